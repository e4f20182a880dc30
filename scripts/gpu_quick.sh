# One GPU call: the suites touched by a change (pass test files / -k as arguments).
mkdir -p gpurun_out
tag=${TAG:-q}
timeout ${TMO:-1500} python -m pytest -x -q -m gpu "$@" > gpurun_out/pytest_$tag.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_$tag.log
