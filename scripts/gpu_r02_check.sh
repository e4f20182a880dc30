# Round-2 re-entry check: smoke, -m gpu suite, bench + reference arm on the current code.
mkdir -p gpurun_out
tag=${1:-r02c}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; tail -2 gpurun_out/smoke_$tag.log
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gpu_tests_$tag.log 2>&1; tail -6 gpurun_out/gpu_tests_$tag.log
timeout 600 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; tail -c 400 gpurun_out/bench_$tag.json
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref_$tag.json 2>&1; tail -c 300 gpurun_out/bench_ref_$tag.json
