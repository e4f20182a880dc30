# mirror / resident decider bring-up: the decision suites, then the bench
mkdir -p gpurun_out
tag=${1:-r02b}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; tail -2 gpurun_out/smoke_$tag.log
timeout 900 python -m pytest -q -m gpu -x tests/test_mirror_gpu.py -s > gpurun_out/mirror_$tag.log 2>&1; tail -15 gpurun_out/mirror_$tag.log
timeout 1500 python -m pytest -q -m gpu tests/test_lockstep_gpu.py tests/test_reference_suites_gpu.py tests/test_engine_gpu.py tests/test_fuzz_gpu.py tests/test_k5_large_gpu.py tests/test_host_cpp.py > gpurun_out/dec_$tag.log 2>&1; tail -15 gpurun_out/dec_$tag.log
timeout 600 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; tail -3 gpurun_out/bench_$tag.err; tail -c 3000 gpurun_out/bench_$tag.json
