# Round-2 last GPU pass: decision suites, K4 crossover, bench line (+ reference arm).
mkdir -p gpurun_out
tag=${1:-r02x}
timeout 1500 python -m pytest -x -q -m gpu -p no:cacheprovider tests/test_host_cpp.py tests/test_mirror_gpu.py tests/test_lockstep_gpu.py tests/test_reference_suites_gpu.py tests/test_fuzz_gpu.py > gpurun_out/dec_tests_$tag.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/dec_tests_$tag.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; tail -1 gpurun_out/smoke_$tag.log
timeout 600 python scripts/crossover_k4_mirror.py > gpurun_out/crossover_k4_mirror_$tag.json 2> /dev/null
timeout 300 python scripts/decider_probe.py gpurun_out/decider_probe_$tag.json > /dev/null 2>&1
timeout 600 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; tail -c 300 gpurun_out/bench_$tag.json
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref_$tag.json 2>&1; tail -c 200 gpurun_out/bench_ref_$tag.json
