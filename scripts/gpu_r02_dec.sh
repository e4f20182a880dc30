# Decision-path change check: the suites that drive K4/K5 through the mirror, then the probe + bench.
mkdir -p gpurun_out
tag=${1:-r02d}
[ -n "$SKIPTESTS" ] || timeout 1500 python -m pytest -x -q -m gpu -p no:cacheprovider tests/test_host_cpp.py tests/test_lockstep_gpu.py tests/test_fuzz_gpu.py tests/test_reference_suites_gpu.py tests/test_wallclock_parity_gpu.py tests/test_mirror_gpu.py tests/test_stall_gpu.py tests/test_wallclock_gpu.py tests/test_fuzz_wallclock_gpu.py tests/test_shared_engine_gpu.py tests/test_k4_large_gpu.py > gpurun_out/dec_tests_$tag.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/dec_tests_$tag.log
timeout 300 python scripts/decider_probe.py gpurun_out/decider_probe_$tag.json > /dev/null 2>&1; cat gpurun_out/decider_probe_$tag.json | head -30
timeout 120 python scripts/mirror_probe.py gpurun_out/mirror_probe_$tag.json > /dev/null 2>&1; cat gpurun_out/mirror_probe_$tag.json | head -40
timeout 600 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; tail -c 600 gpurun_out/bench_$tag.json
