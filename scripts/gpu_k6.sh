tag=${1:-k6a}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_attend_gpu.py -x -q > gpurun_out/attend_tests_$tag.log 2>&1; tail -15 gpurun_out/attend_tests_$tag.log
timeout 600 python scripts/attend_bench.py --out gpurun_out/attend_$tag.json > gpurun_out/attend_bench_$tag.log 2>&1; tail -30 gpurun_out/attend_bench_$tag.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kvf_attend_kernel -s 2 -c 1 -o gpurun_out/prof_k6_$tag python scripts/attend_bench.py --ncu > gpurun_out/ncu_k6_$tag.log 2>&1; tail -3 gpurun_out/ncu_k6_$tag.log
timeout 900 compute-sanitizer --tool memcheck python -m pytest tests/test_attend_gpu.py -x -q -k "shared_prefix or errors" > gpurun_out/attend_memcheck_$tag.log 2>&1; tail -5 gpurun_out/attend_memcheck_$tag.log
