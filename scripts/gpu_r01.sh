set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 600 python bench.py > gpurun_out/bench_r01.json 2> gpurun_out/bench_r01.err; tail -3 gpurun_out/bench_r01.err; cat gpurun_out/bench_r01.json
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref_r01.json 2>&1; cat gpurun_out/bench_ref_r01.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 3 --warmup 3 > gpurun_out/bench_under_ncu.log 2>&1; tail -2 gpurun_out/bench_under_ncu.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kvf_copy_vec -s 2 -c 1 -o gpurun_out/prof_k1 python scripts/profile_kernels.py k1 > gpurun_out/ncu_k1.log 2>&1; tail -3 gpurun_out/ncu_k1.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kvf_copy_vec -s 2 -c 1 -o gpurun_out/prof_k3 python scripts/profile_kernels.py k3 > gpurun_out/ncu_k3.log 2>&1; tail -3 gpurun_out/ncu_k3.log
timeout 300 ncu --set full --clock-control none --import-source on -k regex:kvf_victim -s 2 -c 1 -o gpurun_out/prof_k5 python scripts/profile_kernels.py k5 > gpurun_out/ncu_k5.log 2>&1; tail -3 gpurun_out/ncu_k5.log
ls -la gpurun_out
