# Final round-2 GPU pass: smoke, -m gpu suite, bench (+ reference arm), probes, ncu evidence.
mkdir -p gpurun_out
tag=${1:-r02z}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; tail -2 gpurun_out/smoke_$tag.log
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/gpu_tests_$tag.log 2>&1; tail -4 gpurun_out/gpu_tests_$tag.log
timeout 600 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; tail -c 400 gpurun_out/bench_$tag.json
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref_$tag.json 2>&1; tail -c 300 gpurun_out/bench_ref_$tag.json
timeout 200 python scripts/decider_probe.py gpurun_out/decider_probe_$tag.json > /dev/null 2>&1
timeout 120 python scripts/mirror_probe.py gpurun_out/mirror_probe_$tag.json > /dev/null 2>&1
timeout 900 python scripts/crossover_mirror.py > gpurun_out/crossover_mirror_$tag.json 2> /dev/null
timeout 600 python scripts/crossover_k4_mirror.py > gpurun_out/crossover_k4_mirror_$tag.json 2> /dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_$tag.csv python bench.py --steps 3 --warmup 3 > gpurun_out/bench_under_ncu_$tag.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kvf_copy_vec -s 2 -c 1 -o gpurun_out/prof_k1_$tag python scripts/profile_kernels.py k1 > gpurun_out/ncu_k1_$tag.log 2>&1
KVF_DECIDER=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:kvf_decide_once -s 4 -c 1 -o gpurun_out/prof_k5m_$tag python scripts/profile_kernels.py k5mirror > gpurun_out/ncu_k5m_$tag.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:big_ -s 40 -c 12 -o gpurun_out/prof_k5big_$tag python scripts/profile_kernels.py k5big > gpurun_out/ncu_k5big_$tag.log 2>&1
ls gpurun_out/*$tag*
