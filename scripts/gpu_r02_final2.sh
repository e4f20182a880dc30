# Round-2 final GPU pass after the decision-path rework: smoke, -m gpu suite, bench (+ reference
# arm), probes, ncu evidence, crossovers, compute-sanitizer over the mirror + lockstep suites.
mkdir -p gpurun_out
tag=${1:-r02y}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; tail -2 gpurun_out/smoke_$tag.log
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gpu_tests_$tag.log 2>&1; tail -4 gpurun_out/gpu_tests_$tag.log
timeout 600 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; tail -c 400 gpurun_out/bench_$tag.json
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref_$tag.json 2>&1; tail -c 300 gpurun_out/bench_ref_$tag.json
timeout 300 python scripts/decider_probe.py gpurun_out/decider_probe_$tag.json > /dev/null 2>&1
timeout 120 python scripts/mirror_probe.py gpurun_out/mirror_probe_$tag.json > /dev/null 2>&1
timeout 600 python scripts/attend_bench.py --out gpurun_out/attend_$tag.json > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_$tag.csv python bench.py --steps 3 --warmup 3 > gpurun_out/bench_under_ncu_$tag.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kvf_copy_vec -s 2 -c 1 -o gpurun_out/prof_k1_$tag python scripts/profile_kernels.py k1 > gpurun_out/ncu_k1_$tag.log 2>&1
KVF_DECIDER=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:kvf_decide_once -s 4 -c 1 -o gpurun_out/prof_k5m_$tag python scripts/profile_kernels.py k5mirror > gpurun_out/ncu_k5m_$tag.log 2>&1
timeout 900 python scripts/crossover_mirror.py > gpurun_out/crossover_mirror_$tag.json 2> /dev/null
timeout 600 python scripts/crossover_k4_mirror.py > gpurun_out/crossover_k4_mirror_$tag.json 2> /dev/null
export KVF_SANITIZER=1
: > gpurun_out/sanitize_$tag.txt
for tool in memcheck racecheck; do
  for f in tests/test_mirror_gpu.py tests/test_lockstep_gpu.py tests/test_host_cpp.py; do
    dec=0; [ $f = tests/test_mirror_gpu.py ] && dec=1
    echo "=== $tool: $f (KVF_DECIDER=$dec)" >> gpurun_out/sanitize_$tag.txt
    KVF_DECIDER=$dec timeout 1200 compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
      python -m pytest -x -q -m gpu -p no:cacheprovider $f > gpurun_out/san.tmp 2>&1
    echo "rc=$?" >> gpurun_out/sanitize_$tag.txt
    grep -E "passed|failed|error|ERROR SUMMARY|RACECHECK SUMMARY|Invalid|Hazard" gpurun_out/san.tmp | tail -12 >> gpurun_out/sanitize_$tag.txt
  done
done
rm -f gpurun_out/san.tmp
cat gpurun_out/sanitize_$tag.txt
ls gpurun_out/*$tag*
