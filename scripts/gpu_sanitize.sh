# compute-sanitizer memcheck + racecheck over the multi-stream driver suites.
# Usage: bash scripts/gpu_sanitize.sh [tag]; writes gpurun_out/sanitize_<tag>.txt
mkdir -p gpurun_out
tag=${1:-r02}
out=gpurun_out/sanitize_$tag.txt
: > $out
export KVF_SANITIZER=1  # tests skip their real-time latency assertions (kernels run 10-100x slower)
for tool in memcheck racecheck; do
  for f in tests/test_lockstep_gpu.py tests/test_fuzz_gpu.py tests/test_wallclock_gpu.py tests/test_concurrency_gpu.py tests/test_shared_engine_gpu.py tests/test_wallclock_parity_gpu.py tests/test_mirror_gpu.py; do
    [ -f $f ] || continue
    echo "=== $tool: $f" >> $out
    timeout ${SAN_TMO:-1500} compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
      python -m pytest -x -q -m gpu -p no:cacheprovider $f >> $out.tmp 2>&1
    echo "rc=$?" >> $out
    grep -E "passed|failed|error|ERROR SUMMARY|RACECHECK SUMMARY|Invalid|Hazard" $out.tmp | tail -12 >> $out
    rm -f $out.tmp
  done
done
cat $out
