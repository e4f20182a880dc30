# compute-sanitizer memcheck + racecheck over the multi-stream driver suites.
# Usage: bash scripts/gpu_sanitize.sh [tag]; writes gpurun_out/sanitize_<tag>.txt
mkdir -p gpurun_out
tag=${1:-r02}
out=gpurun_out/sanitize_$tag.txt
: > $out
export KVF_SANITIZER=1  # tests skip their real-time latency assertions (kernels run 10-100x slower)
# compute-sanitizer serialises kernels: a held resident decider CTA would never let the copy
# kernels of a driver run start.  The driver suites therefore run their decisions as one
# launch per request (the same device code: apply records, K4 / K5 bodies); the mirror suite
# exercises the resident CTA itself (no other kernel runs while it is alive there).
for tool in memcheck racecheck; do
  for f in tests/test_lockstep_gpu.py tests/test_fuzz_gpu.py tests/test_wallclock_gpu.py tests/test_concurrency_gpu.py tests/test_shared_engine_gpu.py tests/test_wallclock_parity_gpu.py tests/test_mirror_gpu.py; do
    [ -f $f ] || continue
    dec=0; [ $f = tests/test_mirror_gpu.py ] && dec=1
    echo "=== $tool: $f (KVF_DECIDER=$dec)" >> $out
    KVF_DECIDER=$dec timeout ${SAN_TMO:-1500} compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
      python -m pytest -x -q -m gpu -p no:cacheprovider $f >> $out.tmp 2>&1
    echo "rc=$?" >> $out
    grep -E "passed|failed|error|ERROR SUMMARY|RACECHECK SUMMARY|Invalid|Hazard" $out.tmp | tail -12 >> $out
    rm -f $out.tmp
  done
done
cat $out
