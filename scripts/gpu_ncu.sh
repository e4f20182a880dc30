# ncu evidence only (launch list + per-kernel full captures): bash scripts/gpu_ncu.sh TAG
tag=${1:-r01}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_$tag.csv python bench.py --steps 3 --warmup 3 > gpurun_out/bench_under_ncu_$tag.log 2>&1
for k in k1 k2 k3 k5; do
  pat=kvf_copy_vec; [ $k = k5 ] && pat=kvf_victim
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$pat -s 2 -c 1 -o gpurun_out/prof_${k}_$tag python scripts/profile_kernels.py $k > gpurun_out/ncu_${k}_$tag.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kvf_attend_kernel -s 2 -c 1 -o gpurun_out/prof_k6_$tag python scripts/attend_bench.py --ncu > gpurun_out/ncu_k6_$tag.log 2>&1
ls gpurun_out/*_$tag*
