#!/usr/bin/env bash
# Regenerates every golden fixture in tests/golden/ from the UNMODIFIED reference.
# Needs /root/reference (this container only); builds oracle/_ref first.
#   bash tests/golden/make_golden.sh
# The fixtures are committed; the GPU box never runs this script.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
ROOT="$(cd "$HERE/../.." && pwd)"
make -C "$ROOT/oracle" ref >/dev/null
T="$ROOT/oracle/_ref/ref_trace"
G="$HERE"

# ---- K5 / K4 / step-graph vectors (component level) ---------------------------
"$T" evict seed=1 cases=300 max_nodes=60 > "$G/evict_small.jsonl"
"$T" evict seed=2 cases=24 min_nodes=200 max_nodes=1500 vocab=40 > "$G/evict_medium.jsonl"
"$T" evict_bounded seed=3 cases=80 > "$G/evict_bounded.jsonl"
"$T" prio seed=4 cases=200 > "$G/prio.jsonl"
"$T" steps seed=5 cases=200 > "$G/steps.jsonl"

# ---- BASELINE.json configs, h100-qwen32b timing, Llama-3 geometry -----
# C1 PEER 4-agent cyclic, 2k, 3.0 footprints
"$T" sim fixed=2048 gpu_cap=855638016 > "$G/sim_c1.jsonl"
# C2 PEER 8k, eviction-heavy (3.0 footprints)
"$T" sim fixed=8192 gpu_cap=3271557120 > "$G/sim_c2.jsonl"
# C4 64 workflows, intra-client shared prefixes, 16 GiB budget
"$T" sim fixed=1024 shared_prefix=512 dyn=256 out=256 workflows=64 iterations=4 gpu_cap=17179869184 dump=0 > "$G/sim_c4.jsonl"
# C4 as one of 8 KV-head shards (16 KiB/token, 2 GiB budget); every shard runs this stream
# (it differs from G=1: transfers are 8x shorter while compute is not, so events reorder)
"$T" sim fixed=1024 shared_prefix=512 dyn=256 out=256 workflows=64 iterations=4 gpu_cap=2147483648 bpt=16384 dump=0 > "$G/sim_c4_g8.jsonl"
# C5 Llama-3-70B KV head-sharded: per-shard bytes/token and budget divide by G
for G_ in 1 2 4 8; do
  "$T" sim fixed=2048 bpt=$((327680 / G_)) gpu_cap=$((2139095040 / G_)) > "$G/sim_c5_g${G_}.jsonl"
done

# ---- small configs mirroring the reference's scheduler suite (micro cost, 16 B/token) --
M="profile=micro bpt=16 vocab=50000"
"$T" sim $M topology=SEQUENTIAL agents=2 iterations=1 warmup=0 fixed=32 dyn=8 out=3 gpu_cap=160000 policy=LRU_GPU_ONLY > "$G/sim_m_pipeline.jsonl"
for P in LRU_GPU_ONLY LRU_REACTIVE_HICACHE KVFLOW; do
  "$T" sim $M topology=SEQUENTIAL agents=2 iterations=2 warmup=1 fixed=256 dyn=16 out=0 gpu_cap=7200 policy=$P > "$G/sim_m_gate_${P}.jsonl"
  "$T" sim $M topology=SEQUENTIAL agents=4 iterations=2 warmup=1 fixed=512 dyn=32 out=16 workflows=2 gpu_cap=20800 seed=7 policy=$P > "$G/sim_m_status_${P}.jsonl"
done
"$T" sim $M topology=SEQUENTIAL agents=3 iterations=4 warmup=1 fixed=256 dyn=16 out=8 gpu_cap=11200 seed=3 max_prefetch=1 > "$G/sim_m_prefetch.jsonl"
"$T" sim $M topology=SEQUENTIAL agents=1 iterations=4 warmup=1 fixed=32 dyn=8 out=0 gpu_cap=160000 boundary=heuristic > "$G/sim_m_heuristic.jsonl"
"$T" sim $M topology=CYCLIC agents=3 iterations=4 warmup=1 fixed=64 dyn=8 out=0 gpu_cap=2688 policy=LRU_GPU_ONLY eviction=WA > "$G/sim_m_wa_gpuonly.jsonl"
"$T" sim $M topology=BRANCH_MAX agents=4 iterations=3 warmup=1 fixed=128 dyn=16 out=8 workflows=2 gpu_cap=9000 seed=11 audit=1 > "$G/sim_m_branch_max.jsonl"
"$T" sim $M topology=BRANCH_MIN agents=4 iterations=3 warmup=1 fixed=128 dyn=16 out=8 workflows=2 gpu_cap=9000 seed=12 audit=1 > "$G/sim_m_branch_min.jsonl"
"$T" sim $M topology=PEER_STYLE agents=4 iterations=2 warmup=1 workflows=3 gpu_cap=40000 seed=13 audit=1 > "$G/sim_m_peer_style.jsonl"
"$T" sim $M topology=CYCLIC agents=4 iterations=3 warmup=1 fixed=96 dyn=8 out=8 workflows=3 shared_prefix=32 gpu_cap=9000 seed=14 audit=1 > "$G/sim_m_shared.jsonl"
# C3: 16-agent branch + barrier graph, mixed 1k-8k prompts (component-level harness,
# tests/cpp/c3_harness.hpp); one Llama-3-8B KV head (16 KiB/token), 24k-token budget
"$ROOT/oracle/_ref/ref_c3" 3 4 16384 393216000 > "$G/c3_seed3.jsonl"
"$ROOT/oracle/_ref/ref_c3" 11 6 16384 262144000 > "$G/c3_seed11.jsonl"
for c in "5 4 327680000" "7 5 294912000" "13 4 360448000" "17 6 425984000" "19 3 229376000" "23 5 491520000"; do
  set -- $c
  "$ROOT/oracle/_ref/ref_c3" "$1" "$2" 16384 "$3" > "$G/c3_seed$1.jsonl"
done
echo "golden fixtures regenerated in $G"
