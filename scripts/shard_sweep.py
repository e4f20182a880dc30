"""Per-GPU K1/K2 throughput at each KV-head shard size, measured on one B200.

    python scripts/shard_sweep.py > gpurun_out/shard_sweep.json

With G GPUs every rank moves exactly 1/G of each node over its own PCIe link (no collective),
so the per-GPU rate at the shard's transfer size is what each rank of the scaling run sees
when links are independent; the aggregate is G x that (an upper bound: links behind a shared
PCIe switch or one host memory controller can cap it -- the driver's own N-GPU run decides).
Shapes: C2 (Llama-3-8B, 8192-token node, 128-token suffix) and C5 (Llama-3-70B, 2176-token
node = 2k fixed prompt + suffix + output), shards G = 1, 2, 4, 8 of the 8 KV heads.
"""
import json
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_07400_b200 import _native as N  # noqa: E402
from paper_2507_07400_b200.engine import Engine  # noqa: E402


def measure(layers, G, node_tokens, suffix, steps=8):
    heads = 8 // G
    e = Engine(layers=layers, kv_heads_total=8, kv_heads_local=heads, head_offset=8 - heads,
               gpu_slots=2 * node_tokens + 2 * suffix + 64, host_slots=4 * node_tokens + 16 * suffix + 64)
    rng = np.random.default_rng(G)
    hosts = [e.alloc(N.KVF_TIER_HOST, node_tokens) for _ in range(4)]
    for h in hosts:
        e.fill(N.KVF_TIER_HOST, h, rng.integers(0, 2**63, size=node_tokens, dtype=np.uint64))
    devs = [e.alloc(N.KVF_TIER_DEVICE, node_tokens) for _ in range(2)]
    sdev = [e.alloc(N.KVF_TIER_DEVICE, suffix) for _ in range(2)]
    shost = [e.alloc(N.KVF_TIER_HOST, suffix) for _ in range(16)]
    for r in sdev:
        e.fill(N.KVF_TIER_DEVICE, r, rng.integers(0, 2**63, size=suffix, dtype=np.uint64))
    e.sync()
    k1, k2, span = [], [], []
    for s in range(steps + 3):
        j1 = e.h2d(hosts[s % 4], devs[s % 2])
        j2 = e.d2h(sdev[s % 2], shost[s % 16])
        t1, t2 = e.elapsed_ms(j1), e.elapsed_ms(j2)
        if s >= 3:
            k1.append(t1)
            k2.append(t2)
        e.release(j1)
        e.release(j2)
    ok = e.checksum(N.KVF_TIER_DEVICE, devs[(steps + 2) % 2]) == e.checksum(N.KVF_TIER_HOST, hosts[(steps + 2) % 4])
    nb, sb = node_tokens * e.token_bytes, suffix * e.token_bytes
    e.close()
    return {"G": G, "kv_heads_per_gpu": heads, "node_bytes_per_gpu": nb, "k1_ms": round(statistics.median(k1), 3),
            "k1_gbs_per_gpu": round(nb / (statistics.median(k1) * 1e-3) / 1e9, 2),
            "k2_suffix_bytes_per_gpu": sb, "k2_gbs_per_gpu": round(sb / (statistics.median(k2) * 1e-3) / 1e9, 2),
            "aggregate_k1_gbs_if_links_independent": round(G * nb / (statistics.median(k1) * 1e-3) / 1e9, 1),
            "bytes_equal": bool(ok)}


def main():
    out = {"note": "one B200; per-GPU rate at each shard's transfer size (see module docstring)",
           "C2_llama3_8b": [measure(32, G, 8192, 128) for G in (1, 2, 4, 8)],
           "C5_llama3_70b": [measure(80, G, 2176, 128) for G in (1, 2, 4, 8)]}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
