"""K6 (kvf_decode_attend) measurement: decode attention straight off the slot-run table.

    python scripts/attend_bench.py [--out gpurun_out/attend.json]      # all workloads
    python scripts/attend_bench.py --ncu                                # one C2 layer call (ncu capture)

One step = one decode step of a batch = 32 per-layer K6 calls (the descriptor upload is
cached across the layers of a step).  Algorithmic bytes per call = sum over sequences of
tokens x 2 (K, V) x tpb -- every KV byte of the layer read once; q/out are < 0.1 %.
GB/s is against MEASURED_PEAKS.json hbm_gbs (else the B200_PROFILING.md fallback).
Comparator: the compaction path (K3 gathers every sequence into contiguous staging first),
the copy in-place consumption avoids.  Payload = the engine's hash fill (timing only; the
numerics are pinned by tests/test_attend_gpu.py).
"""
import argparse
import json
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_07400_b200 import _native as N  # noqa: E402
from paper_2507_07400_b200.engine import Engine  # noqa: E402


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        return json.load(open(p))["hbm_gbs"], "measured"
    return 6650.0, "fallback (B200_PROFILING.md)"


def build(e, lens, rng, piece=None):
    seqs = []
    for n in lens:
        if piece is None:
            runs = e.alloc(N.KVF_TIER_DEVICE, n)
        else:
            runs, left = [], n
            while left:
                k = min(left, int(rng.integers(piece[0], piece[1] + 1)))
                runs += e.alloc(N.KVF_TIER_DEVICE, k)
                e.free(N.KVF_TIER_DEVICE, e.alloc(N.KVF_TIER_DEVICE, 1))
                left -= k
        e.fill(N.KVF_TIER_DEVICE, runs, rng.integers(0, 2**63, size=n, dtype=np.uint64))
        seqs.append(runs)
    e.sync()
    return seqs


def step(e, seqs, q, out, group, layers, scale, queued=False):
    seqs = e.attend_runs(seqs)
    if queued:  # hold the compute stream while the calls are enqueued: each job = device time
        e.compute_spin(3_000_000, 1)
    jobs = [e.attend(layer, group, q.data_ptr(), seqs, out.data_ptr(), scale) for layer in range(layers)]
    ms = e.span_ms(jobs[0], jobs[-1])
    per = [e.elapsed_ms(j) for j in jobs]
    for j in jobs:
        e.release(j)
    return ms, per


def step_chained(e, seqs, q, out, group, layers, scale):
    """The decode step's layers as one kvf_decode_attend_layers job (PDL-chained)."""
    j = e.attend_layers(0, group, [q.data_ptr()] * layers, e.attend_runs(seqs), [out.data_ptr()] * layers, scale)
    e.wait(j)
    ms = e.elapsed_ms(j)
    e.release(j)
    return ms


def run(name, kv_local, group, lens, piece=None, steps=5, layers=32):
    rng = np.random.default_rng(1)
    total = sum(lens)
    slack = 2 * len(lens) + (total // 8 if piece else 0) + 4096
    e = Engine(layers=layers, kv_heads_total=8, kv_heads_local=kv_local, head_offset=8 - kv_local,
               gpu_slots=total + slack, host_slots=0)
    seqs = build(e, lens, rng, piece)
    hq = kv_local * group
    q = torch.randn(len(lens), hq, 128, device="cuda").to(torch.bfloat16)
    out = torch.empty_like(q)
    torch.cuda.synchronize()
    scale = 1 / math.sqrt(128)
    for _ in range(2):
        step(e, seqs, q, out, group, layers, scale)
    spans, pers = [], []
    for _ in range(steps):
        ms, per = step(e, seqs, q, out, group, layers, scale)
        spans.append(ms)
        pers += per
    qpers = []
    for _ in range(steps):
        qpers += step(e, seqs, q, out, group, layers, scale, queued=True)[1]
    chained = [step_chained(e, seqs, q, out, group, layers, scale) for _ in range(steps + 2)][2:]
    bytes_layer = total * 2 * e.tpb
    # compaction comparator: K3 gathers every sequence (all layers) into staging, then attend
    st = torch.empty(max(lens) * e.token_bytes, dtype=torch.uint8, device="cuda")
    k3 = []
    for _ in range(2):
        t = 0.0
        for runs in seqs:
            j = e.dev_gather(runs, st.data_ptr())
            e.wait(j)
            t += e.elapsed_ms(j)
            e.release(j)
        k3.append(t)
    del st
    nruns = sum(len(s) for s in seqs)
    e.close()
    peak, src = hbm_peak()
    step_ms = min(spans)
    layer_ms = float(np.median(pers))
    gbs = bytes_layer / (layer_ms * 1e-3) / 1e9
    return {"workload": name, "kv_heads_local": kv_local, "group": group, "batch": len(lens), "tokens": total,
            "runs": nruns, "layers": layers, "bytes_per_layer_call": bytes_layer,
            "step_ms": round(step_ms, 4), "layer_call_ms_median": round(layer_ms, 4),
            "achieved_GBps": round(gbs, 1), "step_GBps": round(bytes_layer * layers / (step_ms * 1e-3) / 1e9, 1),
            "hbm_peak_GBps": peak, "peak_source": src, "frac": round(gbs / peak, 4),
            # the same single-layer calls enqueued behind earlier work (a decoder's steady state)
            "queued_layer_call_us_median": round(float(np.median(qpers)) * 1e3, 2),
            "queued_frac": round(bytes_layer / (float(np.median(qpers)) * 1e-3) / 1e9 / peak, 4),
            "chained_step_ms": round(min(chained), 4),
            "chained_layer_us": round(min(chained) / layers * 1e3, 2),
            "chained_GBps": round(bytes_layer * layers / (min(chained) * 1e-3) / 1e9, 1),
            "chained_frac": round(bytes_layer * layers / (min(chained) * 1e-3) / 1e9 / peak, 4),
            "compaction_k3_ms_per_step": round(min(k3), 3),
            "in_place_saves": f"{min(k3):.2f} ms of K3 copies per step ({2 * bytes_layer * layers / 1e9:.2f} GB moved)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--ncu", action="store_true")
    a = ap.parse_args()
    if a.ncu:  # one warm C2 call for ncu -k regex:kvf_attend -s 2 -c 1
        rng = np.random.default_rng(1)
        e = Engine(layers=32, kv_heads_total=8, gpu_slots=4 * 8320 + 64, host_slots=0)
        seqs = build(e, [8320] * 4, rng)
        q = torch.randn(4, 32, 128, device="cuda").to(torch.bfloat16)
        out = torch.empty_like(q)
        torch.cuda.synchronize()
        for layer in (0, 1, 2, 3):
            j = e.attend(layer, 4, q.data_ptr(), seqs, out.data_ptr(), 0.088)
            e.wait(j)
            print("k6 ms", e.elapsed_ms(j))
            e.release(j)
        e.close()
        return
    res = [
        run("C2 decode: 4 agents x 8320 tokens (8k prefix + suffix), Llama-3-8B, contiguous runs", 8, 4, [8320] * 4),
        run("C2 decode, prefixes fragmented into 16-64-token runs", 8, 4, [8320] * 4, piece=(16, 64)),
        run("C4 decode: 64 workflows x 1792 tokens, Llama-3-8B", 8, 4, [1792] * 64),
        run("C5 decode: Llama-3-70B KV, 1 KV head per GPU (8-way shard), 4 x 8320 tokens", 1, 8, [8320] * 4,
            layers=80),
        run("single long sequence: 1 x 32768 tokens, Llama-3-8B", 8, 4, [32768]),
    ]
    txt = json.dumps(res, indent=1)
    print(txt)
    if a.out:
        with open(a.out, "w") as f:
            f.write(txt)


if __name__ == "__main__":
    main()
