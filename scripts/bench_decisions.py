"""K4/K5 decision latency on the GPU vs tree size, idle and under a concurrent 1 GiB K1.

    python scripts/bench_decisions.py > gpurun_out/decisions.json

Per golden evict/prio case: host round-trip us (pack, H2D, kernel, D2H, sync) and kernel
us (CUDA events on the decision stream), plus the CPU restatement (oracle kvfo_evict,
single thread) on the same tree for scale.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle_ffi import TreeArrays, load_jsonl, oracle_evict  # noqa: E402
from paper_2507_07400_b200 import _native as N  # noqa: E402
from paper_2507_07400_b200.engine import Engine, depth_from_parent  # noqa: E402


def tree_of(c):
    ta = TreeArrays(c)
    t = {k: getattr(ta, k) for k in ("parent", "status", "lock", "rank", "time", "seq", "id", "tokens", "backed")}
    t["depth"] = depth_from_parent(ta.parent)
    t["bpt"] = ta.bpt
    return t


def main():
    e = Engine(layers=32, kv_heads_total=8, head_dim=128, gpu_slots=8192 + 256, host_slots=8192 + 256)
    h = e.alloc(N.KVF_TIER_HOST, 8192)
    d = e.alloc(N.KVF_TIER_DEVICE, 8192)
    cases = sorted(load_jsonl("evict_small.jsonl") + load_jsonl("evict_medium.jsonl"), key=lambda c: len(c["parent"]))
    picks = [cases[int(q * (len(cases) - 1))] for q in (0.0, 0.1, 0.5, 0.8, 0.9, 0.95, 1.0)]
    out = []
    reps = 30
    for c in picks:
        t = tree_of(c)
        row = {"nodes": len(c["parent"])}
        for load in (False, True):
            job = e.h2d(h, d) if load else None
            s0 = e.stats()
            w0 = time.perf_counter()
            for _ in range(reps):
                e.victims(t, c["needed"], c["policy"], c["mode"], c["has_floor"], c["floor"], c["cpu_used"], c["cpu_cap"])
            wall = (time.perf_counter() - w0) / reps * 1e6
            s1 = e.stats()
            if job:
                e.wait(job)
                e.release(job)
            key = "busy_link" if load else "idle"
            row[f"k5_kernel_us_{key}"] = round((s1["decision_kernel_ms"] - s0["decision_kernel_ms"]) / reps * 1e3, 2)
            row[f"k5_call_us_{key}"] = round((s1["decision_call_us"] - s0["decision_call_us"]) / reps, 2)
            row[f"k5_python_us_{key}"] = round(wall, 2)
            row[f"k5_phase_us_{key}"] = [round((b - a) / reps / 1e3, 2) for a, b in zip(s0["k5_phase_ns"], s1["k5_phase_ns"])]
            row[f"k5_phase_kcycles_{key}"] = [round((b - a) / reps / 1e3, 2)
                                              for a, b in zip(s0["k5_phase_cycles"], s1["k5_phase_cycles"])]
        w0 = time.perf_counter()
        for _ in range(reps):
            oracle_evict(c)
        row["cpu_restatement_us_incl_python"] = round((time.perf_counter() - w0) / reps * 1e6, 2)
        out.append(row)
    prio = sorted(load_jsonl("prio.jsonl"), key=lambda c: len(c["parent"]))
    hb = e.alloc(N.KVF_TIER_HOST, 128)
    db = e.alloc(N.KVF_TIER_DEVICE, 128)
    for c in (prio[0], prio[len(prio) // 2], prio[-1]):
        b = c["boundaries"]
        row = {"k4_nodes": len(c["parent"]), "boundaries": len(b)}
        for load in ("idle", "busy_h2d", "busy_both"):
            jobs = [] if load == "idle" else [e.h2d(h, d)] + ([e.d2h(db, hb)] if load == "busy_both" else [])
            s0 = e.stats()
            for _ in range(reps):
                e.priority(c["parent"], [x[0] for x in b], [int(x[1]) for x in b])
            s1 = e.stats()
            for j in jobs:
                e.wait(j)
                e.release(j)
            row[f"k4_kernel_us_{load}"] = round((s1["decision_kernel_ms"] - s0["decision_kernel_ms"]) / reps * 1e3, 2)
            row[f"k4_call_us_{load}"] = round((s1["decision_call_us"] - s0["decision_call_us"]) / reps, 2)
        out.append(row)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
