"""K5 node-count crossover over the HBM tree MIRROR (kvf_tree_victims): the tree is loaded once
(as a cache would have built it up), then each call ships no records -- the steady state of
RadixCache::evict.  Against the UNMODIFIED reference's RadixCache::evict CPU time on the same
random tree (oracle/_ref/ref_trace evict), victims checked against the reference's.  Small
trees go to the resident decider (<= 512 slots) or one-shot launches (<= 4096), larger ones to
the hand-written device-wide path (decide_large.cu).  The snapshot path (kvf_victim_select:
pack + upload per call) is timed beside it.

    python scripts/crossover_mirror.py > profiles/r02_k5_crossover_mirror.json
"""
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle_ffi import ORACLE_DIR, TreeArrays  # noqa: E402
from paper_2507_07400_b200.engine import Engine, Tree, decider_hold, depth_from_parent  # noqa: E402

FIELDS = ("parent", "status", "lock", "rank", "time", "seq", "id", "tokens", "backed")


def time_follows_seq(ta):
    o = np.argsort(ta.seq, kind="stable")
    t, s = ta.time[o], ta.seq[o]
    same = s[1:] == s[:-1]
    return bool(np.all(np.diff(t) >= 0) and np.all(t[1:][same] == t[:-1][same]))


def main():
    ref = os.path.join(ORACLE_DIR, "_ref", "ref_trace")
    e = Engine(layers=1, kv_heads_total=1, head_dim=4, gpu_slots=16, host_slots=16)
    rows = []
    sizes = [int(x) for x in sys.argv[1:]] or [44, 200, 500, 1000, 1500, 4000, 4500, 8000, 12000, 30000, 100000, 150000]
    for nodes in sizes:
        out = subprocess.run([ref, "evict", "seed=7", "cases=2", f"min_nodes={nodes}", f"max_nodes={nodes}",
                              "vocab=200"], capture_output=True, text=True, check=True).stdout
        for line in out.splitlines():
            c = json.loads(line)
            if "error" in c:
                continue
            ta = TreeArrays(c)
            arr = {k: getattr(ta, k) for k in FIELDS}
            args = dict(needed=c["needed"], workflow_aware=c["policy"], offload=c["mode"], has_floor=c["has_floor"],
                        floor=c["floor"], cpu_used=c["cpu_used"], cpu_cap=c["cpu_cap"])
            want = [tuple(v) for v in c["victims"]]
            hint = time_follows_seq(ta)
            with Tree(e, ta.bpt, capacity=ta.n) as t:
                t.load_arrays(arr)
                t.hints(hint)
                decider_hold(e, True)
                calls, kern, ok = [], [], True
                for rep in range(8):
                    s0 = e.stats()
                    t0 = time.perf_counter()
                    sl, act, imm, pend = t.victims(**args)
                    host_us = (time.perf_counter() - t0) * 1e6
                    s1 = e.stats()
                    if rep >= 1:  # the first call ships the whole tree
                        calls.append(s1["decision_call_us"] - s0["decision_call_us"])
                        kern.append((s1["decision_kernel_ms"] - s0["decision_kernel_ms"]) * 1e3)
                    got = [(int(ta.id[v]), int(ta.tokens[v]) * ta.bpt, 0 if a == 0 else 1) for v, a in zip(sl, act)]
                    ok &= got == want and (imm, pend) == (c["immediate"], c["pending"])
                decider_hold(e, False)
            tree = dict(arr)
            tree["depth"] = depth_from_parent(ta.parent)
            tree["bpt"] = ta.bpt
            snap = []
            for rep in range(4):
                s0 = e.stats()
                idx, act, _, _ = e.victims(tree, **args)
                snap.append(e.stats()["decision_call_us"] - s0["decision_call_us"])
            call, k = min(calls), min(kern)
            rows.append({"nodes": ta.n, "victims": len(want), "policy": "WA" if c["policy"] else "LRU",
                         "time_follows_seq": hint, "reference_cpu_us": c["evict_us"],
                         "mirror_call_us": round(call, 1), "mirror_kernel_us": round(k, 1),
                         "call_over_kernel": round(call / k, 2) if k > 0 else None,
                         "snapshot_call_us": round(min(snap), 1),
                         "speedup_vs_cpu": round(c["evict_us"] / call, 2), "parity": ok})
            print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
    e.close()
    print(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()
