"""K5 node-count crossover: GPU victim selection (host round trip through kvf_victim_select)
vs the UNMODIFIED reference's RadixCache::evict CPU time on the same random tree
(oracle/_ref/ref_trace evict, which times the call with steady_clock), with parity checked.

    python scripts/crossover.py > profiles/r01_k5_crossover.json
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle_ffi import ORACLE_DIR, TreeArrays  # noqa: E402
from paper_2507_07400_b200.engine import Engine, depth_from_parent  # noqa: E402


def main():
    ref = os.path.join(ORACLE_DIR, "_ref", "ref_trace")
    e = Engine(layers=1, kv_heads_total=1, head_dim=4, gpu_slots=16, host_slots=16)
    rows = []
    for nodes in (44, 200, 1000, 1500, 4000, 8000, 30000, 100000, 150000):
        out = subprocess.run([ref, "evict", "seed=7", "cases=2", f"min_nodes={nodes}", f"max_nodes={nodes}",
                              "vocab=200"], capture_output=True, text=True, check=True).stdout
        for line in out.splitlines():
            c = json.loads(line)
            if "error" in c:
                continue
            ta = TreeArrays(c)
            tree = {k: getattr(ta, k) for k in ("parent", "status", "lock", "rank", "time", "seq", "id", "tokens",
                                                "backed")}
            tree["depth"] = depth_from_parent(ta.parent)
            tree["bpt"] = ta.bpt
            best, ok = None, True
            for _ in range(5):
                s0 = e.stats()
                idx, act, imm, pend = e.victims(tree, c["needed"], c["policy"], c["mode"], c["has_floor"], c["floor"],
                                                c["cpu_used"], c["cpu_cap"])
                s1 = e.stats()
                us = s1["decision_call_us"] - s0["decision_call_us"]
                kus = (s1["decision_kernel_ms"] - s0["decision_kernel_ms"]) * 1e3
                best = (us, kus) if best is None or us < best[0] else best
                got = [(int(ta.id[v]), int(ta.tokens[v]) * ta.bpt, 0 if a == 0 else 1) for v, a in zip(idx, act)]
                ok &= got == [tuple(v) for v in c["victims"]]
            rows.append({"nodes": ta.n, "victims": len(c["victims"]), "policy": "WA" if c["policy"] else "LRU",
                         "reference_cpu_us": c["evict_us"], "gpu_call_us": round(best[0], 1),
                         "gpu_kernels_us": round(best[1], 1), "speedup": round(c["evict_us"] / best[0], 2),
                         "parity": ok})
            print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
    e.close()
    print(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()
