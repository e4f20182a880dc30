"""K4 node-count sweep over the HBM tree MIRROR: kvf_tree_priorities + kvf_tree_rank_changes
(the tree loaded once; a call ships no records -- the steady state of set_agent_priorities)
vs the UNMODIFIED reference's RadixCache::set_agent_priorities CPU time on the same random
tree and boundaries (oracle/_ref/ref_trace prio time=1), ranks checked equal.

    python scripts/crossover_k4_mirror.py > profiles/r02_k4_crossover_mirror.json
"""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle_ffi import ORACLE_DIR  # noqa: E402
from paper_2507_07400_b200.engine import Engine, Tree, decider_hold  # noqa: E402

SUFFIX = 4611686018427387903


def main():
    ref = os.path.join(ORACLE_DIR, "_ref", "ref_trace")
    e = Engine(layers=1, kv_heads_total=1, head_dim=4, gpu_slots=16, host_slots=16)
    rows = []
    for nodes, agents in ((44, 4), (200, 16), (1000, 64), (1500, 256), (4000, 256), (8000, 256), (30000, 256),
                          (100000, 256), (150000, 256)):
        out = subprocess.run([ref, "prio", "seed=5", "cases=2", f"min_nodes={nodes}", f"max_nodes={nodes}",
                              f"agents={agents}", "time=1"], capture_output=True, text=True, check=True).stdout
        for line in out.splitlines():
            c = json.loads(line)
            b = c["boundaries"]
            parent = c["parent"]
            n = len(parent)
            want = [int(x) for x in c["rank"]]
            with Tree(e, 1, capacity=n) as t:
                t.update({"slot": i, "parent": int(parent[i]), "rank": SUFFIX, "tokens": 1, "id": i, "seq": i,
                          "lock": 1 if i == 0 else 0} for i in range(n))
                decider_hold(e, True)
                calls, ok = [], True
                ranks = [SUFFIX] * n
                for rep in range(6):
                    t0 = time.perf_counter()
                    s0 = e.stats()
                    t.priorities([x[0] for x in b], [int(x[1]) for x in b])
                    ch = t.rank_changes()
                    s1 = e.stats()
                    if rep >= 1:
                        calls.append((time.perf_counter() - t0) * 1e6)
                    for k, v in ch.items():
                        ranks[k] = v
                    ok &= ranks[1:] == want[1:]
                decider_hold(e, False)
            rows.append({"nodes": n, "boundaries": len(b), "reference_cpu_us": c["prio_us"],
                         "mirror_call_us_incl_python": round(min(calls), 1), "parity": ok})
            print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
    e.close()
    print(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()
