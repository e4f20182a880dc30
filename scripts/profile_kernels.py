"""Launch each hot-path kernel at BASELINE configs[1] (C2) sizes for ncu capture.

    ncu --set full --clock-control none --import-source on -k regex:kvf_copy_vec -s 2 -c 1 \
        -o gpurun_out/prof_k1 python scripts/profile_kernels.py k1

k1: 8192-token (1 GiB) H2D gather    k2: 128-token (16 MiB) D2H scatter
k3: 1 GiB HBM gather to staging      k5: victim selection on a 1.4k-node golden tree
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from paper_2507_07400_b200 import _native as N  # noqa: E402
from paper_2507_07400_b200.engine import Engine, depth_from_parent  # noqa: E402


def main(which):
    e = Engine(layers=32, kv_heads_total=8, head_dim=128, gpu_slots=24960, host_slots=4 * 8192 + 1024)
    rng = np.random.default_rng(0)
    h = e.alloc(N.KVF_TIER_HOST, 8192)
    d = e.alloc(N.KVF_TIER_DEVICE, 8192)
    e.fill(N.KVF_TIER_HOST, h, rng.integers(0, 2**63, size=8192, dtype=np.uint64))
    e.fill(N.KVF_TIER_DEVICE, d, rng.integers(0, 2**63, size=8192, dtype=np.uint64))
    e.sync()
    for _ in range(3):
        if which == "k1":
            j = e.h2d(h, d)
        elif which == "k2":
            j = e.d2h(d[:1] if False else [(d[0][0], 128)], [(h[0][0], 128)])
        elif which == "k3":
            import torch
            st = torch.empty(8192 * e.token_bytes, dtype=torch.uint8, device="cuda")
            j = e.dev_gather(d, st.data_ptr())
        else:
            j = None
        if j is not None:
            e.wait(j)
            print(which, f"{e.elapsed_ms(j):.3f} ms")
            e.release(j)
    if which in ("k5", "k5small"):
        from oracle_ffi import TreeArrays, load_jsonl
        if which == "k5":
            c = sorted(load_jsonl("evict_medium.jsonl"), key=lambda c: -len(c["parent"]))[0]
        else:  # a BASELINE-sized tree (~44 nodes, like C1/C2)
            c = min(load_jsonl("evict_small.jsonl"), key=lambda c: abs(len(c["parent"]) - 44))
        ta = TreeArrays(c)
        tree = {k: getattr(ta, k) for k in ("parent", "status", "lock", "rank", "time", "seq", "id", "tokens",
                                            "backed")}
        tree["depth"] = depth_from_parent(ta.parent)
        tree["bpt"] = ta.bpt
        for _ in range(6):
            e.victims(tree, c["needed"], c["policy"], c["mode"], c["has_floor"], c["floor"], c["cpu_used"],
                      c["cpu_cap"])
        print("k5 nodes", ta.n)
    if which in ("k5mirror", "k5big", "k5mirrorsmall"):
        # K5 over the HBM mirror: a 1.4k-node golden tree (one-shot kvf_decide_once; run with
        # KVF_DECIDER=0 so no resident CTA is in the capture) or a 30k-node tree on the
        # hand-written device-wide path (big_* kernels)
        import subprocess
        from oracle_ffi import ORACLE_DIR, TreeArrays, load_jsonl
        from paper_2507_07400_b200.engine import Tree
        if which == "k5mirror":
            c = sorted(load_jsonl("evict_medium.jsonl"), key=lambda c: -len(c["parent"]))[0]
        elif which == "k5mirrorsmall":  # a BASELINE-sized tree (~44 nodes, like C1/C2)
            c = min((x for x in load_jsonl("evict_small.jsonl") if "error" not in x),
                    key=lambda c: abs(len(c["parent"]) - 44))
        else:
            import json
            out = subprocess.run([os.path.join(ORACLE_DIR, "_ref", "ref_trace"), "evict", "seed=7", "cases=1",
                                  "min_nodes=30000", "max_nodes=30000", "vocab=200"], capture_output=True, text=True,
                                 check=True).stdout
            c = json.loads(out.splitlines()[0])
        ta = TreeArrays(c)
        arr = {k: getattr(ta, k) for k in ("parent", "status", "lock", "rank", "time", "seq", "id", "tokens", "backed")}
        with Tree(e, ta.bpt, capacity=ta.n) as t:
            t.load_arrays(arr)
            t.hints(True)
            for _ in range(6):
                t.victims(c["needed"], c["policy"], c["mode"], c["has_floor"], c["floor"], c["cpu_used"], c["cpu_cap"])
        print(which, "nodes", ta.n)
    e.close()


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "k1")
