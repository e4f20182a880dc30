"""K5 above the single-CTA limit (device-wide path, decide_large.cu): victims equal the
UNMODIFIED reference's RadixCache::evict on large random trees built through its own API
(oracle/_ref/ref_trace evict, run live -- the reference is the checker), and the node-count
crossover against the reference's CPU time for the same call."""
import json
import os
import subprocess

import pytest

from oracle_ffi import ORACLE_DIR, TreeArrays

pytestmark = pytest.mark.gpu

REF = os.path.join(ORACLE_DIR, "_ref", "ref_trace")


def ref_cases(seed, nodes, cases=1, vocab=200):
    if not os.path.exists(REF):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    out = subprocess.run([REF, "evict", f"seed={seed}", f"cases={cases}", f"min_nodes={nodes}", f"max_nodes={nodes}",
                          f"vocab={vocab}"], capture_output=True, text=True, check=True, timeout=600).stdout
    return [json.loads(l) for l in out.splitlines() if l.strip()]


def gpu_victims(eng, c):
    from paper_2507_07400_b200.engine import depth_from_parent
    ta = TreeArrays(c)
    tree = {k: getattr(ta, k) for k in ("parent", "status", "lock", "rank", "time", "seq", "id", "tokens", "backed")}
    tree["depth"] = depth_from_parent(ta.parent)
    tree["bpt"] = ta.bpt
    s0 = eng.stats()
    idx, act, imm, pend = eng.victims(tree, c["needed"], c["policy"], c["mode"], c["has_floor"], c["floor"],
                                      c["cpu_used"], c["cpu_cap"])
    s1 = eng.stats()
    got = [(int(ta.id[v]), int(ta.tokens[v]) * ta.bpt, 0 if a == 0 else 1) for v, a in zip(idx, act)]
    return got, (imm, pend), s1["decision_call_us"] - s0["decision_call_us"]


@pytest.fixture(scope="module")
def eng():
    from paper_2507_07400_b200.engine import Engine
    e = Engine(layers=1, kv_heads_total=1, head_dim=4, gpu_slots=16, host_slots=16)
    yield e
    e.close()


@pytest.mark.parametrize("nodes,seed", [(4500, 1), (12000, 2), (30000, 3)])
def test_large_tree_victims_match_reference(eng, nodes, seed):
    for c in ref_cases(seed, nodes, cases=3):
        if "error" in c:
            continue
        got, totals, _ = gpu_victims(eng, c)
        assert got == [tuple(v) for v in c["victims"]], (nodes, c["case"])
        assert totals == (c["immediate"], c["pending"])
