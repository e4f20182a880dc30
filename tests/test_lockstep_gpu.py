"""Decision parity of the full hot path: the C++ lockstep driver (kvf::Simulator) on a GPU
engine vs the UNMODIFIED reference Simulator's golden traces (tests/golden/sim_*.jsonl).

Every transfer here is a real K1/K2 job and every priority/victim decision a K4/K5 call;
the test requires, record for record:
  * the same status transitions (node id, from, to, event index) -- the eviction-victim
    and prefetched-node sequences,
  * the same transfer jobs (id, direction, purpose, node, bytes, virtual times, target),
  * the same per-request traces and run result, and the same final tree dump,
and then checks the bytes: every H2D-loaded node hashes equal to its host copy at the
fence, and every resident/backed node equals its expected payload at the end.
"""
import glob
import os

import pytest

from golden_sim import assert_same_trace, config_from_golden
from oracle_ffi import GOLDEN, load_jsonl

pytestmark = pytest.mark.gpu

S = pytest.importorskip("paper_2507_07400_b200.sim")

SMALL = sorted(os.path.basename(p) for p in glob.glob(os.path.join(GOLDEN, "sim_m_*.jsonl")))
BASELINE = ["sim_c1.jsonl", "sim_c2.jsonl"] + [f"sim_c5_g{g}.jsonl" for g in (1, 2, 4, 8)]


def run_against(fixture, **extra):
    golden = load_jsonl(fixture)
    kw = config_from_golden(golden[0])
    kw.update(extra)
    with S.Sim(verify_loads=1, **kw) as sim:
        sim.run()
        res = sim.result()
        trace = sim.trace()
        checked, bad = sim.verify_resident()
    assert_same_trace(golden[1:], trace)
    assert res["verify_failures"] == 0 and res["verified_loads"] == res["prefetch_jobs"] + res["reactive_jobs"]
    assert bad == 0, f"{bad}/{checked} nodes hold the wrong bytes"
    return res, checked


@pytest.mark.parametrize("fixture", SMALL)
def test_small_configs_match_reference(fixture):
    run_against(fixture, audit=1)


@pytest.mark.parametrize("fixture", BASELINE)
def test_baseline_configs_match_reference(fixture):
    extra = {}
    if fixture.startswith("sim_c5_g"):
        g = int(fixture[len("sim_c5_g"):-len(".jsonl")])
        # Llama-3-70B KV shard: 80 layers, 8/G of the 8 KV heads; take the LAST shard so
        # head_offset != 0 is exercised (decisions are shard-independent).
        extra = dict(layers=80, kv_heads_total=8, kv_heads_local=8 // g, head_offset=8 - 8 // g, head_dim=128)
    res, checked = run_against(fixture, **extra)
    assert checked > 0
    assert res["prefetch_jobs"] == 36 and res["reactive_jobs"] == 3 and res["offload_jobs"] == 43
