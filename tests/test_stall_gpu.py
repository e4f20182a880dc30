"""Prefix-cache-miss stalls with real B200 transfer times in the loop (TransferTiming::Measured):
every transfer runs on the GPU and its measured device time -- not the reference's cost
model -- sets when the workflow sees it land.  Target: zero stall on every
step the reference served by prefetch; the reference's own reactive (stalling) steps are
reported separately.  Also: identical decisions across KV-head shards is exercised by the
C5 parity tests; here the 4-agent PEER workflow runs at G = 1, 2, 4, 8 shard geometry."""
import pytest

from oracle_ffi import load_jsonl

pytestmark = pytest.mark.gpu
S = pytest.importorskip("paper_2507_07400_b200.sim")


def reference_stalls(fixture):
    reqs = [r for r in load_jsonl(fixture) if r["t"] == "req" and r["measured"]]
    return sum(r["stall"] for r in reqs), sum(1 for r in reqs if r["stall"] > 1e-12)


def run_measured(**kw):
    with S.Sim(timing=1, **kw) as s:
        s.run()
        return s.result(), [r for r in s.trace() if r["t"] == "req"]


@pytest.mark.parametrize("fixed,cap,fixture", [(2048, 855638016, "sim_c1.jsonl"), (8192, 3271557120, "sim_c2.jsonl")])
def test_peer_prefetch_steps_never_stall(fixed, cap, fixture):
    res, reqs = run_measured(fixed=fixed, gpu_cap=cap)
    measured = [r for r in reqs if r["measured"]]
    assert len(measured) == 40 and res["prefetch_jobs"] > 0
    # every request that did not have to load its own prefix reactively starts with no stall
    for r in measured:
        if r["loaded_bytes"] == 0:
            assert r["stall"] == 0.0, r
    ref_total, ref_stalled = reference_stalls(fixture)
    assert res["stall_total_s"] <= ref_total + 1e-9
    assert res["stalled_requests"] <= ref_stalled


@pytest.mark.parametrize("g", [2, 4, 8])
def test_sharded_peer_prefetch_steps_never_stall(g):
    res, reqs = run_measured(fixed=2048, gpu_cap=855638016 // g, bytes_per_token=131072 // g, layers=32,
                             kv_heads_total=8, kv_heads_local=8 // g, head_offset=0, head_dim=128)
    for r in reqs:
        if r["measured"] and r["loaded_bytes"] == 0:
            assert r["stall"] == 0.0, r


def issue_order(records):
    """The decisions of a run independent of how the two PCIe directions interleave their
    completions: transfers in issue order (job ids are assigned at issue) and each node's
    sequence of state transitions.  Real B200 link times differ from the cost model's, so an
    offload may land before a concurrently issued prefetch (the trace is in event order)."""
    jobs = [(r["dir"], r["purpose"], r["node"]) for r in sorted((r for r in records if r["t"] == "job"),
                                                                key=lambda r: r["id"])]
    per_node = {}
    for r in records:
        if r["t"] == "tr":
            per_node.setdefault(r["node"], []).append((r["from"], r["to"]))
    return jobs, per_node


@pytest.mark.parametrize("fixed,cap,fixture", [(2048, 855638016, "sim_c1.jsonl"), (8192, 3271557120, "sim_c2.jsonl")])
def test_decisions_robust_to_real_transfer_times(fixed, cap, fixture):
    """SURVEY §7 'hard parts': with the measured B200 transfer times in the loop instead of the
    cost model, the reference's victims and prefetched nodes are chosen, in the same issue order."""
    with S.Sim(timing=1, fixed=fixed, gpu_cap=cap) as s:
        s.run()
        mine = issue_order(s.trace())
    assert mine == issue_order(load_jsonl(fixture))
