"""Wall-clock driver (ClockMode::WallClock): the workflow runs in real time on the
B200.  Transfers land when their CUDA stop events fire, prefill/decode compute is a spin kernel
of the cost-model duration on the engine's compute stream, and dispatch consumes the real
completion state -- the status-aware queue walk of the reference scheduler
(proj/src/scheduler.cpp:177-216) driven by hardware instead of a model.  Stalls are real
seconds.  Bytes are checked end to end (every loaded node and every resident node)."""
import pytest

from conftest import UNDER_SANITIZER

from oracle_ffi import load_jsonl

pytestmark = pytest.mark.gpu
S = pytest.importorskip("paper_2507_07400_b200.sim")

C1 = dict(fixed=2048, gpu_cap=855638016)
C2 = dict(fixed=8192, gpu_cap=3271557120)


def run_wall(**kw):
    kw.setdefault("audit", 1)
    kw.setdefault("verify_loads", 1)
    with S.Sim(clock=1, **kw) as s:
        s.run()
        res = s.result()
        checked, bad = s.verify_resident()
        return res, s.trace(), (checked, bad)


def reqs(trace):
    return [r for r in trace if r["t"] == "req"]


@pytest.mark.parametrize("cfg,fixture", [(C1, "sim_c1.jsonl"), (C2, "sim_c2.jsonl")])
def test_wall_clock_peer_workflow(cfg, fixture):
    res, trace, (checked, bad) = run_wall(**cfg)
    assert res["verify_failures"] == 0 and res["verified_loads"] > 0
    assert checked > 0 and bad == 0
    measured = [r for r in reqs(trace) if r["measured"]]
    assert len(measured) == 40
    ref = load_jsonl(fixture)
    ref_jobs = [r for r in ref if r["t"] == "job"]
    if UNDER_SANITIZER:  # bytes checked above; the rest is about real time
        return
    # the workflow-aware prefetch fires and serves the steps
    assert res["prefetch_jobs"] > 0
    # steps the prefetch served start within host decision latency of being ready (no PCIe wait)
    for r in measured:
        if r["loaded_bytes"] == 0:
            assert r["stall"] < 2e-3, r
    # a real-time run moves the same order of bytes as the reference's modeled one
    ref_loaded = sum(j["bytes"] for j in ref_jobs if j["dir"] == 0)
    assert 0.5 * ref_loaded <= res["loaded_bytes"] <= 1.5 * ref_loaded
    # makespan: real compute is the cost model's, real PCIe is faster than the model's
    ref_res = [r for r in ref if r["t"] == "res"][0]
    assert res["makespan"] <= ref_res["makespan"] * 1.10


def test_wall_clock_hicache_gate_is_enforced_on_the_gpu():
    """LRU_REACTIVE_HICACHE: a request whose prefix is on the host dispatches at once and its
    prefill waits (on the GPU, cudaStreamWaitEvent) for the loads; the measured gate is the
    part of the load the pipelined prefill could not hide."""
    res, trace, (checked, bad) = run_wall(policy="LRU_REACTIVE_HICACHE", **C2)
    assert bad == 0 and res["verify_failures"] == 0
    jobs = {j["node"]: j for j in trace if j["t"] == "job" and j["dir"] == 0}
    gated = [r for r in reqs(trace) if r["loaded_bytes"] > 0]
    assert gated, "C2 under HiCache must reload prefixes"
    for r in gated:
        assert r["stall"] >= 0.0
    assert res["prefetch_jobs"] == 0
    assert len(jobs) > 0


def test_wall_clock_gpu_only_baseline():
    res, trace, (checked, bad) = run_wall(policy="LRU_GPU_ONLY", **C1)
    assert bad == 0
    assert res["loaded_bytes"] == 0 and res["offloaded_bytes"] == 0


def test_prefetch_retry_on_transfer_done():
    """§8f-2 prefetch retry: re-running the step-1 prefetch whenever a transfer lands never
    issues fewer prefetches than arrival-only issue, and keeps every byte intact."""
    base, _, _ = run_wall(**C2)
    retry, trace, (checked, bad) = run_wall(prefetch_retry=1, **C2)
    assert bad == 0 and retry["verify_failures"] == 0
    if UNDER_SANITIZER:
        return
    assert retry["prefetch_jobs"] >= base["prefetch_jobs"]
    assert retry["stall_total_s"] <= base["stall_total_s"] + 0.05


def test_wall_clock_compute_scale_runs_faster():
    res, _, (checked, bad) = run_wall(compute_scale=0.25, **C1)
    assert bad == 0
    if UNDER_SANITIZER:
        return
    ref_res = [r for r in load_jsonl("sim_c1.jsonl") if r["t"] == "res"][0]
    assert res["makespan"] < 0.6 * ref_res["makespan"]


def test_layered_gate_bytes_and_stall():
    """§8f-1 in the driver: HiCache-gated prefills consume layer-pipelined loads (prefill layer
    l waits only for layer l of its loads, on the GPU).  Bytes stay exact; the exposed stall
    is no larger than with the whole-load gate."""
    whole, _, _ = run_wall(policy="LRU_REACTIVE_HICACHE", **C2)
    lay, trace, (checked, bad) = run_wall(policy="LRU_REACTIVE_HICACHE", layered_gate=1, **C2)
    assert bad == 0 and lay["verify_failures"] == 0 and lay["verified_loads"] > 0
    if UNDER_SANITIZER:
        return
    # Real time: which requests find their prefix on the host depends on when write-backs
    # land, so the two runs' reactive-load counts differ (29-40 of 40 seen); compare the stall
    # each reactive load exposes.
    assert lay["reactive_jobs"] > 0 and whole["reactive_jobs"] > 0
    per_lay = lay["stall_total_s"] / lay["reactive_jobs"]
    per_whole = whole["stall_total_s"] / whole["reactive_jobs"]
    assert per_lay <= per_whole * 1.05 + 0.5e-3, (per_lay, per_whole)
