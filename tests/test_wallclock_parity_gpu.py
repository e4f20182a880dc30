"""Wall-clock (real-overlap) mode pinned to the reference's decisions (SURVEY §7 "hard parts":
wall-clock mode must be shown not to reorder).  The workflow runs in real time on the B200 --
transfers land when their CUDA stop events fire, compute is a spin kernel of the cost-model
duration, dispatch consumes the real completion state -- and its transfers in ISSUE order plus
every node's status-transition sequence (the victim and prefetched-node sequences) must equal
the unmodified reference's golden trace.  Completion order is not compared (real PCIe times
are not the cost model's).  C5 runs at the 2/4/8-way KV-head shard geometry of Llama-3-70B.
Reference decision points: proj/src/scheduler.cpp:177-216, :396-435."""
import os
import sys

import pytest

from conftest import UNDER_SANITIZER

pytestmark = pytest.mark.gpu
pytest.importorskip("paper_2507_07400_b200.sim")
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts"))
from wallclock_parity import run_one  # noqa: E402


@pytest.mark.parametrize("cfg", ["c1", "c2", "c5g2", "c5g4", "c5g8"])
def test_wall_clock_decisions_equal_reference(cfg):
    run = run_one(cfg)["runs"][0]
    assert run["issue_order_equal"], run["first_job_divergence"]
    assert run["node_transitions_equal"], run["nodes_differing"]
    b = run["bytes_verified"]
    assert b["load_failures"] == 0 and b["resident_bad"] == 0 and b["loads"] > 0
    if UNDER_SANITIZER:
        return
    # the steps the reference served by prefetch start within host decision latency (no PCIe wait)
    st = run["prefetch_served_stall_us"]
    assert run["prefetch_served_steps"] == 37
    assert st["median"] < 250 and st["max"] < 2000, st
    # north_star: zero prefix-miss stalls on the prefetch-served steps -- none of them was held
    # for KV on the wire or on the host, and no prefill's compute stream waited on a load
    # (GPU-timed); the rest of `stall` is dispatch latency.  The reactive steps do wait.
    lw = run["prefetch_served_load_wait_us"]
    assert lw["zero"] == 37 and lw["max"] == 0.0, lw
    assert all(w > 0 for w in run["reactive_load_wait_ms"])
