"""The fuzz corpus (tests/golden/fuzz/) replayed by the WALL-CLOCK driver (ClockMode::WallClock,
SURVEY §8f-2): the same random workflows, but transfers land when their CUDA events fire and
compute is real spin time, so decisions follow real completion order and may legitimately
differ from the reference's virtual-time trace.  What must hold for every configuration: the
run completes, every request the reference served is served, the ledger audits clean after
every event, and every loaded / resident node holds the right bytes.  Half the cases also
switch on the prefetch retry and the layered HiCache gate."""
import glob
import os

import pytest

from golden_sim import config_from_golden
from oracle_ffi import GOLDEN, load_jsonl

pytestmark = pytest.mark.gpu
S = pytest.importorskip("paper_2507_07400_b200.sim")

FUZZ = sorted(os.path.basename(p) for p in glob.glob(os.path.join(GOLDEN, "fuzz", "sim_[fg]_*.jsonl")))


@pytest.mark.parametrize("fixture", FUZZ)
def test_fuzz_workflow_wall_clock(fixture):
    golden = load_jsonl(os.path.join("fuzz", fixture))
    kw = config_from_golden(golden[0])
    kw.update(audit=1, verify_loads=1)
    extra = int(fixture[-8:-6]) % 2 == 1  # odd cases: retry + layered gate on
    with S.Sim(clock=1, prefetch_retry=int(extra), layered_gate=int(extra), **kw) as s:
        s.run()
        res = s.result()
        trace = s.trace()
        checked, bad = s.verify_resident()
    want = [r for r in golden if r["t"] == "req"]
    got = [r for r in trace if r["t"] == "req"]
    assert len(got) == len(want)
    assert sorted((r["client"], r["agent"], r["iter"]) for r in got) == \
        sorted((r["client"], r["agent"], r["iter"]) for r in want)
    assert res["verify_failures"] == 0 and bad == 0
    assert res["verified_loads"] == res["prefetch_jobs"] + res["reactive_jobs"]
