"""Health check of the oracle build: the reference's OWN unit suites (proj/tests/test_*.cpp,
55 test cases) compiled unmodified, in place, against oracle/_ref/libkvsim_ref.a with the
doctest-compatible shim in oracle/doctest_shim/ (`make -C oracle suites`).

Every case must pass except the reference's own known failures, which must
still fail exactly where the survey recorded them -- so the compiled reference behaves as
its authors' tests say before any golden vector drawn from it is trusted.
"""
import glob
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")
SUITES = ["cost_model", "radix_cache", "scheduler", "step_graph", "tier_manager", "workload"]
# failures of the reference against its own tests (not used as pins)
KNOWN = {"test_scheduler.cpp:310", "test_scheduler.cpp:313", "test_scheduler.cpp:345", "test_scheduler.cpp:418"}


def _bins():
    return [os.path.join(REF, f"suite_{s}") for s in SUITES]


@pytest.mark.skipif(not all(os.path.exists(b) for b in _bins()),
                    reason="oracle/_ref suites not built (needs /root/reference: make -C oracle ref suites)")
def test_reference_suites_pass_except_known_failures():
    failures, cases, passed = set(), 0, 0
    for b in _bins():
        r = subprocess.run([b], capture_output=True, text=True, timeout=600)
        for line in r.stdout.splitlines():
            m = re.match(r"FAIL (\S+):(\d+):", line)
            if m:
                failures.add(f"{os.path.basename(m.group(1))}:{m.group(2)}")
        m = re.search(r"test cases: (\d+) \| (\d+) passed", r.stdout)
        assert m, r.stdout[-2000:]
        cases += int(m.group(1))
        passed += int(m.group(2))
    assert cases == 55
    assert failures == KNOWN, f"unexpected: {sorted(failures - KNOWN)}; missing: {sorted(KNOWN - failures)}"
    assert passed == 52
