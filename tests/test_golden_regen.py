"""The golden generator is pinned: regenerating the deterministic fixtures with the committed
oracle/ref_trace (built from the unmodified reference) reproduces them byte for byte, so a
change to the trace driver (e.g. the timed sweep modes) cannot silently move a golden vector.
(The evict and sim traces carry wall-clock fields and are pinned by their own tests.)"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref", "ref_trace")
GOLDEN = os.path.join(ROOT, "tests", "golden")


@pytest.mark.skipif(not os.path.exists(REF), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("args,fixture", [(["prio", "seed=4", "cases=200"], "prio.jsonl"),
                                          (["steps", "seed=5", "cases=200"], "steps.jsonl")])
def test_deterministic_goldens_regenerate_identically(args, fixture):
    out = subprocess.run([REF, *args], capture_output=True, text=True, timeout=300, check=True).stdout
    assert out == open(os.path.join(GOLDEN, fixture)).read()
