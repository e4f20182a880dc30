"""C3 (BASELINE configs[2]): 16-agent Agent Step Graph with conditional branches (MIN
joins), a 6-way barrier (MAX join), mixed 1k-8k prompts behind a shared system prompt.
The same harness source (tests/cpp/c3_harness.hpp) runs against the UNMODIFIED reference
components (golden tests/golden/c3_*.jsonl, oracle/_ref/ref_c3) and against this repo on
the GPU engine (tests/cpp/c3_kvf): traces must match record for record, and every resident
or backed node must hold its expected bytes."""
import json
import os
import subprocess

import pytest

from oracle_ffi import load_jsonl

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2507_07400_b200")


def _build():
    from paper_2507_07400_b200 import build as B
    B.build_engine()
    B.build_host()
    exe = os.path.join(ROOT, "tests", "cpp", "c3_kvf")
    src = os.path.join(ROOT, "tests", "cpp", "c3_kvf.cpp")
    subprocess.run(["g++", "-std=c++20", "-O2", f"-I{ROOT}/include", f"-I{ROOT}/tests/cpp", src, "-o", exe,
                    f"-L{PKG}", "-lkvflow_driver", "-lkvflow_host", "-lkvflow", f"-Wl,-rpath,{PKG}"], check=True)
    return exe


C3_CASES = [("3", "4", "393216000"), ("11", "6", "262144000"), ("5", "4", "327680000"), ("7", "5", "294912000"),
            ("13", "4", "360448000"), ("17", "6", "425984000"), ("19", "3", "229376000"), ("23", "5", "491520000")]


@pytest.mark.parametrize("fixture,args", [(f"c3_seed{s}.jsonl", [s, it, "16384", cap]) for s, it, cap in C3_CASES])
def test_c3_matches_reference(fixture, args):
    exe = _build()
    r = subprocess.run([exe, *args], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    mine = [json.loads(l) for l in r.stdout.splitlines() if l.strip()]
    golden = load_jsonl(fixture)
    assert not [x for x in mine if x["t"] == "error"]
    by = lambda recs, t: [x for x in recs if x["t"] == t]  # noqa: E731
    for t in ("tr", "req", "skip", "job", "dump"):
        assert by(mine, t) == by(golden, t), t
    b = by(mine, "bytes")[0]
    assert b["checked"] > 0 and b["bad"] == 0
    assert sum(1 for j in by(golden, "job") if j["purpose"] == 1) > 0  # prefetches exercised
