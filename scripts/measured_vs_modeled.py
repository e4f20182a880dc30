"""Where does a measured-timing run (real B200 transfer times in the loop) first leave the
reference's modeled-time decision stream?  Prints the first divergence of the transfer and
transition streams with context, and the per-purpose job counts of both runs."""
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle_ffi import load_jsonl  # noqa: E402
from paper_2507_07400_b200 import sim as S  # noqa: E402
from paper_2507_07400_b200.shard import decision_stream  # noqa: E402


def first_diff(a, b):
    for i, (x, y) in enumerate(zip(a, b)):
        if x != y:
            return i
    return None if len(a) == len(b) else min(len(a), len(b))


def main():
    out = {}
    for fixed, cap, fx in [(2048, 855638016, "sim_c1.jsonl"), (8192, 3271557120, "sim_c2.jsonl")]:
        ref = load_jsonl(fx)
        with S.Sim(timing=1, fixed=fixed, gpu_cap=cap) as s:
            s.run()
            mine = s.trace()
        (mj, mt), (rj, rt) = decision_stream(mine), decision_stream(ref)
        dj, dt = first_diff(mj, rj), first_diff(mt, rt)
        rjobs = [r for r in ref if r["t"] == "job"]
        mjobs = [r for r in mine if r["t"] == "job"]
        out[fx] = {
            "jobs": [len(mj), len(rj)], "trs": [len(mt), len(rt)],
            "first_job_diff": dj, "first_tr_diff": dt,
            "mine_jobs_ctx": mjobs[max(0, (dj or 0) - 3):(dj or 0) + 3] if dj is not None else [],
            "ref_jobs_ctx": rjobs[max(0, (dj or 0) - 3):(dj or 0) + 3] if dj is not None else [],
            "mine_purposes": collections.Counter(r["purpose"] for r in mjobs),
            "ref_purposes": collections.Counter(r["purpose"] for r in rjobs),
        }
    print(json.dumps(out, indent=1, default=str))


if __name__ == "__main__":
    main()
