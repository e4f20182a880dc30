"""Resident-decider round trips on a 44-node mirror (KVF_MIRROR_TRACE): host wait vs device
serve time vs polls, idle and while a K1 keeps the PCIe link busy.  Diagnostics."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/mirror_probe.json"
tr = out + ".trace.jsonl"
if os.path.exists(tr):
    os.remove(tr)
os.environ["KVF_MIRROR_TRACE"] = tr
from oracle_ffi import TreeArrays, load_jsonl  # noqa: E402
from paper_2507_07400_b200 import _native as N  # noqa: E402
from paper_2507_07400_b200.engine import Engine, Tree, decider_hold  # noqa: E402

c = next(x for x in load_jsonl("evict_small.jsonl") if len(x["parent"]) >= 40 and "error" not in x)
ta = TreeArrays(c)
arr = {k: getattr(ta, k) for k in ("parent", "status", "lock", "rank", "time", "seq", "id", "tokens", "backed")}
args = dict(needed=c["needed"], workflow_aware=c["policy"], offload=c["mode"], has_floor=c["has_floor"],
            floor=c["floor"], cpu_used=c["cpu_used"], cpu_cap=c["cpu_cap"])
res = {}
with Engine(layers=32, kv_heads_total=8, head_dim=128, gpu_slots=8192, host_slots=8192) as eng:
    h = eng.alloc(N.KVF_TIER_HOST, 8192)
    d = eng.alloc(N.KVF_TIER_DEVICE, 8192)
    with Tree(eng, ta.bpt) as t:
        t.load_arrays(arr)
        decider_hold(eng, True)
        for label in ("idle", "busy_h2d"):
            job = eng.h2d(h, d) if label == "busy_h2d" else None
            lat = []
            for i in range(60):
                t0 = time.perf_counter()
                t.victims(**args)
                lat.append((time.perf_counter() - t0) * 1e6)
            if job is not None:
                eng.wait(job)
                eng.release(job)
            res[label] = {"k5_call_us_median": round(statistics.median(lat), 2)}
            t0 = time.perf_counter()
            for i in range(60):
                t.priorities([1], [3])
                t.victims(**args)
                t.rank_changes()
            res[label]["k4_k5_pair_us_mean"] = round((time.perf_counter() - t0) / 60 * 1e6, 2)
        decider_hold(eng, False)
    st = eng.stats()
rows = [json.loads(l) for l in open(tr)]
res["trace"] = {k: round(statistics.median(r[k] for r in rows), 2) for k in ("wait_us", "serve_us", "polls")}
res["trace"]["n"] = len(rows)
res["stats"] = {k: st[k] for k in ("resident_served", "oneshot_served", "resident_launches")}
nk5 = 240  # K5 calls above (victims in both loops)
res["k5_phase_us"] = [round(x / nk5 / 1e3, 2) for x in st["k5_phase_ns"]]
res["k5_phase_cycles"] = [round(x / nk5) for x in st["k5_phase_cycles"]]
print(json.dumps(res, indent=1))
json.dump(res, open(out, "w"), indent=1)
