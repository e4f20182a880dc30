"""Per-arrival decision time of the C2 workflow through the resident decider: phase breakdown
(KVF_ARRIVAL_TRACE) + who served the decisions.  Diagnostics for DESIGN §6."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/decider_probe.json"
arr = os.path.join(os.path.dirname(out) or ".", "arrivals_probe.jsonl")
if os.path.exists(arr):
    os.remove(arr)
os.environ["KVF_ARRIVAL_TRACE"] = arr
from paper_2507_07400_b200.sim import Sim  # noqa: E402

FIXED, BPT = 8192, 131072
budget = int(3.0 * (FIXED + 128) * BPT)
res = {}
for label, env in (("resident", "1"), ("oneshot", "0")):
    os.environ["KVF_DECIDER"] = env
    if os.path.exists(arr):
        os.remove(arr)
    runs = []
    for rep in range(3):
        with Sim(fixed=FIXED, dyn=64, out=64, gpu_cap=budget, bytes_per_token=BPT) as s:
            s.run()
            r = s.result()
        runs.append(r)
    rows = [json.loads(l) for l in open(arr)]
    n = len(rows)
    r = runs[-1]
    res[label] = {
        "decision_us_per_agent_step": round(statistics.median(x["decision_us_total"] / x["arrivals"] for x in runs), 2),
        "decision_excl_issue_us_per_agent_step": round(statistics.median(
            (x["decision_us_total"] - x["decision_issue_us"]) / x["arrivals"] for x in runs), 2),
        "arrival_us_median": round(statistics.median(x["us"] for x in rows), 2),
        "priorities_us_median": round(statistics.median(x["priorities_us"] for x in rows), 2),
        "schedule_us_median": round(statistics.median(x["schedule_us"] for x in rows), 2),
        "prefetch_us_median": round(statistics.median(x["prefetch_us"] for x in rows), 2),
        "arrivals": n,
        "k4_calls": r["priority_calls"], "k4_issued": r["priority_issued"], "k4_us_total": round(r["priority_us"], 1), "k4_join_us": round(r["k4_join_us"], 1),
        "k5_calls": r["evict_calls"], "k5_us_total": round(r["k5_us"], 1), "apply_us": round(r["apply_us"], 1),
        "k1_k2_issue_us": round(r["issue_us"], 1), "resident_served": r["resident_served"],
        "oneshot_served": r["oneshot_served"], "resident_launches": r["resident_launches"],
        "mirror_records": r["mirror_records"], "engine_kernel_ms": round(r["engine_decision_kernel_ms"], 3),
    }
    print(label, json.dumps(res[label]), flush=True)
json.dump(res, open(out, "w"), indent=1)
