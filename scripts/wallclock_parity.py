#!/usr/bin/env python3
"""Wall-clock (real-overlap) runs pinned to the reference's decisions.

For each BASELINE config the workflow runs in ClockMode::WallClock on the B200: transfers
land when their CUDA stop events fire, prefill/decode compute is a spin kernel of the
cost-model duration, and dispatch consumes real completion state.  The run's decisions are
then compared with the unmodified reference's golden trace (tests/golden/sim_*.jsonl):

  * transfers in ISSUE order (direction, purpose, node) -- job ids are assigned at issue;
  * every node's sequence of status transitions (the victim and prefetched-node sequences).

Completion order is not compared: real PCIe times are not the cost model's, so a write-back
may land before a concurrently issued prefetch.  The script also reports the stall
distribution on the steps the reference served by prefetch (north_star: zero stall) and the
first divergence, if any.

    python scripts/wallclock_parity.py [--out profiles/r02_wallclock_parity.json] [--configs c1,c2,c5g2,...]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from golden_sim import config_from_golden  # noqa: E402
from oracle_ffi import load_jsonl  # noqa: E402


def c5_extra(g):
    # Llama-3-70B KV shard: 80 layers, 8/G of the 8 KV heads (the last shard: head_offset != 0)
    return dict(layers=80, kv_heads_total=8, kv_heads_local=8 // g, head_offset=8 - 8 // g, head_dim=128)


CONFIGS = {
    "c1": ("sim_c1.jsonl", {}),
    "c2": ("sim_c2.jsonl", {}),
    "c5g1": ("sim_c5_g1.jsonl", c5_extra(1)),
    "c5g2": ("sim_c5_g2.jsonl", c5_extra(2)),
    "c5g4": ("sim_c5_g4.jsonl", c5_extra(4)),
    "c5g8": ("sim_c5_g8.jsonl", c5_extra(8)),
}


def issue_order(records):
    jobs = [(r["dir"], r["purpose"], r["node"]) for r in sorted((r for r in records if r["t"] == "job"),
                                                                key=lambda r: r["id"])]
    per_node = {}
    for r in records:
        if r["t"] == "tr":
            per_node.setdefault(r["node"], []).append((r["from"], r["to"]))
    return jobs, per_node


def first_divergence(a, b):
    for i, (x, y) in enumerate(zip(a, b)):
        if x != y:
            return {"index": i, "reference": list(y), "wallclock": list(x)}
    if len(a) != len(b):
        return {"index": min(len(a), len(b)), "reference_len": len(b), "wallclock_len": len(a)}
    return None


def run_one(name, reps=1):
    from paper_2507_07400_b200.sim import Sim

    fixture, extra = CONFIGS[name]
    golden = load_jsonl(fixture)
    kw = config_from_golden(golden[0])
    kw.update(extra)
    kw.update(clock=1, audit=1, verify_loads=1)
    ref_jobs, ref_nodes = issue_order(golden[1:])
    ref_reqs = {r["id"]: r for r in golden[1:] if r["t"] == "req"}
    runs = []
    for _ in range(reps):
        with Sim(**kw) as s:
            s.run()
            res = s.result()
            trace = s.trace()
            checked, bad = s.verify_resident()
        jobs, nodes = issue_order(trace)
        node_diff = sorted(n for n in set(ref_nodes) | set(nodes) if ref_nodes.get(n) != nodes.get(n))
        # steps the reference served by prefetch: measured, nothing loaded reactively by the step itself
        served = [r for r in trace if r["t"] == "req" and r["measured"] and ref_reqs.get(r["id"], {}).get("loaded_bytes", 1) == 0]
        stalls_us = sorted(1e6 * r["stall"] for r in served)
        waits_us = sorted(1e6 * r["load_wait"] for r in served)
        reactive = [r for r in trace if r["t"] == "req" and r["measured"] and r["loaded_bytes"] > 0]
        runs.append({
            "issue_order_equal": jobs == ref_jobs,
            "node_transitions_equal": not node_diff,
            "jobs": len(jobs), "reference_jobs": len(ref_jobs),
            "first_job_divergence": first_divergence(jobs, ref_jobs),
            "nodes_differing": node_diff[:10],
            "bytes_verified": {"loads": res["verified_loads"], "load_failures": res["verify_failures"],
                               "resident_checked": checked, "resident_bad": bad},
            "prefetch_served_steps": len(served),
            "prefetch_served_stall_us": {"max": round(max(stalls_us), 2) if stalls_us else None,
                                         "median": round(statistics.median(stalls_us), 2) if stalls_us else None,
                                         "p90": round(stalls_us[int(0.9 * (len(stalls_us) - 1))], 2) if stalls_us else None,
                                         "zero": sum(1 for s in stalls_us if s == 0.0),
                                         "under_100us": sum(1 for s in stalls_us if s < 100.0)},
            # the prefix-miss stall proper: GPU-timed waits of the step's prefill on KV loads
            "prefetch_served_load_wait_us": {"max": round(max(waits_us), 2) if waits_us else None,
                                             "zero": sum(1 for s in waits_us if s == 0.0),
                                             "nonzero": [round(s, 2) for s in waits_us if s != 0.0][:10]},
            "reactive_load_wait_ms": [round(1e3 * r["load_wait"], 3) for r in reactive],
            "reactive_steps": len(reactive),
            "reactive_stall_ms": [round(1e3 * r["stall"], 3) for r in reactive],
            "prefetch_jobs": res["prefetch_jobs"], "reactive_jobs": res["reactive_jobs"],
            "offload_jobs": res["offload_jobs"], "makespan_s": round(res["makespan"], 4),
            "reference_makespan_s": [r for r in golden if r["t"] == "res"][0]["makespan"],
            "decision_us_per_arrival": round(res["decision_us_total"] / max(1, res["arrivals"]), 2),
        })
    return {"config": name, "fixture": fixture, "runs": runs}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c2,c5g2,c5g4,c5g8")
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    out = {"what": "wall-clock (real overlap) runs vs the unmodified reference's golden decisions",
           "results": [run_one(c, a.reps) for c in a.configs.split(",")]}
    s = json.dumps(out, indent=1)
    print(s)
    if a.out:
        with open(a.out, "w") as f:
            f.write(s + "\n")


if __name__ == "__main__":
    main()
