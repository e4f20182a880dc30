"""Where does a K4/K5 decision call's time go?  Per-call host phases and the kernel's own
globaltimer window (KVF_DECISION_TRACE, csrc/engine/decide.cu), in three settings:
idle, with a 1 GiB K1 saturating the H2D link, and inside the C2 workflow (bench.py's e2e run).

    python scripts/decision_trace.py --out gpurun_out/decision_trace.json
"""
import argparse
import json
import os
import statistics
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

TRACE = os.path.join(tempfile.mkdtemp(), "dtrace.jsonl")
os.environ["KVF_DECISION_TRACE"] = TRACE  # read once, at the first decision call
ARRIVALS = os.path.join(os.path.dirname(TRACE), "arrivals.jsonl")
os.environ["KVF_ARRIVAL_TRACE"] = ARRIVALS  # per-arrival phases (Simulator::on_arrival)

from oracle_ffi import load_jsonl  # noqa: E402
from paper_2507_07400_b200 import _native as N  # noqa: E402
from paper_2507_07400_b200.engine import Engine  # noqa: E402
from paper_2507_07400_b200.sim import Sim  # noqa: E402

sys.path.insert(0, os.path.join(ROOT, "scripts"))
from bench_decisions import tree_of  # noqa: E402

KEYS = ("pack_us", "launch_call_us", "spin_us", "kernel_us")


def lines():
    if not os.path.exists(TRACE):
        return []
    return [json.loads(x) for x in open(TRACE)]


def summary(rows):
    out = {"calls": len(rows)}
    for kind in ("k4", "k5"):
        rs = [r for r in rows if r["kind"] == kind]
        if rs:
            tot = [r["pack_us"] + r["launch_call_us"] + r["spin_us"] for r in rs]
            out[kind] = {"calls": len(rs), "nodes_median": statistics.median(r["n"] for r in rs),
                         **{k: round(statistics.median(r[k] for r in rs), 2) for k in KEYS},
                         "call_us_median": round(statistics.median(tot), 2), "call_us_mean": round(statistics.mean(tot), 2),
                         "call_us_max": round(max(tot), 2), "first_call": {k: round(rs[0][k], 2) for k in KEYS}}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    res = {}
    e = Engine(layers=32, kv_heads_total=8, head_dim=128, gpu_slots=8192 + 256, host_slots=8192 + 256)
    h = e.alloc(N.KVF_TIER_HOST, 8192)
    d = e.alloc(N.KVF_TIER_DEVICE, 8192)
    cases = sorted(load_jsonl("evict_small.jsonl") + load_jsonl("evict_medium.jsonl"), key=lambda c: len(c["parent"]))
    c5 = min(cases, key=lambda c: abs(len(c["parent"]) - 44))  # the C2 tree size
    t5 = tree_of(c5)
    prio = sorted(load_jsonl("prio.jsonl"), key=lambda c: abs(len(c["parent"]) - 44))[0]
    b = prio["boundaries"]
    for phase in ("idle", "busy_h2d"):
        n0 = len(lines())
        job = e.h2d(h, d) if phase == "busy_h2d" else None
        for _ in range(40):
            e.victims(t5, c5["needed"], c5["policy"], c5["mode"], c5["has_floor"], c5["floor"], c5["cpu_used"],
                      c5["cpu_cap"])
            e.priority(prio["parent"], [x[0] for x in b], [int(x[1]) for x in b])
        if job:
            e.wait(job)
            e.release(job)
        res[phase] = summary(lines()[n0:])
    e.close()
    # the C2 workflow, as bench.py's e2e leg runs it (Llama-3-8B, 1 GPU)
    from paper_2507_07400_b200.shard import plan
    import bench
    sp = plan(0, 1, layers=32, kv_heads=8, head_dim=128, gpu_budget=bench.BUDGET_FULL)
    n0 = len(lines())
    sim = Sim(fixed=bench.FIXED, dyn=bench.DYN, out=bench.OUT, gpu_cap=sp.gpu_budget,
              bytes_per_token=sp.bytes_per_token, device=0, numa_node=N.KVF_NUMA_AUTO, **sp.engine_kwargs())
    sim.run()
    sim.close()
    wf = lines()[n0:]
    res["c2_workflow"] = summary(wf)
    res["c2_workflow_p90"] = {k: round(sorted(r[k] for r in wf)[int(0.9 * (len(wf) - 1))], 2) for k in KEYS} if wf else {}
    res["c2_workflow_slow_calls"] = [
        {**{k: round(r[k], 2) for k in KEYS}, "kind": r["kind"], "n": r["n"], "index": i,
         "overhead_us": round(r["spin_us"] - r["kernel_us"], 2)}
        for i, r in enumerate(wf) if r["pack_us"] + r["launch_call_us"] + r["spin_us"] > 60]
    arr = [json.loads(x) for x in open(ARRIVALS)] if os.path.exists(ARRIVALS) else []
    if arr:
        res["c2_arrivals"] = {"count": len(arr), "us_median": round(statistics.median(a["us"] for a in arr), 2),
                              "us_mean": round(statistics.mean(a["us"] for a in arr), 2),
                              "slowest": sorted(arr, key=lambda a: -a["us"])[:4],
                              "first": arr[:2]}
    res["note"] = ("per call, medians: pack = entry -> launch call; launch_call = cudaLaunchKernel; spin = launch "
                   "returned -> done word seen (host clock); kernel = in-kernel (the GPU's globaltimer); the two "
                   "clock domains are never subtracted from each other")
    s = json.dumps(res, indent=1)
    print(s)
    if a.out:
        open(a.out, "w").write(s)


if __name__ == "__main__":
    main()
