#!/usr/bin/env python3
"""Seeded fuzz corpus of whole-workflow golden traces from the UNMODIFIED reference.

    python tests/golden/make_fuzz.py [--n 40] [--seed 2507]

Draws random Simulator configurations across the reference's own parameter space (topology,
policy, eviction order, agents, prompt / suffix / output lengths, workflows, intra-client
shared prefixes, GPU budget from ~1 to ~4 agent footprints, concurrency caps, prefetch cap,
boundary mode, gate overlap fraction, seeds), runs each through oracle/_ref/ref_trace (the
reference compiled in place) and keeps every configuration the reference completes as
tests/golden/fuzz/sim_f_NN.jsonl -- the trace format tests/test_lockstep_gpu.py replays on the
GPU engine record for record.  Configurations the reference itself rejects (SimError) are
kept too (up to --n-err of them) as fuzz/sim_e_NN.jsonl with a final {"t":"err","code":C}
record: the GPU run must fail with the same ErrorCode after the same status transitions.  Micro cost profile, 16 B/token, so one
configuration runs in well under a second on the GPU.  Needs /root/reference (this container
only); the fixtures are committed and the GPU box never runs this script.
"""
import argparse
import json
import os
import random
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
TRACE = os.path.join(ROOT, "oracle", "_ref", "ref_trace")


def draw(rng, geom="micro"):
    topo = rng.choice(["CYCLIC", "SEQUENTIAL", "BRANCH_MAX", "BRANCH_MIN", "PEER_STYLE"])
    agents = 4 if topo.startswith("BRANCH") else rng.randint(1, 4)  # workload.cpp:35-36
    fixed = rng.choice([16, 32, 64, 96, 128, 256, 512])
    dyn = rng.choice([4, 8, 16, 32])
    out = rng.choice([0, 3, 8, 16])
    workflows = rng.randint(1, 3)
    shared = rng.choice([0, 0, 8, 16, 32]) if fixed > 32 else 0
    footprint = agents * (fixed + dyn + out) * 16
    a = {
        "profile": "micro", "bpt": 16, "vocab": 50000, "topology": topo, "agents": agents,
        "iterations": rng.randint(2, 4), "warmup": rng.randint(0, 1), "fixed": fixed, "dyn": dyn, "out": out,
        "workflows": workflows, "shared_prefix": shared,
        "gpu_cap": int(footprint * workflows * rng.uniform(0.35, 1.4)) // 16 * 16,
        "policy": rng.choice(["LRU_GPU_ONLY", "LRU_REACTIVE_HICACHE", "KVFLOW", "KVFLOW"]),
        "max_running": rng.choice([1, 2, 4, 8]), "max_prefetch": rng.choice([1, 2, 3]),
        "seed": rng.randint(1, 10**6), "audit": 1,
    }
    if rng.random() < 0.3:
        a["eviction"] = "WA"
    if rng.random() < 0.2:
        a["boundary"] = "heuristic"
    if rng.random() < 0.2:
        a["overlap"] = rng.choice([0.0, 0.25, 0.75, 1.0])
    if rng.random() < 0.25:  # bounded CPU tier: fallback discards, and the reference's own
        # remove_node defect surfaces as an InternalError to match
        a["cpu_cap"] = int(footprint * workflows * rng.uniform(0.1, 1.5)) // 16 * 16
    if topo == "PEER_STYLE":  # the generator draws its own lengths
        for k in ("fixed", "dyn", "out", "shared_prefix"):
            a.pop(k)
        a["gpu_cap"] = int(agents * workflows * 900 * 16 * rng.uniform(0.5, 2.0)) // 16 * 16
    if geom == "llama8b":  # real KV bytes: every transfer is megabytes of K1/K2
        scale = 131072 // 16
        a.update(profile="h100-qwen32b", bpt=131072, vocab=32000)
        a["gpu_cap"] *= scale
        if "cpu_cap" in a:
            a["cpu_cap"] *= scale
    return a


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=40)
    ap.add_argument("--seed", type=int, default=2507)
    ap.add_argument("--n-err", type=int, default=12)
    ap.add_argument("--geom", choices=["micro", "llama8b"], default="micro",
                    help="micro: 16 B/token, micro cost profile (sim_f_/sim_e_); llama8b: 128 KiB/token, "
                         "h100-qwen32b profile, shorter prompts (sim_g_)")
    args = ap.parse_args()
    subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True, capture_output=True)
    out_dir = os.path.join(HERE, "fuzz")
    os.makedirs(out_dir, exist_ok=True)
    pre = ("sim_g_",) if args.geom == "llama8b" else ("sim_f_", "sim_e_")
    for f in os.listdir(out_dir):
        if f.startswith(pre):
            os.remove(os.path.join(out_dir, f))
    rng = random.Random(args.seed)
    kept, errs, rejected, tries = [], [], {}, 0
    while len(kept) < args.n and tries < 20 * args.n:
        tries += 1
        a = draw(rng, args.geom)
        r = subprocess.run([TRACE, "sim", *[f"{k}={v}" for k, v in a.items()]], capture_output=True, text=True)
        if r.returncode != 0:
            key = r.stderr.strip().split(":")[0] or f"rc {r.returncode}"
            rejected[key] = rejected.get(key, 0) + 1
            if r.returncode == 3 and key.startswith("SimError") and len(errs) < args.n_err and args.geom == "micro":
                name = f"sim_e_{len(errs):02d}.jsonl"
                code = int(key.split()[1])
                with open(os.path.join(out_dir, name), "w") as f:
                    f.write(r.stdout + json.dumps({"t": "err", "code": code, "args": a}) + "\n")
                errs.append({"file": name, "args": a, "code": code, "message": r.stderr.strip()})
            continue
        lines = r.stdout.splitlines()
        n_tr = sum(1 for l in lines if '"t":"tr"' in l)
        n_job = sum(1 for l in lines if '"t":"job"' in l)
        if n_job == 0 and rng.random() < 0.7:  # keep the corpus transfer-heavy
            continue
        name = f"{'sim_g_' if args.geom == 'llama8b' else 'sim_f_'}{len(kept):02d}.jsonl"
        with open(os.path.join(out_dir, name), "w") as f:
            f.write(r.stdout)
        kept.append({"file": name, "args": a, "transitions": n_tr, "jobs": n_job})
    with open(os.path.join(out_dir, f"MANIFEST{'_llama8b' if args.geom == 'llama8b' else ''}.json"), "w") as f:
        json.dump({"seed": args.seed, "tries": tries, "kept": kept, "errors": errs, "reference_rejected": rejected}, f,
                  indent=1)
    print(f"kept {len(kept)} of {tries}; reference rejected {rejected}; {len(errs)} error fixtures")


if __name__ == "__main__":
    main()
