"""Helpers shared by the lockstep parity tests and smoke(): map a golden trace's recorded
reference arguments onto kvfh_sim_config, and compare traces record for record."""


INT_KEYS = ["agents", "iterations", "warmup", "workflows", "fixed", "dyn", "out", "shared_prefix", "vocab",
            "gpu_cap", "cpu_cap", "seed", "max_running", "max_prefetch", "audit"]


def config_from_golden(cfg_rec):
    a = cfg_rec["args"]
    kw = {k: int(a[k]) for k in INT_KEYS if k in a}
    kw["bytes_per_token"] = int(a.get("bpt", 131072))
    for k in ("topology", "policy", "profile"):
        if k in a:
            kw[k] = a[k]
    if "prefetch" in a:
        kw["prefetch"] = int(a["prefetch"])
    if "eviction" in a:
        kw["eviction"] = 1 if a["eviction"] == "WA" else 0
    if a.get("boundary") == "heuristic":
        kw["heuristic_boundary"] = 1
    if "overlap" in a:
        kw["overlap_fraction"] = float(a["overlap"])
    return kw


def split(records):
    out = {"tr": [], "job": [], "req": [], "res": [], "dump": []}
    for r in records:
        if r["t"] in out:
            out[r["t"]].append(r)
    return out


def assert_same_trace(golden, mine):
    g, m = split(golden), split(mine)
    gtr = [(r["ev"], r["node"], r["from"], r["to"], r["tokens"]) for r in g["tr"]]
    mtr = [(r["ev"], r["node"], r["from"], r["to"], r["tokens"]) for r in m["tr"]]
    assert mtr == gtr, "status-transition (victim / prefetch) sequence differs"
    keys = ["id", "dir", "purpose", "node", "bytes", "enqueue", "start", "complete", "tc", "tn"]
    assert [tuple(r[k] for k in keys) for r in m["job"]] == [tuple(r[k] for k in keys) for r in g["job"]]
    assert [{k: v for k, v in r.items()} for r in m["req"]] == g["req"]
    rk = ["makespan", "end_of_run", "loaded_bytes", "offloaded_bytes", "wasted", "events", "nodes"]
    assert {k: m["res"][0][k] for k in rk} == {k: g["res"][0][k] for k in rk}
    if g["dump"]:
        assert m["dump"][0]["text"] == g["dump"][0]["text"]
