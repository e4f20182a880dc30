"""Summarise ncu captures into profiles/ncu_summary.json (read here, not on the GPU box).

    python scripts/ncu_summary.py TAG        # reads gpurun_out/prof_<k>_<TAG>.ncu-rep, launches_<TAG>.csv

Per kernel: duration, DRAM read/write bytes (the `traffic` of bench.py's roofline), PCIe
rates, launch shape, registers and the algorithmic bytes of that launch.
Launch shares: each kernel's share of device time in the bench's ncu launch list.
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9, "us": 1e-6,
        "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "nsecond": 1e-9, "second": 1.0}
ALGO = {  # algorithmic bytes per launch of the capture in scripts/profile_kernels.py
    "k1": 8192 * 131072, "k2": 128 * 131072, "k3": 2 * 8192 * 131072,
    "k6": 4 * 8320 * 2 * 2048,  # one layer of 4 x 8320-token sequences, K + V (scripts/attend_bench.py --ncu)
}
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size",
        "launch__block_size", "launch__registers_per_thread", "pcie__read_bytes.sum.per_second",
        "pcie__write_bytes.sum.per_second", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "Kernel Name"]


def raw(rep, row=0):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, vals = rows[0], rows[1], rows[2 + row]
    return {w: (units[h.index(w)], vals[h.index(w)]) for w in WANT if w in h}


def all_rows(rep):
    """Every kernel of a multi-kernel capture (the device-wide K5 graph): name, duration, grid."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        if len(vals) < len(h):
            continue
        u = units[h.index("gpu__time_duration.sum")]
        res.append({"kernel": vals[h.index("Kernel Name")],
                    "duration_us": float(vals[h.index("gpu__time_duration.sum")].replace(",", "")) * UNIT.get(u, 1.0) * 1e6,
                    "grid": vals[h.index("launch__grid_size")], "block": vals[h.index("launch__block_size")]})
    return res


def scaled(m, key):
    u, v = m[key]
    return float(v.replace(",", "")) * UNIT.get(u, 1.0)


def kernel(rep, name):
    m = raw(rep)
    d = {"kernel": m["Kernel Name"][1], "duration_s": scaled(m, "gpu__time_duration.sum")}
    rb, wb = scaled(m, "dram__bytes_read.sum"), scaled(m, "dram__bytes_write.sum")
    d.update(dram_read_bytes=rb, dram_write_bytes=wb, dram_traffic_bytes=rb + wb,
             grid=m["launch__grid_size"][1], block=m["launch__block_size"][1],
             registers=m["launch__registers_per_thread"][1])
    for k in ("pcie__read_bytes.sum.per_second", "pcie__write_bytes.sum.per_second",
              "sm__throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed"):
        if k in m:
            d[k] = f"{m[k][1]} {m[k][0]}".strip()
    if name in ALGO:
        d["algorithmic_bytes"] = ALGO[name]
        d["achieved_GBps"] = ALGO[name] / d["duration_s"] / 1e9
    return d


def shares(path):
    rows = list(csv.reader(open(path)))
    i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[i]
    kn, mv = h.index("Kernel Name"), h.index("Metric Value")
    tot, per = 0.0, {}
    for r in rows[i + 1:]:
        if len(r) <= mv or not r[mv].replace(",", "").replace(".", "").isdigit():
            continue
        name = r[kn].split("(")[0].replace("void ", "").replace("<unnamed>::", "").strip()
        t = float(r[mv].replace(",", ""))
        c = per.setdefault(name, [0, 0.0])
        c[0] += 1
        c[1] += t
        tot += t
    return {k: {"launches": n, "share": round(t / tot, 4)} for k, (n, t) in sorted(per.items(), key=lambda x: -x[1][1])}


def main(tag, dst_name="ncu_summary.json"):
    dst = os.path.join(ROOT, "profiles", dst_name)
    # kernels not re-captured under this tag keep their earlier summaries (marked with theirs)
    out = json.load(open(dst)) if os.path.exists(dst) else {}
    prev = out.get("tag")
    for k, v in list(out.items()):
        if isinstance(v, dict) and "kernel" in v and "tag" not in v:
            v["tag"] = prev
    out["tag"] = tag
    for k in ("k1", "k2", "k3", "k5", "k6", "k5m"):
        rep = os.path.join(ROOT, "gpurun_out", f"prof_{k}_{tag}.ncu-rep")
        if os.path.exists(rep):
            out[k] = kernel(rep, k)
            out[k]["tag"] = tag
    rep = os.path.join(ROOT, "gpurun_out", f"prof_k5big_{tag}.ncu-rep")
    if os.path.exists(rep):
        ks = all_rows(rep)
        out["k5_device_wide"] = {"tag": tag, "what": "hand-written device-wide K5 kernels of one 30k-node call",
                                 "kernels": ks, "total_us": round(sum(k["duration_us"] for k in ks), 2)}
    lp = os.path.join(ROOT, "gpurun_out", f"launches_{tag}.csv")
    if os.path.exists(lp):
        out["launch_shares_bench"] = shares(lp)
    with open(dst, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
