"""Bandwidth probe for K1/K2/K3 against copy-engine peaks (run on the GPU box).

  python scripts/probe_copy.py [--tokens 8192] [--reps 5]

Prints one JSON object: measured pinned H2D/D2H copy-engine peaks (torch, CUDA events)
and K1/K2/K3 GB/s per back-end and grid size.  Event timing on the job's own stream.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_07400_b200 import _native as N  # noqa: E402
from paper_2507_07400_b200.engine import Engine  # noqa: E402


def ce_peak(nbytes, reps):
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    out = {}
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
        best = 0.0
        with torch.cuda.stream(s):
            for _ in range(reps + 1):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                fn()
                b.record(s)
                b.synchronize()
                best = max(best, nbytes / (a.elapsed_time(b) * 1e-3) / 1e9)
        out[name] = best
    a = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    best = 0.0
    for _ in range(reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        d.copy_(a)
        e1.record()
        e1.synchronize()
        best = max(best, 2 * nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    out["d2d_rw"] = best
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=8192)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    ntok = args.tokens
    e = Engine(layers=32, kv_heads_total=8, head_dim=128, gpu_slots=ntok * 2 + 64, host_slots=ntok * 2 + 64)
    nbytes = ntok * e.token_bytes
    res = {"tokens": ntok, "bytes": nbytes, "ce": ce_peak(nbytes, args.reps)}
    rng = np.random.default_rng(0)
    cids = rng.integers(0, 2**63, size=ntok, dtype=np.uint64)
    h = e.alloc(N.KVF_TIER_HOST, ntok)
    d = e.alloc(N.KVF_TIER_DEVICE, ntok)
    d2 = e.alloc(N.KVF_TIER_DEVICE, ntok)
    e.fill(N.KVF_TIER_HOST, h, cids)
    e.sync()

    def timed(fn):
        best = 0.0
        for _ in range(args.reps + 1):
            j = fn()
            ms = e.elapsed_ms(j)
            e.release(j)
            best = max(best, nbytes / (ms * 1e-3) / 1e9)
        return best

    res["k1_h2d"], res["k2_d2h"], res["k3_gather"] = {}, {}, {}
    for mode, mname in ((N.KVF_COPY_SM_VEC, "vec"), (N.KVF_COPY_SM_BULK, "bulk"), (N.KVF_COPY_CE, "ce")):
        for ctas in ((8, 16, 32, 64, 148, 296) if mode != N.KVF_COPY_CE else (1,)):
            e.set_copy_mode(mode, ctas)
            try:
                res["k1_h2d"][f"{mname}_{ctas}"] = timed(lambda: e.h2d(h, d))
                res["k2_d2h"][f"{mname}_{ctas}"] = timed(lambda: e.d2h(d, h))
            except Exception as ex:  # report, keep probing the rest
                res["k1_h2d"][f"{mname}_{ctas}"] = str(ex)
    st = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    for ctas in (148, 296, 592, 1184):
        e.set_copy_mode(N.KVF_COPY_SM_VEC, 0, ctas)
        res["k3_gather"][str(ctas)] = 2 * timed(lambda: e.dev_gather(d, st.data_ptr()))
    e.set_copy_mode(N.KVF_COPY_SM_VEC, 0, 0)
    # verify the last H2D landed bit-exact
    e.set_copy_mode(N.KVF_COPY_SM_VEC, 32)
    j = e.h2d(h, d2)
    e.wait(j)
    res["verify_checksum_equal"] = e.checksum(N.KVF_TIER_DEVICE, d2) == e.checksum(N.KVF_TIER_HOST, h)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
