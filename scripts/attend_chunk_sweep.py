"""K6 single-layer call time vs work-item size (chunk tokens per item; 0 = one wave, the default):
more, smaller items let the block scheduler balance the per-SM bandwidth spread over several
waves, at the price of a prologue per item and more partials to combine.  Calls enqueued
behind a spin (device time per call).  Diagnostics for DESIGN §9 item 3."""
import json
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from attend_bench import build, hbm_peak  # noqa: E402
from paper_2507_07400_b200.engine import Engine  # noqa: E402


def sweep(name, kv_local, group, lens, layers, chunks):
    rng = np.random.default_rng(1)
    e = Engine(layers=layers, kv_heads_total=8, kv_heads_local=kv_local, head_offset=8 - kv_local,
               gpu_slots=sum(lens) + 4096 + 2 * len(lens), host_slots=0)
    seqs = e.attend_runs(build(e, lens, rng))
    q = torch.randn(len(lens), kv_local * group, 128, device="cuda").to(torch.bfloat16)
    out = torch.empty_like(q)
    torch.cuda.synchronize()
    peak, _ = hbm_peak()
    nbytes = sum(lens) * 2 * e.tpb
    rows = []
    for ch in chunks:
        per = []
        for rep in range(4):
            e.compute_spin(3_000_000, 1)
            js = [e.attend(l, group, q.data_ptr(), seqs, out.data_ptr(), 1 / math.sqrt(128), chunk=ch) for l in range(layers)]
            e.wait(js[-1])
            if rep:
                per += [e.elapsed_ms(j) for j in js]
            for j in js:
                e.release(j)
        us = float(np.median(per)) * 1e3
        rows.append({"workload": name, "chunk": ch, "us_per_call": round(us, 2), "frac": round(nbytes / (us * 1e-6) / 1e9 / peak, 4)})
        print(json.dumps(rows[-1]), flush=True)
    e.close()
    return rows


if __name__ == "__main__":
    res = []
    res += sweep("C2 2x8320", 8, 4, [8320] * 2, 32, [0, 448, 224, 160, 112, 96, 64])
    res += sweep("C2 4x8320", 8, 4, [8320] * 4, 32, [0, 448, 224, 160, 112])
    res += sweep("C5 70B shard 4x8320", 1, 8, [8320] * 4, 80, [0, 448, 224, 128, 64])
    if len(sys.argv) > 1:
        json.dump(res, open(sys.argv[1], "w"), indent=1)
