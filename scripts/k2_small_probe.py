"""K2 (D2H write-back) efficiency at small sizes -- the 8-way shard's 2 MiB suffixes, C4's
8 MiB segments -- vs CTA count and job timing (events vs kernel stamps), alone and beside a
1 GiB K1.  Diagnostics for the write-back row of DESIGN §7."""
import json
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_07400_b200 import _native as N  # noqa: E402
from paper_2507_07400_b200.engine import Engine  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/k2_small_probe.json"
res = []
# 1 KV head of Llama-3-8B: 32 layers x 2 x 256 B = 16 KiB per token
e = Engine(layers=32, kv_heads_total=8, kv_heads_local=1, head_offset=7, gpu_slots=70000, host_slots=140000)
rng = np.random.default_rng(1)
big_h = e.alloc(N.KVF_TIER_HOST, 65536)  # 1 GiB
big_d = e.alloc(N.KVF_TIER_DEVICE, 65536)
for tokens in (128, 512, 1024):  # 2 / 8 / 16 MiB
    d = e.alloc(N.KVF_TIER_DEVICE, tokens)
    e.fill(N.KVF_TIER_DEVICE, d, rng.integers(0, 2**63, size=tokens, dtype=np.uint64))
    hs = [e.alloc(N.KVF_TIER_HOST, tokens) for _ in range(4)]
    e.sync()
    nbytes = tokens * e.token_bytes
    for ctas in (8, 16, 32):
        e.set_copy_mode(N.KVF_COPY_SM_VEC, ctas, 0)
        for stamps in (False, True):
            e.set_job_timing(stamps)
            for busy in (False, True):
                ts = []
                for rep in range(12):
                    jb = None
                    if busy:
                        e.set_copy_mode(N.KVF_COPY_SM_VEC, 8, 0)
                        jb = e.h2d(big_h, big_d)
                        e.set_copy_mode(N.KVF_COPY_SM_VEC, ctas, 0)
                    j = e.d2h(d, hs[rep % 4])
                    ts.append(e.elapsed_ms(j))
                    e.release(j)
                    if jb is not None:
                        e.wait(jb)
                        e.release(jb)
                ms = statistics.median(ts[2:])
                row = {"mib": nbytes >> 20, "ctas": ctas, "timing": "stamps" if stamps else "events", "beside_k1": busy,
                       "us": round(ms * 1e3, 2), "gbs": round(nbytes / (ms * 1e-3) / 1e9, 2)}
                res.append(row)
                print(json.dumps(row), flush=True)
e.close()
json.dump(res, open(out, "w"), indent=1)
