"""Per-CTA timeline of K6 (KVF_ATTEND_TRACE): prologue, main loop, epilogue, spread.
    KVF_ATTEND_TRACE=gpurun_out/k6_trace.jsonl python scripts/attend_trace.py [lens...]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_07400_b200 import _native as N  # noqa: E402
from paper_2507_07400_b200.engine import Engine  # noqa: E402

path = os.environ["KVF_ATTEND_TRACE"]
lens = [int(x) for x in sys.argv[1:]] or [8320] * 4
e = Engine(layers=32, kv_heads_total=8, gpu_slots=sum(lens) + 64, host_slots=0)
rng = np.random.default_rng(1)
seqs = []
for n in lens:
    r = e.alloc(N.KVF_TIER_DEVICE, n)
    e.fill(N.KVF_TIER_DEVICE, r, rng.integers(0, 2**63, size=n, dtype=np.uint64))
    seqs.append(r)
e.sync()
q = torch.randn(len(lens), 32, 128, device="cuda").to(torch.bfloat16)
out = torch.empty_like(q)
torch.cuda.synchronize()
if os.path.exists(path):
    os.remove(path)
plan = e.attend_runs(seqs)
jobs_ms = []
for layer in range(6):
    j = e.attend(layer, 4, q.data_ptr(), plan, out.data_ptr(), 0.088)
    e.wait(j)
    jobs_ms.append(e.elapsed_ms(j) * 1e3)
    e.release(j)
print("job us (events: kernel + combine):", [round(x, 1) for x in jobs_ms])
rows = [json.loads(l) for l in open(path)]
tb = sum(lens) * 2 * e.tpb
for call in rows[2:]:
    a = np.array(call, dtype=np.float64)
    t0 = a[:, 0].min()
    s, p, l, en = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3, (a[:, 2] - t0) / 1e3, (a[:, 3] - t0) / 1e3
    print(f"CTAs {len(a)} SMs {len(set(a[:,4]))}  span {en.max():.1f} us  start spread {s.max():.2f}  "
          f"prologue {np.median(p - s):.2f} (max {np.max(p - s):.2f})  loop med {np.median(l - p):.1f} "
          f"min {np.min(l - p):.1f} max {np.max(l - p):.1f}  epi {np.median(en - l):.2f}  "
          f"loop-end spread {l.max() - l.min():.1f}  GB/s(span) {tb / en.max() / 1e3:.0f}")
