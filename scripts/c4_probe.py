"""C4 (64 workflows, shared prefixes) as one 8-way KV-head shard through the lockstep driver:
K2 launches and wall time with write-back coalescing across evict calls (default) vs one
launch per evict call vs one launch per write-back.  Traces must be identical."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_07400_b200 import _native as N  # noqa: E402
from paper_2507_07400_b200.sim import Sim  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/c4_probe.json"
kw = dict(topology="CYCLIC", agents=4, iterations=4, workflows=64, fixed=1024, dyn=256, out=256, shared_prefix=512,
          gpu_cap=2147483648, bytes_per_token=16384, layers=32, kv_heads_total=8, kv_heads_local=1, head_offset=7,
          head_dim=128, numa_node=N.KVF_NUMA_AUTO, host_slots=10578034688 // 16384 + 4096)
res, traces = {}, {}
for label, extra in (("coalesced", {}), ("per_evict", {"d2h_coalesce": 0}), ("unbatched", {"d2h_unbatched": 1})):
    with Sim(**kw, **extra) as s:
        t0 = time.perf_counter()
        s.run()
        wall = time.perf_counter() - t0
        r = s.result()
        traces[label] = s.trace()
    res[label] = {"wall_s": round(wall, 4), "offload_jobs": r["offload_jobs"], "d2h_launches": r["d2h_batches"],
                  "kernel_launches": r["kernel_launches"], "offload_device_ms": round(r["offload_device_ms"], 2),
                  "fence_wait_ms": round(r["fence_wait_us"] / 1e3, 2),
                  "moved_gbs_wall": round((r["loaded_bytes"] + r["offloaded_bytes"]) / wall / 1e9, 3)}
    print(label, json.dumps(res[label]), flush=True)
# decision records only (job records carry measured device times)
dec = {k: [l for l in v.splitlines() if '"t":"tr"' in l or '"t":"req"' in l] for k, v in traces.items()}
res["decision_traces_identical"] = dec["coalesced"] == dec["per_evict"] == dec["unbatched"]
print(json.dumps(res, indent=1))
json.dump(res, open(out, "w"), indent=1)
