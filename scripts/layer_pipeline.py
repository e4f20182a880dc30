"""Reactive load with a layer-pipelined consumer vs the reference's gate model.

Scenario (C2 reactive reload): a 8192-token fixed node (1 GiB, 32 layers) comes
back from the host while the request's prefill of its 64 uncached tokens runs layer by
layer (h100-qwen32b profile: prefill_time(64) = 6.84 ms, i.e. 0.214 ms per layer).
  serial:      load everything, then prefill                  (what a plain fence gives)
  pipelined:   layer l's prefill waits only for layer l        (kvf_h2d_gather_layered)
  model gate:  max(0, load - 0.5 * prefill)                    (scheduler.cpp:281)
Exposed stall = total - prefill.  Prints one JSON object.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2507_07400_b200 import _native as N  # noqa: E402
from paper_2507_07400_b200.engine import Engine  # noqa: E402


def main():
    L, ntok, dyn = 32, 8192, 64
    prefill_s = 60e-6 * dyn + 3e-3
    per_layer_ns = int(prefill_s / L * 1e9)
    e = Engine(layers=L, kv_heads_total=8, head_dim=128, gpu_slots=ntok, host_slots=ntok)
    h = e.alloc(N.KVF_TIER_HOST, ntok)
    d = e.alloc(N.KVF_TIER_DEVICE, ntok)
    ready = torch.zeros(L, dtype=torch.int32, device="cuda")
    out = {}
    for mode in ("serial", "pipelined"):
        best = None
        for _ in range(4):
            if mode == "serial":  # a fence on the whole node, then the prefill (device-side wait)
                j, tpl = e.h2d_layered(h, d, ready.data_ptr())
                c = e.compute_begin()
                for l in range(L):
                    e.compute_wait_layer(ready.data_ptr(), l, tpl)
                for _l in range(L):
                    e.compute_spin(per_layer_ns)
                e.compute_end(c)
                total = e.span_ms(j, c)
                first = e.elapsed_ms(j)
            else:
                j, tpl = e.h2d_layered(h, d, ready.data_ptr())
                c = e.compute_begin()
                m0 = None
                for l in range(L):
                    e.compute_wait_layer(ready.data_ptr(), l, tpl)
                    if l == 0:
                        m0 = e.compute_begin()
                        e.compute_end(m0)
                    e.compute_spin(per_layer_ns)
                e.compute_end(c)
                total = e.span_ms(j, c)
                first = e.span_ms(j, m0)
                e.release(m0)
            load = e.elapsed_ms(j)
            e.release(j)
            e.release(c)
            if best is None or total < best["total_ms"]:
                best = {"total_ms": total, "load_ms": load, "first_layer_ready_ms": first}
        best["exposed_stall_ms"] = best["total_ms"] - prefill_s * 1e3
        out[mode] = {k: round(v, 3) for k, v in best.items()}
    load_ms = out["serial"]["load_ms"]
    out["model_gate_ms"] = round(max(0.0, load_ms - 0.5 * prefill_s * 1e3), 3)
    out["prefill_ms"] = round(prefill_s * 1e3, 3)
    out["bytes"] = ntok * e.token_bytes
    e.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
