"""Run the C++ lockstep workflow driver (kvf::Simulator) on a GPU engine shard.

    res, trace = run_sim(fixed=8192, gpu_cap=3271557120)

Config keys are the fields of kvfh_sim_config (include/kvflow_host.h); topology and
policy also accept the reference's names ("CYCLIC", "KVFLOW", ...).
"""
from __future__ import annotations

import ctypes as C
import json

from . import _native as N
from ._host_sigs import SimConfig, SimResult

TOPOLOGIES = ["SEQUENTIAL", "CYCLIC", "BRANCH_MAX", "BRANCH_MIN", "PEER_STYLE"]
POLICIES = ["LRU_GPU_ONLY", "LRU_REACTIVE_HICACHE", "KVFLOW"]
PROFILES = ["h100-qwen32b", "a10g-llama8b", "micro"]


def geometry_for_bpt(bpt):
    """A KV geometry whose per-token bytes equal the ledger's bytes_per_token:
    Llama-3 shapes when they fit (8 KV heads x 128 dims bf16 per layer), else a tiny
    1-layer geometry (the reference test suites use 16 B/token)."""
    per_head_layer = 2 * 128 * 2
    if bpt % (per_head_layer) == 0:
        units = bpt // per_head_layer  # layers * local heads
        for heads in (8, 4, 2, 1):
            if units % heads == 0:
                return dict(layers=units // heads, kv_heads_total=heads, kv_heads_local=heads, head_dim=128)
    if bpt % 8 == 0:  # 1 layer, 1 head, D = bpt / 4
        return dict(layers=1, kv_heads_total=1, kv_heads_local=1, head_dim=bpt // 4)
    raise ValueError(f"bytes_per_token {bpt} has no bf16 geometry")


def make_config(**kw):
    L = N.host_lib()
    c = SimConfig()
    L.kvfh_default_config(C.byref(c))
    if "topology" in kw and isinstance(kw["topology"], str):
        kw["topology"] = TOPOLOGIES.index(kw["topology"])
    if "policy" in kw and isinstance(kw["policy"], str):
        kw["policy"] = POLICIES.index(kw["policy"])
    if "profile" in kw and isinstance(kw["profile"], str):
        kw["profile"] = PROFILES.index(kw["profile"])
    if "bytes_per_token" in kw and "layers" not in kw:
        kw = {**geometry_for_bpt(kw["bytes_per_token"]), **kw}
    for k, v in kw.items():
        if not hasattr(c, k):
            raise KeyError(k)
        setattr(c, k, v)
    return c


class Sim:
    def __init__(self, **kw):
        self._L = N.host_lib()
        self.cfg = make_config(**kw)
        h = C.c_void_p()
        N.check(self._L.kvfh_sim_create(C.byref(self.cfg), C.byref(h)), _HostErr(self._L))
        self.h = h

    def run(self):
        N.check(self._L.kvfh_sim_run(self.h), _HostErr(self._L))
        return self

    def result(self):
        r = SimResult()
        N.check(self._L.kvfh_sim_result_get(self.h, C.byref(r)), _HostErr(self._L))
        return {f: getattr(r, f) for f, _ in SimResult._fields_}

    def trace(self):
        n = C.c_size_t()
        self._L.kvfh_sim_trace(self.h, None, 0, C.byref(n))
        buf = C.create_string_buffer(n.value + 1)
        self._L.kvfh_sim_trace(self.h, buf, n.value, C.byref(n))
        return [json.loads(l) for l in buf.raw[: n.value].decode().splitlines() if l]

    def verify_resident(self):
        k, bad = C.c_uint64(), C.c_uint64()
        N.check(self._L.kvfh_sim_verify_resident(self.h, C.byref(k), C.byref(bad)), _HostErr(self._L))
        return k.value, bad.value

    def close(self):
        if self.h:
            self._L.kvfh_sim_destroy(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


class _HostErr:
    """adapter so N.check reads kvfh_last_error"""

    def __init__(self, L):
        self._L = L

    def kvf_last_error(self):
        return self._L.kvfh_last_error()


def run_sim(**kw):
    with Sim(**kw) as s:
        s.run()
        return s.result(), s.trace()
