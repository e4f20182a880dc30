"""ctypes bindings to the in-tree native libraries.

  libkvflow.so       -- the CUDA engine C-ABI (include/kvflow.h)
  libkvflow_host.so  -- the C++ control plane (include/kvflow/*.hpp)
  libkvflow_driver.so-- harness over it: the synthetic workload generator and the lockstep
                        driver's C-ABI (include/kvflow_host.h) used by tests, smoke(), bench.py

There is no fallback: if a library is missing this raises, and every engine entry point
returns KVF_E_NO_DEVICE when no CUDA device is present.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
ENGINE_SO = os.path.join(PKG, "libkvflow.so")
HOST_SO = os.path.join(PKG, "libkvflow_host.so")
DRIVER_SO = os.path.join(PKG, "libkvflow_driver.so")

KVF_OK = 0
KVF_TIER_DEVICE, KVF_TIER_HOST = 0, 1
KVF_COPY_SM_VEC, KVF_COPY_SM_BULK, KVF_COPY_CE = 0, 1, 2
KVF_NUMA_AUTO = -2
KVF_E_INVALID_ARG, KVF_E_OUT_OF_HOST_SLOTS, KVF_E_NO_DEVICE, KVF_E_UNKNOWN_JOB, KVF_E_TOO_LARGE = 101, 102, 103, 104, 105


class KvfError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"kvflow error {code}: {msg}")
        self.code = code


class Geometry(C.Structure):
    _fields_ = [("layers", C.c_uint32), ("kv_heads_total", C.c_uint32), ("kv_heads_local", C.c_uint32),
                ("head_offset", C.c_uint32), ("head_dim", C.c_uint32), ("dtype_bytes", C.c_uint32)]


class EngineConfig(C.Structure):
    _fields_ = [("device", C.c_int32), ("gpu_slots", C.c_uint64), ("host_slots", C.c_uint64),
                ("pcie_ctas", C.c_uint32), ("pcie_mode", C.c_uint32), ("hbm_ctas", C.c_uint32),
                ("host_numa_node", C.c_int32)]


class Run(C.Structure):
    _fields_ = [("start", C.c_uint64), ("len", C.c_uint64)]


class TreeView(C.Structure):
    _fields_ = [("n", C.c_uint32), ("parent", C.c_void_p), ("depth", C.c_void_p), ("status", C.c_void_p),
                ("lock", C.c_void_p), ("rank", C.c_void_p), ("time", C.c_void_p), ("seq", C.c_void_p),
                ("id", C.c_void_p), ("tokens", C.c_void_p), ("backed", C.c_void_p),
                ("bytes_per_token", C.c_uint64)]


class EvictRequest(C.Structure):
    _fields_ = [("needed", C.c_uint64), ("workflow_aware", C.c_int32), ("offload_mode", C.c_int32),
                ("has_floor", C.c_int32), ("floor", C.c_int64), ("cpu_used", C.c_uint64),
                ("cpu_capacity", C.c_uint64)]


class Stats(C.Structure):
    _fields_ = [("kernel_launches", C.c_uint64), ("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64),
                ("dev_bytes", C.c_uint64), ("h2d_jobs", C.c_uint64), ("d2h_jobs", C.c_uint64),
                ("dev_jobs", C.c_uint64), ("decisions", C.c_uint64), ("decision_kernel_ms", C.c_double),
                ("decision_call_us", C.c_double), ("k5_phase_ns", C.c_double * 5),
                ("k5_phase_cycles", C.c_double * 5), ("stale_errors", C.c_uint64), ("attend_calls", C.c_uint64),
                ("attend_bytes", C.c_uint64), ("resident_served", C.c_uint64), ("oneshot_served", C.c_uint64),
                ("resident_launches", C.c_uint64), ("mirror_records", C.c_uint64)]


class NodeRec(C.Structure):  # kvf_node_rec
    _fields_ = [("slot", C.c_uint32), ("parent", C.c_int32), ("lock", C.c_int32), ("status", C.c_uint8),
                ("backed", C.c_uint8), ("flags", C.c_uint16), ("rank", C.c_int64), ("time", C.c_double),
                ("seq", C.c_uint64), ("id", C.c_uint64), ("tokens", C.c_uint64), ("pad1", C.c_uint64)]


# every symbol include/kvflow.h declares, with its ctypes signature
_ENGINE_SIGS = {
    "kvf_last_error": (C.c_char_p, []),
    "kvf_version": (C.c_char_p, []),
    "kvf_device_count": (C.c_int, [C.POINTER(C.c_int32)]),
    "kvf_device_numa_node": (C.c_int, [C.c_int32, C.POINTER(C.c_int32)]),
    "kvf_engine_create": (C.c_int, [C.POINTER(Geometry), C.POINTER(EngineConfig), C.POINTER(C.c_void_p)]),
    "kvf_engine_destroy": (C.c_int, [C.c_void_p]),
    "kvf_engine_token_bytes": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "kvf_engine_set_copy_mode": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32]),
    "kvf_slots_alloc": (C.c_int, [C.c_void_p, C.c_int32, C.c_uint64, C.POINTER(Run), C.c_uint32,
                                  C.POINTER(C.c_uint32)]),
    "kvf_slots_free": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(Run), C.c_uint32]),
    "kvf_slots_free_count": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "kvf_pool_ptr": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_void_p), C.POINTER(C.c_uint64)]),
    "kvf_h2d_gather": (C.c_int, [C.c_void_p, C.c_uint64, C.POINTER(Run), C.c_uint32, C.POINTER(Run), C.c_uint32]),
    "kvf_d2h_scatter": (C.c_int, [C.c_void_p, C.c_uint64, C.POINTER(Run), C.c_uint32, C.POINTER(Run), C.c_uint32]),
    "kvf_d2h_scatter_batch": (C.c_int, [C.c_void_p, C.c_uint32, C.POINTER(C.c_uint64), C.POINTER(Run),
                                        C.POINTER(C.c_uint32), C.POINTER(Run), C.POINTER(C.c_uint32)]),
    "kvf_kv_append": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint32, C.POINTER(Run), C.c_uint32, C.c_void_p,
                                C.c_void_p, C.c_uint64]),
    "kvf_peer_gather": (C.c_int, [C.c_void_p, C.c_uint64, C.c_void_p, C.POINTER(Run), C.c_uint32, C.POINTER(Run),
                                  C.c_uint32]),
    "kvf_dev_gather": (C.c_int, [C.c_void_p, C.c_uint64, C.POINTER(Run), C.c_uint32, C.c_void_p]),
    "kvf_dev_scatter": (C.c_int, [C.c_void_p, C.c_uint64, C.c_void_p, C.POINTER(Run), C.c_uint32]),
    "kvf_h2d_gather_layered": (C.c_int, [C.c_void_p, C.c_uint64, C.POINTER(Run), C.c_uint32, C.POINTER(Run), C.c_uint32,
                                         C.c_void_p, C.POINTER(C.c_uint32)]),
    "kvf_compute_wait_layer": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint32]),
    "kvf_compute_wait_job": (C.c_int, [C.c_void_p, C.c_uint64]),
    "kvf_compute_wait_job_layer": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint32]),
    "kvf_compute_spin": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint32]),
    "kvf_compute_job_begin": (C.c_int, [C.c_void_p, C.c_uint64]),
    "kvf_compute_job_end": (C.c_int, [C.c_void_p, C.c_uint64]),
    "kvf_job_span_ms": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.POINTER(C.c_float)]),
    "kvf_job_query": (C.c_int, [C.c_void_p, C.c_uint64, C.POINTER(C.c_int32)]),
    "kvf_job_wait": (C.c_int, [C.c_void_p, C.c_uint64]),
    "kvf_job_elapsed_ms": (C.c_int, [C.c_void_p, C.c_uint64, C.POINTER(C.c_float)]),
    "kvf_job_release": (C.c_int, [C.c_void_p, C.c_uint64]),
    "kvf_sync_all": (C.c_int, [C.c_void_p]),
    "kvf_priority_propagate": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p, C.c_uint32,
                                         C.c_void_p]),
    "kvf_victim_select": (C.c_int, [C.c_void_p, C.POINTER(TreeView), C.POINTER(EvictRequest), C.c_void_p,
                                    C.c_void_p, C.POINTER(C.c_uint32), C.POINTER(C.c_uint64),
                                    C.POINTER(C.c_uint64)]),
    "kvf_decode_attend": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p,
                                    C.POINTER(Run), C.c_void_p, C.c_float, C.c_void_p, C.c_uint32]),
    "kvf_decode_attend_layers": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                           C.c_void_p, C.POINTER(Run), C.c_void_p, C.c_float, C.c_void_p, C.c_uint32]),
    "kvf_fill_payload": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(Run), C.c_uint32, C.c_void_p, C.c_uint64]),
    "kvf_checksum": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(Run), C.c_uint32, C.POINTER(C.c_uint64)]),
    "kvf_payload_checksum": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64)]),
    "kvf_read_runs": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(Run), C.c_uint32, C.c_void_p, C.c_uint64]),
    "kvf_get_stats": (C.c_int, [C.c_void_p, C.POINTER(Stats)]),
    "kvf_engine_set_job_timing": (C.c_int, [C.c_void_p, C.c_uint32]),
    "kvf_tree_create": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint32, C.POINTER(C.c_void_p)]),
    "kvf_tree_destroy": (C.c_int, [C.c_void_p]),
    "kvf_tree_set_hints": (C.c_int, [C.c_void_p, C.c_uint32]),
    "kvf_tree_update": (C.c_int, [C.c_void_p, C.POINTER(NodeRec), C.c_uint32]),
    "kvf_tree_priorities": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint32), C.POINTER(C.c_int64), C.c_uint32]),
    "kvf_tree_stage_priorities": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint32), C.POINTER(C.c_int64), C.c_uint32]),
    "kvf_tree_rank_changes": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint32), C.POINTER(C.c_int64), C.c_uint32,
                                        C.POINTER(C.c_uint32)]),
    "kvf_tree_victims": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_uint32), C.POINTER(C.c_uint8), C.c_uint32,
                                   C.POINTER(C.c_uint32), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "kvf_decider_hold": (C.c_int, [C.c_void_p, C.c_int32]),
    "kvf_decider_running": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32)]),
}

_engine = None
_host = None


def engine_lib():
    """Load libkvflow.so (in-tree).  Raises if it was not built."""
    global _engine
    if _engine is None:
        if not os.path.exists(ENGINE_SO):
            raise ImportError(f"{ENGINE_SO} missing: run __graft_entry__.build() (no CPU fallback exists)")
        lib = C.CDLL(ENGINE_SO)
        for name, (res, args) in _ENGINE_SIGS.items():
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        _engine = lib
    return _engine


def host_lib():
    """Load the lockstep driver's C-ABI (libkvflow_driver.so over libkvflow_host.so, the C++
    control plane).  Raises if they were not built."""
    global _host
    if _host is None:
        engine_lib()  # dependencies, loaded first so the loader resolves them in-tree
        for so in (HOST_SO, DRIVER_SO):
            if not os.path.exists(so):
                raise ImportError(f"{so} missing: run __graft_entry__.build()")
        C.CDLL(HOST_SO, mode=C.RTLD_GLOBAL)
        _host = C.CDLL(DRIVER_SO)
        from . import _host_sigs
        _host_sigs.bind(_host)
    return _host


def check(rc, lib=None):
    if rc != KVF_OK:
        L = lib or engine_lib()
        raise KvfError(rc, L.kvf_last_error().decode(errors="replace"))
    return rc


def runs_array(runs):
    arr = (Run * max(1, len(runs)))()
    for i, (s, l) in enumerate(runs):
        arr[i].start = int(s)
        arr[i].len = int(l)
    return arr
