"""ctypes signatures of include/kvflow_host.h."""
import ctypes as C


class SimConfig(C.Structure):
    _fields_ = [
        ("topology", C.c_int32), ("agents", C.c_uint32), ("iterations", C.c_uint32), ("warmup", C.c_uint32),
        ("workflows", C.c_uint32), ("fixed", C.c_uint64), ("dyn", C.c_uint64), ("out", C.c_uint64),
        ("shared_prefix", C.c_uint64), ("vocab", C.c_uint64), ("policy", C.c_int32), ("max_running", C.c_uint32),
        ("max_prefetch", C.c_uint32), ("prefetch", C.c_int32), ("eviction", C.c_int32),
        ("heuristic_boundary", C.c_int32), ("overlap_fraction", C.c_double), ("profile", C.c_int32),
        ("bytes_per_token", C.c_uint64), ("gpu_cap", C.c_uint64), ("cpu_cap", C.c_uint64), ("seed", C.c_uint64),
        ("layers", C.c_uint32), ("kv_heads_total", C.c_uint32), ("kv_heads_local", C.c_uint32),
        ("head_offset", C.c_uint32), ("head_dim", C.c_uint32), ("device", C.c_int32), ("host_slots", C.c_uint64),
        ("pcie_mode", C.c_uint32), ("pcie_ctas", C.c_uint32), ("numa_node", C.c_int32), ("audit", C.c_int32),
        ("verify_loads", C.c_int32), ("timing", C.c_int32), ("clock", C.c_int32), ("compute_scale", C.c_double),
        ("compute_ctas", C.c_uint32), ("prefetch_retry", C.c_int32), ("layered_gate", C.c_int32),
        ("d2h_unbatched", C.c_int32), ("d2h_coalesce", C.c_int32),
    ]


class SimResult(C.Structure):
    _fields_ = [
        ("makespan", C.c_double), ("end_of_run", C.c_double), ("loaded_bytes", C.c_uint64),
        ("offloaded_bytes", C.c_uint64), ("wasted_prefetch_bytes", C.c_uint64), ("events", C.c_uint64),
        ("nodes", C.c_uint64), ("requests", C.c_uint64), ("wall_s", C.c_double), ("arrivals", C.c_uint64),
        ("decision_us_total", C.c_double), ("decision_us_max", C.c_double), ("prefetch_jobs", C.c_uint64),
        ("reactive_jobs", C.c_uint64), ("offload_jobs", C.c_uint64), ("prefetch_bytes", C.c_uint64),
        ("reactive_bytes", C.c_uint64), ("offload_bytes", C.c_uint64), ("prefetch_device_ms", C.c_double),
        ("reactive_device_ms", C.c_double), ("offload_device_ms", C.c_double), ("fence_wait_us", C.c_double),
        ("priority_calls", C.c_uint64), ("evict_calls", C.c_uint64), ("priority_us", C.c_double),
        ("evict_us", C.c_double), ("kernel_launches", C.c_uint64), ("verified_loads", C.c_uint64),
        ("verify_failures", C.c_uint64), ("audits", C.c_uint64), ("d2h_batches", C.c_uint64),
        ("stall_total_s", C.c_double),
        ("stalled_requests", C.c_uint64), ("measured_requests", C.c_uint64),
        ("engine_decisions", C.c_uint64), ("engine_decision_kernel_ms", C.c_double),
        ("engine_decision_call_us", C.c_double),
        ("resident_served", C.c_uint64), ("oneshot_served", C.c_uint64), ("resident_launches", C.c_uint64),
        ("mirror_records", C.c_uint64), ("k4_join_us", C.c_double), ("k5_us", C.c_double), ("apply_us", C.c_double),
        ("issue_us", C.c_double), ("decision_issue_us", C.c_double),
        ("priority_issued", C.c_uint64),
    ]


SIGS = {
    "kvfh_last_error": (C.c_char_p, []),
    "kvfh_default_config": (None, [C.POINTER(SimConfig)]),
    "kvfh_sim_create": (C.c_int, [C.POINTER(SimConfig), C.POINTER(C.c_void_p)]),
    "kvfh_sim_run": (C.c_int, [C.c_void_p]),
    "kvfh_sim_result_get": (C.c_int, [C.c_void_p, C.POINTER(SimResult)]),
    "kvfh_sim_trace": (C.c_int, [C.c_void_p, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "kvfh_sim_verify_resident": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "kvfh_sim_destroy": (C.c_int, [C.c_void_p]),
}


def bind(lib):
    for name, (res, args) in SIGS.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
