"""Thin Python handle over the libkvflow.so C-ABI (include/kvflow.h).

Used by tests, smoke() and bench.py to drive the CUDA engine directly.  The
reference-facing cache-manager API (RadixCache / TierManager / Simulator) is the C++
control plane in include/kvflow/*.hpp; this module is only plumbing.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N


def device_count() -> int:
    n = C.c_int32()
    N.engine_lib().kvf_device_count(C.byref(n))
    return n.value


def device_numa_node(device: int) -> int:
    """NUMA node of the GPU's PCI device (-1 if unknown)."""
    n = C.c_int32()
    N.check(N.engine_lib().kvf_device_numa_node(device, C.byref(n)))
    return n.value


class Engine:
    """One KV-movement engine = one GPU shard (HBM pool + pinned host pool + streams)."""

    def __init__(self, layers=32, kv_heads_total=8, kv_heads_local=None, head_offset=0, head_dim=128,
                 gpu_slots=0, host_slots=0, device=0, pcie_mode=N.KVF_COPY_SM_VEC, pcie_ctas=0, hbm_ctas=0,
                 numa_node=-1):
        L = N.engine_lib()
        self._lib = L
        g = N.Geometry(layers, kv_heads_total, kv_heads_local or kv_heads_total, head_offset, head_dim, 2)
        cfg = N.EngineConfig(device, gpu_slots, host_slots, pcie_ctas, pcie_mode, hbm_ctas, numa_node)
        h = C.c_void_p()
        N.check(L.kvf_engine_create(C.byref(g), C.byref(cfg), C.byref(h)))
        self.h = h
        self.geom = g
        tpb, tb = C.c_uint64(), C.c_uint64()
        N.check(L.kvf_engine_token_bytes(h, C.byref(tpb), C.byref(tb)))
        self.tpb, self.token_bytes = tpb.value, tb.value
        self.gpu_slots, self.host_slots = gpu_slots, host_slots
        self._next_job = 1

    def close(self):
        if self.h:
            self._lib.kvf_engine_destroy(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- pools ---------------------------------------------------------------------
    def alloc(self, tier, tokens, max_runs=4096):
        out = (N.Run * max_runs)()
        n = C.c_uint32()
        N.check(self._lib.kvf_slots_alloc(self.h, tier, tokens, out, max_runs, C.byref(n)))
        return [(out[i].start, out[i].len) for i in range(n.value)]

    def free(self, tier, runs):
        N.check(self._lib.kvf_slots_free(self.h, tier, N.runs_array(runs), len(runs)))

    def free_count(self, tier):
        t, r = C.c_uint64(), C.c_uint64()
        N.check(self._lib.kvf_slots_free_count(self.h, tier, C.byref(t), C.byref(r)))
        return t.value, r.value

    def pool_ptr(self, tier):
        p, s = C.c_void_p(), C.c_uint64()
        N.check(self._lib.kvf_pool_ptr(self.h, tier, C.byref(p), C.byref(s)))
        return p.value, s.value

    def host_pool_array(self):
        """numpy uint8 view of the pinned host pool (for verification only)."""
        p, s = self.pool_ptr(N.KVF_TIER_HOST)
        buf = (C.c_uint8 * (s * self.token_bytes)).from_address(p)
        return np.frombuffer(buf, dtype=np.uint8)

    # ---- jobs ------------------------------------------------------------------------
    def new_job(self):
        j = self._next_job
        self._next_job += 1
        return j

    def h2d(self, host_runs, dev_runs, job=None):
        job = job or self.new_job()
        N.check(self._lib.kvf_h2d_gather(self.h, job, N.runs_array(host_runs), len(host_runs),
                                         N.runs_array(dev_runs), len(dev_runs)))
        return job

    def d2h(self, dev_runs, host_runs, job=None):
        job = job or self.new_job()
        N.check(self._lib.kvf_d2h_scatter(self.h, job, N.runs_array(dev_runs), len(dev_runs),
                                          N.runs_array(host_runs), len(host_runs)))
        return job

    def d2h_batch(self, pairs, jobs=None):
        """One K2 launch for several nodes: pairs = [(dev_runs, host_runs), ...]; returns job ids."""
        jobs = jobs or [self.new_job() for _ in pairs]
        n = len(pairs)
        ids = (C.c_uint64 * max(1, n))(*jobs)
        dc = (C.c_uint32 * max(1, n))(*[len(d) for d, _ in pairs])
        hc = (C.c_uint32 * max(1, n))(*[len(h) for _, h in pairs])
        dev = N.runs_array([r for d, _ in pairs for r in d])
        host = N.runs_array([r for _, h in pairs for r in h])
        N.check(self._lib.kvf_d2h_scatter_batch(self.h, n, ids, dev, dc, host, hc))
        return jobs

    def h2d_layered(self, host_runs, dev_runs, layer_ready_ptr, job=None):
        """Layer-pipelined K1; returns (job, tiles_per_layer)."""
        job = job or self.new_job()
        tpl = C.c_uint32()
        N.check(self._lib.kvf_h2d_gather_layered(self.h, job, N.runs_array(host_runs), len(host_runs),
                                                 N.runs_array(dev_runs), len(dev_runs), layer_ready_ptr,
                                                 C.byref(tpl)))
        return job, tpl.value

    def compute_wait_layer(self, layer_ready_ptr, layer, target):
        N.check(self._lib.kvf_compute_wait_layer(self.h, layer_ready_ptr, layer, target))

    def compute_wait_job(self, job):
        N.check(self._lib.kvf_compute_wait_job(self.h, job))

    def compute_wait_job_layer(self, job, layer):
        N.check(self._lib.kvf_compute_wait_job_layer(self.h, job, layer))

    def compute_spin(self, ns, ctas=1):
        N.check(self._lib.kvf_compute_spin(self.h, int(ns), ctas))

    def compute_begin(self, job=None):
        job = job or self.new_job()
        N.check(self._lib.kvf_compute_job_begin(self.h, job))
        return job

    def compute_end(self, job):
        N.check(self._lib.kvf_compute_job_end(self.h, job))

    def span_ms(self, first_job, last_job):
        ms = C.c_float()
        N.check(self._lib.kvf_job_span_ms(self.h, first_job, last_job, C.byref(ms)))
        return ms.value

    def kv_append(self, layer, runs, k_ptr, v_ptr, ntok, job=None):
        """Write a layer's new K/V rows (device bf16 [ntok][kv_heads_local][128]) into slot runs."""
        job = job or self.new_job()
        N.check(self._lib.kvf_kv_append(self.h, job, layer, N.runs_array(runs), len(runs), k_ptr, v_ptr, ntok))
        return job

    def peer_gather(self, src, src_runs, dst_runs, job=None):
        """Copy a node from another engine's HBM pool (NVLink on another GPU) into dst_runs."""
        job = job or self.new_job()
        N.check(self._lib.kvf_peer_gather(self.h, job, src.h, N.runs_array(src_runs), len(src_runs),
                                          N.runs_array(dst_runs), len(dst_runs)))
        return job

    def dev_gather(self, dev_runs, staging_ptr, job=None):
        job = job or self.new_job()
        N.check(self._lib.kvf_dev_gather(self.h, job, N.runs_array(dev_runs), len(dev_runs), staging_ptr))
        return job

    def dev_scatter(self, staging_ptr, dev_runs, job=None):
        job = job or self.new_job()
        N.check(self._lib.kvf_dev_scatter(self.h, job, staging_ptr, N.runs_array(dev_runs), len(dev_runs)))
        return job

    @staticmethod
    def attend_runs(seq_runs):
        """Pack per-sequence run lists once (a decode step reuses them for every layer)."""
        flat = np.array([r for runs in seq_runs for r in runs] or [(0, 0)], dtype=np.uint64).reshape(-1, 2)
        counts = np.array([len(r) for r in seq_runs], dtype=np.uint32)
        return flat, counts

    def attend(self, layer, group, q_ptr, seq_runs, out_ptr, scale, job=None, chunk=0):
        """K6: decode attention of layer `layer` over each sequence's slot runs, in place
        (q/out: device bf16 [batch][kv_heads_local*group][128]).  Async job on the compute stream.
        seq_runs: list of run lists, or the tuple attend_runs() returned."""
        job = job or self.new_job()
        flat, counts = seq_runs if isinstance(seq_runs, tuple) else self.attend_runs(seq_runs)
        N.check(self._lib.kvf_decode_attend(self.h, job, layer, len(counts), group, q_ptr,
                                            C.cast(flat.ctypes.data, C.POINTER(N.Run)), counts.ctypes.data,
                                            float(scale), out_ptr, chunk))
        return job

    def attend_layers(self, layer0, group, q_ptrs, seq_runs, out_ptrs, scale, job=None, chunk=0):
        """K6 for a decode step's layers layer0 .. layer0+len(q_ptrs)-1 as one chained job
        (q_ptrs[l] / out_ptrs[l]: that layer's device buffers, as for attend())."""
        if len(q_ptrs) != len(out_ptrs):
            raise ValueError("one q and one out pointer per layer")
        job = job or self.new_job()
        flat, counts = seq_runs if isinstance(seq_runs, tuple) else self.attend_runs(seq_runs)
        qa = (C.c_void_p * max(1, len(q_ptrs)))(*q_ptrs)
        oa = (C.c_void_p * max(1, len(out_ptrs)))(*out_ptrs)
        N.check(self._lib.kvf_decode_attend_layers(self.h, job, layer0, len(q_ptrs), len(counts), group, qa,
                                                   C.cast(flat.ctypes.data, C.POINTER(N.Run)), counts.ctypes.data,
                                                   float(scale), oa, chunk))
        return job

    def query(self, job):
        d = C.c_int32()
        N.check(self._lib.kvf_job_query(self.h, job, C.byref(d)))
        return bool(d.value)

    def wait(self, job):
        N.check(self._lib.kvf_job_wait(self.h, job))

    def elapsed_ms(self, job):
        ms = C.c_float()
        N.check(self._lib.kvf_job_elapsed_ms(self.h, job, C.byref(ms)))
        return ms.value

    def release(self, job):
        N.check(self._lib.kvf_job_release(self.h, job))

    def sync(self):
        N.check(self._lib.kvf_sync_all(self.h))

    def set_job_timing(self, stamps):
        """K1/K2 job timing: CUDA timing events (default) or the copy kernels' globaltimer stamps."""
        N.check(self._lib.kvf_engine_set_job_timing(self.h, 1 if stamps else 0))

    def set_copy_mode(self, mode, pcie_ctas=0, hbm_ctas=0):
        N.check(self._lib.kvf_engine_set_copy_mode(self.h, mode, pcie_ctas, hbm_ctas))

    # ---- payload / verification -----------------------------------------------------
    def fill(self, tier, runs, cids):
        cids = np.ascontiguousarray(cids, dtype=np.uint64)
        N.check(self._lib.kvf_fill_payload(self.h, tier, N.runs_array(runs), len(runs), cids.ctypes.data,
                                           len(cids)))

    def checksum(self, tier, runs):
        out = C.c_uint64()
        N.check(self._lib.kvf_checksum(self.h, tier, N.runs_array(runs), len(runs), C.byref(out)))
        return out.value

    def payload_checksum(self, cids):
        cids = np.ascontiguousarray(cids, dtype=np.uint64)
        out = C.c_uint64()
        N.check(self._lib.kvf_payload_checksum(self.h, cids.ctypes.data, len(cids), C.byref(out)))
        return out.value

    def read(self, tier, runs):
        ntok = sum(l for _, l in runs)
        buf = np.zeros(ntok * self.token_bytes, dtype=np.uint8)
        N.check(self._lib.kvf_read_runs(self.h, tier, N.runs_array(runs), len(runs), buf.ctypes.data, buf.nbytes))
        return buf

    def stats(self):
        s = N.Stats()
        N.check(self._lib.kvf_get_stats(self.h, C.byref(s)))
        return {f: (list(getattr(s, f)) if f.startswith("k5_phase") else getattr(s, f)) for f, _ in N.Stats._fields_}

    # ---- decisions ---------------------------------------------------------------------
    def priority(self, parent, bidx, cand):
        parent = np.ascontiguousarray(parent, dtype=np.int32)
        bidx = np.ascontiguousarray(bidx, dtype=np.int32)
        cand = np.ascontiguousarray(cand, dtype=np.int64)
        out = np.zeros(len(parent), dtype=np.int64)
        N.check(self._lib.kvf_priority_propagate(self.h, parent.ctypes.data, len(parent), bidx.ctypes.data,
                                                 cand.ctypes.data, len(bidx), out.ctypes.data))
        return out

    def victims(self, tree, needed, workflow_aware, offload, has_floor=False, floor=0, cpu_used=0, cpu_cap=0):
        """tree: dict of numpy arrays parent/depth/status/lock/rank/time/seq/id/tokens/backed + bpt."""
        arrs = {
            "parent": np.ascontiguousarray(tree["parent"], dtype=np.int32),
            "depth": np.ascontiguousarray(tree["depth"], dtype=np.uint16),
            "status": np.ascontiguousarray(tree["status"], dtype=np.uint8),
            "lock": np.ascontiguousarray(tree["lock"], dtype=np.int32),
            "rank": np.ascontiguousarray(tree["rank"], dtype=np.int64),
            "time": np.ascontiguousarray(tree["time"], dtype=np.float64),
            "seq": np.ascontiguousarray(tree["seq"], dtype=np.uint64),
            "id": np.ascontiguousarray(tree["id"], dtype=np.uint64),
            "tokens": np.ascontiguousarray(tree["tokens"], dtype=np.uint64),
            "backed": np.ascontiguousarray(tree["backed"], dtype=np.uint8),
        }
        n = len(arrs["parent"])
        tv = N.TreeView(n, *(arrs[k].ctypes.data for k in
                             ("parent", "depth", "status", "lock", "rank", "time", "seq", "id", "tokens", "backed")),
                        int(tree["bpt"]))
        req = N.EvictRequest(int(needed), int(bool(workflow_aware)), int(bool(offload)), int(bool(has_floor)),
                             int(floor), int(cpu_used), int(cpu_cap))
        idx = np.zeros(max(1, n), dtype=np.int32)
        act = np.zeros(max(1, n), dtype=np.uint8)
        cnt, imm, pend = C.c_uint32(), C.c_uint64(), C.c_uint64()
        N.check(self._lib.kvf_victim_select(self.h, C.byref(tv), C.byref(req), idx.ctypes.data, act.ctypes.data,
                                            C.byref(cnt), C.byref(imm), C.byref(pend)))
        k = cnt.value
        return idx[:k].copy(), act[:k].copy(), imm.value, pend.value


def depth_from_parent(parent):
    parent = np.asarray(parent)
    d = np.zeros(len(parent), dtype=np.uint16)
    for i in range(1, len(parent)):
        d[i] = d[parent[i]] + 1
    return d


class Tree:
    """A radix tree mirrored in an engine's HBM (kvf_tree, include/kvflow.h): node records in,
    K4 rank changes / K5 victims (as slots) out."""

    def __init__(self, eng, bpt, capacity=0):
        self._lib = eng._lib
        self.eng = eng
        h = C.c_void_p()
        N.check(self._lib.kvf_tree_create(eng.h, int(bpt), int(capacity), C.byref(h)))
        self.h = h
        self.n = 1

    def close(self):
        if self.h:
            self._lib.kvf_tree_destroy(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def hints(self, time_follows_seq):
        N.check(self._lib.kvf_tree_set_hints(self.h, 1 if time_follows_seq else 0))

    def update(self, recs):
        """recs: iterable of dicts slot/parent/lock/status/backed/rank/time/seq/id/tokens."""
        recs = list(recs)
        arr = (N.NodeRec * max(1, len(recs)))()
        for i, r in enumerate(recs):
            arr[i] = N.NodeRec(int(r["slot"]), int(r.get("parent", -1)), int(r.get("lock", 0)),
                               int(r.get("status", 0)), int(r.get("backed", 0)), 0, int(r.get("rank", 0)),
                               float(r.get("time", 0.0)), int(r.get("seq", 0)), int(r.get("id", 0)),
                               int(r.get("tokens", 0)), 0)
            self.n = max(self.n, int(r["slot"]) + 1)
        N.check(self._lib.kvf_tree_update(self.h, arr, len(recs)))

    def load_arrays(self, a, slots=None):
        """Whole-tree records from SoA arrays (index = slot unless `slots` maps them)."""
        n = len(a["parent"])
        sl = list(range(n)) if slots is None else list(slots)
        self.update({"slot": sl[i], "parent": (sl[a["parent"][i]] if a["parent"][i] >= 0 else -1),
                     "lock": a["lock"][i], "status": a["status"][i], "backed": a["backed"][i], "rank": a["rank"][i],
                     "time": a["time"][i], "seq": a["seq"][i], "id": a["id"][i], "tokens": a["tokens"][i]}
                    for i in range(n))

    def priorities(self, bslot, cand):
        b = np.ascontiguousarray(bslot, dtype=np.uint32)
        c = np.ascontiguousarray(cand, dtype=np.int64)
        N.check(self._lib.kvf_tree_priorities(self.h, b.ctypes.data_as(C.POINTER(C.c_uint32)),
                                              c.ctypes.data_as(C.POINTER(C.c_int64)), len(b)))

    def rank_changes(self):
        cap = max(1, self.n)
        s = np.zeros(cap, dtype=np.uint32)
        r = np.zeros(cap, dtype=np.int64)
        k = C.c_uint32()
        N.check(self._lib.kvf_tree_rank_changes(self.h, s.ctypes.data_as(C.POINTER(C.c_uint32)),
                                                r.ctypes.data_as(C.POINTER(C.c_int64)), cap, C.byref(k)))
        return dict(zip(s[:k.value].tolist(), r[:k.value].tolist()))

    def victims(self, needed, workflow_aware, offload, has_floor=False, floor=0, cpu_used=0, cpu_cap=0):
        req = N.EvictRequest(int(needed), int(bool(workflow_aware)), int(bool(offload)), int(bool(has_floor)),
                             int(floor), int(cpu_used), int(cpu_cap))
        cap = max(1, self.n)
        s = np.zeros(cap, dtype=np.uint32)
        a = np.zeros(cap, dtype=np.uint8)
        cnt, imm, pend = C.c_uint32(), C.c_uint64(), C.c_uint64()
        N.check(self._lib.kvf_tree_victims(self.h, C.byref(req), s.ctypes.data_as(C.POINTER(C.c_uint32)),
                                           a.ctypes.data_as(C.POINTER(C.c_uint8)), cap, C.byref(cnt), C.byref(imm),
                                           C.byref(pend)))
        k = cnt.value
        return s[:k].copy(), a[:k].copy(), imm.value, pend.value


def decider_hold(eng, hold):
    N.check(eng._lib.kvf_decider_hold(eng.h, 1 if hold else 0))


def decider_running(eng):
    r = C.c_int32()
    N.check(eng._lib.kvf_decider_running(eng.h, C.byref(r)))
    return bool(r.value)
