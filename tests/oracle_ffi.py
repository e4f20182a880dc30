"""ctypes bindings to oracle/liboracle.so (the CPU restatement) and golden-fixture loaders.

TEST INFRASTRUCTURE ONLY: the oracle is the checker, never the product path.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
ORACLE_DIR = os.path.join(ROOT, "oracle")
_LIB = None


class Geom(C.Structure):
    _fields_ = [("layers", C.c_uint32), ("kv_heads", C.c_uint32), ("head_dim", C.c_uint32),
                ("head_offset", C.c_uint32)]


class Run(C.Structure):
    _fields_ = [("start", C.c_uint64), ("len", C.c_uint64)]


class Tree(C.Structure):
    _fields_ = [("n", C.c_uint32), ("parent", C.c_void_p), ("status", C.c_void_p), ("lock", C.c_void_p),
                ("rank", C.c_void_p), ("time", C.c_void_p), ("seq", C.c_void_p), ("id", C.c_void_p),
                ("tokens", C.c_void_p), ("backed", C.c_void_p), ("bytes_per_token", C.c_uint64)]


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(ORACLE_DIR, "liboracle.so")
        if not os.path.exists(path):
            subprocess.run(["make", "-C", ORACLE_DIR, "liboracle.so"], check=True, capture_output=True)
        L = C.CDLL(path)
        L.kvfo_mix64.restype = C.c_uint64
        L.kvfo_mix64.argtypes = [C.c_uint64]
        L.kvfo_next_cid.restype = C.c_uint64
        L.kvfo_next_cid.argtypes = [C.c_uint64, C.c_int32]
        L.kvfo_payload_elem.restype = C.c_uint16
        L.kvfo_payload_elem.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32]
        L.kvfo_fill.restype = None
        L.kvfo_fill.argtypes = [C.POINTER(Geom), C.c_void_p, C.c_uint64, C.POINTER(Run), C.c_uint32, C.c_void_p]
        L.kvfo_copy_runs.restype = C.c_uint64
        L.kvfo_copy_runs.argtypes = [C.POINTER(Geom), C.c_void_p, C.c_uint64, C.POINTER(Run), C.c_uint32,
                                     C.c_void_p, C.c_uint64, C.POINTER(Run), C.c_uint32, C.c_int]
        L.kvfo_checksum_runs.restype = C.c_uint64
        L.kvfo_checksum_runs.argtypes = [C.POINTER(Geom), C.c_void_p, C.c_uint64, C.POINTER(Run), C.c_uint32]
        L.kvfo_checksum_expected.restype = C.c_uint64
        L.kvfo_checksum_expected.argtypes = [C.POINTER(Geom), C.c_void_p, C.c_uint64]
        L.kvfo_priority.restype = None
        L.kvfo_priority.argtypes = [C.POINTER(Tree), C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p]
        L.kvfo_evict.restype = C.c_int
        L.kvfo_evict.argtypes = [C.POINTER(Tree), C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int64, C.c_uint64,
                                 C.c_uint64, C.c_void_p, C.c_void_p, C.POINTER(C.c_uint32),
                                 C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.kvfo_now.restype = C.c_double
        _LIB = L
    return _LIB


def load_jsonl(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return [json.loads(l) for l in f if l.strip()]


class TreeArrays:
    """Numpy SoA of one golden snapshot (preorder, index 0 = root)."""

    def __init__(self, case):
        self.parent = np.asarray(case["parent"], dtype=np.int32)
        self.status = np.asarray(case["status"], dtype=np.uint8)
        self.lock = np.asarray(case["lock"], dtype=np.int32)
        self.rank = np.asarray([int(x) for x in case["rank"]], dtype=np.int64)
        self.time = np.asarray(case["time"], dtype=np.float64)
        self.seq = np.asarray(case["seq"], dtype=np.uint64)
        self.id = np.asarray(case["id"], dtype=np.uint64)
        self.tokens = np.asarray(case["tokens"], dtype=np.uint64)
        self.backed = np.asarray(case["backed"], dtype=np.uint8)
        self.bpt = int(case["bpt"])
        self.n = len(self.parent)

    def ctree(self):
        t = Tree()
        t.n = self.n
        for f in ("parent", "status", "lock", "rank", "time", "seq", "id", "tokens", "backed"):
            setattr(t, f, getattr(self, f).ctypes.data)
        t.bytes_per_token = self.bpt
        return t


def oracle_evict(case):
    """Run the C restatement of RadixCache::evict on a golden snapshot.
    Returns (rc, [(id, bytes, immediate)], immediate, pending)."""
    L = lib()
    ta = TreeArrays(case)
    t = ta.ctree()
    idx = np.zeros(ta.n + 1, dtype=np.int32)
    act = np.zeros(ta.n + 1, dtype=np.uint8)
    cnt = C.c_uint32()
    imm = C.c_uint64()
    pend = C.c_uint64()
    rc = L.kvfo_evict(C.byref(t), case["needed"], case["policy"], case["mode"], case["has_floor"], case["floor"],
                      case["cpu_used"], case["cpu_cap"], idx.ctypes.data, act.ctypes.data, C.byref(cnt),
                      C.byref(imm), C.byref(pend))
    victims = []
    for k in range(cnt.value):
        v = int(idx[k])
        victims.append((int(ta.id[v]), int(ta.tokens[v]) * ta.bpt, 0 if act[k] == 0 else 1))
    return rc, victims, imm.value, pend.value


def oracle_priority(case):
    L = lib()
    ta = TreeArrays(case)
    t = ta.ctree()
    b = case["boundaries"]
    bidx = np.asarray([x[0] for x in b], dtype=np.int32)
    cand = np.asarray([int(x[1]) for x in b], dtype=np.int64)
    out = ta.rank.copy()
    L.kvfo_priority(C.byref(t), bidx.ctypes.data, cand.ctypes.data, len(b), out.ctypes.data)
    return out


def runs_array(runs):
    arr = (Run * max(1, len(runs)))()
    for i, (s, l) in enumerate(runs):
        arr[i].start = s
        arr[i].len = l
    return arr


def cids_for(tokens, prev=0x6b766600):
    """Content ids of a token sequence (prefix hash), via the oracle's kvfo_next_cid."""
    L = lib()
    out = np.zeros(len(tokens), dtype=np.uint64)
    c = prev
    for i, t in enumerate(tokens):
        c = L.kvfo_next_cid(c, int(t))
        out[i] = c
    return out
