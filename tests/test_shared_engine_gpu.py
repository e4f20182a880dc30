"""One engine shared by a fence thread and a decision thread.

A 1 GiB K1 prefetch is being waited on (kvf_job_wait -> cudaEventSynchronize, ~20 ms) by one
host thread while another thread issues K4 / K5 decisions on the SAME engine.  The fence runs
outside the engine lock, so the decision calls go through at their normal latency instead of
queueing behind the wait; results are checked against the reference's vectors."""
import ctypes as C
import statistics
import threading
import time

import numpy as np
import pytest

from conftest import UNDER_SANITIZER

from oracle_ffi import load_jsonl

pytestmark = pytest.mark.gpu
N = pytest.importorskip("paper_2507_07400_b200._native")
from paper_2507_07400_b200.engine import Engine  # noqa: E402


def test_decisions_do_not_queue_behind_a_fence():
    prio = [c for c in load_jsonl("prio.jsonl") if len(c["parent"]) <= 64][:20]
    assert prio
    with Engine(layers=32, kv_heads_total=8, gpu_slots=8192 + 64, host_slots=8192) as e:
        host = e.alloc(N.KVF_TIER_HOST, 8192)
        dev = e.alloc(N.KVF_TIER_DEVICE, 8192)
        e.fill(N.KVF_TIER_HOST, host, np.arange(8192, dtype=np.uint64))
        e.sync()
        L = e._lib
        cases = []
        for c in prio:
            parent = np.ascontiguousarray(c["parent"], dtype=np.int32)
            bidx = np.ascontiguousarray([x[0] for x in c["boundaries"]], dtype=np.int32)
            cand = np.ascontiguousarray([int(x[1]) for x in c["boundaries"]], dtype=np.int64)
            out = np.zeros(len(parent), dtype=np.int64)
            cases.append((parent, bidx, cand, out, np.asarray([int(x) for x in c["rank"]], dtype=np.int64)))
        in_wait = threading.Event()
        stop = threading.Event()
        errors, lat_waiting, waits = [], [], []

        def fencer():
            try:
                for _ in range(12):
                    j = e.h2d(host, dev)
                    in_wait.set()
                    t0 = time.perf_counter()
                    e.wait(j)
                    waits.append(time.perf_counter() - t0)
                    in_wait.clear()
                    e.release(j)
            except Exception as ex:  # pragma: no cover
                errors.append(repr(ex))
            finally:
                in_wait.clear()
                stop.set()

        def decider():
            k = 0
            try:
                while not stop.is_set():
                    parent, bidx, cand, out, want = cases[k % len(cases)]
                    k += 1
                    during = in_wait.is_set()
                    t0 = time.perf_counter()
                    rc = L.kvf_priority_propagate(e.h, parent.ctypes.data, len(parent), bidx.ctypes.data,
                                                  cand.ctypes.data, len(bidx), out.ctypes.data)
                    dt = time.perf_counter() - t0
                    if rc:
                        errors.append(f"K4 rc {rc}")
                        return
                    if not np.array_equal(out[1:], want[1:]):
                        errors.append("K4 ranks differ from the reference")
                        return
                    if during and in_wait.is_set():
                        lat_waiting.append(dt * 1e6)
            except Exception as ex:  # pragma: no cover
                errors.append(repr(ex))

        threads = [threading.Thread(target=fencer), threading.Thread(target=decider)]
        for t in threads:
            t.start()
        for t in threads:
            t.join(timeout=300)
        assert not errors, errors
        if UNDER_SANITIZER:
            return
        assert statistics.median(waits) > 5e-3  # the fence really blocked for a 1 GiB load
        assert len(lat_waiting) > 100, len(lat_waiting)
        med = statistics.median(lat_waiting)
        # before the fix every call issued during the wait queued for the rest of the ~20 ms fence
        assert med < 30.0, f"median K4 call {med:.1f} us while a K1 fence is held"
        assert max(lat_waiting) < 5000.0
