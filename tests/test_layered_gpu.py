"""Layer-pipelined K1 (kvf_h2d_gather_layered): same bytes as K1, tiles landed
layer by layer, and a compute-stream consumer can start on layer l before later layers land."""
import numpy as np
import pytest

from oracle_ffi import Geom, lib as olib, runs_array as oruns

pytestmark = pytest.mark.gpu
N = pytest.importorskip("paper_2507_07400_b200._native")
torch = pytest.importorskip("torch")
from paper_2507_07400_b200.engine import Engine  # noqa: E402


def test_layered_load_bytes_and_counters():
    L = 8
    with Engine(layers=L, kv_heads_total=8, head_dim=128, gpu_slots=4096, host_slots=4096) as e:
        rng = np.random.default_rng(3)
        ntok = 1500
        cids = rng.integers(0, 2**63, size=ntok, dtype=np.uint64)
        h = e.alloc(N.KVF_TIER_HOST, 700) + e.alloc(N.KVF_TIER_HOST, 800)
        e.fill(N.KVF_TIER_HOST, h, cids)
        d = e.alloc(N.KVF_TIER_DEVICE, 300) + e.alloc(N.KVF_TIER_DEVICE, 1200)
        ready = torch.zeros(L, dtype=torch.int32, device="cuda")
        j, tpl = e.h2d_layered(h, d, ready.data_ptr())
        e.wait(j)
        e.release(j)
        torch.cuda.synchronize()
        assert tpl > 0 and ready.cpu().tolist() == [tpl] * L
        want = np.zeros(ntok * e.token_bytes, dtype=np.uint8)
        olib().kvfo_fill(Geom(L, 8, 128, 0), want.ctypes.data, ntok, oruns([(0, ntok)]), 1, cids.ctypes.data)
        assert np.array_equal(e.read(N.KVF_TIER_DEVICE, d), want)


def test_consumer_starts_before_the_load_finishes():
    L = 32
    with Engine(layers=L, kv_heads_total=8, head_dim=128, gpu_slots=8192, host_slots=8192) as e:
        h = e.alloc(N.KVF_TIER_HOST, 8192)
        d = e.alloc(N.KVF_TIER_DEVICE, 8192)
        ready = torch.zeros(L, dtype=torch.int32, device="cuda")
        for rep in range(2):  # rep 0 also loads the kernels (lazy module loading)
            j, tpl = e.h2d_layered(h, d, ready.data_ptr())
            c0 = e.compute_begin()
            e.compute_wait_layer(ready.data_ptr(), 0, tpl)
            c1 = e.compute_begin()  # layer 0 ready
            e.compute_end(c1)
            e.compute_end(c0)
            first = e.span_ms(j, c1)   # load start -> layer 0 usable
            total = e.elapsed_ms(j)    # load start -> all layers landed
            for x in (j, c0, c1):
                e.release(x)
        assert first < total / 4, (first, total)


def test_engine_owned_counters_recycle_without_reset():
    """layer_ready = NULL: the engine owns the counters (64 slots).  Counters only grow, so a
    slot is reused without a reset and a consumer enqueued late on a recycled slot never
    waits on the next job's progress.  More jobs than slots, each with a per-layer consumer."""
    L = 4
    with Engine(layers=L, kv_heads_total=8, head_dim=128, gpu_slots=2048, host_slots=2048) as e:
        rng = np.random.default_rng(5)
        cids = rng.integers(0, 2**63, size=256, dtype=np.uint64)
        h = e.alloc(N.KVF_TIER_HOST, 256)
        e.fill(N.KVF_TIER_HOST, h, cids)
        d = e.alloc(N.KVF_TIER_DEVICE, 256)
        for k in range(80):
            j, _ = e.h2d_layered(h, d, None)
            c = e.compute_begin()
            for l in range(L):
                e.compute_wait_job_layer(j, l)
            e.compute_end(c)
            e.wait(c)
            e.release(c)
            e.release(j)
        assert e.checksum(N.KVF_TIER_DEVICE, d) == e.checksum(N.KVF_TIER_HOST, h)


def test_engine_owned_counter_slots_are_bounded():
    with Engine(layers=2, kv_heads_total=8, head_dim=128, gpu_slots=1024, host_slots=1024) as e:
        h = e.alloc(N.KVF_TIER_HOST, 8)
        d = e.alloc(N.KVF_TIER_DEVICE, 8)
        jobs = [e.h2d_layered(h, d, None)[0] for _ in range(64)]
        with pytest.raises(N.KvfError) as ei:
            e.h2d_layered(h, d, None)
        assert ei.value.code == N.KVF_E_TOO_LARGE
        for j in jobs:
            e.release(j)
        j, _ = e.h2d_layered(h, d, None)  # a released slot is reusable
        e.release(j)


def test_wait_job_layer_on_a_plain_job_waits_for_the_whole_job():
    with Engine(layers=2, kv_heads_total=8, head_dim=128, gpu_slots=1024, host_slots=1024) as e:
        h = e.alloc(N.KVF_TIER_HOST, 64)
        d = e.alloc(N.KVF_TIER_DEVICE, 64)
        j = e.h2d(h, d)
        c = e.compute_begin()
        e.compute_wait_job_layer(j, 1)
        e.compute_end(c)
        e.wait(c)
        assert e.query(j)
        e.release(c)
        e.release(j)
