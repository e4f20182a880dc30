"""Parity of the CUDA engine (libkvflow.so, via its C-ABI) against the CPU oracle.

Bytes: bit-exact against the oracle's payload restatement and memcpy restatement over
the same slot-run tables (K1 H2D gather, K2 D2H scatter, K3 HBM gather/scatter), in all
copy back-ends.  Decisions: K4/K5 equal to the golden vectors of the UNMODIFIED reference.
"""
import numpy as np
import pytest

from oracle_ffi import Geom, lib as olib, load_jsonl, runs_array as oruns, TreeArrays

pytestmark = pytest.mark.gpu

N = pytest.importorskip("paper_2507_07400_b200._native")
from paper_2507_07400_b200.engine import Engine, depth_from_parent  # noqa: E402

MODES = [N.KVF_COPY_SM_VEC, N.KVF_COPY_SM_BULK, N.KVF_COPY_CE]


def oracle_geom(e):
    g = e.geom
    return Geom(g.layers, g.kv_heads_local, g.head_dim, g.head_offset)


def expected_bytes(e, cids):
    """Logical [plane][token][bytes] image of a node whose tokens have content ids cids."""
    L = olib()
    n = len(cids)
    buf = np.zeros(n * e.token_bytes, dtype=np.uint8)
    L.kvfo_fill(oracle_geom(e), buf.ctypes.data, n, oruns([(0, n)]), 1,
                np.ascontiguousarray(cids, dtype=np.uint64).ctypes.data)
    return buf


def rand_cids(rng, n):
    return rng.integers(0, 2**63, size=n, dtype=np.uint64)


def fragment(e, tier, ntok, rng, pieces=5):
    """Allocate ntok slots as several runs by allocating/freeing a checkerboard first."""
    blockers = []
    runs = []
    left = ntok
    while left > 0:
        take = min(left, int(rng.integers(1, max(2, ntok // pieces + 2))))
        runs += e.alloc(tier, take)
        blockers += e.alloc(tier, int(rng.integers(1, 4)))
        left -= take
    e.free(tier, blockers)
    return runs


@pytest.fixture(scope="module")
def eng():
    e = Engine(layers=4, kv_heads_total=8, head_dim=128, gpu_slots=8192, host_slots=16384)
    yield e
    e.close()


def test_fill_matches_oracle_payload(eng):
    rng = np.random.default_rng(1)
    cids = rand_cids(rng, 777)
    for tier in (N.KVF_TIER_DEVICE, N.KVF_TIER_HOST):
        runs = fragment(eng, tier, len(cids), rng)
        assert len(runs) > 1
        eng.fill(tier, runs, cids)
        got = eng.read(tier, runs)
        assert np.array_equal(got, expected_bytes(eng, cids))
        L = olib()
        want = L.kvfo_checksum_expected(oracle_geom(eng), cids.ctypes.data, len(cids))
        assert eng.checksum(tier, runs) == want
        eng.free(tier, runs)


@pytest.mark.parametrize("mode", MODES)
def test_h2d_d2h_roundtrip_bit_exact(eng, mode):
    """K2 then K1 through fragmented runs on both tiers: bytes equal the oracle's memcpy."""
    rng = np.random.default_rng(2 + mode)
    eng.set_copy_mode(mode)
    L = olib()
    for ntok in (1, 7, 300, 2048):
        cids = rand_cids(rng, ntok)
        d0 = fragment(eng, N.KVF_TIER_DEVICE, ntok, rng)
        eng.fill(N.KVF_TIER_DEVICE, d0, cids)
        h = fragment(eng, N.KVF_TIER_HOST, ntok, rng)
        j = eng.d2h(d0, h)
        eng.wait(j)
        eng.release(j)
        # host pool bytes == oracle memcpy of the device image into the same host runs
        host = eng.host_pool_array()
        want_host = np.zeros_like(host)
        img = expected_bytes(eng, cids)
        L.kvfo_copy_runs(oracle_geom(eng), img.ctypes.data, ntok, oruns([(0, ntok)]), 1, want_host.ctypes.data,
                         eng.host_slots, oruns(h), len(h), 1)
        for s, l in h:  # compare only the node's bytes, plane by plane
            for p in range(eng.geom.layers * 2):
                a = (p * eng.host_slots + s) * eng.tpb
                b = a + l * eng.tpb
                assert np.array_equal(host[a:b], want_host[a:b])
        d1 = fragment(eng, N.KVF_TIER_DEVICE, ntok, rng)
        j = eng.h2d(h, d1)
        eng.wait(j)
        assert eng.elapsed_ms(j) > 0
        eng.release(j)
        assert np.array_equal(eng.read(N.KVF_TIER_DEVICE, d1), img)
        for t, r in ((N.KVF_TIER_DEVICE, d0), (N.KVF_TIER_HOST, h), (N.KVF_TIER_DEVICE, d1)):
            eng.free(t, r)
    eng.set_copy_mode(N.KVF_COPY_SM_VEC)


def test_many_pieces_split_launches(eng):
    """> 48 pieces per job: the engine splits launches; bytes still exact."""
    rng = np.random.default_rng(5)
    ntok = 400
    cids = rand_cids(rng, ntok)
    h = fragment(eng, N.KVF_TIER_HOST, ntok, rng, pieces=150)
    assert len(h) > 48
    eng.fill(N.KVF_TIER_HOST, h, cids)
    d = fragment(eng, N.KVF_TIER_DEVICE, ntok, rng, pieces=90)
    for mode in MODES:
        eng.set_copy_mode(mode)
        j = eng.h2d(h, d)
        eng.wait(j)
        eng.release(j)
        assert np.array_equal(eng.read(N.KVF_TIER_DEVICE, d), expected_bytes(eng, cids))
    eng.set_copy_mode(N.KVF_COPY_SM_VEC)
    eng.free(N.KVF_TIER_HOST, h)
    eng.free(N.KVF_TIER_DEVICE, d)


def test_dev_gather_scatter_k3(eng):
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(6)
    ntok = 1500
    cids = rand_cids(rng, ntok)
    d = fragment(eng, N.KVF_TIER_DEVICE, ntok, rng)
    eng.fill(N.KVF_TIER_DEVICE, d, cids)
    stage = torch.zeros(ntok * eng.token_bytes, dtype=torch.uint8, device="cuda")
    j = eng.dev_gather(d, stage.data_ptr())
    eng.wait(j)
    eng.release(j)
    torch.cuda.synchronize()
    assert np.array_equal(stage.cpu().numpy(), expected_bytes(eng, cids))
    d2 = fragment(eng, N.KVF_TIER_DEVICE, ntok, rng)
    j = eng.dev_scatter(stage.data_ptr(), d2)
    eng.wait(j)
    eng.release(j)
    assert np.array_equal(eng.read(N.KVF_TIER_DEVICE, d2), expected_bytes(eng, cids))
    eng.free(N.KVF_TIER_DEVICE, d)
    eng.free(N.KVF_TIER_DEVICE, d2)


def test_empty_and_invalid_jobs(eng):
    j = eng.h2d([], [])
    eng.wait(j)
    eng.release(j)
    with pytest.raises(N.KvfError):
        eng.h2d([(0, 4)], [(0, 5)])  # token counts differ
    with pytest.raises(N.KvfError):
        eng.h2d([(eng.host_slots, 1)], [(0, 1)])  # out of range
    with pytest.raises(N.KvfError):
        eng.wait(999999)


def test_full_pool_allocation(eng):
    free, _ = eng.free_count(N.KVF_TIER_DEVICE)
    runs = eng.alloc(N.KVF_TIER_DEVICE, free)
    with pytest.raises(N.KvfError) as ex:
        eng.alloc(N.KVF_TIER_DEVICE, 1)
    assert ex.value.code == 10  # OutOfGpuMemory + 1
    eng.free(N.KVF_TIER_DEVICE, runs)
    assert eng.free_count(N.KVF_TIER_DEVICE) == (free, 1)


def test_k4_priority_matches_reference(eng):
    for c in load_jsonl("prio.jsonl"):
        b = c["boundaries"]
        got = eng.priority(c["parent"], [x[0] for x in b], [int(x[1]) for x in b])
        want = np.asarray([int(x) for x in c["rank"]], dtype=np.int64)
        assert np.array_equal(got[1:], want[1:]), c["case"]


@pytest.mark.parametrize("fixture", ["evict_small.jsonl", "evict_medium.jsonl", "evict_bounded.jsonl"])
def test_k5_victims_match_reference(eng, fixture):
    for c in load_jsonl(fixture):
        if "error" in c:
            continue
        ta = TreeArrays(c)
        tree = {k: getattr(ta, k) for k in ("parent", "status", "lock", "rank", "time", "seq", "id", "tokens",
                                            "backed")}
        tree["depth"] = depth_from_parent(ta.parent)
        tree["bpt"] = ta.bpt
        idx, act, imm, pend = eng.victims(tree, c["needed"], c["policy"], c["mode"], c["has_floor"], c["floor"],
                                          c["cpu_used"], c["cpu_cap"])
        got = [(int(ta.id[v]), int(ta.tokens[v]) * ta.bpt, 0 if a == 0 else 1) for v, a in zip(idx, act)]
        assert got == [tuple(v) for v in c["victims"]], (fixture, c["case"])
        assert (imm, pend) == (c["immediate"], c["pending"])


@pytest.mark.parametrize("geom", [
    dict(layers=1, kv_heads_total=1, kv_heads_local=1, head_offset=0, head_dim=4),     # 8 B/token-plane: uint2 path
    dict(layers=2, kv_heads_total=8, kv_heads_local=1, head_offset=5, head_dim=128),   # G = 8 shard, head 5
    dict(layers=3, kv_heads_total=8, kv_heads_local=2, head_offset=6, head_dim=64),    # G = 4 shard, odd layers
    dict(layers=80, kv_heads_total=8, kv_heads_local=1, head_offset=7, head_dim=128),  # Llama-3-70B, G = 8
])
def test_shard_geometries_bit_exact(geom):
    """Every K1/K2/K3 path over shard geometries (head offsets, 8-byte token planes, odd layer
    counts) against the oracle's payload restatement of the same shard; runs end on the last
    slot of each pool."""
    torch = pytest.importorskip("torch")
    slots = 1024
    with Engine(gpu_slots=slots, host_slots=slots, **geom) as e:
        rng = np.random.default_rng(geom["layers"] * 31 + geom["head_offset"])
        ntok = 300
        cids = rand_cids(rng, ntok)
        pre = e.alloc(N.KVF_TIER_HOST, slots - ntok)     # the node ends on the last host slot
        h = e.alloc(N.KVF_TIER_HOST, ntok)
        assert h[-1][0] + h[-1][1] == slots
        e.fill(N.KVF_TIER_HOST, h, cids)
        want = expected_bytes(e, cids)
        assert np.array_equal(e.read(N.KVF_TIER_HOST, h), want)
        d = fragment(e, N.KVF_TIER_DEVICE, ntok, rng, pieces=7)
        for mode in MODES:
            e.set_copy_mode(mode)
            j = e.h2d(h, d)
            e.wait(j)
            e.release(j)
            assert np.array_equal(e.read(N.KVF_TIER_DEVICE, d), want), mode
        e.set_copy_mode(N.KVF_COPY_SM_VEC)
        j, _ = e.h2d_layered(h, d, None)
        e.wait(j)
        e.release(j)
        assert np.array_equal(e.read(N.KVF_TIER_DEVICE, d), want)
        stage = torch.zeros(ntok * e.token_bytes, dtype=torch.uint8, device="cuda")
        j = e.dev_gather(d, stage.data_ptr())
        e.wait(j)
        e.release(j)
        torch.cuda.synchronize()
        assert np.array_equal(stage.cpu().numpy(), want)
        e.free(N.KVF_TIER_HOST, pre)
        h2 = fragment(e, N.KVF_TIER_HOST, ntok, rng, pieces=5)
        j = e.d2h(d, h2)
        e.wait(j)
        e.release(j)
        assert np.array_equal(e.read(N.KVF_TIER_HOST, h2), want)
        assert e.checksum(N.KVF_TIER_HOST, h2) == e.checksum(N.KVF_TIER_DEVICE, d) == e.payload_checksum(cids)


def test_d2h_batch_one_launch_bit_exact(eng):
    """kvf_d2h_scatter_batch: several nodes' write-backs in one K2 launch, each job with its
    own id / events, bytes exact; a bad entry rejects the whole batch before any job exists."""
    rng = np.random.default_rng(21)
    nodes = []
    for ntok in (17, 128, 3, 200):
        cids = rand_cids(rng, ntok)
        d = fragment(eng, N.KVF_TIER_DEVICE, ntok, rng, pieces=3)
        eng.fill(N.KVF_TIER_DEVICE, d, cids)
        h = fragment(eng, N.KVF_TIER_HOST, ntok, rng, pieces=2)
        nodes.append((d, h, cids))
    l0 = eng.stats()["kernel_launches"]
    jobs = eng.d2h_batch([(d, h) for d, h, _ in nodes])
    assert eng.stats()["kernel_launches"] - l0 == 1
    for j, (d, h, cids) in zip(jobs, nodes):
        eng.wait(j)
        assert eng.elapsed_ms(j) >= 0
        eng.release(j)
        assert np.array_equal(eng.read(N.KVF_TIER_HOST, h), expected_bytes(eng, cids))
    d, h, _ = nodes[0]
    with pytest.raises(N.KvfError):  # token counts differ in the 2nd entry
        eng.d2h_batch([(d, h), (nodes[1][0], nodes[2][1])])
    with pytest.raises(N.KvfError):  # duplicate job ids
        eng.d2h_batch([(d, h), (d, h)], jobs=[77, 77])
    j = eng.d2h_batch([(d, h)], jobs=[77])[0]  # nothing of the rejected batches was left behind
    eng.wait(j)
    eng.release(j)
    for d, h, _ in nodes:
        eng.free(N.KVF_TIER_DEVICE, d)
        eng.free(N.KVF_TIER_HOST, h)


def random_case(rng, n):
    parent = [-1] + [int(rng.integers(0, i)) for i in range(1, n)]
    status = [0] + [int(x) for x in rng.choice([0, 0, 0, 1], size=n - 1)]
    return {
        "parent": parent, "status": status,
        "lock": [0] + [int(x) for x in rng.choice([0, 0, 0, 0, 1], size=n - 1)],
        "rank": [int(x) for x in rng.choice([2**62 - 1, 2**61 - 1, 1, 2, 3, 5], size=n)],
        "time": [float(x) for x in rng.integers(0, n // 3 + 1, size=n) * 0.25],  # ties on time
        "seq": [int(x) for x in rng.integers(0, n // 2 + 1, size=n)],            # and on seq
        "id": [int(x) for x in rng.permutation(n) + 1],
        "tokens": [int(x) for x in rng.integers(1, 300, size=n)],
        "backed": [int(x) for x in rng.integers(0, 2, size=n)],
        "bpt": 1024, "policy": int(rng.integers(0, 2)), "mode": int(rng.integers(0, 2)),
        "has_floor": int(rng.integers(0, 2)), "floor": 2, "cpu_used": 0, "cpu_cap": 0,
        "needed": int(rng.integers(1, 150 * n)) * 1024,
    }


def test_k5_every_tree_size_across_the_shared_memory_limits(eng):
    """Random trees of every size class around the single-CTA launch configurations
    (zero-copy staging ~48 KB, block-size steps, the 4096-node limit) against the CPU
    restatement (itself pinned to the reference's 402 golden vectors).  Regression: a 488-node
    tree needed 48,888 B of dynamic + static shared memory, just over the 48 KB default."""
    from oracle_ffi import oracle_evict
    rng = np.random.default_rng(2024)
    sizes = list(range(380, 620, 7)) + [63, 64, 65, 127, 128, 129, 1023, 1024, 1025, 1170, 1171, 2047, 2049, 4095,
                                        4096, 4097]
    checked = 0
    for n in sizes:
        for _ in range(8):  # skip snapshots that hit the reference's remove_node defect (rc 13)
            c = random_case(rng, n)
            rc, want, imm, pend = oracle_evict(c)
            if rc == 0:
                break
        if rc != 0:
            continue
        ta = TreeArrays(c)
        tree = {k: getattr(ta, k) for k in ("parent", "status", "lock", "rank", "time", "seq", "id", "tokens", "backed")}
        tree["depth"] = depth_from_parent(ta.parent)
        tree["bpt"] = ta.bpt
        idx, act, gi, gp = eng.victims(tree, c["needed"], c["policy"], c["mode"], c["has_floor"], c["floor"],
                                       c["cpu_used"], c["cpu_cap"])
        got = [(int(ta.id[v]), int(ta.tokens[v]) * ta.bpt, 0 if a == 0 else 1) for v, a in zip(idx, act)]
        assert got == want and (gi, gp) == (imm, pend), n
        checked += 1
    assert checked >= len(sizes) - 4


def test_stamp_timed_jobs_match_event_timing_and_bytes():
    """KVF_JOB_TIMING_STAMPS: K1 / K2 / K2-batch jobs fenced by a plain stop event and timed by
    the copy kernels' globaltimer stamps -- bytes exact, device time within 10 % of the
    timing-event measurement of the same copy, span over jobs consistent."""
    e = Engine(layers=32, kv_heads_total=8, head_dim=128, gpu_slots=4096, host_slots=8192)
    try:
        rng = np.random.default_rng(5)
        n = 2048  # 256 MiB
        cids = rand_cids(rng, n)
        h = e.alloc(N.KVF_TIER_HOST, n)
        e.fill(N.KVF_TIER_HOST, h, cids)
        want = expected_bytes(e, cids)
        times = {}
        for stamps in (False, True, False, True):
            e.set_job_timing(stamps)
            d = e.alloc(N.KVF_TIER_DEVICE, n)
            j = e.h2d(h, d)
            ms = e.elapsed_ms(j)
            e.release(j)
            assert np.array_equal(e.read(N.KVF_TIER_DEVICE, d), want)
            times.setdefault(stamps, []).append(ms)
            e.free(N.KVF_TIER_DEVICE, d)
        ev, st = min(times[False]), min(times[True])
        assert st > 0 and abs(st - ev) <= 0.1 * ev, (ev, st)
        # K2 batch under stamps: jobs share the launch's stamps; span covers both
        e.set_job_timing(True)
        d = e.alloc(N.KVF_TIER_DEVICE, n)
        e.fill(N.KVF_TIER_DEVICE, d, cids)
        h1, h2 = e.alloc(N.KVF_TIER_HOST, n // 2), e.alloc(N.KVF_TIER_HOST, n // 2)
        # split the device run list in two halves of n/2 tokens
        first, second, left = [], [], n // 2
        for s, l in d:
            if left >= l:
                first.append((s, l))
                left -= l
            elif left > 0:
                first.append((s, left))
                second.append((s + left, l - left))
                left = 0
            else:
                second.append((s, l))
        jobs = e.d2h_batch([(first, h1), (second, h2)])
        a, b = e.elapsed_ms(jobs[0]), e.elapsed_ms(jobs[1])
        span = e.span_ms(jobs[0], jobs[1])
        assert a == b and a > 0 and abs(span - a) < 1e-3
        for j in jobs:
            e.release(j)
        got = e.read(N.KVF_TIER_HOST, h1 + h2)
        assert np.array_equal(got, want)
    finally:
        e.close()
