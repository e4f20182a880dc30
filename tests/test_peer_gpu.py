"""kvf_peer_gather -- NVLink peer fetch from another engine's HBM pool (SURVEY §8f-4 follow-on).

This pool gives one GPU per call, so the two engines here share device 0: the kernel path is
the one a second GPU would use (a K3-style copy reading the peer pool's device addresses;
across GPUs the same loads go over NVLink after cudaDeviceEnablePeerAccess).  Bytes are
compared bit for bit with the oracle's payload restatement over fragmented run tables.
"""
import numpy as np
import pytest

from test_engine_gpu import expected_bytes, fragment, rand_cids

pytestmark = pytest.mark.gpu

N = pytest.importorskip("paper_2507_07400_b200._native")
from paper_2507_07400_b200.engine import Engine  # noqa: E402


@pytest.mark.parametrize("local,offset", [(8, 0), (1, 7), (2, 4)])
def test_peer_gather_bytes_match_oracle(local, offset):
    rng = np.random.default_rng(local * 10 + offset)
    kw = dict(layers=3, kv_heads_total=8, kv_heads_local=local, head_offset=offset, head_dim=128,
              gpu_slots=8192, host_slots=0)
    with Engine(**kw) as a, Engine(**kw) as b:
        cids = rand_cids(rng, 1500)
        src = fragment(a, N.KVF_TIER_DEVICE, len(cids), rng)
        a.fill(N.KVF_TIER_DEVICE, src, cids)           # replica A holds the node (its prefill)
        dst = fragment(b, N.KVF_TIER_DEVICE, len(cids), rng, pieces=9)
        j = b.peer_gather(a, src, dst)                 # replica B pulls it from A's HBM
        b.wait(j)
        b.release(j)
        assert np.array_equal(b.read(N.KVF_TIER_DEVICE, dst), expected_bytes(b, cids))
        assert b.checksum(N.KVF_TIER_DEVICE, dst) == b.payload_checksum(cids)


def test_peer_gather_within_one_engine_and_errors():
    rng = np.random.default_rng(3)
    with Engine(layers=2, kv_heads_total=8, gpu_slots=4096, host_slots=0) as a, \
            Engine(layers=2, kv_heads_total=8, kv_heads_local=4, gpu_slots=4096, host_slots=0) as other:
        cids = rand_cids(rng, 300)
        src = a.alloc(N.KVF_TIER_DEVICE, 300)
        a.fill(N.KVF_TIER_DEVICE, src, cids)
        dst = fragment(a, N.KVF_TIER_DEVICE, 300, rng)
        j = a.peer_gather(a, src, dst)
        a.wait(j)
        a.release(j)
        assert np.array_equal(a.read(N.KVF_TIER_DEVICE, dst), expected_bytes(a, cids))
        with pytest.raises(N.KvfError):
            other.peer_gather(a, src, other.alloc(N.KVF_TIER_DEVICE, 300))   # different shard geometry
        with pytest.raises(N.KvfError):
            a.peer_gather(a, src, a.alloc(N.KVF_TIER_DEVICE, 299))            # token counts differ
        with pytest.raises(N.KvfError):
            a.peer_gather(a, [(4000, 300)], dst)                              # beyond the pool
