"""Multi-GPU host logic on CPU (gloo, world_size 2 and 4): the KV-head shard plan every
rank derives, and the shard-independence of the decision stream."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle_ffi import load_jsonl
from paper_2507_07400_b200.shard import decision_stream, plan


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p = plan(rank, world, layers=80, kv_heads=8, gpu_budget=2_139_095_040)
    got = [None] * world
    dist.all_gather_object(got, (p.rank, p.head_offset, p.kv_heads_local, p.bytes_per_token, p.gpu_budget))
    dist.barrier()
    if rank == 0:
        q.put(got)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_shard_plans_partition_heads_and_bytes(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    heads = sorted(h for _, off, n, _, _ in got for h in range(off, off + n))
    assert heads == list(range(8))                        # disjoint, complete
    assert sum(g[3] for g in got) == 327680                # bytes/token add up (70B KV)
    assert sum(g[4] for g in got) == 2_139_095_040         # budgets add up
    assert len({g[3] for g in got}) == 1                   # equal shards


def test_plan_rejects_bad_splits():
    with pytest.raises(ValueError):
        plan(0, 3)
    with pytest.raises(ValueError):
        plan(2, 2)


def test_reference_decisions_are_shard_independent():
    """The unmodified reference, run at per-shard bytes/token and budget for G = 1, 2, 4, 8,
    issues the identical transfer and transition sequence -- so every rank of a head-sharded
    deployment runs the same decisions, and the G=1 golden trace is every shard's oracle."""
    base = decision_stream(load_jsonl("sim_c5_g1.jsonl"))
    for g in (2, 4, 8):
        assert decision_stream(load_jsonl(f"sim_c5_g{g}.jsonl")) == base
    jobs, _ = base
    assert sum(1 for d, p, _ in jobs if d == 0 and p == 1) == 36  # prefetches
