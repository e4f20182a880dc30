"""KV-head sharding plan for N GPUs of one box.

Rank g of G holds KV heads [g*H/G, (g+1)*H/G) of every token: its engine's geometry has
kv_heads_local = H/G, head_offset = g*H/G, so bytes per token and the GPU budget both
divide by G.  All shards see the same tokens, hence run the identical decision stream
(the C5 golden traces are identical at G = 1, 2, 4, 8); each moves only its own shard over
its own PCIe link.  Nothing here is a collective: torch.distributed is used only for the
barrier and the max-over-ranks timing in bench.py.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class ShardPlan:
    rank: int
    world: int
    layers: int
    kv_heads_total: int
    kv_heads_local: int
    head_offset: int
    head_dim: int
    bytes_per_token: int   # this shard's ledger bytes per token
    gpu_budget: int        # this shard's HBM budget (bytes)

    @property
    def heads(self) -> range:
        return range(self.head_offset, self.head_offset + self.kv_heads_local)

    def engine_kwargs(self) -> dict:
        return dict(layers=self.layers, kv_heads_total=self.kv_heads_total, kv_heads_local=self.kv_heads_local,
                    head_offset=self.head_offset, head_dim=self.head_dim)


def plan(rank: int, world: int, layers: int = 32, kv_heads: int = 8, head_dim: int = 128,
         gpu_budget: int = 3_271_557_120, dtype_bytes: int = 2) -> ShardPlan:
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    if kv_heads % world:
        raise ValueError(f"{kv_heads} KV heads cannot be split across {world} GPUs")
    local = kv_heads // world
    bpt_full = 2 * layers * kv_heads * head_dim * dtype_bytes
    if gpu_budget % bpt_full:
        raise ValueError("the GPU budget must be a whole number of tokens")
    return ShardPlan(rank, world, layers, kv_heads, local, rank * local, head_dim, bpt_full // world,
                     gpu_budget // world)


def decision_stream(records):
    """The shard-independent part of a trace: ordered (direction, purpose, node) of every
    transfer and (node, from, to) of every transition (event indices shift with G: transfer
    times scale with the shard size, compute times do not)."""
    jobs = [(r["dir"], r["purpose"], r["node"]) for r in records if r["t"] == "job"]
    trs = [(r["node"], r["from"], r["to"]) for r in records if r["t"] == "tr"]
    return jobs, trs
