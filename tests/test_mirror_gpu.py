"""Decisions over the HBM tree mirror (kvf_tree_*, csrc/engine/mirror.cu) against the
reference's own vectors and the snapshot path:
  * K5 over the mirror == the unmodified reference's RadixCache::evict on 402 golden
    snapshots (tests/golden/evict_small.jsonl), served by the resident decider CTA (<= 128
    slots) and by one-shot launches (larger / KVF_DECIDER=0);
  * K4 over the mirror == the reference's set_agent_priorities (tests/golden/prio.jsonl),
    reported as rank changes;
  * incremental updates: random mutations (touch, lock, status, backup, removal with slot
    reuse, new nodes) shipped as change records keep the mirror's decisions equal to a fresh
    snapshot's (kvf_victim_select) at every step;
  * the device-wide path (> 4096 slots, hand-written radix sort + chain cut) == the live
    reference at 4.5k / 12k nodes, with and without the time-follows-seq key shortcut;
  * the resident CTA's lifecycle: idle-out, relaunch, hold, a device-wide sync returning."""
import json
import os
import random
import subprocess
import time

import numpy as np
import pytest

from conftest import UNDER_SANITIZER
from oracle_ffi import ORACLE_DIR, TreeArrays, load_jsonl

pytestmark = pytest.mark.gpu

FIELDS = ("parent", "status", "lock", "rank", "time", "seq", "id", "tokens", "backed")


@pytest.fixture(scope="module")
def eng():
    from paper_2507_07400_b200.engine import Engine
    e = Engine(layers=1, kv_heads_total=1, head_dim=4, gpu_slots=16, host_slots=16)
    yield e
    e.close()


def arrays(c):
    ta = TreeArrays(c)
    return {k: getattr(ta, k) for k in FIELDS}, ta


def ref_victims(ta, c):
    return [tuple(v) for v in c["victims"]]


def as_victims(ta, slots, acts, slot_to_index=None):
    out = []
    for s, a in zip(slots, acts):
        i = int(s) if slot_to_index is None else slot_to_index[int(s)]
        out.append((int(ta.id[i]), int(ta.tokens[i]) * ta.bpt, 0 if a == 0 else 1))
    return out


def evict_args(c):
    return dict(needed=c["needed"], workflow_aware=c["policy"], offload=c["mode"], has_floor=c["has_floor"],
                floor=c["floor"], cpu_used=c["cpu_used"], cpu_cap=c["cpu_cap"])


def test_mirror_k5_matches_reference_vectors(eng):
    from paper_2507_07400_b200.engine import Tree
    s0 = eng.stats()
    checked = 0
    for c in load_jsonl("evict_small.jsonl"):
        if "error" in c or c["needed"] == 0:
            continue
        a, ta = arrays(c)
        with Tree(eng, ta.bpt) as t:
            t.load_arrays(a)
            slots, acts, imm, pend = t.victims(**evict_args(c))
        assert as_victims(ta, slots, acts) == ref_victims(ta, c), c["case"]
        assert (imm, pend) == (c["immediate"], c["pending"]), c["case"]
        checked += 1
    s1 = eng.stats()
    assert checked >= 300
    # these trees (<= 128 slots) went to the resident CTA; larger ones (the incremental test
    # below grows to 900 slots) take one-shot launches
    assert s1["resident_served"] - s0["resident_served"] >= checked


def test_mirror_k4_matches_reference_vectors(eng):
    from paper_2507_07400_b200.engine import Tree
    for c in load_jsonl("prio.jsonl"):
        parent = np.asarray(c["parent"], dtype=np.int32)
        n = len(parent)
        suffix = 4611686018427387903  # INT64_MAX / 2
        with Tree(eng, 1) as t:
            t.update({"slot": i, "parent": int(parent[i]), "rank": suffix, "tokens": 1, "id": i, "seq": i,
                      "lock": 1 if i == 0 else 0} for i in range(n))
            t.priorities([x[0] for x in c["boundaries"]], [int(x[1]) for x in c["boundaries"]])
            ch = t.rank_changes()
        got = [ch.get(i, suffix) for i in range(1, n)]
        assert got == [int(x) for x in c["rank"][1:]], c["case"]


def snapshot_victims(eng, live, bpt, args):
    """Reference for a mirror state: the snapshot path over the live nodes (compacted)."""
    from paper_2507_07400_b200.engine import depth_from_parent
    order = sorted(live)  # slots are reused, so parents may sit above children: preorder remap
    index = {}
    seq_order = []
    roots = [s for s in order if live[s]["parent"] < 0]
    assert roots == [0]
    kids = {}
    for s in order:
        p = live[s]["parent"]
        if p >= 0:
            kids.setdefault(p, []).append(s)
    stack = [0]
    while stack:
        s = stack.pop()
        index[s] = len(seq_order)
        seq_order.append(s)
        stack.extend(reversed(kids.get(s, [])))
    tree = {k: np.asarray([live[s][k] if k != "parent" else (index[live[s]["parent"]] if live[s]["parent"] >= 0 else -1)
                           for s in seq_order]) for k in FIELDS}
    tree["depth"] = depth_from_parent(tree["parent"])
    tree["bpt"] = bpt
    idx, act, imm, pend = eng.victims(tree, **args)
    return [(seq_order[int(i)], int(a)) for i, a in zip(idx, act)], imm, pend


@pytest.mark.parametrize("seed,target", [(1, 40), (2, 300), (3, 900)])
def test_mirror_incremental_matches_snapshot(eng, seed, target):
    """Random mutations through change records; the mirror's K5 equals a fresh snapshot's."""
    from paper_2507_07400_b200.engine import Tree
    rng = random.Random(seed)
    bpt = 7
    live = {0: dict(parent=-1, status=0, lock=1, rank=4611686018427387903, time=0.0, seq=0, id=0, tokens=0,
                    backed=0)}
    free = []
    next_id, seq, now = 1, 0, 0.0
    with Tree(eng, bpt) as t:
        t.update([dict(slot=0, **live[0])])
        for step in range(120):
            recs = {}
            for _ in range(rng.randint(1, 12)):
                op = rng.random()
                if len(live) < target and (op < 0.45 or len(live) < 4):
                    slot = min(free) if free else len(live) + len(free)
                    if free:
                        free.remove(slot)
                    par = rng.choice(list(live))
                    seq += 1
                    now += rng.choice([0.0, 0.5])
                    live[slot] = dict(parent=par, status=0, lock=0, rank=rng.choice([4611686018427387903, 1, 3]),
                                      time=now, seq=seq, id=next_id, tokens=rng.randint(1, 9), backed=0)
                    next_id += 1
                    recs[slot] = live[slot]
                    continue
                s = rng.choice([x for x in live if x != 0])
                n = live[s]
                if op < 0.6:
                    seq += 1
                    now += rng.choice([0.0, 0.25])
                    n["time"], n["seq"] = now, seq
                elif op < 0.7:
                    n["lock"] = rng.choice([0, 0, 1])
                elif op < 0.8:
                    n["status"] = rng.choice([0, 0, 1, 2, 3])
                elif op < 0.85:
                    n["backed"] = 1 - n["backed"]
                elif op < 0.9:
                    n["rank"] = rng.choice([4611686018427387903, 2305843009213693951, 0, 1, 2, 5])
                else:  # remove a leaf
                    if any(v["parent"] == s for v in live.values()):
                        continue
                    del live[s]
                    free.append(s)
                    recs[s] = None
                    continue
                recs[s] = n
            t.update([dict(slot=s, **v) if v is not None else dict(slot=s, parent=-1, status=0xFF)
                      for s, v in recs.items()])
            args = dict(needed=rng.randint(1, 120) * bpt, workflow_aware=rng.random() < 0.5,
                        offload=rng.random() < 0.7, has_floor=rng.random() < 0.3, floor=rng.choice([0, 1, 3]),
                        cpu_used=0, cpu_cap=0)
            want, wimm, wpend = snapshot_victims(eng, live, bpt, args)
            slots, acts, imm, pend = t.victims(**args)
            got = [(int(s), int(a)) for s, a in zip(slots, acts)]
            assert got == want, (seed, step)
            assert (imm, pend) == (wimm, wpend), (seed, step)


REF = os.path.join(ORACLE_DIR, "_ref", "ref_trace")


def ref_cases(seed, nodes, cases=1, vocab=200):
    if not os.path.exists(REF):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    out = subprocess.run([REF, "evict", f"seed={seed}", f"cases={cases}", f"min_nodes={nodes}", f"max_nodes={nodes}",
                          f"vocab={vocab}"], capture_output=True, text=True, check=True, timeout=600).stdout
    return [json.loads(l) for l in out.splitlines() if l.strip()]


def time_follows_seq(ta):
    o = np.argsort(ta.seq, kind="stable")
    t, s = ta.time[o], ta.seq[o]
    ok = np.all(np.diff(t) >= 0)
    same = s[1:] == s[:-1]
    return bool(ok and np.all(t[1:][same] == t[:-1][same]))


@pytest.mark.parametrize("nodes,seed", [(4500, 11), (12000, 12)])
def test_mirror_large_matches_reference(eng, nodes, seed):
    from paper_2507_07400_b200.engine import Tree
    for c in ref_cases(seed, nodes, cases=3):
        if "error" in c:
            continue
        a, ta = arrays(c)
        with Tree(eng, ta.bpt) as t:
            t.load_arrays(a)
            t.hints(time_follows_seq(ta))
            slots, acts, imm, pend = t.victims(**evict_args(c))
        assert as_victims(ta, slots, acts) == ref_victims(ta, c), (nodes, c["case"])
        assert (imm, pend) == (c["immediate"], c["pending"])


def test_mirror_large_time_shortcut(eng):
    """A large tree whose stamps follow seq: the shortcut (no time passes) and the full key agree
    with the snapshot path (which always sorts the time word)."""
    from paper_2507_07400_b200.engine import Tree, depth_from_parent
    rng = np.random.default_rng(5)
    n = 9000
    parent = np.zeros(n, dtype=np.int32)
    parent[0] = -1
    for i in range(1, n):
        parent[i] = rng.integers(0, i) if i > 50 else 0
    seq = rng.permutation(n).astype(np.uint64) + 1
    seq[0] = 0
    tree = dict(parent=parent, status=rng.choice([0, 0, 0, 1], n).astype(np.uint8),
                lock=(rng.random(n) < 0.05).astype(np.int32), rank=rng.choice([4611686018427387903, 1, 2, 7], n),
                time=(seq // 4).astype(np.float64), seq=seq, id=np.arange(n, dtype=np.uint64),
                tokens=rng.integers(1, 64, n).astype(np.uint64), backed=(rng.random(n) < 0.3).astype(np.uint8))
    tree["status"][0], tree["lock"][0] = 0, 1
    tree["depth"] = depth_from_parent(parent)
    tree["bpt"] = 3
    for wa in (0, 1):
        args = dict(needed=int(tree["tokens"].sum()) // 3 * 3, workflow_aware=wa, offload=1)
        want_i, want_a, wimm, wpend = eng.victims(tree, **args)
        for hint in (False, True):
            with Tree(eng, 3) as t:
                t.load_arrays(tree)
                t.hints(hint)
                s, a, imm, pend = t.victims(**args)
            assert s.tolist() == want_i.tolist() and a.tolist() == want_a.tolist(), (wa, hint)
            assert (imm, pend) == (wimm, wpend)


def test_resident_lifecycle(eng):
    import torch
    from paper_2507_07400_b200.engine import Tree, decider_hold, decider_running
    c = load_jsonl("evict_small.jsonl")[1]
    a, ta = arrays(c)
    with Tree(eng, ta.bpt) as t:
        t.load_arrays(a)
        want = ref_victims(ta, c)
        s0 = eng.stats()
        for _ in range(20):  # back to back: one resident CTA serves them all
            s, x, _, _ = t.victims(**evict_args(c))
            assert as_victims(ta, s, x) == want
        s1 = eng.stats()
        assert s1["resident_launches"] - s0["resident_launches"] <= 1
        time.sleep(0.01)  # > the 200 us idle limit: the CTA leaves by itself ...
        torch.cuda.synchronize()  # ... so a device-wide sync returns
        assert not decider_running(eng)
        s, x, _, _ = t.victims(**evict_args(c))  # ... and the next request relaunches it
        assert as_victims(ta, s, x) == want
        assert eng.stats()["resident_launches"] == s1["resident_launches"] + 1
        decider_hold(eng, True)  # held: survives idle gaps
        t.victims(**evict_args(c))
        time.sleep(0.01)
        assert decider_running(eng)
        s2 = eng.stats()
        s, x, _, _ = t.victims(**evict_args(c))
        assert as_victims(ta, s, x) == want
        assert eng.stats()["resident_launches"] == s2["resident_launches"]
        decider_hold(eng, False)  # released: gone at once
        assert not decider_running(eng)
        torch.cuda.synchronize()


def test_resident_fast_path_latency(eng):
    """K4 queued + K5 behind it on a 44-node tree: the pair's host round trip (diagnostic bound)."""
    from paper_2507_07400_b200.engine import Tree, decider_hold
    c = next(x for x in load_jsonl("evict_small.jsonl") if len(x["parent"]) >= 40 and "error" not in x)
    a, ta = arrays(c)
    with Tree(eng, ta.bpt) as t:
        t.load_arrays(a)
        decider_hold(eng, True)
        try:
            lat = []
            for _ in range(200):
                t0 = time.perf_counter()
                t.priorities([1], [3])
                t.victims(**evict_args(c))
                t.rank_changes()
                lat.append((time.perf_counter() - t0) * 1e6)
        finally:
            decider_hold(eng, False)
    med = sorted(lat)[len(lat) // 2]
    print(f"K4+K5 pair via the resident decider, {len(a['parent'])} nodes: median {med:.1f} us")
    if not UNDER_SANITIZER:
        assert med < 60


def test_mirror_grows_past_its_capacity_with_a_k4_pending(eng):
    """A tree that outgrows its mirror (1024 -> 6000 slots: a new HBM block, the old slots
    copied, the single-CTA path handing over to the device-wide one) while a queued K4's result
    is still unread: the rank changes survive the move and K4 / K5 agree with the snapshot
    forms on the grown tree."""
    from paper_2507_07400_b200.engine import Tree
    rng = np.random.default_rng(9)
    n = 6000
    parent = np.zeros(n, dtype=np.int32)
    parent[0] = -1
    for i in range(1, n):
        parent[i] = rng.integers(0, i)
    suffix = 4611686018427387903
    recs = [{"slot": i, "parent": int(parent[i]), "lock": 1 if i == 0 else 0, "status": 0, "backed": 0,
             "rank": suffix, "time": float(i), "seq": i, "id": i, "tokens": int(rng.integers(1, 9))} for i in range(n)]
    with Tree(eng, 5) as t:
        t.update(recs[:800])
        bs = [int(x) for x in rng.integers(1, 800, size=6)]
        cands = [1, 2, 3, 4, 5, 6]
        t.priorities(bs, cands)            # queued on the 1024-slot mirror ...
        t.update(recs[800:])               # ... the next request needs 6000 slots
        t.hints(True)
        slots, acts, imm, pend = t.victims(needed=400, workflow_aware=True, offload=True)
        ch = t.rank_changes()              # the K4 result, carried across the move
        want = eng.priority(parent[:800], bs, cands)
        got = [ch.get(i, suffix) for i in range(1, 800)]
        assert got == [int(x) for x in want[1:]]
        # the K5 above ran before the K4's ranks reached the host, on the grown mirror with them
        ranks = np.full(n, suffix, dtype=np.int64)
        ranks[:800] = want
        ranks[0] = suffix
        tree = dict(parent=parent, status=np.zeros(n, np.uint8), lock=(np.arange(n) == 0).astype(np.int32),
                    rank=ranks, time=np.arange(n, dtype=np.float64), seq=np.arange(n, dtype=np.uint64),
                    id=np.arange(n, dtype=np.uint64), tokens=np.array([r["tokens"] for r in recs], np.uint64),
                    backed=np.zeros(n, np.uint8), bpt=5)
        from paper_2507_07400_b200.engine import depth_from_parent
        tree["depth"] = depth_from_parent(parent)
        wi, wa, wimm, wpend = eng.victims(tree, 400, True, True)
        assert slots.tolist() == wi.tolist() and acts.tolist() == wa.tolist() and (imm, pend) == (wimm, wpend)


def test_two_queued_k4_results_read_in_order_across_a_mirror_move(eng):
    """Two K4 requests queued back to back (the engine keeps two result buffers); a third is
    refused until the oldest is read.  The results, read oldest first and applied in order,
    give the second K4's ranks -- also when the mirror is reallocated while both are unread."""
    from paper_2507_07400_b200.engine import Tree
    rng = np.random.default_rng(11)
    n = 3000
    parent = np.zeros(n, dtype=np.int32)
    parent[0] = -1
    for i in range(1, n):
        parent[i] = rng.integers(0, i)
    suffix = 4611686018427387903
    recs = [{"slot": i, "parent": int(parent[i]), "lock": 1 if i == 0 else 0, "status": 0, "backed": 0,
             "rank": suffix, "time": float(i), "seq": i, "id": i, "tokens": 1} for i in range(n)]
    for grow in (False, True):
        with Tree(eng, 5) as t:
            m = 600 if grow else n
            t.update(recs[:m])
            b1, b2 = [int(x) for x in rng.integers(1, m, size=5)], [int(x) for x in rng.integers(1, m, size=4)]
            c1, c2 = [3, 1, 4, 1, 5], [2, 7, 1, 8]
            t.priorities(b1, c1)
            t.priorities(b2, c2)
            with pytest.raises(Exception):
                t.priorities(b1, c1)   # both result buffers unread
            if grow:
                t.update(recs[m:])     # the next request reallocates the mirror (1024 -> 3000+ slots)
                t.victims(needed=1, workflow_aware=True, offload=False)
            host = np.full(m, suffix, dtype=np.int64)
            for _ in range(2):
                for s, r in t.rank_changes().items():
                    host[s] = r
            assert t.rank_changes() == {}
            want = eng.priority(parent[:m], b2, c2)
            assert host[1:].tolist() == [int(x) for x in want[1:]]
