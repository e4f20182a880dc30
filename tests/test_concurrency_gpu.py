"""Several engines driven from several host threads at once -- the one-host-thread-per-GPU
pattern of a multi-GPU box, here all on device 0.  Each thread interleaves K1/K2 transfers
(bytes checked against the payload definition), K4/K5 decisions (checked against the
reference's vectors) and K6 calls; nothing may leak between engines (job ids, workspaces,
decision done words, attention descriptor caches, the per-thread last-error text).
ctypes drops the GIL inside every C-ABI call, so the calls really overlap."""
import threading

import numpy as np
import pytest

from oracle_ffi import TreeArrays, load_jsonl

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
N = pytest.importorskip("paper_2507_07400_b200._native")
from paper_2507_07400_b200.engine import Engine, depth_from_parent  # noqa: E402


def worker(tid, cases, errors):
    try:
        rng = np.random.default_rng(100 + tid)
        with Engine(layers=4, kv_heads_total=8, kv_heads_local=2, head_offset=2 * tid % 8, gpu_slots=8192,
                    host_slots=8192) as e:
            q = torch.randn(2, 8, 128, device="cuda").to(torch.bfloat16)
            out = torch.empty_like(q)
            for it in range(12):
                n = int(rng.integers(50, 900))
                cids = rng.integers(0, 2**63, size=n, dtype=np.uint64)
                h = e.alloc(N.KVF_TIER_HOST, n)
                e.fill(N.KVF_TIER_HOST, h, cids)
                d = e.alloc(N.KVF_TIER_DEVICE, n)
                j = e.h2d(h, d)
                e.wait(j)
                e.release(j)
                assert e.checksum(N.KVF_TIER_DEVICE, d) == e.payload_checksum(cids), "K1 bytes"
                h2 = e.alloc(N.KVF_TIER_HOST, n)
                j = e.d2h(d, h2)
                e.wait(j)
                e.release(j)
                assert e.checksum(N.KVF_TIER_HOST, h2) == e.payload_checksum(cids), "K2 bytes"
                c = cases[(tid * 7 + it) % len(cases)]
                ta = TreeArrays(c)
                tree = {k: getattr(ta, k) for k in ("parent", "status", "lock", "rank", "time", "seq", "id", "tokens",
                                                    "backed")}
                tree["depth"] = depth_from_parent(ta.parent)
                tree["bpt"] = ta.bpt
                idx, act, _, _ = e.victims(tree, c["needed"], c["policy"], c["mode"], c["has_floor"], c["floor"],
                                           c["cpu_used"], c["cpu_cap"])
                got = [(int(ta.id[v]), int(ta.tokens[v]) * ta.bpt, 0 if a == 0 else 1) for v, a in zip(idx, act)]
                assert got == [tuple(v) for v in c["victims"]], "K5 differs from the reference"
                torch.cuda.synchronize()
                ja = e.attend(it % 4, 4, q.data_ptr(), [d, d[:1]], out.data_ptr(), 0.1)
                e.wait(ja)
                e.release(ja)
                assert torch.isfinite(out.float()).all()
                for r in (h, h2):
                    e.free(N.KVF_TIER_HOST, r)
                e.free(N.KVF_TIER_DEVICE, d)
    except Exception as ex:  # pragma: no cover - reported by the test
        errors.append(f"thread {tid}: {ex!r}")


def test_engines_on_concurrent_threads():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cases = load_jsonl("evict_small.jsonl")[:40]
    errors = []
    threads = [threading.Thread(target=worker, args=(t, cases, errors)) for t in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=600)
    assert not errors, errors
