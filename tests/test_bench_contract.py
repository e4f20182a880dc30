"""bench.py contract on the GPU: the N=1 line carries every required key, and the N-rank
code path (torchrun, barrier, max-over-ranks, head-sharded engines) runs -- rehearsed with 2
ranks on one GPU over gloo (the driver's scaling run uses one GPU per rank over NCCL)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REQUIRED = ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
            "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"]


def _last_json(out):
    lines = [l for l in out.splitlines() if l.startswith("{")]
    assert lines, out[-2000:]
    return json.loads(lines[-1])


def test_bench_single_gpu_line():
    r = subprocess.run([sys.executable, "bench.py", "--steps", "3", "--warmup", "3"], cwd=ROOT, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    line = _last_json(r.stdout)
    for k in REQUIRED:
        assert k in line, k
    assert line["value"] > 10 and line["roofline"]["frac"] > 0.5 and line["gpu_launches"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] > 0 and line["parity"]["bench_bytes_checksum_equal"]
    # decisions are inside e2e (symmetric with the reference arm), and C4 has its own line
    assert line["e2e"]["decision_us_per_step"] > 0 and line["e2e"]["value"] <= line["e2e"]["transfer_only_gbs"]
    assert line["e2e_c4"]["value"] > 0 and line["e2e_c4"]["offload_jobs"] == 1261


def test_bench_two_rank_rehearsal():
    env = dict(os.environ, KVF_BENCH_SAME_DEVICE="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29533", "bench.py", "--gpus", "2", "--steps",
                        "2", "--warmup", "3"], cwd=ROOT, capture_output=True, text=True, timeout=1200, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    line = _last_json(r.stdout)
    assert line["n_gpus"] == 2 and line["value"] > 0 and "kv-head shard x2" in line["config"]["parallelism"]
    assert line["cpu_baseline"]["value"] > 0 and line["cpu_baseline"]["cores"] >= 1


def test_reference_arm_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "2", "--warmup", "3"], cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = _last_json(r.stdout)
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["cores"] >= 1
