import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
for p in (HERE, ROOT):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs on the GPU box via gpurun)")


# compute-sanitizer runs (scripts/gpu_sanitize.sh) slow every kernel 10-100x: tests keep their
# parity / byte assertions there and skip the ones about real-time latency
UNDER_SANITIZER = os.environ.get("KVF_SANITIZER") == "1"
