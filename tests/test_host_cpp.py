"""Build and run the C++ unit tests of the host API (tests/cpp/).

test_host_cpu.cpp: step graph, cost model, event queue, radix tree, tier ledger, workload
                   (no GPU; the decision calls are asserted to refuse without an engine)
test_host_gpu.cpp: eviction (K5), priorities (K4), TierManager moving real bytes (K1/K2)
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2507_07400_b200")


def build(name):
    from paper_2507_07400_b200 import build as B
    B.build_engine()
    B.build_host()
    src = os.path.join(ROOT, "tests", "cpp", f"{name}.cpp")
    exe = os.path.join(ROOT, "tests", "cpp", name)
    if not os.path.exists(exe) or os.path.getmtime(exe) < max(os.path.getmtime(src),
                                                               os.path.getmtime(os.path.join(PKG, "libkvflow_host.so"))):
        subprocess.run(["g++", "-std=c++20", "-O1", "-g", "-Wall", "-Wextra", "-Wno-unused-parameter",
                        f"-I{ROOT}/include", f"-I{ROOT}/tests/cpp", src, "-o", exe, f"-L{PKG}", "-lkvflow_driver", "-lkvflow_host",
                        "-lkvflow", f"-Wl,-rpath,{PKG}"], check=True)
    return exe


def run(exe):
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    return r.stdout


def test_host_api_cpu():
    out = run(build("test_host_cpu"))
    assert "20/20 test cases passed" in out or "test cases passed" in out


@pytest.mark.gpu
def test_host_api_gpu():
    run(build("test_host_gpu"))
