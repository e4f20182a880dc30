"""In-tree build of the native libraries (no JIT cache: the .so files travel with gpurun).

  python -m paper_2507_07400_b200.build          # engine + host + oracle (+ oracle/_ref here)

libkvflow.so       nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3  (csrc/engine/*.cu)
libkvflow_host.so  g++ -std=c++20 -O2, links libkvflow.so                      (csrc/host/*.cpp)
oracle/liboracle.so, oracle/_ref/*  test infrastructure (make -C oracle)
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
INC = os.path.join(ROOT, "include")
NVCC = os.environ.get("NVCC", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _run(cmd, cwd=None):
    r = subprocess.run(cmd, cwd=cwd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {cmd[0]} (exit {r.returncode})")
    return r


def _stale(out, srcs):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(s) > t for s in srcs)


def build_engine(force=False):
    srcs = sorted(glob.glob(os.path.join(PKG, "csrc", "engine", "*.cu")))
    deps = srcs + glob.glob(os.path.join(PKG, "csrc", "engine", "*.hpp")) + [os.path.join(INC, "kvflow.h")]
    out = os.path.join(PKG, "libkvflow.so")
    if force or _stale(out, deps):
        _run([NVCC, *ARCH, "-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-shared", f"-I{INC}",
              *srcs, "-o", out])
    return out


def build_host(force=False):
    srcs = sorted(glob.glob(os.path.join(PKG, "csrc", "host", "*.cpp")))
    if not srcs:
        return None
    deps = srcs + glob.glob(os.path.join(INC, "kvflow", "*.hpp")) + [os.path.join(INC, "kvflow.h"),
                                                                     os.path.join(INC, "kvflow_host.h"),
                                                                     os.path.join(PKG, "libkvflow.so")]
    deps = [d for d in deps if os.path.exists(d)]
    out = os.path.join(PKG, "libkvflow_host.so")
    if force or _stale(out, deps):
        _run(["g++", "-std=c++20", "-O2", "-g", "-fPIC", "-shared", "-Wall", "-Wextra", "-Wno-unused-parameter",
              f"-I{INC}", *srcs, "-o", out, f"-L{PKG}", "-lkvflow", "-Wl,-rpath,$ORIGIN",
              ])
    return out


def build_oracle():
    _run(["make", "-C", os.path.join(ROOT, "oracle"), "liboracle.so"])
    if os.path.isdir("/root/reference/proj/src"):
        _run(["make", "-C", os.path.join(ROOT, "oracle"), "ref", "suites"])
        # the reference's own unit suites against OUR host API (tests/refsuite/README.md)
        _run(["make", "-C", os.path.join(ROOT, "tests", "refsuite")])


def build_all(force=False):
    build_engine(force)
    build_host(force)
    build_oracle()


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
    print("built:", ", ".join(os.path.basename(p) for p in glob.glob(os.path.join(PKG, "*.so"))))
