"""In-tree build of the native libraries (no JIT cache: the .so files travel with gpurun).

  python -m paper_2507_07400_b200.build          # engine + host + oracle (+ oracle/_ref here)

libkvflow.so       nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3  (csrc/engine/*.cu)
libkvflow_host.so  g++ -std=c++20 -O2, links libkvflow.so                      (csrc/host/*.cpp)
libkvflow_driver.so  harness: workload generator + driver C-ABI, links both  (csrc/driver/*.cpp)
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


def _parallel(jobs):
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 4))) as ex:
        for f in [ex.submit(_run, j) for j in jobs]:
            f.result()


def build_engine(force=False):
    """One nvcc per .cu in parallel (objects under build/), then one shared link."""
    srcs = sorted(glob.glob(os.path.join(PKG, "csrc", "engine", "*.cu")))
    hdrs = glob.glob(os.path.join(PKG, "csrc", "engine", "*.hpp")) + \
        glob.glob(os.path.join(PKG, "csrc", "engine", "*.cuh")) + [os.path.join(INC, "kvflow.h")]
    out = os.path.join(PKG, "libkvflow.so")
    objdir = os.path.join(ROOT, "build", "engine")
    os.makedirs(objdir, exist_ok=True)
    objs, jobs = [], []
    for s in srcs:
        o = os.path.join(objdir, os.path.basename(s)[:-3] + ".o")
        objs.append(o)
        if force or _stale(o, [s] + hdrs):
            jobs.append([NVCC, *ARCH, "-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC", f"-I{INC}",
                         "-c", s, "-o", o])
    _parallel(jobs)
    if force or _stale(out, objs):
        _run([NVCC, *ARCH, "-shared", *objs, "-o", out])
    return out


GXX = ["g++", "-std=c++20", "-O2", "-g", "-fPIC", "-shared", "-Wall", "-Wextra", "-Wno-unused-parameter"]


def build_host(force=False):
    """libkvflow_host.so: the product control plane (csrc/host: cache, tier manager, step graph,
    cost model, scheduler).  libkvflow_driver.so: harness on top of it (csrc/driver: the
    synthetic workload generator and the lockstep-driver C-ABI of include/kvflow_host.h)."""
    hdrs = glob.glob(os.path.join(INC, "kvflow", "*.hpp")) + [os.path.join(INC, "kvflow.h"),
                                                             os.path.join(INC, "kvflow_host.h")]
    srcs = sorted(glob.glob(os.path.join(PKG, "csrc", "host", "*.cpp")))
    out = os.path.join(PKG, "libkvflow_host.so")
    if force or _stale(out, srcs + hdrs + [os.path.join(PKG, "libkvflow.so")]):
        _run([*GXX, f"-I{INC}", *srcs, "-o", out, f"-L{PKG}", "-lkvflow", "-Wl,-rpath,$ORIGIN"])
    dsrcs = sorted(glob.glob(os.path.join(PKG, "csrc", "driver", "*.cpp")))
    dout = os.path.join(PKG, "libkvflow_driver.so")
    if force or _stale(dout, dsrcs + hdrs + [out]):
        _run([*GXX, f"-I{INC}", *dsrcs, "-o", dout, f"-L{PKG}", "-lkvflow_host", "-lkvflow", "-Wl,-rpath,$ORIGIN"])
    return dout


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
