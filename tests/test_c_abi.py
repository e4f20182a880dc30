"""The C-ABI from plain C: tests/c/abi_check.c includes include/kvflow.h and
include/kvflow_host.h as pedantic C99 (-Werror) and links libkvflow.so + libkvflow_host.so.
CPU: it must build and report the documented no-device failure (no CPU fallback).
GPU: it must move a node host -> HBM -> host through K1/K2 with matching checksums."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2507_07400_b200")


def build(tmp_path):
    if not shutil.which("gcc"):
        pytest.skip("no gcc")
    exe = str(tmp_path / "abi_check")
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Wextra", "-pedantic", "-Werror", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tests", "c", "abi_check.c"), "-o", exe, "-L", LIBDIR, "-lkvflow",
                        "-lkvflow_driver", "-lkvflow_host", f"-Wl,-rpath,{LIBDIR}"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    return exe


def gpu_present():
    from paper_2507_07400_b200.engine import device_count
    return device_count() > 0


def test_c_program_builds_and_fails_loudly_without_gpu(tmp_path):
    exe = build(tmp_path)
    if gpu_present():
        pytest.skip("GPU present (covered by the gpu variant)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0 and r.stdout.startswith("no-device 103"), r.stdout + r.stderr


@pytest.mark.gpu
def test_c_program_round_trip_on_gpu(tmp_path):
    exe = build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "round trip ok" in r.stdout, r.stdout + r.stderr
