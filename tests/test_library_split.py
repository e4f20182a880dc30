"""The product control plane carries no harness code: the synthetic
workload generator (WorkloadController, SURVEY §2 out of scope) and the lockstep driver's
C-ABI live in libkvflow_driver.so; libkvflow_host.so is the cache, tier manager, step graph,
cost model and scheduler (fed by a RequestSource).  CPU-only: reads the dynamic symbols."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2507_07400_b200")


def dyn_symbols(lib):
    path = os.path.join(PKG, lib)
    if not os.path.exists(path):
        pytest.skip(f"{lib} not built")
    out = subprocess.run(["nm", "-DC", "--defined-only", path], capture_output=True, text=True, check=True).stdout
    return out


def test_host_library_has_no_workload_generator_or_driver_abi():
    host = dyn_symbols("libkvflow_host.so")
    assert "WorkloadController" not in host
    assert "kvfh_sim_create" not in host
    assert "kvf::RadixCache::evict" in host and "kvf::Simulator::run" in host
    assert "kvf::Simulator::Simulator(kvf::CostModel const&, kvf::SchedulerConfig const&, std::unique_ptr<kvf::RequestSource" in host


def test_driver_library_holds_the_harness():
    drv = dyn_symbols("libkvflow_driver.so")
    assert "kvf::WorkloadController::start" in drv
    assert "kvfh_sim_create" in drv
    # the reference-signature constructor (WorkloadSpec + seed) is harness-side
    assert "kvf::Simulator::Simulator(kvf::CostModel const&, kvf::SchedulerConfig const&, kvf::WorkloadSpec const&" in drv
