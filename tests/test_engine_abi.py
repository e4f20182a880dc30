"""CPU-side checks of the C-ABI boundary: the library loads, exports every symbol
include/kvflow.h declares, and fails loudly (no CPU fallback) without a GPU."""
import ctypes
import os
import re

import pytest

from paper_2507_07400_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header):
    txt = open(os.path.join(ROOT, "include", header)).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(kvf\w*)\s*\(", txt, re.M)))


def test_engine_exports_every_declared_symbol():
    lib = ctypes.CDLL(N.ENGINE_SO)
    names = declared("kvflow.h")
    assert len(names) >= 25
    for name in names:
        assert hasattr(lib, name), name
    # and the Python bindings cover all of them
    assert set(names) <= set(N._ENGINE_SIGS)


def test_engine_refuses_without_gpu():
    from paper_2507_07400_b200.engine import Engine, device_count
    if device_count() > 0:
        pytest.skip("GPU present")
    with pytest.raises(N.KvfError) as ex:
        Engine(gpu_slots=16, host_slots=16)
    assert ex.value.code == N.KVF_E_NO_DEVICE
