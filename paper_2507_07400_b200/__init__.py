"""paper_2507_07400_b200 -- B200-native KVFlow KV-movement hot path.

Native pieces (built in-tree by __graft_entry__.build()):
  libkvflow.so       CUDA engine: K1 H2D gather, K2 D2H scatter, K3 HBM gather/scatter,
                     K4 priority propagation, K5 victim selection (include/kvflow.h)
  libkvflow_host.so  C++ control plane with the reference cache-manager API
                     (include/kvflow/*.hpp) + its C-ABI (include/kvflow_host.h)
"""
from ._native import KvfError, engine_lib, host_lib  # noqa: F401

__all__ = ["KvfError", "engine_lib", "host_lib"]
