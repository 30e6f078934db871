"""B200-native SuperVoxHenry hot path (arXiv 2105.08627).

libsvh.so (CUDA, sm_100a) behind the C-ABI in include/svh.h; ``svh`` is the
thin ctypes binding; ``parallel`` shards port solves over ranks.
"""
from . import svh  # noqa: F401

__all__ = ["svh"]
