"""B200-native hot path of arXiv 2405.08754 (hierarchical MIG x MPS partitioning + DQN
co-scheduling): libhrp (CUDA, sm_100a) behind a C ABI (include/hrp.h) and a thin ctypes
binding (hrp.py).  See DESIGN.md."""
from . import hrp  # noqa: F401
