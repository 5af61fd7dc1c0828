"""B200-native (sm_100a) DiffKV KV memory manager (arXiv 2412.03131): C-ABI library + thin binding.

The hot path — classify, compact+alloc, quant-write — runs in hand-written CUDA kernels inside
``libdkv.so`` (built in-tree from ``csrc/``).  Importing this package fails if the library is missing.
"""
from . import dkv  # noqa: F401  (raises ImportError if libdkv.so is missing)
from .dkv import *  # noqa: F401,F403
from .pool import Pool, decisions_to_numpy  # noqa: F401
