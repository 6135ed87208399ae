"""contactamg-b200: B200-native (sm_100a) solve path of the fully coupled
saddle-point AMG for mortar contact / mesh-tying systems (arXiv:1912.09056),
behind the reference package's Python API (`contactamg`).

Compute runs in `libcamg.so` (hand-written CUDA, C ABI in include/camg.h);
PyTorch provides device memory and streams only.
"""

from .sparse import BlockVector, SparseMatrix

__all__ = ["SparseMatrix", "BlockVector"]
__version__ = "0.1.0"
