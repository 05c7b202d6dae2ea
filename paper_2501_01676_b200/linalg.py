"""Error type of the reference's dense kernels (reference linalg.py:11).

The dense kernels themselves (pseudo_inverse, parallel_sum, sym_pencil_gevp)
run inside the per-glob CUDA kernels (csrc/globs.cu, csrc/dense_block.cuh)."""

from .engine import NumericalError

__all__ = ["NumericalError"]
