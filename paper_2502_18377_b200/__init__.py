"""B200-native NeuRLP-PDE batched solve (Mechanistic PDE Networks, arXiv 2502.18377).

The hot path lives in ``libmpde.so`` (CUDA C++, sm_100a) behind the C ABI declared in
``include/mpde.h``; ``mpde`` is the thin ctypes binding with the same names.
"""
from . import mpde  # noqa: F401
from .mpde import NeuRLPSolve, Solver  # noqa: F401
