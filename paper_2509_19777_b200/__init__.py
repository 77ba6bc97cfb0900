"""B200-native hPLMM-preconditioned GMRES (arXiv 2509.19777).

The product is ``libhplmm.so`` (C ABI in ``include/hplmm.h``, CUDA for
sm_100a); ``hplmm`` is its thin ctypes binding.  Nothing here imports the
oracle, and there is no CPU fallback.
"""
from .hplmm import ART, OP, HPLMMError, Solver, assemble_bsr, default_options, load  # noqa: F401

__all__ = ["Solver", "load", "default_options", "OP", "ART", "HPLMMError"]
