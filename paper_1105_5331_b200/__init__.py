"""B200-native hot path of ALS-preconditioned N-GMRES for rank-R CP approximation
(arxiv/paper_1105_5331, reference proj/core/). See DESIGN.md.

The compute lives in lib/libcpfit_gpu.so (hand-written sm_100a CUDA behind the C-ABI in
include/cpfit_gpu.h); `api` is the Python mirror of the reference's C++ solver API.
"""
from . import api  # noqa: F401  (raises ImportError if the CUDA library was not built)
from .api import *  # noqa: F401,F403

__all__ = [n for n in dir(api) if not n.startswith("_")]
