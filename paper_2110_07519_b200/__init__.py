"""B200-native MESSI exact 1-NN hot path (arXiv 2110.07519).

The product is ``libmessi.so`` (hand-written sm_100a CUDA behind the C-ABI in
include/messi.h); ``messi`` is its ctypes binding and ``dist`` the row-sharding /
cross-GPU merge plumbing over torch.distributed.  No CPU fallback exists.
"""
from .messi import (Index, MessiError, messi_build, messi_free, messi_query_dtw, messi_query_dtw_batch,  # noqa: F401
                    messi_query_ed, messi_query_ed_batch)

__all__ = ["Index", "MessiError", "messi_build", "messi_free", "messi_query_ed", "messi_query_dtw",
           "messi_query_ed_batch", "messi_query_dtw_batch"]
