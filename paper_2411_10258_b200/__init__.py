"""paper_2411_10258_b200 — B200-native (sm_100a) MDHP-GDS hot path (arxiv 2411.10258).

The product is ``lib/libmdhp.so`` (C ABI in ``include/mdhp.h``); this package is the thin
Python binding over it (``mdhp.py``).  No CPU fallback exists: without the CUDA extension and a
GPU every call raises.
"""
from .mdhp import (FitConfig, Packed, PackedSeq, fit, fit_host, hawkes_features,  # noqa: F401
                   launch_count, lib, loglik_dense, loglik_grad, make_desc, pack_windows,
                   packed_bytes, seq_chunk_hint, seq_fit, seq_loglik_grad, seq_pack)
from . import mdhp  # noqa: F401

__all__ = ["FitConfig", "Packed", "PackedSeq", "fit", "fit_host", "hawkes_features", "launch_count", "lib",
           "loglik_dense", "loglik_grad",
           "make_desc", "pack_windows", "packed_bytes", "seq_chunk_hint", "seq_fit", "seq_loglik_grad", "seq_pack", "mdhp"]
