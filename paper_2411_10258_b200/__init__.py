"""paper_2411_10258_b200 — B200-native (sm_100a) MDHP-GDS hot path (arxiv 2411.10258).

The product is ``lib/libmdhp.so`` (C ABI in ``include/mdhp.h``); this package is the thin
Python binding over it (``mdhp.py``).  No CPU fallback exists: without the CUDA extension and a
GPU every call raises.
"""
from .mdhp import (FitConfig, Packed, fit, fit_host, launch_count, lib, loglik_grad,  # noqa: F401
                   make_desc, pack_windows, packed_bytes)
from . import mdhp  # noqa: F401

__all__ = ["FitConfig", "Packed", "fit", "fit_host", "launch_count", "lib", "loglik_grad",
           "make_desc", "pack_windows", "packed_bytes", "mdhp"]
