"""GPU input synthesis (libmdhp_synth.so, include/synth.h): seeded Ogata-thinned MDHP windows at
the scale of BASELINE.json's configs.  Input generation only (not the hot path)."""
from __future__ import annotations

import ctypes
import os
import subprocess

import torch

from .gen import CONFIGS, STRATEGIES, Recipe

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = os.path.join(HERE, "csrc", "synth.cu")
LIB = os.path.join(HERE, "lib", "libmdhp_synth.so")
_lib = None


def build(force=False) -> str:
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    hdr = os.path.join(ROOT, "include", "synth.h")
    if force or not os.path.exists(LIB) or max(os.path.getmtime(SRC), os.path.getmtime(hdr)) > os.path.getmtime(LIB):
        cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
               "-Xcompiler", "-fPIC", "-shared", "-o", LIB, SRC]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed: " + r.stderr)
    return LIB


class _Recipe(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in ("total_rate", "rate_lo", "rate_hi", "beta_lo", "beta_hi",
                                                "g_self_lo", "g_self_hi", "g_cross_lo", "g_cross_hi",
                                                "rho", "attack_frac", "rho_attack")] + \
               [("k_cross", ctypes.c_int32), ("n_attack", ctypes.c_int32)]


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        P = ctypes.c_void_p
        L.synth_params.restype = ctypes.c_int
        L.synth_params.argtypes = [ctypes.c_int32, ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64,
                                   ctypes.POINTER(_Recipe), P, P, P, P, P]
        L.synth_ogata.restype = ctypes.c_int
        L.synth_ogata.argtypes = [ctypes.c_int32, ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64,
                                  ctypes.c_double, P, P, P, ctypes.c_int64, P, P, P, P, P]
        L.synth_ogata_inject.restype = ctypes.c_int
        L.synth_ogata_inject.argtypes = [ctypes.c_int32, ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64,
                                         ctypes.c_double, P, P, P, ctypes.c_int64, P, P, P, P, P,
                                         ctypes.c_int32, ctypes.c_double, P]
        L.synth_npp.restype = ctypes.c_int
        L.synth_npp.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int32, ctypes.c_double,
                                P, P, P, P]
        L.synth_last_error.restype = ctypes.c_char_p
        _lib = L
    return _lib


def _p(x):
    return None if x is None else ctypes.c_void_p(x.data_ptr())


def _check(rc, what):
    if rc != 0:
        raise RuntimeError(f"{what}: {lib().synth_last_error().decode()}")


def recipe_c(rc: Recipe) -> _Recipe:
    return _Recipe(rc.total_rate, rc.rate_lo, rc.rate_hi, rc.beta_lo, rc.beta_hi, rc.g_self[0], rc.g_self[1],
                   rc.g_cross[0], rc.g_cross[1], rc.rho, rc.attack_frac, rc.rho_attack, rc.k_cross, rc.n_attack)


def make_batch_gpu(rc: Recipe | str, W: int, seed: int = 2024, first_window: int = 0, device="cuda",
                   params=None, max_events=None, stream=None):
    """Simulate W windows on the GPU.  Returns dict of device tensors: t f64[E], mark i32[E],
    win_off i64[W+1], T f64[W], theta f32[W,D], alpha/beta f32[W,D,D], attack u8[W]."""
    if isinstance(rc, str):
        rc = CONFIGS[rc]
    D = rc.D
    st = ctypes.c_void_p((stream or torch.cuda.current_stream()).cuda_stream)
    if params is None:
        th = torch.empty(W, D, dtype=torch.float32, device=device)
        al = torch.empty(W, D, D, dtype=torch.float32, device=device)
        be = torch.empty(W, D, D, dtype=torch.float32, device=device)
        att = torch.empty(W, dtype=torch.uint8, device=device)
        c = recipe_c(rc)
        _check(lib().synth_params(D, W, first_window, seed, ctypes.byref(c), _p(th), _p(al), _p(be), _p(att), st),
               "synth_params")
    else:
        th, al, be = (params[k].to(device=device, dtype=torch.float32).contiguous() for k in ("theta", "alpha", "beta"))
        att = torch.zeros(W, dtype=torch.uint8, device=device)
    cap = int(max_events or max(64, 16 * rc.total_rate * rc.T + 2 * rc.inj_rate))
    counts = torch.empty(W, dtype=torch.int64, device=device)
    strat = STRATEGIES[rc.inject]
    att_p = _p(att) if strat else None
    _check(lib().synth_ogata_inject(D, W, first_window, seed, rc.T, _p(th), _p(al), _p(be), cap, None,
                                    _p(counts), None, None, att_p, strat, rc.inj_rate, st),
           "synth_ogata(count)")
    if bool((counts < 0).any()):
        raise RuntimeError("synth_ogata: a window exceeded max_events")
    off = torch.zeros(W + 1, dtype=torch.int64, device=device)
    torch.cumsum(counts, 0, out=off[1:])
    E = int(off[-1])
    t = torch.empty(max(E, 1), dtype=torch.float64, device=device)[:E]
    m = torch.empty(max(E, 1), dtype=torch.int32, device=device)[:E]
    _check(lib().synth_ogata_inject(D, W, first_window, seed, rc.T, _p(th), _p(al), _p(be), cap, _p(off),
                                    _p(counts), _p(t), _p(m), att_p, strat, rc.inj_rate, st),
           "synth_ogata(write)")
    T = torch.full((W,), rc.T, dtype=torch.float64, device=device)
    return {"D": D, "t": t, "mark": m, "win_off": off, "T": T, "theta": th, "alpha": al, "beta": be,
            "attack": att}


def npp_gpu(strategy: str, W: int, seed: int = 2024, first_window: int = 0, rate: float = 512.0, device="cuda"):
    """Algorithm 4 injection times alone (normalised u in [0, 1]) for W windows -> (u f64[E], off i64[W+1]),
    the same streams synth_ogata_inject superposes on attack windows."""
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    counts = torch.empty(W, dtype=torch.int64, device=device)
    k = STRATEGIES[strategy]
    _check(lib().synth_npp(W, first_window, seed, k, rate, None, _p(counts), None, st), "synth_npp(count)")
    off = torch.zeros(W + 1, dtype=torch.int64, device=device)
    torch.cumsum(counts, 0, out=off[1:])
    u = torch.empty(max(int(off[-1]), 1), dtype=torch.float64, device=device)
    _check(lib().synth_npp(W, first_window, seed, k, rate, _p(off), _p(counts), _p(u), st), "synth_npp(write)")
    return u[:int(off[-1])], off
