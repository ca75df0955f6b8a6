"""fp64 CPU oracle for MDHP-GDS (arxiv 2411.10258) — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2411_10258_b200``) never imports it, and this package imports nothing from the
product path: the two share no code.  The C source is ``oracle/oracle.c``; this module is
only ctypes marshalling around it (numpy in, numpy out).

Functions (see oracle.c for the passages each one follows):
  convert_window   packing definition (Eq.(6), validation S:24-27)
  loglik_def       Eq.(5) P:290-296 written out, O(N^2), with analytic gradients
  loglik_rec       same quantity via the eager Ozaki-style recursion, O(N*D^2)
  fit              projected gradient ascent / Adam on lnL
  loglik_batch, fit_batch   pthread pools over CSR windows
  hawkes_features  MDHP-LSTM Hawkes gate, Eq.(7) third line P:431

Parity status: every function here is pinned by ``tests/test_oracle_pins.py`` (hand values,
closed forms, brute force, quadrature, finite differences, identities, library Adam).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

# status bits (oracle.c OR_*)
OK, EMPTY, UNSORTED, OUT_OF_RANGE, BAD_MARK = 0, 1, 2, 4, 8
SAME_DIM_TIE, DEGENERATE, NONFINITE, DIVERGED, CONVERGED, BAD_T = 16, 32, 64, 128, 256, 512
INVALID_MASK = UNSORTED | OUT_OF_RANGE | BAD_MARK | SAME_DIM_TIE | DEGENERATE | BAD_T
TIME_RAW, TIME_UNIT, TIME_EQ6 = 0, 1, 2


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (plain -O2, IEEE semantics, no fast-math)."""
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        cmd = f"gcc -O2 -ffp-contract=off -fPIC -shared -o {_LIB_PATH} {src} -lm -lpthread"
        rc = os.system(cmd)
        if rc != 0:
            raise RuntimeError(f"oracle build failed: {cmd}")
    return _LIB_PATH


class _FitCfg(ctypes.Structure):
    _fields_ = [
        ("max_iters", ctypes.c_int32), ("optimizer", ctypes.c_int32),
        ("lr", ctypes.c_double), ("b1", ctypes.c_double), ("b2", ctypes.c_double),
        ("eps", ctypes.c_double), ("loss_mean", ctypes.c_int32), ("tol_rel", ctypes.c_double),
        ("patience", ctypes.c_int32), ("min_param", ctypes.c_double),
        ("fit_mask", ctypes.c_uint32), ("max_halvings", ctypes.c_int32),
        ("use_def", ctypes.c_int32),
    ]


@dataclass
class FitConfig:
    """Optimizer definition shared *by specification* with the GPU path.
    Defaults follow SPEC S:182-185 (Adam, lr 0.05, floor 1e-4, tol 1e-6, patience 10)."""
    max_iters: int = 300
    optimizer: str = "adam"        # "gd" | "adam"
    lr: float = 0.05
    b1: float = 0.9
    b2: float = 0.999
    eps: float = 1e-8
    loss: str = "sum"              # "sum" (-lnL) | "mean" (-lnL/N)
    tol_rel: float = 1e-6
    patience: int = 10
    min_param: float = 1e-4
    fit_mask: int = 7              # 1 theta | 2 alpha | 4 beta
    max_halvings: int = 8
    use_def: bool = False

    def _c(self) -> _FitCfg:
        return _FitCfg(self.max_iters, 1 if self.optimizer == "adam" else 0, self.lr, self.b1,
                       self.b2, self.eps, 1 if self.loss == "mean" else 0, self.tol_rel,
                       self.patience, self.min_param, self.fit_mask, self.max_halvings,
                       1 if self.use_def else 0)


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        L.oracle_convert_window.restype = ctypes.c_int
        L.oracle_convert_window.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                            ctypes.c_double, ctypes.c_int, ctypes.c_int64, P, P,
                                            ctypes.c_double, P, P]
        for name in ("oracle_loglik_def", "oracle_loglik_rec"):
            f = getattr(L, name)
            f.restype = ctypes.c_double
            f.argtypes = [ctypes.c_int, ctypes.c_int64, P, P, ctypes.c_double, P, P, P, P, P, P, P]
        L.oracle_fit.restype = ctypes.c_int
        L.oracle_fit.argtypes = [ctypes.c_int, ctypes.c_int64, P, P, ctypes.c_double,
                                 ctypes.POINTER(_FitCfg), P, P, P, P, P, P]
        L.oracle_loglik_batch.restype = None
        L.oracle_loglik_batch.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64, P, P, P, P,
                                          P, P, P, P, P, P, P, ctypes.c_int]
        L.oracle_fit_batch.restype = None
        L.oracle_fit_batch.argtypes = [ctypes.c_int, ctypes.c_int64, P, P, P, P,
                                       ctypes.POINTER(_FitCfg), P, P, P, P, P, P, ctypes.c_int]
        L.oracle_hawkes_features.restype = None
        L.oracle_hawkes_features.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int, P, P, P,
                                             P, P, P, P, P, P]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


TIE_ERROR, TIE_NUDGE = 0, 1


def convert_window(D, t, mark, T, time_mode=TIME_RAW, lo=0.0, hi=1.0, tie_policy=TIE_ERROR):
    """-> (t32 float32[n], T32 float, status int).  Packing definition (oracle.c)."""
    t = _f64(t)
    mark = np.ascontiguousarray(mark, dtype=np.int32)
    out = np.zeros(len(t), dtype=np.float32)
    T32 = np.zeros(1, dtype=np.float32)
    st = lib().oracle_convert_window(int(D), int(time_mode), float(lo), float(hi), int(tie_policy), len(t),
                                     _p(t), _p(mark), float(T), _p(out), _p(T32))
    return out, float(T32[0]), int(st)


def _times(t):
    """Times as fp64: fp32 analysis times are promoted exactly; fp64 times pass through."""
    return np.ascontiguousarray(np.asarray(t), dtype=np.float64)


def _ll(fn, D, t32, mark, T, theta, alpha, beta, grads=True):
    t32 = _times(t32)
    mark = np.ascontiguousarray(mark, dtype=np.int32)
    theta, alpha, beta = _f64(theta).ravel(), _f64(alpha).ravel(), _f64(beta).ravel()
    gt = np.zeros(D) if grads else None
    ga = np.zeros(D * D) if grads else None
    gb = np.zeros(D * D) if grads else None
    gam = np.zeros(1)
    val = fn(int(D), len(t32), _p(t32), _p(mark), float(T), _p(theta), _p(alpha), _p(beta),
             _p(gt), _p(ga), _p(gb), _p(gam))
    out = {"lnl": float(val), "gamma": float(gam[0])}
    if grads:
        out.update(g_theta=gt, g_alpha=ga.reshape(D, D), g_beta=gb.reshape(D, D))
    return out


def loglik_def(D, t32, mark, T, theta, alpha, beta, grads=True):
    """Eq.(5) written out (O(N^2)).  Returns dict(lnl, gamma, g_theta, g_alpha, g_beta)."""
    return _ll(lib().oracle_loglik_def, D, t32, mark, T, theta, alpha, beta, grads)


def loglik_rec(D, t32, mark, T, theta, alpha, beta, grads=True):
    """Eager recursion (O(N*D^2)); same outputs as loglik_def."""
    return _ll(lib().oracle_loglik_rec, D, t32, mark, T, theta, alpha, beta, grads)


def fit(D, t32, mark, T, theta, alpha, beta, cfg: FitConfig, trace=False):
    t32 = _times(t32)
    mark = np.ascontiguousarray(mark, dtype=np.int32)
    th, al, be = _f64(theta).ravel().copy(), _f64(alpha).ravel().copy(), _f64(beta).ravel().copy()
    lnl = np.zeros(1)
    it = np.zeros(1, dtype=np.int32)
    tr = np.full(max(cfg.max_iters, 1), np.nan) if trace else None
    c = cfg._c()
    st = lib().oracle_fit(int(D), len(t32), _p(t32), _p(mark), float(T), ctypes.byref(c),
                          _p(th), _p(al), _p(be), _p(lnl), _p(it), _p(tr))
    out = {"theta": th, "alpha": al.reshape(D, D), "beta": be.reshape(D, D),
           "lnl": float(lnl[0]), "iters": int(it[0]), "status": int(st)}
    if trace:
        out["trace"] = tr[~np.isnan(tr)]   # includes the evaluation that triggered a stop
    return out


def loglik_batch(D, t32, mark, win_off, T, theta, alpha, beta, nthreads=None, use_def=False,
                 grads=True):
    W = len(win_off) - 1
    nthreads = nthreads or os.cpu_count() or 1
    t32 = _times(t32)
    mark = np.ascontiguousarray(mark, dtype=np.int32)
    off = np.ascontiguousarray(win_off, dtype=np.int64)
    T = _f64(T)
    theta, alpha, beta = _f64(theta), _f64(alpha), _f64(beta)
    lnl = np.zeros(W)
    gt = np.zeros((W, D)) if grads else None
    ga = np.zeros((W, D, D)) if grads else None
    gb = np.zeros((W, D, D)) if grads else None
    lib().oracle_loglik_batch(1 if use_def else 0, int(D), W, _p(t32), _p(mark), _p(off), _p(T),
                              _p(theta), _p(alpha), _p(beta), _p(lnl), _p(gt), _p(ga), _p(gb),
                              int(nthreads))
    return {"lnl": lnl, "g_theta": gt, "g_alpha": ga, "g_beta": gb}


def fit_batch(D, t32, mark, win_off, T, theta, alpha, beta, cfg: FitConfig, nthreads=None):
    W = len(win_off) - 1
    nthreads = nthreads or os.cpu_count() or 1
    t32 = _times(t32)
    mark = np.ascontiguousarray(mark, dtype=np.int32)
    off = np.ascontiguousarray(win_off, dtype=np.int64)
    T = _f64(T)
    th = _f64(theta).copy()
    al = _f64(alpha).copy()
    be = _f64(beta).copy()
    lnl = np.zeros(W)
    iters = np.zeros(W, dtype=np.int32)
    status = np.zeros(W, dtype=np.int32)
    c = cfg._c()
    lib().oracle_fit_batch(int(D), W, _p(t32), _p(mark), _p(off), _p(T), ctypes.byref(c),
                           _p(th), _p(al), _p(be), _p(lnl), _p(iters), _p(status), int(nthreads))
    return {"theta": th, "alpha": al, "beta": be, "lnl": lnl, "iters": iters, "status": status}


def hawkes_features(D, theta, alpha, beta, T_span, A, B, C, gross=False):
    """Eq.(7) third line per window: hks[w] = tanh(A alpha_w - B (beta_w T_w) + C theta_w).
    theta [W][D], alpha/beta [W][D][D], T_span [W], A/B [H][D*D], C [H][D].  -> hks [W][H]
    (and sum_k |W_hk X_wk| [W][H] when gross=True).  oracle.c: oracle_hawkes_features."""
    theta = _f64(theta).reshape(-1, D)
    W = theta.shape[0]
    alpha = _f64(alpha).reshape(W, D * D)
    beta = _f64(beta).reshape(W, D * D)
    T_span = _f64(T_span).reshape(W)
    A = _f64(A).reshape(-1, D * D)
    H = A.shape[0]
    B = _f64(B).reshape(H, D * D)
    C = _f64(C).reshape(H, D)
    out = np.empty((W, H))
    g = np.empty((W, H)) if gross else None
    lib().oracle_hawkes_features(int(D), W, H, _p(theta), _p(alpha), _p(beta), _p(T_span), _p(A),
                                 _p(B), _p(C), _p(out), _p(g))
    return (out, g) if gross else out
