"""Thin Python binding of libmdhp.so (include/mdhp.h): argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; torch provides device memory
and streams.  There is no CPU fallback: if the extension is missing or no CUDA device is
present the calls raise.  Function names follow the C ABI.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

from . import build as _build

# status bits (include/mdhp.h)
ST_OK, ST_EMPTY, ST_UNSORTED, ST_OUT_OF_RANGE, ST_BAD_MARK = 0, 1, 2, 4, 8
ST_SAME_DIM_TIE, ST_DEGENERATE, ST_NONFINITE, ST_DIVERGED, ST_CONVERGED, ST_BAD_T = 16, 32, 64, 128, 256, 512
ST_INVALID = ST_UNSORTED | ST_OUT_OF_RANGE | ST_BAD_MARK | ST_SAME_DIM_TIE | ST_DEGENERATE | ST_BAD_T
TIME_RAW, TIME_UNIT, TIME_EQ6 = 0, 1, 2
TIE_ERROR, TIE_NUDGE = 0, 1
OPT_GD, OPT_ADAM = 0, 1
FIT_THETA, FIT_ALPHA, FIT_BETA = 1, 2, 4


class PackDesc(ctypes.Structure):
    _fields_ = [("D", ctypes.c_int32), ("time_mode", ctypes.c_int32),
                ("n_windows", ctypes.c_int64), ("n_events", ctypes.c_int64),
                ("eq6_lo", ctypes.c_double), ("eq6_hi", ctypes.c_double),
                ("tie_policy", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class SeqDesc(ctypes.Structure):
    _fields_ = [("D", ctypes.c_int32), ("chunk_events", ctypes.c_int32),
                ("n_events", ctypes.c_int64), ("T", ctypes.c_double), ("t0", ctypes.c_double),
                ("has_history", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class FitConfigC(ctypes.Structure):
    _fields_ = [("max_iters", ctypes.c_int32), ("optimizer", ctypes.c_int32),
                ("lr", ctypes.c_float), ("adam_b1", ctypes.c_float), ("adam_b2", ctypes.c_float),
                ("adam_eps", ctypes.c_float), ("loss_mean", ctypes.c_int32),
                ("tol_rel", ctypes.c_float), ("patience", ctypes.c_int32),
                ("min_param", ctypes.c_float), ("fit_mask", ctypes.c_uint32),
                ("max_halvings", ctypes.c_int32), ("adam_step0", ctypes.c_int32),
                ("time_chunks", ctypes.c_int32)]


@dataclass
class FitConfig:
    """mdhp_fit_config.  Defaults follow SPEC S:182-185 (Adam, lr 0.05, floor 1e-4,
    tol 1e-6, patience 10); DESIGN.md "Fit" defines the loop."""
    max_iters: int = 300
    optimizer: str = "adam"
    lr: float = 0.05
    b1: float = 0.9
    b2: float = 0.999
    eps: float = 1e-8
    loss: str = "sum"
    tol_rel: float = 1e-6
    patience: int = 10
    min_param: float = 1e-4
    fit_mask: int = 7
    max_halvings: int = 8
    adam_step0: int = 0        # Adam steps already taken when resuming from a returned opt_state
    time_chunks: int = 0        # time chunks per window (D <= 8): 0 = throughput layout
    latency_mode: bool = False  # shorthand for the most time chunks (one window per warp)

    def c(self) -> FitConfigC:
        return FitConfigC(self.max_iters, OPT_ADAM if self.optimizer == "adam" else OPT_GD,
                          self.lr, self.b1, self.b2, self.eps, 1 if self.loss == "mean" else 0,
                          self.tol_rel, self.patience, self.min_param, self.fit_mask,
                          self.max_halvings, self.adam_step0, 32 if self.latency_mode else self.time_chunks)


_lib = None


def lib() -> ctypes.CDLL:
    """Load libmdhp.so (building it with nvcc if stale).  Raises if it cannot be loaded."""
    global _lib
    if _lib is None:
        path = os.environ.get("MDHP_LIB") or _build.LIB   # MDHP_LIB: A/B experiments only
        if not os.path.exists(path):
            path = _build.build()
        L = ctypes.CDLL(path)
        P, I64, I32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
        L.mdhp_packed_bytes.restype = ctypes.c_size_t
        L.mdhp_packed_bytes.argtypes = [ctypes.POINTER(PackDesc)]
        L.mdhp_pack_windows.restype = ctypes.c_int
        L.mdhp_pack_windows.argtypes = [ctypes.POINTER(PackDesc), P, P, P, P, P, ctypes.c_size_t, P, P]
        L.mdhp_loglik_grad.restype = ctypes.c_int
        L.mdhp_loglik_grad.argtypes = [ctypes.POINTER(PackDesc), P, P, P, P, P, P, P, P, P, P]
        L.mdhp_loglik_exact.restype = ctypes.c_int
        L.mdhp_loglik_exact.argtypes = [ctypes.POINTER(PackDesc), P, P, P, P, P, P, P, P, P, P]
        L.mdhp_loglik_dense.restype = ctypes.c_int
        L.mdhp_loglik_dense.argtypes = [ctypes.POINTER(PackDesc), P, P, P, P, P, P, P]
        L.mdhp_hawkes_features.restype = ctypes.c_int
        L.mdhp_hawkes_features.argtypes = [ctypes.c_int32, ctypes.c_int64, ctypes.c_int32, P, P, P, P,
                                           P, P, P, P, P]
        L.mdhp_fit.restype = ctypes.c_int
        L.mdhp_fit.argtypes = [ctypes.POINTER(PackDesc), P, ctypes.POINTER(FitConfigC), P, P, P, P, P,
                               P, P, P, P]
        L.mdhp_fit_host.restype = ctypes.c_int
        L.mdhp_fit_host.argtypes = [ctypes.POINTER(PackDesc), P, P, P, P, ctypes.POINTER(FitConfigC),
                                    P, P, P, P, P, P, P]
        L.mdhp_seq_packed_bytes.restype = ctypes.c_size_t
        L.mdhp_seq_packed_bytes.argtypes = [ctypes.POINTER(SeqDesc)]
        L.mdhp_seq_chunk_hint.restype = ctypes.c_int32
        L.mdhp_seq_chunk_hint.argtypes = [ctypes.c_int32, ctypes.c_int64]
        L.mdhp_seq_pack.restype = ctypes.c_int
        L.mdhp_seq_pack.argtypes = [ctypes.POINTER(SeqDesc), P, P, P, ctypes.c_size_t, P, P]
        L.mdhp_seq_loglik_grad.restype = ctypes.c_int
        L.mdhp_seq_loglik_grad.argtypes = [ctypes.POINTER(SeqDesc), P, P, P, P, P, P, P, P, P]
        L.mdhp_seq_fit.restype = ctypes.c_int
        L.mdhp_seq_fit.argtypes = [ctypes.POINTER(SeqDesc), P, ctypes.POINTER(FitConfigC), P, P, P, P, P,
                                   P, P, P, P]
        L.mdhp_seq_work_bytes.restype = ctypes.c_size_t
        L.mdhp_seq_work_bytes.argtypes = [ctypes.POINTER(SeqDesc)]
        L.mdhp_seq_work_init.restype = ctypes.c_int
        L.mdhp_seq_work_init.argtypes = [ctypes.POINTER(SeqDesc), P, ctypes.POINTER(FitConfigC), P]
        L.mdhp_seq_maps.restype = ctypes.c_int
        L.mdhp_seq_maps.argtypes = [ctypes.POINTER(SeqDesc), P, P, P, P, P, ctypes.c_int32, P]
        L.mdhp_seq_parts.restype = ctypes.c_int
        L.mdhp_seq_parts.argtypes = [ctypes.POINTER(SeqDesc), P, P, P, P, P, P, ctypes.c_int32, P, P, P,
                                     ctypes.c_int32, ctypes.c_int32, P]
        L.mdhp_seq_stats.restype = ctypes.c_int
        L.mdhp_seq_stats.argtypes = [ctypes.POINTER(SeqDesc), P, P, P]
        L.mdhp_seq_stats_combine.restype = ctypes.c_int
        L.mdhp_seq_stats_combine.argtypes = [ctypes.c_int32, ctypes.c_int32, P, P, P]
        L.mdhp_seq_finish.restype = ctypes.c_int
        L.mdhp_seq_finish.argtypes = [ctypes.POINTER(SeqDesc), ctypes.c_int64, P, P, P, P, P, P, P, P, P, P,
                                      ctypes.POINTER(FitConfigC), P, P, P, P, P, ctypes.c_int32, P, P]
        L.mdhp_packed_layout.restype = ctypes.c_int
        L.mdhp_packed_layout.argtypes = [ctypes.POINTER(PackDesc), P]
        L.mdhp_last_error.restype = ctypes.c_char_p
        L.mdhp_launch_count.restype = ctypes.c_uint64
        L.mdhp_version.restype = I32
        _lib = L
    return _lib


def _check(rc: int, what: str):
    if rc != 0:
        raise RuntimeError(f"{what} failed (rc={rc}): {lib().mdhp_last_error().decode()}")


def _ptr(x):
    if x is None:
        return None
    return ctypes.c_void_p(x.data_ptr())


def _dev(x, dtype, name):
    if not isinstance(x, torch.Tensor) or not x.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if x.dtype != dtype or not x.is_contiguous():
        raise TypeError(f"{name} must be a contiguous {dtype} tensor")
    return x


def _size(x, n, name):
    """ValueError unless tensor x holds exactly n elements (the C side trusts the sizes)."""
    if x is not None and x.numel() != n:
        raise ValueError(f"{name} has {x.numel()} elements, expected {n}")
    return x


def _params(W, D, theta, alpha, beta):
    for nm, x in (("theta", theta), ("alpha", alpha), ("beta", beta)):
        _dev(x, torch.float32, nm)
    _size(theta, W * D, "theta"); _size(alpha, W * D * D, "alpha"); _size(beta, W * D * D, "beta")


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def launch_count() -> int:
    return int(lib().mdhp_launch_count())


@dataclass
class Packed:
    """A packed batch: the device buffer plus the descriptor it was packed with."""
    desc: PackDesc
    buf: torch.Tensor          # uint8 device buffer
    status: torch.Tensor       # int32 [W] device

    @property
    def D(self):
        return int(self.desc.D)

    @property
    def W(self):
        return int(self.desc.n_windows)


def make_desc(D, W, E, time_mode=TIME_RAW, eq6_lo=0.0, eq6_hi=1.0, tie_policy=TIE_NUDGE) -> PackDesc:
    return PackDesc(int(D), int(time_mode), int(W), int(E), float(eq6_lo), float(eq6_hi), int(tie_policy), 0)


def packed_layout(desc: PackDesc) -> dict:
    """Section offsets of a packed buffer (mdhp_packed_layout)."""
    arr = (ctypes.c_size_t * 14)()
    _check(lib().mdhp_packed_layout(ctypes.byref(desc), ctypes.cast(arr, ctypes.c_void_p)),
           "mdhp_packed_layout")
    keys = ["begin", "n", "T32", "perm", "t32", "dtp", "mark", "cnt", "umax", "mom", "sort",
            "total", "Epad", "Dp"]
    return dict(zip(keys, [int(v) for v in arr]))


def unpack_views(pk: "Packed") -> dict:
    """Typed views of the packed sections (for tests and tools)."""
    L = packed_layout(pk.desc)
    W, Ep, Dp = pk.W, L["Epad"], L["Dp"]
    b = pk.buf

    def sec(off, n, dt):
        nb = n * torch.tensor([], dtype=dt).element_size()
        return b[off:off + nb].view(dt)
    return {"begin": sec(L["begin"], W, torch.int64), "n": sec(L["n"], W, torch.int32),
            "T32": sec(L["T32"], W, torch.float32), "perm": sec(L["perm"], W, torch.int32),
            "t32": sec(L["t32"], Ep, torch.float32), "dtp": sec(L["dtp"], Ep, torch.float32),
            "mark": sec(L["mark"], Ep, torch.uint8), "cnt": sec(L["cnt"], W * Dp, torch.int32).view(W, Dp),
            "umax": sec(L["umax"], W * Dp, torch.float32).view(W, Dp),
            "mom": sec(L["mom"], W * Dp * 17, torch.float32).view(W, Dp, 17), "Dp": Dp}


def packed_bytes(desc: PackDesc) -> int:
    return int(lib().mdhp_packed_bytes(ctypes.byref(desc)))


def pack_windows(D, t, mark, win_off, T, time_mode=TIME_RAW, eq6_lo=0.0, eq6_hi=1.0,
                 out: Packed | None = None, tie_policy=TIE_NUDGE, stream=None) -> Packed:
    """mdhp_pack_windows on CUDA tensors t f64[E], mark i32[E], win_off i64[W+1], T f64[W]."""
    _dev(t, torch.float64, "t"); _dev(mark, torch.int32, "mark")
    _dev(win_off, torch.int64, "win_off"); _dev(T, torch.float64, "T")
    W = T.numel(); E = t.numel()
    _size(mark, E, "mark"); _size(win_off, W + 1, "win_off")
    desc = make_desc(D, W, E, time_mode, eq6_lo, eq6_hi, tie_policy)
    nb = packed_bytes(desc)
    if nb == 0:
        _check(-2, "mdhp_packed_bytes")
    if out is None or out.buf.numel() < nb or out.status.numel() < W:
        buf = torch.empty(nb, dtype=torch.uint8, device=t.device)
        status = torch.empty(max(W, 1), dtype=torch.int32, device=t.device)
    else:
        buf, status = out.buf, out.status
    rc = lib().mdhp_pack_windows(ctypes.byref(desc), _ptr(t), _ptr(mark), _ptr(win_off), _ptr(T),
                                 _ptr(buf), ctypes.c_size_t(buf.numel()), _ptr(status), _stream(stream))
    _check(rc, "mdhp_pack_windows")
    return Packed(desc, buf, status)


def loglik_grad(pk: Packed, theta, alpha, beta, grads=True, out=None, stream=None, exact=False):
    """mdhp_loglik_grad (exact=True: mdhp_loglik_exact, every window in fp64 on the GPU).
    theta f32[W,D], alpha/beta f32[W,D,D] (CUDA).  Returns dict of tensors."""
    D, W = pk.D, pk.W
    _params(W, D, theta, alpha, beta)
    dev = theta.device
    o = out or {}
    lnl = o.get("lnl") if o.get("lnl") is not None else torch.empty(W, dtype=torch.float64, device=dev)
    gt = ga = gb = None
    if grads:
        gt = o.get("g_theta") if o.get("g_theta") is not None else torch.empty(W, D, dtype=torch.float32, device=dev)
        ga = o.get("g_alpha") if o.get("g_alpha") is not None else torch.empty(W, D, D, dtype=torch.float32, device=dev)
        gb = o.get("g_beta") if o.get("g_beta") is not None else torch.empty(W, D, D, dtype=torch.float32, device=dev)
    _dev(lnl, torch.float64, "lnl"); _size(lnl, W, "lnl")
    for nm, x, n in (("g_theta", gt, W * D), ("g_alpha", ga, W * D * D), ("g_beta", gb, W * D * D)):
        if x is not None:
            _dev(x, torch.float32, nm); _size(x, n, nm)
    fn = lib().mdhp_loglik_exact if exact else lib().mdhp_loglik_grad
    rc = fn(ctypes.byref(pk.desc), _ptr(pk.buf), _ptr(theta), _ptr(alpha),
            _ptr(beta), _ptr(lnl), _ptr(gt), _ptr(ga), _ptr(gb),
            _ptr(pk.status), _stream(stream))
    _check(rc, "mdhp_loglik_exact" if exact else "mdhp_loglik_grad")
    return {"lnl": lnl, "g_theta": gt, "g_alpha": ga, "g_beta": gb}


def loglik_dense(pk: Packed, theta, alpha, beta, out=None, stream=None):
    """mdhp_loglik_dense (ablation f3): lnL by the paper's all-pairs method.  -> lnL f64[W]."""
    _params(pk.W, pk.D, theta, alpha, beta)
    lnl = out if out is not None else torch.empty(pk.W, dtype=torch.float64, device=theta.device)
    _dev(lnl, torch.float64, "out"); _size(lnl, pk.W, "out")
    rc = lib().mdhp_loglik_dense(ctypes.byref(pk.desc), _ptr(pk.buf), _ptr(theta), _ptr(alpha), _ptr(beta),
                                 _ptr(lnl), _ptr(pk.status), _stream(stream))
    _check(rc, "mdhp_loglik_dense")
    return lnl


def hawkes_features(theta, alpha, beta, T_span, A, B, C, out=None, stream=None):
    """mdhp_hawkes_features (row f4): hks[w] = tanh(A alpha_w - B (beta_w T_w) + C theta_w),
    Eq.(7) third line.  theta [W][D], alpha/beta [W][D][D], T_span [W], A/B [H][D*D],
    C [H][D], all fp32 CUDA tensors.  -> hks fp32 [W][H]."""
    for nm, x in (("theta", theta), ("alpha", alpha), ("beta", beta), ("T_span", T_span),
                  ("A", A), ("B", B), ("C", C)):
        _dev(x, torch.float32, nm)
    W, D = theta.shape[0], theta.shape[-1]
    H = A.shape[0]
    _params(W, D, theta, alpha, beta)
    _size(T_span, W, "T_span"); _size(A, H * D * D, "A"); _size(B, H * D * D, "B"); _size(C, H * D, "C")
    hks = out if out is not None else torch.empty(W, H, dtype=torch.float32, device=theta.device)
    _dev(hks, torch.float32, "out"); _size(hks, W * H, "out")
    rc = lib().mdhp_hawkes_features(D, W, H, _ptr(theta), _ptr(alpha), _ptr(beta), _ptr(T_span),
                                    _ptr(A), _ptr(B), _ptr(C), _ptr(hks), _stream(stream))
    _check(rc, "mdhp_hawkes_features")
    return hks


def fit(pk: Packed, theta, alpha, beta, cfg: FitConfig, opt_state=None, trace=False, stream=None):
    """mdhp_fit.  theta/alpha/beta are updated IN PLACE (init in, fitted out)."""
    D, W = pk.D, pk.W
    _params(W, D, theta, alpha, beta)
    if opt_state is not None:
        _dev(opt_state, torch.float32, "opt_state")
        _size(opt_state, 2 * W * (D + 2 * D * D), "opt_state")
    dev = theta.device
    lnl = torch.empty(W, dtype=torch.float64, device=dev)
    iters = torch.empty(W, dtype=torch.int32, device=dev)
    tr = torch.empty(W, max(cfg.max_iters, 1), dtype=torch.float32, device=dev) if trace else None
    c = cfg.c()
    rc = lib().mdhp_fit(ctypes.byref(pk.desc), _ptr(pk.buf), ctypes.byref(c), _ptr(theta),
                        _ptr(alpha), _ptr(beta), _ptr(opt_state), _ptr(lnl), _ptr(iters),
                        _ptr(pk.status), _ptr(tr), _stream(stream))
    _check(rc, "mdhp_fit")
    return {"theta": theta, "alpha": alpha, "beta": beta, "lnl": lnl, "iters": iters,
            "status": pk.status, "trace": tr}


def fit_host(D, t, mark, win_off, T, theta, alpha, beta, cfg: FitConfig, time_mode=TIME_RAW,
             eq6_lo=0.0, eq6_hi=1.0, tie_policy=TIE_NUDGE, stream=None):
    """mdhp_fit_host on CPU tensors (pinned recommended).  theta/alpha/beta updated in place;
    returns dict with lnl, iters, status (CPU tensors)."""
    for nm, x, dt in (("t", t, torch.float64), ("mark", mark, torch.int32), ("win_off", win_off, torch.int64),
                      ("T", T, torch.float64), ("theta", theta, torch.float32),
                      ("alpha", alpha, torch.float32), ("beta", beta, torch.float32)):
        if x.is_cuda or x.dtype != dt or not x.is_contiguous():
            raise TypeError(f"{nm} must be a contiguous CPU {dt} tensor")
    W = T.numel()
    _size(mark, t.numel(), "mark"); _size(win_off, W + 1, "win_off")
    _size(theta, W * D, "theta"); _size(alpha, W * D * D, "alpha"); _size(beta, W * D * D, "beta")
    desc = make_desc(D, W, t.numel(), time_mode, eq6_lo, eq6_hi, tie_policy)
    lnl = torch.empty(W, dtype=torch.float64)
    iters = torch.empty(W, dtype=torch.int32)
    status = torch.empty(W, dtype=torch.int32)
    c = cfg.c()
    rc = lib().mdhp_fit_host(ctypes.byref(desc), _ptr(t), _ptr(mark), _ptr(win_off), _ptr(T),
                             ctypes.byref(c), _ptr(theta), _ptr(alpha), _ptr(beta), _ptr(lnl),
                             _ptr(iters), _ptr(status), _stream(stream))
    _check(rc, "mdhp_fit_host")
    return {"lnl": lnl, "iters": iters, "status": status}


# ------------------------------------------------------------------ long single sequences (a7)
@dataclass
class PackedSeq:
    desc: SeqDesc
    buf: torch.Tensor
    status: torch.Tensor   # int32 [1] device

    @property
    def D(self):
        return int(self.desc.D)


def seq_chunk_hint(D, n_events) -> int:
    """mdhp_seq_chunk_hint: a chunk size whose chunks fill whole waves of the current device."""
    ce = int(lib().mdhp_seq_chunk_hint(int(D), int(n_events)))
    if ce < 0:
        _check(ce, "mdhp_seq_chunk_hint")
    return ce


def seq_pack(D, t, mark, T, chunk_events=256, out: PackedSeq | None = None, t0=0.0, has_history=False,
             stream=None) -> PackedSeq:
    """mdhp_seq_pack on CUDA tensors t f64[N], mark i32[N] (one sequence on [0, T], or one slice of
    it starting after t0 when has_history).  chunk_events=0: mdhp_seq_chunk_hint."""
    _dev(t, torch.float64, "t"); _dev(mark, torch.int32, "mark")
    if not chunk_events:
        chunk_events = seq_chunk_hint(D, t.numel())
    desc = SeqDesc(int(D), int(chunk_events), int(t.numel()), float(T), float(t0), int(bool(has_history)), 0)
    nb = int(lib().mdhp_seq_packed_bytes(ctypes.byref(desc)))
    if nb == 0:
        _check(-2, "mdhp_seq_packed_bytes")
    if out is None or out.buf.numel() < nb:
        buf = torch.empty(nb, dtype=torch.uint8, device=t.device)
        status = torch.zeros(1, dtype=torch.int32, device=t.device)
    else:
        buf, status = out.buf, out.status
    rc = lib().mdhp_seq_pack(ctypes.byref(desc), _ptr(t), _ptr(mark), _ptr(buf), ctypes.c_size_t(buf.numel()),
                             _ptr(status), _stream(stream))
    _check(rc, "mdhp_seq_pack")
    return PackedSeq(desc, buf, status)


def seq_loglik_grad(ps: PackedSeq, theta, alpha, beta, grads=True, stream=None):
    D = ps.D
    _params(1, D, theta, alpha, beta)
    dev = theta.device
    lnl = torch.empty(1, dtype=torch.float64, device=dev)
    gt = torch.empty(D, dtype=torch.float32, device=dev) if grads else None
    ga = torch.empty(D, D, dtype=torch.float32, device=dev) if grads else None
    gb = torch.empty(D, D, dtype=torch.float32, device=dev) if grads else None
    rc = lib().mdhp_seq_loglik_grad(ctypes.byref(ps.desc), _ptr(ps.buf), _ptr(theta), _ptr(alpha), _ptr(beta),
                                    _ptr(lnl), _ptr(gt), _ptr(ga), _ptr(gb), _stream(stream))
    _check(rc, "mdhp_seq_loglik_grad")
    return {"lnl": lnl, "g_theta": gt, "g_alpha": ga, "g_beta": gb}


def seq_fit(ps: PackedSeq, theta, alpha, beta, cfg: FitConfig, opt_state=None, trace=False, stream=None):
    """mdhp_seq_fit; theta [D], alpha/beta [D,D] fp32 CUDA tensors updated in place."""
    D = ps.D
    _params(1, D, theta, alpha, beta)
    if opt_state is not None:
        _dev(opt_state, torch.float32, "opt_state")
        _size(opt_state, 2 * (D + 2 * D * D), "opt_state")
    dev = theta.device
    lnl = torch.empty(1, dtype=torch.float64, device=dev)
    iters = torch.empty(1, dtype=torch.int32, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    tr = torch.empty(max(cfg.max_iters, 1), dtype=torch.float32, device=dev) if trace else None
    c = cfg.c()
    rc = lib().mdhp_seq_fit(ctypes.byref(ps.desc), _ptr(ps.buf), ctypes.byref(c), _ptr(theta), _ptr(alpha),
                            _ptr(beta), _ptr(opt_state), _ptr(lnl), _ptr(iters), _ptr(status), _ptr(tr),
                            _stream(stream))
    _check(rc, "mdhp_seq_fit")
    return {"lnl": lnl, "iters": iters, "status": status, "trace": tr}
