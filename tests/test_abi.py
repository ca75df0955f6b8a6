"""CPU-side checks of the boundary: the library builds for sm_100a, loads, exports every symbol
declared in include/*.h, and rejects bad arguments before touching the GPU."""
import ctypes
import os
import re

import pytest

import paper_2411_10258_b200 as M
from paper_2411_10258_b200 import mdhp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    for fn in os.listdir(os.path.join(ROOT, "include")):
        if not fn.endswith(".h"):
            continue
        src = open(os.path.join(ROOT, "include", fn)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"^[A-Za-z_][\w\s\*]*?\b(mdhp_\w+|synth_\w+)\s*\(", src, flags=re.M):
            names.add((fn, m.group(1)))
    return names


def test_library_exports_every_declared_symbol():
    syms = declared_symbols()
    assert any(n == "mdhp_fit" for _, n in syms)
    libs = {"mdhp.h": M.lib()}
    try:
        from synth import gpu as sg
        libs["synth.h"] = sg.lib()
    except Exception:  # pragma: no cover - synth lib optional until built
        pass
    for fn, name in syms:
        L = libs.get(fn)
        assert L is not None, f"no library for header {fn}"
        assert hasattr(L, name), f"{name} declared in include/{fn} but not exported"


def test_sm100a_cubin():
    """The .so carries sm_100a SASS (cuobjdump lists the architecture)."""
    import subprocess
    r = subprocess.run(["cuobjdump", "--list-elf", M.build.LIB if hasattr(M, "build") else
                        mdhp._build.LIB], capture_output=True, text=True)
    assert "sm_100a" in r.stdout


def test_bad_arguments_rejected_without_gpu():
    L = M.lib()
    d = mdhp.make_desc(0, 1, 1)
    assert L.mdhp_pack_windows(ctypes.byref(d), None, None, None, None, None, 0, None, None) == -2
    d = mdhp.make_desc(33, 1, 1)
    assert mdhp.packed_bytes(d) == 0
    d = mdhp.make_desc(4, 1, 1)
    assert L.mdhp_pack_windows(ctypes.byref(d), None, None, None, None, None, 0, None, None) == -1
    assert b"NULL" in L.mdhp_last_error()
    d = mdhp.make_desc(4, 1, 1, time_mode=mdhp.TIME_EQ6, eq6_lo=1.0, eq6_hi=0.0)
    assert L.mdhp_pack_windows(ctypes.byref(d), None, None, None, None, None, 0, None, None) == -1
    # packed buffer too small
    d = mdhp.make_desc(4, 2, 10)
    fake = ctypes.c_void_p(16)
    assert L.mdhp_pack_windows(ctypes.byref(d), fake, fake, fake, fake, fake, 8, fake, None) == -3
    c = M.FitConfig(lr=-1.0).c()
    assert L.mdhp_fit(ctypes.byref(d), fake, ctypes.byref(c), fake, fake, fake, None, fake, fake,
                      fake, None, None) == -1
    # the chunk-size hint validates its dimensions before touching the device
    assert L.mdhp_seq_chunk_hint(0, 100) == -2 and L.mdhp_seq_chunk_hint(33, 100) == -2
    assert L.mdhp_seq_chunk_hint(4, -1) == -2


def test_layout_is_pure_function():
    a = mdhp.packed_layout(mdhp.make_desc(16, 1000, 10**6))
    b = mdhp.packed_layout(mdhp.make_desc(16, 1000, 10**6))
    assert a == b
    assert a["Dp"] == 16 and a["total"] == mdhp.packed_bytes(mdhp.make_desc(16, 1000, 10**6))
    offs = [a[k] for k in ("begin", "n", "T32", "perm", "t32", "dtp", "mark", "cnt", "umax", "mom", "sort", "total")]
    assert offs == sorted(offs) and all(o % 256 == 0 for o in offs)
    assert mdhp.packed_layout(mdhp.make_desc(5, 3, 7))["Dp"] == 8


def test_no_cpu_fallback():
    import torch
    with pytest.raises(TypeError):
        M.pack_windows(2, torch.zeros(3, dtype=torch.float64), torch.zeros(3, dtype=torch.int32),
                       torch.tensor([0, 3]), torch.ones(1, dtype=torch.float64))


def test_hawkes_features_args_rejected_without_gpu():
    L = M.lib()
    fake = ctypes.c_void_p(16)
    args = [fake] * 7 + [ctypes.c_void_p(256), None]
    assert L.mdhp_hawkes_features(0, 4, 16, *args) == -2          # D out of range
    assert L.mdhp_hawkes_features(33, 4, 16, *args) == -2
    assert L.mdhp_hawkes_features(4, 4, 24, *args) == -2          # H not a multiple of 16
    assert L.mdhp_hawkes_features(4, 4, 272, *args) == -2         # H > 256 not a multiple of 256
    assert L.mdhp_hawkes_features(4, 4, 16, None, *args[1:]) == -1
    assert b"NULL" in L.mdhp_last_error()
    assert L.mdhp_hawkes_features(4, 4, 16, *args[:7], ctypes.c_void_p(260), None) == -1   # unaligned out
