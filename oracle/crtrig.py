"""Correctly-rounded sin/cos for the oracle (test infrastructure only).

Wraps ``oracle/_crtrig.so``, a gcc build (-ffp-contract=off) of the engine's
``exa_math.h``; built on demand with the system C compiler.
"""

from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
SO = HERE / "_crtrig.so"
SRC = HERE / "crtrig.c"
INC = HERE.parent / "paper_2510_12897_b200" / "csrc"

_lib = None


def build(force: bool = False) -> Path:
    deps = [SRC, INC / "exa_math.h", INC / "exa_sincos_table.h"]
    if force or not SO.exists() or any(d.stat().st_mtime > SO.stat().st_mtime for d in deps):
        subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared", f"-I{INC}", str(SRC),
                        "-o", str(SO), "-lm"], check=True)
    return SO


def _load():
    global _lib
    if _lib is None:
        build()
        lib = C.CDLL(str(SO))
        lib.cr_sincos_vec.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64]
        lib.cr_sincos_vec.restype = None
        lib.cr_sincos_fast_vec.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64]
        lib.cr_sincos_fast_vec.restype = None
        lib.cr_sincos_slow_vec.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64]
        lib.cr_sincos_slow_vec.restype = None
        _lib = lib
    return _lib


def sincos(x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    s = np.empty_like(x)
    c = np.empty_like(x)
    _load().cr_sincos_vec(x.ctypes.data, s.ctypes.data, c.ctypes.data, x.size)
    return s, c


def sincos_fast(x):
    """Ziv fast path alone (|x| <= pi/4): (s, c, ok)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    s, c = np.empty_like(x), np.empty_like(x)
    ok = np.empty(x.shape, dtype=np.int32)
    _load().cr_sincos_fast_vec(x.ctypes.data, s.ctypes.data, c.ctypes.data, ok.ctypes.data, x.size)
    return s, c, ok.astype(bool)


def sincos_slow(x):
    """Double-double slow path alone (|x| <= pi/4)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    s, c = np.empty_like(x), np.empty_like(x)
    _load().cr_sincos_slow_vec(x.ctypes.data, s.ctypes.data, c.ctypes.data, x.size)
    return s, c


def sin(x):
    return sincos(x)[0]


def cos(x):
    return sincos(x)[1]


TRIG = (sin, cos)
