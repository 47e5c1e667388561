"""ctypes binding of libexa.so (the C ABI in include/exa.h).

Loading is strict: if the in-tree library is missing or fails to load, every
entry point raises -- there is no CPU fallback anywhere in this package.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(os.environ.get("EXA_LIB", Path(__file__).resolve().parent / "libexa.so"))

MAXF = MAXI = MAXK = 16
NMODES = 6
NKERN = 12
MODE_SET, MODE_CONS, MODE_JAC, MODE_HESS, MODE_OBJV, MODE_GRAD = range(6)
ABI_VERSION = 6

i64, i32, dbl, vp = C.c_int64, C.c_int32, C.c_double, C.c_void_p


class TermDesc(C.Structure):
    _fields_ = [
        ("f_off", i64 * MAXF), ("ix_off", i64 * MAXI), ("rows_off", i64), ("row_ptr_off", i64),
        ("row_ent_off", i64), ("voff", i32 * MAXK), ("nrec", i32), ("pattern", i32), ("kind", i32),
        ("order", i32), ("row_offset", i32), ("cons_direct", i32), ("k", i32), ("pad", i32),
        ("jac0", i64), ("hess0", i64), ("scr0", i64),
    ]


class SegDesc(C.Structure):
    _fields_ = [("term", i32), ("kind", i32), ("cta0", i32), ("nrec", i32)]


class PlanDesc(C.Structure):
    _fields_ = [
        ("abi_version", i32), ("device", i32),
        ("nvar", i64), ("ncon", i64), ("n_jac", i64), ("n_hess", i64),
        ("f64", C.POINTER(dbl)), ("n_f64", i64),
        ("i32", C.POINTER(i32)), ("n_i32", i64),
        ("terms", C.POINTER(TermDesc)), ("n_terms", i32), ("threads", i32 * 2),
        ("segs", C.POINTER(SegDesc) * NKERN), ("n_segs", i32 * NKERN), ("n_ctas", i32 * NKERN),
        ("err_base", (i32 * 2) * NMODES),
        ("n_vscr", i64), ("n_gscr", i64),
        ("leaves", C.POINTER(i64)), ("n_leaves", i32),
        ("obj_prog", C.POINTER(i64)), ("n_prog", i32),
        ("grad_ptr", C.POINTER(i64)), ("grad_ent", C.POINTER(i64)), ("n_grad_ent", i64),
        ("cubin", vp), ("cubin_size", i64),
        ("has_domain_checks", i32),
        ("persist", i32 * NKERN), ("pdl", i32), ("batchable", i32), ("host_fill", C.POINTER(C.c_int64)), ("n_fill_jac", i32), ("n_fill_hess", i32),
        ("host_wzero", C.POINTER(C.c_int64)), ("n_wzero", i32), ("pad_wz", i32),
        ("host_wzero_rows", C.POINTER(C.c_int32)), ("n_wzero_rows", i64),
    ]


# symbol -> (restype, argtypes); every symbol declared in include/exa.h
SIGNATURES = {
    "exa_jit_compile": (C.c_int, [C.c_char_p, C.c_char_p, C.POINTER(C.c_char_p), C.c_int,
                                  C.POINTER(vp), C.POINTER(C.c_size_t), C.POINTER(vp)]),
    "exa_free": (None, [vp]),
    "exa_nvrtc_version": (C.c_int, [C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "exa_plan_create": (C.c_int, [C.POINTER(PlanDesc), C.POINTER(vp)]),
    "exa_plan_destroy": (None, [vp]),
    "exa_plan_info": (C.c_int, [vp, C.POINTER(i64), C.POINTER(i32)]),
    "exa_workspace_create": (C.c_int, [vp, C.POINTER(vp)]),
    "exa_workspace_destroy": (None, [vp]),
    "exa_eval_obj": (C.c_int, [vp, vp, vp, vp, vp]),
    "exa_eval_grad": (C.c_int, [vp, vp, vp, vp, vp]),
    "exa_eval_cons": (C.c_int, [vp, vp, vp, vp, vp]),
    "exa_eval_jac": (C.c_int, [vp, vp, vp, vp, vp]),
    "exa_eval_hess": (C.c_int, [vp, vp, vp, vp, dbl, vp, vp]),
    "exa_eval_set": (C.c_int, [vp, vp, vp, vp, dbl, vp, vp, vp, vp]),
    "exa_eval_set_host": (C.c_int, [vp, vp, vp, vp, dbl, vp, vp, vp, vp]),
    "exa_eval_cons_host": (C.c_int, [vp, vp, vp, vp, vp]),
    "exa_eval_jac_host": (C.c_int, [vp, vp, vp, vp, vp]),
    "exa_eval_hess_host": (C.c_int, [vp, vp, vp, vp, dbl, vp, vp]),
    "exa_host_register": (C.c_int, [vp, C.c_size_t]),
    "exa_host_unregister": (C.c_int, [vp]),
    "exa_eval_set_batch": (C.c_int, [vp, vp, i64, vp, vp, dbl, vp, vp, vp, vp]),
    "exa_segment_sum": (C.c_int, [i64, vp, vp, vp, vp, vp]),
    "exa_pattern_create": (C.c_int, [vp, i64, i64, vp, vp, C.POINTER(vp)]),
    "exa_pattern_create_known": (C.c_int, [vp, i64, i64, vp, vp, vp, vp, C.POINTER(vp)]),
    "exa_pattern_create_direct": (C.c_int, [vp, i64, i64, vp, vp, vp, vp, vp, C.POINTER(vp)]),
    "exa_plan_attach_compressed": (C.c_int, [vp, vp, i64, vp, i64]),
    "exa_pattern_destroy": (None, [vp]),
    "exa_eval_set_compressed": (C.c_int, [vp, vp, vp, vp, vp, vp, dbl, vp, vp, vp, vp]),
    "exa_eval_set_compressed_host": (C.c_int, [vp, vp, vp, vp, vp, vp, dbl, vp, vp, vp, vp]),
    "exa_kkt_values": (C.c_int, [i64, vp, vp, vp, vp, dbl, dbl, vp, vp]),
    "exa_domain_error": (C.c_int, [vp, vp, vp, C.POINTER(i64), C.POINTER(i32), C.POINTER(i64)]),
    "exa_last_error": (C.c_char_p, []),
    "exa_device_sincos": (C.c_int, [vp, vp, vp, i64, vp]),
    "exa_debug_trace": (C.c_int, [vp]),
}

_lib = None


class ExaError(RuntimeError):
    pass


def load():
    """Load libexa.so (build it first if absent in a source checkout)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        from .build import build

        build()
    if not LIB_PATH.exists():  # pragma: no cover
        raise ExaError(f"libexa.so not found at {LIB_PATH}; run __graft_entry__.build()")
    lib = C.CDLL(str(LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int, what: str = "") -> int:
    if rc < 0:
        msg = load().exa_last_error()
        raise ExaError(f"{what}: {msg.decode() if msg else 'error'}")
    return rc


def nvrtc_version() -> str:
    a, b = C.c_int(), C.c_int()
    check(load().exa_nvrtc_version(C.byref(a), C.byref(b)), "nvrtc_version")
    return f"{a.value}.{b.value}"


def jit_compile(src: str, opts, name: str = "exa_gen.cu") -> bytes:
    lib = load()
    arr = (C.c_char_p * len(opts))(*[o.encode() for o in opts])
    out, size, log = vp(), C.c_size_t(), vp()
    rc = lib.exa_jit_compile(src.encode(), name.encode(), arr, len(opts), C.byref(out), C.byref(size), C.byref(log))
    try:
        check(rc, "NVRTC")
        return C.string_at(out, size.value)
    finally:
        if out.value:
            lib.exa_free(out)
        if log.value:
            lib.exa_free(log)
