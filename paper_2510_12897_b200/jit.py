"""Assemble a model's generated kernels into one CUDA module and compile it.

The module holds one device function pair per tape pattern (from
:mod:`.codegen`) and six ``extern "C"`` entry kernels, one per callback mode.
Each CTA serves exactly one *segment* (one term's records, or one
augment-target block's rows), so the pattern ``switch`` is uniform per CTA
and the whole callback set is a single launch.

Compilation goes through NVRTC inside ``libexa.so`` (``exa_jit_compile``)
with ``-arch=sm_100a --fmad=false``.  Cubins are cached in-process and on
disk under ``_jit/`` keyed by the SHA-256 of (source, options, NVRTC
version), so a model family is compiled once per machine.
"""

from __future__ import annotations

import hashlib
import os
import threading
from pathlib import Path

from . import _lib

CSRC = Path(__file__).resolve().parent / "csrc"
CACHE_DIR = Path(os.environ.get("EXA_JIT_CACHE", Path(__file__).resolve().parent / "_jit"))
NVRTC_OPTIONS = ("-arch=sm_100a", "--fmad=false", "-default-device", "-std=c++17", "-lineinfo",
                 "--extra-device-vectorization")
THREADS = int(os.environ.get("EXA_THREADS", "64"))  # CTA size (fused / light kernels)
THREADS_HEAVY = int(os.environ.get("EXA_THREADS_HEAVY", "128"))  # heavy kernels
# tuning knobs (experiments only; defaults are the product configuration)
MIN_BLOCKS = int(os.environ.get("EXA_MINB", "0"))
SINCOS_IMPL = os.environ.get("EXA_SINCOS_IMPL", "cr")
PDL = os.environ.get("EXA_PDL", "0") == "1"  # must match the library's launch attribute  # "cuda" = libdevice sincos, NOT parity-exact

_lock = threading.Lock()
_mem_cache: dict = {}


def _inline_header(name: str, seen: set) -> str:
    if name in seen:
        return ""
    seen.add(name)
    out = []
    for line in (CSRC / name).read_text().splitlines():
        s = line.strip()
        if s.startswith("#pragma once"):
            continue
        if s.startswith("#include \""):
            out.append(_inline_header(s.split('"')[1], seen))
            continue
        if s.startswith("#include <"):
            continue
        out.append(line)
    return "\n".join(out)


_PRELUDE = r"""
// ---- runtime helpers for generated kernels -------------------------------
__device__ __forceinline__ double exa_powi(double a, int n) { return pow(a, (double)n); }
__device__ __forceinline__ void exa_report(const ExaArgs& A, int rank, int instr, long long rec1) {
  atomicMin(A.err, EXA_ERR_KEY(rank, instr, rec1));
}
#define EXA_DOMAIN(instr) exa_report(A, rank, (instr), (long long)r + 1)
#define EXA_REC_ALL 0
#define EXA_REC_FIRST 1
#define EXA_DOMAIN_AT(instr, rec1) exa_report(A, rank, (instr), (rec1))
// programmatic dependent launch: release the next kernel early; wait for the
// previous one before the first access to caller memory (x, y, outputs)
#if EXA_PDL
#define EXA_GRID_WAIT() asm volatile("griddepcontrol.wait;" ::: "memory")
#define EXA_GRID_RELEASE() asm volatile("griddepcontrol.launch_dependents;" ::: "memory")
#else
#define EXA_GRID_WAIT() do {} while (0)
#define EXA_GRID_RELEASE() do {} while (0)
#endif
"""

_COMMON = r"""
// ---- dispatch ------------------------------------------------------------
template <int MODE>
__device__ __forceinline__ void exa_dispatch_term(const ExaTerm& T, int r, const ExaArgs& A, int rank) {
  switch (T.pattern) {
@TERM_CASES@
    default: break;
  }
}

__device__ __forceinline__ double exa_dispatch_val(const ExaTerm& T, int r, const ExaArgs& A, int rank) {
  switch (T.pattern) {
@VAL_CASES@
    default: return 0.0;
  }
}

__device__ __forceinline__ int exa_rank(const ExaTerm& T, const ExaArgs& A) {
  return T.order + (T.kind == EXA_OBJ ? A.obj_base : A.con_base);
}

// Serial row sum (rows with more than 32 contributions): zero-fill, base
// slice-add, then each augment in registration order, records in order
// (reference autodiff.py:573-580).  val(term, record) evaluates one record.
template <class VAL>
__device__ __forceinline__ void exa_row(const ExaTerm& T, int r, const ExaArgs& A, VAL val) {
  EXA_GRID_WAIT();
  double acc = 0.0 + exa_dispatch_val(T, r, A, exa_rank(T, A));
  const int e1 = __ldg(T.row_ptr + r + 1);
  for (int e = __ldg(T.row_ptr + r); e < e1; ++e) {
    const int2 ent = __ldg(reinterpret_cast<const int2*>(T.row_ent) + e);
    acc = acc + val(ent.x, ent.y);
  }
  A.c[T.row_offset + r] = acc;
}

// Warp-parallel row sums with the same rounding: every lane evaluates one
// contribution (row base at position 0, then the row's augment records in
// reference order); the row total is then folded LEFT TO RIGHT through the
// lanes with shuffles, i.e. ((0 + base) + a1) + a2 + ... exactly as numpy's
// slice-add followed by np.add.at.  Rows never straddle a warp.
template <class VAL>
__device__ __forceinline__ void exa_rowfold(const ExaTerm& T, int slot, const ExaArgs& A, VAL val) {
  const int lane = threadIdx.x & 31;
  const int2 e = __ldg(reinterpret_cast<const int2*>(T.row_ent) + slot);
  EXA_GRID_WAIT();
  const bool pad = e.x < 0;
  const int p = pad ? 0 : ((e.x >> 16) & 0x3fff);
  const double v = pad ? 0.0 : val(e.x & (0xffff | (1 << 30)), e.y);
  double acc = (p == 0) ? 0.0 + v : v;
  const unsigned pmax = __reduce_max_sync(0xffffffffu, (unsigned)p);
  for (unsigned s = 1; s <= pmax; ++s) {
    const double up = __shfl_up_sync(0xffffffffu, acc, 1);
    if ((unsigned)p == s) acc = up + v;
  }
  const int pn = __shfl_down_sync(0xffffffffu, pad ? -1 : p, 1);
  const int r0 = __shfl_sync(0xffffffffu, e.y, lane - p);
  if (!pad && (lane == 31 || pn <= 0)) A.c[T.row_offset + r0] = acc;
}
"""

_KERNELS_GENERIC = r"""
// ---- metadata: constant memory (small models) or global memory -----------
#if EXA_META_CONST
__constant__ ExaTerm exa_terms_c[EXA_CMAX_TERMS];
__constant__ ExaSeg exa_segs_c[EXA_CMAX_SEGS];
#define EXA_TERM(i) exa_terms_c[(i)]
#else
#define EXA_TERM(i) terms[(i)]
#endif

template <int MODE>
__device__ __forceinline__ void exa_kernel_body(const ExaTerm* __restrict__ terms, const ExaSeg* __restrict__ segs,
                                                const int* __restrict__ cta_seg, const ExaArgs& A) {
#if EXA_META_CONST
  int lo = A.seg_off, hi = A.seg_off + A.n_segs - 1;
  const int b = (int)blockIdx.x;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (exa_segs_c[mid].cta0 <= b) lo = mid; else hi = mid - 1;
  }
  const ExaSeg sg = exa_segs_c[lo];
#else
  const ExaSeg sg = segs[__ldg(cta_seg + blockIdx.x)];
#endif
  const int kind = sg.kind & 0xff, rpt = sg.kind >> 8;
  const ExaTerm& T = EXA_TERM(sg.term);
  auto val = [&](int t, int rec) -> double {
    const ExaTerm& U = EXA_TERM(t);
    return exa_dispatch_val(U, rec, A, exa_rank(U, A));
  };
  const int r0 = (int)(blockIdx.x - sg.cta0) * (int)blockDim.x * rpt + (int)threadIdx.x;
  if (kind == EXA_SEG_TERM) {
    for (int q = 0; q < rpt; ++q) {
      const int r = r0 + q * (int)blockDim.x;
      if (r < sg.nrec) exa_dispatch_term<MODE>(T, r, A, exa_rank(T, A));
    }
    return;
  }
  if (r0 >= sg.nrec) return;
  if (kind == EXA_SEG_FOLD) exa_rowfold(T, r0, A, val);
  else exa_row(T, r0, A, val);
}
"""

_ENTRIES = r"""
#define EXA_ENTRY(NAME, MODE, BOUNDS)                                                          \
  extern "C" __global__ void __launch_bounds__(BOUNDS) NAME(                                  \
      const ExaTerm* __restrict__ terms, const ExaSeg* __restrict__ segs,                     \
      const int* __restrict__ cta_seg, ExaArgs A) {                                           \
    EXA_GRID_RELEASE();                                                                        \
    exa_kernel_body<MODE>(terms, segs, cta_seg, A);                                            \
  }

EXA_ENTRY(exa_k_set_h, EXA_M_CONS | EXA_M_JAC | EXA_M_HESS, @BOUNDS_H@)
EXA_ENTRY(exa_k_set_l, EXA_M_CONS | EXA_M_JAC | EXA_M_HESS, @BOUNDS_L@)
EXA_ENTRY(exa_k_cons_h, EXA_M_CONS, @BOUNDS_H@)
EXA_ENTRY(exa_k_cons_l, EXA_M_CONS, @BOUNDS_L@)
EXA_ENTRY(exa_k_jac_h, EXA_M_JAC, @BOUNDS_H@)
EXA_ENTRY(exa_k_jac_l, EXA_M_JAC, @BOUNDS_L@)
EXA_ENTRY(exa_k_hess_h, EXA_M_HESS, @BOUNDS_H@)
EXA_ENTRY(exa_k_hess_l, EXA_M_HESS, @BOUNDS_L@)
EXA_ENTRY(exa_k_objv_h, EXA_M_OBJV, @BOUNDS_H@)
EXA_ENTRY(exa_k_objv_l, EXA_M_OBJV, @BOUNDS_L@)
EXA_ENTRY(exa_k_grad_h, EXA_M_GRAD, @BOUNDS_H@)
EXA_ENTRY(exa_k_grad_l, EXA_M_GRAD, @BOUNDS_L@)
"""

_MODE_BITS = ("EXA_M_CONS | EXA_M_JAC | EXA_M_HESS", "EXA_M_CONS", "EXA_M_JAC", "EXA_M_HESS",
              "EXA_M_OBJV", "EXA_M_GRAD")


def _specialised_kernels(layout) -> str:
    """Kernel bodies with the model's metadata as compile-time constants.

    Every term becomes an ``exa_init_T<t>`` that fills a local ExaTerm from
    literals and the blob base pointers; after inlining, addresses are
    ``blob + constant`` and the CTA -> segment dispatch is a chain of uniform
    comparisons with literals -- no metadata loads on the critical path."""
    out = []
    for t, d in enumerate(layout.term_descs()):
        lines = [f"__device__ __forceinline__ void exa_init_T{t}(ExaTerm& T, const ExaArgs& A) {{"]
        for i, off in enumerate(d["f_off"]):
            lines.append(f"  T.f[{i}] = A.f64 + {off}LL;")
        for i, off in enumerate(d["ix_off"]):
            lines.append(f"  T.ix[{i}] = A.i32 + {off}LL;")
        lines.append(f"  T.rows = {'A.i32 + %dLL' % d['rows_off'] if d['rows_off'] >= 0 else '0'};")
        lines.append(f"  T.row_ptr = {'A.i32 + %dLL' % d['row_ptr_off'] if d['row_ptr_off'] >= 0 else '0'};")
        lines.append("  T.row_ent = " + (f"reinterpret_cast<const int2*>(A.i32 + {d['row_ent_off']}LL);"
                                          if d["row_ent_off"] >= 0 else "0;"))
        for s, vo in enumerate(d["voff"]):
            lines.append(f"  T.voff[{s}] = {vo};")
        for k in ("nrec", "pattern", "kind", "order", "row_offset", "cons_direct", "k"):
            lines.append(f"  T.{k} = {d[k]};")
        for k in ("jac0", "hess0", "scr0"):
            lines.append(f"  T.{k} = {d[k]}LL;")
        lines.append("}")
        out.append("\n".join(lines))
    # per augment-target block: value of any contributing (term, record)
    for t, members in layout.row_members().items():
        lines_c = []
        for u in members:
            pc = layout.patterns[layout.term_pid[u]]
            lines_c.append(f"      case {u}: {{ ExaTerm U; exa_init_T{u}(U, A); return exa_val_{layout.term_pid[u]}(U, rec, A, exa_rank(U, A)); }}")
            if pc.valx_ok:  # pre-resolved slot: rec is the global variable id
                lines_c.append(f"      case {u | (1 << 30)}: return exa_valx_{layout.term_pid[u]}(__ldg(A.x + rec));")
        cases = "\n".join(lines_c)
        out.append(f"""__device__ __forceinline__ double exa_rowval_T{t}(int term, int rec, const ExaArgs& A) {{
  switch (term) {{
{cases}
      default: return 0.0;
  }}
}}""")
    for gid, (pid, grp, members) in enumerate(getattr(layout, "groups", [])):
        out.append(layout.patterns[pid].group_source(gid, members))
    for m, name in enumerate(KERNEL_NAMES):
        m_ = m
        for half, suffix in ((0, "_h"), (1, "_l")):
            kid = 2 * m + half
            threads = layout.threads[half]
            body = [f"extern \"C\" __global__ void __launch_bounds__(@BOUNDS_{'H' if half == 0 else 'L'}@) {name}{suffix}(",
                    "    const ExaTerm* __restrict__ terms, const ExaSeg* __restrict__ segs,",
                    "    const int* __restrict__ cta_seg, ExaArgs A) {",
                    "  EXA_GRID_RELEASE();",
                    "  const int b = (int)blockIdx.x;"]
            for (t, kind, cta0, nrec, rpt) in layout.mode_segments(kid):
                n_cta = (nrec + threads * rpt - 1) // (threads * rpt)
                body.append(f"  if (b < {cta0 + n_cta}) {{")
                if kind == 3:  # term group: t is the group id
                    pid, grp, _ = layout.groups[t]
                    for gm, u in enumerate(grp):
                        body.append(f"    ExaTerm T{gm}; exa_init_T{u}(T{gm}, A);")
                    body.append(f"    const int r = (b - {cta0}) * {threads} + (int)threadIdx.x;")
                    body.append(f"    if (r >= {nrec}) return;")
                    tl = ", ".join(f"T{gm}" for gm in range(len(grp)))
                    rl = ", ".join(f"exa_rank(T{gm}, A)" for gm in range(len(grp)))
                    body.append(f"    exa_grp_{t}<{_MODE_BITS[m_]}>({tl}, r, A, {rl});")
                    body.append("    return;")
                    body.append("  }")
                    continue
                body.append(f"    ExaTerm T; exa_init_T{t}(T, A);")
                if kind == 0:
                    body.append(f"    const int r0 = (b - {cta0}) * {threads * rpt} + (int)threadIdx.x;")
                    body.append("#pragma unroll")
                    body.append(f"    for (int q = 0; q < {rpt}; ++q) {{")
                    body.append(f"      const int r = r0 + q * {threads};")
                    body.append(f"      if (r < {nrec}) exa_term_{layout.term_pid[t]}<{_MODE_BITS[m]}>(T, r, A, exa_rank(T, A));")
                    body.append("    }")
                else:
                    body.append(f"    const int r = (b - {cta0}) * {threads} + (int)threadIdx.x;")
                    body.append(f"    if (r >= {nrec}) return;")
                    fn = "exa_rowfold" if kind == 2 else "exa_row"
                    body.append(f"    {fn}(T, r, A, [&](int u, int rec) {{ return exa_rowval_T{t}(u, rec, A); }});")
                body.append("    return;")
                body.append("  }")
            body.append("}")
            out.append("\n".join(body))
    return "\n\n".join(out)


KERNEL_NAMES = ("exa_k_set", "exa_k_cons", "exa_k_jac", "exa_k_hess", "exa_k_objv", "exa_k_grad")


def module_source(patterns, meta_const: bool = True, layout=None) -> str:
    """CUDA source of a model's module.

    ``layout`` given -> *model-specialised* module: term metadata and the
    CTA -> segment map are compiled in as constants (used for models with at
    most ``device.META_CONST_MAX_TERMS`` terms).  Otherwise a generic module
    that reads the term/segment tables at run time, from constant memory when
    ``meta_const`` or from global memory (very large term counts)."""
    seen: set = set()
    parts = ["// generated by paper_2510_12897_b200.jit",
             f"#define EXA_META_CONST {1 if (meta_const and layout is None) else 0}",
             f"#define EXA_PDL {1 if PDL else 0}",
             _inline_header("exa_device.h", seen), _inline_header("exa_math.h", seen), _PRELUDE]
    if SINCOS_IMPL == "cuda":
        parts.append("#define exa_sincos(x, s, c) sincos((x), (s), (c))")
    for pc in patterns:
        parts.append(f"// ---- pattern {pc.pid}: k={pc.k}, {len(pc.tape.instr)} instrs")
        parts.append(pc.source)
    term_cases = "\n".join(
        f"    case {pc.pid}: exa_term_{pc.pid}<MODE>(T, r, A, rank); break;" for pc in patterns)
    val_cases = "\n".join(f"    case {pc.pid}: return exa_val_{pc.pid}(T, r, A, rank);" for pc in patterns)
    parts.append(_COMMON.replace("@TERM_CASES@", term_cases).replace("@VAL_CASES@", val_cases))
    if layout is None:
        parts.append(_KERNELS_GENERIC)
        parts.append(_ENTRIES)
    else:
        parts.append(_specialised_kernels(layout))
    bl = f"{THREADS}, {MIN_BLOCKS}" if MIN_BLOCKS else str(THREADS)
    return "\n".join(parts).replace("@BOUNDS_L@", bl).replace("@BOUNDS_H@", str(THREADS_HEAVY))


def compile_module(src: str) -> bytes:
    """NVRTC -> sm_100a cubin (cached)."""
    opts = NVRTC_OPTIONS
    key = hashlib.sha256((src + "\0" + " ".join(opts) + "\0" + _lib.nvrtc_version()).encode()).hexdigest()
    with _lock:
        got = _mem_cache.get(key)
        if got is not None:
            return got
        path = CACHE_DIR / f"{key}.cubin"
        if path.is_file():
            data = path.read_bytes()
        else:
            # the source is kept beside the cubin under the name NVRTC records in
            # -lineinfo, so `ncu --import-source on` resolves generated lines
            src_path = CACHE_DIR / f"{key}.cu"
            try:
                CACHE_DIR.mkdir(parents=True, exist_ok=True)
                src_path.write_text(src)
            except OSError:
                pass
            data = _lib.jit_compile(src, opts, name=str(src_path))
            try:
                CACHE_DIR.mkdir(parents=True, exist_ok=True)
                tmp = path.with_suffix(f".tmp{os.getpid()}")
                tmp.write_bytes(data)
                tmp.replace(path)
            except OSError:
                pass
        _mem_cache[key] = data
        return data
