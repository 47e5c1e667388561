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
import re
import threading
from pathlib import Path

import numpy as np

from . import _lib
from .codegen import group_source

CSRC = Path(__file__).resolve().parent / "csrc"
CACHE_DIR = Path(os.environ.get("EXA_JIT_CACHE", Path(__file__).resolve().parent / "_jit"))
NVRTC_OPTIONS = ("-arch=sm_100a", "--fmad=false", "-default-device", "-std=c++17", "-lineinfo",
                 "--extra-device-vectorization")
# CTA size of the fused kernels: "auto" = 32 threads when the whole set fits
# one wave of 32-thread CTAs (single instances: fine-grained balance of the
# long flow CTAs over the SMs), else 256 (batched sets of many waves: fewer
# CTA launches; N-1 1024 x case2000 1187 -> 1011 us, MP96 46.0 -> 43.8 us)
THREADS_ENV = os.environ.get("EXA_THREADS", "auto")
THREADS_HEAVY = int(os.environ.get("EXA_THREADS_HEAVY", "128"))  # heavy kernels (EXA_SPLIT experiment)
SM_COUNT = 148
# tuning knobs (experiments only; defaults are the product configuration)
MINB_ENV = os.environ.get("EXA_MINB")  # default: 1024 threads/SM -> <= 64 registers


def choose_threads(n_threads: int) -> int:
    """CTA size for a set kernel that needs ``n_threads`` threads in total."""
    if THREADS_ENV != "auto":
        return int(THREADS_ENV)
    return 32 if (n_threads + 31) // 32 <= SM_COUNT * 32 else 256


def min_blocks(threads: int) -> int:
    return int(MINB_ENV) if MINB_ENV is not None else max(1, 1024 // threads)
SC_TABLE = os.environ.get("EXA_SC_TABLE", "global")  # sin/cos table: "global" (L1/L2) or "const"
# sin/cos slow path (Ziv's rare fallback) inline behind a warp-uniform branch
# instead of an out-of-line call (whose ABI spills live values around it)
SC_SLOW_INLINE = os.environ.get("EXA_SC_SLOW_INLINE", "0") == "1"
SINCOS_IMPL = os.environ.get("EXA_SINCOS_IMPL", "cr")  # "cuda" = libdevice sincos, NOT parity-exact
# Persistent specialised kernels (experiment, off): each real CTA runs PERSIST
# virtual CTAs of THREADS threads side by side and strides over the model's
# virtual CTAs.  Measured slower than one CTA per virtual CTA (static
# assignment cannot balance the long flow CTAs).
PERSIST = int(os.environ.get("EXA_PERSIST", "0"))
TRACE = os.environ.get("EXA_TRACE", "0") == "1"  # per-warp timeline (diagnostics builds)
# bulk L2 prefetch of x, y per set (one-wave sets): +2% before the evict-first
# cache policy, -0.5% after it (5.66 vs 5.63 us at case13659); off by default
PREFETCH_XY = os.environ.get("EXA_PREFETCH_XY", "0") == "1"
PREFETCH_CHUNK = int(os.environ.get("EXA_PREFETCH_CHUNK", "32768"))
# Programmatic dependent launch: a CTA releases the next grid once its work is
# issued; the next grid's CTAs load their (immutable) plan data before
# griddepcontrol.wait, so back-to-back sets overlap one's drain with the next's
# launch and first DRAM round trip (case13659: 8.8 -> 8.3 us per set).  The
# library sets the launch attribute only for modules built with the waits.
PDL = os.environ.get("EXA_PDL", "1") == "1"
PDL_EARLY = os.environ.get("EXA_PDL_EARLY", "0") == "1"
# row buckets' release point: 1 = once their entry gathers are issued, 2 = right
# after the wait, 0 = CTA end; "auto" = 2 for one-wave sets (case13659: 0 ->
# 1 6.53 -> 6.40 us; with the evict-first cache policy 2 beats 1, 5.99 ->
# 5.92), 0 for many-wave ones (MP96: 1 costs 2%, N-1 1%)
PDL_MID_BKT = os.environ.get("EXA_PDL_MID_BKT", "auto")


def _bkt_release(threads: int) -> int:
    if PDL_MID_BKT == "auto":
        return 2 if threads == 32 else 0
    return int(PDL_MID_BKT)
PDL_MID = int(os.environ.get("EXA_PDL_MID", "1"))
ST_CS = os.environ.get("EXA_ST_CS", "1") == "1"  # evict-first stores of the c / J / H outputs
LD_CS = os.environ.get("EXA_LD_CS", "1") == "1"  # evict-first loads of the per-record parameters
_LD_RES = (re.compile(r"__ldg\((T\d*\.(?:f|ix)\[[^\]]*\] \+ (?:r|o))\)"),
           re.compile(r"__ldg\((reinterpret_cast<const int2\*>\(A\.i32 \+ \d+LL\) \+ [^;]*?)\)(?=;)"),
           re.compile(r"__ldg\((A\.i32 \+ \d+LL \+ q)\)"),
           re.compile(r"__ldg\(((?:T\d*|U\d+)\.rows \+ [^)]*)\)"))
_ST_RE = re.compile(r"\b(Cout|A\.c)\[([^\]\[]*)\] = ([^;]*);")
_ST_JH_RE = re.compile(r"\b(Jout|Hout)\[([^\]\[]*)\] = ([^;]*);")  # release point inside term groups (see EXA_GRID_RELEASE_MID)

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
#if EXA_PDL_EARLY
// release right after the wait: the next grid launches once every CTA of this
// one is past its wait (so at most one grid runs ahead) and its resident CTAs
// fetch their plan data while this grid computes
#define EXA_GRID_WAIT() asm volatile("griddepcontrol.wait;\n\tgriddepcontrol.launch_dependents;" ::: "memory")
#define EXA_GRID_RELEASE() do {} while (0)
#else
#define EXA_GRID_WAIT() asm volatile("griddepcontrol.wait;" ::: "memory")
#define EXA_GRID_RELEASE() asm volatile("griddepcontrol.launch_dependents;" ::: "memory")
#endif
#else
#define EXA_GRID_WAIT() do {} while (0)
#define EXA_GRID_RELEASE() do {} while (0)
#endif
// release the dependent grid from inside the term groups: 1 (default) = once
// a group's gathers are issued, 2 = once its sin/cos are done, 0 = only at
// CTA end (row buckets and terms always release at CTA end).  The next grid's
// CTAs take slots as this grid's CTAs exit and load their plan data during
// this grid's store tail.  case13659 (buckets dispatched first) 6.94 / 6.70 /
// 6.53 us for 0 / 2 / 1; MP96 41.44 (2) -> 41.26 (1)
#if EXA_PDL && EXA_PDL_MID
#define EXA_GRID_RELEASE_MID(k) do { if ((k) == EXA_PDL_MID) asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); } while (0)
#else
#define EXA_GRID_RELEASE_MID(k) do {} while (0)
#endif
// diagnostics (EXA_TRACE=1 builds only): per warp and virtual CTA, 12 words
// (SM id, virtual CTA, clock64 start/end, globaltimer start/end, 4 phase
// stamps of lane 0 (clock64, 0 = not reached), 2 unused) into A.trace
#if EXA_TRACE
__device__ __forceinline__ long long exa_gtimer() { long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__shared__ long long exa_tp_s[EXA_TRACE_NT][4];
// phase stamp k once `dep` is available (the asm input waits on its scoreboard)
#define EXA_TP(k, dep)                                                          \
  do {                                                                          \
    long long t_;                                                               \
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t_) : "d"((double)(dep)));     \
    exa_tp_s[threadIdx.x][k] = t_;                                              \
  } while (0)
#define EXA_TRACE_BEGIN() const long long exa_c0_ = clock64(), exa_g0_ = exa_gtimer(); \
  exa_tp_s[threadIdx.x][0] = exa_tp_s[threadIdx.x][1] = exa_tp_s[threadIdx.x][2] = exa_tp_s[threadIdx.x][3] = 0
#define EXA_TRACE_END(b, tid, nthreads)                                                       \
  do {                                                                                      \
    __syncwarp();                                                                           \
    if (A.trace && ((tid) & 31) == 0) {                                                     \
      unsigned smid; asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));                      \
      long long* tr_ = A.trace + 12LL * ((long long)(b) * ((nthreads) / 32) + (tid) / 32);  \
      tr_[0] = smid; tr_[1] = (b); tr_[2] = exa_c0_; tr_[3] = clock64();                    \
      tr_[4] = exa_g0_; tr_[5] = exa_gtimer();                                              \
      for (int k_ = 0; k_ < 4; ++k_) tr_[6 + k_] = exa_tp_s[threadIdx.x][k_];               \
    }                                                                                       \
  } while (0)
#else
#define EXA_TRACE_BEGIN() do {} while (0)
#define EXA_TRACE_END(b, tid, nthreads) do {} while (0)
#define EXA_TP(k, dep) do {} while (0)
#endif
"""

_PREFETCH = r"""
// per-record parameter loads (see _cache_hints): evict-first (LDH = 1) when a
// launch evaluates one set; the strided-batch kernel (LDH = 0) reads the same
// parameters for every set of the launch, so there they stay in L2.  LDH is a
// template parameter of the generated functions; this is the default outside.
// Bit 2 of LDH (compressed-set kernels, exa_k_setc_*) keeps the raw J / H
// slots in L2 (plain instead of evict-first stores): the segmented sum reads
// them right back and the next set overwrites the workspace scratch.
constexpr int LDH = 1;
#define EXA_LDP(p) ((LDH & 1) ? __ldcs(p) : __ldg(p))
#define EXA_STO(p, v) do { if (LDH & 2) *(p) = (v); else __stcs((p), (v)); } while (0)
// Bulk L2 prefetch of the gathered inputs: CTA b < n prefetches chunk b of x
// (then of y).  The first random gathers of a set would otherwise miss L2
// (the previous set used other buffers) and go to DRAM one 32-B sector at a
// time; a prefetch is only a read into L2, so issuing it before
// griddepcontrol.wait is safe (L2 is the point of coherence).
__device__ __forceinline__ void exa_prefetch_l2(const void* base, long long bytes, int chunk, int c) {
  const long long off = (long long)c * chunk;
  if (off >= bytes) return;
  const char* p = reinterpret_cast<const char*>(base) + off;
  long long len = bytes - off < chunk ? bytes - off : chunk;
  len &= ~15LL;
  if (len <= 0 || (reinterpret_cast<unsigned long long>(p) & 15)) return;
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"((unsigned)len) : "memory");
}
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
// ---- metadata: run-time term / segment tables in global memory -----------
#define EXA_TERM(i) terms[(i)]

template <int MODE>
__device__ __forceinline__ void exa_kernel_body(const ExaTerm* __restrict__ terms, const ExaSeg* __restrict__ segs,
                                                const int* __restrict__ cta_seg, const ExaArgs& A) {
  const ExaSeg sg = segs[__ldg(cta_seg + blockIdx.x)];
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
#define EXA_ENTRY(NAME, MODE, ...)                                                             \
  extern "C" __global__ void __launch_bounds__(__VA_ARGS__) NAME(                             \
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


def _specialised_kernels(layout, compressed: bool = False) -> str:
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
        lines.append(f"  T.per = {d.get('per', 0)}; T.fmask = {d.get('fmask', 0)}u; T.imask = {d.get('imask', 0)}u;"
                     f" T.kcol = {d.get('kcol', -1)}; T.g0 = {d.get('g0', 0)};")
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
    # row buckets: value of one pre-resolved augment entry (gid | sel << 29)
    # given its gathered variable, and (set kernel) its J/H slot stores.  The
    # last augment is the default case, so every path is branch-free selects.
    for t, info in getattr(layout, "buckets", {}).items():
        augs = info["augs"]
        cases = "\n".join(f"    case {sel}: return exa_valx_{layout.term_pid[u]}(xv);"
                           for sel, u in enumerate(augs[:-1]))
        last = f"    default: return exa_valx_{layout.term_pid[augs[-1]]}(xv);"
        out.append(f"""__device__ __forceinline__ double exa_bkval_T{t}(const int e, const double xv) {{
  switch ((unsigned)e >> 29) {{
{cases}
{last}
  }}
}}""")
        descs = layout.term_descs()
        oc = []
        for sel, u in enumerate(augs):
            lab = f"    case {sel}:" if sel < len(augs) - 1 else "    default:"
            oc.append(f"{lab} exa_termx_{layout.term_pid[u]}(xv, w, jv, hv); j0 = {descs[u]['jac0']}LL;"
                      f" h0 = {descs[u]['hess0']}LL; break;")
        ocases = "\n".join(oc)
        out.append(f"""template <int WJ, int WH, int LDH = 1>
__device__ __forceinline__ void exa_bkout_T{t}(const int e, const double xv, const double w, const int rec, const ExaArgs& A) {{
  double jv, hv;
  long long j0, h0;
  switch ((unsigned)e >> 29) {{
{ocases}
  }}
  double* __restrict__ Jout = A.J;  // restrict: later gathers may be hoisted above these stores
  double* __restrict__ Hout = A.H;
  if (WJ) Jout[j0 + rec] = jv;
  if (WH) Hout[h0 + rec] = hv;
}}""")
    jdir = getattr(layout, "jdirect", {}) if compressed else {}
    hloc = getattr(layout, "hlocal", {}) if compressed else {}

    def member_meta(gid, m, u, mem):
        if not compressed:
            return mem
        extra = {"cmp": True}
        if u in jdir:
            extra["jc0"] = jdir[u]
            # many-wave sets (256-thread CTAs): stage the warp's direct entries
            # in shared memory and store them coalesced (MP96 compressed set
            # 111 -> 99 us); one-wave sets store them where they are computed
            # (case13659 14.3 vs 15.8 us staged: the extra barriers sit on the
            # critical path)
            extra["jst"] = ("member" if layout.threads[1] > 32
                            else ("group" if os.environ.get("EXA_JST_ONEWAVE") == "1" else None))
        cls = hloc.get(gid, {}).get(m)
        if cls:
            extra["hcls"] = {pair: (c, q, size, zero) for pair, (c, q, size, _off, zero) in cls.items()}
            extra["hcls_pos"] = [(c, q, size, off) for (c, q, size, off, _zero) in cls.values()]
        return dict(mem, **extra)

    for gid, (pid, grp, members) in enumerate(getattr(layout, "groups", [])):
        augs = [(layout.patterns[layout.term_pid[u]], off, m, s_, _aug_row_source(layout, grp, members, u, off))
                for (u, off, m, s_) in getattr(layout, "group_augs", {}).get(gid, [])]
        out.append(group_source(gid, [(layout.patterns[layout.term_pid[u]], member_meta(gid, m, u, mem))
                                      for m, (u, mem) in enumerate(zip(grp, members))],
                                augs, relax=layout.relax))
    if compressed:  # the compressed-set module: set kernels only
        for half, suffix in ((0, "_h"), (1, "_l")):
            out.append(_kernel_source(layout, 0, half, "exa_k_setc" + suffix, ldh=3))
    else:
        for m, name in enumerate(KERNEL_NAMES):
            for half, suffix in ((0, "_h"), (1, "_l")):
                out.append(_kernel_source(layout, m, half, name + suffix))
    return _cache_hints("\n\n".join(out))


def _aug_row_source(layout, grp, members, u, off):
    """(group index column id, constant) when an attached augment's rows are
    ``constant + that index column`` record for record (OPF: the balance row
    of the bus a flow's from-/to-end index names, ``row_offset + i``): the
    group then loads the row's multiplier directly, without the augment's
    row column in between (exact zero-sign mode: its w * 0 Hessian entry).
    None otherwise."""
    a = layout.terms[u]
    n = layout.terms[grp[0]].nrec
    rows = np.asarray(a.rows, dtype=np.int64)[off:off + n]
    for m, t in enumerate(grp):
        tp = layout.terms[t]
        for c, nm in enumerate(tp.tape.index_names):
            col = np.asarray(tp.table.indices[nm], dtype=np.int64)
            if col.size != n:
                continue
            d = rows - col
            if d.size and np.all(d == d[0]):
                return members[m]["cols"][c], int(d[0])
    return None


def _cache_hints(src: str) -> str:
    """L2 policy of the generated code's global accesses (a rewrite of the
    emitted statements):

    * c / J / H are written once and never read back by the kernel: streamed
      past L2 with evict-first stores (``st.global.cs``), keeping L2 for x, y
      and the next set's loads (case13659 6.36 -> 6.27 us, MP96 41.1 -> 40.0);
    * per-record parameters (field and index columns, row-bucket entries and
      rows, augment row ids) are read once per set: evict-first loads
      (``ld.global.cs``), so they do not displace the gathered x / y lines
      (case13659 6.27 -> 6.10 us, MP96 40.0 -> 39.4, N-1 -0.5%).
    x and y keep ``__ldg`` (gathered, reused across records)."""
    if ST_CS:
        src = _ST_RE.sub(r"__stcs(&\1[\2], \3);", src)
        src = _ST_JH_RE.sub(r"EXA_STO(&\1[\2], \3);", src)
    if LD_CS:
        for pat in _LD_RES:
            src = pat.sub(r"EXA_LDP(\1)", src)
    return src


def _mode_outputs(m):
    """(row value, J slots, H slots) a bucket segment produces in kernel m."""
    return m in (0, 1), m in (0, 2), m in (0, 3)


def _warp_row_source(layout, t, bi, cta0, n_cta, threads, m):
    """Long rows of a bucketed block: one warp per row.  Lane 0 evaluates the
    base term, lane l > 0 augment entry l-1; the row total is folded left to
    right through the lanes with shuffles -- ((0 + base) + a1) + a2 ... as the
    reference's slice-add + np.add.at (autodiff.py:573-580).  In the jac /
    hess kernels only the J / H slots of the base term and the augments."""
    want_v, want_j, want_h = _mode_outputs(m)
    bk = layout.buckets[t]["buckets"][bi]
    n = bk["n"]
    pid = layout.term_pid[t]
    base_mode = " | ".join(x for x, w in (("EXA_M_JAC", want_j), ("EXA_M_HESS", want_h)) if w)
    L = [f"  if (b < {cta0 + n_cta}) {{", f"    ExaTerm T; exa_init_T{t}(T, A);"]
    for i, off in enumerate(bk["f_off"]):
        L.append(f"    T.f[{i}] = A.f64 + {off}LL;")
    for i, off in enumerate(bk["ix_off"]):
        L.append(f"    T.ix[{i}] = A.i32 + {off}LL;")
    L.append("    T.fmask = 0u; T.imask = 0u;  // bucket-order copies are per row")
    LW = bk["d"]  # lanes per row: 32, or 16 (two rows per warp)
    if LW == 32:
        L += [f"    const int q = (b - {cta0}) * {threads // 32} + tid / 32;",
              "    const int lane = tid & 31;",
              f"    if (q >= {n}) return;  // warp-uniform"]
    else:  # the second half of the last warp may redo row n-1 (same values, same slots)
        L += [f"    const int q = min((b - {cta0}) * {threads // 16} + tid / 16, {n - 1});",
              "    const int lane = tid & 15;"]
    L += [f"    const int r = __ldg(A.i32 + {bk['rows_off']}LL + q);",
          f"    const int2 er = __ldg(reinterpret_cast<const int2*>(A.i32 + {bk['pair_off']}LL) + {LW} * q + lane);",
          "    const int e = er.x, rc = er.y;",
          "    EXA_GRID_WAIT();"]
    if _bkt_release(threads):  # warp rows: release right after the wait
        L.append("    EXA_GRID_RELEASE();")
    L.append("    const double wrow = " + ("__ldg(A.y + T.row_offset + r);" if want_h else "0.0;"))
    L += ["    double v = 0.0;",
          "    if (lane == 0) {"]
    if want_v:
        L.append(f"      v = exa_val_{pid}<LDH>(T, q, A, exa_rank(T, A));")
    if base_mode and layout.buckets[t]["base_k"]:
        L.append(f"      exa_term_{pid}<{base_mode}, LDH>(T, q, A, exa_rank(T, A), r);")
    L += ["    } else {",
          f"      const double xv = __ldg(A.x + (e & {(1 << 29) - 1} & ~(e >> 31)));"]
    if want_v:
        L.append(f"      v = exa_bkval_T{t}(e, xv);")
    if want_j or want_h:
        L.append(f"      if (e >= 0 && rc >= 0) exa_bkout_T{t}<{int(want_j)}, {int(want_h)}, LDH>(e, xv, wrow, rc, A);")
    L.append("    }")
    if want_v:
        if LW == 32:
            L += ["    const int d = __popc(__ballot_sync(0xffffffffu, e >= 0));  // entries in lanes 1..d",
                  "    const int dm = d;"]
        else:  # per half: own count d, loop to the larger of the two halves' counts
            L += ["    const unsigned bal = __ballot_sync(0xffffffffu, e >= 0);",
                  "    const int d = __popc((bal >> (tid & 16)) & 0xffffu);  // entries in lanes 1..d",
                  "    const int dm = max(__popc(bal & 0xffffu), __popc(bal >> 16));"]
        L += ["    double acc = lane == 0 ? 0.0 + v : v;",
              "    for (int s = 1; s <= dm; ++s) {",
              f"      const double up = __shfl_up_sync(0xffffffffu, acc, 1, {LW});",
              "      if (lane == s && s <= d) acc = up + v;",
              "    }",
              "    if (lane == d) A.c[T.row_offset + r] = acc;"]
    L += ["    return;", "  }"]
    return L


def _kernel_source(layout, m, half, kname, ldh: int = 1) -> str:
    """One entry kernel of a specialised module.

    ``exa_vb_<kname>(b, tid, A)`` evaluates virtual CTA ``b`` (the segment
    table's CTA numbering, ``threads`` threads).  Classic mode: one real CTA
    per virtual CTA.  Persistent mode (``layout.persist[kid] = V > 0``): a
    real CTA of ``V * threads`` threads holds V virtual CTAs; slot j of real
    CTA c serves virtual CTAs ``c + G*j + G*V*k`` (G = gridDim.x, k = 0, 1,
    ...), so every segment is spread over all SMs.  With ``EXA_TRACE`` each
    warp records (SM, clock64 start, end, virtual CTA) per virtual CTA."""
    kid = 2 * m + half
    threads = layout.threads[half]
    V = layout.persist[kid]
    bounds = "@BOUNDS_H@" if half == 0 else "@BOUNDS_L@"
    if V:
        bounds = f"{threads * V}, {max(1, min_blocks(threads) // V)}"
    segs = layout.mode_segments(kid)
    n_vb = sum((nrec + threads * rpt - 1) // (threads * rpt) for (_, _, _, nrec, rpt) in segs)
    fn_body = [f"template <int LDH>\n__device__ __forceinline__ void exa_vb_{kname}(const int b, const int tid, const ExaArgs& A) {{"]
    for (t, kind, cta0, nrec, rpt) in segs:
        n_cta = (nrec + threads * rpt - 1) // (threads * rpt)
        b_ = [f"  if (b < {cta0 + n_cta}) {{"]
        if kind & 15 == 4 and layout.buckets[t]["buckets"][kind >> 4]["d"] >= 16:
            fn_body += _warp_row_source(layout, t, kind >> 4, cta0, n_cta, threads, m)
            continue
        if kind & 15 == 4:  # row bucket of augment-target block t: one thread per row
            bk = layout.buckets[t]["buckets"][kind >> 4]
            dd, n = bk["d"], bk["n"]
            b_.append(f"    ExaTerm T; exa_init_T{t}(T, A);")
            for i, off in enumerate(bk["f_off"]):
                b_.append(f"    T.f[{i}] = A.f64 + {off}LL;")
            for i, off in enumerate(bk["ix_off"]):
                b_.append(f"    T.ix[{i}] = A.i32 + {off}LL;")
            b_.append("    T.fmask = 0u; T.imask = 0u;  // bucket-order copies are per row")
            b_.append(f"    const int q = (b - {cta0}) * {threads} + tid;")
            b_.append(f"    if (q >= {n}) return;")
            b_.append(f"    const int r = __ldg(A.i32 + {bk['rows_off']}LL + q);")
            # width class dd: entries k <= dd/2 always present, later ones may be -1
            always = dd // 2 + 1 if dd > 1 else dd
            # set kernel: row value, base term's and augments' J/H slots; cons:
            # the value; jac / hess: only their slots
            want_v, want_j, want_h = _mode_outputs(m)
            info = layout.buckets[t]
            need_x = want_v or not all(getattr(layout.patterns[layout.term_pid[u]], "termx_const", False)
                                       for u in info["augs"])
            base_mode = " | ".join(x for x, w in (("EXA_M_JAC", want_j), ("EXA_M_HESS", want_h)) if w)
            # chunks of 8 entries: loads, gathers (unconditional), in-order adds
            for c0 in range(0, max(dd, 1), 8):
                ks = range(c0, min(dd, c0 + 8))
                for k in ks:
                    b_.append(f"    const int2 er{k} = __ldg(reinterpret_cast<const int2*>(A.i32 + {bk['pair_off']}LL) + {k * n} + q);")
                    b_.append(f"    const int e{k} = er{k}.x, rc{k} = er{k}.y;")
                if c0 == 0:
                    b_.append(f"    EXA_TP(0, {'e0' if dd else 'r'});")
                    b_.append("    EXA_GRID_WAIT();")
                    if _bkt_release(threads) == 2:
                        b_.append("    EXA_GRID_RELEASE();")
                    b_.append("    const double wrow = " + ("__ldg(A.y + T.row_offset + r);" if want_h else "0.0;"))
                    if want_v:
                        # base value first: its gathers issue with the entries' (a later
                        # re-load behind the base J/H stores would cost a round trip)
                        b_.append(f"    const double base = exa_val_{layout.term_pid[t]}<LDH>(T, q, A, exa_rank(T, A));")
                for k in ks:
                    # pad entries (-1) gather x[0]: branch-free, selected away below
                    xv = f"__ldg(A.x + (e{k} & {(1 << 29) - 1} & ~(e{k} >> 31)))" if need_x else "0.0"
                    b_.append(f"    const double xv{k} = {xv};")
                    if want_v:
                        b_.append(f"    const double v{k} = exa_bkval_T{t}(e{k}, xv{k});")
                if c0 == 0:
                    if ks and need_x:
                        b_.append("    EXA_TP(1, " + " + ".join(f"xv{k}" for k in ks) + ");")
                        if _bkt_release(threads) == 1:
                            b_.append("    EXA_GRID_RELEASE();")
                    # base term J/H after the entry gathers are issued (in-order issue:
                    # its stores wait on its own gather and would hold the others back)
                    if base_mode and info["base_k"]:
                        b_.append(f"    exa_term_{layout.term_pid[t]}<{base_mode}, LDH>(T, q, A, exa_rank(T, A), r);")
                    if want_v:
                        # reference order: zero-fill, base slice-add, augments in order (autodiff.py:573-580)
                        b_.append("    double acc = 0.0 + base;")
                for k in ks:
                    if want_v:
                        if k < always:
                            b_.append(f"    acc = acc + v{k};")
                        else:
                            b_.append(f"    acc = e{k} >= 0 ? acc + v{k} : acc;")
                    if want_j or want_h:
                        cond = f"if (rc{k} >= 0) " if k < always else f"if (e{k} >= 0 && rc{k} >= 0) "
                        b_.append(f"    {cond}exa_bkout_T{t}<{int(want_j)}, {int(want_h)}, LDH>(e{k}, xv{k}, wrow, rc{k}, A);")
            if want_v:
                b_.append("    A.c[T.row_offset + r] = acc;")
            b_.append("    return;")
            b_.append("  }")
            fn_body += b_
            continue
        if kind == 3:  # term group: t is the group id
            pid, grp, _ = layout.groups[t]
            for gm, u in enumerate(grp):
                b_.append(f"    ExaTerm T{gm}; exa_init_T{u}(T{gm}, A);")
            gaugs = getattr(layout, "group_augs", {}).get(t, [])
            for k, (u, _, _, _) in enumerate(gaugs):
                b_.append(f"    ExaTerm U{k}; exa_init_T{u}(U{k}, A);")
            tl = ", ".join([f"T{gm}" for gm in range(len(grp))] + [f"U{k}" for k in range(len(gaugs))])
            rl = ", ".join(f"exa_rank(T{gm}, A)" for gm in range(len(grp)))
            if rpt == 1:
                b_.append(f"    const int r = (b - {cta0}) * {threads} + tid;")
                b_.append(f"    if (r >= {nrec}) return;")
                b_.append(f"    exa_grp_{t}<{_MODE_BITS[m]}, LDH>({tl}, r, A, {rl});")
            else:
                b_.append(f"    const int r0 = (b - {cta0}) * {threads * rpt} + tid;")
                b_.append("#pragma unroll")
                b_.append(f"    for (int q = 0; q < {rpt}; ++q) {{")
                b_.append(f"      const int r = r0 + q * {threads};")
                b_.append(f"      if (r < {nrec}) exa_grp_{t}<{_MODE_BITS[m]}, LDH>({tl}, r, A, {rl});")
                b_.append("    }")
        else:
            b_.append(f"    ExaTerm T; exa_init_T{t}(T, A);")
            if kind == 0:
                b_.append(f"    const int r0 = (b - {cta0}) * {threads * rpt} + tid;")
                b_.append("#pragma unroll")
                b_.append(f"    for (int q = 0; q < {rpt}; ++q) {{")
                b_.append(f"      const int r = r0 + q * {threads};")
                b_.append(f"      if (r < {nrec}) exa_term_{layout.term_pid[t]}<{_MODE_BITS[m]}, LDH>(T, r, A, exa_rank(T, A));")
                b_.append("    }")
            else:  # fold rows are padded to whole warps: a warp never splits here
                b_.append(f"    const int r = (b - {cta0}) * {threads} + tid;")
                b_.append(f"    if (r >= {nrec}) return;")
                fn = "exa_rowfold" if kind == 2 else "exa_row"
                b_.append(f"    {fn}(T, r, A, [&](int u, int rec) {{ return exa_rowval_T{t}(u, rec, A); }});")
        b_.append("    return;")
        b_.append("  }")
        fn_body += b_
    fn_body.append("}")
    plan = layout.plan
    body = [f"extern \"C\" __global__ void __launch_bounds__({bounds}) {kname}(",
            "    const ExaTerm* __restrict__ terms, const ExaSeg* __restrict__ segs,",
            "    const int* __restrict__ cta_seg, ExaArgs A) {",
            # strided batches (exa_eval_set_batch): set blockIdx.y; 0 for single sets
            "  { const long long k_ = blockIdx.y;",
            f"    A.x += k_ * {plan.nvar}LL; A.y += k_ * {plan.ncon}LL; A.c += k_ * {plan.ncon}LL;",
            f"    A.J += k_ * {plan.n_jac_slots}LL; A.H += k_ * {plan.n_hess_slots}LL; }}"]
    # single-wave sets only (measured: +2% at case13659; batched sets, whose x
    # and y are tens of MB, lose 3-4% to the extra L2 traffic)
    if PREFETCH_XY and not V and threads == 32:
        nvar, ncon = layout.plan.nvar, layout.plan.ncon
        ch = PREFETCH_CHUNK
        ncx = (8 * nvar + ch - 1) // ch
        body.append(f"  if (threadIdx.x == 0 && blockIdx.x < {ncx}) exa_prefetch_l2(A.x, {8 * nvar}LL, {ch}, (int)blockIdx.x);")
        if m in (0, 3):  # set / hess kernels gather multipliers too
            ncy = (8 * ncon + ch - 1) // ch
            body.append(f"  if (threadIdx.x == 0 && blockIdx.x >= {ncx} && blockIdx.x < {ncx + ncy}) "
                        f"exa_prefetch_l2(A.y, {8 * ncon}LL, {ch}, (int)blockIdx.x - {ncx});")
    if V:
        body += [f"  const int tid = (int)threadIdx.x % {threads};",
                 f"  for (int b = (int)blockIdx.x + (int)gridDim.x * ((int)threadIdx.x / {threads}); b < {n_vb};"
                 f" b += (int)gridDim.x * {V}) {{",
                 "    EXA_TRACE_BEGIN();",
                 f"    exa_vb_{kname}<@LDH@>(b, tid, A);",
                 f"    EXA_TRACE_END(b, tid, {threads});",
                 "  }"]
    else:
        perm = getattr(layout, "cta_perm_off", None)
        b0 = f"__ldg(A.i32 + {perm}LL + blockIdx.x)" if (perm is not None and kid == 1) else "(int)blockIdx.x"
        body += ["  EXA_TRACE_BEGIN();",
                 f"  const int vb_ = {b0};",
                 f"  exa_vb_{kname}<@LDH@>(vb_, (int)threadIdx.x, A);",
                 f"  EXA_TRACE_END(vb_, (int)threadIdx.x, {threads});"]
    # release the dependent grid only when this CTA's work is issued (an early
    # release lets later grids' waiting CTAs take the slots this grid needs)
    body.append("  EXA_GRID_RELEASE();")
    body.append("}")
    entry = "\n".join(body)
    out = "\n".join(fn_body) + "\n" + entry.replace("@LDH@", str(ldh))
    if m == 0 and half == 1 and ldh == 1:  # strided-batch entry (exa_eval_set_batch): parameters stay in L2
        out += "\n" + entry.replace("@LDH@", "0").replace(f" {kname}(", f" {kname.replace('_set_', '_setb_')}(", 1)
    return out


KERNEL_NAMES = ("exa_k_set", "exa_k_cons", "exa_k_jac", "exa_k_hess", "exa_k_objv", "exa_k_grad")


def module_source(patterns, layout=None, threads: int = 32, compressed: bool = False) -> str:
    """CUDA source of a model's module.

    ``layout`` given -> *model-specialised* module: term metadata and the
    CTA -> segment map are compiled in as constants (used for models with at
    most ``device.META_CONST_MAX_TERMS`` terms).  Otherwise a generic module
    that reads the term/segment tables from global memory at run time."""
    seen: set = set()
    parts = ["// generated by paper_2510_12897_b200.jit",
             f"#define EXA_PDL {1 if PDL else 0}",
             f"#define EXA_PDL_EARLY {1 if PDL_EARLY else 0}",
             f"#define EXA_PDL_MID {PDL_MID}",
             f"#define EXA_TRACE {1 if TRACE else 0}",
             "#define EXA_SC_CONST 1" if SC_TABLE == "const" else "",
             "#define EXA_SC_SLOW_INLINE 1" if SC_SLOW_INLINE else "",
             f"#define EXA_TRACE_NT {max(threads, THREADS_HEAVY) * max(1, PERSIST)}",
             _inline_header("exa_device.h", seen), _inline_header("exa_math.h", seen), _PRELUDE]
    if SINCOS_IMPL == "cuda":
        parts.append("#define exa_sincos(x, s, c) sincos((x), (s), (c))")
    for pc in patterns:
        parts.append(f"// ---- pattern {pc.pid}: k={pc.k}, {len(pc.tape.instr)} instrs")
        parts.append(pc.source)
    term_cases = "\n".join(
        f"    case {pc.pid}: exa_term_{pc.pid}<MODE>(T, r, A, rank); break;" for pc in patterns)
    val_cases = "\n".join(f"    case {pc.pid}: return exa_val_{pc.pid}(T, r, A, rank);" for pc in patterns)
    parts.append(_PREFETCH)
    parts.append(_COMMON.replace("@TERM_CASES@", term_cases).replace("@VAL_CASES@", val_cases))
    if layout is None:
        parts.append(_KERNELS_GENERIC)
        parts.append(_ENTRIES)
    else:
        parts.append(_specialised_kernels(layout, compressed))
    bl = f"{threads}, {min_blocks(threads)}"
    # warps per CTA of the largest kernel (per-warp shared stages, EXA_JST)
    parts.insert(1, f"#define EXA_JST_WARPS {max(threads, THREADS_HEAVY) // 32}")
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
