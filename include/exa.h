/*
 * exa.h -- C ABI of libexa.so, the B200 (sm_100a) callback engine.
 *
 * Drop-in boundary for the reference's callback set
 * (/root/reference/pkg/src/simdnlp/autodiff.py):
 *
 *   exa_eval_obj   <- eval_objective(model, x) -> float          autodiff.py:536-547
 *   exa_eval_grad  <- eval_gradient(model, x, out_g)             autodiff.py:550-563
 *   exa_eval_cons  <- eval_constraints(model, x, out_c)          autodiff.py:566-580
 *   exa_eval_jac   <- eval_jacobian(model, x, out_vals)          autodiff.py:588-602
 *   exa_eval_hess  <- eval_hessian(model, x, mult, w, out_vals)  autodiff.py:615-652
 *   exa_eval_set   <- cons + jac + hess in one launch (the benchmarked unit)
 *   exa_segment_sum <- CompressedPattern.sum_values(raw)         autodiff.py:672-674
 *   exa_domain_error <- EvalDomainError(op, record, kind, block) autodiff.py:30-47
 *   exa_plan_create  <- ModelCore.compile / build_plan           core.py:246-280,
 *                                                                 autodiff.py:453-508
 *
 * Conventions (reference contract):
 *  - all arrays passed to exa_eval_* are DEVICE pointers on the plan's device;
 *    outputs are caller-owned and overwritten in full (grad/cons zero-filled
 *    semantics, every raw Jacobian/Hessian slot written);
 *  - evaluation is asynchronous on `stream`; no allocation, no host sync
 *    (exa_domain_error synchronises the stream to read the error word);
 *  - results are run-to-run bitwise deterministic: no floating-point atomics,
 *    fixed reduction orders equal to the reference's;
 *  - status: 0 ok, < 0 invalid argument / CUDA failure (exa_last_error());
 *  - a plan is immutable after creation and shareable across threads
 *    (reference core.py:301-305); all mutable evaluation state (obj/grad
 *    scratch, the domain-error word, host-path staging, the light kernels'
 *    aux stream) lives in an ExaWorkspace.  A workspace serves one evaluation
 *    at a time: concurrent callers pass one workspace each
 *    (exa_workspace_create); NULL selects the plan's default workspace, for
 *    single-threaded callers.  The Python layer gives every thread its own.
 */
#ifndef EXA_H
#define EXA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EXA_ABI_VERSION 6
#define EXA_MAXF 16
#define EXA_MAXI 16
#define EXA_MAXK 16

/* callback modes: indices into ExaPlanDesc.segs */
#define EXA_MODE_SET 0
#define EXA_MODE_CONS 1
#define EXA_MODE_JAC 2
#define EXA_MODE_HESS 3
#define EXA_MODE_OBJV 4
#define EXA_MODE_GRAD 5
#define EXA_NMODES 6
/* each callback runs as up to two concurrent kernels: heavy patterns
 * (transcendentals / many slots, small CTAs) and light ones (large CTAs, few
 * registers); kernel id = 2 * mode + {0 heavy, 1 light} */
#define EXA_NKERN 12

typedef struct ExaPlan ExaPlan;
typedef struct ExaWorkspace ExaWorkspace;
typedef void* exa_stream_t; /* a cudaStream_t; NULL = legacy default stream */

/* One objective block / constraint block / augment (reference TermPlan,
 * autodiff.py:413-423).  Offsets index the f64 / i32 blobs of the plan
 * descriptor; -1 = absent. */
typedef struct ExaTermDesc {
  int64_t f_off[EXA_MAXF];  /* real field columns (fp64, nrec each)          */
  int64_t ix_off[EXA_MAXI]; /* index columns (int32 in-block positions)       */
  int64_t rows_off;         /* augments: int32 global rows                    */
  int64_t row_ptr_off;      /* augment-target blocks: int32 CSR ptr (nrec+1)  */
  int64_t row_ent_off;      /*   int32 pairs (term, record), reference order  */
  int32_t voff[EXA_MAXK];   /* variable-block offset of each slot             */
  int32_t nrec, pattern, kind, order, row_offset, cons_direct, k, pad;
  int64_t jac0, hess0, scr0;
} ExaTermDesc;

/* A run of CTAs serving one term (kind 0) or one block's rows (kind 1). */
typedef struct ExaSegDesc {
  int32_t term, kind, cta0, nrec;
} ExaSegDesc;

typedef struct ExaPlanDesc {
  int32_t abi_version; /* EXA_ABI_VERSION */
  int32_t device;      /* CUDA ordinal */
  int64_t nvar, ncon, n_jac, n_hess;
  const double* f64;
  int64_t n_f64;
  const int32_t* i32;
  int64_t n_i32;
  const ExaTermDesc* terms;
  int32_t n_terms;
  int32_t threads[2]; /* CTA size of the heavy / light kernels of the module */
  const ExaSegDesc* segs[EXA_NKERN];
  int32_t n_segs[EXA_NKERN];
  int32_t n_ctas[EXA_NKERN];
  int32_t err_base[EXA_NMODES][2]; /* domain-error rank offsets: {objective, constraint} */
  /* objective: per-record value scratch, leaves and combine program
     (numpy pairwise summation order) */
  int64_t n_vscr, n_gscr;
  const int64_t* leaves; /* pairs (scratch start, length) */
  int32_t n_leaves;
  const int64_t* obj_prog; /* triples (opcode, a, b); see exa_capi.cu */
  int32_t n_prog;
  /* gradient: CSR over variables (nvar+1), entries = G index | group flag << 62 */
  const int64_t* grad_ptr;
  const int64_t* grad_ent;
  int64_t n_grad_ent;
  /* the model's generated kernels (cubin for sm_100a from exa_jit_compile) */
  const void* cubin;
  int64_t cubin_size;
  int32_t has_domain_checks;
  /* persistent kernels: persist[kid] = V > 0 -> the kernel's real CTAs hold V
     virtual CTAs (threads[kid & 1] threads each) and stride over n_ctas[kid]
     virtual CTAs; the grid is one wave (occupancy x SM count) */
  int32_t persist[EXA_NKERN];
  /* the module was built with programmatic-dependent-launch waits: launch
     with cudaLaunchAttributeProgrammaticStreamSerialization */
  int32_t pdl;
  /* the module's set kernel offsets x, mult, c, jac, hess by blockIdx.y times
     nvar, ncon, ncon, n_jac, n_hess (strided batches, exa_eval_set_batch) */
  int32_t batchable;
  /* host path (exa_eval_set_host): raw J / H slot runs whose value is the same
     constant for every record and call, int64 triples (first slot, length,
     IEEE-754 bits of the value): the first n_fill_jac index J, the next
     n_fill_hess index H, sorted and disjoint.  They are filled on the host
     instead of being copied from the device.  May be null / 0. */
  const int64_t* host_fill;
  int32_t n_fill_jac, n_fill_hess;
  /* host path, exact zero-sign modules: raw H slot runs holding the
     reference's weight * z (z = a structural +-0.0 of the pattern; the
     weight is the row's multiplier or obj_weight), int64 quadruples (first
     slot, length, offset into host_wzero_rows or -1 = obj_weight, IEEE-754
     bits of z), sorted, disjoint from each other and from the host_fill H
     runs.  Slot i of a run = mult_host[host_wzero_rows[offset + i]] * z,
     computed by host threads from the caller's multipliers (sign of zero and
     NaN / inf propagation as the reference's autodiff.py:652).  May be 0. */
  const int64_t* host_wzero;
  int32_t n_wzero, pad_wz;
  const int32_t* host_wzero_rows;
  int64_t n_wzero_rows;
} ExaPlanDesc;

/* ---- build-time: JIT ---------------------------------------------------- */
int exa_jit_compile(const char* src, const char* name, const char* const* opts, int n_opts,
                    void** cubin, size_t* cubin_size, char** log);
void exa_free(void* p);
int exa_nvrtc_version(int* major, int* minor);

/* ---- plans and workspaces ----------------------------------------------- */
int exa_plan_create(const ExaPlanDesc* desc, ExaPlan** out);
void exa_plan_destroy(ExaPlan* plan);
int exa_plan_info(const ExaPlan* plan, int64_t* bytes_device, int32_t* regs_set_kernel);
int exa_workspace_create(ExaPlan* plan, ExaWorkspace** out);
void exa_workspace_destroy(ExaWorkspace* ws);

/* ---- the callbacks (device pointers) ------------------------------------ */
int exa_eval_obj(ExaPlan* plan, ExaWorkspace* ws, const double* x, double* out_scalar,
                 exa_stream_t stream);
int exa_eval_grad(ExaPlan* plan, ExaWorkspace* ws, const double* x, double* g, exa_stream_t stream);
int exa_eval_cons(ExaPlan* plan, ExaWorkspace* ws, const double* x, double* c, exa_stream_t stream);
int exa_eval_jac(ExaPlan* plan, ExaWorkspace* ws, const double* x, double* jac, exa_stream_t stream);
int exa_eval_hess(ExaPlan* plan, ExaWorkspace* ws, const double* x, const double* mult,
                  double obj_weight, double* hess, exa_stream_t stream);
int exa_eval_set(ExaPlan* plan, ExaWorkspace* ws, const double* x, const double* mult,
                 double obj_weight, double* c, double* jac, double* hess, exa_stream_t stream);
/* nsets independent callback sets of the same model in ONE launch (strided
 * batch: set k reads x + k*nvar, mult + k*ncon and writes c + k*ncon,
 * jac + k*n_jac, hess + k*n_hess; one obj_weight).  For throughput on
 * independent evaluation points (scenario streams, multi-start, parallel
 * trial points); each set's results are bitwise those of exa_eval_set.
 * Plans with domain-checked operations or generic modules return an error. */
int exa_eval_set_batch(ExaPlan* plan, ExaWorkspace* ws, int64_t nsets, const double* x, const double* mult,
                       double obj_weight, double* c, double* jac, double* hess, exa_stream_t stream);
/* exa_eval_set with HOST buffers (the reference-facing drop-in path: numpy
 * arrays in, numpy arrays out): copies x, mult to the workspace's device
 * staging, evaluates, copies c and the x-dependent J/H ranges back -- all
 * asynchronous on `stream` (synchronise it before reading the outputs;
 * page-locked output arrays are written by one store kernel through their
 * device mapping, EXA_D2H=dma selects copy-engine transfers) -- and writes the plan's
 * constant J/H runs (ExaPlanDesc.host_fill) into jac/hess with host threads
 * before returning.  Pinned host memory makes the copies asynchronous, so
 * sets on distinct workspaces and streams overlap their H2D copy, kernel and
 * D2H copy. */
int exa_eval_set_host(ExaPlan* plan, ExaWorkspace* ws, const double* x_host, const double* mult_host,
                      double obj_weight, double* c_host, double* jac_host, double* hess_host,
                      exa_stream_t stream);
/* The separate callbacks with HOST buffers (the reference IPM calls
 * eval_constraints / eval_jacobian / eval_hessian with numpy arrays every
 * iteration; autodiff.py:566,588,615): same staging, copies and constant-run
 * fill as exa_eval_set_host.  Pageable (unregistered) host buffers go through
 * the workspace's pinned staging and the call returns with the outputs
 * complete; pinned buffers are filled asynchronously on `stream`. */
int exa_eval_cons_host(ExaPlan* plan, ExaWorkspace* ws, const double* x_host, double* c_host, exa_stream_t stream);
int exa_eval_jac_host(ExaPlan* plan, ExaWorkspace* ws, const double* x_host, double* jac_host, exa_stream_t stream);
int exa_eval_hess_host(ExaPlan* plan, ExaWorkspace* ws, const double* x_host, const double* mult_host,
                       double obj_weight, double* hess_host, exa_stream_t stream);
/* Page-lock a caller's pageable host range in place (cudaHostRegister,
 * portable + mapped) so the *_host entries above use it like page-locked
 * memory: inputs without staging, outputs written through their device
 * mapping.  The caller unregisters it (exa_host_unregister, same ptr) before
 * freeing it.  Non-zero status (message in exa_last_error) when the range
 * cannot be locked -- e.g. it overlaps a registered one; it stays pageable.
 * The Python mirror does this for numpy arrays passed again and again
 * (a solver's scratch buffers, reference solver.py:249-295). */
int exa_host_register(void* ptr, size_t bytes);
int exa_host_unregister(void* ptr);
/* ---- compressed values (what the reference solver consumes) ------------ */
/* A compressed pattern on the plan's device (reference compress_coordinates /
 * CompressedPattern, autodiff.py:660-689): nnz compressed entries over n_raw
 * raw slots; entry k = 0 + sum of raw[ent[e]], e in [ptr[k], ptr[k+1]), in
 * increasing e (np.bincount order, bit-identical to sum_values).  ptr: int64
 * [nnz + 1] from 0 to n_raw; ent: int32 [n_raw] raw slot ids.  Host arrays,
 * copied to the device. */
typedef struct ExaPattern ExaPattern;
int exa_pattern_create(ExaPlan* plan, int64_t n_raw, int64_t nnz, const int64_t* ptr, const int32_t* ent,
                       ExaPattern** out);
/* The same, told which raw slots the plan's set kernel writes as the same
 * constant on every call (known[r] != 0: raw slot r always holds
 * known_val[r]; the plan's constant Jacobian slots and, under the zero-sign
 * relaxation, its structural-zero Hessian pairs -- HostLayout fill runs).
 * The compressed sum then skips known +0.0 slots (exact: a fold that starts
 * at +0.0 never holds -0.0) and takes known constants from the pattern
 * instead of gathering them; valid only with exa_eval_set_compressed on a
 * plan whose kernels write those values. */
int exa_pattern_create_known(ExaPlan* plan, int64_t n_raw, int64_t nnz, const int64_t* ptr, const int32_t* ent,
                             const uint8_t* known, const double* known_val, ExaPattern** out);
/* A pattern for the compressed-set kernels (exa_plan_attach_compressed):
 * direct[r] != 0 flags raw slot r as folded into its compressed entry by the
 * set kernel itself (np.bincount's fold order); an entry whose slots other
 * than known +0.0 are all direct is left out of the segmented sum, an entry
 * mixing direct and other slots is an error.  Used by
 * exa_eval_set_compressed only on a plan with the compressed-set module. */
int exa_pattern_create_direct(ExaPlan* plan, int64_t n_raw, int64_t nnz, const int64_t* ptr, const int32_t* ent,
                              const uint8_t* known, const double* known_val, const uint8_t* direct,
                              ExaPattern** out);
void exa_pattern_destroy(ExaPattern* pattern);
/* Attach the compressed-set module of a plan: a cubin (exa_jit_compile) with
 * set kernels exa_k_setc_h / exa_k_setc_l that write the direct compressed
 * Jacobian entries (ExaArgs.Jc) and the group-local compressed Hessian
 * entries (ExaArgs.Hc, positions hpos[class * nrec + record], -1 = the
 * record writes its raw slots instead) and keep every other raw slot in L2
 * for the segmented sum.  Built host-side from the same layout as the
 * plan's module (paper_2510_12897_b200.device); hpos is copied. */
int exa_plan_attach_compressed(ExaPlan* plan, const void* cubin, int64_t cubin_size, const int32_t* hpos,
                               int64_t n_hpos);
/* cons + COMPRESSED Jacobian and Hessian values of one point: the set kernel
 * writes the raw slots into the workspace's scratch and the two segmented
 * sums run in one programmatic-dependent launch behind it (reference
 * solver._Scratch.jac / .hess = eval_* + sum_values, solver.py:282-295).
 * jac_c has jpat's nnz entries, hess_c hpat's; a NULL pattern writes that
 * output's raw slots instead.  Device pointers; asynchronous on `stream`. */
int exa_eval_set_compressed(ExaPlan* plan, ExaWorkspace* ws, const ExaPattern* jpat, const ExaPattern* hpat,
                            const double* x, const double* mult, double obj_weight, double* c, double* jac_c,
                            double* hess_c, exa_stream_t stream);
/* The same with HOST buffers: H2D x, mult; D2H c and the compressed values
 * only (the raw slots never cross PCIe).  Pinned buffers: asynchronous on
 * `stream`; pageable ones: complete on return. */
int exa_eval_set_compressed_host(ExaPlan* plan, ExaWorkspace* ws, const ExaPattern* jpat, const ExaPattern* hpat,
                                 const double* x_host, const double* mult_host, double obj_weight, double* c_host,
                                 double* jac_c_host, double* hess_c_host, exa_stream_t stream);
/* out[k] = 0 + sum_{e in [ptr[k], ptr[k+1])} raw[ent[e]], sequentially in e
 * order (np.bincount order); with ent sorted by raw slot within each k this is
 * CompressedPattern.sum_values.  All pointers are device pointers. */
int exa_segment_sum(int64_t nnz, const int64_t* ptr, const int32_t* ent, const double* raw,
                    double* out, exa_stream_t stream);

/* Solver-side consumer of the compressed callbacks: the
 * values of the reference IPM's KKT matrix (solver.py:421-456: H block
 * W + W^T - diag W, + sigma on the primal/slack diagonal, Jacobian and slack
 * coupling blocks, fixed rows/columns, + delta_w on free diagonals, - delta_c
 * on the dual diagonal) in a lower-triangle CSR whose pattern and per-entry
 * descriptors (int32 pairs, see kkt.py) are built once on the host.  All
 * pointers are device pointers; bit-identical to the reference's dense K. */
int exa_kkt_values(int64_t n, const int32_t* desc, const double* hvals, const double* jvals,
                   const double* sigma, double delta_w, double delta_c, double* out, exa_stream_t stream);

/* Synchronises `stream`; returns 1 and fills the location if the last
 * evaluation on `ws` hit a numeric-domain violation, 0 if not, < 0 on error.
 * rank = term rank in the callback's evaluation order, instr = tape index,
 * record = -1 when the failing operand was a constant. */
int exa_domain_error(ExaPlan* plan, ExaWorkspace* ws, exa_stream_t stream, int64_t* rank,
                     int32_t* instr, int64_t* record);

/* ---- diagnostics -------------------------------------------------------- */
const char* exa_last_error(void);
/* Timeline buffer for modules generated with EXA_TRACE=1 (8 int64 words per
 * warp and virtual CTA: SM id, virtual CTA, clock64 start/end, globaltimer
 * start/end, 2 unused);
 * NULL disables.  Process-global; not for production use. */
int exa_debug_trace(void* device_buffer);
int exa_device_sincos(const double* x, double* s, double* c, int64_t n, exa_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* EXA_H */
