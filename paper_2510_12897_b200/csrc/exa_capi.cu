// exa_capi.cu -- libexa.so: C ABI, plan management, NVRTC JIT, and the static
// aggregation kernels of the B200 callback engine.  See include/exa.h.
//
// Static kernels here (the generated per-model kernels live in the JIT module):
//   exa_obj_leaves / exa_obj_combine  objective sum in numpy's pairwise order
//                                      (reference eval_objective, autodiff.py:536-547)
//   exa_grad_reduce                    dense gradient, bincount order per variable
//                                      (reference eval_gradient, autodiff.py:550-563)
//   exa_compress_reduce                CompressedPattern.sum_values (autodiff.py:672-674)
//   exa_sincos_kernel                  device check of exa_sincos (diagnostics)
// All reductions are sequential per output element in the reference's order:
// deterministic, no floating-point atomics.

#include <cuda_runtime.h>
#include <nvrtc.h>

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <map>
#include <mutex>
#include <set>
#include <unordered_map>
#include <string>
#include <thread>
#include <vector>

#include "../../include/exa.h"
#include "exa_device.h"
#include "exa_math.h"

static_assert(sizeof(ExaSegDesc) == sizeof(ExaSeg), "segment layout");

namespace {

thread_local std::string g_err;
static long long* g_trace = nullptr;  // exa_debug_trace: timeline buffer for EXA_TRACE modules

int fail(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return -1;
}

#define CU(call)                                                                             \
  do {                                                                                       \
    cudaError_t e_ = (call);                                                                 \
    if (e_ != cudaSuccess) return fail("%s failed: %s", #call, cudaGetErrorString(e_));      \
  } while (0)

template <class T>
int dev_upload(T** dst, const T* src, size_t n) {
  *dst = nullptr;
  if (n == 0) return 0;
  CU(cudaMalloc((void**)dst, n * sizeof(T)));
  CU(cudaMemcpy(*dst, src, n * sizeof(T), cudaMemcpyHostToDevice));
  return 0;
}

const char* kKernelNames[EXA_NKERN] = {
    "exa_k_set_h",  "exa_k_set_l",  "exa_k_cons_h", "exa_k_cons_l", "exa_k_jac_h",  "exa_k_jac_l",
    "exa_k_hess_h", "exa_k_hess_l", "exa_k_objv_h", "exa_k_objv_l", "exa_k_grad_h", "exa_k_grad_l"};

// objective combine program opcodes (see paper_2510_12897_b200/device.py)
enum { OP_LEAF = 0, OP_ADD = 1, OP_CONST = 2, OP_ZERO_PLUS = 3, OP_TOTAL_ADD = 4 };

}  // namespace

struct ExaWorkspace {
  ExaPlan* plan = nullptr;
  double* V = nullptr;
  double* G = nullptr;
  double* leafsum = nullptr;
  unsigned long long* err = nullptr;
  cudaStream_t aux = nullptr;   // second stream: light kernel runs beside the heavy one
  cudaEvent_t fork = nullptr, join = nullptr;
  /* device staging for exa_eval_set_host (allocated on first use); dJ / dH
     are also the raw-slot scratch of exa_eval_set_compressed */
  double *dx = nullptr, *dy = nullptr, *dc = nullptr, *dJ = nullptr, *dH = nullptr;
  /* compressed J / H staging of exa_eval_set_compressed_host */
  double *dJc = nullptr, *dHc = nullptr;
  int64_t cap_Jc = 0, cap_Hc = 0;
  /* pinned host staging for pageable callers: x, mult | c, J ranges, H ranges */
  double* hstage = nullptr;
  std::vector<cudaEvent_t> chunk_ev;
  /* guards the lazy staging allocation (a workspace serves one evaluation at
     a time; concurrent callers use one workspace each) */
  std::mutex mu;
};

struct ExaObjNode;

/* one CTA's share of the host path's D2H: output slots [a, e) of output arr */
struct ExaD2HChunk {
  int64_t a, e;
  int32_t arr, pad;
};
constexpr int64_t kD2HChunk = 2048;  // doubles per CTA (16 KB)

struct ExaPlan {
  int device = 0;
  int64_t nvar = 0, ncon = 0, n_jac = 0, n_hess = 0;
  int threads[2] = {128, 256};
  double* f64 = nullptr;
  int32_t* i32 = nullptr;
  ExaTerm* terms = nullptr;
  int32_t n_terms = 0;
  ExaSeg* segs[EXA_NKERN] = {};
  int* cta_seg[EXA_NKERN] = {};
  int n_ctas[EXA_NKERN] = {};
  int persist[EXA_NKERN] = {};  /* virtual CTAs per real CTA (0 = classic grid) */
  int batchable = 0;            /* module offsets x/y/c/J/H by blockIdx.y (exa_eval_set_batch) */
  int grid[EXA_NKERN] = {};     /* real CTAs launched */
  int err_base[EXA_NMODES][2] = {};
  int64_t n_vscr = 0, n_gscr = 0;
  int64_t* leaves = nullptr;
  int32_t n_leaves = 0;
  int64_t obj_leaf_max = 0; /* longest pairwise leaf (numpy: <= 128) */
  int64_t* prog = nullptr;
  int32_t n_prog = 0;
  ExaObjNode* onodes = nullptr; /* the combine program as a level-ordered DAG */
  double* oinit = nullptr;
  int32_t* olvl = nullptr;
  int32_t n_onodes = 0, n_olvl = 0;
  int64_t* grad_ptr = nullptr;
  int64_t* grad_ent = nullptr;
  int has_checks = 0;
  cudaLibrary_t lib = nullptr;
  cudaKernel_t kern[EXA_NKERN] = {};
  cudaKernel_t kern_batch = nullptr; /* strided-batch set kernel (parameters kept in L2), if the module has one */
  /* compressed-set module (exa_plan_attach_compressed): set kernels that write
     the direct compressed Jacobian entries themselves and keep the other raw
     slots in L2 for the segmented sum */
  cudaLibrary_t lib_cmp = nullptr;
  cudaKernel_t kern_cmp[2] = {};
  int32_t* hpos = nullptr; /* group-local compressed H entry per (class, record), -1 = not local */
  ExaWorkspace* dflt = nullptr;
  size_t bytes = 0;
  int pdl = 0;
  /* host path: constant runs filled on the host, (first, length, value) */
  struct Run { int64_t a, n; double v; };
  std::vector<Run> fill_jac, fill_hess;
  /* ... and weighted-zero runs (exact zero-sign modules): slot a + i holds
     mult[rows[off + i]] * z (off < 0: obj_weight * z) */
  struct WRun { int64_t a, n, off; double z; };
  std::vector<WRun> fill_wz;
  std::vector<int32_t> wz_rows;
  /* ... and the complementary slot ranges copied D2H, (first, length) */
  std::vector<std::pair<int64_t, int64_t>> copy_jac, copy_hess;
  /* the same ranges (c whole, then J, then H) cut into CTA chunks for the
     device-to-host store kernel; chunks [d2h_c[k], d2h_c[k + 1]) belong to
     output k (0 = c, 1 = J, 2 = H) */
  struct ExaD2HChunk* d2h = nullptr;
  int d2h_c[4] = {};
  /* ... and as copy-engine operations: rows x [a, a + n) at pitch (slots) of
     output arr; consecutive ranges of equal length and stride are one 2D copy
     (a transfer costs the engine ~3.6 us on top of its bytes: 20 ranges of a
     case13659 set run at 42 GB/s one by one, at the full 56 GB/s as rows of
     one 2D copy -- tools/micro/d2hstore.cu) */
  struct Op { int arr, rows; int64_t a, n, pitch; };
  std::vector<Op> d2h_ops;
};

/* A compressed pattern (reference CompressedPattern, autodiff.py:660-674) on
 * the plan's device: compressed entry k sums raw slots ent[ptr[k] .. ptr[k+1])
 * in increasing slot order (np.bincount order). */
struct ExaPattern {
  int device = 0;
  int64_t n_raw = 0, nnz = 0;
  /* entries written directly by the compressed-set kernels (their single raw
     slot is flagged direct at creation): not folded here */
  bool direct = false;
  /* CTA chunks of the compressed sum.  Each entry's raw slots, in increasing
     slot order, minus the slots known to hold +0.0 on every call (dropping
     them from a fold that starts at +0.0 is exact), form its *stage*; chunk b
     covers entries [chk[b], chk[b+1]) whose stages fit one CTA's shared
     memory (cap = 256 * ipt slots, at most cap entries) -- or a single
     longer entry.  Per chunk: gathered
     slots [che[b], che[b+1]) of src (raw slot id) / dst (stage position),
     sorted by src so that a warp's gathers hit runs of consecutive raw slots;
     known constant slots [chc[b], chc[b+1]) of cpos (stage position) / cid
     (index into cval).  Per chunk entry slot, entries by decreasing stage
     length (the threads of a warp fold stages of similar length): edesc =
     stage start | length << 16, eout = the compressed entry.  A long entry
     keeps every non-skipped slot in src, in slot order. */
  int32_t nch = 0, ipt = 8;
  int32_t* chk = nullptr;
  int32_t* che = nullptr;
  int32_t* chc = nullptr;
  int32_t* src = nullptr;
  uint16_t* dst = nullptr;
  uint16_t* cpos = nullptr;
  uint16_t* cid = nullptr;
  uint32_t* edesc = nullptr; /* per entry slot of a chunk, longest stage first: start | len << 16 */
  int32_t* eout = nullptr;   /* ... and the compressed entry it folds */
  double* cval = nullptr;
};

// ---------------------------------------------------------------------------
// static kernels
// ---------------------------------------------------------------------------

// One leaf of numpy's pairwise summation (numpy/_core/src/umath/loops_utils.h.src
// pairwise_sum): n < 8 -> plain loop; 8 <= n <= 128 -> 8 strided accumulators,
// combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the tail.
__global__ void exa_obj_leaves(const double* __restrict__ V, const int64_t* __restrict__ leaves,
                               int n_leaves, double* __restrict__ out) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= n_leaves) return;
  const double* a = V + leaves[2 * l];
  const int64_t n = leaves[2 * l + 1];
  double res;
  if (n < 8) {
    res = 0.0;
    for (int64_t i = 0; i < n; ++i) res = res + a[i];
  } else {
    double r0 = a[0], r1 = a[1], r2 = a[2], r3 = a[3], r4 = a[4], r5 = a[5], r6 = a[6], r7 = a[7];
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8) {
      r0 = r0 + a[i + 0];
      r1 = r1 + a[i + 1];
      r2 = r2 + a[i + 2];
      r3 = r3 + a[i + 3];
      r4 = r4 + a[i + 4];
      r5 = r5 + a[i + 5];
      r6 = r6 + a[i + 6];
      r7 = r7 + a[i + 7];
    }
    res = ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7));
    for (; i < n; ++i) res = res + a[i];
  }
  out[l] = res;
}

// The pairwise tree above the leaves plus the Python-level `total += s_t`
// accumulation over objective blocks, replayed by one thread.  The program's
// stack depth is validated on the host at plan creation (prog_depth).
#define EXA_OBJ_STACK 96
__global__ void exa_obj_combine(const int64_t* __restrict__ prog, int n_prog,
                                const double* __restrict__ leafsum, double* __restrict__ out) {
  double stack[EXA_OBJ_STACK];
  int sp = 0;
  double total = 0.0;
  for (int p = 0; p < n_prog; ++p) {
    const int64_t op = prog[3 * p], a = prog[3 * p + 1];
    switch ((int)op) {
      case OP_LEAF: stack[sp++] = leafsum[a]; break;
      case OP_ADD: {
        const double b = stack[--sp];
        const double x = stack[--sp];
        stack[sp++] = x + b;
        break;
      }
      case OP_CONST: stack[sp++] = __longlong_as_double((long long)a); break;
      case OP_ZERO_PLUS: stack[sp - 1] = 0.0 + stack[sp - 1]; break;
      case OP_TOTAL_ADD: total = total + stack[--sp]; break;
      default: break;
    }
  }
  *out = total;
}

// The same objective sum as exa_obj_leaves + exa_obj_combine, as two
// programmatic-dependent launches behind the objective-value kernel:
//  * exa_obj_leaves2: one warp per pairwise leaf (lanes load the leaf's
//    <= 128 values at once, lane 0 replays numpy's accumulator order);
//  * exa_obj_dag: one CTA evaluates the combine program as a DAG ordered by
//    level (level 0: the leaves in leaf order, then the constants; a node of
//    level L > 0 adds two lower nodes, or is 0 + a node), one __syncthreads
//    per level.  Every add is the program's own operation on the same
//    operands, so the value is bit-identical.  Its node table is staged in
//    shared memory before griddepcontrol.wait.
#define EXA_OBJ_THREADS 512
#define EXA_OBJ_LEAF_MAX 128
#define EXA_OBJ_LEAF_WARPS 4
__global__ void __launch_bounds__(32 * EXA_OBJ_LEAF_WARPS) exa_obj_leaves2(const double* V,
                                                                         const int64_t* __restrict__ leaves,
                                                                         int n_leaves, double* __restrict__ out) {
  __shared__ double wbuf[EXA_OBJ_LEAF_WARPS][EXA_OBJ_LEAF_MAX];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int l = blockIdx.x * EXA_OBJ_LEAF_WARPS + warp;
  int64_t st = 0;
  int n = 0;
  if (l < n_leaves) {
    st = __ldg(leaves + 2 * l);
    n = (int)__ldg(leaves + 2 * l + 1);
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (l >= n_leaves) return;
  double* wb = wbuf[warp];
  double v[EXA_OBJ_LEAF_MAX / 32];
#pragma unroll
  for (int j = 0; j < EXA_OBJ_LEAF_MAX / 32; ++j) v[j] = lane + 32 * j < n ? V[st + lane + 32 * j] : 0.0;
#pragma unroll
  for (int j = 0; j < EXA_OBJ_LEAF_MAX / 32; ++j) wb[lane + 32 * j] = v[j];
  __syncwarp();
  if (lane != 0) return;
  double res;
  if (n < 8) {
    res = 0.0;
    for (int i = 0; i < n; ++i) res = res + wb[i];
  } else {
    double r0 = wb[0], r1 = wb[1], r2 = wb[2], r3 = wb[3], r4 = wb[4], r5 = wb[5], r6 = wb[6], r7 = wb[7];
    int i = 8;
    for (; i < n - (n % 8); i += 8) {
      r0 = r0 + wb[i + 0];
      r1 = r1 + wb[i + 1];
      r2 = r2 + wb[i + 2];
      r3 = r3 + wb[i + 3];
      r4 = r4 + wb[i + 4];
      r5 = r5 + wb[i + 5];
      r6 = r6 + wb[i + 6];
      r7 = r7 + wb[i + 7];
    }
    res = ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7));
    for (; i < n; ++i) res = res + wb[i];
  }
  out[l] = res;
}
struct ExaObjNode {
  int32_t op, a, b, pad; /* op: 0 leaf / constant (value preset), 1 add, 2 zero-plus */
};
__global__ void __launch_bounds__(EXA_OBJ_THREADS) exa_obj_dag(const double* leafsum, int n_leaves,
                                                             const ExaObjNode* __restrict__ nodes, int n_nodes,
                                                             const double* __restrict__ init,
                                                             const int32_t* __restrict__ lvl, int n_lvl,
                                                             double* __restrict__ out) {
  extern __shared__ double osm[];
  double* nv = osm;                                                       // [n_nodes]
  ExaObjNode* sn = reinterpret_cast<ExaObjNode*>(nv + ((n_nodes + 1) & ~1));  // [n_nodes]
  int32_t* sl = reinterpret_cast<int32_t*>(sn + n_nodes);                 // [n_lvl + 1]
  const int tid = threadIdx.x;
  for (int i0 = n_leaves; i0 < n_nodes; i0 += 4 * EXA_OBJ_THREADS) {  // 4 loads per thread in flight
    ExaObjNode t[4];
    double c[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int i = i0 + tid + EXA_OBJ_THREADS * j;
      if (i < n_nodes) {
        t[j] = nodes[i];
        c[j] = __ldg(init + i);
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int i = i0 + tid + EXA_OBJ_THREADS * j;
      if (i < n_nodes) {
        sn[i] = t[j];
        nv[i] = c[j];
      }
    }
  }
  for (int i = tid; i <= n_lvl; i += EXA_OBJ_THREADS) sl[i] = __ldg(lvl + i);
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  for (int i0 = 0; i0 < n_leaves; i0 += 4 * EXA_OBJ_THREADS) {
    double c[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int i = i0 + tid + EXA_OBJ_THREADS * j;
      c[j] = i < n_leaves ? leafsum[i] : 0.0;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int i = i0 + tid + EXA_OBJ_THREADS * j;
      if (i < n_leaves) nv[i] = c[j];
    }
  }
  __syncthreads();
  for (int L = 1; L < n_lvl; ++L) {
    const int i1 = sl[L + 1];
    for (int i = sl[L] + tid; i < i1; i += EXA_OBJ_THREADS) {
      const ExaObjNode nd = sn[i];
      nv[i] = nd.op == 1 ? nv[nd.a] + nv[nd.b] : 0.0 + nv[nd.a];
    }
    __syncthreads();
  }
  if (tid == 0) *out = n_nodes ? nv[n_nodes - 1] : 0.0;
}
#define EXA_OBJ_FUSED_SMEM_MAX (160 * 1024)
static size_t obj_dag_smem(int n_nodes, int n_lvl) {
  return sizeof(double) * (size_t)((n_nodes + 1) & ~1) + sizeof(ExaObjNode) * (size_t)n_nodes +
         sizeof(int32_t) * (size_t)(n_lvl + 1);
}

// The combine program as a level-ordered DAG (see exa_obj_fused).  Returns
// false if the program is malformed.  Node n_nodes - 1 is the total.
static bool obj_dag(const int64_t* prog, int n_prog, int n_leaves, std::vector<ExaObjNode>& nodes,
                    std::vector<double>& init, std::vector<int32_t>& lvl) {
  struct N { int op; int64_t a, b; int level; double c; };
  std::vector<N> g;
  std::vector<int64_t> st;
  for (int l = 0; l < n_leaves; ++l) g.push_back({0, l, 0, 0, 0.0});
  auto cnst = [&](double c) { g.push_back({3, 0, 0, 0, c}); return (int64_t)g.size() - 1; };
  int64_t total = cnst(0.0);
  for (int q = 0; q < n_prog; ++q) {
    const int64_t op = prog[3 * q], a = prog[3 * q + 1];
    switch ((int)op) {
      case OP_LEAF: if (a < 0 || a >= n_leaves) return false; st.push_back(a); break;
      case OP_CONST: { double c; std::memcpy(&c, &a, 8); st.push_back(cnst(c)); break; }
      case OP_ADD: {
        if (st.size() < 2) return false;
        const int64_t y = st.back(); st.pop_back();
        const int64_t x = st.back(); st.pop_back();
        g.push_back({1, x, y, 1 + std::max(g[x].level, g[y].level), 0.0});
        st.push_back((int64_t)g.size() - 1);
        break;
      }
      case OP_ZERO_PLUS: {
        if (st.empty()) return false;
        const int64_t x = st.back();
        g.push_back({2, x, 0, 1 + g[x].level, 0.0});
        st.back() = (int64_t)g.size() - 1;
        break;
      }
      case OP_TOTAL_ADD: {
        if (st.empty()) return false;
        const int64_t y = st.back(); st.pop_back();
        g.push_back({1, total, y, 1 + std::max(g[total].level, g[y].level), 0.0});
        total = (int64_t)g.size() - 1;
        break;
      }
      default: return false;
    }
  }
  if (g.size() >= (size_t)INT32_MAX) return false;
  /* order: leaves (leaf order), constants, then by level; the total last */
  const int64_t n = (int64_t)g.size();
  std::vector<int64_t> order;
  for (int64_t i = 0; i < n_leaves; ++i) order.push_back(i);
  for (int64_t i = n_leaves; i < n; ++i)
    if (g[i].op == 3) order.push_back(i);
  std::vector<int64_t> rest;
  for (int64_t i = n_leaves; i < n; ++i)
    if (g[i].op != 3 && i != total) rest.push_back(i);
  std::stable_sort(rest.begin(), rest.end(), [&](int64_t x, int64_t y) { return g[x].level < g[y].level; });
  order.insert(order.end(), rest.begin(), rest.end());
  if (total >= n_leaves && g[total].op != 3) order.push_back(total);
  else if (total != order.back()) {  /* no objective block: the total is the constant 0 */
    g.push_back({2, total, 0, 1 + g[total].level, 0.0});
    order.push_back((int64_t)g.size() - 1);
  }
  std::vector<int64_t> pos(g.size());
  for (size_t i = 0; i < order.size(); ++i) pos[order[i]] = (int64_t)i;
  nodes.assign(order.size(), ExaObjNode{0, 0, 0, 0});
  init.assign(order.size(), 0.0);
  lvl.assign(1, 0);
  int cur = 0;
  for (size_t i = 0; i < order.size(); ++i) {
    const N& x = g[order[i]];
    if (x.op == 3) init[i] = x.c;
    if (x.op == 1 || x.op == 2) nodes[i] = ExaObjNode{x.op, (int32_t)pos[x.a], (int32_t)pos[x.op == 1 ? x.b : 0], 0};
    /* level boundaries: level 0 = leaves + constants; the total may sit alone
       at the end (its level can be below the last non-total node's) */
    const int L = (x.op == 0 || x.op == 3) ? 0 : std::max(cur, x.level);
    while (cur < L) { lvl.push_back((int32_t)i); ++cur; }
  }
  lvl.push_back((int32_t)order.size());
  return true;
}

// Stack depth of an objective combine program, or -1 if it is malformed
// (unknown opcode, pop from an empty stack, leaf index out of range).
static int prog_depth(const int64_t* prog, int n_prog, int n_leaves) {
  int sp = 0, mx = 0;
  for (int p = 0; p < n_prog; ++p) {
    const int64_t op = prog[3 * p], a = prog[3 * p + 1];
    switch ((int)op) {
      case OP_LEAF:
        if (a < 0 || a >= n_leaves) return -1;
        ++sp;
        break;
      case OP_CONST: ++sp; break;
      case OP_ADD: if (sp < 2) return -1; --sp; break;
      case OP_ZERO_PLUS: if (sp < 1) return -1; break;
      case OP_TOTAL_ADD: if (sp < 1) return -1; --sp; break;
      default: return -1;
    }
    if (sp > mx) mx = sp;
  }
  return mx;
}

// g[v] = ((0 + B_1) + B_2) + ..., B_k = sequential bincount sum of group k.
__global__ void exa_grad_reduce(int64_t nvar, const int64_t* __restrict__ ptr, const int64_t* __restrict__ ent,
                                const double* __restrict__ G, double* __restrict__ g) {
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nvar) return;
  double acc = 0.0, grp = 0.0;
  bool open = false;
  const int64_t e1 = ptr[v + 1];
  for (int64_t e = ptr[v]; e < e1; ++e) {
    const int64_t en = ent[e];
    if (en >> 62) {
      if (open) acc = acc + grp;
      grp = 0.0;
      open = true;
    }
    grp = grp + G[en & ((1LL << 62) - 1)];
  }
  if (open) acc = acc + grp;
  g[v] = acc;
}

// compressed[k] = 0 + sum of raw slots mapped to k, in slot order (np.bincount).
// The raw loads of an entry are issued together (8 at a time) before the
// in-order adds, so a long segment costs a few load latencies, not one each.
__global__ void exa_compress_reduce(int64_t nnz, const int64_t* __restrict__ ptr, const int32_t* __restrict__ ent,
                                    const double* __restrict__ raw, double* __restrict__ out) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nnz) return;
  double acc = 0.0;
  const int64_t e1 = ptr[k + 1];
  int64_t e = ptr[k];
  for (; e + 8 <= e1; e += 8) {
    double v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = __ldg(raw + __ldg(ent + e + j));
#pragma unroll
    for (int j = 0; j < 8; ++j) acc = acc + v[j];
  }
  for (; e < e1; ++e) acc = acc + __ldg(raw + __ldg(ent + e));
  out[k] = acc;
}

// Compressed J and H of one callback set in one launch, one CTA per chunk of
// compressed entries (chunks [0, nchJ) are J's, the rest H's).  Launched as a
// programmatic dependent of the set kernel: before griddepcontrol.wait a CTA
// loads its chunk's slot map and writes the known constant slots into its
// shared-memory stage (plan data only); then it gathers the set's raw slots
// in ADDRESS order into the stage (ENTRY order), and each thread folds its
// entries' stages in increasing slot order (np.bincount's order: compressed[k]
// = ((0 + r_1) + r_2) + ...) and writes them coalesced.  A chunk holding one
// entry longer than the stage is folded by one thread from global memory.
#define EXA_CMP_THREADS 256
// gathers per thread (stage = 256 * IPT slots); EXA_CMP_IPT picks it when a
// pattern is created (chunks are sized for it)
static int cmp_ipt_env() {
  const char* e = getenv("EXA_CMP_IPT");
  const int v = e ? atoi(e) : 4;  // case13659 set + compress: 4 -> 18.2 us, 8 -> 21.8, 16 -> 24.1
  return (v == 1 || v == 2 || v == 4 || v == 8 || v == 12 || v == 16) ? v : 4;
}
struct ExaCmpArgs {
  const int32_t *chk, *che, *chc, *src;
  const uint16_t *dst, *cpos, *cid;
  const uint32_t* edesc;
  const int32_t* eout;
  const double* cval;
  const double* raw;
  double* out;
};
template <int IPT>
__device__ __forceinline__ void exa_cmp_chunk(const ExaCmpArgs& P, int b, bool first, double* vals, uint32_t* sdesc,
                                              int32_t* sord) {
  constexpr int EXA_CMP_IPT = IPT;
  constexpr int EXA_CMP_CAP = EXA_CMP_THREADS * IPT;
  const int tid = threadIdx.x;
  const int k0 = __ldg(P.chk + b), k1 = __ldg(P.chk + b + 1);
  const int g0 = __ldg(P.che + b), g1 = __ldg(P.che + b + 1);
  const int c0 = __ldg(P.chc + b), c1 = __ldg(P.chc + b + 1);
  const int ng = g1 - g0, nc = c1 - c0, nk = k1 - k0;
  if (ng + nc > EXA_CMP_CAP) {  // one long entry: its slots in increasing order
    if (first) {
      asm volatile("griddepcontrol.wait;" ::: "memory");
      asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    }
    if (tid == 0) {
      double acc = 0.0;
      for (int e = g0; e < g1; ++e) acc = acc + P.raw[__ldg(P.src + e)];
      P.out[__ldg(P.eout + k0)] = acc;
    }
    return;
  }
  // nc, nk <= EXA_CMP_CAP: fixed trip counts, so every load of a loop is
  // issued before its first shared-memory store (one DRAM latency, not IPT)
  {
    int cp[EXA_CMP_IPT], ci[EXA_CMP_IPT];
#pragma unroll
    for (int j = 0; j < EXA_CMP_IPT; ++j) {
      const int i = tid + EXA_CMP_THREADS * j;
      cp[j] = i < nc ? (int)__ldg(P.cpos + c0 + i) : -1;
      ci[j] = i < nc ? (int)__ldg(P.cid + c0 + i) : 0;
    }
    uint32_t dd[EXA_CMP_IPT];
    int32_t oo[EXA_CMP_IPT];
#pragma unroll
    for (int j = 0; j < EXA_CMP_IPT; ++j) {
      const int i = tid + EXA_CMP_THREADS * j;
      dd[j] = i < nk ? __ldg(P.edesc + k0 + i) : 0u;
      oo[j] = i < nk ? __ldg(P.eout + k0 + i) : 0;
    }
#pragma unroll
    for (int j = 0; j < EXA_CMP_IPT; ++j)
      if (cp[j] >= 0) vals[cp[j]] = __ldg(P.cval + ci[j]);
#pragma unroll
    for (int j = 0; j < EXA_CMP_IPT; ++j) {
      const int i = tid + EXA_CMP_THREADS * j;
      if (i < nk) {
        sdesc[i] = dd[j];
        sord[i] = oo[j];
      }
    }
  }
  int idx[EXA_CMP_IPT], pos[EXA_CMP_IPT];
#pragma unroll
  for (int j = 0; j < EXA_CMP_IPT; ++j) {
    const int e = tid + EXA_CMP_THREADS * j;
    idx[j] = e < ng ? __ldg(P.src + g0 + e) : -1;
    pos[j] = e < ng ? (int)__ldg(P.dst + g0 + e) : 0;
  }
  if (first) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  }
  double v[EXA_CMP_IPT];
#pragma unroll
  for (int j = 0; j < EXA_CMP_IPT; ++j) v[j] = idx[j] >= 0 ? P.raw[idx[j]] : 0.0;  // plain loads: the set wrote them
#pragma unroll
  for (int j = 0; j < EXA_CMP_IPT; ++j)
    if (idx[j] >= 0) vals[pos[j]] = v[j];
  __syncthreads();
  for (int i = tid; i < nk; i += EXA_CMP_THREADS) {
    const uint32_t d = sdesc[i];
    int e = (int)(d & 0xffffu);
    const int z = e + (int)(d >> 16);
    double acc = 0.0;
    for (; e + 4 <= z; e += 4) {  // four stage loads in flight, adds in slot order
      const double a0 = vals[e], a1 = vals[e + 1], a2 = vals[e + 2], a3 = vals[e + 3];
      acc = acc + a0;
      acc = acc + a1;
      acc = acc + a2;
      acc = acc + a3;
    }
    for (; e < z; ++e) acc = acc + vals[e];
    P.out[sord[i]] = acc;
  }
}

// One CTA per chunk (launched with nch CTAs; the loop also serves smaller
// grids).  Measured: a no-op launch of this kernel behind every case13659 set
// already adds 4.2 us (1,831 CTAs; 2.8 us with 458), but a persistent grid
// sized to the resident capacity, folding its chunks one after another, is
// slower (22.1 vs 18.0 us per set + compression).
template <int IPT, int MINB>
__global__ void __launch_bounds__(EXA_CMP_THREADS, MINB) exa_compress2_kernel(int nchJ, int nch, ExaCmpArgs J,
                                                                             ExaCmpArgs H, int probe) {
  constexpr int EXA_CMP_CAP = EXA_CMP_THREADS * IPT;
  extern __shared__ double vals[];                                     // [EXA_CMP_CAP] stage
  uint32_t* sdesc = reinterpret_cast<uint32_t*>(vals + EXA_CMP_CAP);  // [EXA_CMP_CAP]
  int32_t* sord = reinterpret_cast<int32_t*>(sdesc + EXA_CMP_CAP);    // [EXA_CMP_CAP]
  if (probe == 1) {  // timing probe (EXA_CMP_PROBE=1): the launch and its dependency only
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    return;
  }
  bool first = true;
  for (int b = blockIdx.x; b < nch; b += gridDim.x) {
    if (!first) __syncthreads();  // the previous chunk's stage is free
    const bool isJ = b < nchJ;
    exa_cmp_chunk<IPT>(isJ ? J : H, isJ ? b : b - nchJ, first, vals, sdesc, sord);
    first = false;
  }
}

// KKT assembly (reference solver.py:421-456): one thread per lower-triangle
// CSR entry; desc = (kind << 29 | a, b).  Kinds and their exact arithmetic:
//   0 H off-diagonal        (h + 0) - 0              (W + W^T - diag W)
//   1 diagonal with H       (((h + h) - h) + sigma[b]) + delta_w
//   2 diagonal without H    (0 + sigma[b]) + delta_w
//   3 Jacobian              j
//   4 slack coupling        -1
//   5 dual diagonal         delta_c != 0 ? 0 - delta_c : 0
//   6 fixed row/col         0
//   7 fixed diagonal        1
__device__ __forceinline__ double exa_kkt_entry(int2 d, const double* __restrict__ h, const double* __restrict__ j,
                                                const double* __restrict__ sigma, double dw, double dc) {
  const int kind = (int)((unsigned)d.x >> 29);
  const int a = d.x & ((1 << 29) - 1);
  switch (kind) {
    case 0: { const double hv = __ldg(h + a); return (hv + 0.0) - 0.0; }
    case 1: { const double hv = __ldg(h + a); return (((hv + hv) - hv) + __ldg(sigma + d.y)) + dw; }
    case 2: return (0.0 + __ldg(sigma + d.y)) + dw;
    case 3: return __ldg(j + a);
    case 4: return -1.0;
    case 5: return dc != 0.0 ? 0.0 - dc : 0.0;
    case 6: return 0.0;
    default: return 1.0;
  }
}

// 4 entries per thread, strided by the grid so loads stay coalesced: all four
// descriptors are loaded before any value gather (memory-level parallelism).
__global__ void __launch_bounds__(256) exa_kkt_kernel(int64_t n, const int2* __restrict__ desc,
                                                      const double* __restrict__ h, const double* __restrict__ j,
                                                      const double* __restrict__ sigma, double dw, double dc,
                                                      double* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t p0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int2 d[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int64_t p = p0 + u * stride;
    d[u] = p < n ? __ldg(desc + p) : make_int2(6 << 29, 0);
  }
  double v[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) v[u] = exa_kkt_entry(d[u], h, j, sigma, dw, dc);
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int64_t p = p0 + u * stride;
    if (p < n) out[p] = v[u];
  }
}

__global__ void exa_sincos_kernel(const double* __restrict__ x, double* __restrict__ s, double* __restrict__ c,
                                  int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double sv, cv;
  exa_sincos(x[i], &sv, &cv);
  s[i] = sv;
  c[i] = cv;
}

static inline unsigned grid_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" {

const char* exa_last_error(void) { return g_err.c_str(); }

int exa_debug_trace(void* device_buffer) {
  g_trace = reinterpret_cast<long long*>(device_buffer);
  return 0;
}

void exa_free(void* p) { free(p); }

int exa_nvrtc_version(int* major, int* minor) {
  if (nvrtcVersion(major, minor) != NVRTC_SUCCESS) return fail("nvrtcVersion failed");
  return 0;
}

int exa_jit_compile(const char* src, const char* name, const char* const* opts, int n_opts, void** cubin,
                    size_t* cubin_size, char** log) {
  if (!src || !cubin || !cubin_size) return fail("exa_jit_compile: null argument");
  *cubin = nullptr;
  *cubin_size = 0;
  if (log) *log = nullptr;
  nvrtcProgram prog;
  nvrtcResult r = nvrtcCreateProgram(&prog, src, name ? name : "exa_gen.cu", 0, nullptr, nullptr);
  if (r != NVRTC_SUCCESS) return fail("nvrtcCreateProgram: %s", nvrtcGetErrorString(r));
  r = nvrtcCompileProgram(prog, n_opts, opts);
  size_t log_size = 0;
  nvrtcGetProgramLogSize(prog, &log_size);
  std::string lg(log_size, '\0');
  if (log_size) nvrtcGetProgramLog(prog, &lg[0]);
  if (log && log_size > 1) {
    *log = (char*)malloc(log_size);
    memcpy(*log, lg.data(), log_size);
  }
  if (r != NVRTC_SUCCESS) {
    nvrtcDestroyProgram(&prog);
    return fail("NVRTC compile failed: %s\n%.4000s", nvrtcGetErrorString(r), lg.c_str());
  }
  size_t n = 0;
  if (nvrtcGetCUBINSize(prog, &n) != NVRTC_SUCCESS || n == 0) {
    nvrtcDestroyProgram(&prog);
    return fail("nvrtcGetCUBINSize failed (was -arch=sm_100a given?)");
  }
  void* buf = malloc(n);
  nvrtcGetCUBIN(prog, (char*)buf);
  nvrtcDestroyProgram(&prog);
  *cubin = buf;
  *cubin_size = n;
  return 0;
}

static int ws_alloc(ExaPlan* p, ExaWorkspace** out) {
  ExaWorkspace* w = new ExaWorkspace();
  w->plan = p;
  if (p->n_vscr) CU(cudaMalloc((void**)&w->V, p->n_vscr * sizeof(double)));
  if (p->n_gscr) CU(cudaMalloc((void**)&w->G, p->n_gscr * sizeof(double)));
  if (p->n_leaves) CU(cudaMalloc((void**)&w->leafsum, p->n_leaves * sizeof(double)));
  CU(cudaMalloc((void**)&w->err, sizeof(unsigned long long)));
  CU(cudaMemset(w->err, 0xff, sizeof(unsigned long long)));
  CU(cudaStreamCreateWithFlags(&w->aux, cudaStreamNonBlocking));
  CU(cudaEventCreateWithFlags(&w->fork, cudaEventDisableTiming));
  CU(cudaEventCreateWithFlags(&w->join, cudaEventDisableTiming));
  *out = w;
  return 0;
}

void exa_workspace_destroy(ExaWorkspace* w) {
  if (!w) return;
  cudaFree(w->V);
  cudaFree(w->G);
  cudaFree(w->leafsum);
  cudaFree(w->err);
  cudaFree(w->dx);
  cudaFree(w->dy);
  cudaFree(w->dc);
  cudaFree(w->dJ);
  cudaFree(w->dH);
  cudaFree(w->dJc);
  cudaFree(w->dHc);
  if (w->hstage) cudaFreeHost(w->hstage);
  for (cudaEvent_t e : w->chunk_ev) cudaEventDestroy(e);
  if (w->fork) cudaEventDestroy(w->fork);
  if (w->join) cudaEventDestroy(w->join);
  if (w->aux) cudaStreamDestroy(w->aux);
  delete w;
}

int exa_workspace_create(ExaPlan* p, ExaWorkspace** out) {
  if (!p || !out) return fail("exa_workspace_create: null argument");
  CU(cudaSetDevice(p->device));
  return ws_alloc(p, out);
}

void exa_plan_destroy(ExaPlan* p) {
  if (!p) return;
  cudaSetDevice(p->device);
  exa_workspace_destroy(p->dflt);
  cudaFree(p->f64);
  cudaFree(p->i32);
  cudaFree(p->terms);
  for (int m = 0; m < EXA_NKERN; ++m) {
    cudaFree(p->segs[m]);
    cudaFree(p->cta_seg[m]);
  }
  cudaFree(p->leaves);
  cudaFree(p->prog);
  cudaFree(p->onodes);
  cudaFree(p->oinit);
  cudaFree(p->olvl);
  cudaFree(p->grad_ptr);
  cudaFree(p->grad_ent);
  cudaFree(p->d2h);
  if (p->lib_cmp) cudaLibraryUnload(p->lib_cmp);
  cudaFree(p->hpos);
  if (p->lib) cudaLibraryUnload(p->lib);
  delete p;
}

int exa_plan_create(const ExaPlanDesc* d, ExaPlan** out) {
  if (!d || !out) return fail("exa_plan_create: null argument");
  *out = nullptr;
  if (d->abi_version != EXA_ABI_VERSION) return fail("ABI version %d != %d", d->abi_version, EXA_ABI_VERSION);
  if (!d->cubin || d->cubin_size <= 0) return fail("exa_plan_create: no kernel module");
  CU(cudaSetDevice(d->device));
  ExaPlan* p = new ExaPlan();
  int rc = 0;
  auto bail = [&](int code) {
    exa_plan_destroy(p);
    return code;
  };
  p->device = d->device;
  p->nvar = d->nvar;
  p->ncon = d->ncon;
  p->n_jac = d->n_jac;
  p->n_hess = d->n_hess;
  {
    // programmatic dependent launch only for modules built with the waits;
    // EXA_PDL=0 in the environment turns it off for experiments
    const char* e = getenv("EXA_PDL");
    p->pdl = (d->pdl && !(e && e[0] == '0')) ? 1 : 0;
  }
  p->batchable = d->batchable && !d->has_domain_checks;
  {
    // host-filled runs; the complement of each output's runs is copied D2H
    auto take = [&](const int64_t* tr, int n, int64_t total, std::vector<ExaPlan::Run>& fill,
                    std::vector<std::pair<int64_t, int64_t>>* spans) -> int {
      for (int i = 0; i < n; ++i) {
        const int64_t a = tr[3 * i], len = tr[3 * i + 1];
        double v;
        std::memcpy(&v, &tr[3 * i + 2], sizeof v);
        if (len <= 0 || a < 0 || a + len > total) return fail("host_fill: run out of range");
        fill.push_back({a, len, v});
        spans->push_back({a, len});
      }
      return 0;
    };
    auto complement = [&](std::vector<std::pair<int64_t, int64_t>>& spans, int64_t total,
                          std::vector<std::pair<int64_t, int64_t>>& copy) -> int {
      std::sort(spans.begin(), spans.end());
      int64_t at = 0;
      for (auto& sp : spans) {
        if (sp.first < at) return fail("host_fill: runs must be disjoint");
        if (sp.first > at) copy.push_back({at, sp.first - at});
        at = sp.first + sp.second;
      }
      if (at < total) copy.push_back({at, total - at});
      return 0;
    };
    const int nj = d->host_fill ? d->n_fill_jac : 0, nh = d->host_fill ? d->n_fill_hess : 0;
    std::vector<std::pair<int64_t, int64_t>> sj, sh;
    if ((rc = take(d->host_fill, nj, d->n_jac, p->fill_jac, &sj))) return bail(rc);
    if ((rc = take(d->host_fill ? d->host_fill + 3 * nj : nullptr, nh, d->n_hess, p->fill_hess, &sh)))
      return bail(rc);
    const int nw = d->host_wzero ? d->n_wzero : 0;
    for (int i = 0; i < nw; ++i) {
      const int64_t* q = d->host_wzero + 4 * i;
      double z;
      std::memcpy(&z, &q[3], sizeof z);
      if (q[1] <= 0 || q[0] < 0 || q[0] + q[1] > d->n_hess || (q[2] >= 0 && q[2] + q[1] > d->n_wzero_rows))
        return bail(fail("host_wzero: run out of range"));
      p->fill_wz.push_back({q[0], q[1], q[2], z});
      sh.push_back({q[0], q[1]});
    }
    if (d->n_wzero_rows > 0) {
      p->wz_rows.assign(d->host_wzero_rows, d->host_wzero_rows + d->n_wzero_rows);
      for (int32_t r : p->wz_rows)
        if (r < 0 || r >= d->ncon) return bail(fail("host_wzero_rows: row out of range"));
    }
    if ((rc = complement(sj, d->n_jac, p->copy_jac))) return bail(rc);
    if ((rc = complement(sh, d->n_hess, p->copy_hess))) return bail(rc);
    // constant runs shorter than EXA_D2H_GAP slots between two copied ranges
    // are copied with them instead of filled on the host (one transfer fewer)
    const char* ge = std::getenv("EXA_D2H_GAP");
    const int64_t gap = ge ? std::atoll(ge) : 0;
    auto merge = [&](std::vector<std::pair<int64_t, int64_t>>& cp) {
      std::vector<std::pair<int64_t, int64_t>> out;
      for (auto& r : cp) {
        if (!out.empty() && r.first - (out.back().first + out.back().second) <= gap)
          out.back().second = r.first + r.second - out.back().first;
        else
          out.push_back(r);
      }
      cp.swap(out);
    };
    auto inside = [](const std::vector<std::pair<int64_t, int64_t>>& cp, int64_t a) {
      auto it = std::upper_bound(cp.begin(), cp.end(), std::make_pair(a, INT64_MAX));
      return it != cp.begin() && a < std::prev(it)->first + std::prev(it)->second;
    };
    if (gap > 0) {
      merge(p->copy_jac);
      merge(p->copy_hess);
      auto drop = [&](auto& runs, const std::vector<std::pair<int64_t, int64_t>>& cp) {
        runs.erase(std::remove_if(runs.begin(), runs.end(), [&](const auto& r) { return inside(cp, r.a); }), runs.end());
      };
      drop(p->fill_jac, p->copy_jac);
      drop(p->fill_hess, p->copy_hess);
      drop(p->fill_wz, p->copy_hess);
    }
    {
      auto ops = [&](int arr, const std::vector<std::pair<int64_t, int64_t>>& cp) {
        for (size_t i = 0; i < cp.size();) {
          size_t j = i + 1;
          const int64_t pitch = j < cp.size() ? cp[j].first - cp[i].first : 0;
          while (j < cp.size() && cp[j].second == cp[i].second && cp[j].first - cp[j - 1].first == pitch) ++j;
          p->d2h_ops.push_back({arr, (int)(j - i), cp[i].first, cp[i].second, j - i > 1 ? pitch : cp[i].second});
          i = j;
        }
      };
      std::vector<std::pair<int64_t, int64_t>> call;
      if (d->ncon) call.push_back({0, d->ncon});
      ops(0, call);
      ops(1, p->copy_jac);
      ops(2, p->copy_hess);
    }
    std::vector<ExaD2HChunk> ch;
    auto cut = [&](int arr, const std::vector<std::pair<int64_t, int64_t>>& rs) {
      p->d2h_c[arr] = (int)ch.size();
      for (auto& r : rs)
        for (int64_t o = 0; o < r.second; o += kD2HChunk)
          ch.push_back({r.first + o, r.first + std::min(r.second, o + kD2HChunk), arr, 0});
    };
    std::vector<std::pair<int64_t, int64_t>> call;
    if (d->ncon) call.push_back({0, d->ncon});
    cut(0, call);
    cut(1, p->copy_jac);
    cut(2, p->copy_hess);
    p->d2h_c[3] = (int)ch.size();
    if (!ch.empty()) {
      CU(cudaMalloc((void**)&p->d2h, ch.size() * sizeof(ExaD2HChunk)));
      CU(cudaMemcpy(p->d2h, ch.data(), ch.size() * sizeof(ExaD2HChunk), cudaMemcpyHostToDevice));
    }
  }
  p->threads[0] = d->threads[0] > 0 ? d->threads[0] : 128;
  p->threads[1] = d->threads[1] > 0 ? d->threads[1] : 256;
  p->n_terms = d->n_terms;
  p->has_checks = d->has_domain_checks;
  p->n_vscr = d->n_vscr;
  p->n_gscr = d->n_gscr;
  if ((rc = dev_upload(&p->f64, d->f64, (size_t)d->n_f64))) return bail(rc);
  if ((rc = dev_upload(&p->i32, d->i32, (size_t)d->n_i32))) return bail(rc);
  p->bytes += d->n_f64 * 8 + d->n_i32 * 4;

  // terms: translate blob offsets into device pointers
  std::vector<ExaTerm> terms(d->n_terms);
  for (int t = 0; t < d->n_terms; ++t) {
    const ExaTermDesc& s = d->terms[t];
    ExaTerm& T = terms[t];
    memset(&T, 0, sizeof T);
    for (int i = 0; i < EXA_MAXF; ++i) T.f[i] = s.f_off[i] >= 0 ? p->f64 + s.f_off[i] : nullptr;
    for (int i = 0; i < EXA_MAXI; ++i) T.ix[i] = s.ix_off[i] >= 0 ? p->i32 + s.ix_off[i] : nullptr;
    T.rows = s.rows_off >= 0 ? p->i32 + s.rows_off : nullptr;
    T.row_ptr = s.row_ptr_off >= 0 ? p->i32 + s.row_ptr_off : nullptr;
    T.row_ent = s.row_ent_off >= 0 ? reinterpret_cast<const int2*>(p->i32 + s.row_ent_off) : nullptr;
    for (int i = 0; i < EXA_MAXK; ++i) T.voff[i] = s.voff[i];
    T.nrec = s.nrec;
    T.pattern = s.pattern;
    T.kind = s.kind;
    T.order = s.order;
    T.row_offset = s.row_offset;
    T.cons_direct = s.cons_direct;
    T.k = s.k;
    T.jac0 = s.jac0;
    T.hess0 = s.hess0;
    T.scr0 = s.scr0;
    if (s.row_ent_off >= 0 && (s.row_ent_off & 1)) return bail(fail("term %d: row entries misaligned", t));
  }
  if ((rc = dev_upload(&p->terms, terms.data(), terms.size()))) return bail(rc);
  p->bytes += terms.size() * sizeof(ExaTerm);

  for (int m = 0; m < EXA_NMODES; ++m) {
    p->err_base[m][0] = d->err_base[m][0];
    p->err_base[m][1] = d->err_base[m][1];
  }
  for (int kid = 0; kid < EXA_NKERN; ++kid) {
    const int ns = d->n_segs[kid];
    const int th = p->threads[kid & 1];
    p->n_ctas[kid] = d->n_ctas[kid];
    if (ns == 0) continue;
    if ((rc = dev_upload(&p->segs[kid], reinterpret_cast<const ExaSeg*>(d->segs[kid]), (size_t)ns))) return bail(rc);
    std::vector<int> map(d->n_ctas[kid], -1);
    for (int s = 0; s < ns; ++s) {
      const ExaSegDesc& sg = d->segs[kid][s];
      const int rpt = (sg.kind >> 8) > 0 ? (sg.kind >> 8) : 1;  // records per thread
      const int nc = (sg.nrec + th * rpt - 1) / (th * rpt);
      for (int c = 0; c < nc; ++c) {
        if (sg.cta0 + c >= d->n_ctas[kid]) return bail(fail("kernel %d: segment %d overflows the grid", kid, s));
        map[sg.cta0 + c] = s;
      }
    }
    for (int c = 0; c < d->n_ctas[kid]; ++c)
      if (map[c] < 0) return bail(fail("kernel %d: CTA %d has no segment", kid, c));
    if ((rc = dev_upload(&p->cta_seg[kid], map.data(), map.size()))) return bail(rc);
    p->bytes += ns * sizeof(ExaSeg) + map.size() * sizeof(int);
  }

  p->n_leaves = d->n_leaves;
  p->n_prog = d->n_prog;
  for (int l = 0; l < d->n_leaves; ++l)
    if (d->leaves[2 * l + 1] > p->obj_leaf_max) p->obj_leaf_max = d->leaves[2 * l + 1];
  {
    const int depth = d->n_prog ? prog_depth(d->obj_prog, d->n_prog, d->n_leaves) : 0;
    if (depth < 0) return bail(fail("objective combine program is malformed"));
    if (depth > EXA_OBJ_STACK)
      return bail(fail("objective combine program needs a stack of %d > %d entries", depth, EXA_OBJ_STACK));
  }
  if ((rc = dev_upload(&p->leaves, d->leaves, (size_t)d->n_leaves * 2))) return bail(rc);
  if ((rc = dev_upload(&p->prog, d->obj_prog, (size_t)d->n_prog * 3))) return bail(rc);
  {
    std::vector<ExaObjNode> nodes;
    std::vector<double> init;
    std::vector<int32_t> lvl;
    if (!obj_dag(d->obj_prog, d->n_prog, d->n_leaves, nodes, init, lvl))
      return bail(fail("objective combine program is malformed"));
    p->n_onodes = (int32_t)nodes.size();
    p->n_olvl = (int32_t)lvl.size() - 1;
    if ((rc = dev_upload(&p->onodes, nodes.data(), nodes.size()))) return bail(rc);
    if ((rc = dev_upload(&p->oinit, init.data(), init.size()))) return bail(rc);
    if ((rc = dev_upload(&p->olvl, lvl.data(), lvl.size()))) return bail(rc);
  }
  if (d->grad_ptr) {
    if ((rc = dev_upload(&p->grad_ptr, d->grad_ptr, (size_t)d->nvar + 1))) return bail(rc);
    if ((rc = dev_upload(&p->grad_ent, d->grad_ent, (size_t)d->n_grad_ent))) return bail(rc);
  }

  cudaError_t e = cudaLibraryLoadData(&p->lib, d->cubin, nullptr, nullptr, 0, nullptr, nullptr, 0);
  if (e != cudaSuccess) return bail(fail("cudaLibraryLoadData: %s", cudaGetErrorString(e)));
  int n_sm = 0;
  CU(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, p->device));
  for (int kid = 0; kid < EXA_NKERN; ++kid) {
    e = cudaLibraryGetKernel(&p->kern[kid], p->lib, kKernelNames[kid]);
    if (e != cudaSuccess)
      return bail(fail("cudaLibraryGetKernel(%s): %s", kKernelNames[kid], cudaGetErrorString(e)));
    const int V = d->persist[kid];
    p->persist[kid] = V > 0 ? V : 0;
    p->grid[kid] = p->n_ctas[kid];
    if (V > 0 && p->n_ctas[kid] > 0) {
      // one wave: as many real CTAs as can be co-resident, never more than needed
      int occ = 0;
      CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)p->kern[kid], p->threads[kid & 1] * V, 0));
      if (occ < 1) return bail(fail("kernel %s: zero occupancy", kKernelNames[kid]));
      const int need = (p->n_ctas[kid] + V - 1) / V;
      p->grid[kid] = need < occ * n_sm ? need : occ * n_sm;
    }
  }
  // the strided-batch entry exists in model-specialised modules only (the
  // descriptor says so): no failing symbol lookup for generic modules
  if (d->batchable && cudaLibraryGetKernel(&p->kern_batch, p->lib, "exa_k_setb_l") != cudaSuccess) {
    cudaGetLastError();
    p->kern_batch = nullptr;
  }
  if ((rc = ws_alloc(p, &p->dflt))) return bail(rc);
  *out = p;
  return 0;
}

int exa_plan_info(const ExaPlan* p, int64_t* bytes, int32_t* regs) {
  if (!p) return fail("exa_plan_info: null plan");
  if (bytes) *bytes = (int64_t)p->bytes;
  if (regs) {
    cudaFuncAttributes a;
    const int kid = p->n_ctas[2 * EXA_MODE_SET] > 0 ? 2 * EXA_MODE_SET : 2 * EXA_MODE_SET + 1;
    CU(cudaFuncGetAttributes(&a, (const void*)p->kern[kid]));
    *regs = a.numRegs;
  }
  return 0;
}

static int launch_kid(ExaPlan* p, ExaWorkspace* w, int kid, ExaArgs A, cudaStream_t st, unsigned nbatch = 1,
                      bool cmp = false) {
  const ExaTerm* terms = p->terms;
  const ExaSeg* segs = p->segs[kid];
  const int* cmap = p->cta_seg[kid];
  void* args[] = {(void*)&terms, (void*)&segs, (void*)&cmap, (void*)&A};
  // Programmatic dependent launch: this kernel may be scheduled while the
  // previous work on the stream drains; it loads the (immutable) plan data,
  // then waits (griddepcontrol.wait) before touching caller buffers.
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p->grid[kid], nbatch);
  cfg.blockDim = dim3(p->threads[kid & 1] * (p->persist[kid] ? p->persist[kid] : 1));
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = p->pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const bool batch_kernel = nbatch > 1 && kid == 2 * EXA_MODE_SET + 1 && p->kern_batch;
  cudaKernel_t k = batch_kernel ? p->kern_batch : p->kern[kid];
  if (cmp) k = p->kern_cmp[kid & 1];
  CU(cudaLaunchKernelExC(&cfg, (const void*)k, args));
  return 0;
}

// One callback = its heavy kernel on `st` and its light kernel on the
// workspace's aux stream, forked/joined with events (graph-capturable).
static int launch_mode(ExaPlan* p, ExaWorkspace* w, int mode, ExaArgs& A, cudaStream_t st, unsigned nbatch = 1,
                       bool cmp = false) {
  A.err = w->err;
  A.trace = g_trace;
  A.obj_base = p->err_base[mode][0];
  A.con_base = p->err_base[mode][1];
  A.f64 = p->f64;
  A.i32 = p->i32;
  const int kh = 2 * mode, kl = 2 * mode + 1;
  const bool h = p->n_ctas[kh] > 0, l = p->n_ctas[kl] > 0;
  int rc = 0;
  if (h && l) {
    // heavy first: its few, long-lived CTAs must become resident before the
    // light kernel's many short CTAs fill every SM
    CU(cudaEventRecord(w->fork, st));
    CU(cudaStreamWaitEvent(w->aux, w->fork, 0));
    if ((rc = launch_kid(p, w, kh, A, st, nbatch, cmp))) return rc;
    if ((rc = launch_kid(p, w, kl, A, w->aux, nbatch, cmp))) return rc;
    CU(cudaEventRecord(w->join, w->aux));
    CU(cudaStreamWaitEvent(st, w->join, 0));
  } else if (h) {
    rc = launch_kid(p, w, kh, A, st, nbatch, cmp);
  } else if (l) {
    rc = launch_kid(p, w, kl, A, st, nbatch, cmp);
  }
  return rc;
}

static int reset_err(ExaPlan* p, ExaWorkspace* w, cudaStream_t st) {
  if (p->has_checks) CU(cudaMemsetAsync(w->err, 0xff, sizeof(unsigned long long), st));
  return 0;
}

// Launches go to the plan's device: make it current for the call (and restore
// the caller's device after), so a caller whose current device differs gets
// the plan's kernels on the plan's device instead of a launch error.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) == cudaSuccess && prev != dev) cudaSetDevice(dev);
    else prev = -1;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

#define EXA_PROLOGUE()                                      \
  if (!p) return fail("null plan");                         \
  DeviceGuard dguard_(p->device);                           \
  ExaWorkspace* w = ws ? ws : p->dflt;                      \
  cudaStream_t st = (cudaStream_t)stream;                   \
  ExaArgs A;                                                \
  memset(&A, 0, sizeof A);                                  \
  if (int rc_ = reset_err(p, w, st)) return rc_;

static int eval_set(ExaPlan* p, ExaWorkspace* ws, const double* x, const double* mult, double w_obj, double* c,
                    double* jac, double* hess, exa_stream_t stream, double* jac_c, double* hess_c) {
  EXA_PROLOGUE();
  A.x = x;
  A.y = mult;
  A.w = w_obj;
  A.c = c;
  A.J = jac;
  A.H = hess;
  A.Jc = jac_c;
  A.Hc = hess_c;
  A.hpos = hess_c ? p->hpos : nullptr;  // no compressed Hessian: raw slots everywhere
  return launch_mode(p, w, EXA_MODE_SET, A, st, 1, jac_c != nullptr || hess_c != nullptr);
}

int exa_eval_set(ExaPlan* p, ExaWorkspace* ws, const double* x, const double* mult, double w_obj, double* c,
                 double* jac, double* hess, exa_stream_t stream) {
  return eval_set(p, ws, x, mult, w_obj, c, jac, hess, stream, nullptr, nullptr);
}

int exa_eval_set_batch(ExaPlan* p, ExaWorkspace* ws, int64_t nsets, const double* x, const double* mult,
                       double w_obj, double* c, double* jac, double* hess, exa_stream_t stream) {
  if (!p) return fail("null plan");
  if (nsets < 0 || nsets > 65535) return fail("exa_eval_set_batch: nsets %lld outside [0, 65535]", (long long)nsets);
  if (!p->batchable) return fail("exa_eval_set_batch: this plan's module does not support batches");
  if (nsets == 0) return 0;
  EXA_PROLOGUE();
  A.x = x;
  A.y = mult;
  A.w = w_obj;
  A.c = c;
  A.J = jac;
  A.H = hess;
  return launch_mode(p, w, EXA_MODE_SET, A, st, (unsigned)nsets);
}

// ---------------------------------------------------------------------------
// host fill of constant output runs: a small persistent pool of threads (the
// caller included) writes the runs in 256 KB pieces; a run of +0.0 is a memset
// ---------------------------------------------------------------------------
namespace {
struct FillPool {
  // dst[0, n) = v, or (src) = src[0, n) once event ev (if any) has completed
  struct Piece {
    double* dst; int64_t n; double v; const double* src = nullptr; cudaEvent_t ev = nullptr;
    const int32_t* rows = nullptr; const double* mult = nullptr;  // weighted zeros: dst[i] = mult[rows[i]] * v
  };
  std::mutex call_mu;  // one fill at a time
  std::mutex mu;
  std::condition_variable cv;
  std::vector<std::thread> workers;
  const std::vector<Piece>* job = nullptr;
  uint64_t gen = 0;
  std::atomic<size_t> next{0};
  std::atomic<int> active{0};

  static void run(const Piece& q) {
    if (q.rows) {
      for (int64_t i = 0; i < q.n; ++i) q.dst[i] = q.mult[q.rows[i]] * q.v;
    } else if (q.src) {
      if (q.ev) cudaEventSynchronize(q.ev);
      std::memcpy(q.dst, q.src, q.n * sizeof(double));
    } else if (q.v == 0.0 && !std::signbit(q.v)) {
      std::memset(q.dst, 0, q.n * sizeof(double));
    } else {
      for (int64_t i = 0; i < q.n; ++i) q.dst[i] = q.v;
    }
  }
  void drain(const std::vector<Piece>& pcs) {
    for (size_t i; (i = next.fetch_add(1)) < pcs.size();) run(pcs[i]);
  }
  explicit FillPool(int n) {
    for (int t = 0; t < n; ++t)
      workers.emplace_back([this] {
        uint64_t seen = 0;
        for (;;) {
          const std::vector<Piece>* j;
          {
            std::unique_lock<std::mutex> lk(mu);
            cv.wait(lk, [&] { return gen != seen; });
            seen = gen;
            j = job;
            active.fetch_add(1);
          }
          if (j) drain(*j);
          active.fetch_sub(1);
        }
      });
    for (auto& t : workers) t.detach();
  }
  void fill(const std::vector<Piece>& pcs) {
    std::lock_guard<std::mutex> g(call_mu);
    int64_t bytes = 0;
    for (auto& q : pcs) bytes += q.n * 8;
    next.store(0);
    if (!workers.empty() && bytes > (1 << 20)) {
      {
        std::lock_guard<std::mutex> lk(mu);
        job = &pcs;
        ++gen;
      }
      cv.notify_all();
      drain(pcs);
      // every piece is claimed; wait for the workers still writing one
      {
        std::lock_guard<std::mutex> lk(mu);
        job = nullptr;
      }
      while (active.load() > 0) std::this_thread::yield();
    } else {
      drain(pcs);
    }
  }
};

FillPool& fill_pool() {
  static FillPool* pool = [] {
    int n = (int)std::thread::hardware_concurrency() / 2;
    if (const char* e = std::getenv("EXA_HOST_FILL_THREADS")) n = std::atoi(e);
    if (n > 8) n = 8;
    return new FillPool(n > 0 ? n - 1 : 0);  // the caller is the n-th
  }();
  return *pool;
}
}  // namespace

constexpr int64_t kPiece = 32768;  // doubles (256 KB) per host-pool piece

static void add_fill(const ExaPlan* p, double* jac, double* hess, const double* mult, double w_obj,
                     std::vector<FillPool::Piece>& pcs) {
  for (auto* rs : {&p->fill_jac, &p->fill_hess}) {
    double* out = rs == &p->fill_jac ? jac : hess;
    if (!out) continue;
    for (auto& r : *rs)
      for (int64_t o = 0; o < r.n; o += kPiece) pcs.push_back({out + r.a + o, r.n - o < kPiece ? r.n - o : kPiece, r.v});
  }
  if (!hess) return;
  for (auto& r : p->fill_wz)
    for (int64_t o = 0; o < r.n; o += kPiece) {
      const int64_t n = r.n - o < kPiece ? r.n - o : kPiece;
      if (r.off < 0) {  // objective weight: a constant run
        pcs.push_back({hess + r.a + o, n, w_obj * r.z});
      } else {
        FillPool::Piece q{hess + r.a + o, n, r.z};
        q.rows = p->wz_rows.data() + r.off + o;
        q.mult = mult;
        pcs.push_back(q);
      }
    }
}

static bool pageable(const void* ptr) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

// Host path, pinned outputs: the x-dependent output ranges stored by SMs
// straight into the caller's page-locked arrays (mapped into the device's
// address space), one launch for all ranges -- every copy-engine transfer
// adds ~3.6 us of engine time (tools/micro/d2hstore.cu).  One CTA per chunk;
// 16-byte accesses when source and destination share their alignment.
__global__ void __launch_bounds__(128) exa_d2h_store(const ExaD2HChunk* __restrict__ ch, int c0, double* d0, double* d1,
                                                     double* d2, const double* s0, const double* s1, const double* s2) {
  const ExaD2HChunk q = ch[c0 + blockIdx.x];
  double* dst = q.arr == 0 ? d0 : (q.arr == 1 ? d1 : d2);
  const double* src = q.arr == 0 ? s0 : (q.arr == 1 ? s1 : s2);
  int64_t a = q.a;
  const int64_t e = q.e;
  if (((reinterpret_cast<uintptr_t>(dst) ^ reinterpret_cast<uintptr_t>(src)) & 15) == 0) {
    if (reinterpret_cast<uintptr_t>(dst + a) & 15) {
      if (threadIdx.x == 0) dst[a] = __ldcs(src + a);
      ++a;
    }
    const int64_t nv = (e - a) >> 1;
    double2* dv = reinterpret_cast<double2*>(dst + a);
    const double2* sv = reinterpret_cast<const double2*>(src + a);
    for (int64_t i = threadIdx.x; i < nv; i += blockDim.x) dv[i] = __ldcs(sv + i);
    if (((e - a) & 1) && threadIdx.x == 0) dst[e - 1] = __ldcs(src + e - 1);
  } else {
    for (int64_t i = a + threadIdx.x; i < e; i += blockDim.x) dst[i] = __ldcs(src + i);
  }
}

// device address of a page-locked host array, or null (pageable / not mapped /
// not 8-byte aligned: those take the copy-engine path)
static double* mapped(void* h) {
  if (!h || (reinterpret_cast<uintptr_t>(h) & 7)) return nullptr;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, h) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return a.type == cudaMemoryTypeHost ? static_cast<double*>(a.devicePointer) : nullptr;
}

// D2H ranges (dst host, src device, doubles) of one host-path set
struct Range { double* dst; const double* src; int64_t n; };

static std::vector<Range> d2h_ranges(const ExaPlan* p, const ExaWorkspace* w, double* c, double* jac, double* hess) {
  std::vector<Range> r;
  if (c && p->ncon) r.push_back({c, w->dc, p->ncon});
  if (jac)
    for (auto& q : p->copy_jac) r.push_back({jac + q.first, w->dJ + q.first, q.second});
  if (hess)
    for (auto& q : p->copy_hess) r.push_back({hess + q.first, w->dH + q.first, q.second});
  return r;
}

// Device staging of a workspace, sized for its plan (first use; caller holds w->mu).
static int ws_staging(ExaPlan* p, ExaWorkspace* w) {
  if (w->dx) return 0;
  CU(cudaSetDevice(p->device));
  CU(cudaMalloc((void**)&w->dx, (p->nvar > 0 ? p->nvar : 1) * sizeof(double)));
  CU(cudaMalloc((void**)&w->dy, (p->ncon > 0 ? p->ncon : 1) * sizeof(double)));
  CU(cudaMalloc((void**)&w->dc, (p->ncon > 0 ? p->ncon : 1) * sizeof(double)));
  CU(cudaMalloc((void**)&w->dJ, (p->n_jac > 0 ? p->n_jac : 1) * sizeof(double)));
  CU(cudaMalloc((void**)&w->dH, (p->n_hess > 0 ? p->n_hess : 1) * sizeof(double)));
  return 0;
}

// Host-buffer form of one callback (mode SET, CONS, JAC or HESS): H2D of the
// inputs the mode reads, the device callback on the workspace's staging, D2H
// of its x-dependent output ranges, constant runs filled on the host.  Null
// output pointers are the outputs the mode does not produce.
static int host_eval(ExaPlan* p, ExaWorkspace* ws, int mode, const double* x, const double* mult, double w_obj,
                     double* c, double* jac, double* hess, cudaStream_t st) {
  if (!p) return fail("null plan");
  DeviceGuard dguard(p->device);
  ExaWorkspace* w = ws ? ws : p->dflt;
  std::unique_lock<std::mutex> lazy(w->mu);
  if (int rc_ = ws_staging(p, w)) return rc_;
  if (mode != EXA_MODE_SET && mode != EXA_MODE_HESS) mult = nullptr;
  if (mode != EXA_MODE_SET && mode != EXA_MODE_CONS) c = nullptr;
  if (mode != EXA_MODE_SET && mode != EXA_MODE_JAC) jac = nullptr;
  if (mode != EXA_MODE_SET && mode != EXA_MODE_HESS) hess = nullptr;
  const bool pg_in = (p->nvar && pageable(x)) || (mult && p->ncon && pageable(mult));
  const bool pg_out = (c && p->ncon && pageable(c)) || (jac && p->n_jac && pageable(jac)) ||
                      (hess && p->n_hess && pageable(hess));
  if ((pg_in || pg_out) && !w->hstage) {  // pinned staging for pageable callers (numpy arrays)
    CU(cudaHostAlloc((void**)&w->hstage, (p->nvar + 2 * p->ncon + p->n_jac + p->n_hess + 1) * sizeof(double),
                     cudaHostAllocDefault));
  }
  lazy.unlock();
  const double* xs = x;
  const double* ys = mult;
  if (pg_in) {  // pageable inputs: host threads copy them into pinned staging, then one DMA each
    std::vector<FillPool::Piece> pcs;
    for (int64_t o = 0; o < p->nvar; o += kPiece)
      pcs.push_back({w->hstage + o, p->nvar - o < kPiece ? p->nvar - o : kPiece, 0.0, x + o});
    for (int64_t o = 0; mult && o < p->ncon; o += kPiece)
      pcs.push_back({w->hstage + p->nvar + o, p->ncon - o < kPiece ? p->ncon - o : kPiece, 0.0, mult + o});
    CU(cudaStreamSynchronize(st));  // the staging may still feed an earlier set's H2D
    fill_pool().fill(pcs);
    xs = w->hstage;
    ys = w->hstage + p->nvar;
  }
  if (p->nvar) CU(cudaMemcpyAsync(w->dx, xs, p->nvar * sizeof(double), cudaMemcpyHostToDevice, st));
  if (mult && p->ncon) CU(cudaMemcpyAsync(w->dy, ys, p->ncon * sizeof(double), cudaMemcpyHostToDevice, st));
  int rc = 0;
  switch (mode) {
    case EXA_MODE_SET: rc = exa_eval_set(p, w, w->dx, w->dy, w_obj, w->dc, w->dJ, w->dH, st); break;
    case EXA_MODE_CONS: rc = exa_eval_cons(p, w, w->dx, w->dc, st); break;
    case EXA_MODE_JAC: rc = exa_eval_jac(p, w, w->dx, w->dJ, st); break;
    case EXA_MODE_HESS: rc = exa_eval_hess(p, w, w->dx, w->dy, w_obj, w->dH, st); break;
    default: return fail("host_eval: mode %d has no host form", mode);
  }
  if (rc) return rc;
  std::vector<FillPool::Piece> pcs;
  if (pg_out) {
    // pageable outputs: DMA each range, in 2 MB chunks, into pinned staging
    // (event per chunk); host threads copy chunk k into the caller's arrays
    // while later chunks are still in flight.  Returns with outputs complete.
    constexpr int64_t kChunk = 262144;  // doubles
    double* hs = w->hstage + p->nvar + p->ncon;
    int64_t at = 0;
    size_t ne = 0;
    for (const Range& r : d2h_ranges(p, w, c, jac, hess)) {
      for (int64_t o = 0; o < r.n; o += kChunk) {
        const int64_t n = r.n - o < kChunk ? r.n - o : kChunk;
        CU(cudaMemcpyAsync(hs + at, r.src + o, n * sizeof(double), cudaMemcpyDeviceToHost, st));
        if (ne == w->chunk_ev.size()) {
          cudaEvent_t e;
          CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
          w->chunk_ev.push_back(e);
        }
        cudaEvent_t e = w->chunk_ev[ne++];
        CU(cudaEventRecord(e, st));
        for (int64_t q = 0; q < n; q += kPiece)
          pcs.push_back({r.dst + o + q, n - q < kPiece ? n - q : kPiece, 0.0, hs + at + q, e});
        at += n;
      }
    }
  } else {
    // pinned outputs: everything but the constant runs crosses PCIe while
    // the constant runs are written on the host.  Default: one store kernel
    // into the mapped arrays (case13659 e2e 4.09k sets/s); EXA_D2H=dma, or
    // arrays not mapped: copy-engine transfers, 2D where ranges repeat at a
    // constant stride (3.54k: every transfer adds ~3.6 us of engine time)
    static const bool dma = [] { const char* e = std::getenv("EXA_D2H"); return e && std::strcmp(e, "dma") == 0; }();
    double *mc = dma ? nullptr : mapped(c), *mj = dma ? nullptr : mapped(jac), *mh = dma ? nullptr : mapped(hess);
    // the wanted outputs must be consecutive in chunk order (c, J, H)
    const bool want[3] = {c != nullptr, jac != nullptr, hess != nullptr}, got[3] = {mc != nullptr, mj != nullptr, mh != nullptr};
    int k0 = 0, k1 = 3;
    while (k0 < 3 && !want[k0]) ++k0;
    while (k1 > k0 && !want[k1 - 1]) --k1;
    bool ok = !dma;
    for (int k = k0; k < k1; ++k) ok = ok && want[k] && got[k];
    const int c0 = p->d2h_c[k0 < 3 ? k0 : 3], n_ch = p->d2h_c[k1 > k0 ? k1 : k0 < 3 ? k0 : 3] - c0;
    if (ok && n_ch > 0) {
      exa_d2h_store<<<n_ch, 128, 0, st>>>(p->d2h, c0, mc, mj, mh, w->dc, w->dJ, w->dH);
      CU(cudaGetLastError());
    } else {
      double* dst[3] = {c, jac, hess};
      const double* src[3] = {w->dc, w->dJ, w->dH};
      for (const ExaPlan::Op& o : p->d2h_ops) {
        if (!dst[o.arr]) continue;
        if (o.rows == 1)
          CU(cudaMemcpyAsync(dst[o.arr] + o.a, src[o.arr] + o.a, o.n * sizeof(double), cudaMemcpyDeviceToHost, st));
        else
          CU(cudaMemcpy2DAsync(dst[o.arr] + o.a, o.pitch * sizeof(double), src[o.arr] + o.a, o.pitch * sizeof(double),
                               o.n * sizeof(double), o.rows, cudaMemcpyDeviceToHost, st));
      }
    }
  }
  add_fill(p, jac, hess, mult, w_obj, pcs);
  if (!pcs.empty()) fill_pool().fill(pcs);
  return 0;
}

int exa_eval_set_host(ExaPlan* p, ExaWorkspace* ws, const double* x, const double* mult, double w_obj, double* c,
                      double* jac, double* hess, exa_stream_t stream) {
  return host_eval(p, ws, EXA_MODE_SET, x, mult, w_obj, c, jac, hess, (cudaStream_t)stream);
}

int exa_eval_cons_host(ExaPlan* p, ExaWorkspace* ws, const double* x, double* c, exa_stream_t stream) {
  return host_eval(p, ws, EXA_MODE_CONS, x, nullptr, 0.0, c, nullptr, nullptr, (cudaStream_t)stream);
}

int exa_eval_jac_host(ExaPlan* p, ExaWorkspace* ws, const double* x, double* jac, exa_stream_t stream) {
  return host_eval(p, ws, EXA_MODE_JAC, x, nullptr, 0.0, nullptr, jac, nullptr, (cudaStream_t)stream);
}

int exa_eval_hess_host(ExaPlan* p, ExaWorkspace* ws, const double* x, const double* mult, double w_obj,
                       double* hess, exa_stream_t stream) {
  return host_eval(p, ws, EXA_MODE_HESS, x, mult, w_obj, nullptr, nullptr, hess, (cudaStream_t)stream);
}

// Page-lock a caller's pageable range in place, mapped and portable, so the
// host-buffer entries treat it like page-locked memory (H2D without staging,
// D2H by the store kernel through its device mapping).  A failure (range
// already registered, memory limits) leaves it pageable and clears the error.
int exa_host_register(void* ptr, size_t bytes) {
  if (!ptr || !bytes) return fail("exa_host_register: empty range");
  const cudaError_t e = cudaHostRegister(ptr, bytes, cudaHostRegisterPortable | cudaHostRegisterMapped);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail("exa_host_register: cudaHostRegister failed: %s", cudaGetErrorString(e));
  }
  return 0;
}

int exa_host_unregister(void* ptr) {
  const cudaError_t e = cudaHostUnregister(ptr);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail("exa_host_unregister: cudaHostUnregister failed: %s", cudaGetErrorString(e));
  }
  return 0;
}

static int pattern_build(ExaPlan* p, int64_t n_raw, int64_t nnz, const int64_t* ptr, const int32_t* ent,
                         const uint8_t* known, const double* known_val, ExaPattern** out,
                         const uint8_t* direct = nullptr) {
  if (!p || !out || n_raw < 0 || nnz < 0 || (nnz && !ptr) || (n_raw && !ent) || (known && !known_val))
    return fail("exa_pattern_create: invalid argument");
  *out = nullptr;
  if (ptr && (ptr[0] != 0 || ptr[nnz] != n_raw)) return fail("exa_pattern_create: ptr must run from 0 to n_raw");
  for (int64_t k = 0; k < nnz; ++k)
    if (ptr[k + 1] < ptr[k]) return fail("exa_pattern_create: ptr must be non-decreasing");
  for (int64_t e = 0; e < n_raw; ++e)
    if (ent[e] < 0 || ent[e] >= n_raw) return fail("exa_pattern_create: raw slot %lld out of range", (long long)e);
  if (n_raw >= INT32_MAX || nnz >= INT32_MAX) return fail("exa_pattern_create: more than 2^31 - 1 slots");
  const int ipt = cmp_ipt_env(), EXA_CMP_CAP = EXA_CMP_THREADS * ipt;
  /* per raw slot: 0 = gathered, 1 = known +0.0 (dropped), 2 = known constant */
  auto cls = [&](int32_t r) -> int {
    if (!known || !known[r]) return 0;
    uint64_t bits;
    std::memcpy(&bits, known_val + r, 8);
    return bits == 0 ? 1 : 2;
  };
  std::vector<int32_t> stage_len((size_t)nnz);
  for (int64_t k = 0; k < nnz; ++k) {
    int32_t L = 0;
    for (int64_t e = ptr[k]; e < ptr[k + 1]; ++e) L += cls(ent[e]) != 1;
    stage_len[k] = L;
  }
  /* chunks of consecutive entries (ordering the entries by the record that
     produces their slots, so that gathers become runs, measured slower:
     case13659 18.0 vs 18.2 us, MP96 149 vs 131 us) */
  // entries written directly by the compressed-set kernels: exactly one raw
  // slot, flagged direct; they are left out of the chunks
  std::vector<int32_t> order;
  order.reserve((size_t)nnz);
  for (int64_t k = 0; k < nnz; ++k) {
    // an entry is left out when every slot that is not a known +0.0 is
    // direct (folded by the set kernel); a partly direct entry is an error
    int n_dir = 0, n_other = 0;
    if (direct)
      for (int64_t e = ptr[k]; e < ptr[k + 1]; ++e) {
        if (direct[ent[e]]) ++n_dir;
        else if (cls(ent[e]) != 1) ++n_other;
      }
    if (n_dir && n_other)
      return fail("exa_pattern_create_direct: entry %lld mixes %d direct with %d other slots", (long long)k, n_dir,
                  n_other);
    if (!n_dir) order.push_back((int32_t)k);
  }
  const int64_t n_fold = (int64_t)order.size();
  std::vector<int32_t> chk{0}, che{0}, chc{0}, src, eout((size_t)n_fold);
  std::vector<uint16_t> dst, cpos, cid;
  std::vector<uint32_t> edesc((size_t)n_fold);
  std::vector<int32_t> est((size_t)n_fold);
  std::vector<double> cval;
  std::unordered_map<uint64_t, uint16_t> cmap;
  std::vector<std::pair<int32_t, int32_t>> gat;
  for (int64_t q0 = 0; q0 < n_fold;) {
    int64_t q1 = q0 + 1, tot = stage_len[order[q0]];
    while (q1 < n_fold && q1 - q0 < EXA_CMP_CAP && tot + stage_len[order[q1]] <= EXA_CMP_CAP) tot += stage_len[order[q1++]];
    if (tot > EXA_CMP_CAP) {  // one long entry: every non-dropped slot gathered, slot order
      const int64_t k = order[q0];
      for (int64_t e = ptr[k]; e < ptr[k + 1]; ++e)
        if (cls(ent[e]) != 1) src.push_back(ent[e]), dst.push_back(0);
      edesc[q0] = 0;
      eout[q0] = (int32_t)k;
    } else {
      gat.clear();
      int32_t pos = 0;
      for (int64_t q = q0; q < q1; ++q) {
        const int64_t k = order[q];
        est[q] = pos;
        for (int64_t e = ptr[k]; e < ptr[k + 1]; ++e) {
          const int c = cls(ent[e]);
          if (c == 1) continue;
          uint16_t id = 0;
          bool as_const = false;
          if (c == 2) {
            uint64_t bits;
            std::memcpy(&bits, known_val + ent[e], 8);
            auto it = cmap.find(bits);
            if (it != cmap.end()) {
              id = it->second;
              as_const = true;
            } else if (cval.size() < 65535) {
              id = (uint16_t)cval.size();
              cmap.emplace(bits, id);
              cval.push_back(known_val[ent[e]]);
              as_const = true;
            }
          }
          if (as_const) {
            cpos.push_back((uint16_t)pos);
            cid.push_back(id);
          } else {
            gat.emplace_back(ent[e], pos);
          }
          ++pos;
        }
      }
      std::sort(gat.begin(), gat.end());
      for (auto& g : gat) src.push_back(g.first), dst.push_back((uint16_t)g.second);
      /* entry slots of the chunk, longest stage first (stable) */
      std::vector<int64_t> qs;
      for (int64_t q = q0; q < q1; ++q) qs.push_back(q);
      std::stable_sort(qs.begin(), qs.end(),
                       [&](int64_t x, int64_t y) { return stage_len[order[x]] > stage_len[order[y]]; });
      for (int64_t i = 0; i < q1 - q0; ++i) {
        const int64_t q = qs[i];
        edesc[q0 + i] = (uint32_t)est[q] | ((uint32_t)stage_len[order[q]] << 16);
        eout[q0 + i] = order[q];
      }
    }
    chk.push_back((int32_t)q1);
    che.push_back((int32_t)src.size());
    chc.push_back((int32_t)cpos.size());
    q0 = q1;
  }
  DeviceGuard g(p->device);
  ExaPattern* q = new ExaPattern();
  q->device = p->device;
  q->n_raw = n_raw;
  q->nnz = nnz;
  q->direct = direct != nullptr;
  q->nch = (int32_t)(chk.size() - 1);
  q->ipt = ipt;
  int rc = dev_upload(&q->chk, chk.data(), chk.size());
  if (!rc) rc = dev_upload(&q->che, che.data(), che.size());
  if (!rc) rc = dev_upload(&q->chc, chc.data(), chc.size());
  if (!rc) rc = dev_upload(&q->src, src.data(), src.size());
  if (!rc) rc = dev_upload(&q->dst, dst.data(), dst.size());
  if (!rc) rc = dev_upload(&q->cpos, cpos.data(), cpos.size());
  if (!rc) rc = dev_upload(&q->cid, cid.data(), cid.size());
  if (!rc) rc = dev_upload(&q->edesc, edesc.data(), edesc.size());
  if (!rc) rc = dev_upload(&q->eout, eout.data(), eout.size());
  if (!rc) rc = dev_upload(&q->cval, cval.data(), cval.size());
  if (rc) {
    exa_pattern_destroy(q);
    return rc;
  }
  *out = q;
  return 0;
}

int exa_pattern_create_known(ExaPlan* p, int64_t n_raw, int64_t nnz, const int64_t* ptr, const int32_t* ent,
                             const uint8_t* known, const double* known_val, ExaPattern** out) {
  return pattern_build(p, n_raw, nnz, ptr, ent, known, known_val, out);
}

int exa_pattern_create_direct(ExaPlan* p, int64_t n_raw, int64_t nnz, const int64_t* ptr, const int32_t* ent,
                              const uint8_t* known, const double* known_val, const uint8_t* direct,
                              ExaPattern** out) {
  if (!direct) return fail("exa_pattern_create_direct: null direct mask");
  return pattern_build(p, n_raw, nnz, ptr, ent, known, known_val, out, direct);
}

int exa_plan_attach_compressed(ExaPlan* p, const void* cubin, int64_t cubin_size, const int32_t* hpos,
                               int64_t n_hpos) {
  if (!p || !cubin || cubin_size <= 0 || n_hpos < 0 || (n_hpos && !hpos))
    return fail("exa_plan_attach_compressed: invalid argument");
  if (p->lib_cmp) return 0;  // attached once per plan
  DeviceGuard g(p->device);
  if (n_hpos) {
    for (int64_t i = 0; i < n_hpos; ++i)
      if (hpos[i] < -1) return fail("exa_plan_attach_compressed: bad entry position %d", hpos[i]);
    if (int rc = dev_upload(&p->hpos, hpos, (size_t)n_hpos)) return rc;
  }
  cudaLibrary_t lib = nullptr;
  cudaError_t e = cudaLibraryLoadData(&lib, cubin, nullptr, nullptr, 0, nullptr, nullptr, 0);
  if (e != cudaSuccess) return fail("cudaLibraryLoadData (compressed module): %s", cudaGetErrorString(e));
  cudaKernel_t k[2];
  for (int h = 0; h < 2; ++h)
    if ((e = cudaLibraryGetKernel(&k[h], lib, h ? "exa_k_setc_l" : "exa_k_setc_h")) != cudaSuccess) {
      cudaLibraryUnload(lib);
      return fail("cudaLibraryGetKernel(exa_k_setc_%s): %s", h ? "l" : "h", cudaGetErrorString(e));
    }
  p->kern_cmp[0] = k[0];
  p->kern_cmp[1] = k[1];
  p->lib_cmp = lib;
  return 0;
}

int exa_pattern_create(ExaPlan* p, int64_t n_raw, int64_t nnz, const int64_t* ptr, const int32_t* ent,
                       ExaPattern** out) {
  return pattern_build(p, n_raw, nnz, ptr, ent, nullptr, nullptr, out);
}

void exa_pattern_destroy(ExaPattern* q) {
  if (!q) return;
  cudaFree(q->chk);
  cudaFree(q->che);
  cudaFree(q->chc);
  cudaFree(q->src);
  cudaFree(q->dst);
  cudaFree(q->cpos);
  cudaFree(q->cid);
  cudaFree(q->edesc);
  cudaFree(q->eout);
  cudaFree(q->cval);
  delete q;
}

// raw J / H of the set into the workspace scratch, then both segmented sums in
// one programmatic-dependent launch (a NULL pattern: that output gets the raw
// slots themselves)
static int set_compressed(ExaPlan* p, ExaWorkspace* w, const ExaPattern* jp, const ExaPattern* hp, const double* x,
                          const double* mult, double w_obj, double* c, double* jc, double* hc, cudaStream_t st) {
  if ((jp && jp->n_raw != p->n_jac) || (hp && hp->n_raw != p->n_hess))
    return fail("exa_eval_set_compressed: pattern does not match the plan's raw J / H slots");
  if ((jp && jp->device != p->device) || (hp && hp->device != p->device))
    return fail("exa_eval_set_compressed: pattern on another device");
  if (jp && hp && jp->ipt != hp->ipt) return fail("exa_eval_set_compressed: patterns chunked for different EXA_CMP_IPT");
  double* rawJ = jp ? w->dJ : jc;
  double* rawH = hp ? w->dH : hc;
  if ((jp && jp->direct) || (hp && hp->direct)) {
    if (!(p->kern_cmp[0] && p->kern_cmp[1]))
      return fail("exa_eval_set_compressed: direct pattern but no compressed-set module attached");
    if (hp && hp->direct && !p->hpos)
      return fail("exa_eval_set_compressed: direct Hessian pattern but the plan has no entry positions");
  }
  // direct J pattern: the compressed-set kernels write the direct entries into
  // jc themselves and every other raw slot into the workspace scratch
  int rc = eval_set(p, w, x, mult, w_obj, c, rawJ, rawH, (exa_stream_t)st, jp && jp->direct ? jc : nullptr,
                    hp && hp->direct ? hc : nullptr);
  if (rc) return rc;
  const int nchJ = jp ? jp->nch : 0, nchH = hp ? hp->nch : 0;
  if (nchJ + nchH == 0) return 0;
  ExaCmpArgs aJ = {}, aH = {};
  if (jp) aJ = ExaCmpArgs{jp->chk, jp->che, jp->chc, jp->src, jp->dst, jp->cpos, jp->cid, jp->edesc, jp->eout, jp->cval,
                          rawJ, jc};
  if (hp) aH = ExaCmpArgs{hp->chk, hp->che, hp->chc, hp->src, hp->dst, hp->cpos, hp->cid, hp->edesc, hp->eout, hp->cval,
                          rawH, hc};
  static const int probe = getenv("EXA_CMP_PROBE") ? atoi(getenv("EXA_CMP_PROBE")) : 0;
  const int nch = nchJ + nchH;
  const int ipt = jp ? jp->ipt : hp->ipt;
  const void* fn = ipt == 1 ? (const void*)exa_compress2_kernel<1, 8>
                 : ipt == 2 ? (const void*)exa_compress2_kernel<2, 8>
                 : ipt == 4 ? (const void*)exa_compress2_kernel<4, 6>
                 : ipt == 12 ? (const void*)exa_compress2_kernel<12, 4>
                 : ipt == 16 ? (const void*)exa_compress2_kernel<16, 3>
                             : (const void*)exa_compress2_kernel<8, 6>;
  const size_t smem = (size_t)EXA_CMP_THREADS * ipt * 16;
  if (smem > 48 * 1024) {  // opt in once per (device, kernel)
    static std::mutex mu;
    static std::set<std::pair<int, const void*>> done;
    std::lock_guard<std::mutex> lk(mu);
    if (done.insert({p->device, fn}).second) CU(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  }
  void* args[] = {(void*)&nchJ, (void*)&nch, (void*)&aJ, (void*)&aH, (void*)&probe};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)nch);
  cfg.blockDim = dim3(EXA_CMP_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = p->pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CU(cudaLaunchKernelExC(&cfg, fn, args));
  return 0;
}

int exa_eval_set_compressed(ExaPlan* p, ExaWorkspace* ws, const ExaPattern* jpat, const ExaPattern* hpat,
                            const double* x, const double* mult, double w_obj, double* c, double* jac_c,
                            double* hess_c, exa_stream_t stream) {
  if (!p) return fail("null plan");
  DeviceGuard dguard(p->device);
  ExaWorkspace* w = ws ? ws : p->dflt;
  {
    std::lock_guard<std::mutex> lazy(w->mu);
    if (int rc_ = ws_staging(p, w)) return rc_;
  }
  return set_compressed(p, w, jpat, hpat, x, mult, w_obj, c, jac_c, hess_c, (cudaStream_t)stream);
}

int exa_eval_set_compressed_host(ExaPlan* p, ExaWorkspace* ws, const ExaPattern* jpat, const ExaPattern* hpat,
                                 const double* x, const double* mult, double w_obj, double* c, double* jac_c,
                                 double* hess_c, exa_stream_t stream) {
  if (!p) return fail("null plan");
  if (!jpat || !hpat) return fail("exa_eval_set_compressed_host: both patterns are required");
  DeviceGuard dguard(p->device);
  cudaStream_t st = (cudaStream_t)stream;
  ExaWorkspace* w = ws ? ws : p->dflt;
  {
    std::lock_guard<std::mutex> lazy(w->mu);
    if (int rc_ = ws_staging(p, w)) return rc_;
    if (w->cap_Jc < jpat->nnz) {
      cudaFree(w->dJc);
      w->dJc = nullptr;
      CU(cudaMalloc((void**)&w->dJc, (jpat->nnz > 0 ? jpat->nnz : 1) * sizeof(double)));
      w->cap_Jc = jpat->nnz;
    }
    if (w->cap_Hc < hpat->nnz) {
      cudaFree(w->dHc);
      w->dHc = nullptr;
      CU(cudaMalloc((void**)&w->dHc, (hpat->nnz > 0 ? hpat->nnz : 1) * sizeof(double)));
      w->cap_Hc = hpat->nnz;
    }
  }
  if (p->nvar) CU(cudaMemcpyAsync(w->dx, x, p->nvar * sizeof(double), cudaMemcpyHostToDevice, st));
  if (p->ncon) CU(cudaMemcpyAsync(w->dy, mult, p->ncon * sizeof(double), cudaMemcpyHostToDevice, st));
  if (int rc = set_compressed(p, w, jpat, hpat, w->dx, w->dy, w_obj, w->dc, w->dJc, w->dHc, st)) return rc;
  if (p->ncon) CU(cudaMemcpyAsync(c, w->dc, p->ncon * sizeof(double), cudaMemcpyDeviceToHost, st));
  if (jpat->nnz) CU(cudaMemcpyAsync(jac_c, w->dJc, jpat->nnz * sizeof(double), cudaMemcpyDeviceToHost, st));
  if (hpat->nnz) CU(cudaMemcpyAsync(hess_c, w->dHc, hpat->nnz * sizeof(double), cudaMemcpyDeviceToHost, st));
  if (pageable(c) || pageable(jac_c) || pageable(hess_c) || pageable(x) || pageable(mult))
    CU(cudaStreamSynchronize(st));  // pageable copies: complete on return
  return 0;
}

int exa_eval_cons(ExaPlan* p, ExaWorkspace* ws, const double* x, double* c, exa_stream_t stream) {
  EXA_PROLOGUE();
  A.x = x;
  A.c = c;
  return launch_mode(p, w, EXA_MODE_CONS, A, st);
}

int exa_eval_jac(ExaPlan* p, ExaWorkspace* ws, const double* x, double* jac, exa_stream_t stream) {
  EXA_PROLOGUE();
  A.x = x;
  A.J = jac;
  return launch_mode(p, w, EXA_MODE_JAC, A, st);
}

int exa_eval_hess(ExaPlan* p, ExaWorkspace* ws, const double* x, const double* mult, double w_obj,
                  double* hess, exa_stream_t stream) {
  EXA_PROLOGUE();
  A.x = x;
  A.y = mult;
  A.w = w_obj;
  A.H = hess;
  return launch_mode(p, w, EXA_MODE_HESS, A, st);
}

int exa_eval_obj(ExaPlan* p, ExaWorkspace* ws, const double* x, double* out, exa_stream_t stream) {
  EXA_PROLOGUE();
  A.x = x;
  A.V = w->V;
  int rc = launch_mode(p, w, EXA_MODE_OBJV, A, st);
  if (rc) return rc;
  const size_t smem = obj_dag_smem(p->n_onodes, p->n_olvl);
  if (p->obj_leaf_max <= EXA_OBJ_LEAF_MAX && smem <= EXA_OBJ_FUSED_SMEM_MAX && w->leafsum) {
    if (smem > 48 * 1024) {  // opt in once per device
      static std::mutex mu;
      static bool done[64] = {};
      std::lock_guard<std::mutex> lk(mu);
      if (p->device < 64 && !done[p->device]) {
        CU(cudaFuncSetAttribute(exa_obj_dag, cudaFuncAttributeMaxDynamicSharedMemorySize, EXA_OBJ_FUSED_SMEM_MAX));
        done[p->device] = true;
      }
    }
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = p->pdl ? 1 : 0;
    cudaLaunchConfig_t cfg = {};
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (p->n_leaves) {
      cfg.gridDim = dim3((unsigned)((p->n_leaves + EXA_OBJ_LEAF_WARPS - 1) / EXA_OBJ_LEAF_WARPS));
      cfg.blockDim = dim3(32 * EXA_OBJ_LEAF_WARPS);
      const double* V = w->V;
      void* a1[] = {(void*)&V, (void*)&p->leaves, (void*)&p->n_leaves, (void*)&w->leafsum};
      CU(cudaLaunchKernelExC(&cfg, (const void*)exa_obj_leaves2, a1));
    }
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(EXA_OBJ_THREADS);
    cfg.dynamicSmemBytes = smem;
    const double* ls = w->leafsum;
    void* a2[] = {(void*)&ls, (void*)&p->n_leaves, (void*)&p->onodes, (void*)&p->n_onodes, (void*)&p->oinit,
                  (void*)&p->olvl, (void*)&p->n_olvl, (void*)&out};
    CU(cudaLaunchKernelExC(&cfg, (const void*)exa_obj_dag, a2));
    return 0;
  }
  if (p->n_leaves) {
    exa_obj_leaves<<<grid_for(p->n_leaves, 128), 128, 0, st>>>(w->V, p->leaves, p->n_leaves, w->leafsum);
    CU(cudaGetLastError());
  }
  exa_obj_combine<<<1, 1, 0, st>>>(p->prog, p->n_prog, w->leafsum, out);
  CU(cudaGetLastError());
  return 0;
}

int exa_eval_grad(ExaPlan* p, ExaWorkspace* ws, const double* x, double* g, exa_stream_t stream) {
  EXA_PROLOGUE();
  A.x = x;
  A.G = w->G;
  int rc = launch_mode(p, w, EXA_MODE_GRAD, A, st);
  if (rc) return rc;
  if (p->nvar) {
    if (p->grad_ptr) {
      exa_grad_reduce<<<grid_for(p->nvar, 256), 256, 0, st>>>(p->nvar, p->grad_ptr, p->grad_ent, w->G, g);
      CU(cudaGetLastError());
    } else {
      CU(cudaMemsetAsync(g, 0, p->nvar * sizeof(double), st));
    }
  }
  return 0;
}

int exa_kkt_values(int64_t n, const int32_t* desc, const double* hvals, const double* jvals, const double* sigma,
                   double delta_w, double delta_c, double* out, exa_stream_t stream) {
  if (n < 0) return fail("exa_kkt_values: negative size");
  if (n == 0) return 0;
  if (!desc || !out || !sigma) return fail("exa_kkt_values: null argument");
  exa_kkt_kernel<<<grid_for((n + 3) / 4, 256), 256, 0, (cudaStream_t)stream>>>(
      n, reinterpret_cast<const int2*>(desc), hvals, jvals, sigma, delta_w, delta_c, out);
  CU(cudaGetLastError());
  return 0;
}

int exa_segment_sum(int64_t nnz, const int64_t* ptr, const int32_t* ent, const double* raw, double* out,
                    exa_stream_t stream) {
  if (nnz <= 0) return 0;
  if (!ptr || !ent || !raw || !out) return fail("exa_segment_sum: null argument");
  exa_compress_reduce<<<grid_for(nnz, 256), 256, 0, (cudaStream_t)stream>>>(nnz, ptr, ent, raw, out);
  CU(cudaGetLastError());
  return 0;
}

int exa_domain_error(ExaPlan* p, ExaWorkspace* ws, exa_stream_t stream, int64_t* rank, int32_t* instr,
                     int64_t* record) {
  if (!p) return fail("null plan");
  if (!p->has_checks) return 0;
  ExaWorkspace* w = ws ? ws : p->dflt;
  unsigned long long key = 0;
  CU(cudaMemcpyAsync(&key, w->err, sizeof key, cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  CU(cudaStreamSynchronize((cudaStream_t)stream));
  if (key == EXA_ERR_NONE) return 0;
  if (rank) *rank = (int64_t)(key >> 44);
  if (instr) *instr = (int32_t)((key >> 32) & 0xfff);
  if (record) *record = (int64_t)(key & 0xffffffffull) - 1;
  return 1;
}

int exa_device_sincos(const double* x, double* s, double* c, int64_t n, exa_stream_t stream) {
  if (n <= 0) return 0;
  exa_sincos_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(x, s, c, n);
  CU(cudaGetLastError());
  return 0;
}

}  // extern "C"
