// What can ONE launch moving one case13659 set's bytes (7 MB read, 18.8 MB
// written) achieve back to back in a CUDA graph?  Variants: naive 3-phase,
// interleaved vector loads/stores (many CTAs), persistent (148*k CTAs), and
// persistent + programmatic dependent launch (reads of immutable data before
// griddepcontrol.wait).  11 rotating replicas (> 2x L2).
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

// one "item" = 16 B read (if i < nin2) and 16*ratio B written
template <int PDL>
__global__ void __launch_bounds__(256) inter_k(const double2* __restrict__ in, long long nin2, double2* __restrict__ out,
                                               long long nout2) {
  if (PDL) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  // reads first (immutable inputs), kept in registers
  double2 acc = make_double2(0, 0);
  double2 v[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    long long k = tid + u * nt;
    v[u] = k < nin2 ? __ldg(in + k) : make_double2(0, 0);
  }
  for (long long k = tid + 4 * nt; k < nin2; k += nt) { double2 a = __ldg(in + k); acc.x += a.x; acc.y += a.y; }
  if (PDL) asm volatile("griddepcontrol.wait;" ::: "memory");
#pragma unroll
  for (int u = 0; u < 4; ++u) { acc.x += v[u].x; acc.y += v[u].y; }
  for (long long k = tid; k < nout2; k += nt) out[k] = acc;
}

__global__ void naive_k(const double* __restrict__ in, long long nin, double* __restrict__ out, long long nout) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  long long stride = (long long)gridDim.x * blockDim.x;
  double acc = 0;
  for (long long k = i; k < nin; k += stride) acc += __ldg(in + k);
  for (long long k = i; k < nout; k += stride) out[k] = acc;
}

__global__ void empty_k() {}

int main() {
  const long long nin = 7000000 / 8, nout = 18800000 / 8;
  const int R = 11;
  std::vector<double*> ins(R), outs(R);
  for (int r = 0; r < R; ++r) {
    CK(cudaMalloc(&ins[r], nin * 8)); cudaMemset(ins[r], 0, nin * 8);
    CK(cudaMalloc(&outs[r], nout * 8));
  }
  cudaStream_t s; cudaStreamCreate(&s);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto launch) {
    cudaGraph_t g; cudaGraphExec_t ge;
    const int S = 64 * R;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < S; ++i) launch(i % R);
    cudaStreamEndCapture(s, &g);
    if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) { printf("%s: instantiate failed\n", name); return; }
    cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
    cudaEventRecord(e0, s);
    for (int rep = 0; rep < 5; ++rep) cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double us = ms * 1e3 / (5.0 * S);
    printf("%-40s %6.2f us/launch  %6.0f GB/s\n", name, us, (nin + nout) * 8 / us / 1e3);
    cudaGraphExecDestroy(ge); cudaGraphDestroy(g);
    cudaError_t e = cudaGetLastError(); if (e) printf("err %s\n", cudaGetErrorString(e));
  };
  timeit("empty 1 CTA", [&](int r) { empty_k<<<1, 32, 0, s>>>(); });
  timeit("empty 5463x64", [&](int r) { empty_k<<<5463, 64, 0, s>>>(); });
  timeit("empty 1184x256", [&](int r) { empty_k<<<1184, 256, 0, s>>>(); });
  for (int blocks : {1529, 148 * 8}) {
    char nm[64]; snprintf(nm, 64, "naive grid %d", blocks);
    timeit(nm, [&](int r) { naive_k<<<blocks, 256, 0, s>>>(ins[r], nin, outs[r], nout); });
  }
  for (int blocks : {148 * 2, 148 * 4, 148 * 8, 2296, 4592}) {
    char nm[64]; snprintf(nm, 64, "interleaved grid %d", blocks);
    timeit(nm, [&](int r) { inter_k<0><<<blocks, 256, 0, s>>>((const double2*)ins[r], nin / 2, (double2*)outs[r], nout / 2); });
    snprintf(nm, 64, "interleaved+PDL grid %d", blocks);
    timeit(nm, [&](int r) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = blocks; cfg.blockDim = 256; cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, inter_k<1>, (const double2*)ins[r], nin / 2, (double2*)outs[r], nout / 2);
    });
  }
  // big copy for reference
  {
    double *a, *b; long long n = 1ll << 28;
    cudaMalloc(&a, n * 8); cudaMalloc(&b, n * 8);
    cudaMemcpyAsync(b, a, n * 8, cudaMemcpyDeviceToDevice, s);
    cudaEventRecord(e0, s);
    for (int i = 0; i < 5; ++i) cudaMemcpyAsync(b, a, n * 8, cudaMemcpyDeviceToDevice, s);
    cudaEventRecord(e1, s); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("memcpy 2 GiB: %.0f GB/s (r+w)\n", 2.0 * n * 8 * 5 / (ms * 1e-3) / 1e9);
  }
  return 0;
}
