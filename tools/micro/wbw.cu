// Write bandwidth into HBM through L2 for one set's output volume (18.8 MB per
// launch, 11 rotating buffers > L2), by allocation kind: cudaMalloc vs
// cuMemCreate without / with generic compression.  Graph of 64 launches.
#include <cstdio>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>
#define CK(x) do { auto e_ = (x); if (e_ != 0) { printf("%s:%d err %d\n", __FILE__, __LINE__, (int)e_); return 1; } } while (0)

__global__ void __launch_bounds__(256) wr(double* __restrict__ out, long long n, double seed, int zeros) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  long long st = (long long)gridDim.x * blockDim.x;
  // zeros: the second half of every 64 KB block is 0.0 (like the structural-zero Hessian columns)
  for (long long i = t; i < n; i += st)
    out[i] = (zeros && (i & 8191) >= 4096) ? 0.0 : seed * (double)(i ^ 0x5bd1e995) + 0.1234567;
}
__global__ void __launch_bounds__(256) rw(const double* __restrict__ in, long long nin, double* __restrict__ out, long long n) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  long long st = (long long)gridDim.x * blockDim.x;
  double acc = 0;
  for (long long i = t; i < nin; i += st) acc += __ldg(in + i);
  for (long long i = t; i < n; i += st) out[i] = acc * (double)(i ^ 0x5bd1e995) + 0.1234567;
}

static int alloc_vmm(double** p, size_t bytes, int comp) {
  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = 0;
  prop.allocFlags.compressionType = comp ? CU_MEM_ALLOCATION_COMP_GENERIC : CU_MEM_ALLOCATION_COMP_NONE;
  size_t gran = 0;
  CK(cuMemGetAllocationGranularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  size_t sz = (bytes + gran - 1) / gran * gran;
  CUmemGenericAllocationHandle h;
  CK(cuMemCreate(&h, sz, &prop, 0));
  CUdeviceptr d;
  CK(cuMemAddressReserve(&d, sz, 0, 0, 0));
  CK(cuMemMap(d, sz, 0, h, 0));
  CUmemAccessDesc acc = {};
  acc.location = prop.location;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(d, sz, &acc, 1));
  *p = (double*)d;
  return 0;
}

int main() {
  cudaFree(0);
  const long long n = 18800000 / 8, nin = 7000000 / 8;
  const int R = 11;
  cudaStream_t s; cudaStreamCreate(&s);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  double* in[R];
  for (int r = 0; r < R; ++r) { cudaMalloc(&in[r], nin * 8); cudaMemset(in[r], 0, nin * 8); }
  for (int kind = 0; kind < 3; ++kind) {
    std::vector<double*> b(R);
    for (int r = 0; r < R; ++r) {
      if (kind == 0) CK(cudaMalloc(&b[r], n * 8));
      else if (alloc_vmm(&b[r], n * 8, kind == 2)) return 1;
    }
    for (int mode = 0; mode < 3; ++mode) {
      cudaGraph_t g; cudaGraphExec_t ge;
      cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
      for (int i = 0; i < 64 * R; ++i) {
        if (mode == 0) wr<<<148 * 8, 256, 0, s>>>(b[i % R], n, 1.0 + i, 0);
        else if (mode == 2) wr<<<148 * 8, 256, 0, s>>>(b[i % R], n, 1.0 + i, 1);
        else rw<<<148 * 8, 256, 0, s>>>(in[i % R], nin, b[i % R], n);
      }
      cudaStreamEndCapture(s, &g);
      cudaGraphInstantiate(&ge, g, 0);
      cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
      cudaEventRecord(e0, s);
      for (int k = 0; k < 3; ++k) cudaGraphLaunch(ge, s);
      cudaEventRecord(e1, s); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double us = ms * 1e3 / (3.0 * 64 * R);
      double bytes = n * 8.0 + (mode == 1 ? nin * 8.0 : 0);
      printf("%-28s %-14s %6.2f us/launch  %6.0f GB/s\n", kind == 0 ? "cudaMalloc" : (kind == 1 ? "cuMemCreate COMP_NONE" : "cuMemCreate COMP_GENERIC"),
             mode == 1 ? "read7+write19" : (mode == 2 ? "write 18.8MB 50% 0" : "write 18.8MB"), us, bytes / us / 1e3);
      cudaGraphExecDestroy(ge); cudaGraphDestroy(g);
    }
    CUmemAllocationProp pr = {};
  }
  return 0;
}
