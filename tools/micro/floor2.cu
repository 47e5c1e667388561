// Floor with gathers: per launch, read 7 MB + write 18.8 MB coalesced AND do
// G random 8-byte gathers from a 1 MB (x-sized) array -- the access mix of one
// case13659 callback set.  CUDA graph of back-to-back launches, 11 rotating sets.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
__global__ void mix_k(const double* __restrict__ in, long long nin, double* __restrict__ out, long long nout,
                      const double* __restrict__ x, const int* __restrict__ idx, long long ng) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  long long stride = (long long)gridDim.x * blockDim.x;
  double acc = 0;
  for (long long k = i; k < nin; k += stride) acc += __ldg(in + k);
  for (long long k = i; k < ng; k += stride) acc += __ldg(x + __ldg(idx + k));
  for (long long k = i; k < nout; k += stride) out[k] = acc;
}
int main() {
  const long long nin = 7000000 / 8, nout = 18800000 / 8, nx = 1000000 / 8;
  const int R = 11;
  std::vector<double*> ins(R), outs(R), xs(R);
  std::vector<int*> idxs(R);
  for (long long ng : {0LL, 250000LL, 565000LL, 1000000LL}) {
    for (int r = 0; r < R; ++r) {
      cudaMalloc(&ins[r], nin * 8); cudaMemset(ins[r], 0, nin * 8);
      cudaMalloc(&outs[r], nout * 8);
      cudaMalloc(&xs[r], nx * 8); cudaMemset(xs[r], 0, nx * 8);
      std::vector<int> h(ng > 0 ? ng : 1);
      for (auto& v : h) v = rand() % nx;
      cudaMalloc(&idxs[r], h.size() * 4); cudaMemcpy(idxs[r], h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    }
    cudaStream_t s; cudaStreamCreate(&s);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int blocks : {148 * 8, 1529}) {
      cudaGraph_t g; cudaGraphExec_t ge;
      const int S = 64 * R;
      cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
      for (int i = 0; i < S; ++i)
        mix_k<<<blocks, 256, 0, s>>>(ins[i % R], nin, outs[i % R], nout, xs[i % R], idxs[i % R], ng);
      cudaStreamEndCapture(s, &g);
      cudaGraphInstantiate(&ge, g, 0);
      cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
      cudaEventRecord(e0, s);
      for (int rep = 0; rep < 3; ++rep) cudaGraphLaunch(ge, s);
      cudaEventRecord(e1, s); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("gathers %7lld grid %5d: %.2f us per launch\n", ng, blocks, ms * 1e3 / (3.0 * S));
      cudaGraphExecDestroy(ge); cudaGraphDestroy(g);
    }
    for (int r = 0; r < R; ++r) { cudaFree(ins[r]); cudaFree(outs[r]); cudaFree(xs[r]); cudaFree(idxs[r]); }
  }
  return 0;
}
