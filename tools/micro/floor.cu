// Floor for one-launch-per-set: CUDA graph of back-to-back launches of
// (a) an empty kernel, (b) a pure streaming kernel moving the same bytes as one
// case13659 callback set (7 MB read, 18.8 MB written), rotating 11 buffers.
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
__global__ void empty_k() {}
__global__ void stream_k(const double* __restrict__ in, long long nin, double* __restrict__ out, long long nout) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  long long stride = (long long)gridDim.x * blockDim.x;
  double acc = 0;
  for (long long k = i; k < nin; k += stride) acc += __ldg(in + k);
  for (long long k = i; k < nout; k += stride) out[k] = acc;
}
int main() {
  const long long nin = 7000000 / 8, nout = 18800000 / 8;
  const int R = 11;
  std::vector<double*> ins(R), outs(R);
  for (int r = 0; r < R; ++r) { cudaMalloc(&ins[r], nin * 8); cudaMemset(ins[r], 0, nin * 8); cudaMalloc(&outs[r], nout * 8); }
  cudaStream_t s; cudaStreamCreate(&s);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int variant = 0; variant < 5; ++variant) {
    int blocks = (variant == 0) ? 1529 : (variant == 1 ? 148 * 4 : (variant == 2 ? 148 * 8 : (variant == 3 ? 1529 : 148 * 16)));
    int threads = 256;
    cudaGraph_t g; cudaGraphExec_t ge;
    const int S = 64 * R;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < S; ++i) {
      if (variant == 0) empty_k<<<blocks, threads, 0, s>>>();
      else stream_k<<<blocks, threads, 0, s>>>(ins[i % R], nin, outs[i % R], nout);
    }
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
    cudaEventRecord(e0, s);
    for (int rep = 0; rep < 3; ++rep) cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double us = ms * 1e3 / (3.0 * S);
    printf("%s grid %d: %.2f us per launch  (%.0f GB/s for 25.8 MB)\n", variant == 0 ? "empty " : "stream", blocks, us,
           variant == 0 ? 0.0 : 25.8e6 / (us * 1e-6) / 1e9);
    cudaGraphExecDestroy(ge); cudaGraphDestroy(g);
  }
  return 0;
}
