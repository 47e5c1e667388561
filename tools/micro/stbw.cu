// Per-SM global store / load throughput microbenchmark (B200).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void st64(double* __restrict__ out, long long n_per_thread, long long stride) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  #pragma unroll 4
  for (long long k = 0; k < n_per_thread; ++k) out[i + k * stride] = (double)k;
}
__global__ void st128(double2* __restrict__ out, long long n_per_thread, long long stride) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  #pragma unroll 4
  for (long long k = 0; k < n_per_thread; ++k) out[i + k * stride] = make_double2(k, k);
}
__global__ void ld64(const double* __restrict__ in, double* out, long long n_per_thread, long long stride) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  double acc = 0;
  #pragma unroll 8
  for (long long k = 0; k < n_per_thread; ++k) acc += __ldg(in + i + k * stride);
  if (acc == 12345.678) out[0] = acc;
}
int main() {
  const long long N = 1LL << 24;  // 16M doubles = 128 MB
  double* buf; cudaMalloc(&buf, N * 8 * 2);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = 148;
  for (int blocks_per_sm : {1, 2, 4, 8}) {
    int threads = 256, blocks = sms * blocks_per_sm;
    long long total_threads = (long long)threads * blocks;
    for (long long bytes_target : {8LL << 20, 32LL << 20}) {
      long long npt = bytes_target / 8 / total_threads;
      if (npt < 1) npt = 1;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        st64<<<blocks, threads>>>(buf, npt, total_threads);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
      }
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double bytes = 8.0 * npt * total_threads;
      printf("STG.64  %d CTA/SM, %6.1f MB: %7.2f us  %7.1f GB/s  %5.1f B/clk/SM\n", blocks_per_sm, bytes / 1e6, ms * 1e3,
             bytes / ms / 1e6, bytes / (ms * 1e-3) / 1.965e9 / sms);
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        st128<<<blocks, threads>>>((double2*)buf, (npt + 1) / 2, total_threads);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
      }
      cudaEventElapsedTime(&ms, e0, e1);
      bytes = 16.0 * ((npt + 1) / 2) * total_threads;
      printf("STG.128 %d CTA/SM, %6.1f MB: %7.2f us  %7.1f GB/s  %5.1f B/clk/SM\n", blocks_per_sm, bytes / 1e6, ms * 1e3,
             bytes / ms / 1e6, bytes / (ms * 1e-3) / 1.965e9 / sms);
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        ld64<<<blocks, threads>>>(buf, buf + N, npt, total_threads);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
      }
      cudaEventElapsedTime(&ms, e0, e1);
      bytes = 8.0 * npt * total_threads;
      printf("LDG.64  %d CTA/SM, %6.1f MB: %7.2f us  %7.1f GB/s  %5.1f B/clk/SM\n", blocks_per_sm, bytes / 1e6, ms * 1e3,
             bytes / ms / 1e6, bytes / (ms * 1e-3) / 1.965e9 / sms);
    }
  }
  // empty kernel launch cost
  for (int rep = 0; rep < 3; ++rep) { cudaEventRecord(e0); st64<<<sms * 8, 256>>>(buf, 0, 1); cudaEventRecord(e1); cudaEventSynchronize(e1); }
  float ms; cudaEventElapsedTime(&ms, e0, e1); printf("empty 1184-CTA kernel: %.2f us\n", ms * 1e3);
  return 0;
}
