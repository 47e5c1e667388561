// FP64 latency / throughput microbenchmark (B200): dependent DFMA/DADD chains.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat_fma(double* out, double a, double b, int n, long long* cyc) {
  double x = out[threadIdx.x];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = fma(x, a, b); x = fma(x, a, b); x = fma(x, a, b); x = fma(x, a, b); }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat_add(double* out, double a, int n, long long* cyc) {
  double x = out[threadIdx.x];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = x + a; x = x - a; x = x + a; x = x - a; }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void thr_fma(double* out, double a, double b, int n, long long* cyc) {
  double x0 = out[threadIdx.x], x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
    x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
  }
  long long t1 = clock64();
  out[threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void lat_ldg(const long long* __restrict__ chain, int n, long long* cyc, long long* sink) {
  long long p = 0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) p = chain[p];
  long long t1 = clock64();
  sink[0] = p;
  cyc[0] = t1 - t0;
}
int main() {
  double* d; long long* c; long long h[64];
  cudaMalloc(&d, 1024 * 8); cudaMemset(d, 0, 1024 * 8); cudaMalloc(&c, 64 * 8);
  int n = 10000;
  lat_fma<<<1, 1>>>(d, 0.999, 1e-3, n, c); cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
  lat_fma<<<1, 1>>>(d, 0.999, 1e-3, n, c); cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cycles\n", h[0] / (4.0 * n));
  lat_add<<<1, 1>>>(d, 0.5, n, c); cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
  lat_add<<<1, 1>>>(d, 0.5, n, c); cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
  printf("DADD dependent latency: %.2f cycles\n", h[0] / (4.0 * n));
  for (int warps = 1; warps <= 32; warps *= 2) {
    thr_fma<<<1, 32 * warps>>>(d, 0.999, 1e-3, n, c); cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
    thr_fma<<<1, 32 * warps>>>(d, 0.999, 1e-3, n, c); cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
    double per = h[0] / (8.0 * n);
    printf("DFMA 8-chain, %2d warps/SM: %.2f cycles per warp-iteration step -> %.1f DFMA/clk/SM\n",
           warps, per, 32.0 * warps / per);
  }
  // pointer chase for L2 / DRAM latency
  const long long N = 1 << 24;  // 128 MB
  long long* chain; cudaMalloc(&chain, N * 8);
  long long* hc = (long long*)malloc(N * 8);
  for (long long s : {1LL << 10, 1LL << 16, 1LL << 24}) {
    long long stride = 4099;  // pseudo-random walk within s elements
    for (long long i = 0; i < s; ++i) hc[i] = (i + stride * 16 + 7) % s;
    cudaMemcpy(chain, hc, s * 8, cudaMemcpyHostToDevice);
    lat_ldg<<<1, 1>>>(chain, 2000, c, c + 8); cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
    lat_ldg<<<1, 1>>>(chain, 2000, c, c + 8); cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
    printf("pointer chase over %lld KB: %.1f cycles per load\n", s * 8 / 1024, h[0] / 2000.0);
  }
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0); printf("clock %d kHz\n", clk);
  return 0;
}
