// SM stores into mapped page-locked host memory (the host path's D2H of one
// case13659 set: 11.66 MB in 20 ranges): store width x chunk size x threads,
// against one DMA of the same bytes, and a DMA + store-kernel split.
// nvcc -O3 -std=c++17 -cudart shared -gencode arch=compute_100a,code=sm_100a -o d2hstore d2hstore.cu
#include <chrono>
#include <cstdio>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>

static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
struct Ch { long long a, e; };

template <int W>  // bytes per thread access: 8, 16, 32
__global__ void st(const Ch* __restrict__ ch, const double* __restrict__ src, double* dst) {
  const Ch q = ch[blockIdx.x];
  constexpr int D = W / 8;
  long long a = q.a;  // chunks are 32-byte aligned in this test
  const long long nv = (q.e - a) / D;
  for (long long i = threadIdx.x; i < nv; i += blockDim.x) {
    const double* s = src + a + i * D;
    double* d = dst + a + i * D;
    if (W == 8) *d = __ldcs(s);
    if (W == 16) *reinterpret_cast<double2*>(d) = __ldcs(reinterpret_cast<const double2*>(s));
    if (W == 32) {
      double x0, x1, x2, x3;
      asm volatile("ld.global.cs.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(x0), "=d"(x1), "=d"(x2), "=d"(x3) : "l"(s));
      asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(d), "d"(x0), "d"(x1), "d"(x2), "d"(x3) : "memory");
    }
  }
}

int main() {
  const long long total = 18800000 / 8, n = 11660000 / 8;
  const int NR = 20, reps = 100, R = 3;
  double* dev;
  cudaMalloc(&dev, total * 8);
  cudaMemset(dev, 0, total * 8);
  std::vector<double*> host(R);
  for (auto& h : host) { cudaHostAlloc(&h, total * 8, cudaHostAllocDefault); memset(h, 1, total * 8); }
  cudaStream_t s, s2;
  cudaStreamCreate(&s);
  cudaStreamCreate(&s2);
  const long long step = (total / NR) & ~3LL, len = (n / NR) & ~3LL;
  {
    double t0 = now();
    for (int i = 0; i < reps; ++i) cudaMemcpyAsync(host[i % R], dev, NR * len * 8, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    double dt = now() - t0;
    printf("one DMA %.2f MB: %.1f GB/s %.1f us\n", NR * len * 8 / 1e6, NR * len * 8.0 * reps / dt / 1e9, dt / reps * 1e6);
  }
  for (int chunk : {1024, 2048, 4096, 8192, 16384}) {
    std::vector<Ch> ch;
    for (int r = 0; r < NR; ++r)
      for (long long o = 0; o < len; o += chunk) ch.push_back({r * step + o, r * step + std::min(len, o + chunk)});
    Ch* dch;
    cudaMalloc(&dch, ch.size() * sizeof(Ch));
    cudaMemcpy(dch, ch.data(), ch.size() * sizeof(Ch), cudaMemcpyHostToDevice);
    for (int th : {64, 128, 256, 512}) {
      for (int W : {8, 16, 32}) {
        auto launch = [&](int i) {
          if (W == 8) st<8><<<ch.size(), th, 0, s>>>(dch, dev, host[i % R]);
          if (W == 16) st<16><<<ch.size(), th, 0, s>>>(dch, dev, host[i % R]);
          if (W == 32) st<32><<<ch.size(), th, 0, s>>>(dch, dev, host[i % R]);
        };
        for (int i = 0; i < 3; ++i) launch(i);
        cudaStreamSynchronize(s);
        double t0 = now();
        for (int i = 0; i < reps; ++i) launch(i);
        cudaStreamSynchronize(s);
        double dt = now() - t0;
        printf("store W=%2d chunk=%5d th=%3d CTAs=%5zu: %.1f GB/s %.1f us\n", W, chunk, th, ch.size(),
               NR * len * 8.0 * reps / dt / 1e9, dt / reps * 1e6);
      }
    }
    cudaFree(dch);
  }
  // split: the first K ranges by DMA on s2, the rest by a W=16 store kernel on s
  for (int K : {2, 5, 10}) {
    std::vector<Ch> ch;
    for (int r = K; r < NR; ++r)
      for (long long o = 0; o < len; o += 4096) ch.push_back({r * step + o, r * step + std::min(len, o + 4096)});
    Ch* dch;
    cudaMalloc(&dch, ch.size() * sizeof(Ch));
    cudaMemcpy(dch, ch.data(), ch.size() * sizeof(Ch), cudaMemcpyHostToDevice);
    double t0 = now();
    for (int i = 0; i < reps; ++i) {
      for (int r = 0; r < K; ++r) cudaMemcpyAsync(host[i % R] + r * step, dev + r * step, len * 8, cudaMemcpyDeviceToHost, s2);
      st<16><<<ch.size(), 256, 0, s>>>(dch, dev, host[i % R]);
    }
    cudaDeviceSynchronize();
    double dt = now() - t0;
    printf("split K=%2d DMA ranges + store kernel: %.1f GB/s %.1f us\n", K, NR * len * 8.0 * reps / dt / 1e9, dt / reps * 1e6);
    cudaFree(dch);
  }
  // per-range DMAs spread over S streams (fork / join with events): the copy
  // engines overlap each other's per-transfer latency
  for (int S : {1, 2, 3, 4, 6}) {
    std::vector<cudaStream_t> ss(S);
    for (auto& q : ss) cudaStreamCreateWithFlags(&q, cudaStreamNonBlocking);
    cudaEvent_t fork, join[8];
    cudaEventCreateWithFlags(&fork, cudaEventDisableTiming);
    for (int k = 0; k < S; ++k) cudaEventCreateWithFlags(&join[k], cudaEventDisableTiming);
    double t0 = now(), iss = 0;
    for (int i = 0; i < reps; ++i) {
      double a = now();
      cudaEventRecord(fork, s);
      for (int k = 0; k < S; ++k) cudaStreamWaitEvent(ss[k], fork, 0);
      for (int r = 0; r < NR; ++r)
        cudaMemcpyAsync(host[i % R] + r * step, dev + r * step, len * 8, cudaMemcpyDeviceToHost, ss[r % S]);
      for (int k = 0; k < S; ++k) { cudaEventRecord(join[k], ss[k]); cudaStreamWaitEvent(s, join[k], 0); }
      iss += now() - a;
      if (i % 3 == 2) cudaStreamSynchronize(s);  // keep the queues short (a caller syncs per set)
    }
    cudaStreamSynchronize(s);
    double dt = now() - t0;
    printf("DMA %d ranges over %d streams: %.1f GB/s %.1f us, issue %.1f us per set\n", NR, S, NR * len * 8.0 * reps / dt / 1e9,
           dt / reps * 1e6, iss / reps * 1e6);
  }
  // 2D copies: the 20 ranges as ONE 2D copy (equal lengths, constant stride)
  {
    double t0 = now(), iss = 0;
    for (int i = 0; i < reps; ++i) {
      double a = now();
      cudaMemcpy2DAsync(host[i % R], step * 8, dev, step * 8, len * 8, NR, cudaMemcpyDeviceToHost, s);
      iss += now() - a;
    }
    cudaStreamSynchronize(s);
    double dt = now() - t0;
    printf("one 2D DMA of %d rows: %.1f GB/s %.1f us, issue %.1f us per set\n", NR, NR * len * 8.0 * reps / dt / 1e9,
           dt / reps * 1e6, iss / reps * 1e6);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
