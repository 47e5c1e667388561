// Memory-system rates that bound the set kernel: random 8-byte gathers from
// an L2-resident 1 MB array (through L1 / bypassing L1), scattered 8-byte
// stores, coalesced stores.  Each config: mean of 50 back-to-back launches.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

template <int K, bool CG>
__global__ void __launch_bounds__(256) gather_k(const double* __restrict__ x, const int* __restrict__ idx, long long n,
                                                double* __restrict__ out) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  int id[K];
#pragma unroll
  for (int k = 0; k < K; ++k) id[k] = __ldg(idx + k * n + t);
  double acc = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) acc += CG ? __ldcg(x + id[k]) : __ldg(x + id[k]);
  out[t] = acc;
}

template <int K>
__global__ void __launch_bounds__(256) scatter_k(const int* __restrict__ idx, long long n, double* __restrict__ out) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
#pragma unroll
  for (int k = 0; k < K; ++k) out[__ldg(idx + k * n + t)] = (double)t;
}

__global__ void __launch_bounds__(256) stream_st(long long n, double* __restrict__ out) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (long long i = t; i < n; i += (long long)gridDim.x * blockDim.x) out[i] = (double)i;
}

__global__ void empty_k() {}

int main() {
  const int nx = 1 << 17;  // 1 MB of doubles
  double* x; cudaMalloc(&x, nx * 8); cudaMemset(x, 0, nx * 8);
  const long long NT = 148LL * 2048 * 2;  // threads
  const int KMAX = 8;
  std::vector<int> h(NT * KMAX);
  for (auto& v : h) v = rand() % nx;
  int* idx; cudaMalloc(&idx, h.size() * 4); cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  const long long NS = 20000000 / 8;  // 20 MB scatter target
  std::vector<int> hs(NT * KMAX);
  for (auto& v : hs) v = rand() % NS;
  int* sidx; cudaMalloc(&sidx, hs.size() * 4); cudaMemcpy(sidx, hs.data(), hs.size() * 4, cudaMemcpyHostToDevice);
  double* out; cudaMalloc(&out, NS * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto T = [&](const char* name, double units, auto launch) {
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int i = 0; i < 50; ++i) launch();
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double us = ms * 1e3 / 50;
    printf("%-44s %8.2f us  %8.1f G units/s\n", name, us, units / us / 1e3);
  };
  T("empty", 1, [&] { empty_k<<<1, 32>>>(); });
  for (long long nt : {NT / 8, NT / 2, NT}) {
    int grid = (int)((nt + 255) / 256);
    char b[80];
    snprintf(b, 80, "gather K=1 ldg  threads=%lld", nt); T(b, nt * 1.0, [&] { gather_k<1, false><<<grid, 256>>>(x, idx, nt, out); });
    snprintf(b, 80, "gather K=4 ldg  threads=%lld", nt); T(b, nt * 4.0, [&] { gather_k<4, false><<<grid, 256>>>(x, idx, nt, out); });
    snprintf(b, 80, "gather K=8 ldg  threads=%lld", nt); T(b, nt * 8.0, [&] { gather_k<8, false><<<grid, 256>>>(x, idx, nt, out); });
    snprintf(b, 80, "gather K=8 ldcg threads=%lld", nt); T(b, nt * 8.0, [&] { gather_k<8, true><<<grid, 256>>>(x, idx, nt, out); });
    snprintf(b, 80, "scatter K=1 threads=%lld", nt); T(b, nt * 1.0, [&] { scatter_k<1><<<grid, 256>>>(sidx, nt, out); });
    snprintf(b, 80, "scatter K=4 threads=%lld", nt); T(b, nt * 4.0, [&] { scatter_k<4><<<grid, 256>>>(sidx, nt, out); });
  }
  T("stream store 18.8 MB (G doubles)", 18.8e6 / 8, [&] { stream_st<<<148 * 8, 256>>>(18800000 / 8, out); });
  return 0;
}
