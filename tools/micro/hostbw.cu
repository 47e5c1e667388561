// Host-side limits of the host-buffer callback path (exa_eval_set_host):
// pinned D2H bandwidth for one set's copied bytes as one DMA, as per-range
// DMAs (CPU issue cost), and as a kernel storing straight into the mapped
// pinned buffer; host fill / negate-copy throughput with T threads; both at once.
// nvcc -O3 -std=c++17 -cudart shared -gencode arch=compute_100a,code=sm_100a -o hostbw hostbw.cu
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>
#include <cuda_runtime.h>

static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

// T threads each write their share of n doubles: memset (neg = 0) or dst = -src (neg = 1)
static void host_pass(double* dst, const double* src, int64_t n, int T, int neg) {
  std::vector<std::thread> th;
  for (int t = 0; t < T; ++t)
    th.emplace_back([=] {
      int64_t a = n * t / T, b = n * (t + 1) / T;
      if (!neg) std::memset(dst + a, 0, (b - a) * 8);
      else for (int64_t i = a; i < b; ++i) dst[i] = -src[i];
    });
  for (auto& x : th) x.join();
}

struct Rg { int64_t off, n; };
// ranges copied device -> mapped host memory: CTA b takes 2048-double chunks of the
// concatenated ranges; 16-byte stores when dst / src are 16-byte aligned
__global__ void __launch_bounds__(256) to_host(const Rg* __restrict__ rg, int nr, const int64_t* __restrict__ chunk0,
                                               const double* __restrict__ src, double* dst) {
  // find the range of this CTA's chunk (few ranges: linear scan)
  int r = 0;
  while (r + 1 < nr && chunk0[r + 1] <= blockIdx.x) ++r;
  const int64_t c = blockIdx.x - chunk0[r];
  const int64_t a = rg[r].off + c * 2048, e = min(rg[r].off + rg[r].n, a + 2048);
  for (int64_t i = a + threadIdx.x; i < e; i += blockDim.x) dst[i] = __ldg(src + i);
}

int main() {
  const int64_t out_n = 18800000 / 8, d2h_full = 11660000 / 8, d2h_dedup = 8060000 / 8, fill_n = 7200000 / 8,
                neg_n = 3600000 / 8;
  const int R = 3, reps = 200, NRG = 24;
  double* dev;
  cudaMalloc(&dev, out_n * 8);
  cudaMemset(dev, 0, out_n * 8);
  std::vector<double*> host(R);
  for (auto& h : host) { cudaHostAlloc(&h, out_n * 8, cudaHostAllocDefault); std::memset(h, 1, out_n * 8); }
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int64_t n : {d2h_full, d2h_dedup}) {
    for (int i = 0; i < 5; ++i) cudaMemcpyAsync(host[i % R], dev, n * 8, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    double t0 = now();
    for (int i = 0; i < reps; ++i) cudaMemcpyAsync(host[i % R], dev, n * 8, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    double dt = now() - t0;
    printf("D2H one DMA %.2f MB: %.1f GB/s, %.1f us per set\n", n * 8 / 1e6, n * 8.0 * reps / dt / 1e9, dt / reps * 1e6);
    // NRG ranges with gaps (every other 1/(2 NRG) of the output)
    std::vector<Rg> rg;
    const int64_t step = out_n / NRG, len = n / NRG;
    for (int k = 0; k < NRG; ++k) rg.push_back({k * step, len});
    double issue = 0;
    t0 = now();
    for (int i = 0; i < reps; ++i) {
      double a = now();
      for (auto& q : rg) cudaMemcpyAsync(host[i % R] + q.off, dev + q.off, q.n * 8, cudaMemcpyDeviceToHost, s);
      issue += now() - a;
    }
    cudaStreamSynchronize(s);
    dt = now() - t0;
    printf("D2H %d DMAs %.2f MB: %.1f GB/s, %.1f us per set, CPU issue %.1f us per set\n", NRG, n * 8 / 1e6,
           n * 8.0 * reps / dt / 1e9, dt / reps * 1e6, issue / reps * 1e6);
    // kernel stores into mapped pinned memory
    std::vector<int64_t> c0(NRG + 1, 0);
    for (int k = 0; k < NRG; ++k) c0[k + 1] = c0[k] + (rg[k].n + 2047) / 2048;
    Rg* drg;
    int64_t* dc0;
    cudaMalloc(&drg, NRG * sizeof(Rg));
    cudaMalloc(&dc0, (NRG + 1) * 8);
    cudaMemcpy(drg, rg.data(), NRG * sizeof(Rg), cudaMemcpyHostToDevice);
    cudaMemcpy(dc0, c0.data(), (NRG + 1) * 8, cudaMemcpyHostToDevice);
    for (int th : {128, 256}) {
      for (int i = 0; i < 3; ++i) to_host<<<c0[NRG], th, 0, s>>>(drg, NRG, dc0, dev, host[i % R]);
      cudaStreamSynchronize(s);
      cudaEventRecord(e0, s);
      t0 = now();
      for (int i = 0; i < reps; ++i) to_host<<<c0[NRG], th, 0, s>>>(drg, NRG, dc0, dev, host[i % R]);
      cudaEventRecord(e1, s);
      cudaStreamSynchronize(s);
      dt = now() - t0;
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("kernel -> mapped host %.2f MB (%lld CTAs x %d): %.1f GB/s, %.1f us per set (events %.1f us)  err=%s\n",
             n * 8 / 1e6, (long long)c0[NRG], th, n * 8.0 * reps / dt / 1e9, dt / reps * 1e6, ms * 1e3 / reps,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  for (int T : {1, 2, 4, 8, 12, 16}) {
    for (int neg = 0; neg < 2; ++neg) {
      int64_t n = neg ? neg_n : fill_n;
      double t0 = now();
      for (int i = 0; i < 50; ++i) host_pass(host[i % R] + (neg ? fill_n : 0), host[(i + 1) % R], n, T, neg);
      double dt = now() - t0;
      printf("host %s %.2f MB, %2d threads: %.1f GB/s written, %.1f us per set\n", neg ? "negate-copy" : "memset", n * 8 / 1e6,
             T, n * 8.0 * 50 / dt / 1e9, dt / 50 * 1e6);
    }
  }
  // concurrent: D2H stream running while T threads fill (+ negate)
  for (int T : {4, 8}) {
    for (int64_t n : {d2h_full, d2h_dedup}) {
      std::atomic<bool> stop{false};
      std::atomic<int64_t> sets{0};
      std::thread filler([&] {
        int i = 0;
        while (!stop.load()) {
          host_pass(host[i % R], nullptr, fill_n, T, 0);
          if (n == d2h_dedup) host_pass(host[i % R] + fill_n, host[(i + 1) % R] + fill_n, neg_n, T, 1);
          ++i;
          sets.fetch_add(1);
        }
      });
      double t0 = now();
      for (int i = 0; i < reps; ++i) cudaMemcpyAsync(host[(i + 1) % R] + fill_n + neg_n, dev, n * 8, cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
      double dt = now() - t0;
      stop.store(true);
      filler.join();
      printf("concurrent T=%d D2H %.2f MB: D2H %.1f GB/s (%.1f us/set); host passes %.1f us/set\n", T, n * 8 / 1e6,
             n * 8.0 * reps / dt / 1e9, dt / reps * 1e6, dt / sets.load() * 1e6);
    }
  }
  printf("hardware_concurrency %u\n", std::thread::hardware_concurrency());
  return 0;
}
