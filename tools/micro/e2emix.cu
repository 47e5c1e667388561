// Host path balance: a store kernel pushing D MB per set into page-locked
// memory while T host threads write F MB (memset) + N MB (negate-copy) per set
// into other page-locked arrays -- does moving bytes from PCIe to host threads
// pay on this host?  nvcc -O3 -std=c++17 -cudart shared -gencode arch=compute_100a,code=sm_100a -o e2emix e2emix.cu -lpthread
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>
#include <cuda_runtime.h>

static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

__global__ void st(const double2* __restrict__ src, double2* dst, long long n2) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n2; i += (long long)gridDim.x * blockDim.x)
    dst[i] = __ldcs(src + i);
}

int main() {
  const long long out_n = 18800000 / 8;
  const int R = 3, sets = 300;
  double* dev;
  cudaMalloc(&dev, out_n * 8);
  cudaMemset(dev, 0, out_n * 8);
  std::vector<double*> host(R);
  for (auto& h : host) { cudaHostAlloc(&h, 3 * out_n * 8, cudaHostAllocDefault); memset(h, 1, 3 * out_n * 8); }
  cudaStream_t s;
  cudaStreamCreate(&s);
  struct Cfg { double d, f, n; };
  for (int T : {4, 8}) {
    for (Cfg c : {Cfg{11.66, 7.2, 0}, Cfg{10.33, 7.2, 1.33}, Cfg{9.36, 7.2, 2.3}, Cfg{11.66, 0, 0}, Cfg{0, 7.2, 0}, Cfg{0, 7.2, 2.3}}) {
      const long long d2 = (long long)(c.d * 1e6 / 16), fn = (long long)(c.f * 1e6 / 8), nn = (long long)(c.n * 1e6 / 8);
      // one "set" = kernel on the stream + host pass on the caller's threads; the
      // caller waits for set i-2's kernel before reusing its buffer (3 in flight)
      std::vector<cudaEvent_t> ev(R);
      for (auto& e : ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
      double t0 = now();
      for (int i = 0; i < sets; ++i) {
        double* h = host[i % R];
        cudaEventSynchronize(ev[i % R]);
        if (d2) st<<<592, 256, 0, s>>>(reinterpret_cast<const double2*>(dev), reinterpret_cast<double2*>(h), d2);
        cudaEventRecord(ev[i % R], s);
        std::vector<std::thread> th;
        for (int t = 0; t < T; ++t)
          th.emplace_back([=] {
            double* dst = h + out_n;  // host-written part (disjoint from the kernel's)
            long long a = fn * t / T, b = fn * (t + 1) / T;
            memset(dst + a, 0, (b - a) * 8);
            const double* src = h;
            double* nd = dst + fn;
            long long p = nn * t / T, q = nn * (t + 1) / T;
            for (long long k = p; k < q; ++k) nd[k] = -src[k];
          });
        for (auto& x : th) x.join();
      }
      cudaStreamSynchronize(s);
      double dt = now() - t0;
      printf("T=%d D2H %.2f MB + memset %.2f MB + negate %.2f MB: %.1f us per set (%.0f sets/s)\n", T, c.d, c.f, c.n,
             dt / sets * 1e6, sets / dt);
      for (auto& e : ev) cudaEventDestroy(e);
    }
  }
  return 0;
}
