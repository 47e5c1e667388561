// SM -> mapped page-locked host memory with TMA bulk copies: each CTA moves
// 16 KB chunks device -> shared (cp.async.bulk, mbarrier) -> host
// (cp.async.bulk.global.shared::cta), against plain 16-byte stores.
// nvcc -O3 -std=c++17 -cudart shared -gencode arch=compute_100a,code=sm_100a -o tmastore tmastore.cu
#include <chrono>
#include <cstdio>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>

static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// CB bytes per chunk, NB chunks in flight per CTA (ring of NB buffers)
template <int CB, int NB>
__global__ void __launch_bounds__(32) tma(const char* __restrict__ src, char* dst, long long nchunks) {
  extern __shared__ __align__(128) char buf[];
  __shared__ __align__(8) unsigned long long bar[NB];
  if (threadIdx.x == 0) {
    for (int b = 0; b < NB; ++b) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&bar[b])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncwarp();
  if (threadIdx.x != 0) return;
  int it = 0;
  for (long long c = blockIdx.x; c < nchunks; c += gridDim.x, ++it) {
    const int b = it % NB;
    const unsigned ph = (it / NB) & 1;
    char* sb = buf + b * CB;
    if (it >= NB) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(NB - 1) : "memory");  // buffer b free
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&bar[b])), "r"(CB));
    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_addr(sb)), "l"(src + c * CB), "r"(CB), "r"(smem_addr(&bar[b])) : "memory");
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }"
                 ::"r"(smem_addr(&bar[b])), "r"(ph) : "memory");
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + c * CB), "r"(smem_addr(sb)), "r"(CB)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void st16(const double2* __restrict__ src, double2* dst, long long n2) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n2; i += (long long)gridDim.x * blockDim.x)
    dst[i] = __ldcs(src + i);
}

int main() {
  const long long bytes = 11665408;  // multiple of 16 KB
  const int R = 3, reps = 100;
  char* dev;
  cudaMalloc(&dev, bytes);
  cudaMemset(dev, 1, bytes);
  std::vector<char*> host(R);
  for (auto& h : host) { cudaHostAlloc(&h, bytes, cudaHostAllocDefault); memset(h, 0, bytes); }
  cudaStream_t s;
  cudaStreamCreate(&s);
  auto time_it = [&](const char* what, auto launch) {
    for (int i = 0; i < 3; ++i) launch(i);
    cudaStreamSynchronize(s);
    double t0 = now();
    for (int i = 0; i < reps; ++i) launch(i);
    cudaStreamSynchronize(s);
    double dt = now() - t0;
    printf("%-40s %.1f GB/s %.1f us  err=%s\n", what, bytes * (double)reps / dt / 1e9, dt / reps * 1e6,
           cudaGetErrorString(cudaGetLastError()));
  };
  time_it("DMA one copy", [&](int i) { cudaMemcpyAsync(host[i % R], dev, bytes, cudaMemcpyDeviceToHost, s); });
  time_it("st16 592x256", [&](int i) {
    st16<<<592, 256, 0, s>>>((const double2*)dev, (double2*)host[i % R], bytes / 16);
  });
  char name[64];
  for (int grid : {148, 296, 592}) {
    {
      constexpr int CB = 16384, NB = 4;
      cudaFuncSetAttribute(tma<CB, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, CB * NB);
      snprintf(name, sizeof name, "tma 16KB x4 grid %d", grid);
      time_it(name, [&](int i) { tma<CB, NB><<<grid, 32, CB * NB, s>>>(dev, host[i % R], bytes / CB); });
    }
    {
      constexpr int CB = 8192, NB = 4;
      cudaFuncSetAttribute(tma<CB, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, CB * NB);
      snprintf(name, sizeof name, "tma 8KB x4 grid %d", grid);
      time_it(name, [&](int i) { tma<CB, NB><<<grid, 32, CB * NB, s>>>(dev, host[i % R], bytes / CB); });
    }
    {
      constexpr int CB = 32768, NB = 2;
      cudaFuncSetAttribute(tma<CB, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, CB * NB);
      snprintf(name, sizeof name, "tma 32KB x2 grid %d", grid);
      time_it(name, [&](int i) { tma<CB, NB><<<grid, 32, CB * NB, s>>>(dev, host[i % R], bytes / CB); });
    }
  }
  // correctness of the last copy
  cudaDeviceSynchronize();
  long long bad = 0;
  for (long long i = 0; i < bytes; ++i) bad += host[2][i] != 1;
  printf("mismatching bytes in last buffer: %lld\n", bad);
  return 0;
}
