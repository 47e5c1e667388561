// Latency cost of sin/cos variants inside a flow-like chain: per thread
// gather two angles (random bus ids), d = a - b, sincos(d), store s and c.
// 40934 threads (two branch-flow groups of case13659), graph of 64 launches.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include <cuda_runtime.h>
#include "../../paper_2510_12897_b200/csrc/exa_math.h"

template <int V>
__global__ void __launch_bounds__(64) k(const double* __restrict__ x, const int* __restrict__ ia, const int* __restrict__ ib,
                                        int n, double* __restrict__ s, double* __restrict__ c) {
  int r = blockIdx.x * 64 + threadIdx.x;
  if (r >= n) return;
  double d = __ldg(x + __ldg(ia + r)) - __ldg(x + __ldg(ib + r));
  double sv, cv;
  if (V == 0) sincos(d, &sv, &cv);
  else if (V == 1) exa_sincos(d, &sv, &cv);
  else if (V == 2) { if (!exa_sincos_fast(fabs(d), &sv, &cv)) { sv = 0; cv = 0; } if (d < 0) sv = -sv; }
  else { sv = d; cv = 1.0 - d; }
  s[r] = sv;
  c[r] = cv;
}

int main() {
  const int nb = 13659, n = 40934, R = 11;
  std::vector<double> hx(nb);
  for (auto& v : hx) v = (rand() / (double)RAND_MAX - 0.5) * 0.5;
  std::vector<int> ha(n), hb(n);
  for (int i = 0; i < n; ++i) { ha[i] = rand() % nb; hb[i] = rand() % nb; }
  double *x, *s, *c; int *ia, *ib;
  cudaMalloc(&x, nb * 8); cudaMemcpy(x, hx.data(), nb * 8, cudaMemcpyHostToDevice);
  cudaMalloc(&ia, n * 4); cudaMemcpy(ia, ha.data(), n * 4, cudaMemcpyHostToDevice);
  cudaMalloc(&ib, n * 4); cudaMemcpy(ib, hb.data(), n * 4, cudaMemcpyHostToDevice);
  cudaMalloc(&s, n * 8 * R); cudaMalloc(&c, n * 8 * R);
  cudaStream_t st; cudaStreamCreate(&st);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[] = {"libdevice sincos", "exa_sincos (CR)", "exa fast path only", "no trig"};
  for (int v = 0; v < 4; ++v) {
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < 64; ++i) {
      double* so = s + (i % R) * n; double* co = c + (i % R) * n;
      int grid = (n + 63) / 64;
      if (v == 0) k<0><<<grid, 64, 0, st>>>(x, ia, ib, n, so, co);
      if (v == 1) k<1><<<grid, 64, 0, st>>>(x, ia, ib, n, so, co);
      if (v == 2) k<2><<<grid, 64, 0, st>>>(x, ia, ib, n, so, co);
      if (v == 3) k<3><<<grid, 64, 0, st>>>(x, ia, ib, n, so, co);
    }
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, st); cudaStreamSynchronize(st);
    cudaEventRecord(e0, st);
    for (int i = 0; i < 10; ++i) cudaGraphLaunch(ge, st);
    cudaEventRecord(e1, st); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-24s %.3f us/launch\n", names[v], ms * 1e3 / 640);
  }
  return 0;
}
