// Per-reflector cycle count of the n <= 32 stacked-triangle combine
// (k_tree_factor_w32's loop, instrumented copy): where do ~1.5 K cycles go?
#include <cstdio>
#include "../paper_0809_2407_b200/csrc/tsqr_device.cuh"
using namespace tsqr;
__device__ long long g_c[8];
__global__ void kf(double* Rslots, int n, double* Ynode, double* taunode) {
  const int lane = threadIdx.x & 31;
  __shared__ double Ras[32][33];
  __shared__ double vs[32];
  double* Ra = Rslots;
  const double* Rb = Rslots + n * n;
  double cb[32];
#pragma unroll
  for (int r = 0; r < 32; ++r) {
    const bool ok = (r < n && lane < n && lane >= r);
    Ras[r][lane] = ok ? Ra[r * n + lane] : 0.0;
    cb[r] = ok ? Rb[r * n + lane] : 0.0;
  }
  __syncwarp();
  const double diag = Ras[lane][lane];
  long long acc[5] = {0, 0, 0, 0, 0};
#pragma unroll 1
  for (int j = 0; j < n; ++j) {
    long long t0 = clock64();
    double s4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int r = 0; r < 32; ++r) s4[r & 3] = fma(cb[r], cb[r], s4[r & 3]);
    const double sg = __shfl_sync(FULL, (s4[0] + s4[1]) + (s4[2] + s4[3]), j);
    const double x0 = __shfl_sync(FULL, diag, j);
    double beta, tau, scale;
    house_lean(x0, sg, beta, tau, scale);
    long long t1 = clock64();
    if (lane == j) {
#pragma unroll
      for (int r = 0; r < 32; ++r) vs[r] = cb[r] * scale;
    }
    __syncwarp();
    long long t2 = clock64();
    const double raj = Ras[j][lane];
    double d4[4] = {raj, 0.0, 0.0, 0.0};
#pragma unroll
    for (int r = 0; r < 32; ++r) d4[r & 3] = fma(vs[r], cb[r], d4[r & 3]);
    const double d = (d4[0] + d4[1]) + (d4[2] + d4[3]);
    const double w = (lane > j) ? tau * d : 0.0;
    long long t3 = clock64();
#pragma unroll
    for (int r = 0; r < 32; ++r) cb[r] = fma(-vs[r], w, cb[r]);
    if (lane > j) Ras[j][lane] = raj - w;
    if (lane == j) {
      Ras[j][j] = beta;
#pragma unroll
      for (int r = 0; r < 32; ++r) cb[r] = vs[r];
    }
    if (lane == 0 && taunode) taunode[j] = tau;
    __syncwarp();
    long long t4 = clock64();
    acc[0] += t1 - t0; acc[1] += t2 - t1; acc[2] += t3 - t2; acc[3] += t4 - t3;
  }
#pragma unroll
  for (int r = 0; r < 32; ++r) {
    if (r < n && lane < n) {
      Ra[r * n + lane] = (lane >= r) ? Ras[r][lane] : 0.0;
      if (Ynode) Ynode[r * n + lane] = (lane >= r) ? cb[r] : 0.0;
    }
  }
  if (lane == 0) for (int i = 0; i < 4; ++i) g_c[i] = acc[i];
}
int main() {
  const int n = 32;
  double h[2 * n * n];
  for (int i = 0; i < 2 * n * n; ++i) h[i] = ((i * 7919) % 1000) / 1000.0 - 0.5;
  double *R, *Y, *t;
  cudaMalloc(&R, sizeof(h)); cudaMalloc(&Y, n * n * 8); cudaMalloc(&t, n * 8);
  for (int it = 0; it < 3; ++it) {
    cudaMemcpy(R, h, sizeof(h), cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kf<<<1, 32>>>(R, n, Y, t);
    cudaEventRecord(e1); cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long c[8]; cudaMemcpyFromSymbol(c, g_c, sizeof(c));
    printf("%.1f us; per reflector: house %.0f, v stage %.0f, dot %.0f, update %.0f cycles\n", ms * 1e3,
           c[0] / 32.0, c[1] / 32.0, c[2] / 32.0, c[3] / 32.0);
  }
  return 0;
}
