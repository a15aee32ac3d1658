// Is DFMA a separate pipe from DMMA on sm_100a?  Runs fixed work per warp with
// (a) all warps DMMA, (b) all warps DFMA, (c) warps 0-3 DMMA + warps 4-7 DFMA
// (one of each per SM sub-partition), (d) each warp interleaving both, and
// reports combined FP64 TF/s.  Then the latency of a dependent DFMA chain on
// an idle sub-partition vs next to a DMMA-saturating warp.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mix_probe tools/mix_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

// kind per warp: 0 = DMMA (8 chains), 1 = DFMA (16 chains), 2 = both interleaved
__global__ void __launch_bounds__(256) k_mix(double* out, int iters, int mode) {
  const int w = threadIdx.x >> 5;
  int kind = mode == 0 ? 0 : mode == 1 ? 1 : mode == 2 ? (w < 4 ? 0 : 1) : 2;
  double acc[8][2];
  double a[16];
#pragma unroll
  for (int i = 0; i < 8; ++i) { acc[i][0] = 0.0; acc[i][1] = 0.0; }
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-7 + i;
  const double av = 1.0 + threadIdx.x * 1e-9, bv = 0.5, b = 1.0000001, c = 1e-9;
  if (kind == 0) {
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) dmma(acc[i][0], acc[i][1], av, bv);
    }
  } else if (kind == 1) {
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int i = 0; i < 16; ++i) a[i] = fma(a[i], b, c);
    }
  } else {
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        dmma(acc[i][0], acc[i][1], av, bv);
#pragma unroll
        for (int j = 0; j < 16; ++j) a[j] = fma(a[j], b, c);
      }
    }
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  if (s == 12345.678) out[0] = s;
}

// latency: warp 0 runs a dependent DFMA chain; warps 4 (same sub-partition)
// hammer DMMA when `noise` = 1, DFMA when 2, nothing when 0.
__global__ void __launch_bounds__(256) k_lat(long long* cyc, double* out, int iters, int noise) {
  const int w = threadIdx.x >> 5;
  if (w == 0) {
    double x = threadIdx.x * 1e-9 + 1.0;
    const double b = 1.0000001, c = 1e-9;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int j = 0; j < 16; ++j) x = fma(x, b, c);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
    if (x == 12345.678) out[0] = x;
  } else if (w == 4 && noise) {
    double acc[8][2];
    double a[16];
#pragma unroll
    for (int i = 0; i < 8; ++i) { acc[i][0] = 0.0; acc[i][1] = 0.0; }
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-7 + i;
    const double av = 1.0, bv = 0.5, b = 1.0000001, c = 1e-9;
    for (int it = 0; it < iters / 4; ++it) {
      if (noise == 1) {
#pragma unroll
        for (int i = 0; i < 8; ++i) dmma(acc[i][0], acc[i][1], av, bv);
      } else {
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int i = 0; i < 16; ++i) a[i] = fma(a[i], b, c);
      }
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
#pragma unroll
    for (int i = 0; i < 16; ++i) s += a[i];
    if (s == 12345.678) out[0] = s;
  }
}

int main() {
  double* d;
  long long* cyc;
  cudaMalloc(&d, 64);
  cudaMalloc(&cyc, 64);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4000;
  const char* names[] = {"all DMMA", "all DFMA", "4 DMMA + 4 DFMA warps", "interleaved in each warp"};
  for (int mode = 0; mode < 4; ++mode) {
    for (int cps : {1, 2}) {
      k_mix<<<sms * cps, 256>>>(d, 50, mode);
      cudaEventRecord(e0);
      k_mix<<<sms * cps, 256>>>(d, iters, mode);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      // per warp per iter: DMMA warp 8 x 256 FMA; DFMA warp 8 x 16 x 32 FMA (= 4096, same)
      double fma_dmma = 8.0 * 256, fma_dfma = 8.0 * 16 * 32;
      double per_cta;
      if (mode == 0) per_cta = 8 * fma_dmma;
      else if (mode == 1) per_cta = 8 * fma_dfma;
      else if (mode == 2) per_cta = 4 * fma_dmma + 4 * fma_dfma;
      else per_cta = 8 * (fma_dmma + fma_dfma);
      double tf = 2.0 * per_cta * iters * sms * cps / (ms * 1e-3) / 1e12;
      printf("%-28s ctas/SM %d: %.3f ms  %.2f TF/s\n", names[mode], cps, ms, tf);
    }
  }
  long long h;
  for (int noise = 0; noise < 3; ++noise) {
    k_lat<<<1, 256>>>(cyc, d, 64, noise);
    k_lat<<<1, 256>>>(cyc, d, 2000, noise);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("dependent DFMA latency, neighbour %s: %.2f cycles\n",
           noise == 0 ? "idle" : noise == 1 ? "DMMA" : "DFMA", (double)h / (2000 * 16));
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
