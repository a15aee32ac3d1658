// Latency microbenchmarks (one warp, dependent chains), cycles per op.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(long long* out, double seed, int iters) {
  double a = seed + threadIdx.x * 1e-9, b = 1.0000001, c = 1e-9;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { a = fma(a, b, c); a = fma(a, b, c); a = fma(a, b, c); a = fma(a, b, c); }
  t1 = clock64(); if (threadIdx.x == 0) out[0] = (t1 - t0); 
  // DMUL chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { a = a * b; a = a * b; a = a * b; a = a * b; }
  t1 = clock64(); if (threadIdx.x == 0) out[1] = (t1 - t0);
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { a = a + c; a = a + c; a = a + c; a = a + c; }
  t1 = clock64(); if (threadIdx.x == 0) out[2] = (t1 - t0);
  // sqrt chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { a = sqrt(a + 1.5); }
  t1 = clock64(); if (threadIdx.x == 0) out[3] = (t1 - t0) * 4;
  // drcp chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { a = __drcp_rn(a + 1.5); }
  t1 = clock64(); if (threadIdx.x == 0) out[4] = (t1 - t0) * 4;
  // div chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { a = 3.0 / (a + 1.5); }
  t1 = clock64(); if (threadIdx.x == 0) out[5] = (t1 - t0) * 4;
  // shfl chain (double)
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { a = __shfl_sync(0xffffffff, a, (threadIdx.x + 1) & 31) + c; }
  t1 = clock64(); if (threadIdx.x == 0) out[6] = (t1 - t0) * 4;
  // membar.cta
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { __threadfence_block(); a = a + c; }
  t1 = clock64(); if (threadIdx.x == 0) out[7] = (t1 - t0) * 4;
  // syncwarp
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { __syncwarp(); a = a + c; }
  t1 = clock64(); if (threadIdx.x == 0) out[8] = (t1 - t0) * 4;
  if (a == 1234.5) out[9] = 1;
}
__global__ void k_lds(long long* out, int iters) {
  __shared__ double s[1024];
  for (int i = threadIdx.x; i < 1024; i += 32) s[i] = (double)((i * 7 + 1) & 1023);
  __syncwarp();
  int idx = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) { idx = (int)s[idx]; idx = (int)s[idx]; idx = (int)s[idx]; idx = (int)s[idx]; }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[10] = t1 - t0;
  if (idx == 12345) out[11] = 1;
}
int main() {
  long long* d; cudaMalloc(&d, 16 * sizeof(long long));
  int iters = 4096;
  k<<<1, 32>>>(d, 1.0, 16); k<<<1, 32>>>(d, 1.0, iters);
  k_lds<<<1, 32>>>(d, iters);
  long long h[16]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const char* names[] = {"dfma", "dmul", "dadd", "sqrt(+dadd)", "drcp_rn(+dadd)", "div(+dadd)", "shfl(+dadd)", "membar.cta(+dadd)", "syncwarp(+dadd)"};
  for (int i = 0; i < 9; ++i) printf("%-20s %.1f cycles\n", names[i], (double)h[i] / (4.0 * iters));
  printf("%-20s %.1f cycles (incl. f2i)\n", "lds.64+cvt", (double)h[10] / (4.0 * iters));
  return 0;
}
