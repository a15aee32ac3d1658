// DMMA m8n8k4.f64 latency (dependent accumulator chain) and per-warp issue
// interval (independent chains), one CTA; cycles per DMMA.
#include <cstdio>
#include "../paper_0809_2407_b200/csrc/tsqr_device.cuh"
using namespace tsqr;
template <int CH>
__global__ void k(long long* out, int iters, double a, double b) {
  double d[CH][2];
  for (int c = 0; c < CH; ++c) { d[c][0] = threadIdx.x * 1e-3 + c; d[c][1] = 1.0; }
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) dmma(d[c][0], d[c][1], a, b);
  long long t1 = clock64();
  double s = 0;
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1];
  if ((threadIdx.x & 31) == 0) out[threadIdx.x >> 5] = t1 - t0;
  if (s == 1234.5) out[63] = 1;
}
int main() {
  long long* d;
  cudaMalloc(&d, 64 * sizeof(long long));
  long long h[64];
  const int it = 4096;
#define RUN(CH, W)                                                          \
  k<CH><<<1, 32 * W>>>(d, 16, 1e-9, 1e-9);                                  \
  k<CH><<<1, 32 * W>>>(d, it, 1e-9, 1e-9);                                  \
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);                      \
  printf("chains %d warps %d: %.1f cycles per DMMA per warp\n", CH, W, (double)h[0] / (it * CH));
  RUN(1, 1) RUN(2, 1) RUN(4, 1) RUN(8, 1) RUN(4, 4) RUN(4, 8) RUN(8, 8)
  return 0;
}
