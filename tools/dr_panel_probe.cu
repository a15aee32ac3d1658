// Latency of the DMMA ring's Level-2 panel step (dr_panel): each warp factors
// its own 16 x 8 panel against private pivot rows, `iters` times; cycles per
// generation (8 generations per call).
#include <cstdio>
#include "../paper_0809_2407_b200/csrc/tsqr_device.cuh"
namespace tsqr {
#include "../paper_0809_2407_b200/csrc/dmma_ring.cuh"
}
using namespace tsqr;
__global__ void kp(long long* out, int iters) {
  __shared__ double Rs[8][8 * 10 + 128 + 8];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* R = Rs[w];
  for (int i = lane; i < 8 * 10 + 136; i += 32) R[i] = 0.01 * (i % 7);
  __syncwarp();
  double x[4];
  for (int k = 0; k < 4; ++k) x[k] = 0.1 * (lane + k) - 1.0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    dr_panel(x, R, 10, R + 8 * 10, R + 8 * 10 + 64);
    for (int k = 0; k < 4; ++k) x[k] += 0.5;
  }
  long long t1 = clock64();
  if (lane == 0) out[w] = t1 - t0;
  if (x[0] == 1234.5) out[9] = 1;
}
int main() {
  long long* d;
  cudaMalloc(&d, 16 * sizeof(long long));
  for (int W : {1, 2, 4, 8}) {
    kp<<<1, 32 * W>>>(d, 10);
    kp<<<1, 32 * W>>>(d, 200);
    long long h[16];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("warps %d: %.0f cycles per generation (%s)\n", W, h[0] / (200.0 * 8), cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
