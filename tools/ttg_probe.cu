// Latency of tt_gen (tall-tile generation, owner column through shared memory) alone:
// NG generation warps, optionally next to DMMA warps.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/ttg_probe tools/ttg_probe.cu
#include <cstdio>
#include "../paper_0809_2407_b200/csrc/tsqr_device.cuh"
namespace tsqr {
#include "../paper_0809_2407_b200/csrc/dmma_ring.cuh"
#include "../paper_0809_2407_b200/csrc/split_leaf.cuh"
#include "../paper_0809_2407_b200/csrc/tm_leaf.cuh"
#include "../paper_0809_2407_b200/csrc/tm_tall.cuh"
}
using namespace tsqr;

template <int K, int NG, int PAIR>
__global__ void __launch_bounds__(512, 1) k_g(long long* out, double* sink, int panels, int mode) {
  __shared__ __align__(16) double Rs[NG][8 * 10], gsa[NG][72], xsa[NG][16 * K];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2;
  if (w < NG) {
    double x[K];
#pragma unroll
    for (int k = 0; k < K; ++k) x[k] = ((((lane * 2654435761u) ^ (k * 40503u + 12345u)) * 2246822519u >> 8) & 0xffff) / 32768.0 - 1.0;
    for (int i = lane; i < 80; i += 32) Rs[w][i] = (i % 11 == 0) ? 30.0 : 0.1;
    __syncwarp();
    long long t0 = clock64();
    for (int p = 0; p < panels; ++p) {
      double* gs = gsa[w];
      tt_gen<0, K, false>(x, Rs[w], gs, gs + 64, xsa[w]);
      tt_gen<1, K, false>(x, Rs[w] + 10, gs, gs + 64, xsa[w] + 4 * K);
      tt_gen<2, K, false>(x, Rs[w] + 20, gs, gs + 64, xsa[w]);
      tt_gen<3, K, false>(x, Rs[w] + 30, gs, gs + 64, xsa[w] + 4 * K);
      tt_gen<4, K, false>(x, Rs[w] + 40, gs, gs + 64, xsa[w]);
      tt_gen<5, K, false>(x, Rs[w] + 50, gs, gs + 64, xsa[w] + 4 * K);
      tt_gen<6, K, false>(x, Rs[w] + 60, gs, gs + 64, xsa[w]);
      tt_gen<7, K, false>(x, Rs[w] + 70, gs, gs + 64, xsa[w] + 4 * K);
      __syncwarp();
#pragma unroll
      for (int k = 0; k < K; ++k) x[k] = (((((lane + 7 * p) * 2654435761u) ^ (k * 40503u + 12345u + p)) * 2246822519u >> 8) & 0xffff) / 32768.0 - 1.0;
      for (int i = lane; i < 80; i += 32) Rs[w][i] = (i % 11 == 0) ? 30.0 : 0.1;
      __syncwarp();
    }
    long long t1 = clock64();
    if (lane == 0 && w == 0) out[0] = t1 - t0;
    double z = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) z += x[k];
    if (z == 1234.5) sink[0] = z;
  } else if (mode == 1) {
    double acc[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
    const double av = 1.0 + lane * 1e-9, bv = 0.5;
    for (int it = 0; it < panels * (K / 2 + 2); ++it)
#pragma unroll
      for (int i = 0; i < 8; ++i) dmma(acc[i][0], acc[i][1], av, bv);
    double z = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) z += acc[i][0] + acc[i][1];
    if (z == 1234.5) sink[0] = z;
  }
}

template <int K, int NG, int PAIR>
void run(long long* d, double* s, int mode, int warps, const char* what) {
  const int panels = 64;
  long long h;
  k_g<K, NG, PAIR><<<1, 32 * warps>>>(d, s, 4, mode);
  k_g<K, NG, PAIR><<<1, 32 * warps>>>(d, s, panels, mode);
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%-60s %.0f cycles per generation\n", what, (double)h / (panels * 8));
}

int main() {
  long long* d;
  double* s;
  cudaMalloc(&d, 64);
  cudaMalloc(&s, 8);
  run<8, 1, 0>(d, s, 0, 1, "single: 1 gen warp, 32 rows, alone");
  run<16, 1, 0>(d, s, 0, 1, "single: 1 gen warp, 64 rows, alone");
  run<16, 4, 0>(d, s, 0, 4, "single: 4 gen warps (1 per SMSP), 64 rows");
  run<16, 4, 0>(d, s, 1, 8, "single: 4 gen warps, 64 rows, 4 DMMA warps");
  run<16, 4, 0>(d, s, 1, 12, "single: 4 gen warps, 64 rows, 8 DMMA warps");
  run<8, 8, 0>(d, s, 1, 16, "single: 8 gen warps, 32 rows, 8 DMMA warps");
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
