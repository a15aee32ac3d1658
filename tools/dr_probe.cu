// Phase-cycle probe of the DMMA warp ring leaf (k_leaf_dmma): 148 leaves of
// 8192 x 128 N(0,1)-ish data, per-warp clock64 sums over CTA 0.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DDR_PROBE -o tools/dr_probe tools/dr_probe.cu
#include <cstdio>
#include <vector>
#include <random>
#include "../paper_0809_2407_b200/csrc/tsqr_device.cuh"
namespace tsqr {
#include "../paper_0809_2407_b200/csrc/dmma_ring.cuh"
}
using namespace tsqr;
#ifndef DR_NPX
#define DR_NPX 128
#endif
#ifndef DR_KERNEL
#define DR_KERNEL k_leaf_dmma
#endif
int main(int argc, char** argv) {
  const int P = argc > 1 ? atoi(argv[1]) : 148;
  const int64_t b = argc > 2 ? atoll(argv[2]) : 8192, n = DR_NPX, m = b * P;
  std::vector<double> h(m * n);
  std::mt19937_64 rng(1);
  std::normal_distribution<double> nd;
  for (auto& x : h) x = nd(rng);
  double *A, *R;
  int* flag;
  cudaMalloc(&A, m * n * 8);
  cudaMalloc(&R, P * n * n * 8);
  cudaMalloc(&flag, 4);
  cudaMemcpy(A, h.data(), m * n * 8, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(DR_KERNEL<DR_NPX, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)DmmaRingSmem<DR_NPX>::bytes);
  for (int it = 0; it < 2; ++it) {
    unsigned long long z[8] = {};
    cudaMemcpyToSymbol(g_dr_cycles, z, sizeof(z));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    DR_KERNEL<DR_NPX, true, false><<<P, 256, DmmaRingSmem<DR_NPX>::bytes>>>(A, n, m, n, P, b, nullptr, 0, nullptr, 0, R, flag, 0);
    cudaEventRecord(e1);
    cudaError_t e = cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaMemcpyFromSymbol(z, g_dr_cycles, sizeof(z));
    const double tiles = b / 16.0;  // per CTA
    printf("%s  %.3f ms  per tile (cycles, summed over warps / tiles): c0 %.0f c1 %.0f c2 %.0f c3 %.0f c4 %.0f | total/warp %.0f\n",
           cudaGetErrorString(e), ms, z[0] / tiles, z[1] / tiles, z[2] / tiles, z[3] / tiles, z[4] / tiles,
           z[5] / 8.0);
  }
  return 0;
}
