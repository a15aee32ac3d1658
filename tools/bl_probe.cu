// Phase cycles of k_leaf_blocked (block 0, thread 0): panel, G/T + W, update.
#define BL_PROBE
#include "../paper_0809_2407_b200/csrc/tsqr_sm100.cu"
#include <cstdio>
#include <vector>
#include <random>
int main() {
  const int P = 148; const int64_t base = 8192, m = P * base; const int n = 128;
  std::vector<double> h(m * n); std::mt19937_64 g(1); std::normal_distribution<double> d;
  for (auto& x : h) x = d(g);
  double *A, *R; int* flag; cudaMalloc(&A, m * n * 8); cudaMalloc(&R, P * n * n * 8); cudaMalloc(&flag, 4);
  cudaMemcpy(A, h.data(), m * n * 8, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k_leaf_blocked, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)BlockedSmem::bytes);
  unsigned long long z[4] = {0, 0, 0, 0};
  cudaMemcpyToSymbol(g_bl_cycles, z, sizeof(z));
  k_leaf_blocked<<<P, 256, BlockedSmem::bytes>>>(A, n, m, n, P, base, R, flag);
  cudaDeviceSynchronize();
  unsigned long long c[4]; cudaMemcpyFromSymbol(c, g_bl_cycles, sizeof(c));
  const double tiles = base / 128.0;
  printf("per tile (summed over warps): panel %.0f, G/T+W %.0f, update %.0f cycles (err %s)\n", c[0] / tiles, c[1] / tiles,
         c[2] / tiles, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
