// Phase-cycle probe of the TMEM split-role ring (k_leaf_tm<G>), CTA 0 sums,
// per tile.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DSP_PROBE -o tools/tm_probe tools/tm_probe.cu
#include <cstdio>
#include <random>
#include <vector>
#include "../paper_0809_2407_b200/csrc/tsqr_device.cuh"
namespace tsqr {
#include "../paper_0809_2407_b200/csrc/dmma_ring.cuh"
#include "../paper_0809_2407_b200/csrc/split_leaf.cuh"
#include "../paper_0809_2407_b200/csrc/tm_leaf.cuh"
}
using namespace tsqr;
template <int G>
void run(double* A, double* R, int* flag, int P, int64_t b) {
  const int64_t n = 128, m = b * P;
  cudaFuncSetAttribute(k_leaf_tm<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TmSmem<G>::bytes);
  for (int it = 0; it < 2; ++it) {
    unsigned long long z[16] = {};
    cudaMemcpyToSymbol(g_sp_cycles, z, sizeof(z));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_leaf_tm<G><<<P, TmCfg<G>::THREADS, TmSmem<G>::bytes>>>(A, n, m, n, P, b, R, flag);
    cudaEventRecord(e1);
    cudaError_t e = cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaMemcpyFromSymbol(z, g_sp_cycles, sizeof(z));
    const double tiles = b / 16.0;
    if (it)
      printf("G=%d %s %.3f ms | per tile: gen total %.0f: ring wait %.0f, gens %.0f, publish %.0f, "
             "ufirst wait %.0f, p1 wait %.0f, upd %.0f, load %.0f | update warps: work %.0f\n",
             G, cudaGetErrorString(e), ms, z[7] / tiles, z[0] / tiles, z[1] / tiles, z[2] / tiles,
             z[3] / tiles, z[4] / tiles, z[5] / tiles, z[6] / tiles, z[10] / tiles);
  }
}
int main(int argc, char** argv) {
  const int P = argc > 1 ? atoi(argv[1]) : 148;
  const int64_t b = argc > 2 ? atoll(argv[2]) : 8192, n = 128, m = b * P;
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
  run<12>(A, R, flag, P, b);
  run<16>(A, R, flag, P, b);
  return 0;
}
