// A/B + phase probe of the tall-tile TMEM leaf (k_leaf_tt<H>) against k_leaf_tm<16>.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 [-DSP_PROBE] -o tools/tt_probe tools/tt_probe.cu
//   tools/tt_probe [P=148] [b=8192] [n=128]
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>
#include "../paper_0809_2407_b200/csrc/tsqr_device.cuh"
namespace tsqr {
#include "../paper_0809_2407_b200/csrc/dmma_ring.cuh"
#include "../paper_0809_2407_b200/csrc/split_leaf.cuh"
#include "../paper_0809_2407_b200/csrc/tm_leaf.cuh"
#include "../paper_0809_2407_b200/csrc/tm_tall.cuh"
}
using namespace tsqr;

static std::vector<double> g_ref;

template <typename KERN, typename LAUNCH>
void run(const char* name, KERN kern, LAUNCH launch, size_t smem, double* A, double* R, int* flag, int P,
         int64_t b, int64_t n, int64_t m, double tiles_rows) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  float best = 1e30f;
  cudaError_t e = cudaSuccess;
  for (int it = 0; it < 4; ++it) {
#ifdef SP_PROBE
    unsigned long long z[16] = {};
    cudaMemcpyToSymbol(g_sp_cycles, z, sizeof(z));
#endif
    cudaMemset(R, 0, (size_t)P * n * n * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    e = cudaDeviceSynchronize();
    if (e != cudaSuccess) break;
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
#ifdef SP_PROBE
    if (it == 3) {
      cudaMemcpyFromSymbol(z, g_sp_cycles, sizeof(z));
      const double tiles = b / tiles_rows;
      printf("   per tile: gen total %.0f: ring wait %.0f, gens %.0f, publish %.0f, stage %.0f, ufirst wait %.0f, "
             "p1 wait %.0f, upd %.0f, load %.0f | update warps (sum): yrdy wait %.0f, ver_u wait %.0f, work %.0f\n",
             z[7] / tiles, z[0] / tiles, z[11] / tiles, z[2] / tiles, z[1] / tiles, z[3] / tiles, z[4] / tiles,
             z[5] / tiles, z[6] / tiles, z[8] / tiles, z[9] / tiles, z[10] / tiles);
    }
#endif
  }
  std::vector<double> h((size_t)P * n * n);
  cudaMemcpy(h.data(), R, h.size() * 8, cudaMemcpyDeviceToHost);
  double err = 0.0, nrm = 0.0;
  if (g_ref.empty()) g_ref = h;
  for (int l = 0; l < P; ++l)
    for (int r = 0; r < n; ++r) {
      const double* a = &h[(size_t)l * n * n + r * n];
      const double* c = &g_ref[(size_t)l * n * n + r * n];
      const double sa = a[r] < 0 ? -1.0 : 1.0, sc = c[r] < 0 ? -1.0 : 1.0;
      for (int j = 0; j < n; ++j) {
        err = fmax(err, fabs(sa * a[j] - sc * c[j]));
        nrm = fmax(nrm, fabs(c[j]));
      }
    }
  const double flops = 2.0 * m * n * n;
  printf("%-14s %s %.3f ms  %.2f TF/s  max|dR|/max|R| = %.2e (%.1f eps)\n", name, cudaGetErrorString(e), best,
         flops / best / 1e9, err / nrm, err / nrm / 2.22e-16);
  fflush(stdout);
}

int main(int argc, char** argv) {
  const int P = argc > 1 ? atoi(argv[1]) : 148;
  const int64_t b = argc > 2 ? atoll(argv[2]) : 8192, n = argc > 3 ? atoll(argv[3]) : 128, m = b * P;
  std::vector<double> h((size_t)m * n);
  std::mt19937_64 rng(1);
  std::normal_distribution<double> nd;
  for (auto& x : h) x = nd(rng);
  double *A, *R;
  int* flag;
  cudaMalloc(&A, (size_t)m * n * 8);
  cudaMalloc(&R, (size_t)P * n * n * 8);
  cudaMalloc(&flag, 4);
  cudaMemcpy(A, h.data(), (size_t)m * n * 8, cudaMemcpyHostToDevice);
  printf("P=%d b=%lld n=%lld\n", P, (long long)b, (long long)n);
  run("tm16 (H=16)", k_leaf_tm<16>,
      [&] { k_leaf_tm<16><<<P, TmCfg<16>::THREADS, TmSmem<16>::bytes>>>(A, n, m, (int)n, P, b, R, flag); },
      TmSmem<16>::bytes, A, R, flag, P, b, n, m, 16.0);
#define TT_RUN(NAME, H, UW)                                                                          \
  run(NAME, k_leaf_tt<H, UW, false>,                                                                 \
      [&] {                                                                                          \
        k_leaf_tt<H, UW, false><<<P, TtCfg<H, UW>::THREADS, TtSmem<H>::bytes>>>(                     \
            A, n, m, (int)n, P, b, R, flag, nullptr, 0, nullptr, 0, 0);                              \
      },                                                                                             \
      TtSmem<H>::bytes, A, R, flag, P, b, n, m, (double)H)
  TT_RUN("tt H=32 UW=1", 32, 1);
  TT_RUN("tt H=64 UW=1", 64, 1);
  return 0;
}
