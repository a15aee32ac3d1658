// Fraction of ring-tile time spent spinning on the version counters.
#define TSQR_SPIN_PROBE 1
#include "../paper_0809_2407_b200/csrc/tsqr_sm100.cu"
#include <cstdio>
#include <vector>
#include <random>
int main(int argc, char** argv) {
  int n = argc > 1 ? atoi(argv[1]) : 128;
  int leaves = 148; long long rows = 8192; long long m = leaves * rows;
  std::vector<double> h(m * n); std::mt19937_64 g(1); std::normal_distribution<double> d;
  for (auto& x : h) x = d(g);
  double *A, *R; int* flag;
  cudaMalloc(&A, m * n * 8); cudaMalloc(&R, (size_t)leaves * n * n * 8); cudaMalloc(&flag, 4);
  cudaMemcpy(A, h.data(), m * n * 8, cudaMemcpyHostToDevice);
  for (int it = 0; it < 2; ++it) {
    unsigned long long z[2] = {0, 0};
    cudaMemcpyToSymbol(g_spin_cycles, z, sizeof(z));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    int rc = tsqr_f64_leaf_factor(A, n, m, n, leaves, nullptr, 0, nullptr, 0, R, flag, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    cudaMemcpyFromSymbol(z, g_spin_cycles, sizeof(z));
    printf("rc=%d n=%d %.3f ms  spin/total cycles = %.3f (spin %.3e, total %.3e)\n", rc, n, ms,
           (double)z[0] / z[1], (double)z[0], (double)z[1]);
  }
  return 0;
}
