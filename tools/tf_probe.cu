// Phase probe of k_tree_factor_dmma128: cycles in the panel owners' generations, publication,
// and the next owner's block update.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DTF_PROBE -o tools/tf_probe tools/tf_probe.cu
#include <cstdio>
#include <random>
#include <vector>
#include "../paper_0809_2407_b200/csrc/tsqr_device.cuh"
namespace tsqr {
#include "../paper_0809_2407_b200/csrc/dmma_ring.cuh"
#include "../paper_0809_2407_b200/csrc/tree_factor128.cuh"
}
using namespace tsqr;
int main() {
  const int n = 128;
  std::vector<double> h(2 * n * n, 0.0);
  std::mt19937_64 rng(1);
  std::normal_distribution<double> nd;
  for (int s = 0; s < 2; ++s)
    for (int r = 0; r < n; ++r)
      for (int c = r; c < n; ++c) h[s * n * n + r * n + c] = nd(rng) + (r == c ? 20.0 : 0.0);
  double *R, *Y, *tau;
  int* ev;
  cudaMalloc(&R, 2 * n * n * 8);
  cudaMalloc(&Y, n * n * 8);
  cudaMalloc(&tau, n * 8);
  cudaMalloc(&ev, 12);
  int hev[3] = {0, 1, 0};
  cudaMemcpy(ev, hev, 12, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k_tree_factor_dmma128, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TreeFactor128Smem::bytes);
  for (int it = 0; it < 3; ++it) {
    cudaMemcpy(R, h.data(), 2 * n * n * 8, cudaMemcpyHostToDevice);
    unsigned long long z[8] = {};
    cudaMemcpyToSymbol(g_tf_cycles, z, sizeof(z));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_tree_factor_dmma128<<<1, TF_W * 32, TreeFactor128Smem::bytes>>>(R, n, ev, Y, tau);
    cudaEventRecord(e1);
    cudaError_t e = cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaMemcpyFromSymbol(z, g_tf_cycles, sizeof(z));
    printf("%s %.1f us | main loop %llu cycles: generations %llu (%.0f each), publish %llu (%.0f per panel), next owner's update %llu (%.0f per panel)\n",
           cudaGetErrorString(e), ms * 1e3, z[3], z[0], z[0] / 128.0, z[1], z[1] / 16.0, z[2], z[2] / 15.0);
  }
  return 0;
}
