// Per-column latency of the ring chain step with 1, 2, 4, 8 warps per CTA (one CTA per SM).
#include "../paper_0809_2407_b200/csrc/tsqr_sm100.cu"
#include <cstdio>
#include <vector>
#include <random>
template <int NP, int HT, int RW>
__global__ void __launch_bounds__(RW * 32, 1)
k_chain_rw(const double* __restrict__ A, int64_t lda, int n, int64_t rows, double* Rio) {
  constexpr int S = NP / 32;
  extern __shared__ __align__(16) double sm[];
  double* Rs = sm;
  double* vbuf = Rs + NP * NP;
  int* ver = reinterpret_cast<int*>(vbuf + RW * 2 * HT);
  const int w = threadIdx.x >> 5;
  for (int idx = threadIdx.x; idx < NP * NP; idx += RW * 32) Rs[idx] = (idx / NP == idx % NP) ? 1.0 : 0.0;
  for (int j = threadIdx.x; j < NP; j += RW * 32) ver[j] = 0;
  __syncthreads();
  const double* Al = A + (int64_t)blockIdx.x * rows * lda;
  const int T = (int)(rows / HT);
  bool bad = false;
  double X[HT][S];
  for (int t = w; t < T; t += RW) {
    load_rows<HT, S>(X, Al + (int64_t)t * HT * lda, lda, HT, n, 0, bad);
#ifdef RING3
    ring_factor_tile3<NP, HT>(X, Rs, ver, n, t, nullptr);
#else
#ifdef RING3
    ring_factor_tile3<NP, HT>(X, Rs, ver, n, t, nullptr);
#else
    ring_factor_tile<NP, HT>(X, Rs, ver, vbuf + w * 2 * HT, n, t, nullptr);
#endif
#endif
  }
  __syncthreads();
  if (threadIdx.x == 0) Rio[blockIdx.x] = Rs[NP * NP - 1] + (bad ? 1.0 : 0.0);
}
#ifndef HTV
#define HTV 16
#endif
template <int RW>
void run(const double* A, double* R, int64_t rows) {
  const size_t sm = sizeof(double) * (128 * 128 + RW * 2 * HTV) + 4 * 128;
  cudaFuncSetAttribute(k_chain_rw<128, HTV, RW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k_chain_rw<128, HTV, RW><<<148, RW * 32, sm>>>(A, 128, 128, rows, R);
  cudaEventRecord(e0);
  k_chain_rw<128, HTV, RW><<<148, RW * 32, sm>>>(A, 128, 128, rows, R);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double cols = (double)(rows / HTV) * 128 / RW;  // column steps per warp
  printf("HT=%d warps=%d: %.3f ms (%.1f rows/us/SM), %.0f cycles per column step per warp, err=%s\n",
         HTV, RW, ms, rows / (ms * 1e3), ms * 1e-3 * 1.92e9 / cols, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  const int64_t rows = 6144;
  const int64_t m = 148 * rows;
  std::vector<double> h(m * 128); std::mt19937_64 g(1); std::normal_distribution<double> d;
  for (auto& x : h) x = d(g);
  double *A, *R; cudaMalloc(&A, m * 128 * 8); cudaMalloc(&R, 148 * 8);
  cudaMemcpy(A, h.data(), m * 128 * 8, cudaMemcpyHostToDevice);
#ifdef ONLY_RW
  run<ONLY_RW>(A, R, rows);
#else
  run<1>(A, R, rows); run<2>(A, R, rows); run<4>(A, R, rows); run<8>(A, R, rows);
#endif
}
