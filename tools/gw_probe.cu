// Latency probe for a "generation warp": one warp holds a 128-row panel of 8
// (W2 = 1: 16, the panel plus the next block at Level 2) columns in registers
// (lane (g, q) holds rows 8b + 2q + e of column g) and runs Householder
// generations back to back, no barriers; warps 1..7 optionally run dummy DMMA
// work (mode 1) to load the FP64 pipe like trailing-update warps would.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/gw_probe tools/gw_probe.cu
#include <cstdio>
#include "../paper_0809_2407_b200/csrc/tsqr_device.cuh"
namespace tsqr {
#include "../paper_0809_2407_b200/csrc/dmma_ring.cuh"
}
using namespace tsqr;

template <int I, int W2, int K>
__device__ __forceinline__ void gw_gen(double (&x)[K], double (&xb)[K], const double (&rg)[8],
                                       const double (&rgb)[8], double* Rs, double* gs, int g, int q) {
  double xi[K];
#pragma unroll
  for (int k = 0; k < K; ++k) xi[k] = __shfl_sync(FULL, x[k], 4 * I + q);
  double a[4] = {0.0, 0.0, 0.0, 0.0}, b[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int k = 0; k < K; ++k) a[k & 3] = fma(xi[k], x[k], a[k & 3]);
  if (W2) {
#pragma unroll
    for (int k = 0; k < K; ++k) b[k & 3] = fma(xi[k], xb[k], b[k & 3]);
  }
  double pd = (a[0] + a[1]) + (a[2] + a[3]);
  double pb = (b[0] + b[1]) + (b[2] + b[3]);
  pd += __shfl_xor_sync(FULL, pd, 1);
  if (W2) pb += __shfl_xor_sync(FULL, pb, 1);
  pd += __shfl_xor_sync(FULL, pd, 2);
  if (W2) pb += __shfl_xor_sync(FULL, pb, 2);
  const double s = __shfl_sync(FULL, pd, 4 * I);
  const double x0 = __shfl_sync(FULL, rg[I], 4 * I);
  double beta, tau, scale, invb;
  house_fast(x0, s, beta, tau, scale, invb);
  const double tw = fma(scale, pd, rg[I]);
  const bool upd = g > I, own = g == I;
  const double f = upd ? tw * invb : (own ? scale : 0.0);
#pragma unroll
  for (int k = 0; k < K; ++k) x[k] = fma(f, xi[k], own ? 0.0 : x[k]);
  if (W2) {
    const double twb = fma(scale, pb, rgb[I]);
    const double fb = twb * invb;
#pragma unroll
    for (int k = 0; k < K; ++k) xb[k] = fma(fb, xi[k], xb[k]);
    Rs[64 + I * 8 + g] = rgb[I] - tau * twb;
  }
  double* dst = upd ? Rs + I * 8 + g : (own ? Rs + I * 8 + I : gs + g * 8 + I);
  *dst = upd ? rg[I] - tau * tw : (own ? beta : scale * (s - s + pd));
  gs[64 + I] = tau;
}

template <int W2, int K, int NG>
__global__ void __launch_bounds__(512, 1) k_gw(long long* out, double* sink, int panels, int mode) {
  __shared__ double Rs[NG][128], gsa[NG][72];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  if (w < NG) {
    double* gs = gsa[w];
    double x[K], xb[K], rg[8], rgb[8];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      x[k] = 1.0 + 0.01 * ((lane * 37 + k * 11) % 17);
      xb[k] = 0.5 + 0.01 * ((lane * 13 + k * 7) % 19);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      rg[i] = (i == g) ? 30.0 : 0.1 * i;
      rgb[i] = 0.2 * i;
    }
    long long t0 = clock64();
    for (int p = 0; p < panels; ++p) {
      gw_gen<0, W2, K>(x, xb, rg, rgb, Rs[w], gs, g, q);
      gw_gen<1, W2, K>(x, xb, rg, rgb, Rs[w], gs, g, q);
      gw_gen<2, W2, K>(x, xb, rg, rgb, Rs[w], gs, g, q);
      gw_gen<3, W2, K>(x, xb, rg, rgb, Rs[w], gs, g, q);
      gw_gen<4, W2, K>(x, xb, rg, rgb, Rs[w], gs, g, q);
      gw_gen<5, W2, K>(x, xb, rg, rgb, Rs[w], gs, g, q);
      gw_gen<6, W2, K>(x, xb, rg, rgb, Rs[w], gs, g, q);
      gw_gen<7, W2, K>(x, xb, rg, rgb, Rs[w], gs, g, q);
      // next panel: reuse the (now reflector) values as fresh data
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const double t = x[k];
        x[k] = xb[k] + 1.0;
        xb[k] = t * 0.5 + 0.25;
      }
    }
    long long t1 = clock64();
    if (lane == 0 && w == 0) out[0] = t1 - t0;
    double z = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) z += x[k] + xb[k];
    if (z == 1234.5) sink[0] = z;
  } else if (mode == 1) {
    double acc[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
    const double av = 1.0 + lane * 1e-9, bv = 0.5;
    for (int it = 0; it < panels * (K / 4 + 2); ++it)
#pragma unroll
      for (int i = 0; i < 8; ++i) dmma(acc[i][0], acc[i][1], av, bv);
    double z = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) z += acc[i][0] + acc[i][1];
    if (z == 1234.5) sink[0] = z;
  }
}

template <int W2, int K, int NG>
void run(long long* d, double* s, int mode, int warps, const char* what) {
  const int panels = 64;
  long long h;
  k_gw<W2, K, NG><<<1, 32 * warps>>>(d, s, 4, mode);
  k_gw<W2, K, NG><<<1, 32 * warps>>>(d, s, panels, mode);
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%-60s %.0f cycles per generation\n", what, (double)h / (panels * 8));
}

int main() {
  long long* d;
  double* s;
  cudaMalloc(&d, 64);
  cudaMalloc(&s, 8);
  run<0, 32, 1>(d, s, 0, 8, "1 gen warp, 128 rows x 8, alone");
  run<0, 32, 1>(d, s, 1, 8, "1 gen warp, 128 rows x 8, 7 DMMA warps");
  run<0, 4, 1>(d, s, 0, 8, "1 gen warp, 16 rows x 8, alone");
  run<0, 4, 8>(d, s, 0, 8, "8 gen warps, 16 rows x 8, no DMMA");
  run<0, 4, 8>(d, s, 1, 16, "8 gen warps, 16 rows x 8, 8 DMMA warps");
  run<1, 4, 8>(d, s, 1, 16, "8 gen warps, 16 rows x 16 (L2 next block), 8 DMMA warps");
  run<0, 8, 8>(d, s, 1, 16, "8 gen warps, 32 rows x 8, 8 DMMA warps");
  run<0, 8, 4>(d, s, 1, 12, "4 gen warps, 32 rows x 8, 8 DMMA warps");
  run<0, 4, 8>(d, s, 1, 12, "8 gen warps, 16 rows x 8, 4 DMMA warps");
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
