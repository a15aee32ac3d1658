// Where a generation's cycles go: tt_gen with clock reads between its phases (one warp alone).
#include <cstdio>
#include "../paper_0809_2407_b200/csrc/tsqr_device.cuh"
namespace tsqr {
#include "../paper_0809_2407_b200/csrc/dmma_ring.cuh"
}
using namespace tsqr;
__device__ long long g_ph[8];
#define TK(v) const long long v = clock64()
template <int I, int K>
__device__ __forceinline__ void gen_p(double (&x)[K], double* Rrow, double* gs, double* taus, double* xs,
                                      long long (&ph)[8]) {
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, q = lane & 3;
  double2* buf = reinterpret_cast<double2*>(xs + (I & 1) * 4 * K) + q;
  TK(t0);
  if (g == I) {
#pragma unroll
    for (int k2 = 0; k2 < K / 2; ++k2) buf[4 * k2] = make_double2(x[2 * k2], x[2 * k2 + 1]);
  }
  const double x0 = Rrow[I];
  const double rgi = Rrow[g];
  __syncwarp();
  double xi[K];
#pragma unroll
  for (int k2 = 0; k2 < K / 2; ++k2) {
    const double2 t = buf[4 * k2];
    xi[2 * k2] = t.x;
    xi[2 * k2 + 1] = t.y;
  }
  double a[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) a[k] = xi[k] * x[k];
  TK(t1);
#pragma unroll
  for (int k = 4; k < K; ++k) a[k & 3] = fma(xi[k], x[k], a[k & 3]);
  double pd = (a[0] + a[1]) + (a[2] + a[3]);
  if (pd == 1234.5678) pd += 1.0;  // force completion before the clock read
  TK(t2);
  pd += __shfl_xor_sync(FULL, pd, 1);
  pd += __shfl_xor_sync(FULL, pd, 2);
  const double s = __shfl_sync(FULL, pd, 4 * I);
  double sdep = s;
  if (sdep == 1234.5678) sdep += 1.0;
  TK(t3);
  double beta, tau, scale, invb;
  house_fast(x0, sdep, beta, tau, scale, invb);
  double dep = scale + invb + tau;
  if (dep == 1234.5678) scale += 1.0;
  TK(t4);
  const double tw = fma(scale, pd, rgi);
  const double wv = tau * tw;
  const bool upd = g > I, own = (g == I);
  const double f = upd ? tw * invb : (own ? scale - 1.0 : 0.0);
#pragma unroll
  for (int k = 0; k < K; ++k) x[k] = fma(f, xi[k], x[k]);
  double* dst = upd ? Rrow + g : (own ? Rrow + I : gs + g * 8 + I);
  *dst = upd ? rgi - wv : (own ? beta : scale * pd);
  taus[I] = tau;
  double xd = x[K - 1];
  if (xd == 1234.5678) x[0] += 1.0;
  TK(t5);
  ph[0] += t1 - t0; ph[1] += t2 - t1; ph[2] += t3 - t2; ph[3] += t4 - t3; ph[4] += t5 - t4;
}
template <int K>
__global__ void k(double* sink, int panels) {
  __shared__ __align__(16) double Rs[80], gsa[72], xsa[8 * K];
  const int lane = threadIdx.x & 31;
  double x[K];
  long long ph[8] = {};
#pragma unroll
  for (int k = 0; k < K; ++k) x[k] = ((((lane * 2654435761u) ^ (k * 40503u + 12345u)) * 2246822519u >> 8) & 0xffff) / 32768.0 - 1.0;
  for (int i = lane; i < 80; i += 32) Rs[i] = (i % 11 == 0) ? 30.0 : 0.1;
  __syncwarp();
  for (int p = 0; p < panels; ++p) {
    gen_p<0, K>(x, Rs, gsa, gsa + 64, xsa, ph);
    gen_p<1, K>(x, Rs + 10, gsa, gsa + 64, xsa, ph);
    gen_p<2, K>(x, Rs + 20, gsa, gsa + 64, xsa, ph);
    gen_p<3, K>(x, Rs + 30, gsa, gsa + 64, xsa, ph);
    gen_p<4, K>(x, Rs + 40, gsa, gsa + 64, xsa, ph);
    gen_p<5, K>(x, Rs + 50, gsa, gsa + 64, xsa, ph);
    gen_p<6, K>(x, Rs + 60, gsa, gsa + 64, xsa, ph);
    gen_p<7, K>(x, Rs + 70, gsa, gsa + 64, xsa, ph);
    __syncwarp();
#pragma unroll
    for (int k = 0; k < K; ++k) x[k] = (((((lane + 7 * p) * 2654435761u) ^ (k * 40503u + 12345u + p)) * 2246822519u >> 8) & 0xffff) / 32768.0 - 1.0;
    for (int i = lane; i < 80; i += 32) Rs[i] = (i % 11 == 0) ? 30.0 : 0.1;
    __syncwarp();
  }
  if (lane == 0) for (int i = 0; i < 8; ++i) g_ph[i] = ph[i];
  double z = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) z += x[k];
  if (z == 1234.5) sink[0] = z;
}
template <int K>
void run(double* s) {
  const int panels = 64;
  long long h[8];
  k<K><<<1, 32>>>(s, panels);
  cudaMemcpyFromSymbol(h, g_ph, sizeof(h));
  const double n = panels * 8;
  printf("K=%2d: broadcast (STS, barrier, LDS, first products) %.0f | dot chain + adds %.0f | shuffle reduce + fetch %.0f | "
         "house_fast %.0f | scalars + update + stores %.0f | sum %.0f\n",
         K, h[0] / n, h[1] / n, h[2] / n, h[3] / n, h[4] / n, (h[0] + h[1] + h[2] + h[3] + h[4]) / n);
}
int main() {
  double* s;
  cudaMalloc(&s, 8);
  run<4>(s);
  run<8>(s);
  run<16>(s);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
