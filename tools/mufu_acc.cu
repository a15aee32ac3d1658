#include <cstdio>
#include <cmath>
__global__ void k(const double* x, double* r1, double* r2, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double a = x[i], y, z;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(z) : "d"(a));
  r1[i] = y; r2[i] = z;
}
int main() {
  const int n = 1 << 20;
  double *x, *r1, *r2; cudaMallocManaged(&x, n * 8); cudaMallocManaged(&r1, n * 8); cudaMallocManaged(&r2, n * 8);
  unsigned long long s = 88172645463325252ull;
  for (int i = 0; i < n; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; x[i] = ldexp((double)(s >> 11) / 9007199254740992.0 + 0.5, (int)(s % 200) - 100); }
  k<<<(n + 255) / 256, 256>>>(x, r1, r2, n); cudaDeviceSynchronize();
  double e1 = 0, e2 = 0;
  for (int i = 0; i < n; ++i) {
    double t1 = 1.0 / sqrt(x[i]), t2 = 1.0 / x[i];
    e1 = fmax(e1, fabs(r1[i] - t1) / t1); e2 = fmax(e2, fabs(r2[i] - t2) / t2);
  }
  printf("rsqrt.approx.f64 max rel err %.3e (2^%.1f)\nrcp.approx.f64   max rel err %.3e (2^%.1f)\n", e1, log2(e1), e2, log2(e2));
}
