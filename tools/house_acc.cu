// Accuracy of the DMMA ring's reflector scalars (house_fast, dmma_ring.cuh):
// max relative error of nrm = sqrt(x0^2 + sigma) and of 1/(|x0| + nrm)
// against long double on the host, over random (x0, sigma) spanning 2^-100..2^100.
#include <cstdio>
#include <cmath>
#include "../paper_0809_2407_b200/csrc/tsqr_device.cuh"
namespace tsqr {
#include "../paper_0809_2407_b200/csrc/dmma_ring.cuh"
}
using namespace tsqr;
__global__ void k(const double* x0, const double* sg, double* nrm, double* sc, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double beta, tau, scale, invb;
  house_fast(x0[i], sg[i], beta, tau, scale, invb);
  nrm[i] = fabs(beta);
  sc[i] = fabs(scale);
}
int main() {
  const int n = 1 << 22;
  double *x, *s, *a, *b;
  cudaMallocManaged(&x, n * 8); cudaMallocManaged(&s, n * 8); cudaMallocManaged(&a, n * 8); cudaMallocManaged(&b, n * 8);
  unsigned long long st = 88172645463325252ull;
  auto rnd = [&]() { st ^= st << 13; st ^= st >> 7; st ^= st << 17; return st; };
  for (int i = 0; i < n; ++i) {
    const int ex = (int)(rnd() % 200) - 100;
    x[i] = ldexp((double)(rnd() >> 11) / 9007199254740992.0 - 0.5, ex);
    s[i] = ldexp((double)(rnd() >> 11) / 9007199254740992.0, ex + (int)(rnd() % 9) - 4);
  }
  k<<<(n + 255) / 256, 256>>>(x, s, a, b, n);
  cudaDeviceSynchronize();
  long double e1 = 0, e2 = 0;
  for (int i = 0; i < n; ++i) {
    if (s[i] == 0.0) continue;
    const long double X = x[i], S = s[i];
    const long double N = sqrtl(X * X + S), R = 1.0L / (fabsl(X) + N);
    e1 = fmaxl(e1, fabsl(a[i] - N) / N);
    e2 = fmaxl(e2, fabsl(b[i] - R) / R);
  }
  printf("house_fast: nrm max rel err %.3Le (%.2Lf ulp), 1/(|x0|+nrm) max rel err %.3Le (%.2Lf ulp)\n", e1,
         e1 / 1.1102230246251565e-16L, e2, e2 / 1.1102230246251565e-16L);
  return 0;
}
