// Verifies the fragment layout assumed for mma.sync.m8n8k4.f64 (A row, B col):
// A: lane holds A[lane/4][lane%4]; B: lane holds B[lane%4][lane/4];
// C/D: lane holds C[lane/4][2*(lane%4) + {0,1}].
#include <cstdio>
__global__ void k(const double* A, const double* B, double* C) {
  const int l = threadIdx.x;
  double a = A[(l / 4) * 4 + (l % 4)];
  double b = B[(l % 4) * 8 + (l / 4)];
  double c0 = 0.0, c1 = 0.0, d0, d1;
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};"
               : "=d"(d0), "=d"(d1) : "d"(a), "d"(b), "d"(c0), "d"(c1));
  C[(l / 4) * 8 + 2 * (l % 4)] = d0;
  C[(l / 4) * 8 + 2 * (l % 4) + 1] = d1;
}
int main() {
  double hA[32], hB[32], hC[64], ref[64];
  for (int i = 0; i < 32; ++i) { hA[i] = 1.0 + i * 0.5; hB[i] = 2.0 - i * 0.25; }
  for (int r = 0; r < 8; ++r)
    for (int c = 0; c < 8; ++c) {
      double s = 0; for (int k = 0; k < 4; ++k) s += hA[r * 4 + k] * hB[k * 8 + c];
      ref[r * 8 + c] = s;
    }
  double *A, *B, *C; cudaMalloc(&A, 256); cudaMalloc(&B, 256); cudaMalloc(&C, 512);
  cudaMemcpy(A, hA, 256, cudaMemcpyHostToDevice); cudaMemcpy(B, hB, 256, cudaMemcpyHostToDevice);
  k<<<1, 32>>>(A, B, C);
  cudaMemcpy(hC, C, 512, cudaMemcpyDeviceToHost);
  double err = 0; for (int i = 0; i < 64; ++i) err = fmax(err, fabs(hC[i] - ref[i]));
  printf("dmma m8n8k4 layout max err = %g (%s)\n", err, err < 1e-12 ? "OK" : "MISMATCH");
  return 0;
}
