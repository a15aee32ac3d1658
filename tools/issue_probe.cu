// Single-warp issue rate of independent FP64 instructions (is one warp able to keep the
// FP64 pipe of its sub-partition busy?).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/issue_probe tools/issue_probe.cu
#include <cstdio>
template <int NCH>
__global__ void k(long long* out, double* sink, int iters, int warps_active) {
  double a[NCH];
  const double m = 1.0 + 1e-9 * threadIdx.x, c = 1e-3;
#pragma unroll
  for (int i = 0; i < NCH; ++i) a[i] = 1.0 + i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) a[i] = fma(a[i], m, c);
  }
  long long t1 = clock64();
  double z = 0;
#pragma unroll
  for (int i = 0; i < NCH; ++i) z += a[i];
  if (z == 1234.5) sink[0] = z;
  if (threadIdx.x == 0) out[0] = t1 - t0;
}
template <int NCH>
void run(long long* d, double* s, int threads) {
  long long h;
  const int iters = 2000;
  k<NCH><<<1, threads>>>(d, s, 10, 0);
  k<NCH><<<1, threads>>>(d, s, iters, 0);
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%d warps, %2d independent DFMA chains: %.2f cycles per DFMA per warp\n", threads / 32, NCH,
         (double)h / (iters * NCH));
}
int main() {
  long long* d;
  double* s;
  cudaMalloc(&d, 64);
  cudaMalloc(&s, 8);
  run<1>(d, s, 32);
  run<2>(d, s, 32);
  run<4>(d, s, 32);
  run<8>(d, s, 32);
  run<16>(d, s, 32);
  run<8>(d, s, 128);
  run<8>(d, s, 256);
  run<8>(d, s, 512);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
