// DMMA m8n8k4 f64: dependent-chain latency and per-warp throughput vs independent chains and warps per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_lat tools/dmma_lat.cu
#include <cstdio>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int NCH>
__global__ void k(long long* out, double* sink, int iters) {
  double a[NCH][2];
  const double av = 1.0 + 1e-9 * threadIdx.x, bv = 0.5;
#pragma unroll
  for (int i = 0; i < NCH; ++i) a[i][0] = a[i][1] = i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) dmma(a[i][0], a[i][1], av, bv);
  }
  long long t1 = clock64();
  double z = 0;
#pragma unroll
  for (int i = 0; i < NCH; ++i) z += a[i][0] + a[i][1];
  if (z == 1234.5) sink[0] = z;
  if (threadIdx.x == 0) out[0] = t1 - t0;
}
// accumulator feeds the A operand of the next DMMA (the W -> T^T W -> C chain)
__global__ void k_a(long long* out, double* sink, int iters) {
  double d0 = 1.0, d1 = 2.0;
  const double bv = 0.5;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    double e0 = 0.0, e1 = 0.0;
    dmma(e0, e1, d0, bv);
    d0 = e0;
    d1 = e1;
  }
  long long t1 = clock64();
  if (d0 + d1 == 1234.5) sink[0] = d0;
  if (threadIdx.x == 0) out[0] = t1 - t0;
}
template <int NCH>
void run(long long* d, double* s, int threads) {
  long long h;
  const int iters = 2000;
  k<NCH><<<1, threads>>>(d, s, 10);
  k<NCH><<<1, threads>>>(d, s, iters);
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%2d warps/SM, %2d independent accumulators per warp: %.1f cycles per DMMA per warp\n", threads / 32, NCH,
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
  run<1>(d, s, 128);
  run<4>(d, s, 128);
  run<8>(d, s, 128);
  run<1>(d, s, 256);
  run<2>(d, s, 256);
  run<4>(d, s, 256);
  run<8>(d, s, 256);
  run<4>(d, s, 512);
  long long h;
  k_a<<<1, 32>>>(d, s, 2000);
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("accumulator -> A operand dependent chain: %.1f cycles per DMMA\n", (double)h / 2000);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
