// FP64 TSQR / CAQR kernels for B200 (sm_100a) and their C-ABI.
//
// Kernels (all FP64, see tsqr_device.cuh for the register layout):
//   k_leaf_factor   : one CTA per leaf row-block: dense first tile (CTA sweep)
//                     then the flat chain of triangle-on-rectangle tiles as a
//                     warp ring.  Reads A once; writes R (and optionally the
//                     implicit-Q storage Y, tau).            [SURVEY 8(a) a3,a10]
//   k_tree_factor   : one CTA per combine event of one tree level: QR of two
//                     stacked n x n triangles on the sparsity profile.  [a9]
//   k_tree_apply    : Q or Q^T of a stacked node factor applied to the two
//                     n-row blocks of C it acts on (tree walk / CAQR).  [a11,a12]
//   k_leaf_apply    : Q or Q^T of a leaf chain applied to the leaf's rows of C
//                     (explicit Q, implicit-Q apply, CAQR trailing update). [a6,a12]
//   k_block_factor  : single-CTA DENSE / TRIRECT factorization of a small block
//                     (kernel-level API mirrors of qr_unblocked, qr_triangle_on_rect).
//   k_peak_probe    : DFMA / DMMA throughput microbenchmark.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "tsqr_device.cuh"
#include "../../include/caqr_sm100.h"

using namespace tsqr;

// ---------------------------------------------------------------------------
// error plumbing
// ---------------------------------------------------------------------------
static thread_local char g_err[512];
static int set_err(int code, const char* msg) {
  snprintf(g_err, sizeof(g_err), "%s", msg);
  return code;
}
static int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    snprintf(g_err, sizeof(g_err), "%s: %s", what, cudaGetErrorString(e));
    return CAQR_ERR_CUDA;
  }
  return CAQR_OK;
}
static int padded(int64_t n) { return n <= 32 ? 32 : (n <= 64 ? 64 : (n <= 128 ? 128 : 0)); }

// ---------------------------------------------------------------------------
// leaf factorization
// ---------------------------------------------------------------------------
// Ring warps per CTA for the chain kernel (tunable: 8 warps x 255 registers
// or 12 warps x 168 registers; the register file is split over 4 SMSPs).
static int g_ring_warps = 8;

template <int NP>
struct DenseSmem {
  static constexpr int HW = Geo<NP>::HW;
  static constexpr size_t bytes = sizeof(double) * ((size_t)WARPS * NP + WARPS * HW + WARPS + 2);
};
template <int NP, int RWN>
struct ChainSmem {
  static constexpr int HW = Geo<NP>::HW;
  static constexpr size_t bytes =
      sizeof(double) * ((size_t)NP * NP + RWN * HW) + sizeof(int) * NP;
};

// Dense first tile of every leaf: rows [0, H0) (zero padded), CTA sweep.
// Writes the leaf's R into its slot, tile 0 of Y (LAPACK layout) and tau.
template <int NP>
__global__ void __launch_bounds__(THREADS, 1)
k_leaf_dense(const double* __restrict__ A, int64_t lda, int64_t m, int n, int P, int64_t base,
             double* Y, int64_t ldy, double* tau, int64_t tau_stride, double* Rout, int* flag) {
  constexpr int S = Geo<NP>::S, HW = Geo<NP>::HW;
  extern __shared__ __align__(16) double sm[];
  double* part = sm;
  double* vbuf = part + WARPS * NP;
  double* red = vbuf + WARPS * HW;
  double* sx0 = red + WARPS;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  bool bad = false;
  const int leaf = blockIdx.x;
  const int64_t r0 = (int64_t)leaf * base;
  const int64_t b = (leaf == P - 1) ? m - r0 : base;
  double* tl = tau ? tau + (int64_t)leaf * tau_stride : nullptr;
  double X[HW][S];
  const int valid = (int)min64((int64_t)HW, b - (int64_t)w * HW);
  load_rows<HW, S>(X, A + (r0 + (int64_t)w * HW) * lda, lda, valid, n, 0, bad);
  cta_factor<NP, HW, DENSE>(X, nullptr, n, tl, red, sx0, part, vbuf);
  if (Y) store_rows<HW, S>(X, Y + (r0 + (int64_t)w * HW) * ldy, ldy, valid, n, 0);
  double* Ro = Rout + (int64_t)leaf * n * n;
#pragma unroll
  for (int k = 0; k < HW; ++k) {
    const int r = w * HW + k;
    if (r < n) {
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const int c = 32 * s + lane;
        if (c < n) Ro[r * n + c] = (c >= r) ? X[k][s] : 0.0;
      }
    }
  }
  if (bad && flag) atomicOr(flag, 1);
}

// Flat chain of triangle-on-rectangle tiles after the dense tile, as a warp
// ring: R starts from the leaf's slot and is written back to it.
template <int NP, int RING_WARPS>
__global__ void __launch_bounds__(RING_WARPS * 32, 1)
k_leaf_chain(const double* __restrict__ A, int64_t lda, int64_t m, int n, int P, int64_t base,
             double* Y, int64_t ldy, double* tau, int64_t tau_stride, double* Rio, int* flag) {
  constexpr int S = Geo<NP>::S, HW = Geo<NP>::HW, H0 = WARPS * HW;
  constexpr int NT = RING_WARPS * 32;
  extern __shared__ __align__(16) double sm[];
  double* Rs = sm;
  double* vbuf = Rs + NP * NP;
  int* ver = reinterpret_cast<int*>(vbuf + RING_WARPS * HW);
  const int w = threadIdx.x >> 5;
  bool bad = false;
  const int leaf = blockIdx.x;
  const int64_t r0 = (int64_t)leaf * base;
  const int64_t b = (leaf == P - 1) ? m - r0 : base;
  const int64_t rest = b - H0;
  const int T = rest > 0 ? (int)((rest + HW - 1) / HW) : 0;
  if (T == 0) return;
  double* tl = tau ? tau + (int64_t)leaf * tau_stride : nullptr;
  double* Rl = Rio + (int64_t)leaf * n * n;
  for (int idx = threadIdx.x; idx < NP * NP; idx += NT) {
    const int r = idx / NP, c = idx - r * NP;
    Rs[idx] = (r < n && c < n && c >= r) ? Rl[r * n + c] : 0.0;
  }
  for (int j = threadIdx.x; j < NP; j += NT) ver[j] = 0;
  __syncthreads();
  double X[HW][S];
  for (int t = w; t < T; t += RING_WARPS) {
    const int64_t row = r0 + H0 + (int64_t)t * HW;
    const int valid = (int)min64((int64_t)HW, r0 + b - row);
    load_rows<HW, S>(X, A + row * lda, lda, valid, n, 0, bad);
    ring_factor_tile<NP, HW>(X, Rs, ver, vbuf + w * HW, n, t, tl ? tl + (int64_t)(t + 1) * n : nullptr);
    if (Y) store_rows<HW, S>(X, Y + row * ldy, ldy, valid, n, 0);
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < n * n; idx += NT) {
    const int r = idx / n, c = idx - r * n;
    Rl[idx] = (c >= r) ? Rs[r * NP + c] : 0.0;
  }
  if (bad && flag) atomicOr(flag, 1);
}

// ---------------------------------------------------------------------------
// tree combine: [R_a; R_b] -> R_a' with STACKED factor (Ybot, tau)
// events: int32 triples (receiver slot, partner slot, node id)
// ---------------------------------------------------------------------------
template <int NP>
struct TreeSmem {
  static constexpr int RW = NP / WARPS;
  static constexpr size_t bytes = sizeof(double) * ((size_t)NP * NP + WARPS * NP + WARPS * RW + WARPS + 2);
};

template <int NP>
__global__ void __launch_bounds__(THREADS, 1)
k_tree_factor(double* Rslots, int n, const int* __restrict__ ev, double* Ynode, double* taunode) {
  constexpr int S = NP / 32, RW = NP / WARPS;
  extern __shared__ __align__(16) double sm[];
  double* Ps = sm;
  double* part = Ps + NP * NP;
  double* vbuf = part + WARPS * NP;
  double* red = vbuf + WARPS * RW;
  double* sx0 = red + WARPS;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int a = ev[3 * blockIdx.x], b = ev[3 * blockIdx.x + 1], id = ev[3 * blockIdx.x + 2];
  const double* Ra = Rslots + (int64_t)a * n * n;
  const double* Rb = Rslots + (int64_t)b * n * n;
  for (int idx = threadIdx.x; idx < NP * NP; idx += THREADS) {
    const int r = idx / NP, c = idx - r * NP;
    Ps[idx] = (r < n && c < n && c >= r) ? Ra[r * n + c] : 0.0;
  }
  double X[RW][S];
#pragma unroll
  for (int k = 0; k < RW; ++k) {
    const int r = w * RW + k;
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int c = 32 * s + lane;
      X[k][s] = (r < n && c < n && c >= r) ? Rb[r * n + c] : 0.0;
    }
  }
  __syncthreads();
  cta_factor<NP, RW, STACKED>(X, Ps, n, taunode + (int64_t)id * n, red, sx0, part, vbuf);
  __syncthreads();
  double* Ro = Rslots + (int64_t)a * n * n;
  for (int idx = threadIdx.x; idx < n * n; idx += THREADS) {
    const int r = idx / n, c = idx - r * n;
    Ro[idx] = (c >= r) ? Ps[r * NP + c] : 0.0;
  }
  double* Yo = Ynode + (int64_t)id * n * n;
#pragma unroll
  for (int k = 0; k < RW; ++k) {
    const int r = w * RW + k;
    if (r >= n) continue;
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int c = 32 * s + lane;
      if (c < n) Yo[r * n + c] = X[k][s];
    }
  }
}

// ---------------------------------------------------------------------------
// tree apply: [C_a; C_b] <- Q_node^(T?) [C_a; C_b] on one column block.
// C_a = C + a*slot_rows*ldc, C_b = C + b*slot_rows*ldc (n rows each).
// ---------------------------------------------------------------------------
template <int NP, int KBS>
struct TreeApplySmem {
  static constexpr size_t bytes = sizeof(double) * ((size_t)NP * 32 * KBS + 2 * WARPS * 32 * KBS);
};

template <int NP, int KBS, bool TRANS>
__global__ void __launch_bounds__(THREADS, 1)
k_tree_apply(const double* __restrict__ Ynode, const double* __restrict__ taunode, int n,
             const int* __restrict__ ev, double* C, int64_t ldc, int64_t slot_rows, int64_t ncols,
             int zero_partner) {
  constexpr int RW = NP / WARPS, KB = 32 * KBS;
  extern __shared__ __align__(16) double sm[];
  double* Ps = sm;
  double* part = Ps + NP * KB;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int a = ev[3 * blockIdx.x], b = ev[3 * blockIdx.x + 1], id = ev[3 * blockIdx.x + 2];
  const int col0 = blockIdx.y * KB;
  double* Ca = C + (int64_t)a * slot_rows * ldc;
  double* Cb = C + (int64_t)b * slot_rows * ldc;
  for (int idx = threadIdx.x; idx < NP * KB; idx += THREADS) {
    const int r = idx / KB, c = idx - r * KB;
    Ps[idx] = (r < n && col0 + c < ncols) ? Ca[(int64_t)r * ldc + col0 + c] : 0.0;
  }
  double X[RW][KBS];
  bool bad = false;
  if (zero_partner) {
#pragma unroll
    for (int k = 0; k < RW; ++k)
#pragma unroll
      for (int s = 0; s < KBS; ++s) X[k][s] = 0.0;
  } else {
    const int valid = max(0, min(RW, n - w * RW));
    load_rows<RW, KBS>(X, Cb + (int64_t)w * RW * ldc + col0, ldc, valid,
                       (int)min64(ncols - col0, KB), 0, bad);
  }
  __syncthreads();
  const double* Yn = Ynode + (int64_t)id * n * n;
  auto ycol = [&](int r, int j) { return __ldg(Yn + (int64_t)r * n + j); };
  cta_apply<RW, KBS, STACKED, TRANS>(X, Ps, n, ycol, taunode + (int64_t)id * n, part, col0, false);
  __syncthreads();
  for (int idx = threadIdx.x; idx < n * KB; idx += THREADS) {
    const int r = idx / KB, c = idx - r * KB;
    if (col0 + c < ncols) Ca[(int64_t)r * ldc + col0 + c] = Ps[r * KB + c];
  }
  const int valid = max(0, min(RW, n - w * RW));
  store_rows<RW, KBS>(X, Cb + (int64_t)w * RW * ldc + col0, ldc, valid,
                      (int)min64(ncols - col0, KB), 0);
}

// ---------------------------------------------------------------------------
// leaf apply: C[leaf rows] <- Q_leaf^(T?) C[leaf rows], one column block per CTA.
// Qt: dense tile 0 forward, then the ring forward over the chain tiles.
// Q : ring backward over the chain tiles, then dense tile 0 backward.
// S (nullable): source of the leaf's top n rows for Q (explicit-Q formation),
// leaf i's block at S + i*s_slot_rows*lds.  zero_init: C tiles start at zero.
// ---------------------------------------------------------------------------
template <int NP, int KBS>
struct LeafApplySmem {
  static constexpr size_t bytes =
      sizeof(double) * ((size_t)NP * 32 * KBS + 2 * WARPS * 32 * KBS) + sizeof(int) * NP;
};

template <int NP, int KBS, bool TRANS>
__global__ void __launch_bounds__(THREADS, 1)
k_leaf_apply(const double* __restrict__ Y, int64_t ldy, const double* __restrict__ tau,
             int64_t tau_stride, int64_t m, int n, int P, int64_t base, double* C, int64_t ldc,
             int64_t ncols, const double* __restrict__ S, int64_t lds, int64_t s_slot_rows,
             int zero_init, int tri_skip) {
  constexpr int HW = Geo<NP>::HW, H0 = WARPS * HW, KB = 32 * KBS;
  extern __shared__ __align__(16) double sm[];
  double* Cs = sm;
  double* part = Cs + NP * KB;
  int* ver = reinterpret_cast<int*>(part + 2 * WARPS * KB);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int leaf = blockIdx.x;
  const int col0 = blockIdx.y * KB;
  const int ncb = (int)min64(ncols - col0, KB);
  const int64_t r0 = (int64_t)leaf * base;
  const int64_t b = (leaf == P - 1) ? m - r0 : base;
  const double* tl = tau + (int64_t)leaf * tau_stride;
  const double* Yl = Y + r0 * ldy;
  double* Cl = C + r0 * ldc + col0;
  const int64_t rest = b - H0;
  const int T = rest > 0 ? (int)((rest + HW - 1) / HW) : 0;
  const bool tskip = tri_skip != 0;
  bool bad = false;
  double X[HW][KBS];
  auto ycol = [&](int r, int j) { return (r < b) ? __ldg(Yl + (int64_t)r * ldy + j) : 0.0; };
  const int v0 = (int)max64(0, min64((int64_t)HW, b - (int64_t)w * HW));
  if (TRANS) {
    load_rows<HW, KBS>(X, Cl + (int64_t)w * HW * ldc, ldc, v0, ncb, 0, bad);
    cta_apply<HW, KBS, DENSE, true>(X, nullptr, n, ycol, tl, part, col0, false);
    // rows < n become the ring's pivot rows; rows >= n are final
#pragma unroll
    for (int k = 0; k < HW; ++k) {
      const int r = w * HW + k;
      if (r < NP) {
#pragma unroll
        for (int s = 0; s < KBS; ++s) Cs[r * KB + 32 * s + lane] = (r < n) ? X[k][s] : 0.0;
      }
    }
    {
      const int lo = max(0, n - w * HW);
      store_rows<HW, KBS>(X, Cl + (int64_t)w * HW * ldc, ldc, v0, ncb, 0, lo);
    }
    for (int j = threadIdx.x; j < NP; j += THREADS) ver[j] = 0;
    __syncthreads();
    for (int t = w; t < T; t += WARPS) {
      const int64_t row = H0 + (int64_t)t * HW;
      const int valid = (int)min64((int64_t)HW, b - row);
      load_rows<HW, KBS>(X, Cl + row * ldc, ldc, valid, ncb, 0, bad);
      ring_apply_tile<HW, KBS, true>(X, Cs, ver, Yl + row * ldy, ldy, valid, tl + (int64_t)(t + 1) * n,
                                     n, t, col0, false);
      store_rows<HW, KBS>(X, Cl + row * ldc, ldc, valid, ncb, 0);
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < n * KB; idx += THREADS) {
      const int r = idx / KB, c = idx - r * KB;
      if (c < ncb) Cl[(int64_t)r * ldc + c] = Cs[idx];
    }
  } else {
    const double* Sl = S ? S + (int64_t)leaf * s_slot_rows * lds + col0 : nullptr;
    for (int idx = threadIdx.x; idx < NP * KB; idx += THREADS) {
      const int r = idx / KB, c = idx - r * KB;
      double x = 0.0;
      if (r < n && c < ncb) x = Sl ? Sl[(int64_t)r * lds + c] : Cl[(int64_t)r * ldc + c];
      Cs[idx] = x;
    }
    for (int j = threadIdx.x; j < NP; j += THREADS) ver[j] = 0;
    __syncthreads();
    for (int o = w; o < T; o += WARPS) {
      const int t = T - 1 - o;
      const int64_t row = H0 + (int64_t)t * HW;
      const int valid = (int)min64((int64_t)HW, b - row);
      if (zero_init) {
#pragma unroll
        for (int k = 0; k < HW; ++k)
#pragma unroll
          for (int s = 0; s < KBS; ++s) X[k][s] = 0.0;
      } else {
        load_rows<HW, KBS>(X, Cl + row * ldc, ldc, valid, ncb, 0, bad);
      }
      ring_apply_tile<HW, KBS, false>(X, Cs, ver, Yl + row * ldy, ldy, valid, tl + (int64_t)(t + 1) * n,
                                      n, o, col0, tskip);
      store_rows<HW, KBS>(X, Cl + row * ldc, ldc, valid, ncb, 0);
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < HW; ++k) {
      const int r = w * HW + k;
#pragma unroll
      for (int s = 0; s < KBS; ++s) {
        double x = 0.0;
        if (r < n) x = Cs[r * KB + 32 * s + lane];
        else if (!zero_init && k < v0 && 32 * s + lane < ncb) x = Cl[(int64_t)r * ldc + 32 * s + lane];
        X[k][s] = x;
      }
    }
    __syncthreads();
    cta_apply<HW, KBS, DENSE, false>(X, nullptr, n, ycol, tl, part, col0, tskip);
    store_rows<HW, KBS>(X, Cl + (int64_t)w * HW * ldc, ldc, v0, ncb, 0);
  }
}

// ---------------------------------------------------------------------------
// small single-CTA factorizations for the kernel-level API mirrors
//   DENSE  : QR of a block of up to WARPS*RW rows (qr_unblocked)
//   TRIRECT: QR of [R; B] with B up to WARPS*RW rows (qr_triangle_on_rect)
// ---------------------------------------------------------------------------
template <int NP, int RW, int MODE>
__global__ void __launch_bounds__(THREADS, 1)
k_block_factor(const double* __restrict__ A, int64_t lda, int rows, int n, double* Rio,
               double* Yout, int64_t ldy, double* tau, int* flag) {
  constexpr int S = NP / 32;
  extern __shared__ __align__(16) double sm[];
  double* Ps = sm;
  double* part = Ps + NP * NP;
  double* vbuf = part + WARPS * NP;
  double* red = vbuf + WARPS * RW;
  double* sx0 = red + WARPS;
  const int w = threadIdx.x >> 5;
  bool bad = false;
  if (MODE == TRIRECT || MODE == STACKEDQ) {
    for (int idx = threadIdx.x; idx < NP * NP; idx += THREADS) {
      const int r = idx / NP, c = idx - r * NP;
      Ps[idx] = (r < n && c < n && c >= r) ? Rio[r * n + c] : 0.0;
    }
  }
  double X[RW][S];
  const int valid = max(0, min(RW, rows - w * RW));
  load_rows<RW, S>(X, A + (int64_t)w * RW * lda, lda, valid, n, 0, bad);
  __syncthreads();
  cta_factor<NP, RW, MODE>(X, Ps, n, tau, red, sx0, part, vbuf);
  __syncthreads();
  store_rows<RW, S>(X, Yout + (int64_t)w * RW * ldy, ldy, valid, n, 0);
  if (MODE == DENSE) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int k = 0; k < RW; ++k) {
      const int r = w * RW + k;
      if (r >= n) continue;
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const int c = 32 * s + lane;
        if (c < n) Rio[r * n + c] = (c >= r) ? X[k][s] : 0.0;
      }
    }
  }
  if (MODE == TRIRECT || MODE == STACKEDQ) {
    for (int idx = threadIdx.x; idx < n * n; idx += THREADS) {
      const int r = idx / n, c = idx - r * n;
      Rio[idx] = (c >= r) ? Ps[r * NP + c] : 0.0;
    }
  }
  if (bad && flag) atomicOr(flag, 1);
}

// Single-CTA application of a DENSE (rows <= 128) or TRIRECT (rectangle rows
// <= 128) factor: C block rows in registers; for TRIRECT the n pivot rows Ct
// (the identity-top part of the factor) live in shared memory.
template <int RW, int KBS, int MODE, bool TRANS>
__global__ void __launch_bounds__(THREADS, 1)
k_block_apply(const double* __restrict__ Yf, int64_t ldy, int rows, int n,
              const double* __restrict__ tau, double* Ct, int64_t ldt, double* C, int64_t ldc,
              int64_t ncols) {
  constexpr int KB = 32 * KBS;
  extern __shared__ __align__(16) double sm[];
  double* Ps = sm;
  double* part = Ps + 128 * KB;
  const int w = threadIdx.x >> 5;
  const int col0 = blockIdx.x * KB;
  const int ncb = (int)min64(ncols - col0, KB);
  if (MODE == TRIRECT) {
    for (int idx = threadIdx.x; idx < 128 * KB; idx += THREADS) {
      const int r = idx / KB, c = idx - r * KB;
      Ps[idx] = (r < n && c < ncb) ? Ct[(int64_t)r * ldt + col0 + c] : 0.0;
    }
  }
  double X[RW][KBS];
  bool bad = false;
  const int valid = max(0, min(RW, rows - w * RW));
  load_rows<RW, KBS>(X, C + (int64_t)w * RW * ldc + col0, ldc, valid, ncb, 0, bad);
  __syncthreads();
  auto ycol = [&](int r, int j) { return (r < rows) ? __ldg(Yf + (int64_t)r * ldy + j) : 0.0; };
  cta_apply<RW, KBS, MODE, TRANS>(X, Ps, n, ycol, tau, part, col0, false);
  __syncthreads();
  store_rows<RW, KBS>(X, C + (int64_t)w * RW * ldc + col0, ldc, valid, ncb, 0);
  if (MODE == TRIRECT) {
    for (int idx = threadIdx.x; idx < n * KB; idx += THREADS) {
      const int r = idx / KB, c = idx - r * KB;
      if (c < ncb) Ct[(int64_t)r * ldt + col0 + c] = Ps[idx];
    }
  }
}

// ---------------------------------------------------------------------------
// FP64 pipe microbenchmark: DFMA chains vs DMMA m8n8k4.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_peak_dfma(double* out, int iters) {
  double a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-7 + i;
  const double b = 1.0000001, c = 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fma(a[i], b, c);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void __launch_bounds__(256) k_peak_dmma(double* out, int iters) {
  double acc[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { acc[i][0] = 0.0; acc[i][1] = 0.0; }
  const double av = 1.0 + threadIdx.x * 1e-9, bv = 0.5;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(av), "d"(bv));
    }
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.678) out[0] = s;
}

// ===========================================================================
// C-ABI
// ===========================================================================
template <class K>
static int prep(K kernel, size_t smem) {
  static_assert(sizeof(K) > 0, "");
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) {
    snprintf(g_err, sizeof(g_err), "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    return CAQR_ERR_CUDA;
  }
  return CAQR_OK;
}

extern "C" {

int caqr_sm100_abi_version(void) { return CAQR_SM100_ABI_VERSION; }

const char* tsqr_last_error(void) { return g_err; }

int tsqr_f64_geometry(int64_t n, int64_t* np, int64_t* h0, int64_t* ht) {
  const int p = padded(n);
  if (n < 1 || !p) return set_err(CAQR_ERR_ARG, "n must be in [1, 128]");
  int hw = p == 32 ? Geo<32>::HW : (p == 64 ? Geo<64>::HW : Geo<128>::HW);
  if (np) *np = p;
  if (ht) *ht = hw;
  if (h0) *h0 = (int64_t)WARPS * hw;
  return CAQR_OK;
}

int tsqr_f64_leaf_factor(const double* A, int64_t lda, int64_t m, int64_t n, int64_t P, double* Y,
                         int64_t ldy, double* tau, int64_t tau_stride, double* R, int* flag,
                         void* stream) {
  const int p = padded(n);
  if (!p || !A || !R || P < 1 || m < n * P || lda < n || (Y && ldy < n))
    return set_err(CAQR_ERR_ARG, "tsqr_f64_leaf_factor: bad arguments");
  if ((Y == nullptr) != (tau == nullptr)) return set_err(CAQR_ERR_ARG, "Y and tau go together");
  const int64_t base = m / P;
  if (base < n) return set_err(CAQR_ERR_ARG, "leaf shorter than n");
  cudaStream_t st = (cudaStream_t)stream;
  const int grid = (int)P;
#define CHAIN_LAUNCH(NPV, RWN)                                                                  \
  {                                                                                             \
    rc = prep(k_leaf_chain<NPV, RWN>, ChainSmem<NPV, RWN>::bytes);                              \
    if (rc) return rc;                                                                          \
    k_leaf_chain<NPV, RWN><<<grid, RWN * 32, ChainSmem<NPV, RWN>::bytes, st>>>(A, lda, m,       \
        (int)n, (int)P, base, Y, ldy, tau, tau_stride, R, flag);                                \
  }
#define LEAF_CASE(NPV)                                                                          \
  case NPV: {                                                                                   \
    int rc = prep(k_leaf_dense<NPV>, DenseSmem<NPV>::bytes);                                    \
    if (rc) return rc;                                                                          \
    k_leaf_dense<NPV><<<grid, THREADS, DenseSmem<NPV>::bytes, st>>>(A, lda, m, (int)n, (int)P,  \
        base, Y, ldy, tau, tau_stride, R, flag);                                                \
    if (m - base * (P - 1) > (int64_t)WARPS * Geo<NPV>::HW) {                                    \
      if (g_ring_warps == 12) CHAIN_LAUNCH(NPV, 12) else CHAIN_LAUNCH(NPV, 8)                   \
    }                                                                                           \
    break;                                                                                      \
  }
  switch (p) { LEAF_CASE(32) LEAF_CASE(64) LEAF_CASE(128) }
#undef LEAF_CASE
#undef CHAIN_LAUNCH
  return check_launch("k_leaf_dense/k_leaf_chain");
}

int tsqr_f64_tree_factor_level(double* Rslots, int64_t n, const int32_t* events, int64_t nev,
                               double* Ynode, double* taunode, void* stream) {
  const int p = padded(n);
  if (!p || !Rslots || !events || !Ynode || !taunode || nev < 0)
    return set_err(CAQR_ERR_ARG, "tsqr_f64_tree_factor_level: bad arguments");
  if (nev == 0) return CAQR_OK;
  cudaStream_t st = (cudaStream_t)stream;
#define TREE_CASE(NPV)                                                                   \
  case NPV: {                                                                            \
    int rc = prep(k_tree_factor<NPV>, TreeSmem<NPV>::bytes);                             \
    if (rc) return rc;                                                                   \
    k_tree_factor<NPV><<<(int)nev, THREADS, TreeSmem<NPV>::bytes, st>>>(Rslots, (int)n,  \
        events, Ynode, taunode);                                                         \
    break;                                                                               \
  }
  switch (p) { TREE_CASE(32) TREE_CASE(64) TREE_CASE(128) }
#undef TREE_CASE
  return check_launch("k_tree_factor");
}

int tsqr_f64_tree_apply_level(const double* Ynode, const double* taunode, int64_t n,
                              const int32_t* events, int64_t nev, double* C, int64_t ldc,
                              int64_t slot_rows, int64_t ncols, int transpose, int zero_partner,
                              void* stream) {
  const int p = padded(n);
  if (!p || !Ynode || !taunode || !events || !C || ncols < 1 || ldc < ncols)
    return set_err(CAQR_ERR_ARG, "tsqr_f64_tree_apply_level: bad arguments");
  if (nev == 0) return CAQR_OK;
  cudaStream_t st = (cudaStream_t)stream;
  constexpr int KBS = 2;
  dim3 grid((unsigned)nev, (unsigned)((ncols + 32 * KBS - 1) / (32 * KBS)));
#define TA_CASE(NPV)                                                                            \
  case NPV: {                                                                                   \
    const size_t sm = TreeApplySmem<NPV, KBS>::bytes;                                           \
    if (transpose) {                                                                            \
      int rc = prep(k_tree_apply<NPV, KBS, true>, sm); if (rc) return rc;                       \
      k_tree_apply<NPV, KBS, true><<<grid, THREADS, sm, st>>>(Ynode, taunode, (int)n, events,   \
          C, ldc, slot_rows, ncols, zero_partner);                                              \
    } else {                                                                                    \
      int rc = prep(k_tree_apply<NPV, KBS, false>, sm); if (rc) return rc;                      \
      k_tree_apply<NPV, KBS, false><<<grid, THREADS, sm, st>>>(Ynode, taunode, (int)n, events,  \
          C, ldc, slot_rows, ncols, zero_partner);                                              \
    }                                                                                           \
    break;                                                                                      \
  }
  switch (p) { TA_CASE(32) TA_CASE(64) TA_CASE(128) }
#undef TA_CASE
  return check_launch("k_tree_apply");
}

int tsqr_f64_leaf_apply(const double* Y, int64_t ldy, const double* tau, int64_t tau_stride,
                        int64_t m, int64_t n, int64_t P, double* C, int64_t ldc, int64_t ncols,
                        const double* S, int64_t lds, int64_t s_slot_rows, int transpose,
                        int zero_init, int tri_skip, void* stream) {
  const int p = padded(n);
  if (!p || !Y || !tau || !C || P < 1 || m < n * P || ncols < 1 || ldc < ncols)
    return set_err(CAQR_ERR_ARG, "tsqr_f64_leaf_apply: bad arguments");
  if (transpose && (S || zero_init || tri_skip))
    return set_err(CAQR_ERR_ARG, "S / zero_init / tri_skip only apply to Q (not Q^T)");
  const int64_t base = m / P;
  cudaStream_t st = (cudaStream_t)stream;
  const int kbs = (p == 128) ? 4 : 1;
  dim3 grid((unsigned)P, (unsigned)((ncols + 32 * kbs - 1) / (32 * kbs)));
#define LA_CASE(NPV, KB_)                                                                         \
  case NPV: {                                                                                     \
    const size_t sm = LeafApplySmem<NPV, KB_>::bytes;                                             \
    if (transpose) {                                                                              \
      int rc = prep(k_leaf_apply<NPV, KB_, true>, sm); if (rc) return rc;                         \
      k_leaf_apply<NPV, KB_, true><<<grid, THREADS, sm, st>>>(Y, ldy, tau, tau_stride, m, (int)n, \
          (int)P, base, C, ldc, ncols, S, lds, s_slot_rows, zero_init, tri_skip);                 \
    } else {                                                                                      \
      int rc = prep(k_leaf_apply<NPV, KB_, false>, sm); if (rc) return rc;                        \
      k_leaf_apply<NPV, KB_, false><<<grid, THREADS, sm, st>>>(Y, ldy, tau, tau_stride, m,        \
          (int)n, (int)P, base, C, ldc, ncols, S, lds, s_slot_rows, zero_init, tri_skip);         \
    }                                                                                             \
    break;                                                                                        \
  }
  switch (p) { LA_CASE(32, 1) LA_CASE(64, 1) LA_CASE(128, 4) }
#undef LA_CASE
  return check_launch("k_leaf_apply");
}

int tsqr_f64_block_factor(const double* A, int64_t lda, int64_t rows, int64_t n, double* R,
                          double* Y, int64_t ldy, double* tau, int mode, int* flag, void* stream) {
  const int p = padded(n);
  if (!p || !A || !R || !Y || !tau || rows < 1 || (mode == 0 && rows < n) ||
      (mode != 0 && mode != 2 && mode != 3))
    return set_err(CAQR_ERR_ARG, "tsqr_f64_block_factor: bad arguments");
  constexpr int RWMAX = 16;
  if (rows > WARPS * RWMAX) return set_err(CAQR_ERR_ARG, "block too tall for the single-CTA kernel");
  cudaStream_t st = (cudaStream_t)stream;
#define BF_CASE(NPV)                                                                            \
  case NPV: {                                                                                   \
    const size_t sm = sizeof(double) * ((size_t)NPV * NPV + WARPS * NPV + WARPS * RWMAX + WARPS + 2); \
    if (mode == 0) {                                                                            \
      int rc = prep(k_block_factor<NPV, RWMAX, DENSE>, sm); if (rc) return rc;                  \
      k_block_factor<NPV, RWMAX, DENSE><<<1, THREADS, sm, st>>>(A, lda, (int)rows, (int)n, R,   \
          Y, ldy, tau, flag);                                                                   \
    } else if (mode == 3) {                                                                     \
      int rc = prep(k_block_factor<NPV, RWMAX, STACKEDQ>, sm); if (rc) return rc;               \
      k_block_factor<NPV, RWMAX, STACKEDQ><<<1, THREADS, sm, st>>>(A, lda, (int)rows, (int)n,   \
          R, Y, ldy, tau, flag);                                                                \
    } else {                                                                                    \
      int rc = prep(k_block_factor<NPV, RWMAX, TRIRECT>, sm); if (rc) return rc;                \
      k_block_factor<NPV, RWMAX, TRIRECT><<<1, THREADS, sm, st>>>(A, lda, (int)rows, (int)n, R, \
          Y, ldy, tau, flag);                                                                   \
    }                                                                                           \
    break;                                                                                      \
  }
  switch (p) { BF_CASE(32) BF_CASE(64) BF_CASE(128) }
#undef BF_CASE
  return check_launch("k_block_factor");
}

int tsqr_f64_block_apply(const double* Y, int64_t ldy, int64_t rows, int64_t n, const double* tau,
                         double* Ctop, int64_t ldt, double* C, int64_t ldc, int64_t ncols, int mode,
                         int transpose, void* stream) {
  if (n < 1 || n > 128 || rows < 1 || rows > 128 || !Y || !tau || !C || ncols < 1 ||
      (mode == 2 && !Ctop) || (mode == 0 && rows < n) || (mode != 0 && mode != 2))
    return set_err(CAQR_ERR_ARG, "tsqr_f64_block_apply: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  constexpr int RW = 16, KBS = 1;
  const size_t sm = sizeof(double) * ((size_t)128 * 32 * KBS + 2 * WARPS * 32 * KBS);
  dim3 grid((unsigned)((ncols + 32 * KBS - 1) / (32 * KBS)));
#define BA_LAUNCH(MD, TR)                                                                      \
  {                                                                                            \
    int rc = prep(k_block_apply<RW, KBS, MD, TR>, sm); if (rc) return rc;                      \
    k_block_apply<RW, KBS, MD, TR><<<grid, THREADS, sm, st>>>(Y, ldy, (int)rows, (int)n, tau,  \
        Ctop, ldt, C, ldc, ncols);                                                             \
  }
  if (mode == 0) { if (transpose) BA_LAUNCH(DENSE, true) else BA_LAUNCH(DENSE, false) }
  else { if (transpose) BA_LAUNCH(TRIRECT, true) else BA_LAUNCH(TRIRECT, false) }
#undef BA_LAUNCH
  return check_launch("k_block_apply");
}

int caqr_tune(int key, int value) {
  if (key == CAQR_TUNE_RING_WARPS) {
    if (value != 8 && value != 12) return set_err(CAQR_ERR_ARG, "ring warps must be 8 or 12");
    g_ring_warps = value;
    return CAQR_OK;
  }
  return set_err(CAQR_ERR_ARG, "unknown tuning key");
}

int caqr_f64_peak_probe(double* scratch, int mode, int iters, int blocks, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (mode == 0) k_peak_dfma<<<blocks, 256, 0, st>>>(scratch, iters);
  else k_peak_dmma<<<blocks, 256, 0, st>>>(scratch, iters);
  return check_launch("k_peak_probe");
}

}  // extern "C"
