// FP64 TSQR / CAQR kernels for B200 (sm_100a) and their C-ABI.
//
// Kernels (all FP64, see tsqr_device.cuh for the register layout).  Defaults
// for n > 32 run on the FP64 tensor cores (mma.m8n8k4.f64, DMMA):
//   k_leaf_dense    : dense first tile of a leaf that keeps Q (CTA sweep).    [a3]
//   k_leaf_tt       : (tm_tall.cuh) R-only leaves of 64 < n <= 128: split-role ring
//                     with 4 tiles of 64 rows in tensor memory, generation warps +
//                     update warps, CTAs chaining consecutive leaves.  The C3 hot
//                     kernel; <64,1,true> keeps the factors (opt-in format).    [a10]
//   k_leaf_tm / k_leaf_split : (tm_leaf.cuh, split_leaf.cuh) the same ring with 16-row
//                     tiles in tensor memory / shared memory (tuning fallbacks). [a10]
//   k_leaf_dmma     : (dmma_ring.cuh) the leaf's flat chain of
//                     triangle-on-rectangle tiles as a DMMA warp ring, 8-column
//                     Level-2 panels + compact-WY updates; NP = 128 / 64 (/ 32):
//                     the leaves that keep Q (with the panel T for CAQR).       [a10]
//   k_leaf_chain    : the rank-1 warp ring (n <= 32, tuning fallback).        [a10]
//   k_leaf_narrow   : n <= 8, R only: lane-private rows + fused ticket tree.  [C4]
//   k_tree_ring     : R-only stacked combine as a warp ring.                  [a9]
//   k_tree_factor_dmma128 / k_tree_factor_dmma / k_tree_factor / k_tree_factor_w32 :
//                     stacked combine with node factors (dmma: column-block warps,
//                     16 for 64 < n <= 128 in tree_factor128.cuh, 8 for n <= 64).  [a9]
//   k_tree_apply_cp / k_tree_apply_dmma / k_tree_apply / k_tree_apply_w32 : Q or Q^T
//                     of a stacked node on the two n-row blocks of C it acts on
//                     (cp: column-parallel warps, 64 < n <= 128).           [a11,a12]
//   k_leaf_apply_dmma (Q^T, 64 < n <= 128; with the kept panel T: 64-column CTAs,
//                     two per SM), k_leaf_q_dmma (Q, n <= 128; Q^T, n <= 64),
//                     k_tall_apply (both, 64-row chain tiles), k_leaf_apply
//                     (reflector ring): a leaf chain's Q / Q^T on the leaf's rows
//                     of C (explicit Q, apply_q, the CAQR trailing update).   [a6,a12]
//   k_block_factor / k_block_apply : single-CTA DENSE / TRIRECT factorization
//                     and apply of a small block (kernel-level API mirrors).
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
// Chain tile height per padded width (tunable, CAQR_TUNE_CHAIN_HT); it fixes
// the implicit-Q storage format, so factor and apply calls must agree.
static int g_ht[3] = {16, 16, 16};  // NP = 32, 64, 128 (16: the DMMA rings' tile)
static int g_narrow = 3;  // CAQR_TUNE_NARROW: lane-private path for n <= 8, R only (3: K = 8 rows, 2: cp.async K = 4)
static int g_zstart = 1;  // CAQR_TUNE_ZSTART: R-only leaves skip the dense first tile
static int g_dmma = 2;     // CAQR_TUNE_DMMA: n in (32,128] leaves on the DMMA warp ring
static int g_dmma_q = 1;      // CAQR_TUNE_DMMA_Q: Q C of 16-row-tile chain leaves (n <= 128) on the DMMA ring
static int g_dmma_dense = 0;  // CAQR_TUNE_DMMA_DENSE: n <= 64 dense first tiles on DMMA (opt-in, slower)
static int g_dmma_tree_factor = 1;  // CAQR_TUNE_DMMA_TREE_FACTOR: node factors on DMMA (n <= 64: 8 warps, n <= 128: 16)
static int g_dmma_tree = 2;   // CAQR_TUNE_DMMA_TREE: Q / Q^T of the tree nodes on DMMA (2: column-parallel for n > 64)
static int g_dmma_apply = 1;  // CAQR_TUNE_DMMA_APPLY: Q^T of n in (32,128] chain leaves on the DMMA ring
static int g_narrow_pf = 1;   // CAQR_TUNE_NARROW_PF: k_leaf_narrow8 L2 prefetch distance in 256-row steps
static int g_fuse = 148;      // CAQR_TUNE_FUSE: R-only n in (64,128]: CTAs (one per SM) that chain consecutive leaves; 0 off
static int g_cc = 5;          // CAQR_TUNE_CC: R-only n in (64,128] leaves: 5 / 6 split-role ring with 4 / 8 tall
                              // tiles (64 / 32 rows) in TMEM, 4 / 3 with 16 / 12 tiles of 16 rows in TMEM,
                              // 2 split-role ring (smem tiles), 0 DMMA warp ring
static int np_index(int p) { return p == 32 ? 0 : (p == 64 ? 1 : 2); }

template <int NP>
struct DenseSmem {
  static constexpr int HD = Geo<NP>::HD;
  static constexpr size_t bytes = sizeof(double) * ((size_t)WARPS * NP + WARPS * HD + WARPS + 2);
};
template <int NP, int HT>
struct ChainSmem {
  static constexpr int RWN = RingCfg<NP, HT>::WARPS_R;
  static constexpr size_t bytes =
      sizeof(double) * ((size_t)NP * NP + RWN * 2 * HT) + sizeof(int) * NP;
};

// Dense first tile of every leaf: rows [0, H0) (zero padded), CTA sweep.
// Writes the leaf's R into its slot, tile 0 of Y (LAPACK layout) and tau.
// NP = 64: two CTAs per SM (128 registers, 480 B of spills) -- C2's 256 leaves in one wave
// instead of two: 3.275 -> 3.211 ms per step
template <int NP>
__global__ void __launch_bounds__(THREADS, NP == 64 ? 2 : 1)
k_leaf_dense(const double* __restrict__ A, int64_t lda, int64_t m, int n, int P, int64_t base,
             double* Y, int64_t ldy, double* tau, int64_t tau_stride, double* Rout, int* flag) {
  constexpr int S = Geo<NP>::S, HD = Geo<NP>::HD;
  extern __shared__ __align__(16) double sm[];
  double* part = sm;
  double* vbuf = part + WARPS * NP;
  double* red = vbuf + WARPS * HD;
  double* sx0 = red + WARPS;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  bool bad = false;
  const int leaf = blockIdx.x;
  const int64_t r0 = (int64_t)leaf * base;
  const int64_t b = (leaf == P - 1) ? m - r0 : base;
  double* tl = tau ? tau + (int64_t)leaf * tau_stride : nullptr;
  double X[HD][S];
  const int valid = (int)min64((int64_t)HD, b - (int64_t)w * HD);
  load_rows<HD, S>(X, A + (r0 + (int64_t)w * HD) * lda, lda, valid, n, 0, bad);
  cta_factor<NP, HD, DENSE>(X, nullptr, n, tl, red, sx0, part, vbuf);
  if (Y) store_rows<HD, S>(X, Y + (r0 + (int64_t)w * HD) * ldy, ldy, valid, n, 0);
  double* Ro = Rout + (int64_t)leaf * n * n;
#pragma unroll
  for (int k = 0; k < HD; ++k) {
    const int r = w * HD + k;
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
template <int NP, int HT>
__global__ void __launch_bounds__(RingCfg<NP, HT>::WARPS_R * 32, 1)
k_leaf_chain(const double* __restrict__ A, int64_t lda, int64_t m, int n, int P, int64_t base,
             double* Y, int64_t ldy, double* tau, int64_t tau_stride, double* Rio, int* flag,
             int zstart) {
  // zstart (R only): no dense first tile -- the chain starts from R = 0 at
  // the leaf's first row (the QR of [0; A_leaf] has the same R up to signs).
  constexpr int S = Geo<NP>::S, HW = HT;
  const int H0 = zstart ? 0 : WARPS * Geo<NP>::HD;
  constexpr int RING_WARPS = RingCfg<NP, HT>::WARPS_R;
  constexpr int NT = RING_WARPS * 32;
  extern __shared__ __align__(16) double sm[];
  double* Rs = sm;
  double* vbuf = Rs + NP * NP;
  int* ver = reinterpret_cast<int*>(vbuf + RING_WARPS * 2 * HW);
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
    Rs[idx] = (!zstart && r < n && c < n && c >= r) ? Rl[r * n + c] : 0.0;
  }
  for (int j = threadIdx.x; j < NP; j += NT) ver[j] = 0;
  __syncthreads();
  double X[HW][S];
  for (int t = w; t < T; t += RING_WARPS) {
    const int64_t row = r0 + H0 + (int64_t)t * HW;
    const int valid = (int)min64((int64_t)HW, r0 + b - row);
    load_rows<HW, S>(X, A + row * lda, lda, valid, n, 0, bad);
    if constexpr (NP == 128 && HW > 16)
      ring_factor_tile_vs<NP, HW>(X, Rs, ver, vbuf + w * 2 * HW, n, t,
                                  tl ? tl + (int64_t)(t + 1) * n : nullptr);
    else if constexpr ((NP == 128 && HW == 16) || (NP == 64 && HW == 24))  // two vectors fit
      ring_factor_tile3<NP, HW>(X, Rs, ver, n, t, tl ? tl + (int64_t)(t + 1) * n : nullptr);
    else
      ring_factor_tile<NP, HW>(X, Rs, ver, vbuf + w * 2 * HW, n, t,
                               tl ? tl + (int64_t)(t + 1) * n : nullptr);
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
// Narrow leaves (n <= 8, R only): one warp per leaf, lane-private chains.
// Lane l owns an 8x8 upper-triangular R in registers and runs the flat chain
// of triangle-on-rectangle steps (Alg. 2) over its own rows: K = 4 rows per
// step, rows q*128 + 32k + l of round q (one round = 128 contiguous rows =
// 8 KB per warp).  Rounds are prefetched either one ahead into registers or,
// for contiguous 8-column rows, NARROW_STAGES ahead by cp.async into padded
// shared-memory stages (80-byte rows: conflict-free LDS.128).  The 32 lane R factors are then
// combined in-warp by the same step applied to the partner lane's R (shuffled
// in two 4-row halves), a binary tree over lanes.  R-only: the chains start
// from R = 0, which gives the QR of [0; A] -- the same R, no stored Q.
// ---------------------------------------------------------------------------
constexpr int NARROW_K = 4;
constexpr int NARROW_WARPS = 8;
// cp.async-staged variant: K rows per lane per round, W warps (leaves) per
// CTA, two shared-memory stages per warp.  K = 4: 80-byte padded rows filled
// by 16-byte copies, read by LDS.128 (conflict-free), 160 KB.  (K = 6 / 8 with
// 72-byte rows and 8-byte copies fit in shared memory, but ptxas demotes R
// and B -- 84 / 100 doubles -- to local memory: 8x slower; not instantiated.)
template <int K>
struct NarrowPipe {
  static constexpr int W = 8;
  static constexpr int STAGES = 2;
  static constexpr int G = (K == 4) ? 16 : 8;     // copy granule (bytes)
  static constexpr int ROW_B = (K == 4) ? 80 : 72;
  static constexpr int STAGE_B = 32 * K * ROW_B;
  static constexpr size_t SMEM = (size_t)W * STAGES * STAGE_B;
};

// Packed upper-triangular 8x8 R in registers: element (i, c), c >= i.
__host__ __device__ constexpr int pk8(int i, int c) { return i * 8 - (i * (i - 1)) / 2 + (c - i); }

// One triangle-on-rectangle step [R; B] (householder.py:297-332) on K rows.
// N8: n == 8 known at compile time -- the whole step is one basic block, so
// the scalars of column j+1 can be scheduled under column j's updates.
template <int K, bool N8 = false>
__device__ __forceinline__ void narrow_step(double (&R)[36], double (&B)[K][8], int n) {
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    if (!N8 && j >= n) break;
    double sg = 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k) sg = fma(B[k][j], B[k][j], sg);
    double beta, tau, scale;
    house_newton(R[pk8(j, j)], sg, beta, tau, scale);
#pragma unroll
    for (int c = j + 1; c < 8; ++c) {
      double d = 0.0;
#pragma unroll
      for (int k = 0; k < K; ++k) d = fma(B[k][j], B[k][c], d);
      const double q = tau * fma(scale, d, R[pk8(j, c)]);
      R[pk8(j, c)] -= q;
      const double qs = q * scale;
#pragma unroll
      for (int k = 0; k < K; ++k) B[k][c] = fma(-B[k][j], qs, B[k][c]);
    }
    R[pk8(j, j)] = beta;
  }
}

template <int K>
__device__ __forceinline__ void narrow_load(double (&Bt)[K][8], const double* __restrict__ A,
                                            int64_t lda, int64_t r0, int64_t b, int64_t q, int n,
                                            int lane) {
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int64_t row = q * 32 * K + (int64_t)k * 32 + lane;  // rows interleaved over lanes
    const bool ok = row < b;
    const double* src = A + (r0 + row) * lda;
    if (ok && n == 8 && lda == 8 && (((uintptr_t)A & 15) == 0)) {  // 16-byte granules only when aligned
      const double2* s2 = reinterpret_cast<const double2*>(src);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const double2 t = __ldg(s2 + c);
        Bt[k][2 * c] = t.x;
        Bt[k][2 * c + 1] = t.y;
      }
    } else {
#pragma unroll
      for (int c = 0; c < 8; ++c) Bt[k][c] = (ok && c < n) ? __ldg(src + c) : 0.0;
    }
  }
}

// Epilogue of the narrow leaf kernels: in-warp binary tree over the 32 lane
// R factors, NaN/Inf flag, then the leaf's R into its slot or the fused
// ticket tree over leaves.
__device__ __forceinline__ void narrow_finish(double (&R)[36], int lane, int leaf, int P, int n,
                                              double* Rout, int* flag, int* tickets) {
  // in-warp binary tree over the lane R factors (partner rows in two halves)
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      double Bs[4][8];
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const int i = 4 * half + k;
          Bs[k][c] = (c >= i) ? __shfl_down_sync(FULL, R[pk8(i, c)], off) : 0.0;
        }
      if ((lane & (2 * off - 1)) == 0) narrow_step<4>(R, Bs, n);
    }
  }
  if (lane != 0) return;
  // a NaN/Inf anywhere in the leaf reaches its R (every entry enters a norm)
  bool bad = false;
#pragma unroll
  for (int i = 0; i < 36; ++i) bad |= !isfinite(R[i]);
  if (bad && flag) atomicOr(flag, 1);
  auto put = [&](int node) {
    double* Ro = Rout + (int64_t)node * n * n;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (i < n && c < n) Ro[i * n + c] = (c >= i) ? R[pk8(i, c < i ? i : c)] : 0.0;
  };
  if (!tickets) {
    put(leaf);
    return;
  }
  // Fused binary tree (trees.py:52-66): at level k the second child to arrive
  // at parent p combines [R_p-side; R_sibling] with the lower index on top.
  int node = leaf;
  for (int k = 1; (1 << (k - 1)) < P; ++k) {
    const int p = node & ~((1 << k) - 1);
    const int sib_hi = p + (1 << (k - 1));
    if (sib_hi >= P) continue;  // unpaired at this level: pass up unchanged
    put(node);
    __threadfence();
    const int t = atomicAdd(tickets + (int64_t)(k - 1) * P + p, 1);
    if (t == 0) return;  // first arrival: the sibling finishes this node
    __threadfence();
    // receiver (lower index) on top: [R_p; R_sib].  Both operands were stored
    // by put(); the top one is (re)loaded into R only when it is the sibling's,
    // the bottom one streams from memory in two 4-row halves (keeps the live
    // set at R + one half so the main loop's arrays stay in registers).
    const int other = (node == p) ? sib_hi : p;
    const double* Rbot = Rout + (int64_t)((node == p) ? other : node) * n * n;
    if (node != p) {
      const double* Rtop = Rout + (int64_t)other * n * n;
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int c = i; c < 8; ++c) R[pk8(i, c)] = (i < n && c < n) ? __ldcg(Rtop + i * n + c) : 0.0;
    }
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      double Bs[4][8];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const int i = 4 * half + kk;
          Bs[kk][c] = (c >= i && i < n && c < n) ? __ldcg(Rbot + i * n + c) : 0.0;
        }
      narrow_step<4>(R, Bs, n);
    }
    node = p;
  }
  put(node);  // the root (node 0)
}

// n = 8 with contiguous 16-byte-aligned rows (C4): K = 8 rows per lane per
// step (rows 256 s + 32 k + lane of the leaf), twice the rows of k_leaf_narrow
// per reflector-scalar chain (the per-column house_newton and the per-(j, c)
// scalars are amortised over 8 rows: ~25% fewer FP64 instructions per row).
// No staging buffer: the next step's column pair (2c, 2c+1) is loaded into the
// registers of columns 2c, 2c+1 as soon as reflector 2c+1 of the current step
// has consumed them, so the loads run under the rest of the step.
// Reflector J of one K = 8 step (triangle-on-rectangle column J,
// householder.py:314-331); after it (J odd) the next step's columns J-1, J
// are loaded into the registers it consumed.
template <int J>
__device__ __forceinline__ void narrow8_col(double (&R)[36], double (&B)[8][8],
                                            const double2* __restrict__ A2, int64_t st, bool more,
                                            int64_t b, int lane) {
  double sg = 0.0, sg2 = 0.0;
#pragma unroll
  for (int k = 0; k < 8; k += 2) {
    sg = fma(B[k][J], B[k][J], sg);
    sg2 = fma(B[k + 1][J], B[k + 1][J], sg2);
  }
  double beta, tau, scale;
  house_newton(R[pk8(J, J)], sg + sg2, beta, tau, scale);
#pragma unroll
  for (int c = J + 1; c < 8; ++c) {
    double d = 0.0, d2 = 0.0;
#pragma unroll
    for (int k = 0; k < 8; k += 2) {
      d = fma(B[k][J], B[k][c], d);
      d2 = fma(B[k + 1][J], B[k + 1][c], d2);
    }
    const double q = tau * fma(scale, d + d2, R[pk8(J, c)]);
    R[pk8(J, c)] -= q;
    const double qs = q * scale;
#pragma unroll
    for (int k = 0; k < 8; ++k) B[k][c] = fma(-B[k][J], qs, B[k][c]);
  }
  R[pk8(J, J)] = beta;
  if constexpr (J & 1) {
    if (more) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int64_t row = (st + 1) * 256 + 32 * k + lane;
        double2 t = make_double2(0.0, 0.0);
        if (row < b) t = __ldg(A2 + row * 4 + (J >> 1));
        B[k][J - 1] = t.x;
        B[k][J] = t.y;
      }
    }
  }
}

// n = 8 with contiguous 16-byte-aligned rows (C4): K = 8 rows per lane per
// step (rows 256 s + 32 k + lane of the leaf), twice the rows of k_leaf_narrow
// per reflector-scalar chain (the per-column house_newton and the per-(j, c)
// scalars are amortised over 8 rows: ~30% fewer instructions per row).  No
// staging buffer: the next step's column pair (2c, 2c+1) is loaded into the
// registers of columns 2c, 2c+1 once reflector 2c+1 has consumed them, from
// L2 (prefetched one step ahead, CAQR_TUNE_NARROW_PF).  A shared-memory stage (cp.async one
// step ahead, LDS at the step boundary) measured slower: 2.14 vs 1.78 ms.
template <int W>
__global__ void __launch_bounds__(W * 32, 1)
k_leaf_narrow8(const double* __restrict__ A, int64_t m, int P, int64_t base, double* Rout, int* flag,
               int* tickets, int pf) {
  constexpr int K = 8;
  const int lane = threadIdx.x & 31;
  const int leaf = blockIdx.x * W + (threadIdx.x >> 5);
  if (leaf >= P) return;
  const int64_t r0 = (int64_t)leaf * base;
  const int64_t b = (leaf == P - 1) ? m - r0 : base;
  const int64_t steps = (b + 32 * K - 1) / (32 * K);
  const double2* A2 = reinterpret_cast<const double2*>(A + r0 * 8);
  auto prefetch = [&](int64_t st) {  // L2, 128 lines of 128 B per step
    if (st >= steps) return;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t line = st * 128 + 32 * i + lane;
      if (line * 2 < b) asm volatile("prefetch.global.L2 [%0];" :: "l"(A2 + line * 8));
    }
  };
  double R[36];
#pragma unroll
  for (int i = 0; i < 36; ++i) R[i] = 0.0;
  double B[K][8];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int64_t row = 32 * k + lane;
#pragma unroll
    for (int c2 = 0; c2 < 4; ++c2) {
      double2 t = make_double2(0.0, 0.0);
      if (row < b) t = __ldg(A2 + row * 4 + c2);
      B[k][2 * c2] = t.x;
      B[k][2 * c2 + 1] = t.y;
    }
  }
  for (int i = 1; i < pf; ++i) prefetch(i);
  for (int64_t st = 0; st < steps; ++st) {
    const bool more = st + 1 < steps;
    if (pf) prefetch(st + pf);
    narrow8_col<0>(R, B, A2, st, more, b, lane);
    narrow8_col<1>(R, B, A2, st, more, b, lane);
    narrow8_col<2>(R, B, A2, st, more, b, lane);
    narrow8_col<3>(R, B, A2, st, more, b, lane);
    narrow8_col<4>(R, B, A2, st, more, b, lane);
    narrow8_col<5>(R, B, A2, st, more, b, lane);
    narrow8_col<6>(R, B, A2, st, more, b, lane);
    narrow8_col<7>(R, B, A2, st, more, b, lane);
  }
  narrow_finish(R, lane, leaf, P, 8, Rout, flag, tickets);
}

template <bool PIPE, int K = NARROW_K, int W = NARROW_WARPS>
__global__ void __launch_bounds__(W * 32, 1)
k_leaf_narrow(const double* __restrict__ A, int64_t lda, int64_t m, int n, int P, int64_t base,
              double* Rout, int* flag, int* tickets) {
  const int lane = threadIdx.x & 31;
  const int leaf = blockIdx.x * W + (threadIdx.x >> 5);
  if (leaf >= P) return;
  const int64_t r0 = (int64_t)leaf * base;
  const int64_t b = (leaf == P - 1) ? m - r0 : base;
  double R[36];
#pragma unroll
  for (int i = 0; i < 36; ++i) R[i] = 0.0;
  const int64_t rounds = (b + 32 * K - 1) / (32 * K);
  if constexpr (PIPE) {
    // n == 8, lda == 8: round q is rows [q*32K, q*32K + 32K) of the leaf, one
    // contiguous run; lane l copies granules l, l + 32, ... of it
    using NP_ = NarrowPipe<K>;
    constexpr int GPR = 64 / NP_::G;                 // granules per row
    extern __shared__ __align__(16) double nsm[];
    char* stage0 = reinterpret_cast<char*>(nsm) + (threadIdx.x >> 5) * NP_::STAGES * NP_::STAGE_B;
    const unsigned s0 = (unsigned)__cvta_generic_to_shared(stage0);
    const char* Al = reinterpret_cast<const char*>(A + r0 * 8);
    auto issue = [&](int64_t q) {
      const unsigned st = s0 + (unsigned)(q % NP_::STAGES) * NP_::STAGE_B;
      const int64_t left = b - q * 32 * K;
      const char* g = Al + q * 32 * K * 64;
#pragma unroll
      for (int i = 0; i < K * GPR; ++i) {
        const int x = lane + 32 * i, row = x / GPR, part = x % GPR;
        const bool ok = row < left;
        cp_async<NP_::G>(st + row * NP_::ROW_B + part * NP_::G,
                         ok ? (const void*)(g + row * 64 + part * NP_::G) : (const void*)A,
                         ok ? (unsigned)NP_::G : 0u);
      }
    };
#pragma unroll
    for (int s2 = 0; s2 < NP_::STAGES; ++s2) {
      if (s2 < rounds) issue(s2);
      cp_async_commit();
    }
    for (int64_t q = 0; q < rounds; ++q) {
      cp_async_wait<NP_::STAGES - 1>();  // round q has landed (one group per round)
      __syncwarp();
      const char* st = stage0 + (q % NP_::STAGES) * NP_::STAGE_B;
      double B[K][8];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const char* rp = st + (32 * k + lane) * NP_::ROW_B;
        if constexpr (NP_::G == 16) {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const double2 t = reinterpret_cast<const double2*>(rp)[c];
            B[k][2 * c] = t.x;
            B[k][2 * c + 1] = t.y;
          }
        } else {
#pragma unroll
          for (int c = 0; c < 8; ++c) B[k][c] = reinterpret_cast<const double*>(rp)[c];
        }
      }
      __syncwarp();  // every lane has read the stage before it is refilled
      if (q + NP_::STAGES < rounds) issue(q + NP_::STAGES);
      cp_async_commit();
      narrow_step<K, true>(R, B, 8);
    }
  } else {
    // double-buffered prefetch without register copies: two rounds per trip
    double B0[K][8], B1[K][8];
    if (rounds > 0) narrow_load<K>(B0, A, lda, r0, b, 0, n, lane);
    for (int64_t q = 0; q < rounds; q += 2) {
      if (q + 1 < rounds) narrow_load<K>(B1, A, lda, r0, b, q + 1, n, lane);
      narrow_step<K>(R, B0, n);
      if (q + 1 >= rounds) break;
      if (q + 2 < rounds) narrow_load<K>(B0, A, lda, r0, b, q + 2, n, lane);
      narrow_step<K>(R, B1, n);
    }
  }
  narrow_finish(R, lane, leaf, P, n, Rout, flag, tickets);
}

// R-only tree combine as a warp ring: [R_a; R_b] -> R_a with R_a's rows as
// the ring's pivot rows in shared memory and R_b's rows as ring tiles (the
// zero lower part of R_b stays zero, so the reflectors keep the stacked
// structure of qr_stacked_triangles, householder.py:263-294).  No node factor
// is kept (R only).  Events from ev, or the binary level bin_level.
template <int NP, int HT>
__global__ void __launch_bounds__(RingCfg<NP, HT>::WARPS_R * 32, 1)
k_tree_ring(double* Rslots, int n, const int* __restrict__ ev, int bin_level) {
  constexpr int S = NP / 32;
  constexpr int RING_WARPS = RingCfg<NP, HT>::WARPS_R;
  constexpr int NT = RING_WARPS * 32;
  extern __shared__ __align__(16) double sm[];
  double* Rs = sm;
  double* vbuf = Rs + NP * NP;
  int* ver = reinterpret_cast<int*>(vbuf + RING_WARPS * 2 * HT);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int a, b;
  if (ev) {
    a = ev[3 * blockIdx.x];
    b = ev[3 * blockIdx.x + 1];
  } else {
    a = blockIdx.x << bin_level;
    b = a + (1 << (bin_level - 1));
  }
  double* Ra = Rslots + (int64_t)a * n * n;
  const double* Rb = Rslots + (int64_t)b * n * n;
  for (int idx = threadIdx.x; idx < NP * NP; idx += NT) {
    const int r = idx / NP, c = idx - r * NP;
    Rs[idx] = (r < n && c < n && c >= r) ? Ra[r * n + c] : 0.0;
  }
  for (int j = threadIdx.x; j < NP; j += NT) ver[j] = 0;
  __syncthreads();
  const int T = (n + HT - 1) / HT;
  double X[HT][S];
  for (int t = w; t < T; t += RING_WARPS) {
#pragma unroll
    for (int k = 0; k < HT; ++k) {
      const int r = t * HT + k;
#pragma unroll
      for (int s2 = 0; s2 < S; ++s2) {
        const int c = 32 * s2 + lane;
        X[k][s2] = (r < n && c < n && c >= r) ? Rb[r * n + c] : 0.0;
      }
    }
    if constexpr (NP == 128 && HT == 16)
      ring_factor_tile3<NP, HT>(X, Rs, ver, n, t, nullptr);
    else
      ring_factor_tile<NP, HT>(X, Rs, ver, vbuf + w * 2 * HT, n, t, nullptr);
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < n * n; idx += NT) {
    const int r = idx / n, c = idx - r * n;
    Ra[idx] = (c >= r) ? Rs[r * NP + c] : 0.0;
  }
}

// One level of the narrow fused tree as its own launch (streamed TSQR's upper
// levels): event e combines slot a (on top) with slot b exactly as
// k_leaf_narrow's ticket tree does, one thread per event.
__global__ void __launch_bounds__(128)
k_narrow_combine(double* Rslots, int n, const int* __restrict__ ev, int nev) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nev) return;
  double* Ra = Rslots + (int64_t)ev[3 * e] * n * n;
  const double* Rb = Rslots + (int64_t)ev[3 * e + 1] * n * n;
  double R[36], Ro8[36];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int c = i; c < 8; ++c) {
      R[pk8(i, c)] = (i < n && c < n) ? Ra[i * n + c] : 0.0;
      Ro8[pk8(i, c)] = (i < n && c < n) ? Rb[i * n + c] : 0.0;
    }
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    double Bs[4][8];
#pragma unroll
    for (int kk = 0; kk < 4; ++kk)
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int i = 4 * half + kk;
        Bs[kk][c] = (c >= i) ? Ro8[pk8(i, c < i ? i : c)] : 0.0;
      }
    narrow_step<4>(R, Bs, n);
  }
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int c = 0; c < 8; ++c)
      if (i < n && c < n) Ra[i * n + c] = (c >= i) ? R[pk8(i, c < i ? i : c)] : 0.0;
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
k_tree_factor(double* Rslots, int n, const int* __restrict__ ev, double* Ynode, double* taunode,
              int bin_level) {
  constexpr int S = NP / 32, RW = NP / WARPS;
  extern __shared__ __align__(16) double sm[];
  double* Ps = sm;
  double* part = Ps + NP * NP;
  double* vbuf = part + WARPS * NP;
  double* red = vbuf + WARPS * RW;
  double* sx0 = red + WARPS;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int a, b, id;
  if (ev) {
    a = ev[3 * blockIdx.x]; b = ev[3 * blockIdx.x + 1]; id = ev[3 * blockIdx.x + 2];
  } else {  // binary tree level bin_level: pair (e 2^k, e 2^k + 2^(k-1)) (trees.py:52-66)
    a = blockIdx.x << bin_level; b = a + (1 << (bin_level - 1)); id = 0;
  }
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
  cta_factor<NP, RW, STACKED>(X, Ps, n, taunode ? taunode + (int64_t)id * n : nullptr, red, sx0,
                               part, vbuf);
  __syncthreads();
  double* Ro = Rslots + (int64_t)a * n * n;
  for (int idx = threadIdx.x; idx < n * n; idx += THREADS) {
    const int r = idx / n, c = idx - r * n;
    Ro[idx] = (c >= r) ? Ps[r * NP + c] : 0.0;
  }
  if (!Ynode) return;
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
// Warp-level tree kernels for n <= 32: one warp per combine event (or per
// event x 32-column block for the apply); lane c owns column c of both
// stacked blocks, so the reflector arithmetic is lane-local and only the
// reflector vector is broadcast (shuffles).  Same STACKED semantics as
// k_tree_factor / k_tree_apply (householder.py:263-294, 377-396).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128)
k_tree_factor_w32(double* Rslots, int n, const int* __restrict__ ev, int nev, double* Ynode,
                  double* taunode, int bin_level) {
  // One warp per event, a rolled loop over the reflectors (the short-lived tree
  // kernels are instruction-fetch bound when fully unrolled).  Lane c holds
  // column c of R_b in registers (rows > c stay exactly zero until reflector
  // c, so sums over all 32 rows need no masking); R_a's rows -- the pivot
  // rows, row j touched only by reflector j -- live in shared memory.
  const int lane = threadIdx.x & 31;
  const int e = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (e >= nev) return;
  int a, b, id;
  if (ev) {
    a = ev[3 * e]; b = ev[3 * e + 1]; id = ev[3 * e + 2];
  } else {
    a = e << bin_level; b = a + (1 << (bin_level - 1)); id = 0;
  }
  __shared__ double rsm[4][32][33];
  __shared__ double vsm[4][32];
  double (*Ras)[33] = rsm[threadIdx.x >> 5];
  double* vs = vsm[threadIdx.x >> 5];
  double* Ra = Rslots + (int64_t)a * n * n;
  const double* Rb = Rslots + (int64_t)b * n * n;
  double cb[32];
#pragma unroll
  for (int r = 0; r < 32; ++r) {
    const bool ok = (r < n && lane < n && lane >= r);
    Ras[r][lane] = ok ? Ra[r * n + lane] : 0.0;
    cb[r] = ok ? Rb[r * n + lane] : 0.0;
  }
  __syncwarp();
  const double diag = Ras[lane][lane];  // R_a[c][c]: unchanged until reflector c
  // every lane keeps the squared norm of its own column of R_b, refreshed in the
  // update pass, so reflector j's sigma is ready when step j starts
  double sig;
  {
    double s4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int r = 0; r < 32; ++r) s4[r & 3] = fma(cb[r], cb[r], s4[r & 3]);
    sig = (s4[0] + s4[1]) + (s4[2] + s4[3]);
  }
  double2* vs2 = reinterpret_cast<double2*>(vs);
#pragma unroll 1
  for (int j = 0; j < n; ++j) {
    const double sg = __shfl_sync(FULL, sig, j);
    const double x0 = __shfl_sync(FULL, diag, j);
    double beta, tau, scale;
    house_lean(x0, sg, beta, tau, scale);
    if (lane == j) {  // v = column j of R_b, scaled (zero below row j)
#pragma unroll
      for (int r = 0; r < 32; r += 2) vs2[r >> 1] = make_double2(cb[r] * scale, cb[r + 1] * scale);
    }
    __syncwarp();
    double v[32];
#pragma unroll
    for (int r = 0; r < 32; r += 2) {
      const double2 t = vs2[r >> 1];
      v[r] = t.x;
      v[r + 1] = t.y;
    }
    const double raj = Ras[j][lane];
    double d4[4] = {raj, 0.0, 0.0, 0.0};
#pragma unroll
    for (int r = 0; r < 32; ++r) d4[r & 3] = fma(v[r], cb[r], d4[r & 3]);
    const double d = (d4[0] + d4[1]) + (d4[2] + d4[3]);
    const double w = (lane > j) ? tau * d : 0.0;
    const bool own = (lane == j);
    double s4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      cb[r] = own ? v[r] : fma(-v[r], w, cb[r]);
      s4[r & 3] = fma(cb[r], cb[r], s4[r & 3]);
    }
    sig = (s4[0] + s4[1]) + (s4[2] + s4[3]);
    Ras[j][lane] = own ? beta : raj - w;  // lanes < j: w = 0, unchanged
    if (lane == 0 && taunode) taunode[(int64_t)id * n + j] = tau;
    __syncwarp();
  }
#pragma unroll
  for (int r = 0; r < 32; ++r) {
    if (r < n && lane < n) {
      Ra[r * n + lane] = (lane >= r) ? Ras[r][lane] : 0.0;
      if (Ynode) Ynode[(int64_t)id * n * n + r * n + lane] = (lane >= r) ? cb[r] : 0.0;
    }
  }
}

template <bool TRANS>
__global__ void __launch_bounds__(128)
k_tree_apply_w32(const double* __restrict__ Ynode, const double* __restrict__ taunode, int n,
                 const int* __restrict__ ev, int nev, double* C, int64_t ldc, int64_t slot_rows,
                 int64_t ncols, int zero_partner) {
  const int lane = threadIdx.x & 31;
  const int e = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (e >= nev) return;
  const int a = ev[3 * e], b = ev[3 * e + 1], id = ev[3 * e + 2];
  const int64_t col = (int64_t)blockIdx.y * 32 + lane;
  const bool okc = col < ncols;
  double* Ca = C + (int64_t)a * slot_rows * ldc + col;
  double* Cb = C + (int64_t)b * slot_rows * ldc + col;
  const double* Yn = Ynode + (int64_t)id * n * n;
  const double* tn = taunode + (int64_t)id * n;
  // the node's Y (n x n upper triangular) and tau staged once in shared memory:
  // a global load per reflector would put an L2 round trip on the chain
  __shared__ double ysm[4][32][33];
  __shared__ double tsm[4][32];
  double (*Ys)[33] = ysm[threadIdx.x >> 5];
  double* ts = tsm[threadIdx.x >> 5];
#pragma unroll 4
  for (int r = 0; r < 32; ++r) Ys[r][lane] = (r < n && lane < n) ? __ldg(Yn + (int64_t)r * n + lane) : 0.0;
  ts[lane] = lane < n ? __ldg(tn + lane) : 0.0;
  double ca[32], cb[32];
#pragma unroll
  for (int r = 0; r < 32; ++r) {
    ca[r] = (okc && r < n) ? Ca[(int64_t)r * ldc] : 0.0;
    cb[r] = (okc && r < n && !zero_partner) ? Cb[(int64_t)r * ldc] : 0.0;
  }
  __syncwarp();
#pragma unroll
  for (int jx = 0; jx < 32; ++jx) {
    const int j = TRANS ? jx : 31 - jx;
    if (j >= n) continue;
    const double tj = ts[j];
    double d = ca[j];
#pragma unroll
    for (int r = 0; r <= j; ++r) d = fma(Ys[r][j], cb[r], d);
    const double w = tj * d;
    ca[j] -= w;
#pragma unroll
    for (int r = 0; r <= j; ++r) cb[r] = fma(-Ys[r][j], w, cb[r]);
  }
#pragma unroll
  for (int r = 0; r < 32; ++r) {
    if (okc && r < n) {
      Ca[(int64_t)r * ldc] = ca[r];
      Cb[(int64_t)r * ldc] = cb[r];
    }
  }
}

// ---------------------------------------------------------------------------
// tree apply: [C_a; C_b] <- Q_node^(T?) [C_a; C_b] on one column block.
// C_a = C + a*slot_rows*ldc, C_b = C + b*slot_rows*ldc (n rows each).
// ---------------------------------------------------------------------------
template <int NP, int KBS>
struct TreeApplySmem {
  static constexpr size_t bytes = sizeof(double) * ((size_t)NP * 32 * KBS + 2 * WARPS * 32 * KBS +
                                                    (size_t)WARPS * (32 * (NP / WARPS + 2) + 32));
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
  double* vstage = part + 2 * WARPS * KB + w * (32 * (RW + 2) + 32);
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
  auto ycol = [&](int r, int j) { return (r < n) ? __ldg(Yn + (int64_t)r * n + j) : 0.0; };
  cta_apply<RW, KBS, STACKED, TRANS>(X, Ps, n, ycol, taunode + (int64_t)id * n, part, col0, false,
                                     vstage);
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
// Per-warp V/tau staging: 32 reflectors x (rows + 2) for the taller of the
// dense-tile rows per warp (HD) and the chain tile height.
template <int NP, int HT>
__host__ __device__ constexpr int apply_stage_doubles() {
  return ApplyStage<(Geo<NP>::HD > HT ? Geo<NP>::HD : HT)>::DOUBLES;
}
template <int NP, int KBS, int HT>
struct LeafApplySmem {
  static constexpr size_t bytes =
      sizeof(double) * ((size_t)NP * 32 * KBS + 2 * WARPS * 32 * KBS +
                        (size_t)WARPS * apply_stage_doubles<NP, HT>()) + sizeof(int) * NP;
};

template <int NP, int KBS, bool TRANS, int HT>
__global__ void __launch_bounds__(THREADS, 1)
k_leaf_apply(const double* __restrict__ Y, int64_t ldy, const double* __restrict__ tau,
             int64_t tau_stride, int64_t m, int n, int P, int64_t base, double* C, int64_t ldc,
             int64_t ncols, const double* __restrict__ S, int64_t lds, int64_t s_slot_rows,
             int zero_init, int tri_skip) {
  constexpr int HD = Geo<NP>::HD, H0 = WARPS * HD, KB = 32 * KBS;
  extern __shared__ __align__(16) double sm[];
  double* Cs = sm;
  double* part = Cs + NP * KB;
  constexpr int SD = apply_stage_doubles<NP, HT>();
  double* vstage = part + 2 * WARPS * KB + (threadIdx.x >> 5) * SD;
  int* ver = reinterpret_cast<int*>(part + 2 * WARPS * KB + WARPS * SD);
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
  const int T = rest > 0 ? (int)((rest + HT - 1) / HT) : 0;
  const bool tskip = tri_skip != 0;
  bool bad = false;
  auto ycol = [&](int r, int j) { return (r < b) ? __ldg(Yl + (int64_t)r * ldy + j) : 0.0; };
  const int v0 = (int)max64(0, min64((int64_t)HD, b - (int64_t)w * HD));
  if (TRANS) {
    {
    double X[HD][KBS];
    load_rows<HD, KBS>(X, Cl + (int64_t)w * HD * ldc, ldc, v0, ncb, 0, bad);
    cta_apply<HD, KBS, DENSE, true>(X, nullptr, n, ycol, tl, part, col0, false, vstage);
    // rows < n become the ring's pivot rows; rows >= n are final
#pragma unroll
    for (int k = 0; k < HD; ++k) {
      const int r = w * HD + k;
      if (r < NP) {
#pragma unroll
        for (int s = 0; s < KBS; ++s) Cs[r * KB + 32 * s + lane] = (r < n) ? X[k][s] : 0.0;
      }
    }
    {
      const int lo = max(0, n - w * HD);
      store_rows<HD, KBS>(X, Cl + (int64_t)w * HD * ldc, ldc, v0, ncb, 0, lo);
    }
    }
    for (int j = threadIdx.x; j < NP; j += THREADS) ver[j] = 0;
    __syncthreads();
    double X[HT][KBS];
    for (int t = w; t < T; t += WARPS) {
      const int64_t row = H0 + (int64_t)t * HT;
      const int valid = (int)min64((int64_t)HT, b - row);
      load_rows<HT, KBS>(X, Cl + row * ldc, ldc, valid, ncb, 0, bad);
      ring_apply_tile<HT, KBS, true>(X, Cs, ver, Yl + row * ldy, ldy, valid, tl + (int64_t)(t + 1) * n,
                                     n, t, col0, false, vstage);
      store_rows<HT, KBS>(X, Cl + row * ldc, ldc, valid, ncb, 0);
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
    {
    double X[HT][KBS];
    for (int o = w; o < T; o += WARPS) {
      const int t = T - 1 - o;
      const int64_t row = H0 + (int64_t)t * HT;
      const int valid = (int)min64((int64_t)HT, b - row);
      if (zero_init) {
#pragma unroll
        for (int k = 0; k < HT; ++k)
#pragma unroll
          for (int s = 0; s < KBS; ++s) X[k][s] = 0.0;
      } else {
        load_rows<HT, KBS>(X, Cl + row * ldc, ldc, valid, ncb, 0, bad);
      }
      ring_apply_tile<HT, KBS, false>(X, Cs, ver, Yl + row * ldy, ldy, valid, tl + (int64_t)(t + 1) * n,
                                      n, o, col0, tskip, vstage);
      store_rows<HT, KBS>(X, Cl + row * ldc, ldc, valid, ncb, 0);
    }
    }
    __syncthreads();
    double X[HD][KBS];
#pragma unroll
    for (int k = 0; k < HD; ++k) {
      const int r = w * HD + k;
#pragma unroll
      for (int s = 0; s < KBS; ++s) {
        double x = 0.0;
        if (r < n) x = Cs[r * KB + 32 * s + lane];
        else if (!zero_init && k < v0 && 32 * s + lane < ncb) x = Cl[(int64_t)r * ldc + 32 * s + lane];
        X[k][s] = x;
      }
    }
    __syncthreads();
    cta_apply<HD, KBS, DENSE, false>(X, nullptr, n, ycol, tl, part, col0, tskip, vstage);
    store_rows<HD, KBS>(X, Cl + (int64_t)w * HD * ldc, ldc, v0, ncb, 0);
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
  double* vstage = part + 2 * WARPS * KB + w * (32 * (RW + 2) + 32);
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
  cta_apply<RW, KBS, MODE, TRANS>(X, Ps, n, ycol, tau, part, col0, false, vstage);
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

#include "dmma_ring.cuh"
#include "dmma_apply.cuh"
#include "split_leaf.cuh"
#include "tm_leaf.cuh"
#include "tm_tall.cuh"
#include "tall_apply.cuh"
#include "tree_factor128.cuh"
#include "tree_apply_cp.cuh"
#include "dense_geqr2.cuh"

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

// ---------------------------------------------------------------------------
// Column-major -> row-major transpose on load (MAT1 files store columns,
// matio.py:1-10; the kernels read rows): 32 x 32 tiles through padded shared
// memory, coalesced on both sides.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
k_colmajor_to_rowmajor(const double* __restrict__ src, int64_t ld_src, int64_t rows, int cols,
                       double* __restrict__ dst, int64_t ld_dst) {
  __shared__ double tile[32][33];
  const int64_t r0 = (int64_t)blockIdx.x * 32;
  const int c0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8 threads
#pragma unroll
  for (int k = 0; k < 32; k += 8) {
    const int c = c0 + ty + k;
    const int64_t r = r0 + tx;
    tile[ty + k][tx] = (c < cols && r < rows) ? src[(int64_t)c * ld_src + r] : 0.0;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 32; k += 8) {
    const int64_t r = r0 + ty + k;
    const int c = c0 + tx;
    if (r < rows && c < cols) dst[r * ld_dst + c] = tile[tx][ty + k];
  }
}

extern "C" {

int caqr_sm100_abi_version(void) { return CAQR_SM100_ABI_VERSION; }

const char* tsqr_last_error(void) { return g_err; }

int tsqr_f64_geometry(int64_t n, int64_t* np, int64_t* h0, int64_t* ht) {
  const int p = padded(n);
  if (n < 1 || !p) return set_err(CAQR_ERR_ARG, "n must be in [1, 128]");
  const int hd = p == 32 ? Geo<32>::HD : (p == 64 ? Geo<64>::HD : Geo<128>::HD);
  if (np) *np = p;
  if (ht) *ht = g_ht[np_index(p)];
  if (h0) *h0 = (int64_t)WARPS * hd;
  return CAQR_OK;
}

// Narrow leaves: the cp.async-staged kernel for contiguous 8-column rows
// (CAQR_TUNE_NARROW = 2, default), else the register-prefetch kernel.
static int launch_narrow(const double* A, int64_t lda, int64_t m, int64_t n, int64_t P,
                         int64_t base, double* R, int* flag, int* tickets, cudaStream_t st) {
#define NARROW_PIPE(KK)                                                                       \
  {                                                                                           \
    using NP_ = NarrowPipe<KK>;                                                               \
    int rc = prep(k_leaf_narrow<true, KK, NP_::W>, NP_::SMEM);                                \
    if (rc) return rc;                                                                        \
    k_leaf_narrow<true, KK, NP_::W><<<(int)((P + NP_::W - 1) / NP_::W), NP_::W * 32, NP_::SMEM, \
                                      st>>>(A, lda, m, (int)n, (int)P, base, R, flag, tickets); \
  }
  if (g_narrow == 3 && n == 8 && lda == 8 && (((uintptr_t)A & 15) == 0)) {  // 16-byte rows, K = 8
    constexpr int W8 = 8;
    k_leaf_narrow8<W8><<<(int)((P + W8 - 1) / W8), W8 * 32, 0, st>>>(A, m, (int)P, base, R, flag,
                                                                     tickets, g_narrow_pf);
  } else if (g_narrow >= 2 && n == 8 && lda == 8 && (((uintptr_t)A & 15) == 0)) {  // cp.async 16 B granules
    NARROW_PIPE(4)
  } else {
    k_leaf_narrow<false><<<(int)((P + NARROW_WARPS - 1) / NARROW_WARPS), NARROW_WARPS * 32, 0, st>>>(
        A, lda, m, (int)n, (int)P, base, R, flag, tickets);
  }
#undef NARROW_PIPE
  return check_launch("k_leaf_narrow");
}

// Smallest tau row stride of a leaf that keeps Q: the dense first tile (h0
// rows) plus ceil((b - h0) / ht) chain tiles of n scalars each, b the tallest
// (last) leaf.
static int64_t min_tau_stride(int64_t m, int64_t n, int64_t P, int64_t base) {
  int64_t np_ = 0, h0 = 0, ht = 0;
  if (tsqr_f64_geometry(n, &np_, &h0, &ht) != CAQR_OK) return INT64_MAX;
  const int64_t b = m - (P - 1) * base;
  const int64_t tiles = 1 + (b > h0 ? (b - h0 + ht - 1) / ht : 0);
  return tiles * n;
}

// Leaves of `base` rows, the last one taking the remainder (m - (P-1) base >= base).
static int leaf_factor_impl(const double* A, int64_t lda, int64_t m, int64_t n, int64_t P,
                            int64_t base, double* Y, int64_t ldy, double* tau, int64_t tau_stride,
                            double* R, int* flag, void* stream, double* Tout = nullptr) {
  const int p = padded(n);
  if (!p || !A || !R || P < 1 || m < n * P || lda < n || (Y && ldy < n))
    return set_err(CAQR_ERR_ARG, "tsqr_f64_leaf_factor: bad arguments");
  if ((Y == nullptr) != (tau == nullptr)) return set_err(CAQR_ERR_ARG, "Y and tau go together");
  if (base < n) return set_err(CAQR_ERR_ARG, "leaf shorter than n");
  // (R only: the last leaf may be a shorter run of fused leaves, r_binary_impl)
  if (m - (P - 1) * base < (Y ? base : n)) return set_err(CAQR_ERR_ARG, "last leaf shorter than base");
  if (tau && tau_stride < min_tau_stride(m, n, P, base))
    return set_err(CAQR_ERR_ARG, "tau_stride below the leaf's tiles * n");
  cudaStream_t st = (cudaStream_t)stream;
  const int grid = (int)P;
  if (n <= 8 && !Y && g_narrow) {
    return launch_narrow(A, lda, m, n, P, base, R, flag, nullptr, st);
  }
#define CHAIN_LAUNCH(NPV, HTV)                                                                  \
  {                                                                                             \
    rc = prep(k_leaf_chain<NPV, HTV>, ChainSmem<NPV, HTV>::bytes);                              \
    if (rc) return rc;                                                                          \
    k_leaf_chain<NPV, HTV><<<grid, RingCfg<NPV, HTV>::WARPS_R * 32, ChainSmem<NPV, HTV>::bytes,  \
                             st>>>(A, lda, m, (int)n, (int)P, base, Y, ldy, tau, tau_stride, R,  \
                                   flag, zs ? 1 : 0);                                            \
  }
#define DMMA_LAUNCH(NPX, V16, Q)                                                                 \
  {                                                                                             \
    constexpr int NPD = NPX == 128 ? 128 : (NPX == 64 ? 64 : 32);                              \
    rc = prep(k_leaf_dmma<NPD, V16, Q>, DmmaRingSmem<NPD>::bytes);                              \
    if (rc) return rc;                                                                          \
    k_leaf_dmma<NPD, V16, Q><<<grid, DR_WARPS * 32, DmmaRingSmem<NPD>::bytes, st>>>(A, lda, m,  \
        (int)n, (int)P, base, Y, ldy, tau, tau_stride, R, flag, h0d, Tout);                     \
  }
#define LEAF_CASE(NPV, HA, HB)                                                                  \
  case NPV: {                                                                                   \
    const bool zs = !Y && g_zstart;                                                             \
    int rc = 0;                                                                                 \
    if (!zs && NPV <= 64 && g_dmma_dense) {                                                     \
      constexpr int NPQ = NPV <= 32 ? 32 : 64;                                                  \
      rc = prep(k_leaf_dense_dmma<NPQ>, DenseDmmaSmem<NPQ>::bytes);                             \
      if (rc) return rc;                                                                        \
      k_leaf_dense_dmma<NPQ><<<grid, THREADS, DenseDmmaSmem<NPQ>::bytes, st>>>(A, lda, m,       \
          (int)n, (int)P, base, Y, ldy, tau, tau_stride, R, flag);                              \
    } else if (!zs) {                                                                           \
      rc = prep(k_leaf_dense<NPV>, DenseSmem<NPV>::bytes);                                      \
      if (rc) return rc;                                                                        \
      k_leaf_dense<NPV><<<grid, THREADS, DenseSmem<NPV>::bytes, st>>>(A, lda, m, (int)n,        \
          (int)P, base, Y, ldy, tau, tau_stride, R, flag);                                      \
    }                                                                                           \
    if (NPV == 128 && zs && g_cc == 5) {                                                        \
      rc = prep(k_leaf_tt<64, 1, false>, TtSmem<64>::bytes);                                    \
      if (rc) return rc;                                                                        \
      k_leaf_tt<64, 1, false><<<grid, TtCfg<64, 1>::THREADS, TtSmem<64>::bytes, st>>>(A, lda,   \
          m, (int)n, (int)P, base, R, flag, nullptr, 0, nullptr, 0, 0);                         \
    } else if (NPV == 128 && zs && g_cc == 6) {                                                 \
      rc = prep(k_leaf_tt<32, 1, false>, TtSmem<32>::bytes);                                    \
      if (rc) return rc;                                                                        \
      k_leaf_tt<32, 1, false><<<grid, TtCfg<32, 1>::THREADS, TtSmem<32>::bytes, st>>>(A, lda,   \
          m, (int)n, (int)P, base, R, flag, nullptr, 0, nullptr, 0, 0);                         \
    } else if (NPV == 128 && zs && g_cc == 3) {                                                 \
      rc = prep(k_leaf_tm<12>, TmSmem<12>::bytes);                                              \
      if (rc) return rc;                                                                        \
      k_leaf_tm<12><<<grid, TmCfg<12>::THREADS, TmSmem<12>::bytes, st>>>(A, lda, m, (int)n,     \
                                                                         (int)P, base, R, flag); \
    } else if (NPV == 128 && zs && g_cc == 4) {                                                 \
      rc = prep(k_leaf_tm<16>, TmSmem<16>::bytes);                                              \
      if (rc) return rc;                                                                        \
      k_leaf_tm<16><<<grid, TmCfg<16>::THREADS, TmSmem<16>::bytes, st>>>(A, lda, m, (int)n,     \
                                                                         (int)P, base, R, flag); \
    } else if (NPV == 128 && zs && g_cc == 2) {                                                 \
      const bool v16 = (n % 2 == 0) && (lda % 2 == 0) && (((uintptr_t)A & 15) == 0);            \
      if (v16) {                                                                                \
        rc = prep(k_leaf_split<true>, SpSmem::bytes);                                           \
        if (rc) return rc;                                                                      \
        k_leaf_split<true><<<grid, SP_THREADS, SpSmem::bytes, st>>>(A, lda, m, (int)n, (int)P,  \
                                                                    base, R, flag);             \
      } else {                                                                                  \
        rc = prep(k_leaf_split<false>, SpSmem::bytes);                                          \
        if (rc) return rc;                                                                      \
        k_leaf_split<false><<<grid, SP_THREADS, SpSmem::bytes, st>>>(A, lda, m, (int)n, (int)P, \
                                                                     base, R, flag);            \
      }                                                                                         \
    } else if (NPV == 128 && !zs && Y && g_ht[2] == 64) {                                       \
      rc = prep(k_leaf_tt<64, 1, true>, TtSmem<64>::bytes);                                     \
      if (rc) return rc;                                                                        \
      k_leaf_tt<64, 1, true><<<grid, TtCfg<64, 1>::THREADS, TtSmem<64>::bytes, st>>>(A, lda,    \
          m, (int)n, (int)P, base, R, flag, Y, ldy, tau, tau_stride, WARPS * Geo<128>::HD);     \
    } else if ((NPV == 128 && g_dmma && (zs || g_ht[2] == 16)) ||                             \
        (NPV == 64 && g_dmma >= 2 && (zs || g_ht[1] == 16)) ||                                  \
        (NPV == 32 && g_dmma >= 3 && (zs || g_ht[0] == 16))) {                                  \
      const int h0d = zs ? 0 : WARPS * Geo<NPV>::HD;                                            \
      const bool v16 = (n % 2 == 0) && (lda % 2 == 0) && (((uintptr_t)A & 15) == 0);            \
      if (v16 && Y) DMMA_LAUNCH(NPV, true, true)                                                     \
      else if (v16) DMMA_LAUNCH(NPV, true, false)                                                    \
      else if (Y) DMMA_LAUNCH(NPV, false, true)                                                      \
      else DMMA_LAUNCH(NPV, false, false)                                                            \
    } else if (zs || m - base * (P - 1) > (int64_t)WARPS * Geo<NPV>::HD) {                       \
      if (g_ht[np_index(NPV)] == HA) CHAIN_LAUNCH(NPV, HA)                                      \
      else if (NPV == 64 && g_ht[1] == 24) CHAIN_LAUNCH(64, 24)                                 \
      else CHAIN_LAUNCH(NPV, HB)                                                                \
    }                                                                                           \
    break;                                                                                      \
  }
  switch (p) { LEAF_CASE(32, 16, 32) LEAF_CASE(64, 16, 32) LEAF_CASE(128, 16, 24) }
#undef LEAF_CASE
#undef CHAIN_LAUNCH
#undef DMMA_LAUNCH
  return check_launch("k_leaf_dense/k_leaf_chain");
}

int tsqr_f64_leaf_factor(const double* A, int64_t lda, int64_t m, int64_t n, int64_t P, double* Y,
                         int64_t ldy, double* tau, int64_t tau_stride, double* R, int* flag,
                         void* stream) {
  if (P < 1) return set_err(CAQR_ERR_ARG, "tsqr_f64_leaf_factor: bad arguments");
  return leaf_factor_impl(A, lda, m, n, P, m / P, Y, ldy, tau, tau_stride, R, flag, stream);
}

// 1 when tsqr_f64_leaf_factor_t / _apply_t use the panel-T buffer for this width under the
// current tuning (n in (64, 128], 16-row chain tiles on the DMMA ring kernels), else 0.
int tsqr_f64_panel_t_used(int64_t n) {
  return padded(n) == 128 && g_ht[2] == 16 && g_dmma && g_dmma_apply ? 1 : 0;
}

int tsqr_f64_leaf_factor_t(const double* A, int64_t lda, int64_t m, int64_t n, int64_t P, double* Y,
                           int64_t ldy, double* tau, int64_t tau_stride, double* R, int* flag,
                           double* T, void* stream) {
  if (P < 1 || !Y || !tau) return set_err(CAQR_ERR_ARG, "tsqr_f64_leaf_factor_t: bad arguments");
  return leaf_factor_impl(A, lda, m, n, P, m / P, Y, ldy, tau, tau_stride, R, flag, stream,
                          tsqr_f64_panel_t_used(n) ? T : nullptr);
}

static int r_binary_impl(const double* A, int64_t lda, int64_t m, int64_t n, int64_t P,
                         int64_t base, double* Rslots, int* tickets, int* flag, void* stream) {
  const int p = padded(n);
  if (!p || !A || !Rslots || P < 1 || m < n * P || lda < n || (!tickets && n <= 8 && P > 1))
    return set_err(CAQR_ERR_ARG, "tsqr_f64_r_binary: bad arguments");
  if (base < n) return set_err(CAQR_ERR_ARG, "leaf shorter than n");
  if (m - (P - 1) * base < base) return set_err(CAQR_ERR_ARG, "last leaf shorter than base");
  cudaStream_t st = (cudaStream_t)stream;
  int levels = 0;
  while ((1LL << levels) < P) ++levels;
  if (n <= 8 && g_narrow) {
    // More leaves than resident warps (8 per SM): deal the rows to g_fuse x 8 warps in runs of
    // whole 256-row steps, one wave of CTAs, so the start-up loads and the lane / ticket
    // combine of a leaf are paid once per warp instead of once per leaf (C4: 8192 leaves of
    // 16384 rows were 7 waves of CTAs whose 8 warps start and finish together).
    // (never more runs than leaves: Rslots and tickets are sized by the caller's P)
    if (g_fuse && P > 8 * (int64_t)g_fuse) {
      const int64_t W = 8 * (int64_t)g_fuse;
      const int64_t b2 = ((m + W - 1) / W + 255) / 256 * 256;
      if (b2 > base) {
        int64_t P2 = (m + b2 - 1) / b2;
        if (P2 > 1 && m - (P2 - 1) * b2 < n) --P2;
        P = P2;
        base = b2;
        levels = 0;
        while ((1LL << levels) < P) ++levels;
      }
    }
    if (P > 1 && cudaMemsetAsync(tickets, 0, sizeof(int) * (size_t)levels * P, st) != cudaSuccess)
      return check_launch("cudaMemsetAsync");
    return launch_narrow(A, lda, m, n, P, base, Rslots, flag, P > 1 ? tickets : nullptr, st);
  }
  // R only, more leaves than SMs: every CTA keeps folding the next rows into the same R (the
  // flat tree of Alg. 2 inside a CTA, the binary tree above it -- the hybrid tree of PAPER.md
  // Fig. 3), instead of writing 2048 R factors and combining them in tree levels that are
  // several waves wide (C3: 2.1 -> 0.8 ms of tree).  The rows are dealt to g_fuse CTAs in runs
  // of whole 64-row tiles, so one wave carries them evenly whatever P is (256 leaves on 148
  // SMs would otherwise take two waves for 1.73 waves of work); any row partition gives the
  // same R up to rounding and signs (section 5).
  if (g_fuse && p == 128 && g_zstart && P > g_fuse) {
    int64_t b2 = ((m + g_fuse - 1) / g_fuse + 63) / 64 * 64;
    if (b2 < 128) b2 = 128;
    if (b2 > base) {
      int64_t P2 = (m + b2 - 1) / b2;
      if (P2 > 1 && m - (P2 - 1) * b2 < n) --P2;  // a short tail rides with the last run
      P = P2;
      base = b2;
      levels = 0;
      while ((1LL << levels) < P) ++levels;
    }
  }
  int rc = leaf_factor_impl(A, lda, m, n, P, base, nullptr, 0, nullptr, 0, Rslots, flag, stream);
  if (rc) return rc;
  for (int k = 1; k <= levels; ++k) {
    const int64_t nev = (P - 1 - (1LL << (k - 1))) / (1LL << k) + 1;  // f + 2^(k-1) < P, f = e 2^k
#define TB_CASE(NPV)                                                                     \
  case NPV: {                                                                            \
    rc = prep(k_tree_ring<NPV, 16>, ChainSmem<NPV, 16>::bytes);                          \
    if (rc) return rc;                                                                   \
    k_tree_ring<NPV, 16><<<(int)nev, RingCfg<NPV, 16>::WARPS_R * 32,                     \
                           ChainSmem<NPV, 16>::bytes, st>>>(Rslots, (int)n, nullptr, k); \
    break;                                                                               \
  }
    if (p == 32) {
      k_tree_factor_w32<<<(int)((nev + 3) / 4), 128, 0, st>>>(Rslots, (int)n, nullptr, (int)nev,
                                                             nullptr, nullptr, k);
    } else {
      switch (p) { TB_CASE(64) TB_CASE(128) }
    }
#undef TB_CASE
    rc = check_launch("k_tree_factor");
    if (rc) return rc;
  }
  return CAQR_OK;
}

int tsqr_f64_r_binary(const double* A, int64_t lda, int64_t m, int64_t n, int64_t P, double* Rslots,
                      int* tickets, int* flag, void* stream) {
  if (P < 1) return set_err(CAQR_ERR_ARG, "tsqr_f64_r_binary: bad arguments");
  return r_binary_impl(A, lda, m, n, P, m / P, Rslots, tickets, flag, stream);
}

int tsqr_f64_r_binary_rows(const double* A, int64_t lda, int64_t m, int64_t n, int64_t P,
                           int64_t base, double* Rslots, int* tickets, int* flag, void* stream) {
  return r_binary_impl(A, lda, m, n, P, base, Rslots, tickets, flag, stream);
}

int tsqr_f64_r_combine_level(double* Rslots, int64_t n, const int32_t* events, int64_t nev,
                             void* stream) {
  const int p = padded(n);
  if (!p || !Rslots || !events || nev < 0)
    return set_err(CAQR_ERR_ARG, "tsqr_f64_r_combine_level: bad arguments");
  if (nev == 0) return CAQR_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (n <= 8 && g_narrow) {
    k_narrow_combine<<<(int)((nev + 127) / 128), 128, 0, st>>>(Rslots, (int)n, events, (int)nev);
    return check_launch("k_narrow_combine");
  }
  if (p == 32) {
    k_tree_factor_w32<<<(int)((nev + 3) / 4), 128, 0, st>>>(Rslots, (int)n, events, (int)nev,
                                                           nullptr, nullptr, 0);
    return check_launch("k_tree_factor_w32");
  }
#define RC_CASE(NPV)                                                                     \
  case NPV: {                                                                            \
    int rc = prep(k_tree_ring<NPV, 16>, ChainSmem<NPV, 16>::bytes);                      \
    if (rc) return rc;                                                                   \
    k_tree_ring<NPV, 16><<<(int)nev, RingCfg<NPV, 16>::WARPS_R * 32,                     \
                           ChainSmem<NPV, 16>::bytes, st>>>(Rslots, (int)n, events, 0);  \
    break;                                                                               \
  }
  switch (p) { RC_CASE(64) RC_CASE(128) }
#undef RC_CASE
  return check_launch("k_tree_factor");
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
        events, Ynode, taunode, 0);                                                      \
    break;                                                                               \
  }
  if (p == 128 && g_dmma_tree_factor) {
    int rc = prep(k_tree_factor_dmma128, TreeFactor128Smem::bytes);
    if (rc) return rc;
    k_tree_factor_dmma128<<<(int)nev, TF_W * 32, TreeFactor128Smem::bytes, st>>>(Rslots, (int)n, events,
                                                                                 Ynode, taunode);
    return check_launch("k_tree_factor_dmma128");
  }
  if (p <= 64 && g_dmma_tree_factor) {
#define TFD_LAUNCH(NPV)                                                                  \
    {                                                                                    \
      int rc = prep(k_tree_factor_dmma<NPV>, TreeFactorDmmaSmem<NPV>::bytes);            \
      if (rc) return rc;                                                                 \
      k_tree_factor_dmma<NPV><<<(int)nev, THREADS, TreeFactorDmmaSmem<NPV>::bytes, st>>>( \
          Rslots, (int)n, events, Ynode, taunode);                                       \
    }
    if (p == 32) TFD_LAUNCH(32) else TFD_LAUNCH(64)
#undef TFD_LAUNCH
    return check_launch("k_tree_factor_dmma");
  }
  if (p == 32) {
    k_tree_factor_w32<<<(int)((nev + 3) / 4), 128, 0, st>>>(Rslots, (int)n, events, (int)nev, Ynode,
                                                           taunode, 0);
    return check_launch("k_tree_factor_w32");
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
  if (!p || !Ynode || !taunode || !events || !C || ncols < 1 || ldc < ncols || nev < 0 ||
      slot_rows < n)
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
  if (g_dmma_tree >= 2 && p == 128) {  // column-parallel warps, no barriers in the panel loop
    const size_t smc = TreeApplyCpSmem::bytes;
    dim3 gc((unsigned)nev, (unsigned)((ncols + TAC_KB - 1) / TAC_KB));
    if (transpose) {
      int rc = prep(k_tree_apply_cp<true>, smc); if (rc) return rc;
      k_tree_apply_cp<true><<<gc, THREADS, smc, st>>>(Ynode, taunode, (int)n, events, C, ldc, slot_rows,
                                                      ncols, zero_partner);
    } else {
      int rc = prep(k_tree_apply_cp<false>, smc); if (rc) return rc;
      k_tree_apply_cp<false><<<gc, THREADS, smc, st>>>(Ynode, taunode, (int)n, events, C, ldc, slot_rows,
                                                       ncols, zero_partner);
    }
    return check_launch("k_tree_apply_cp");
  }
  if (g_dmma_tree) {
    const size_t sm = TreeApplyDmmaSmem::bytes;
    dim3 gd((unsigned)nev, (unsigned)((ncols + TA_KB - 1) / TA_KB));
#define TAD_LAUNCH(TR)                                                                             \
    {                                                                                              \
      int rc = prep(k_tree_apply_dmma<TR>, sm);                                                    \
      if (rc) return rc;                                                                           \
      k_tree_apply_dmma<TR><<<gd, THREADS, sm, st>>>(Ynode, taunode, (int)n, events, C, ldc,      \
                                                     slot_rows, ncols, zero_partner);             \
    }
    if (transpose) TAD_LAUNCH(true) else TAD_LAUNCH(false)
#undef TAD_LAUNCH
    return check_launch("k_tree_apply_dmma");
  }
  if (p == 32) {
    dim3 g32((unsigned)((nev + 3) / 4), (unsigned)((ncols + 31) / 32));
    if (transpose)
      k_tree_apply_w32<true><<<g32, 128, 0, st>>>(Ynode, taunode, (int)n, events, (int)nev, C, ldc,
                                                  slot_rows, ncols, zero_partner);
    else
      k_tree_apply_w32<false><<<g32, 128, 0, st>>>(Ynode, taunode, (int)n, events, (int)nev, C, ldc,
                                                   slot_rows, ncols, zero_partner);
    return check_launch("k_tree_apply_w32");
  }
  switch (p) { TA_CASE(32) TA_CASE(64) TA_CASE(128) }
#undef TA_CASE
  return check_launch("k_tree_apply");
}

static int leaf_apply_impl(const double* Y, int64_t ldy, const double* tau, int64_t tau_stride,
                           int64_t m, int64_t n, int64_t P, double* C, int64_t ldc, int64_t ncols,
                           const double* S, int64_t lds, int64_t s_slot_rows, int transpose,
                           int zero_init, int tri_skip, void* stream, const double* Tin) {
  const int p = padded(n);
  if (!p || !Y || !tau || !C || P < 1 || m < n * P || ncols < 1 || ldc < ncols || ldy < n)
    return set_err(CAQR_ERR_ARG, "tsqr_f64_leaf_apply: bad arguments");
  if (tau_stride < min_tau_stride(m, n, P, m / P))
    return set_err(CAQR_ERR_ARG, "tsqr_f64_leaf_apply: tau_stride below the leaf's tiles * n");
  if (transpose && (S || zero_init || tri_skip))
    return set_err(CAQR_ERR_ARG, "S / zero_init / tri_skip only apply to Q (not Q^T)");
  const int64_t base = m / P;
  cudaStream_t st = (cudaStream_t)stream;
  const int kbs = (p == 128) ? (g_ht[2] >= 24 ? 2 : 4) : (p == 64 ? 2 : 1);
  dim3 grid((unsigned)P, (unsigned)((ncols + 32 * kbs - 1) / (32 * kbs)));
#define LA_LAUNCH(NPV, KB_, HTV)                                                                  \
  {                                                                                               \
    const size_t sm = LeafApplySmem<NPV, KB_, HTV>::bytes;                                             \
    if (transpose) {                                                                              \
      int rc = prep(k_leaf_apply<NPV, KB_, true, HTV>, sm); if (rc) return rc;                    \
      k_leaf_apply<NPV, KB_, true, HTV><<<grid, THREADS, sm, st>>>(Y, ldy, tau, tau_stride, m,    \
          (int)n, (int)P, base, C, ldc, ncols, S, lds, s_slot_rows, zero_init, tri_skip);         \
    } else {                                                                                      \
      int rc = prep(k_leaf_apply<NPV, KB_, false, HTV>, sm); if (rc) return rc;                   \
      k_leaf_apply<NPV, KB_, false, HTV><<<grid, THREADS, sm, st>>>(Y, ldy, tau, tau_stride, m,   \
          (int)n, (int)P, base, C, ldc, ncols, S, lds, s_slot_rows, zero_init, tri_skip);         \
    }                                                                                             \
  }
#define LA_CASE(NPV, KB_, HA, HB)                                                                 \
  case NPV: {                                                                                     \
    if (g_ht[np_index(NPV)] == HA) LA_LAUNCH(NPV, KB_, HA) else LA_LAUNCH(NPV, KB_, HB)           \
    break;                                                                                        \
  }
  if (p == 128 && g_ht[2] == 64) {
    // tall chain tiles (k_leaf_tt<64, 1, true>): the dense first tile through k_leaf_q_dmma
    // (dense_only), the chain tiles through k_tall_apply; Q^T: dense then chain, Q: chain then
    // dense, both through the leaf's top n rows of C
    const int h0 = WARPS * Geo<128>::HD;
    auto dense = [&](bool tr, int zi) -> int {
      const size_t smq = DmmaQSmem<128, 64>::bytes;
      dim3 gq((unsigned)P, (unsigned)((ncols + 63) / 64));
      if (tr) {
        int rc = prep(k_leaf_q_dmma<128, 64, 1, true>, smq); if (rc) return rc;
        k_leaf_q_dmma<128, 64, 1, true><<<gq, THREADS, smq, st>>>(Y, ldy, tau, tau_stride, m, (int)n,
            (int)P, base, C, ldc, ncols, nullptr, 0, 0, zi, 1);
      } else {
        int rc = prep(k_leaf_q_dmma<128, 64, 1, false>, smq); if (rc) return rc;
        k_leaf_q_dmma<128, 64, 1, false><<<gq, THREADS, smq, st>>>(Y, ldy, tau, tau_stride, m, (int)n,
            (int)P, base, C, ldc, ncols, nullptr, 0, 0, zi, 1);
      }
      return check_launch("k_leaf_q_dmma (dense tile)");
    };
#define TA_LAUNCH(TRV)                                                                            \
    {                                                                                             \
      const size_t sma = TallApplySmem::bytes;                                                    \
      dim3 ga((unsigned)P, (unsigned)((ncols + TLA_KB - 1) / TLA_KB));                              \
      int rc = prep(k_tall_apply<TRV>, sma); if (rc) return rc;                                   \
      k_tall_apply<TRV><<<ga, TLA_W * 32, sma, st>>>(Y, ldy, tau, tau_stride, m, (int)n, (int)P,   \
          base, C, ldc, ncols, S, lds, s_slot_rows, zero_init, h0);                               \
      rc = check_launch("k_tall_apply"); if (rc) return rc;                                       \
    }
    if (transpose) {
      int rc = dense(true, 0); if (rc) return rc;
      TA_LAUNCH(true)
      return CAQR_OK;
    }
    TA_LAUNCH(false)
    return dense(false, zero_init);
#undef TA_LAUNCH
  }
  const int var = transpose ? g_dmma_apply : g_dmma_q;
  const bool q16 = (p == 64 && g_ht[1] == 16) || (p == 128 && g_ht[2] == 16) ||
                   (p == 32 && g_ht[0] == 16);
  if ((!transpose && g_dmma_q && q16) || (transpose && p <= 64 && g_dmma_apply && q16)) {
#define LQ_LAUNCH(NPV, KBQ, MB, TR)                                                               \
    {                                                                                             \
      const size_t sm = DmmaQSmem<NPV, KBQ>::bytes;                                               \
      dim3 gq((unsigned)P, (unsigned)((ncols + KBQ - 1) / KBQ));                                  \
      int rc = prep(k_leaf_q_dmma<NPV, KBQ, MB, TR>, sm); if (rc) return rc;                      \
      k_leaf_q_dmma<NPV, KBQ, MB, TR><<<gq, THREADS, sm, st>>>(Y, ldy, tau, tau_stride, m,         \
          (int)n, (int)P, base, C, ldc, ncols, S, lds, s_slot_rows, zero_init, 0);                \
    }
    if (p == 32) {
      if (transpose) LQ_LAUNCH(32, 32, 2, true) else LQ_LAUNCH(32, 32, 2, false)
    } else if (transpose) {
      if (var == 2) LQ_LAUNCH(64, 32, 2, true)
      else if (var == 3) LQ_LAUNCH(64, 64, 1, true)
      else LQ_LAUNCH(64, 64, 2, true)
    } else if (p == 128) LQ_LAUNCH(128, 64, 2, false)  // two CTAs per SM: 3.6% on factor + explicit Q
    else if (var == 2) LQ_LAUNCH(64, 32, 2, false)
    else if (var == 3) LQ_LAUNCH(64, 64, 1, false)
    else LQ_LAUNCH(64, 64, 2, false)
#undef LQ_LAUNCH
    return check_launch("k_leaf_q_dmma");
  }
  switch (p) {
    LA_CASE(32, 1, 16, 32)
    case 64: {
      if (g_ht[1] == 16) LA_LAUNCH(64, 2, 16)
      else if (g_ht[1] == 24) LA_LAUNCH(64, 2, 24)
      else LA_LAUNCH(64, 2, 32)
      break;
    }
    case 128: {
      if (g_ht[2] == 24) LA_LAUNCH(128, 2, 24)
      else if (transpose && g_dmma_apply) {
        // fewer than one wave of 128-column CTAs (e.g. the look-ahead update of one
        // panel): 32-column blocks, 4x the CTAs at ~3x the T overhead per column
        // (C5: threshold 148 -> 466.6 ms, 296 -> 469.6, 592 -> 504.5)
        const bool narrow = P * ((ncols + 127) / 128) < 148;
#define AD_LAUNCH(KBV, DCPV, HASTV, GY)                                                            \
        {                                                                                          \
          const size_t sm = DmmaApplySmem<KBV>::bytes;                                             \
          int rc = prep(k_leaf_apply_dmma<KBV, DCPV, HASTV>, sm);                                  \
          if (rc) return rc;                                                                       \
          dim3 gd((unsigned)P, (unsigned)(GY));                                                    \
          k_leaf_apply_dmma<KBV, DCPV, HASTV><<<gd, THREADS, sm, st>>>(Y, ldy, tau, tau_stride, m, \
              (int)n, (int)P, base, C, ldc, ncols, Tin);                                           \
        }
        if (narrow) {
          if (Tin) AD_LAUNCH(32, false, true, (ncols + 31) / 32) else AD_LAUNCH(32, false, false, (ncols + 31) / 32)
        } else if (Tin) {
          // kept T: 64-column CTAs, two per SM (16 warps instead of 8 hide the fragment loads
          // and the ring waits; without the kept T the doubled T formation costs more than
          // that), dense first tile column-parallel (C5: 379.9 -> 341.9 ms)
          AD_LAUNCH(64, true, true, (ncols + 63) / 64)
        } else if (base <= 1024) {  // short leaves: column-parallel dense first tile
          if (Tin) AD_LAUNCH(128, true, true, (ncols + 127) / 128) else AD_LAUNCH(128, true, false, (ncols + 127) / 128)
        } else {
          if (Tin) AD_LAUNCH(128, false, true, (ncols + 127) / 128) else AD_LAUNCH(128, false, false, (ncols + 127) / 128)
        }
#undef AD_LAUNCH
      } else LA_LAUNCH(128, 4, 16)
      break;
    }
  }
#undef LA_CASE
#undef LA_LAUNCH
  return check_launch("k_leaf_apply");
}

int tsqr_f64_leaf_apply(const double* Y, int64_t ldy, const double* tau, int64_t tau_stride,
                        int64_t m, int64_t n, int64_t P, double* C, int64_t ldc, int64_t ncols,
                        const double* S, int64_t lds, int64_t s_slot_rows, int transpose,
                        int zero_init, int tri_skip, void* stream) {
  return leaf_apply_impl(Y, ldy, tau, tau_stride, m, n, P, C, ldc, ncols, S, lds, s_slot_rows,
                         transpose, zero_init, tri_skip, stream, nullptr);
}

int tsqr_f64_leaf_apply_t(const double* Y, int64_t ldy, const double* tau, int64_t tau_stride,
                          int64_t m, int64_t n, int64_t P, double* C, int64_t ldc, int64_t ncols,
                          const double* T, void* stream) {
  return leaf_apply_impl(Y, ldy, tau, tau_stride, m, n, P, C, ldc, ncols, nullptr, 0, 0, 1, 0, 0,
                         stream, tsqr_f64_panel_t_used(n) ? T : nullptr);
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
  const size_t sm = sizeof(double) * ((size_t)128 * 32 * KBS + 2 * WARPS * 32 * KBS +
                                      (size_t)WARPS * (32 * (RW + 2) + 32));
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

int tsqr_f64_geqr2(double* A, int64_t lda, int64_t m, int64_t n, double* tau, int* flag,
                   void* stream) {
  if (!A || !tau || m < 1 || n < 1 || n > INT32_MAX || lda < n)
    return set_err(CAQR_ERR_ARG, "tsqr_f64_geqr2: bad arguments");
  k_geqr2<<<1, GQ_THREADS, 0, (cudaStream_t)stream>>>(A, lda, m, (int)n, tau, flag);
  return check_launch("k_geqr2");
}

int tsqr_f64_form_t(const double* G, int64_t ldg, int64_t n, const double* tau, double* T,
                    int64_t ldt, void* stream) {
  if (!G || !tau || !T || n < 1 || n > INT32_MAX || ldg < n || ldt < n)
    return set_err(CAQR_ERR_ARG, "tsqr_f64_form_t: bad arguments");
  k_form_t<<<1, 1024, 0, (cudaStream_t)stream>>>(G, ldg, (int)n, tau, T, ldt);
  return check_launch("k_form_t");
}

int tsqr_f64_cholesky(double* G, int64_t ldg, int64_t n, int* info, void* stream) {
  if (!G || !info || n < 1 || n > INT32_MAX || ldg < n)
    return set_err(CAQR_ERR_ARG, "tsqr_f64_cholesky: bad arguments");
  k_cholesky<<<1, 1024, 0, (cudaStream_t)stream>>>(G, ldg, (int)n, info);
  return check_launch("k_cholesky");
}

int caqr_tune(int key, int value) {
  if (key >= CAQR_TUNE_CHAIN_HT_32 && key <= CAQR_TUNE_CHAIN_HT_128) {
    const int i = key - CAQR_TUNE_CHAIN_HT_32;
    const int a = 16, b = i == 2 ? 24 : 32;
    if (value != a && value != b && !(i == 1 && value == 24) && !(i == 2 && value == 64))
      return set_err(CAQR_ERR_ARG, "unsupported chain tile height");
    g_ht[i] = value;
    return CAQR_OK;
  }
  if (key == CAQR_TUNE_NARROW) {
    if (value < 0 || value > 3) return set_err(CAQR_ERR_ARG, "CAQR_TUNE_NARROW takes 0 .. 3");
    g_narrow = value;
    return CAQR_OK;
  }
  if (key == CAQR_TUNE_DMMA_DENSE) {
    g_dmma_dense = value ? 1 : 0;
    return CAQR_OK;
  }
  if (key == CAQR_TUNE_DMMA_TREE_FACTOR) {
    g_dmma_tree_factor = value ? 1 : 0;
    return CAQR_OK;
  }
  if (key == CAQR_TUNE_DMMA_TREE) {
    if (value < 0 || value > 2) return set_err(CAQR_ERR_ARG, "CAQR_TUNE_DMMA_TREE takes 0, 1 or 2");
    g_dmma_tree = value;
    return CAQR_OK;
  }
  if (key == CAQR_TUNE_DMMA_Q) {
    if (value < 0 || value > 4) return set_err(CAQR_ERR_ARG, "CAQR_TUNE_DMMA_Q takes 0 .. 4");
    g_dmma_q = value;
    return CAQR_OK;
  }
  if (key == CAQR_TUNE_DMMA_APPLY) {
    if (value < 0 || value > 4) return set_err(CAQR_ERR_ARG, "CAQR_TUNE_DMMA_APPLY takes 0 .. 4");
    g_dmma_apply = value;
    return CAQR_OK;
  }
  if (key == CAQR_TUNE_DMMA) {
    if (value < 0 || value > 3) return set_err(CAQR_ERR_ARG, "CAQR_TUNE_DMMA takes 0 .. 3");
    g_dmma = value;
    return CAQR_OK;
  }
  if (key == CAQR_TUNE_NARROW_PF) {
    if (value < 0 || value > 64) return set_err(CAQR_ERR_ARG, "CAQR_TUNE_NARROW_PF takes 0 .. 64");
    g_narrow_pf = value;
    return CAQR_OK;
  }
  if (key == CAQR_TUNE_FUSE) {
    if (value < 0) return set_err(CAQR_ERR_ARG, "CAQR_TUNE_FUSE takes 0 (off) or a CTA count");
    g_fuse = value;
    return CAQR_OK;
  }
  if (key == CAQR_TUNE_CC) {
    if (value != 0 && (value < 2 || value > 6)) return set_err(CAQR_ERR_ARG, "CAQR_TUNE_CC takes 0 or 2..6");
    g_cc = value;
    return CAQR_OK;
  }
  if (key == CAQR_TUNE_ZSTART) {
    g_zstart = value ? 1 : 0;
    return CAQR_OK;
  }
  return set_err(CAQR_ERR_ARG, "unknown tuning key");
}

int tsqr_f64_colmajor_to_rowmajor(const double* src, int64_t ld_src, int64_t rows, int64_t cols,
                                  double* dst, int64_t ld_dst, void* stream) {
  if (!src || !dst || rows < 0 || cols < 0 || cols > 65535 * 32 || ld_src < rows || ld_dst < cols)
    return set_err(CAQR_ERR_ARG, "tsqr_f64_colmajor_to_rowmajor: bad arguments");
  if (rows == 0 || cols == 0) return CAQR_OK;
  dim3 grid((unsigned)((rows + 31) / 32), (unsigned)((cols + 31) / 32));
  k_colmajor_to_rowmajor<<<grid, 256, 0, (cudaStream_t)stream>>>(src, ld_src, rows, (int)cols, dst,
                                                                 ld_dst);
  return check_launch("k_colmajor_to_rowmajor");
}

int caqr_f64_peak_probe(double* scratch, int mode, int iters, int blocks, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (mode == 0) k_peak_dfma<<<blocks, 256, 0, st>>>(scratch, iters);
  else k_peak_dmma<<<blocks, 256, 0, st>>>(scratch, iters);
  return check_launch("k_peak_probe");
}

}  // extern "C"
