// Device building blocks for the FP64 TSQR / CAQR kernels (sm_100a).
//
// Register layout shared by every kernel ("column-owned warp tiles"):
//   a CTA has WARPS = 8 warps; warp w holds RW consecutive rows of a block,
//   lane l holds the columns c = 32*s + l for the S = NP/32 column slots.
//   Column dot products over a warp's rows are therefore lane-local FMA
//   chains (no shuffles); only reductions ACROSS warps go through shared
//   memory.  NP is n rounded up to 32/64/128; padded columns are zero and stay
//   exactly zero through every reflector (their R row entries are zero).
//
// Two execution patterns:
//   * cta_factor / cta_apply: CTA-cooperative sweep over a block held by all
//     8 warps (dense first tile of a leaf, stacked-triangle tree combine,
//     triangle-on-rectangle).  Two __syncthreads per reflector (factor) or one
//     (apply, double-buffered partials).
//   * ring_factor_tile / ring_apply_tile: the flat-tree chain of
//     triangle-on-rectangle steps (Alg. 2 of the paper) as a systolic ring:
//     each warp owns one HW-row tile, the n pivot rows (R, or the top block of
//     C) live in shared memory and flow warp -> warp through per-row version
//     counters, so no CTA barrier is ever taken inside the chain.
//
// Reflector conventions follow pkg/src/caqr/householder.py:9-11,89-114.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace tsqr {

constexpr int WARPS = 8;
constexpr int THREADS = WARPS * 32;
constexpr unsigned FULL = 0xffffffffu;

__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }

enum Mode { DENSE = 0, STACKED = 1, TRIRECT = 2, STACKEDQ = 3 };

// Per padded width: S column slots per lane, HD rows per warp in the dense
// first tile (H0 = 8*HD >= NP rows).  The chain tile height HT is a separate,
// tunable template parameter of the chain / apply kernels.
template <int NP> struct Geo;
template <> struct Geo<32>  { static constexpr int S = 1, HD = 32; };
template <> struct Geo<64>  { static constexpr int S = 2, HD = 16; };
template <> struct Geo<128> { static constexpr int S = 4, HD = 16; };
// Warps of the factorization ring for a chain tile height (register budget:
// 16 warps -> 128 regs, 8 warps -> 255 regs per thread).
template <int NP, int HT> struct RingCfg {
  static constexpr int WARPS_R = (HT * (NP / 32) <= 32 && HT <= 16) ? 16 : 8;
};

// house_gen scalars (householder.py:97-113): given x0 and sigma = ||x[1:]||^2
// return beta, tau and the scale 1/(x0 - beta) applied to x[1:].
__device__ __forceinline__ void house_scalars(double x0, double sigma, double& beta,
                                              double& tau, double& scale) {
  if (sigma == 0.0) {
    scale = 0.0;
    if (x0 == 0.0) { tau = 0.0; beta = 0.0; }
    else if (x0 >= 0.0) { tau = 0.0; beta = x0; }
    else { tau = 2.0; beta = -x0; }
    return;
  }
  const double nrm = sqrt(fma(x0, x0, sigma));
  beta = (x0 >= 0.0) ? -nrm : nrm;
  // x0 - beta and beta carry the same sign and |x0 - beta| >= |beta| > 0
  scale = __drcp_rn(x0 - beta);
  tau = (beta - x0) * __drcp_rn(beta);
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];"
               : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.cta.shared::cta.b32 [%0], %1;"
               :: "r"((unsigned)__cvta_generic_to_shared(p)), "r"(v) : "memory");
}

// Warp waits until ver[j] == target (lane 0 polls, then the warp syncs).
__device__ __forceinline__ void ring_wait(const int* ver, int target, int lane) {
  if (lane == 0) {
    while (ld_acquire(ver) != target) { }
  }
  __syncwarp();
  __threadfence_block();
}
__device__ __forceinline__ void ring_signal(int* ver, int value, int lane) {
  __syncwarp();
  if (lane == 0) {
    __threadfence_block();
    st_release(ver, value);
  }
}

// cp.async granules (8 or 16 bytes, zero fill when bytes < G)
template <int G>
__device__ __forceinline__ void cp_async(unsigned dst, const void* src, unsigned bytes) {
  if constexpr (G == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" :: "r"(dst), "l"(src), "r"(bytes)
                 : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" :: "r"(dst), "l"(src), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" :: "n"(N) : "memory"); }

// FP64 tensor-core MMA, D = A B + D (m8n8k4, A row-major 8x4, B col-major 4x8):
// lane (g = lane/4, q = lane%4) supplies A[g][q], B[q][g] and holds D[g][2q], D[g][2q+1]
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// ---------------------------------------------------------------------------
// Tile load / store (row-major global, leading dimension ld, zero padding)
// ---------------------------------------------------------------------------
template <int RW, int S>
__device__ __forceinline__ void load_rows(double (&X)[RW][S], const double* __restrict__ src,
                                          int64_t ld, int rows_valid, int ncols, int col0,
                                          bool& bad) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < RW; ++k) {
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int c = col0 + 32 * s + lane;
      double x = 0.0;
      if (k < rows_valid && c < ncols) x = __ldg(src + (int64_t)k * ld + c);
      bad |= !isfinite(x);
      X[k][s] = x;
    }
  }
}

template <int RW, int S>
__device__ __forceinline__ void store_rows(const double (&X)[RW][S], double* dst, int64_t ld,
                                           int rows_valid, int ncols, int col0, int row_lo = 0) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < RW; ++k) {
    if (k < row_lo || k >= rows_valid) continue;
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int c = col0 + 32 * s + lane;
      if (c < ncols) dst[(int64_t)k * ld + c] = X[k][s];
    }
  }
}

// Leaner reflector scalars for the pipelined ring: y = rsqrt(a) refined from
// the MUFU seed (~2^-20) is accurate to a few ulp, so
// nrm = a*y needs no correction and tau = 1 + |x0|/nrm = 1 + |x0|*y needs no
// division; scale = 1/(x0 - beta) = sign(x0)/(|x0| + nrm).  Conventions of
// house_gen (householder.py:101-111), branch-free.
// Two-Newton-step variant (the narrow n <= 8 kernel keeps it: its lane-private
// chains schedule better with it -- measured, C4 2.10 vs 2.20 ms).
__device__ __forceinline__ void house_newton(double x0, double sigma, double& beta, double& tau,
                                             double& scale) {
  const double a = fma(x0, x0, sigma);
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
  const double h = 0.5 * a;
  y = y * fma(-h * y, y, 1.5);
  y = y * fma(-h * y, y, 1.5);
  const double nrm = a * y;
  const double ax = fabs(x0);
  const double d = ax + nrm;
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  r = r * fma(-d, r, 2.0);
  r = r * fma(-d, r, 2.0);
  const bool pos = (x0 >= 0.0);
  const bool z = (sigma == 0.0);
  beta = z ? ax : (pos ? -nrm : nrm);
  tau = z ? (pos ? 0.0 : 2.0) : fma(ax, y, 1.0);
  scale = z ? 0.0 : (pos ? r : -r);
}
__device__ __forceinline__ double neg_alu(double x) {  // sign flip on the ALU, off the FP64 pipe
  return __hiloint2double(__double2hiint(x) ^ (int)0x80000000, __double2loint(x));
}
__device__ __forceinline__ void house_lean(double x0, double sigma, double& beta, double& tau,
                                           double& scale) {
  // MUFU seeds (~2^-20) refined by one third-order step each (error ~2^-60, within
  // 2.3 / 3.5 ulp: tools/house_acc.cu): y (1 + e/2 + 3e^2/8) with e = 1 - a y^2,
  // and r (1 + e + e^2) with e = 1 - d r; the reciprocal is seeded from the rsqrt
  // seed so the two MUFU latencies overlap
  const double a = fma(x0, x0, sigma);
  const double ax = fabs(x0);
  double y, r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
  const double d0 = fma(a, y, ax);
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d0));
  {
    const double e = fma(-a * y, y, 1.0);
    y = fma(y, e * fma(e, 0.375, 0.5), y);
  }
  const double nrm = a * y;
  const double d = ax + nrm;
  {
    const double e = fma(-d, r, 1.0);
    r = fma(r, fma(e, e, e), r);
  }
  const bool pos = (x0 >= 0.0);
  const bool z = (sigma == 0.0);
  beta = z ? ax : (pos ? neg_alu(nrm) : nrm);
  tau = z ? (pos ? 0.0 : 2.0) : fma(ax, y, 1.0);
  scale = z ? 0.0 : (pos ? r : neg_alu(r));
}

// ---------------------------------------------------------------------------
// CTA-cooperative factorization sweep.
//   DENSE  : pivot row j is row j of the block (internal), support rows r >= j
//            -> qr_unblocked on the block (householder.py:128-145).
//   STACKED: pivot rows external (Ps, stride NP), support rows r <= j
//            -> qr_stacked_triangles q=2 with X = lower triangle (:263-294).
//   TRIRECT: pivot rows external, support all rows
//            -> qr_triangle_on_rect with X = rectangle (:297-332).
// Block row r = w*RW + k.  tau_out[j] written by thread 0 (nullable).
// smem: red[WARPS], sx0[1], part[WARPS*NP], vbuf[WARPS*RW].
// ---------------------------------------------------------------------------
// Columns 32 s .. 32 s + 31 (s a template parameter: with s a loop variable nvcc kept the
// outer loop rolled -- the inner loop returns early -- and the tile X[.][s] went to local
// memory, 587 LDL / STL in k_leaf_dense<128>).  Returns true when column n was reached.
template <int NP, int RW, int MODE, int s>
__device__ __forceinline__ bool cta_factor_seg(double (&X)[RW][NP / 32], double* Ps, int n,
                                               double* tau_out, double* red, double* sx0,
                                               double* part, double* vbuf) {
  constexpr int S = NP / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  {
    for (int jj = 0; jj < 32; ++jj) {
      const int j = 32 * s + jj;
      if (j >= n) return true;
      const int pw = j / RW;
      // -- 1. partial sigma of column j over this warp's support rows
      double sga[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int k = 0; k < RW; ++k) {
        const int r = w * RW + k;
        const bool in = (MODE == DENSE) ? (r > j)
                        : (MODE == STACKED ? (r <= j) : (MODE == STACKEDQ ? (r % n) <= j : true));
        const double x = in ? X[k][s] : 0.0;
        sga[k & 3] = fma(x, x, sga[k & 3]);
      }
      const double sg = (sga[0] + sga[1]) + (sga[2] + sga[3]);
      if (lane == jj) red[w] = sg;
      if (MODE == DENSE && w == pw && lane == jj) {
        // (selp in inline asm: written as `if (k == kk) x0 = X[k][s]` nvcc turns the chain into
        // X[kk][s], a dynamic index that moves the whole tile X to local memory)
        double x0 = 0.0;
        const int kk = j - pw * RW;
#pragma unroll
        for (int k = 0; k < RW; ++k)
          asm("{\n\t.reg .pred p;\n\tsetp.eq.s32 p, %2, %3;\n\tselp.f64 %0, %1, %0, p;\n\t}"
              : "+d"(x0) : "d"(X[k][s]), "r"(k), "r"(kk));
        *sx0 = x0;
      }
      __syncthreads();
      double rq[WARPS];
#pragma unroll
      for (int q = 0; q < WARPS; ++q) rq[q] = red[q];
#pragma unroll
      for (int h = WARPS / 2; h >= 1; h /= 2)
#pragma unroll
        for (int q = 0; q < h; ++q) rq[q] += rq[q + h];
      const double sigma = rq[0];
      const double x0 = (MODE == DENSE) ? *sx0 : Ps[j * NP + j];
      double beta, tau, scale;
      house_lean(x0, sigma, beta, tau, scale);
      const bool wact = (MODE == DENSE) ? (w >= pw) : (MODE == STACKED ? (w <= pw) : true);
      double v[RW];
      double pold[S];
      if (wact) {
        // -- 2. reflector entries for this warp's rows (lane jj owns column j)
        if (lane == jj) {
#pragma unroll
          for (int k = 0; k < RW; ++k) {
            const int r = w * RW + k;
            const bool in = (MODE == DENSE) ? (r > j)
                            : (MODE == STACKED ? (r <= j) : (MODE == STACKEDQ ? (r % n) <= j : true));
            double vk = 0.0;
            if (in) vk = X[k][s] * scale;
            else if (MODE == DENSE && r == j) vk = 1.0;
            vbuf[w * RW + k] = vk;
            if (in) X[k][s] = vk;
            else if (MODE == DENSE && r == j) X[k][s] = beta;
          }
        }
        __syncwarp();
        // NP = 128: v stays in shared memory (warp-private segment, rewritten only after the
        // next CTA barrier): 32 registers less where the tile alone takes 128
#define VV(k) (NP == 128 ? vbuf[w * RW + (k)] : v[k])
        if (NP != 128) {
#pragma unroll
          for (int k = 0; k < RW; ++k) v[k] = vbuf[w * RW + k];
        }
        // -- 3. partial dots with the trailing columns
#pragma unroll
        for (int s2 = s; s2 < S; ++s2) {
          double pa[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
          for (int k = 0; k < RW; ++k) pa[k & 3] = fma(VV(k), X[k][s2], pa[k & 3]);
          double p = (pa[0] + pa[1]) + (pa[2] + pa[3]);
          if (MODE != DENSE && w == 0) {
            pold[s2] = Ps[j * NP + 32 * s2 + lane];
            p += pold[s2];
          }
          part[w * NP + 32 * s2 + lane] = p;
        }
      }
      __syncthreads();
      if (wact) {
        const int q0 = (MODE == DENSE) ? pw : 0;
        const int q1 = (MODE == STACKED) ? pw : WARPS - 1;
        // -- 4. rank-1 update of the trailing columns
#pragma unroll
        for (int s2 = s; s2 < S; ++s2) {
          const int c = 32 * s2 + lane;
          if (s2 > s || lane > jj) {
            // the partials of warps q0 .. q1, all loads in flight at once; two running sums by
            // the parity of q: the same two sums as pairing from q0 (swapped when q0 is odd)
            double t0 = 0.0, t1 = 0.0;
#pragma unroll
            for (int q = 0; q < WARPS; ++q) {
              const double pv = part[q * NP + c];
              const double pz = (q >= q0 && q <= q1) ? pv : 0.0;
              if (q & 1) t1 += pz;
              else t0 += pz;
            }
            const double wv = tau * (t0 + t1);
#pragma unroll
            for (int k = 0; k < RW; ++k) X[k][s2] = fma(-VV(k), wv, X[k][s2]);
            if (MODE != DENSE && w == 0) Ps[j * NP + c] = pold[s2] - wv;
          }
        }
        if (MODE != DENSE && w == 0 && lane == jj) Ps[j * NP + j] = beta;
      }
      if (threadIdx.x == 0 && tau_out) tau_out[j] = tau;
    }
  }
  return false;
}

#undef VV

template <int NP, int RW, int MODE>
__device__ __forceinline__ void cta_factor(double (&X)[RW][NP / 32], double* Ps, int n,
                                           double* tau_out, double* red, double* sx0,
                                           double* part, double* vbuf) {
  constexpr int S = NP / 32;
  if (cta_factor_seg<NP, RW, MODE, 0>(X, Ps, n, tau_out, red, sx0, part, vbuf)) return;
  if constexpr (S > 1) {
    if (cta_factor_seg<NP, RW, MODE, 1>(X, Ps, n, tau_out, red, sx0, part, vbuf)) return;
  }
  if constexpr (S > 2) {
    if (cta_factor_seg<NP, RW, MODE, 2>(X, Ps, n, tau_out, red, sx0, part, vbuf)) return;
    cta_factor_seg<NP, RW, MODE, 3>(X, Ps, n, tau_out, red, sx0, part, vbuf);
  }
}

// Branch-free reflector scalars for the pipelined ring.  Same conventions
// as house_scalars (householder.py:101-111); sqrt and reciprocals from the
// MUFU seeds refined by Newton steps (within 1 ulp), so the whole computation
// schedules as straight-line code next to independent DFMA work.
__device__ __forceinline__ double rsqrt_nr(double a) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
  const double h = 0.5 * a;
  y = y * fma(-h * y, y, 1.5);
  y = y * fma(-h * y, y, 1.5);
  return y;
}
__device__ __forceinline__ double rcp_nr(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  r = r * fma(-d, r, 2.0);
  r = r * fma(-d, r, 2.0);
  const double e = fma(-d, r, 1.0);
  return fma(r, e, r);
}
// Outputs beta, tau and scale = 1/(x0 - beta) (0 when sigma == 0).
__device__ __forceinline__ void house_fast(double x0, double sigma, double& beta, double& tau,
                                           double& scale) {
  const double a = fma(x0, x0, sigma);
  const double y = rsqrt_nr(a);
  double nrm = a * y;
  nrm = fma(0.5 * y, fma(-nrm, nrm, a), nrm);
  const double b = (x0 >= 0.0) ? -nrm : nrm;
  const double d = x0 - b;
  const double sc = rcp_nr(d);
  const double tg = -d * rcp_nr(b);
  const bool z = (sigma == 0.0);
  beta = z ? fabs(x0) : b;
  tau = z ? ((x0 < 0.0) ? 2.0 : 0.0) : tg;
  scale = z ? 0.0 : sc;
}

// ---------------------------------------------------------------------------
#ifdef TSQR_SPIN_PROBE
__device__ unsigned long long g_spin_cycles[2];
#endif


// Raw dot products of the broadcast column v with this lane's columns in
// slots [s0, S) (the next reflector's p, before its scalars are known).
template <int NP, int HT, int s0>
__device__ __forceinline__ void raw_dots(const double (&X)[HT][NP / 32], const double (&v)[HT],
                                         double (&p)[NP / 32]) {
  constexpr int S = NP / 32;
#pragma unroll
  for (int s2 = s0; s2 < S; ++s2) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
    for (int k = 0; k < HT; k += 4) {
      a0 = fma(v[k], X[k][s2], a0);
      a1 = fma(v[k + 1], X[k + 1][s2], a1);
      a2 = fma(v[k + 2], X[k + 2][s2], a2);
      a3 = fma(v[k + 3], X[k + 3][s2], a3);
    }
    p[s2] = (a0 + a1) + (a2 + a3);
  }
}

// One reflector step of the ring.  Entering step j: v = raw column x_j,
// p[s2] = x_j . X[:, c] for this lane's columns (raw dots), and the scalars
// (beta, tau, scale) of reflector j.  s = slot of column j (lane jj), SN =
// slot of column j+1.  The critical path is only: coefficient and rank-1
// update of column j+1 -> its norm -> sqrt / reciprocal of reflector j+1.
// The other columns' updates, the R row write-back, the broadcast of x_{j+1}
// and the next raw dots are issued while those scalars are in flight.
template <int NP, int HT, int s, int SN>
__device__ __forceinline__ void ring_step(double (&X)[HT][NP / 32], double (&v)[HT],
                                          double (&p)[NP / 32], double (&mysc)[NP / 32],
                                          double& beta, double& tau, double& scale, double* Rs,
                                          int* ver, double* vb, int n, int t, int jj,
                                          double* tau_tile) {
  constexpr int S = NP / 32;
  const int lane = threadIdx.x & 31;
  const int j = 32 * s + jj;
  const int jn = j + 1;
  const bool more = (SN < S) && (jn < n);
  constexpr int SNc = (SN < S) ? SN : S - 1;
  double* Rj = Rs + j * NP;
  // (1) ring: R row j+1 as left by the previous tile
  double x0n = 1.0;
  if (more) {
#ifdef TSQR_SPIN_PROBE
    const long long t0_ = clock64();
#endif
    while (ld_acquire(ver + jn) != t) { }
#ifdef TSQR_SPIN_PROBE
    if (lane == 0) atomicAdd(&g_spin_cycles[0], clock64() - t0_);
#endif
    x0n = Rs[jn * NP + jn];
  }
  // (2) slot SN: coefficient, rank-1 update fused with the next column's norm
  double sg = 0.0;
  if (SN < S) {
    const double r = Rj[32 * SNc + lane];
    const bool act = (SNc > s) || (lane > jj);
    const double q = act ? tau * fma(scale, p[SNc], r) : 0.0;
    const double w = q * scale;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
    for (int k = 0; k < HT; k += 4) {
      X[k][SNc] = fma(-v[k], w, X[k][SNc]);
      X[k + 1][SNc] = fma(-v[k + 1], w, X[k + 1][SNc]);
      X[k + 2][SNc] = fma(-v[k + 2], w, X[k + 2][SNc]);
      X[k + 3][SNc] = fma(-v[k + 3], w, X[k + 3][SNc]);
      s0 = fma(X[k][SNc], X[k][SNc], s0);
      s1 = fma(X[k + 1][SNc], X[k + 1][SNc], s1);
      s2 = fma(X[k + 2][SNc], X[k + 2][SNc], s2);
      s3 = fma(X[k + 3][SNc], X[k + 3][SNc], s3);
    }
    sg = (s0 + s1) + (s2 + s3);
    if (32 * SNc + lane > j) Rj[32 * SNc + lane] = r - q;
  }
  sg = __shfl_sync(FULL, sg, jn & 31);
  // (3) scalars of reflector j+1 (latency) || the remaining columns of reflector j
  double nbeta, ntau, nscale;
  house_lean(x0n, sg, nbeta, ntau, nscale);
#pragma unroll
  for (int s2 = s; s2 < S; ++s2) {
    if (s2 == SN) continue;
    if (s2 == s && SN != s) continue;  // jj == 31: nothing of slot s lies right of j
    const double r = Rj[32 * s2 + lane];
    const bool act = (s2 > s) || (lane > jj);
    const double q = act ? tau * fma(scale, p[s2], r) : 0.0;
    const double w = q * scale;
#pragma unroll
    for (int k = 0; k < HT; ++k) X[k][s2] = fma(-v[k], w, X[k][s2]);
    if (32 * s2 + lane > j) Rj[32 * s2 + lane] = r - q;
  }
  if (lane == jj) Rj[j] = beta;
  if (lane == 0 && tau_tile) tau_tile[j] = tau;
  // (4) hand R row j to the next tile
  __syncwarp();
  if (lane == 0) {
    __threadfence_block();
    st_release(ver + j, t + 1);
  }
  if (!more) return;
  // (5) broadcast x_{j+1} (raw) and form its dot products with the updated tile
  if (lane == (jn & 31)) {
    mysc[SNc] = nscale;
#pragma unroll
    for (int k = 0; k < HT; k += 2)
      *reinterpret_cast<double2*>(vb + k) = make_double2(X[k][SNc], X[k + 1][SNc]);
  }
  __syncwarp();
#pragma unroll
  for (int k = 0; k < HT; k += 2) {
    const double2 t2 = *reinterpret_cast<const double2*>(vb + k);
    v[k] = t2.x;
    v[k + 1] = t2.y;
  }
  __syncwarp();  // vb may be overwritten in the next step
  raw_dots<NP, HT, SNc>(X, v, p);
  beta = nbeta;
  tau = ntau;
  scale = nscale;
}

template <int NP, int HT, int s>
__device__ __forceinline__ void ring_slot(double (&X)[HT][NP / 32], double (&v)[HT],
                                          double (&p)[NP / 32], double (&mysc)[NP / 32],
                                          double& beta, double& tau, double& scale, double* Rs,
                                          int* ver, double* vb, int n, int t, double* tau_tile) {
  for (int jj = 0; jj < 31; ++jj) {
    if (32 * s + jj >= n) return;
    ring_step<NP, HT, s, s>(X, v, p, mysc, beta, tau, scale, Rs, ver, vb, n, t, jj, tau_tile);
  }
  if (32 * s + 31 >= n) return;
  ring_step<NP, HT, s, s + 1>(X, v, p, mysc, beta, tau, scale, Rs, ver, vb, n, t, 31, tau_tile);
}

// ---------------------------------------------------------------------------
// Ring step, register-broadcast form.  Same arithmetic as ring_step, but the
// raw column x_{j+1} is broadcast by shuffles into a second vector (vn) right
// after its rank-1 update, so its dot products and the scalars of reflector
// j+1 overlap the rest of reflector j's update; the two vectors swap roles
// every step (ring_slot3 unrolls by two).  Pivot rows are acquired two at a
// time (spin on even steps only) and the R row hand-off is a plain release
// after __syncwarp (which orders the other lanes' R stores before it).
// ---------------------------------------------------------------------------
template <int NP, int HT, int s, int SN, bool SPIN>
__device__ __forceinline__ void ring_step3(double (&X)[HT][NP / 32], const double (&v)[HT],
                                           double (&vn)[HT], double (&p)[NP / 32],
                                           double (&mysc)[NP / 32], double& beta, double& tau,
                                           double& scale, double* Rs, int* ver, int n, int t,
                                           int jj, double* tau_tile) {
  constexpr int S = NP / 32;
  const int lane = threadIdx.x & 31;
  const int j = 32 * s + jj;
  const int jn = j + 1;
  const bool more = (SN < S) && (jn < n);
  constexpr int SNc = (SN < S) ? SN : S - 1;
  double* Rj = Rs + j * NP;
  double x0n = 1.0;
  if (more) {
    if (SPIN) {
      const int jw = (jn + 1 < n) ? jn + 1 : jn;
      while (ld_acquire(ver + jw) != t) { }
    }
    x0n = Rs[jn * NP + jn];
  }
  double sg = 0.0;
  if (SN < S) {
    const double r = Rj[32 * SNc + lane];
    const bool act = (SNc > s) || (lane > jj);
    const double q = act ? tau * fma(scale, p[SNc], r) : 0.0;
    const double w = q * scale;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
    for (int k = 0; k < HT; k += 4) {
      X[k][SNc] = fma(-v[k], w, X[k][SNc]);
      X[k + 1][SNc] = fma(-v[k + 1], w, X[k + 1][SNc]);
      X[k + 2][SNc] = fma(-v[k + 2], w, X[k + 2][SNc]);
      X[k + 3][SNc] = fma(-v[k + 3], w, X[k + 3][SNc]);
      s0 = fma(X[k][SNc], X[k][SNc], s0);
      s1 = fma(X[k + 1][SNc], X[k + 1][SNc], s1);
      s2 = fma(X[k + 2][SNc], X[k + 2][SNc], s2);
      s3 = fma(X[k + 3][SNc], X[k + 3][SNc], s3);
    }
    sg = (s0 + s1) + (s2 + s3);
    if (32 * SNc + lane > j) Rj[32 * SNc + lane] = r - q;
  }
  const int src = jn & 31;
  sg = __shfl_sync(FULL, sg, src);
  if (more) {
#pragma unroll
    for (int k = 0; k < HT; ++k) vn[k] = __shfl_sync(FULL, X[k][SNc], src);
  }
  double nbeta, ntau, nscale;
  house_lean(x0n, sg, nbeta, ntau, nscale);
#pragma unroll
  for (int s2 = s; s2 < S; ++s2) {
    if (s2 == SN) continue;
    if (s2 == s && SN != s) continue;
    const double r = Rj[32 * s2 + lane];
    const bool act = (s2 > s) || (lane > jj);
    const double q = act ? tau * fma(scale, p[s2], r) : 0.0;
    const double w = q * scale;
#pragma unroll
    for (int k = 0; k < HT; ++k) X[k][s2] = fma(-v[k], w, X[k][s2]);
    if (32 * s2 + lane > j) Rj[32 * s2 + lane] = r - q;
  }
  if (lane == jj) Rj[j] = beta;
  if (lane == 0 && tau_tile) tau_tile[j] = tau;
  __syncwarp();
  if (lane == 0) st_release(ver + j, t + 1);
  if (!more) return;
  if (lane == src) mysc[SNc] = nscale;
  raw_dots<NP, HT, SNc>(X, vn, p);
  beta = nbeta;
  tau = ntau;
  scale = nscale;
}

template <int NP, int HT, int s>
__device__ __forceinline__ void ring_slot3(double (&X)[HT][NP / 32], double (&va)[HT],
                                           double (&vb)[HT], double (&p)[NP / 32],
                                           double (&mysc)[NP / 32], double& beta, double& tau,
                                           double& scale, double* Rs, int* ver, int n, int t,
                                           double* tau_tile) {
  for (int jj = 0; jj < 30; jj += 2) {
    if (32 * s + jj >= n) return;
    ring_step3<NP, HT, s, s, true>(X, va, vb, p, mysc, beta, tau, scale, Rs, ver, n, t, jj, tau_tile);
    if (32 * s + jj + 1 >= n) return;
    ring_step3<NP, HT, s, s, false>(X, vb, va, p, mysc, beta, tau, scale, Rs, ver, n, t, jj + 1,
                                    tau_tile);
  }
  if (32 * s + 30 >= n) return;
  ring_step3<NP, HT, s, s, true>(X, va, vb, p, mysc, beta, tau, scale, Rs, ver, n, t, 30, tau_tile);
  if (32 * s + 31 >= n) return;
  ring_step3<NP, HT, s, s + 1, false>(X, vb, va, p, mysc, beta, tau, scale, Rs, ver, n, t, 31,
                                      tau_tile);
}

template <int NP, int HW>
__device__ __forceinline__ void ring_factor_tile3(double (&X)[HW][NP / 32], double* Rs, int* ver,
                                                  int n, int t, double* tau_tile) {
  constexpr int S = NP / 32;
  const int lane = threadIdx.x & 31;
  double mysc[S];
#pragma unroll
  for (int s = 0; s < S; ++s) mysc[s] = 1.0;
  double va[HW], vb[HW];
  double p[S];
  double beta, tau, scale;
  {
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int k = 0; k < HW; k += 2) {
      s0 = fma(X[k][0], X[k][0], s0);
      s1 = fma(X[k + 1][0], X[k + 1][0], s1);
    }
    const double sg = __shfl_sync(FULL, s0 + s1, 0);
#pragma unroll
    for (int k = 0; k < HW; ++k) va[k] = __shfl_sync(FULL, X[k][0], 0);
    while (ld_acquire(ver) != t) { }
    house_lean(Rs[0], sg, beta, tau, scale);
    if (lane == 0) mysc[0] = scale;
    raw_dots<NP, HW, 0>(X, va, p);
  }
  ring_slot3<NP, HW, 0>(X, va, vb, p, mysc, beta, tau, scale, Rs, ver, n, t, tau_tile);
  if constexpr (S > 1) ring_slot3<NP, HW, 1>(X, va, vb, p, mysc, beta, tau, scale, Rs, ver, n, t, tau_tile);
  if constexpr (S > 2) ring_slot3<NP, HW, 2>(X, va, vb, p, mysc, beta, tau, scale, Rs, ver, n, t, tau_tile);
  if constexpr (S > 3) ring_slot3<NP, HW, 3>(X, va, vb, p, mysc, beta, tau, scale, Rs, ver, n, t, tau_tile);
#pragma unroll
  for (int s = 0; s < S; ++s)
#pragma unroll
    for (int k = 0; k < HW; ++k) X[k][s] *= mysc[s];
}

// ---------------------------------------------------------------------------
// Shared-vector variant of the ring step: the broadcast column x_j is read
// from a double-buffered per-warp shared slot (vb + (j&1)*HT) at its point of
// use instead of being held in registers, which frees 2*HT registers per
// thread for taller tiles (HT = 24 at n = 128).
// ---------------------------------------------------------------------------
template <int NP, int HT, int s0>
__device__ __forceinline__ void raw_dots_vs(const double (&X)[HT][NP / 32], const double* vx,
                                            double (&p)[NP / 32]) {
  constexpr int S = NP / 32;
  double a[S][2];
#pragma unroll
  for (int s2 = s0; s2 < S; ++s2) { a[s2][0] = 0.0; a[s2][1] = 0.0; }
#pragma unroll
  for (int k = 0; k < HT; k += 2) {
    const double2 v2 = *reinterpret_cast<const double2*>(vx + k);
#pragma unroll
    for (int s2 = s0; s2 < S; ++s2) {
      a[s2][0] = fma(v2.x, X[k][s2], a[s2][0]);
      a[s2][1] = fma(v2.y, X[k + 1][s2], a[s2][1]);
    }
  }
#pragma unroll
  for (int s2 = s0; s2 < S; ++s2) p[s2] = a[s2][0] + a[s2][1];
}

template <int NP, int HT, int s, int SN>
__device__ __forceinline__ void ring_step_vs(double (&X)[HT][NP / 32], double (&p)[NP / 32],
                                             double (&mysc)[NP / 32], double& beta, double& tau,
                                             double& scale, double* Rs, int* ver, double* vb,
                                             int n, int t, int jj, double* tau_tile) {
  constexpr int S = NP / 32;
  const int lane = threadIdx.x & 31;
  const int j = 32 * s + jj;
  const int jn = j + 1;
  const bool more = (SN < S) && (jn < n);
  constexpr int SNc = (SN < S) ? SN : S - 1;
  double* Rj = Rs + j * NP;
  const double* vx = vb + (j & 1) * HT;   // x_j
  double* vnx = vb + (jn & 1) * HT;       // x_{j+1}
  double x0n = 1.0;
  if (more) {
    while (ld_acquire(ver + jn) != t) { }
    x0n = Rs[jn * NP + jn];
  }
  double sg = 0.0;
  if (SN < S) {
    const double r = Rj[32 * SNc + lane];
    const bool act = (SNc > s) || (lane > jj);
    const double q = act ? tau * fma(scale, p[SNc], r) : 0.0;
    const double w = q * scale;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
    for (int k = 0; k < HT; k += 4) {
      const double2 va = *reinterpret_cast<const double2*>(vx + k);
      const double2 vc = *reinterpret_cast<const double2*>(vx + k + 2);
      X[k][SNc] = fma(-va.x, w, X[k][SNc]);
      X[k + 1][SNc] = fma(-va.y, w, X[k + 1][SNc]);
      X[k + 2][SNc] = fma(-vc.x, w, X[k + 2][SNc]);
      X[k + 3][SNc] = fma(-vc.y, w, X[k + 3][SNc]);
      s0 = fma(X[k][SNc], X[k][SNc], s0);
      s1 = fma(X[k + 1][SNc], X[k + 1][SNc], s1);
      s2 = fma(X[k + 2][SNc], X[k + 2][SNc], s2);
      s3 = fma(X[k + 3][SNc], X[k + 3][SNc], s3);
    }
    sg = (s0 + s1) + (s2 + s3);
    if (32 * SNc + lane > j) Rj[32 * SNc + lane] = r - q;
  }
  sg = __shfl_sync(FULL, sg, jn & 31);
  double nbeta, ntau, nscale;
  house_lean(x0n, sg, nbeta, ntau, nscale);
#pragma unroll
  for (int s2 = s; s2 < S; ++s2) {
    if (s2 == SN) continue;
    if (s2 == s && SN != s) continue;
    const double r = Rj[32 * s2 + lane];
    const bool act = (s2 > s) || (lane > jj);
    const double q = act ? tau * fma(scale, p[s2], r) : 0.0;
    const double w = q * scale;
#pragma unroll
    for (int k = 0; k < HT; k += 2) {
      const double2 va = *reinterpret_cast<const double2*>(vx + k);
      X[k][s2] = fma(-va.x, w, X[k][s2]);
      X[k + 1][s2] = fma(-va.y, w, X[k + 1][s2]);
    }
    if (32 * s2 + lane > j) Rj[32 * s2 + lane] = r - q;
  }
  if (lane == jj) Rj[j] = beta;
  if (lane == 0 && tau_tile) tau_tile[j] = tau;
  __syncwarp();  // R row j written; every lane is done with x_{j-1} in vnx
  if (lane == 0) {
    __threadfence_block();
    st_release(ver + j, t + 1);
  }
  if (!more) return;
  if (lane == (jn & 31)) {
    mysc[SNc] = nscale;
#pragma unroll
    for (int k = 0; k < HT; k += 2)
      *reinterpret_cast<double2*>(vnx + k) = make_double2(X[k][SNc], X[k + 1][SNc]);
  }
  __syncwarp();
  raw_dots_vs<NP, HT, SNc>(X, vnx, p);
  beta = nbeta;
  tau = ntau;
  scale = nscale;
}

template <int NP, int HT, int s>
__device__ __forceinline__ void ring_slot_vs(double (&X)[HT][NP / 32], double (&p)[NP / 32],
                                             double (&mysc)[NP / 32], double& beta, double& tau,
                                             double& scale, double* Rs, int* ver, double* vb,
                                             int n, int t, double* tau_tile) {
  for (int jj = 0; jj < 31; ++jj) {
    if (32 * s + jj >= n) return;
    ring_step_vs<NP, HT, s, s>(X, p, mysc, beta, tau, scale, Rs, ver, vb, n, t, jj, tau_tile);
  }
  if (32 * s + 31 >= n) return;
  ring_step_vs<NP, HT, s, s + 1>(X, p, mysc, beta, tau, scale, Rs, ver, vb, n, t, 31, tau_tile);
}

// Same contract as ring_factor_tile; vb holds 2*HT doubles for this warp.
template <int NP, int HW>
__device__ __forceinline__ void ring_factor_tile_vs(double (&X)[HW][NP / 32], double* Rs, int* ver,
                                                    double* vb, int n, int t, double* tau_tile) {
  constexpr int S = NP / 32;
  const int lane = threadIdx.x & 31;
  double mysc[S];
#pragma unroll
  for (int s = 0; s < S; ++s) mysc[s] = 1.0;
  double p[S];
  double beta, tau, scale;
  {
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int k = 0; k < HW; k += 2) {
      s0 = fma(X[k][0], X[k][0], s0);
      s1 = fma(X[k + 1][0], X[k + 1][0], s1);
    }
    const double sg = __shfl_sync(FULL, s0 + s1, 0);
    while (ld_acquire(ver) != t) { }
    house_lean(Rs[0], sg, beta, tau, scale);
    __syncwarp();
    if (lane == 0) {
      mysc[0] = scale;
#pragma unroll
      for (int k = 0; k < HW; k += 2)
        *reinterpret_cast<double2*>(vb + k) = make_double2(X[k][0], X[k + 1][0]);
    }
    __syncwarp();
    raw_dots_vs<NP, HW, 0>(X, vb, p);
  }
  ring_slot_vs<NP, HW, 0>(X, p, mysc, beta, tau, scale, Rs, ver, vb, n, t, tau_tile);
  if constexpr (S > 1) ring_slot_vs<NP, HW, 1>(X, p, mysc, beta, tau, scale, Rs, ver, vb, n, t, tau_tile);
  if constexpr (S > 2) ring_slot_vs<NP, HW, 2>(X, p, mysc, beta, tau, scale, Rs, ver, vb, n, t, tau_tile);
  if constexpr (S > 3) ring_slot_vs<NP, HW, 3>(X, p, mysc, beta, tau, scale, Rs, ver, vb, n, t, tau_tile);
#pragma unroll
  for (int s = 0; s < S; ++s)
#pragma unroll
    for (int k = 0; k < HW; ++k) X[k][s] *= mysc[s];
}

// ---------------------------------------------------------------------------
// Ring tile: one warp applies the n reflectors of its triangle-on-rectangle
// tile [R; X] (householder.py:297-332), R rows taken from / returned to Rs
// (stride NP) under the version protocol ver[j] == t.  The broadcast vector
// is the RAW column x (v = scale * x); scale is folded into the coefficients
// and applied to the stored Y at the end, so on return X holds the tile's V
// (the stored rectangle of the factor).
// ---------------------------------------------------------------------------
template <int NP, int HW>
__device__ __forceinline__ void ring_factor_tile(double (&X)[HW][NP / 32], double* Rs, int* ver,
                                                 double* vb, int n, int t, double* tau_tile) {
  constexpr int S = NP / 32;
  const int lane = threadIdx.x & 31;
#ifdef TSQR_SPIN_PROBE
  const long long tstart = clock64();
#endif
  double mysc[S];
#pragma unroll
  for (int s = 0; s < S; ++s) mysc[s] = 1.0;
  double v[HW];
  double p[S];
  double beta, tau, scale;
  {  // prologue: reflector 0
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int k = 0; k < HW; k += 2) {
      s0 = fma(X[k][0], X[k][0], s0);
      s1 = fma(X[k + 1][0], X[k + 1][0], s1);
    }
    const double sg = __shfl_sync(FULL, s0 + s1, 0);
    while (ld_acquire(ver) != t) { }
    house_lean(Rs[0], sg, beta, tau, scale);
    if (lane == 0) {
      mysc[0] = scale;
#pragma unroll
      for (int k = 0; k < HW; k += 2)
        *reinterpret_cast<double2*>(vb + k) = make_double2(X[k][0], X[k + 1][0]);
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < HW; k += 2) {
      const double2 t2 = *reinterpret_cast<const double2*>(vb + k);
      v[k] = t2.x;
      v[k + 1] = t2.y;
    }
    __syncwarp();
    raw_dots<NP, HW, 0>(X, v, p);
  }
  ring_slot<NP, HW, 0>(X, v, p, mysc, beta, tau, scale, Rs, ver, vb, n, t, tau_tile);
  if constexpr (S > 1) ring_slot<NP, HW, 1>(X, v, p, mysc, beta, tau, scale, Rs, ver, vb, n, t, tau_tile);
  if constexpr (S > 2) ring_slot<NP, HW, 2>(X, v, p, mysc, beta, tau, scale, Rs, ver, vb, n, t, tau_tile);
  if constexpr (S > 3) ring_slot<NP, HW, 3>(X, v, p, mysc, beta, tau, scale, Rs, ver, vb, n, t, tau_tile);
#pragma unroll
  for (int s = 0; s < S; ++s)
#pragma unroll
    for (int k = 0; k < HW; ++k) X[k][s] *= mysc[s];
#ifdef TSQR_SPIN_PROBE
  if (lane == 0) atomicAdd(&g_spin_cycles[1], clock64() - tstart);
#endif
}

// ---------------------------------------------------------------------------
// CTA-cooperative application of a DENSE (internal pivot, support r >= j) or
// STACKED (external pivot rows Ps, support r <= j) factor to a block of C
// columns held in registers.  Forward order (Q^T) or reverse (Q).
// Ycol(r, j) gives the stored reflector entry for block row r.
// Lane columns: col0 + 32*s + lane; tri_skip skips slots whose columns are
// all < j (valid when C's columns < j are known to be zero, e.g. forming Q).
// smem part: 2*WARPS*KB (double buffered -> one barrier per reflector).
// ---------------------------------------------------------------------------
template <int RW, int KBS, int MODE, bool TRANS, class YF>
__device__ __forceinline__ void cta_apply(double (&X)[RW][KBS], double* Ps, int n, YF Ycol,
                                          const double* __restrict__ tau, double* part,
                                          int col0, bool tri_skip, double* vs) {
  constexpr int KB = 32 * KBS;
  constexpr int LD = RW + 2;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double* vt = vs + 32 * LD;
  const int nb = (n + 31) / 32;
  for (int bx = 0; bx < nb; ++bx) {
    const int jb = TRANS ? bx : nb - 1 - bx;
    {  // stage this warp's rows of the block's 32 reflector columns, transposed
      const int c = 32 * jb + lane;
      __syncwarp();
#pragma unroll
      for (int k = 0; k < RW; k += 2) {
        const double a0 = (c < n) ? Ycol(w * RW + k, c) : 0.0;
        const double a1 = (c < n) ? Ycol(w * RW + k + 1, c) : 0.0;
        *reinterpret_cast<double2*>(vs + lane * LD + k) = make_double2(a0, a1);
      }
      vt[lane] = (c < n) ? __ldg(tau + c) : 0.0;
      __syncwarp();
    }
    const int jlim = min(32, n - 32 * jb);
    for (int jx = 0; jx < jlim; ++jx) {
      const int jj = TRANS ? jx : jlim - 1 - jx;
      const int j = 32 * jb + jj;
      const int pw = j / RW;
      const bool wact = (MODE == DENSE) ? (w >= pw) : (MODE == STACKED ? (w <= pw) : true);
      double* pb = part + (j & 1) * WARPS * KB;
      const double tj = vt[jj];
      double v[RW];
      double pold[KBS];
      if (wact) {
#pragma unroll
        for (int k = 0; k < RW; k += 2) {
          const double2 t2 = *reinterpret_cast<const double2*>(vs + jj * LD + k);
          v[k] = t2.x;
          v[k + 1] = t2.y;
        }
#pragma unroll
        for (int k = 0; k < RW; ++k) {
          const int r = w * RW + k;
          if (MODE == DENSE) v[k] = (r > j) ? v[k] : (r == j ? 1.0 : 0.0);
          else if (MODE == STACKED) v[k] = (r <= j) ? v[k] : 0.0;
        }
#pragma unroll
        for (int s2 = 0; s2 < KBS; ++s2) {
          if (tri_skip && col0 + 32 * s2 + 31 < j) continue;
          double p0 = 0.0, p1 = 0.0;
#pragma unroll
          for (int k = 0; k < RW; k += 2) {
            p0 = fma(v[k], X[k][s2], p0);
            p1 = fma(v[k + 1], X[k + 1][s2], p1);
          }
          double p = p0 + p1;
          if (MODE != DENSE && w == 0) {
            pold[s2] = Ps[j * KB + 32 * s2 + lane];
            p += pold[s2];
          }
          pb[w * KB + 32 * s2 + lane] = p;
        }
      }
      __syncthreads();
      if (wact && tj != 0.0) {
        const int q0 = (MODE == DENSE) ? pw : 0;
        const int q1 = (MODE == STACKED) ? pw : WARPS - 1;
#pragma unroll
        for (int s2 = 0; s2 < KBS; ++s2) {
          if (tri_skip && col0 + 32 * s2 + 31 < j) continue;
          const int c = 32 * s2 + lane;
          double t0 = 0.0, t1 = 0.0;
          int q = q0;
          for (; q + 1 <= q1; q += 2) {
            t0 += pb[q * KB + c];
            t1 += pb[(q + 1) * KB + c];
          }
          if (q <= q1) t0 += pb[q * KB + c];
          const double wv = tj * (t0 + t1);
#pragma unroll
          for (int k = 0; k < RW; ++k) X[k][s2] = fma(-v[k], wv, X[k][s2]);
          if (MODE != DENSE && w == 0) Ps[j * KB + c] = pold[s2] - wv;
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Ring application of one triangle-on-rectangle tile factor (V: HW x n rows
// at Vt with stride ldv, rows >= vrows treated as zero) to [Cs; X]:
// Cs = pivot rows (stride KB) in smem, X = this warp's tile of C.
// ---------------------------------------------------------------------------
// Shared-memory staging per warp for ring_apply_tile: the tile's V columns of
// one block of 32 reflectors, transposed (row stride HW + 2 doubles: 16-byte
// aligned rows, 2-way conflicts on the transposing stores), plus their tau.
template <int HW>
struct ApplyStage {
  static constexpr int LD = HW + 2;
  static constexpr int DOUBLES = 32 * LD + 32;
};

template <int HW, int KBS, bool TRANS>
__device__ __forceinline__ void ring_apply_tile(double (&X)[HW][KBS], double* Cs, int* ver,
                                                const double* __restrict__ Vt, int64_t ldv,
                                                int vrows, const double* __restrict__ tau,
                                                int n, int order, int col0, bool tri_skip,
                                                double* vs) {
  constexpr int KB = 32 * KBS;
  constexpr int LD = ApplyStage<HW>::LD;
  const int lane = threadIdx.x & 31;
  double* vt = vs + 32 * LD;
  const int nb = (n + 31) / 32;
  for (int bx = 0; bx < nb; ++bx) {
    const int jb = TRANS ? bx : nb - 1 - bx;
    // stage V[:, 32 jb + lane] (coalesced rows) and tau, transposed
    {
      const int c = 32 * jb + lane;
      __syncwarp();
#pragma unroll
      for (int k = 0; k < HW; k += 2) {
        const double a0 = (k < vrows && c < n) ? __ldg(Vt + (int64_t)k * ldv + c) : 0.0;
        const double a1 = (k + 1 < vrows && c < n) ? __ldg(Vt + (int64_t)(k + 1) * ldv + c) : 0.0;
        *reinterpret_cast<double2*>(vs + lane * LD + k) = make_double2(a0, a1);
      }
      vt[lane] = (c < n) ? __ldg(tau + c) : 0.0;
      __syncwarp();
    }
    const int jlim = min(32, n - 32 * jb);
    // one reflector at a time; the pivot rows are acquired two at a time
    // (a spin on even steps only), a zero tau simply gives w = 0, and the
    // hand-off is __syncwarp (orders the lanes' Cs stores) + lane 0 release.
    for (int jx = 0; jx < jlim; ++jx) {
      const int jj = TRANS ? jx : jlim - 1 - jx;
      const int j = 32 * jb + jj;
      const double tj = vt[jj];
      double v[HW];
#pragma unroll
      for (int k = 0; k < HW; k += 2) {
        const double2 t2 = *reinterpret_cast<const double2*>(vs + jj * LD + k);
        v[k] = t2.x;
        v[k + 1] = t2.y;
      }
      if ((jx & 1) == 0) {
        const int jw = (jx + 1 < jlim) ? (TRANS ? j + 1 : j - 1) : j;
        while (ld_acquire(ver + jw) != order) { }
      }
#pragma unroll
      for (int s2 = 0; s2 < KBS; ++s2) {
        if (tri_skip && col0 + 32 * s2 + 31 < j) continue;
        const double cold = Cs[j * KB + 32 * s2 + lane];
        double p0 = cold, p1 = 0.0, p2 = 0.0, p3 = 0.0;
#pragma unroll
        for (int k = 0; k < HW; k += 4) {
          p0 = fma(v[k], X[k][s2], p0);
          p1 = fma(v[k + 1], X[k + 1][s2], p1);
          p2 = fma(v[k + 2], X[k + 2][s2], p2);
          p3 = fma(v[k + 3], X[k + 3][s2], p3);
        }
        const double wv = tj * ((p0 + p1) + (p2 + p3));
        Cs[j * KB + 32 * s2 + lane] = cold - wv;
#pragma unroll
        for (int k = 0; k < HW; ++k) X[k][s2] = fma(-v[k], wv, X[k][s2]);
      }
      __syncwarp();
      if (lane == 0) st_release(ver + j, order + 1);
    }
  }
}

}  // namespace tsqr
