// DMMA warp ring leaf (R only, 64 < n <= 128).
//
// The flat chain of triangle-on-rectangle steps of a leaf (Alg. 2,
// PAPER.md:840-866; one step = qr_triangle_on_rect, householder.py:297-332)
// run as a warp ring like k_leaf_chain -- warp w owns 16-row tiles
// t = w, w+8, ..., the pivot rows R live in shared memory -- but each tile step
// is BLOCKED: 8-column panels are factored Level-2 inside the warp and the
// trailing update of each panel is the compact-WY product (householder.py:
// 175-186 with V = [I; Y])
//
//     W  = R_p,trail + Y^T C          (4 DMMA per 8-column block)
//     W' = T^T W                      (2 DMMA)
//     R_p,trail -= W',  C -= Y W'     (4 DMMA)
//
// on the FP64 tensor cores (mma.m8n8k4.f64).  One DMMA issues 256 FMAs, so the
// issue slots the rank-1 ring spent on DFMA go to the panel reflectors.
//
// Register layout: the tile (16 x 128) is held as 2 x 16 blocks of 8 x 8 in
// the DMMA accumulator layout of C^T: lane (g = lane/4, q = lane%4) holds
// C[8 b + 2 q + e][8 cb + g], e = 0, 1.  With the rows of every k-step
// permuted to {2 q + s}, that same register is the A operand of C^T Y and the
// accumulator of C^T -= W'^T Y^T, so the tile never leaves registers.  The
// panel being factored is always register block 0: after each panel the
// blocks shift down by one.
//
// Pivot rows: R is stored panel-packed in shared memory (panel p = rows
// 8p..8p+7, columns 8p..127, row stride 130 - 8p).  Tile t may factor panel p
// once tile t-1 has (ver1[p] == t) and may update R_p,trail once tile t-1 has
// (ver2[p] == t) -- the ring of k_leaf_chain at panel granularity.
// Included by tsqr_sm100.cu (namespace tsqr).

constexpr int DR_WARPS = 8;
constexpr int DR_H = 16;            // tile rows per warp
constexpr int DR_NP = 128;          // padded width
constexpr int DR_NCB = DR_NP / 8;   // 8-column blocks
constexpr int DR_SLD = DR_NP + 2;   // staging row stride (doubles): conflict-free fragment loads
constexpr int DR_SCR = 336;         // per-warp scratch (V^T staging 16 x 12, G, T, tau)
__host__ __device__ constexpr int dr_ldr(int p) { return DR_NP - 8 * p + 2; }
__host__ __device__ constexpr int dr_pbase(int p) { return 8 * (p * (DR_NP + 2) - 4 * p * (p - 1)); }
struct DmmaRingSmem {
  static constexpr int RP = dr_pbase(DR_NCB);
  static constexpr size_t doubles = (size_t)RP + DR_WARPS * DR_H * DR_SLD + DR_WARPS * DR_SCR;
  static constexpr size_t bytes = sizeof(double) * doubles + sizeof(int) * 2 * DR_NCB;
};

// Stage tile rows [row0, row0 + valid) of A into the warp's staging buffer
// (cp.async, zero fill below `valid`); V16: 16-byte granules (n, lda even).
template <bool V16>
__device__ __forceinline__ void dr_issue(double* stage, const double* __restrict__ A, int64_t lda,
                                         int64_t row0, int valid, int n) {
  const int lane = threadIdx.x & 31;
  const unsigned sb = (unsigned)__cvta_generic_to_shared(stage);
  if constexpr (V16) {
    const int cpr = n >> 1;
#pragma unroll 4
    for (int idx = lane; idx < DR_H * 64; idx += 32) {
      const int r = idx >> 6, c2 = idx & 63;
      if (c2 < cpr) {
        const bool ok = r < valid;
        const double* src = ok ? A + (row0 + r) * lda + 2 * c2 : A;
        cp_async<16>(sb + 8u * (unsigned)(r * DR_SLD + 2 * c2), src, ok ? 16u : 0u);
      }
    }
  } else {
#pragma unroll 4
    for (int idx = lane; idx < DR_H * DR_NP; idx += 32) {
      const int r = idx >> 7, c = idx & 127;
      if (c < n) {
        const bool ok = r < valid;
        const double* src = ok ? A + (row0 + r) * lda + c : A;
        cp_async<8>(sb + 8u * (unsigned)(r * DR_SLD + c), src, ok ? 8u : 0u);
      }
    }
  }
  cp_async_commit();
}

// Level-2 factorisation of the panel held in x[4] (= C[b][0][e]: rows
// 8b + 2q + e, column pc + g) against the pivot rows Rpan (row stride ldr).
// On return x holds the panel's Y (tile part of V), Rpan the updated R_pp,
// gs[s][i] = Y_s^T Y_i (s < i) and taus[i] = tau_i.  Every lane evaluates the
// reflector scalars (house_gen, householder.py:97-113) redundantly from the
// broadcast column, so only two 4-lane reductions sit on the critical path.
__device__ __forceinline__ void dr_panel(double (&x)[4], double* Rpan, int ldr, double* gs,
                                         double* taus) {
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, q = lane & 3;
#ifdef DR_ROLLED
#pragma unroll 1
#else
#pragma unroll
#endif
  for (int i = 0; i < 8; ++i) {
    const int src = 4 * i + q;
    double xi[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) xi[k] = __shfl_sync(FULL, x[k], src);
    const double rgi = Rpan[i * ldr + g];  // row i of R_pp changes only at reflector i
    const double x0 = __shfl_sync(FULL, rgi, 4 * i);
    double s = xi[0] * xi[0], s2 = xi[2] * xi[2];
    s = fma(xi[1], xi[1], s);
    s2 = fma(xi[3], xi[3], s2);
    double pd = xi[0] * x[0], pd2 = xi[2] * x[2];
    pd = fma(xi[1], x[1], pd);
    pd2 = fma(xi[3], x[3], pd2);
    s += s2;
    pd += pd2;
    s += __shfl_xor_sync(FULL, s, 1);
    pd += __shfl_xor_sync(FULL, pd, 1);
    s += __shfl_xor_sync(FULL, s, 2);
    pd += __shfl_xor_sync(FULL, pd, 2);
    double beta, tau, scale;
    house_lean(x0, s, beta, tau, scale);
    const double wv = tau * fma(scale, pd, rgi);
    const bool upd = g > i;
    const double f = upd ? -scale * wv : 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) x[k] = (g == i) ? xi[k] * scale : fma(f, xi[k], x[k]);
    if (q == 0) {
      if (upd) Rpan[i * ldr + g] = rgi - wv;
      else if (g == i) Rpan[i * ldr + i] = beta;
      else gs[g * 8 + i] = scale * pd;
    }
    if (lane == 0) taus[i] = tau;
  }
}

// T of the panel (dlarft forward/columnwise, householder.py:148-164, with
// V^T V = I + G): lane l < 8 runs the recurrence for row l of T.
__device__ __forceinline__ void dr_form_t(const double* gs, const double* taus, double* ts) {
  const int lane = threadIdx.x & 31;
  if (lane < 8) {
    const int l = lane;
    double Tl[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) Tl[c] = (c == l) ? taus[l] : 0.0;
#pragma unroll
    for (int i = 1; i < 8; ++i) {
      double z = 0.0;
#pragma unroll
      for (int s = 0; s < i; ++s) z = fma(Tl[s], gs[s * 8 + i], z);  // Tl[s] = 0 for s < l
      if (l < i) Tl[i] = -taus[i] * z;
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) ts[l * 8 + c] = Tl[c];
  }
}

#ifdef DR_PROBE
__device__ unsigned long long g_dr_cycles[8];
#define DR_TICK(v) const long long v = clock64()
#define DR_ADD(i, a, b) \
  if (lane == 0 && blockIdx.x == 0) atomicAdd(&g_dr_cycles[i], (unsigned long long)((b) - (a)))
#else
#define DR_TICK(v)
#define DR_ADD(i, a, b)
#endif

// Ring wait, warp-uniform: lane 0 polls and broadcasts, so the warp never
// diverges around the spin (a diverged warp runs every later shuffle through
// the slow collective path).
#ifndef DR_SLEEP
#define DR_SLEEP 0
#endif
__device__ __forceinline__ void dr_wait(const int* ver, int target, int lane) {
  for (;;) {
    int v = 0;
    if (lane == 0) v = ld_acquire(ver);
    v = __shfl_sync(FULL, v, 0);
    if (v == target) break;
    if (DR_SLEEP) __nanosleep(DR_SLEEP);
  }
  __threadfence_block();
}

template <bool V16>
__global__ void __launch_bounds__(DR_WARPS * 32, 1)
k_leaf_dmma(const double* __restrict__ A, int64_t lda, int64_t m, int n, int P, int64_t base,
            double* Rio, int* flag) {
  extern __shared__ __align__(16) double sm[];
  double* Rp = sm;
  double* stage_all = Rp + DmmaRingSmem::RP;
  double* scr_all = stage_all + DR_WARPS * DR_H * DR_SLD;
  int* ver = reinterpret_cast<int*>(scr_all + DR_WARPS * DR_SCR);  // ver1[16], ver2[16]
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, q = lane & 3;
  const int leaf = blockIdx.x;
  const int64_t r0 = (int64_t)leaf * base;
  const int64_t b = (leaf == P - 1) ? m - r0 : base;
  const int T = (int)((b + DR_H - 1) / DR_H);
  const int npan = (n + 7) >> 3;
  for (int i = threadIdx.x; i < DmmaRingSmem::RP; i += DR_WARPS * 32) Rp[i] = 0.0;
  if (threadIdx.x < 2 * DR_NCB) ver[threadIdx.x] = 0;
  __syncthreads();
  double* stage = stage_all + w * DR_H * DR_SLD;
  double* vs = scr_all + w * DR_SCR;  // 16 x 12
  double* gs = vs + 192;
  double* ts = gs + 64;
  double* taus = ts + 64;
  bool bad = false;
  if (w < T) {
    const int64_t row = r0 + (int64_t)w * DR_H;
    dr_issue<V16>(stage, A, lda, row, (int)min64(DR_H, r0 + b - row), n);
  }
  DR_TICK(k0_);
  for (int t = w; t < T; t += DR_WARPS) {
    cp_async_wait<0>();
    __syncwarp();
    double C[2][DR_NCB][2];
#pragma unroll
    for (int bb = 0; bb < 2; ++bb)
#pragma unroll
      for (int cb = 0; cb < DR_NCB; ++cb)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = 8 * cb + g;
          double v = stage[(8 * bb + 2 * q + e) * DR_SLD + c];
          v = (c < n) ? v : 0.0;
          bad |= !isfinite(v);
          C[bb][cb][e] = v;
        }
    __syncwarp();
    if (t + DR_WARPS < T) {
      const int64_t row = r0 + (int64_t)(t + DR_WARPS) * DR_H;
      dr_issue<V16>(stage, A, lda, row, (int)min64(DR_H, r0 + b - row), n);
    }
    for (int p = 0; p < npan; ++p) {
      const int ldr = dr_ldr(p);
      double* Rpan = Rp + dr_pbase(p);
      // ---- panel p: Level-2 against R_pp ----
      DR_TICK(c0_);
      dr_wait(ver + p, t, lane);
      DR_TICK(c1_);
      double x[4] = {C[0][0][0], C[0][0][1], C[1][0][0], C[1][0][1]};
      dr_panel(x, Rpan, ldr, gs, taus);
      ring_signal(ver + p, t + 1, lane);
      DR_TICK(c2_);
      DR_ADD(0, c0_, c1_);
      DR_ADD(1, c1_, c2_);
      const int nlive = npan - p;  // register blocks 0 .. nlive-1 are live
      if (nlive <= 1) dr_wait(ver + DR_NCB + p, t, lane);  // keep the versions monotone
      else {
        // V^T in the B layout of C^T -= W'^T Y^T: vb[b][s] = Y[8b + g][2q + s]
#pragma unroll
        for (int k = 0; k < 4; ++k) vs[(8 * (k >> 1) + 2 * q + (k & 1)) * 12 + g] = x[k];
        __syncwarp();
        dr_form_t(gs, taus, ts);
        double vb[2][2];
#pragma unroll
        for (int bb = 0; bb < 2; ++bb)
#pragma unroll
          for (int s = 0; s < 2; ++s) vb[bb][s] = vs[(8 * bb + g) * 12 + 2 * q + s];
        __syncwarp();
        const double tb0 = ts[(2 * q) * 8 + g], tb1 = ts[(2 * q + 1) * 8 + g];
        DR_TICK(c3_);
        DR_ADD(2, c2_, c3_);
        // ---- trailing update of panel p ----
        dr_wait(ver + DR_NCB + p, t, lane);
        DR_TICK(c4_);
        DR_ADD(3, c3_, c4_);
        double* rrow = Rpan + (2 * q) * ldr + g;
#pragma unroll
        for (int cb = 1; cb < DR_NCB; ++cb) {
#ifdef DR_NO_UPDATE
          if (cb < 0) {
#else
          if (cb < nlive) {
#endif
            double* rp0 = rrow + 8 * cb;
            const double ro0 = rp0[0], ro1 = rp0[ldr];
            double wa0 = ro0, wa1 = ro1, wb0 = 0.0, wb1 = 0.0;
            dmma(wa0, wa1, C[0][cb][0], x[0]);
            dmma(wb0, wb1, C[1][cb][0], x[2]);
            dmma(wa0, wa1, C[0][cb][1], x[1]);
            dmma(wb0, wb1, C[1][cb][1], x[3]);
            wa0 += wb0;
            wa1 += wb1;
            double u0 = 0.0, u1 = 0.0;
            dmma(u0, u1, wa0, tb0);
            dmma(u0, u1, wa1, tb1);
            rp0[0] = ro0 - u0;
            rp0[ldr] = ro1 - u1;
            dmma(C[0][cb][0], C[0][cb][1], -u0, vb[0][0]);
            dmma(C[1][cb][0], C[1][cb][1], -u0, vb[1][0]);
            dmma(C[0][cb][0], C[0][cb][1], -u1, vb[0][1]);
            dmma(C[1][cb][0], C[1][cb][1], -u1, vb[1][1]);
          }
        }
        DR_TICK(c5_);
        DR_ADD(4, c4_, c5_);
      }
      ring_signal(ver + DR_NCB + p, t + 1, lane);
      // shift the register blocks: the next panel becomes block 0
#pragma unroll
      for (int cb = 0; cb + 1 < DR_NCB; ++cb)
#pragma unroll
        for (int bb = 0; bb < 2; ++bb) {
          C[bb][cb][0] = C[bb][cb + 1][0];
          C[bb][cb][1] = C[bb][cb + 1][1];
        }
    }
  }
  DR_TICK(k1_);
  DR_ADD(5, k0_, k1_);
  __syncthreads();
  double* Rl = Rio + (int64_t)leaf * n * n;
  for (int idx = threadIdx.x; idx < n * n; idx += DR_WARPS * 32) {
    const int r = idx / n, c = idx - r * n;
    const int p = r >> 3;
    Rl[idx] = (c >= r) ? Rp[dr_pbase(p) + (r & 7) * dr_ldr(p) + (c - 8 * p)] : 0.0;
  }
  if (bad && flag) atomicOr(flag, 1);
}
