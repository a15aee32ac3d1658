// Split-role ring with TALL tiles in tensor memory (k_leaf_tt<H>, H = 32 or 64
// rows per tile): the C3 R-only leaf (64 < n <= 128).
//
// k_leaf_tm (tm_leaf.cuh) keeps 16 tiles of 16 rows in TMEM; its phase probe
// shows the shared FP64 pipe saturated during the generation phases with only
// half of the issued work useful: per 16-row tile the 128 reflector
// generations (~30 FP64 warp instructions each), the 16 T formations and the
// 120 T^T W products cost as much as the 1024 useful DMMAs.  All three are per
// TILE, not per row, so this kernel folds H = 32 / 64 rows per step of the
// flat chain (Alg. 2; one step = qr_triangle_on_rect,
// householder.py:297-332, with an H x n rectangle): the same 256 rows in TMEM
// (8 / 4 slots), a half / a quarter of the per-row overhead:
//
//   pipe work per row (DMMA = 16 sub-partition cycles)   H = 16    32    64
//     useful compact-WY DMMAs                               64    64    64
//     T^T W, T formation, reflector scalars                 64    33    20
//
// Layout: block b (columns 8b..8b+7) of the tile in slot s is K = H/4 doubles
// per lane, lane (g, q) holding rows 8i + 2q + e of column 8b + g (the DMMA
// accumulator layout of C^T, i = 0..H/8-1), = H/2 TMEM columns of the 32 lanes
// of sub-partition s % 4.  Within a generation the owner column goes to the
// other lanes through shared memory (K/2 STS.128 + K/2 LDS.128 per lane)
// instead of 2K SHFL: the shuffle unit (one warp instruction per 4 cycles per
// sub-partition) was the larger part of a tall generation (tools/gw_probe.cu).
//
//   G = 256/H generation warps (warp s = slot s): the reflector chain of the
//     slot's tile, Y_p / T_p, and the update of the next panel's block;
//   G update warps (warp G + s, same sub-partition): the slot's other trailing
//     blocks, and the staging of the slot's NEXT tile: block b goes global ->
//     shared (cp.async, issued a panel ahead) -> the TMEM columns of block b as
//     soon as the generation warp has taken the current tile's block b (its
//     ver_p1 signal), so the chain warp never touches global memory after its
//     first tile.  (Two update warps per slot measured slower: 13.6 vs 14.3
//     TF/s; a generation warp's FP64 instructions wait for every DMMA on its
//     sub-partition.)
//
// Counters and TMEM hand-offs as in k_leaf_tm.  The arithmetic is that of
// k_leaf_dmma with taller rectangles (same reflectors up to summation order),
// so R agrees with the 16-row kernels to rounding, not bitwise.
// Included by tsqr_sm100.cu (namespace tsqr), after tm_leaf.cuh.

template <int H, int UWN = 1>
struct TtCfg {
  static constexpr int G = 256 / H;             // generation warps = tiles in flight
  static constexpr int UW = UWN;                // update warps per slot
  static constexpr int U = G * UW;
  static constexpr int THREADS = (G + U) * 32;
  static constexpr int K = H / 4;               // doubles per lane per block
  static constexpr int NB = H / 8;              // 8-row blocks
};
template <int H>
struct TtSmem {  // offsets in doubles, then ints
  static constexpr int G = TtCfg<H>::G;
  static constexpr int R = 0;
  static constexpr int YN = R + dr_pbase<128>(16);  // [slot][2 parities][H x 8] Y_p, natural
  static constexpr int YF = YN + G * 2 * H * 8;     // [slot][2 parities][K][32] Y_p, fragment order
  static constexpr int TB = YF + G * 2 * H * 8;     // [slot][2 parities][32][2] T
  static constexpr int GS = TB + G * 2 * 64;        // [slot][72] G, tau
  static constexpr int XS = GS + G * 72;            // [slot][2][H] owner column of a generation
  static constexpr int STG = XS + G * 2 * H;        // [slot][H x 8] next tile's block p
  static constexpr int doubles = STG + G * H * 8;
  static constexpr int NCNT = 4 * 16 + 3 * G + 4;
  static constexpr size_t bytes = sizeof(double) * doubles + sizeof(int) * NCNT;
};

__device__ __forceinline__ void tt_ld16_issue(uint32_t* r, uint32_t taddr) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
      "%13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tt_st16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
      "%13, %14, %15, %16};"
      :: "r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]),
         "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
         "r"(r[15])
      : "memory");
}
// one block (K doubles per lane) TMEM -> registers; issue and completion split so
// two blocks can be in flight
template <int K>
__device__ __forceinline__ void tt_ld_issue(uint32_t (&r)[2 * K], uint32_t taddr) {
#pragma unroll
  for (int c = 0; c < K / 8; ++c) tt_ld16_issue(r + 16 * c, taddr + 16 * c);
}
template <int K>
__device__ __forceinline__ void tt_unpack(double (&x)[K], const uint32_t (&r)[2 * K]) {
#pragma unroll
  for (int k = 0; k < K; ++k) x[k] = __hiloint2double((int)r[2 * k + 1], (int)r[2 * k]);
}
template <int K>
__device__ __forceinline__ void tt_ld(double (&x)[K], uint32_t taddr) {
  uint32_t r[2 * K];
  tt_ld_issue<K>(r, taddr);
  tm_ld_wait();
  tt_unpack<K>(x, r);
}
template <int K>
__device__ __forceinline__ void tt_st(uint32_t taddr, const double (&x)[K]) {
  uint32_t r[2 * K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    r[2 * k] = (uint32_t)__double2loint(x[k]);
    r[2 * k + 1] = (uint32_t)__double2hiint(x[k]);
  }
#pragma unroll
  for (int c = 0; c < K / 8; ++c) tt_st16(taddr + 16 * c, r + 16 * c);
}

// One generation (reflector I of the panel) on an H x 8 block: dr_gen's
// arithmetic (the one-FMA R-only form) with K elements per lane; the owner
// column x_I reaches the other column groups through xs (the caller alternates
// two buffers: the warp barrier of generation I+1 separates the reads of
// generation I from the writes of generation I+2).
template <int I, int K, bool EXACT>
__device__ __forceinline__ void tt_gen(double (&x)[K], double* Rrow, double* gs, double* taus,
                                       double* xs) {
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, q = lane & 3;
  double2* buf = reinterpret_cast<double2*>(xs) + q;
  if (g == I) {
#pragma unroll
    for (int k2 = 0; k2 < K / 2; ++k2) buf[4 * k2] = make_double2(x[2 * k2], x[2 * k2 + 1]);
  }
  const double x0 = Rrow[I];   // R[pc+I][pc+I]: read before the barrier, rewritten (beta) after it
  const double rgi = Rrow[g];  // R[pc+I][pc+g]
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
#pragma unroll
  for (int k = 4; k < K; ++k) a[k & 3] = fma(xi[k], x[k], a[k & 3]);
  double pd = (a[0] + a[1]) + (a[2] + a[3]);
  pd = dr_quad_sum(pd);
  const double s = __shfl_sync(FULL, pd, 4 * I);
  double beta, tau, scale, invb;
  house_fast(x0, s, beta, tau, scale, invb);
  const double tw = fma(scale, pd, rgi);  // R[I][g] + v^T x_g
  const double wv = tau * tw;
  const bool upd = g > I, own = (g == I);
  // kept factors (EXACT): the owner column becomes v = fma(scale, x_I, 0), one rounding (dr_gen)
  const double f = upd ? tw * invb : (own ? (EXACT ? scale : scale - 1.0) : 0.0);
#pragma unroll
  for (int k = 0; k < K; ++k) x[k] = fma(f, xi[k], (EXACT && own) ? 0.0 : x[k]);
  double* dst = upd ? Rrow + g : (own ? Rrow + I : gs + g * 8 + I);
  *dst = upd ? rgi - wv : (own ? beta : scale * pd);
  taus[I] = tau;
}

// Compact-WY update of NBLK 8-column blocks (c[j]) by the panel, DMMAs of the
// blocks interleaved (independent accumulation chains side by side); NBLK = 1
// splits the Y^T C accumulation in four chains instead.  y = Y_p (fragment
// order, the B operand of C^T Y), vb[i][s] = Y[8i + g][2q + s] (the B operand
// of W'^T Y^T), tb = T; rp[j] = the block's pivot rows R_p,blk (row stride ldr).
template <int K, int NBLK>
__device__ __forceinline__ void tt_upd(double (&c)[NBLK][K], const double (&y)[K],
                                       const double (&vb)[K / 2][2], double tb0, double tb1,
                                       double* const (&rp)[NBLK], int ldr) {
#ifdef TT_NOUPD
  if (threadIdx.x >= 32 * TT_NOUPD) return;  // probe only: update warps skip the DMMAs (wrong R)
#endif
  double ro0[NBLK], ro1[NBLK], w0[NBLK], w1[NBLK];
#pragma unroll
  for (int j = 0; j < NBLK; ++j) {
    ro0[j] = rp[j][0];
    ro1[j] = rp[j][ldr];
    w0[j] = ro0[j];
    w1[j] = ro1[j];
  }
  if constexpr (NBLK == 1) {
    double v0 = 0.0, v1 = 0.0, s0 = 0.0, s1 = 0.0, t0 = 0.0, t1 = 0.0;
#pragma unroll
    for (int k = 0; k < K; k += 4) {
      dmma(w0[0], w1[0], c[0][k], y[k]);
      dmma(v0, v1, c[0][k + 1], y[k + 1]);
      dmma(s0, s1, c[0][k + 2], y[k + 2]);
      dmma(t0, t1, c[0][k + 3], y[k + 3]);
    }
    w0[0] = (w0[0] + v0) + (s0 + t0);
    w1[0] = (w1[0] + v1) + (s1 + t1);
  } else {
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
      for (int j = 0; j < NBLK; ++j) dmma(w0[j], w1[j], c[j][k], y[k]);
  }
  double u0[NBLK], u1[NBLK];
#pragma unroll
  for (int j = 0; j < NBLK; ++j) u0[j] = u1[j] = 0.0;
#pragma unroll
  for (int j = 0; j < NBLK; ++j) dmma(u0[j], u1[j], w0[j], tb0);
#pragma unroll
  for (int j = 0; j < NBLK; ++j) dmma(u0[j], u1[j], w1[j], tb1);
#pragma unroll
  for (int j = 0; j < NBLK; ++j) {
    rp[j][0] = ro0[j] - u0[j];
    rp[j][ldr] = ro1[j] - u1[j];
    u0[j] = -u0[j];
    u1[j] = -u1[j];
  }
#pragma unroll
  for (int i = 0; i < K / 2; ++i)
#pragma unroll
    for (int j = 0; j < NBLK; ++j) dmma(c[j][2 * i], c[j][2 * i + 1], u0[j], vb[i][0]);
#pragma unroll
  for (int i = 0; i < K / 2; ++i)
#pragma unroll
    for (int j = 0; j < NBLK; ++j) dmma(c[j][2 * i], c[j][2 * i + 1], u1[j], vb[i][1]);
}


// Q = false: R only, the chain starts from R = 0 at the leaf's first row (h0 = 0).
// Q = true: the chain continues from the leaf's R slot after a dense first tile of h0 rows
// (k_leaf_dense) and keeps every tile's TRI_ON_RECT factor: Y rows h0 + H t.., tau at
// (t + 1) * n, the layout of k_leaf_dmma with H-row tiles.  Y may alias A (a tile's rows
// are on chip before its first panel is stored).
template <int H, int UWN, bool Q>
__global__ void __launch_bounds__(TtCfg<H, UWN>::THREADS, 1)
k_leaf_tt(const double* __restrict__ A, int64_t lda, int64_t m, int n, int P, int64_t base,
          double* Rio, int* flag, double* Y, int64_t ldy, double* tau, int64_t tau_stride, int h0) {
  using Cfg = TtCfg<H, UWN>;
  using Sm = TtSmem<H>;
  constexpr int G = Cfg::G, K = Cfg::K, UW = Cfg::UW, THREADS = Cfg::THREADS;
  // (two update warps per slot ran correctly until the next tile's staging moved to the update
  // warp; with it the UW = 2 build returned a wrong R in tools/tt_probe.cu and was dropped)
  static_assert(UW == 1, "one update warp per slot");
  extern __shared__ __align__(16) double sm[];
  double* Rp = sm + Sm::R;
  int* cnt = reinterpret_cast<int*>(sm + Sm::doubles);
  int* ver_pp = cnt;
  int* ver_p1 = cnt + 16;
  int* ver_u = cnt + 32;  // [UW][16]
  int* yrdy = cnt + 64;
  int* ufirst = yrdy + G;
  int* staged = ufirst + G;  // slot s: tiles staged for the generation warp by the update warp
  uint32_t* tbase_s = reinterpret_cast<uint32_t*>(staged + G);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, q = lane & 3;
  const int leaf = blockIdx.x;
  const int64_t bl = (leaf == P - 1) ? m - (int64_t)leaf * base : base;
  if (bl - h0 <= 0) return;  // the dense tile was the whole leaf: R is already in its slot
  const int64_t r0 = (int64_t)leaf * base + h0, b = bl - h0;  // the chain's rows
  const int T = (int)((b + H - 1) / H);
  const int npan = (n + 7) >> 3;
  double* Rl0 = Rio + (int64_t)leaf * n * n;
  for (int i = threadIdx.x; i < Sm::YN; i += THREADS) {
    double v = 0.0;
    if (Q) {  // panel-packed index -> (r, c)
      int pp = 0;
      while (pp + 1 < 16 && dr_pbase<128>(pp + 1) <= i) ++pp;
      const int off = i - dr_pbase<128>(pp), ld = dr_ldr<128>(pp);
      const int r = 8 * pp + off / ld, c = 8 * pp + off % ld;
      if (r < n && c < n && c >= r) v = Rl0[r * n + c];
    }
    Rp[i] = v;
  }
  double* tl = Q ? tau + (int64_t)leaf * tau_stride : nullptr;
  for (int i = threadIdx.x; i < 4 * 16 + 3 * G; i += THREADS) cnt[i] = 0;
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;"
                 :: "r"((unsigned)__cvta_generic_to_shared(tbase_s)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tm_fence_before();
  __syncthreads();
  tm_fence_after();
  const uint32_t tbase = *tbase_s;
  auto taddr = [&](int s, int blk) -> uint32_t {
    return tbase + ((uint32_t)(32 * (s & 3)) << 16) + (uint32_t)((s >> 2) * (8 * H) + (H / 2) * blk);
  };
  // row of element k of lane (., q)
  auto erow = [&](int k) -> int { return 8 * (k >> 1) + 2 * q + (k & 1); };
  if (w < G) {
    // ============================ generation warp ============================
    const int s = w;
    double* gs = sm + Sm::GS + s * 72;
    double* taus = gs + 64;
    double* xs = sm + Sm::XS + s * 2 * H;
    double2* tbs = reinterpret_cast<double2*>(sm + Sm::TB + s * 128);
    auto prefetch = [&](int t) {
      if (t >= T) return;
      const int64_t row = r0 + (int64_t)t * H;
      const int rows = (int)min64(H, r0 + b - row);
      const int lpr = (n * 8 + 127) / 128;
      for (int i = lane; i < rows * lpr; i += 32) {
        const double* a = A + (row + i / lpr) * lda + (i % lpr) * 16;
        asm volatile("prefetch.global.L2 [%0];" :: "l"(a));
      }
    };
    prefetch(s);
    int lt = 0;
    SP_TICK(k0_);
    for (int t = s; t < T; t += G, ++lt) {
      SP_TICK(l0_);
      // tile t: block 0 into registers, blocks 1.. in the slot's TMEM columns.  The
      // slot's first tile is loaded here; every later tile was staged block by
      // block during the previous tile by the slot's update warp (block b once
      // this warp had taken it), off this warp's chain.
      const int64_t row0 = r0 + (int64_t)t * H;
      double x[K];
      if (lt > 0) {
        sp_wait_ge(staged + s, lt, lane);
        tm_fence_after();
        tt_ld<K>(x, taddr(s, 0));
      }
#pragma unroll 1
      for (int blk = 0; blk < (lt > 0 ? 0 : 16); ++blk) {
        double v[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const int64_t row = row0 + erow(k);
          const int col = 8 * blk + g;
          v[k] = (row < r0 + b && col < n) ? __ldg(A + row * lda + col) : 0.0;
        }
        if (blk == 0) {
#pragma unroll
          for (int k = 0; k < K; ++k) x[k] = v[k];
        } else {
          tt_st<K>(taddr(s, blk), v);
        }
      }
      tm_st_wait();
      tm_fence_before();  // published by the first yrdy release below
      prefetch(t + G);
      SP_TICK(l1_);
      SP_ADD(6, l0_, l1_);
      for (int p = 0; p < npan; ++p) {
        const int job = lt * 16 + p;
        const int ldr = dr_ldr<128>(p);
        double* Rpan = Rp + dr_pbase<128>(p);
        SP_TICK(a0_);
        dr_wait(ver_pp + p, t, lane);
        SP_TICK(a1_);
        SP_ADD(0, a0_, a1_);
        tt_gen<0, K, Q>(x, Rpan, gs, taus, xs);
        tt_gen<1, K, Q>(x, Rpan + ldr, gs, taus, xs + H);
        tt_gen<2, K, Q>(x, Rpan + 2 * ldr, gs, taus, xs);
        tt_gen<3, K, Q>(x, Rpan + 3 * ldr, gs, taus, xs + H);
        tt_gen<4, K, Q>(x, Rpan + 4 * ldr, gs, taus, xs);
        tt_gen<5, K, Q>(x, Rpan + 5 * ldr, gs, taus, xs + H);
        tt_gen<6, K, Q>(x, Rpan + 6 * ldr, gs, taus, xs);
        tt_gen<7, K, Q>(x, Rpan + 7 * ldr, gs, taus, xs + H);
        SP_TICK(g1_);
        SP_ADD(11, a1_, g1_);
        dr_signal(ver_pp + p, t + 1, lane);
        if (Q) {  // the tile's factor for panel p: Y (= x) and tau
          const int c = 8 * p + g;
#pragma unroll
          for (int k = 0; k < K; ++k) {
            const int64_t row = row0 + erow(k);
            if (row < r0 + b && c < n) Y[row * ldy + c] = x[k];
          }
          if (lane < 8 && 8 * p + lane < n) tl[(int64_t)(t + 1) * n + 8 * p + lane] = taus[lane];
        }
        if (p + 1 >= npan) break;
        SP_TICK(a2_);
        // publish Y_p (natural layout: the B operand of Y^T; fragment order: the B
        // operand of C^T Y for the update warps) and T_p
        double* yn = sm + Sm::YN + (s * 2 + (p & 1)) * H * 8;
        double* yf = sm + Sm::YF + (s * 2 + (p & 1)) * H * 8;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          yn[erow(k) * 8 + g] = x[k];
          yf[k * 32 + lane] = x[k];
        }
        __syncwarp();
        double vb[K / 2][2], tb0, tb1;
#pragma unroll
        for (int i = 0; i < K / 2; ++i) {
          const double2 t2 = *reinterpret_cast<const double2*>(yn + (8 * i + g) * 8 + 2 * q);
          vb[i][0] = t2.x;
          vb[i][1] = t2.y;
        }
        dr_form_t(gs, taus, tb0, tb1);
        tbs[(p & 1) * 32 + lane] = make_double2(tb0, tb1);
        dr_signal(yrdy + s, job + 1, lane);
        SP_TICK(a3_);
        SP_ADD(2, a2_, a3_);
        SP_TICK(a7_);
        SP_ADD(1, a3_, a7_);
        // hand-off: block p+1 (panel p-1 applied by an update warp), panel p here
        if (p >= 1) sp_wait_ge(ufirst + s, job, lane);
        SP_TICK(a4_);
        SP_ADD(3, a7_, a4_);
        tm_fence_after();
        double c1[1][K];
        tt_ld<K>(c1[0], taddr(s, p + 1));
        dr_wait(ver_p1 + p, t, lane);
        SP_TICK(a5_);
        SP_ADD(4, a4_, a5_);
        double* const rp1[1] = {Rpan + 2 * q * ldr + 8 + g};
        tt_upd<K, 1>(c1, x, vb, tb0, tb1, rp1, ldr);
        tm_fence_before();
        dr_signal(ver_p1 + p, t + 1, lane);  // also: block p+1 is in registers, its TMEM columns free
        SP_TICK(a6_);
        SP_ADD(5, a5_, a6_);
#pragma unroll
        for (int k = 0; k < K; ++k) x[k] = c1[0][k];
      }
    }
    SP_TICK(k1_);
    SP_ADD(7, k0_, k1_);
  } else {
    // ============================== update warp ==============================
    const int u = w - G;
    const int s = u % G, hf = u / G;  // slot (same sub-partition: G % 4 == 0), block parity
    int* vu = ver_u + hf * 16;
    const double2* tbs = reinterpret_cast<const double2*>(sm + Sm::TB + s * 128);
    double* stg = sm + Sm::STG + s * H * 8;
    const bool v16 = ((lda & 1) == 0) && ((n & 1) == 0) && (((uintptr_t)A & 15) == 0);
    int lt = 0;
    for (int t = s; t < T; t += G, ++lt) {
      const bool more = hf == 0 && t + G < T;  // this warp stages the slot's next tile
      const int64_t nrow0 = r0 + (int64_t)(t + G) * H;
      const int nvalid = more ? (int)min64(H, r0 + b - nrow0) : 0;
      // next tile's block bk: global -> shared stage (issued a job ahead, lands under the
      // updates) -> the block's TMEM columns once the generation warp has taken the old block
      auto stage_issue = [&](int bk) {
        const unsigned sb = (unsigned)__cvta_generic_to_shared(stg);
        if (v16) {
#pragma unroll
          for (int i = 0; i < H / 8; ++i) {
            const int x2 = lane + 32 * i, r = x2 >> 2, c2 = x2 & 3;
            const bool ok = r < nvalid && 8 * bk + 2 * c2 < n;
            cp_async<16>(sb + 8u * (unsigned)(r * 8 + 2 * c2),
                         ok ? A + (nrow0 + r) * lda + 8 * bk + 2 * c2 : A, ok ? 16u : 0u);
          }
        } else {
#pragma unroll
          for (int i = 0; i < H / 4; ++i) {
            const int x1 = lane + 32 * i, r = x1 >> 3, c = x1 & 7;
            const bool ok = r < nvalid && 8 * bk + c < n;
            cp_async<8>(sb + 8u * (unsigned)(r * 8 + c), ok ? A + (nrow0 + r) * lda + 8 * bk + c : A,
                        ok ? 8u : 0u);
          }
        }
        cp_async_commit();
      };
      auto stage_move = [&](int bk) {
        cp_async_wait<0>();
        __syncwarp();
        double v[K];
#pragma unroll
        for (int k = 0; k < K; ++k) v[k] = stg[erow(k) * 8 + g];
        __syncwarp();
        tt_st<K>(taddr(s, bk), v);
      };
      double keep[1][K];  // block p+2 between jobs p-1 and p
      for (int p = 0; p + 1 < npan; ++p) {
        const int job = lt * 16 + p;
        const int ldr = dr_ldr<128>(p);
        double* Rpan = Rp + dr_pbase<128>(p);
        SP_TICK(u0_);
        sp_wait_ge(yrdy + s, job + 1, lane);
        tm_fence_after();
        SP_TICK(u1_);
        SP_ADD(8, u0_, u1_);
        double y[K], vb[K / 2][2], tb0 = 0.0, tb1 = 0.0;
        if (p + 2 < npan) {
        const double* yn = sm + Sm::YN + (s * 2 + (p & 1)) * H * 8;
        const double* yf = sm + Sm::YF + (s * 2 + (p & 1)) * H * 8;
#pragma unroll
        for (int k = 0; k < K; ++k) y[k] = yf[k * 32 + lane];
#pragma unroll
        for (int i = 0; i < K / 2; ++i) {
          const double2 t2 = *reinterpret_cast<const double2*>(yn + (8 * i + g) * 8 + 2 * q);
          vb[i][0] = t2.x;
          vb[i][1] = t2.y;
        }
        const double2 tb = tbs[(p & 1) * 32 + lane];
        tb0 = tb.x;
        tb1 = tb.y;
        dr_wait(vu + p, t, lane);
        SP_TICK(u2_);
        SP_ADD(9, u1_, u2_);
        double* rrow = Rpan + 2 * q * ldr + g - 8 * p;  // + 8 * bb: block bb's pivot rows
        {  // the generation warp's next look-ahead block first: block p+2, still in this
           // warp's registers from job p-1 (it was updated last there and not stored)
          if (p == 0) tt_ld<K>(keep[0], taddr(s, 2));
          double* const rp[1] = {rrow + 8 * (p + 2)};
          tt_upd<K, 1>(keep, y, vb, tb0, tb1, rp, ldr);
          tt_st<K>(taddr(s, p + 2), keep[0]);
          tm_st_wait();
          tm_fence_before();
          dr_signal(ufirst + s, job + 1, lane);
        }
        SP_TICK(u2e_);
        SP_ADD(10, u2_, u2e_);
        }
        // staging of the slot's next tile, after the hand-off block (which the generation
        // warp is waiting for): block p (in flight since job p-1) into its TMEM columns, then
        // block p+1 into the stage
        if (more) {
          if (p == 0) {
            stage_issue(0);  // taken by the generation warp at the tile's start
          } else {
            sp_wait_ge(ver_p1 + p - 1, t + 1, lane);  // block p taken (hand-off of panel p-1)
            tm_fence_after();
          }
          stage_move(p);
          stage_issue(p + 1);
        }
        if (p + 2 < npan) {
        SP_TICK(u2b_);
        double* rrow = Rpan + 2 * q * ldr + g - 8 * p;
        int bb = p + 4;
        for (; bb + 1 < npan; bb += 2) {
          double c[2][K];
          {
            uint32_t ra[2 * K], rb[2 * K];
            tt_ld_issue<K>(ra, taddr(s, bb));
            tt_ld_issue<K>(rb, taddr(s, bb + 1));
            tm_ld_wait();
            tt_unpack<K>(c[0], ra);
            tt_unpack<K>(c[1], rb);
          }
          double* const rp[2] = {rrow + 8 * bb, rrow + 8 * (bb + 1)};
          tt_upd<K, 2>(c, y, vb, tb0, tb1, rp, ldr);
          tt_st<K>(taddr(s, bb), c[0]);
          tt_st<K>(taddr(s, bb + 1), c[1]);
        }
        if (bb < npan) {
          double c[1][K];
          tt_ld<K>(c[0], taddr(s, bb));
          double* const rp[1] = {rrow + 8 * bb};
          tt_upd<K, 1>(c, y, vb, tb0, tb1, rp, ldr);
          tt_st<K>(taddr(s, bb), c[0]);
        }
        if (p + 3 < npan) {  // block p+3 last, kept in registers: the next job's first block
          tt_ld<K>(keep[0], taddr(s, p + 3));
          double* const rp[1] = {rrow + 8 * (p + 3)};
          tt_upd<K, 1>(keep, y, vb, tb0, tb1, rp, ldr);
        }
        tm_st_wait();
        dr_signal(vu + p, t + 1, lane);
        SP_TICK(u3_);
        SP_ADD(10, u2b_, u3_);
        }
      }
      if (more) {
        sp_wait_ge(ver_p1 + npan - 2, t + 1, lane);  // the last block taken
        tm_fence_after();
        stage_move(npan - 1);
        tm_st_wait();
        tm_fence_before();
        dr_signal(staged + s, lt + 1, lane);
      }
    }
  }
  tm_fence_before();
  __syncthreads();
  tm_fence_after();
  if (w == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tbase) : "memory");
  // NaN / Inf anywhere in the leaf reaches R (see k_leaf_dmma)
  bool bad = false;
  double* Rl = Rio + (int64_t)leaf * n * n;
  for (int idx = threadIdx.x; idx < n * n; idx += THREADS) {
    const int r = idx / n, c = idx - r * n;
    const int pn = r >> 3;
    const double v = (c >= r) ? Rp[dr_pbase<128>(pn) + (r & 7) * dr_ldr<128>(pn) + (c - 8 * pn)] : 0.0;
    bad |= !isfinite(v);
    Rl[idx] = v;
  }
  if (bad && flag) atomicOr(flag, 1);
}
