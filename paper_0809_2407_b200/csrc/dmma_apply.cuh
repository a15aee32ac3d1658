// FP64-tensor-core (DMMA) apply and tree kernels: k_leaf_apply_dmma (below),
// k_leaf_q_dmma (leaf Q / Q^T), k_tree_apply_dmma (node Q / Q^T) and
// k_tree_factor_dmma (node factor, n <= 64).
//
// DMMA leaf apply: C[leaf rows] <- Q_leaf^T C for the chain leaves of n in
// (64, 128] (Y / tau in the layout of k_leaf_chain<128, 16> / k_leaf_dmma) --
// the CAQR trailing update, _apply_yt with transpose (householder.py:175-186,
// :209), one (leaf, 128-column block) per CTA.
//
// The dense first tile (V unit lower trapezoidal, LAPACK layout) is applied
// in compact WY too, 8 reflectors per panel with the tile's rows spread over
// the warps (partial G / W in shared memory, two barriers per panel); its top
// n rows then become the pivot rows Cs (shared memory, row stride KB + 2).  The chain tiles then run as the DMMA warp ring: warp w owns
// tiles w, w+8, ..., holds its 16 x 128 tile of C in registers in the DMMA
// accumulator layout of k_leaf_dmma, and applies each 8-reflector panel of
// the tile's TRI_ON_RECT factor in compact-WY form on the tensor cores:
//
//   G = Y_p^T Y_p (4 DMMA), T from G and tau by the Neumann product (10 DMMA)
//   per 8-column block: W = Cs_p + Y_p^T C (4), W' = T^T W (2), Cs_p -= W',
//   C -= Y_p W' (4)
//
// Tile t may update the pivot rows of panel p once tile t-1 has (ver[p] == t).
// Included by tsqr_sm100.cu (namespace tsqr) after dmma_ring.cuh.

// KB = columns per CTA: 128 for full-width trailing updates, 32 when the
// launch has few CTAs (the look-ahead update of the next panel's 128 columns:
// 4x the CTAs, each a quarter of the column work).
template <int KB>
struct DmmaApplySmem {
  static constexpr int LDC = KB + 2;  // pivot-row stride (doubles)
  // pivot rows (also the dense phase's W / G, or its staged V: 9 x 8 x 136 doubles, trapezoidal)
  static constexpr size_t doubles = (size_t)DR_NP * LDC > 9792 ? (size_t)DR_NP * LDC : 9792;
  static constexpr size_t tdense = KB >= 64 ? 16 * 64 : 0;  // the dense tile's 16 panel T (column-parallel phase)
  static constexpr size_t bytes = sizeof(double) * (doubles + tdense) + sizeof(int) * DR_NCB;
  static_assert(WARPS * 8 * KB + WARPS * 64 + 8 * KB <= DR_NP * LDC, "dense-phase scratch fits in Cs");
};

// Panel p of a chain tile: Y fragments (x: B operand of C^T Y; vb: B operand
// of Y^T) and the tau values the T build needs (tau_g, tau_{2q}, tau_{2q+1}).
struct DaPanel {
  double x[4], vb[2][2], tg, tq0, tq1;
};
template <bool TAUS = true>
__device__ __forceinline__ void da_load_panel(DaPanel& P, const double* __restrict__ Yt,
                                              int64_t ldy, const double* __restrict__ tt, int valid,
                                              int n, int pc) {
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, q = lane & 3;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int r = 8 * (k >> 1) + 2 * q + (k & 1), c = pc + g;
    P.x[k] = (r < valid && c < n) ? __ldg(Yt + (int64_t)r * ldy + c) : 0.0;
  }
#pragma unroll
  for (int bb = 0; bb < 2; ++bb)
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int r = 8 * bb + g, c = pc + 2 * q + s;
      P.vb[bb][s] = (r < valid && c < n) ? __ldg(Yt + (int64_t)r * ldy + c) : 0.0;
    }
  if constexpr (TAUS) {
    P.tg = (pc + g < n) ? __ldg(tt + pc + g) : 0.0;
    P.tq0 = (pc + 2 * q < n) ? __ldg(tt + pc + 2 * q) : 0.0;
    P.tq1 = (pc + 2 * q + 1 < n) ? __ldg(tt + pc + 2 * q + 1) : 0.0;
  }
}

// TR: tb[s] = T[2q+s][g] of the panel (the B operand of W'^T = W^T T, for Q^T)
// from Y and tau, all in registers: G = Y^T Y is symmetric, so both the
// accumulator and the B layout of M come from the same G fragment (same
// Neumann product as dr_form_t).  !TR: tb[s] = T[g][2q+s] (W'^T = W^T T^T, for
// Q): the polynomial of M^T = (the B layout of M read as the A layout) gives
// P(M)^T, and T = P(M)^T D.
template <bool TR = true>
__device__ __forceinline__ void da_form_t_g(const DaPanel& P, const double (&G)[2], double& tb0,
                                            double& tb1) {
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, q = lane & 3;
  const double tq[2] = {P.tq0, P.tq1};
  double MA[2], MB[2];
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const int c = 2 * q + e;
    const double ma = (c < g) ? tq[e] * G[e] : 0.0;  // M[g][c] = tau_c G[c][g]
    const double mb = (g < c) ? P.tg * G[e] : 0.0;   // M[c][g] = tau_g G[g][c]
    MA[e] = TR ? ma : mb;
    MB[e] = TR ? mb : ma;
  }
  double M2A[2] = {0.0, 0.0}, M2B[2] = {0.0, 0.0};
  dmma(M2A[0], M2A[1], MA[0], MB[0]);
  dmma(M2B[0], M2B[1], MB[0], MA[0]);
  dmma(M2A[0], M2A[1], MA[1], MB[1]);
  dmma(M2B[0], M2B[1], MB[1], MA[1]);
  double M4B[2] = {0.0, 0.0}, M3A[2] = {0.0, 0.0};
  dmma(M4B[0], M4B[1], M2B[0], M2A[0]);
  dmma(M3A[0], M3A[1], MA[0], M2B[0]);
  dmma(M4B[0], M4B[1], M2B[1], M2A[1]);
  dmma(M3A[0], M3A[1], MA[1], M2B[1]);
  double P1[2];
#pragma unroll
  for (int e = 0; e < 2; ++e) P1[e] = ((2 * q + e == g) ? 1.0 : 0.0) - MA[e] + M2A[e] - M3A[e];
  double PA[2] = {P1[0], P1[1]};
  dmma(PA[0], PA[1], P1[0], M4B[0]);
  dmma(PA[0], PA[1], P1[1], M4B[1]);
  tb0 = (TR ? P.tg : P.tq0) * PA[0];
  tb1 = (TR ? P.tg : P.tq1) * PA[1];
}
template <bool TR = true>
__device__ __forceinline__ void da_form_t(const DaPanel& P, double& tb0, double& tb1) {
  double G[2] = {0.0, 0.0};
#pragma unroll
  for (int k = 0; k < 4; ++k) dmma(G[0], G[1], P.x[k], P.x[k]);
  da_form_t_g<TR>(P, G, tb0, tb1);
}

// Panel P of the dense first tile on a warp's 8 NJ columns (column-parallel dense phase of
// k_leaf_apply_dmma<64 NJ>): c[j][2 rb + e] = C[8 rb + 2q + e][8j + g]; V (unit lower trapezoidal,
// zero above row 8P) staged in shared memory with row stride LDV; tb = T_P^T as the B operand.
// offset of panel p in the staged V: rows 8p .. 127 of its 8 columns, row stride 9
__host__ __device__ constexpr int da_voff(int p) { return 9 * (128 * p - 4 * p * (p - 1)); }
template <int P, int NJ>
__device__ __forceinline__ void da_dense_panel(double (&c)[NJ][32], const double* Vall, const double* tdn,
                                               int lane, int g, int q) {
  constexpr int LDV = 9;
  const double* Vs = Vall + da_voff(P) - 8 * P * LDV;  // row r of the panel at Vs[r * LDV + .]
  const double tb0 = tdn[P * 64 + 2 * lane], tb1 = tdn[P * 64 + 2 * lane + 1];
  double w0[NJ] = {}, w1[NJ] = {}, v0[NJ] = {}, v1[NJ] = {};
#pragma unroll
  for (int rb = P; rb < 16; ++rb) {
    const double y0 = Vs[(8 * rb + 2 * q) * LDV + g], y1 = Vs[(8 * rb + 2 * q + 1) * LDV + g];
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      dmma(w0[j], w1[j], c[j][2 * rb], y0);
      dmma(v0[j], v1[j], c[j][2 * rb + 1], y1);
    }
  }
  double u0[NJ] = {}, u1[NJ] = {};
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    dmma(u0[j], u1[j], w0[j] + v0[j], tb0);
    dmma(u0[j], u1[j], w1[j] + v1[j], tb1);
  }
#pragma unroll
  for (int rb = P; rb < 16; ++rb) {
    const double vb0 = Vs[(8 * rb + g) * LDV + 2 * q], vb1 = Vs[(8 * rb + g) * LDV + 2 * q + 1];
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      dmma(c[j][2 * rb], c[j][2 * rb + 1], -u0[j], vb0);
      dmma(c[j][2 * rb], c[j][2 * rb + 1], -u1[j], vb1);
    }
  }
}

// DCP (KB = 64 or 128): the dense first tile column-parallel (below)
template <int KB, bool DCP = false, bool HAST = false>
__global__ void __launch_bounds__(THREADS, KB == 64 ? 2 : 1)
k_leaf_apply_dmma(const double* __restrict__ Y, int64_t ldy, const double* __restrict__ tau,
                  int64_t tau_stride, int64_t m, int n, int P, int64_t base, double* C, int64_t ldc,
                  int64_t ncols, const double* __restrict__ Tin = nullptr) {
  // HAST: Tin holds the chain tiles' panel T stored by k_leaf_dmma (Tout), read instead of formed
  constexpr int H0 = WARPS * Geo<128>::HD, CB = KB / 8;  // dense first tile: 128 rows
  constexpr int DA_KB = KB, DA_LDC = DmmaApplySmem<KB>::LDC;
  extern __shared__ __align__(16) double sm[];
  double* Cs = sm;
  int* ver = reinterpret_cast<int*>(Cs + DmmaApplySmem<KB>::doubles + DmmaApplySmem<KB>::tdense);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int leaf = blockIdx.x;
  const int col0 = blockIdx.y * DA_KB;
  const int ncb = (int)min64(ncols - col0, DA_KB);
  const int64_t r0 = (int64_t)leaf * base;
  const int64_t b = (leaf == P - 1) ? m - r0 : base;
  const double* tl = tau + (int64_t)leaf * tau_stride;
  const double* Yl = Y + r0 * ldy;
  double* Cl = C + r0 * ldc + col0;
  const int64_t rest = b - H0;
  const int T = rest > 0 ? (int)((rest + DR_H - 1) / DR_H) : 0;
  const int npan = (n + 7) >> 3;
  if constexpr (KB >= 64 && DCP) {
    constexpr int NJ = KB / 64;  // 8-column blocks per warp
    // Dense first tile, COLUMN-parallel (as k_tree_apply_cp): V (128 x 128, unit lower
    // trapezoidal, LAPACK layout) staged in the pivot-row area, the 16 panel T formed once per
    // CTA (warp w: panels w, w + 8), then warp w applies all 16 panels to its 16 columns x 128
    // rows in registers -- two barriers for the tile instead of two per panel (the row-split
    // phase below, kept for the 32-column CTAs), and rows above 8p are skipped.  A quarter to a
    // half of the rows of CAQR's late panels are dense first tiles.
    double* Vs = Cs;
    double* tdn = Cs + DmmaApplySmem<KB>::doubles;  // [16][64], before ver
    {  // V trapezoid (panel p: rows 8p .. 127): cp.async for the strict lower part (zero fill
       // above it and past b / n), 1 on the diagonal
      const unsigned sbv = (unsigned)__cvta_generic_to_shared(Vs);
      for (int idx = threadIdx.x; idx < 128 * 128; idx += THREADS) {
        const int r = idx >> 7, c = idx & 127, p = c >> 3;
        if (r < 8 * p) continue;
        const int o = da_voff(p) + (r - 8 * p) * 9 + (c & 7);
        if (r == c) {
          Vs[o] = (r < b && c < n) ? 1.0 : 0.0;
        } else {
          const bool ok = r > c && r < b && c < n;
          cp_async<8>(sbv + 8u * (unsigned)o, ok ? Yl + (int64_t)r * ldy + c : Yl, ok ? 8u : 0u);
        }
      }
      cp_async_commit();
    }
    double c[NJ][32];
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const int r = 8 * (k >> 1) + 2 * q + (k & 1), cc = 8 * NJ * w + 8 * j + g;
        c[j][k] = (r < b && cc < ncb) ? Cl[(int64_t)r * ldc + cc] : 0.0;
      }
    cp_async_wait<0>();
    __syncthreads();
    for (int p = w; p < 16; p += WARPS) {
      const int pc = 8 * p;
      double G[2] = {0.0, 0.0}, G2[2] = {0.0, 0.0};
      for (int rb = p; rb < 16; ++rb) {
        const double* vp = Vs + da_voff(p) - pc * 9;
        const double y0 = vp[(8 * rb + 2 * q) * 9 + g], y1 = vp[(8 * rb + 2 * q + 1) * 9 + g];
        dmma(G[0], G[1], y0, y0);
        dmma(G2[0], G2[1], y1, y1);
      }
      G[0] += G2[0];
      G[1] += G2[1];
      DaPanel Pn;
      Pn.x[0] = Pn.x[1] = Pn.x[2] = Pn.x[3] = 0.0;
      Pn.tg = (pc + g < n) ? __ldg(tl + pc + g) : 0.0;
      Pn.tq0 = (pc + 2 * q < n) ? __ldg(tl + pc + 2 * q) : 0.0;
      Pn.tq1 = (pc + 2 * q + 1 < n) ? __ldg(tl + pc + 2 * q + 1) : 0.0;
      double tb0, tb1;
      da_form_t_g(Pn, G, tb0, tb1);
      tdn[p * 64 + 2 * lane] = tb0;
      tdn[p * 64 + 2 * lane + 1] = tb1;
    }
    __syncthreads();
#define DA_DP(PV) if (PV < npan) da_dense_panel<PV, NJ>(c, Vs, tdn, lane, g, q);
    DA_DP(0) DA_DP(1) DA_DP(2) DA_DP(3) DA_DP(4) DA_DP(5) DA_DP(6) DA_DP(7)
    DA_DP(8) DA_DP(9) DA_DP(10) DA_DP(11) DA_DP(12) DA_DP(13) DA_DP(14) DA_DP(15)
#undef DA_DP
    __syncthreads();  // every warp is done with V before the pivot rows take its place
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const int r = 8 * (k >> 1) + 2 * q + (k & 1), cc = 8 * NJ * w + 8 * j + g;
        if (r < n) Cs[r * DA_LDC + cc] = c[j][k];
        else if (r < b && cc < ncb) Cl[(int64_t)r * ldc + cc] = c[j][k];  // final rows
      }
#pragma unroll 1
    for (int idx = threadIdx.x; idx < (DR_NP - n) * KB; idx += THREADS)  // padded pivot rows
      Cs[(n + idx / KB) * DA_LDC + idx % KB] = 0.0;
  } else
  {  // dense first tile (LAPACK layout: V unit lower trapezoidal) in compact WY on the
     // tensor cores, 8 reflectors per panel: warp w holds rows 16w.. of the tile;
     // per panel partial G = V^T V and W = V^T C per warp (shared memory), then T
     // and W' = T^T W per column block, then C -= V W'.  Two barriers per panel.
    double* wpart = Cs;                       // [warp][refl 8][KB]  (Cs is free until the end)
    double* gpart = wpart + WARPS * 8 * KB;   // [warp][8 x 8]
    double* wfin = gpart + WARPS * 64;        // [refl 8][KB]
    double Cd[CB][2][2];
#pragma unroll
    for (int cb = 0; cb < CB; ++cb)
#pragma unroll
      for (int bb = 0; bb < 2; ++bb)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int r = 16 * w + 8 * bb + 2 * q + e, c = 8 * cb + g;
          Cd[cb][bb][e] = (r < b && c < ncb) ? Cl[(int64_t)r * ldc + c] : 0.0;
        }
    auto vdense = [&](int r, int c) {  // V[r][c] of the dense tile
      return (r >= b || c >= n) ? 0.0 : (r > c ? __ldg(Yl + (int64_t)r * ldy + c) : (r == c ? 1.0 : 0.0));
    };
    for (int p = 0; p < npan; ++p) {
      const int pc = 8 * p;
      const int wmin = pc >> 4;  // warps holding rows >= pc
      const bool active = w >= wmin;
      double x[4], vb[2][2];
      if (active) {
#pragma unroll
        for (int k = 0; k < 4; ++k) x[k] = vdense(16 * w + 8 * (k >> 1) + 2 * q + (k & 1), pc + g);
#pragma unroll
        for (int bb = 0; bb < 2; ++bb)
#pragma unroll
          for (int sx = 0; sx < 2; ++sx) vb[bb][sx] = vdense(16 * w + 8 * bb + g, pc + 2 * q + sx);
        double G[2] = {0.0, 0.0};
#pragma unroll
        for (int k = 0; k < 4; ++k) dmma(G[0], G[1], x[k], x[k]);
        gpart[w * 64 + g * 8 + 2 * q] = G[0];
        gpart[w * 64 + g * 8 + 2 * q + 1] = G[1];
#pragma unroll
        for (int cb = 0; cb < CB; ++cb) {
          double w0 = 0.0, w1 = 0.0;
          dmma(w0, w1, Cd[cb][0][0], x[0]);
          dmma(w0, w1, Cd[cb][1][0], x[2]);
          dmma(w0, w1, Cd[cb][0][1], x[1]);
          dmma(w0, w1, Cd[cb][1][1], x[3]);
          double* wp = wpart + (w * 8 + 2 * q) * KB + 8 * cb + g;
          wp[0] = w0;
          wp[KB] = w1;
        }
      }
      __syncthreads();
      {
        double G[2] = {0.0, 0.0};
        for (int w2 = wmin; w2 < WARPS; ++w2) {
          G[0] += gpart[w2 * 64 + g * 8 + 2 * q];
          G[1] += gpart[w2 * 64 + g * 8 + 2 * q + 1];
        }
        DaPanel Pn;
        Pn.x[0] = Pn.x[1] = Pn.x[2] = Pn.x[3] = 0.0;
        Pn.tg = (pc + g < n) ? __ldg(tl + pc + g) : 0.0;
        Pn.tq0 = (pc + 2 * q < n) ? __ldg(tl + pc + 2 * q) : 0.0;
        Pn.tq1 = (pc + 2 * q + 1 < n) ? __ldg(tl + pc + 2 * q + 1) : 0.0;
        double tb0, tb1;
        da_form_t_g(Pn, G, tb0, tb1);
        for (int cb = w; cb < CB; cb += WARPS) {
          double w0 = 0.0, w1 = 0.0;
          for (int w2 = wmin; w2 < WARPS; ++w2) {
            const double* wp = wpart + (w2 * 8 + 2 * q) * KB + 8 * cb + g;
            w0 += wp[0];
            w1 += wp[KB];
          }
          double u0 = 0.0, u1 = 0.0;
          dmma(u0, u1, w0, tb0);
          dmma(u0, u1, w1, tb1);
          wfin[(2 * q) * KB + 8 * cb + g] = u0;
          wfin[(2 * q + 1) * KB + 8 * cb + g] = u1;
        }
      }
      __syncthreads();
      if (active) {
#pragma unroll
        for (int cb = 0; cb < CB; ++cb) {
          const double u0 = wfin[(2 * q) * KB + 8 * cb + g];
          const double u1 = wfin[(2 * q + 1) * KB + 8 * cb + g];
#pragma unroll
          for (int bb = 0; bb < 2; ++bb) dmma(Cd[cb][bb][0], Cd[cb][bb][1], -u0, vb[bb][0]);
#pragma unroll
          for (int bb = 0; bb < 2; ++bb) dmma(Cd[cb][bb][0], Cd[cb][bb][1], -u1, vb[bb][1]);
        }
      }
    }
    __syncthreads();  // wpart / wfin (in Cs) consumed before Cs is filled
#pragma unroll
    for (int cb = 0; cb < CB; ++cb)
#pragma unroll
      for (int bb = 0; bb < 2; ++bb)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int r = 16 * w + 8 * bb + 2 * q + e, c = 8 * cb + g;
          Cs[r * DA_LDC + c] = (r < n) ? Cd[cb][bb][e] : 0.0;
          if (r >= n && r < b && c < ncb) Cl[(int64_t)r * ldc + c] = Cd[cb][bb][e];  // final rows
        }
  }
  if (threadIdx.x < DR_NCB) ver[threadIdx.x] = 0;
  __syncthreads();
  for (int t = w; t < T; t += WARPS) {
    const int64_t row = H0 + (int64_t)t * DR_H;
    const int valid = (int)min64(DR_H, b - row);
    double Ct[CB][2][2];
#pragma unroll
    for (int cb = 0; cb < CB; ++cb)
#pragma unroll
      for (int bb = 0; bb < 2; ++bb)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int r = 8 * bb + 2 * q + e, c = 8 * cb + g;
          Ct[cb][bb][e] = (r < valid && c < ncb) ? Cl[(row + r) * ldc + c] : 0.0;
        }
    const double* Yt = Yl + row * ldy;
    const double* tt = tl + (int64_t)(t + 1) * n;
    DaPanel cur, nxt;
    da_load_panel<!HAST>(cur, Yt, ldy, tt, valid, n, 0);
    // T of panel p+1 is formed in the same basic block as panel p's block
    // updates (its DMMA chain runs under them); for the last panel it works on
    // stale data and is discarded
    nxt = cur;
    double tb0, tb1;
    const double2* Tt = HAST ? reinterpret_cast<const double2*>(Tin) +
                                   ((int64_t)(leaf * (tau_stride / n) + t + 1) * 16) * 32 + lane
                             : nullptr;
    if constexpr (HAST) {
      const double2 t2 = __ldg(Tt);
      tb0 = t2.x;
      tb1 = t2.y;
    } else {
      da_form_t(cur, tb0, tb1);
    }
    for (int p = 0; p < npan; ++p) {
      if (p + 1 < npan) da_load_panel<!HAST>(nxt, Yt, ldy, tt, valid, n, 8 * (p + 1));
      dr_wait(ver + p, t, lane);
      double* rrow = Cs + (8 * p + 2 * q) * DA_LDC + g;
      double tn0, tn1;
      if constexpr (HAST) {
        const double2 t2 = __ldg(Tt + (p + 1 < npan ? p + 1 : p) * 32);
        tn0 = t2.x;
        tn1 = t2.y;
      } else {
        da_form_t(nxt, tn0, tn1);
      }
      // all blocks, unguarded (columns >= ncb are zero in Ct and Cs and never
      // stored): one basic block, so ptxas interleaves the blocks' DMMA chains
#pragma unroll
      for (int cb = 0; cb < CB; ++cb)
        dr_upd(Ct[cb], cur.x, cur.vb, tb0, tb1, rrow + 8 * cb, DA_LDC);
      dr_signal(ver + p, t + 1, lane);
      cur = nxt;
      tb0 = tn0;
      tb1 = tn1;
    }
#pragma unroll
    for (int cb = 0; cb < CB; ++cb)
#pragma unroll
      for (int bb = 0; bb < 2; ++bb)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int r = 8 * bb + 2 * q + e, c = 8 * cb + g;
          if (r < valid && c < ncb) Cl[(row + r) * ldc + c] = Ct[cb][bb][e];
        }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < n * DA_KB; idx += THREADS) {
    const int r = idx / DA_KB, c = idx - r * DA_KB;
    if (c < ncb) Cl[(int64_t)r * ldc + c] = Cs[r * DA_LDC + c];
  }
}

// ---------------------------------------------------------------------------
// DMMA leaf Q: C[leaf rows] <- Q_leaf C for the chain leaves of n in (32, 64]
// (NP = 64) or (64, 128] (NP = 128) with 16-row chain tiles -- explicit-Q
// formation and apply_q (householder.py:377-404; the order of k_leaf_apply's
// Q branch).  One (leaf, KB-column block) per CTA.  S (nullable): the leaf's
// top n rows come from S + leaf * s_slot_rows * lds (the tree's Q block);
// zero_init: the other rows start at zero.
//
// Q_leaf = Q_dense Q_1 ... Q_{T-1}, every tile factor a product of 8-reflector
// panels I - V T V^T, so the chain tiles run as the DMMA warp ring BACKWARD
// (tile T-1 first, warp w takes the w-th tile from the end) with the panels in
// reverse order:
//   W = Cs_p + Y_p^T C (4 DMMA per 8-column block), W' = T W (2),
//   Cs_p -= W', C -= Y_p W' (4)
// (dr_upd with T^T's B layout, da_form_t<false>), then the dense first tile
// (H0 = 8 x HD rows, RG 16-row groups per warp) in compact WY with its panels
// in reverse order.
// ---------------------------------------------------------------------------
template <int NP, int KB>
struct DmmaQSmem {
  static constexpr int LDC = KB + 2;
  static constexpr int SCR = WARPS * 8 * KB + WARPS * 64 + 8 * KB;  // dense phase: W, G, W'
  static constexpr size_t doubles = (size_t)NP * LDC + SCR;
  static constexpr size_t bytes = sizeof(double) * doubles + sizeof(int) * (NP / 8);
};

template <int NP, int KB, int MB, bool TR>
__global__ void __launch_bounds__(THREADS, MB)
k_leaf_q_dmma(const double* __restrict__ Y, int64_t ldy, const double* __restrict__ tau,
              int64_t tau_stride, int64_t m, int n, int P, int64_t base, double* C, int64_t ldc,
              int64_t ncols, const double* __restrict__ S, int64_t lds, int64_t s_slot_rows,
              int zero_init, int dense_only) {
  // dense_only: the leaf's chain tiles are not in this kernel's 16-row format (tall tiles:
  // k_tall_apply runs them before / after this launch); only the dense first tile is applied
  using SMQ = DmmaQSmem<NP, KB>;
  constexpr int HD = Geo<NP>::HD, H0 = WARPS * HD, RG = HD / 16, CB = KB / 8, LDC = SMQ::LDC;
  extern __shared__ __align__(16) double sm[];
  double* Cs = sm;                       // pivot rows, NP x LDC
  double* wpart = Cs + NP * LDC;         // [warp][refl 8][KB]
  double* gpart = wpart + WARPS * 8 * KB;  // [warp][8 x 8]
  double* wfin = gpart + WARPS * 64;       // [refl 8][KB]
  int* ver = reinterpret_cast<int*>(sm + SMQ::doubles);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int leaf = blockIdx.x;
  const int col0 = blockIdx.y * KB;
  const int ncb = (int)min64(ncols - col0, KB);
  const int64_t r0 = (int64_t)leaf * base;
  const int64_t b = (leaf == P - 1) ? m - r0 : base;
  const double* tl = tau + (int64_t)leaf * tau_stride;
  const double* Yl = Y + r0 * ldy;
  double* Cl = C + r0 * ldc + col0;
  const double* Sl = S ? S + (int64_t)leaf * s_slot_rows * lds + col0 : nullptr;
  const int64_t rest = b - H0;
  const int T = (rest > 0 && !dense_only) ? (int)((rest + DR_H - 1) / DR_H) : 0;
  const int npan = (n + 7) >> 3;
  for (int idx = threadIdx.x; idx < NP * KB; idx += THREADS) {
    const int r = idx / KB, c = idx - r * KB;
    double x = 0.0;
    if (r < n && c < ncb) x = Sl ? Sl[(int64_t)r * lds + c] : Cl[(int64_t)r * ldc + c];
    Cs[r * LDC + c] = x;
  }
  if (threadIdx.x < NP / 8) ver[threadIdx.x] = 0;
  __syncthreads();
  auto chain = [&]() {
  for (int o = w; o < T; o += WARPS) {
    const int t = TR ? o : T - 1 - o;
    const int64_t row = H0 + (int64_t)t * DR_H;
    const int valid = (int)min64(DR_H, b - row);
    double Ct[CB][2][2];
#pragma unroll
    for (int cb = 0; cb < CB; ++cb)
#pragma unroll
      for (int bb = 0; bb < 2; ++bb)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int r = 8 * bb + 2 * q + e, c = 8 * cb + g;
          Ct[cb][bb][e] = (!zero_init && r < valid && c < ncb) ? Cl[(row + r) * ldc + c] : 0.0;
        }
    const double* Yt = Yl + row * ldy;
    const double* tt = tl + (int64_t)(t + 1) * n;
    DaPanel cur, nxt;
    da_load_panel(cur, Yt, ldy, tt, valid, n, TR ? 0 : 8 * (npan - 1));
    nxt = cur;
    double tb0, tb1;
    da_form_t<TR>(cur, tb0, tb1);
    for (int i = 0; i < npan; ++i) {
      const int p = TR ? i : npan - 1 - i;
      if (i + 1 < npan) da_load_panel(nxt, Yt, ldy, tt, valid, n, 8 * (TR ? p + 1 : p - 1));
      dr_wait(ver + p, o, lane);
      double* rrow = Cs + (8 * p + 2 * q) * LDC + g;
      double tn0, tn1;
      da_form_t<TR>(nxt, tn0, tn1);  // stale for the last panel, discarded
#pragma unroll
      for (int cb = 0; cb < CB; ++cb)
        dr_upd(Ct[cb], cur.x, cur.vb, tb0, tb1, rrow + 8 * cb, LDC);
      dr_signal(ver + p, o + 1, lane);
      cur = nxt;
      tb0 = tn0;
      tb1 = tn1;
    }
#pragma unroll
    for (int cb = 0; cb < CB; ++cb)
#pragma unroll
      for (int bb = 0; bb < 2; ++bb)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int r = 8 * bb + 2 * q + e, c = 8 * cb + g;
          if (r < valid && c < ncb) Cl[(row + r) * ldc + c] = Ct[cb][bb][e];
        }
  }
  };
  if (!TR) {
    chain();
    __syncthreads();
  }
  // dense first tile: warp w holds rows HD w + 16 j + .., j < RG
  double Cd[RG][CB][2][2];
#pragma unroll
  for (int j = 0; j < RG; ++j)
#pragma unroll
    for (int cb = 0; cb < CB; ++cb)
#pragma unroll
      for (int bb = 0; bb < 2; ++bb)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int r = HD * w + 16 * j + 8 * bb + 2 * q + e, c = 8 * cb + g;
          double x = 0.0;
          if (r < n) x = Cs[r * LDC + c];
          else if (!zero_init && r < b && c < ncb) x = Cl[(int64_t)r * ldc + c];
          Cd[j][cb][bb][e] = x;
        }
  auto vdense = [&](int r, int c) {  // V[r][c] of the dense tile (unit lower trapezoidal)
    return (r >= b || c >= n) ? 0.0 : (r > c ? __ldg(Yl + (int64_t)r * ldy + c) : (r == c ? 1.0 : 0.0));
  };
  for (int i = 0; i < npan; ++i) {
    const int p = TR ? i : npan - 1 - i;
    const int pc = 8 * p;
    const int wmin = pc / HD;  // warps holding rows >= pc
    const bool active = w >= wmin;
    double x[RG][4], vb[RG][2][2];
    if (active) {
      double G[2] = {0.0, 0.0};
#pragma unroll
      for (int j = 0; j < RG; ++j) {
        const int rb = HD * w + 16 * j;
#pragma unroll
        for (int k = 0; k < 4; ++k) x[j][k] = vdense(rb + 8 * (k >> 1) + 2 * q + (k & 1), pc + g);
#pragma unroll
        for (int bb = 0; bb < 2; ++bb)
#pragma unroll
          for (int sx = 0; sx < 2; ++sx) vb[j][bb][sx] = vdense(rb + 8 * bb + g, pc + 2 * q + sx);
#pragma unroll
        for (int k = 0; k < 4; ++k) dmma(G[0], G[1], x[j][k], x[j][k]);
      }
      gpart[w * 64 + g * 8 + 2 * q] = G[0];
      gpart[w * 64 + g * 8 + 2 * q + 1] = G[1];
#pragma unroll
      for (int cb = 0; cb < CB; ++cb) {
        double w0 = 0.0, w1 = 0.0;
#pragma unroll
        for (int j = 0; j < RG; ++j) {
          dmma(w0, w1, Cd[j][cb][0][0], x[j][0]);
          dmma(w0, w1, Cd[j][cb][1][0], x[j][2]);
          dmma(w0, w1, Cd[j][cb][0][1], x[j][1]);
          dmma(w0, w1, Cd[j][cb][1][1], x[j][3]);
        }
        double* wp = wpart + (w * 8 + 2 * q) * KB + 8 * cb + g;
        wp[0] = w0;
        wp[KB] = w1;
      }
    }
    __syncthreads();
    {
      double G[2] = {0.0, 0.0};
      for (int w2 = wmin; w2 < WARPS; ++w2) {
        G[0] += gpart[w2 * 64 + g * 8 + 2 * q];
        G[1] += gpart[w2 * 64 + g * 8 + 2 * q + 1];
      }
      DaPanel Pn;
      Pn.x[0] = Pn.x[1] = Pn.x[2] = Pn.x[3] = 0.0;
      Pn.tg = (pc + g < n) ? __ldg(tl + pc + g) : 0.0;
      Pn.tq0 = (pc + 2 * q < n) ? __ldg(tl + pc + 2 * q) : 0.0;
      Pn.tq1 = (pc + 2 * q + 1 < n) ? __ldg(tl + pc + 2 * q + 1) : 0.0;
      double tb0, tb1;
      da_form_t_g<TR>(Pn, G, tb0, tb1);
      for (int cb = w; cb < CB; cb += WARPS) {
        double w0 = 0.0, w1 = 0.0;
        for (int w2 = wmin; w2 < WARPS; ++w2) {
          const double* wp = wpart + (w2 * 8 + 2 * q) * KB + 8 * cb + g;
          w0 += wp[0];
          w1 += wp[KB];
        }
        double u0 = 0.0, u1 = 0.0;
        dmma(u0, u1, w0, tb0);
        dmma(u0, u1, w1, tb1);
        wfin[(2 * q) * KB + 8 * cb + g] = u0;
        wfin[(2 * q + 1) * KB + 8 * cb + g] = u1;
      }
    }
    __syncthreads();
    if (active) {
#pragma unroll
      for (int cb = 0; cb < CB; ++cb) {
        const double u0 = wfin[(2 * q) * KB + 8 * cb + g];
        const double u1 = wfin[(2 * q + 1) * KB + 8 * cb + g];
#pragma unroll
        for (int j = 0; j < RG; ++j) {
#pragma unroll
          for (int bb = 0; bb < 2; ++bb) dmma(Cd[j][cb][bb][0], Cd[j][cb][bb][1], -u0, vb[j][bb][0]);
#pragma unroll
          for (int bb = 0; bb < 2; ++bb) dmma(Cd[j][cb][bb][0], Cd[j][cb][bb][1], -u1, vb[j][bb][1]);
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < RG; ++j)
#pragma unroll
    for (int cb = 0; cb < CB; ++cb)
#pragma unroll
      for (int bb = 0; bb < 2; ++bb)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int r = HD * w + 16 * j + 8 * bb + 2 * q + e, c = 8 * cb + g;
          if (TR && r < n) Cs[r * LDC + c] = Cd[j][cb][bb][e];  // the chain's pivot rows
          else if (r < b && c < ncb) Cl[(int64_t)r * ldc + c] = Cd[j][cb][bb][e];
        }
  if (TR) {
    __syncthreads();
    chain();
    __syncthreads();
    for (int idx = threadIdx.x; idx < n * KB; idx += THREADS) {
      const int r = idx / KB, c = idx - r * KB;
      if (c < ncb) Cl[(int64_t)r * ldc + c] = Cs[r * LDC + c];
    }
  }
}

// ---------------------------------------------------------------------------
// DMMA tree apply: [C_a; C_b] <- Q_node^T [C_a; C_b] for a STACKED node
// (qr_stacked_triangles, q = 2: reflector j = [e_j; Y[0..j][j]], householder.py:
// 263-294, 335-374 with the identity top) -- the CAQR tree-level update.
// One (event, 64-column block) per CTA; warp w holds rows 16w.. of C_b in
// registers, C_a (the pivot rows) lives in shared memory.  Per 8-reflector
// panel p (Y's rows > 8p+7 are zero, so warps below them sit out):
//   partial G_w = Y_w^T Y_w and W_w = Y_w^T C_b,w (active warps)  | barrier
//   every warp: T from sum G; warp w forms W' = T^T (C_a,p + sum W_w) for its
//   column block, C_a,p -= W'                                       | barrier
//   active warps: C_b,w -= Y_w W'
// Two barriers per 8 reflectors instead of one per reflector.
// ---------------------------------------------------------------------------
constexpr int TA_KB = 64;
constexpr int TA_LDC = TA_KB + 2;
struct TreeApplyDmmaSmem {
  // C_a, partial W, final W', then per-panel partial G (16 x 8 warps) and T (16 x 64)
  static constexpr size_t doubles = (size_t)DR_NP * TA_LDC + WARPS * 8 * TA_KB + WARPS * 64 + 8 * TA_KB +
                                    (size_t)DR_NCB * WARPS * 64 + DR_NCB * 64;
  static constexpr size_t bytes = sizeof(double) * doubles;
};

// TR = false: Q_node [C_a; C_b] (explicit Q / apply_q walking the tree down):
// panels in reverse order with T instead of T^T; zero_partner: C_b starts at 0.
template <bool TR>
__global__ void __launch_bounds__(THREADS, 1)
k_tree_apply_dmma(const double* __restrict__ Ynode, const double* __restrict__ taunode, int n,
                  const int* __restrict__ ev, double* C, int64_t ldc, int64_t slot_rows,
                  int64_t ncols, int zero_partner) {
  extern __shared__ __align__(16) double sm[];
  double* Ca = sm;                           // 128 x 66
  double* wpart = Ca + DR_NP * TA_LDC;       // [warp][refl 8][col 64]
  double* gpart = wpart + WARPS * 8 * TA_KB; // [warp][8 x 8]
  double* wfin = gpart + WARPS * 64;         // [refl 8][col 64]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int a = ev[3 * blockIdx.x], b = ev[3 * blockIdx.x + 1], id = ev[3 * blockIdx.x + 2];
  const int col0 = blockIdx.y * TA_KB;
  const int ncb = (int)min64(ncols - col0, TA_KB);
  double* Cag = C + (int64_t)a * slot_rows * ldc + col0;
  double* Cbg = C + (int64_t)b * slot_rows * ldc + col0;
  const double* Yn = Ynode + (int64_t)id * n * n;
  const double* tn = taunode + (int64_t)id * n;
  for (int idx = threadIdx.x; idx < DR_NP * TA_KB; idx += THREADS) {
    const int r = idx / TA_KB, c = idx - r * TA_KB;
    Ca[r * TA_LDC + c] = (r < n && c < ncb) ? Cag[(int64_t)r * ldc + c] : 0.0;
  }
  double Cb[TA_KB / 8][2][2];
#pragma unroll
  for (int cb = 0; cb < TA_KB / 8; ++cb)
#pragma unroll
    for (int bb = 0; bb < 2; ++bb)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = 16 * w + 8 * bb + 2 * q + e, c = 8 * cb + g;
        Cb[cb][bb][e] = (!zero_partner && r < n && c < ncb) ? Cbg[(int64_t)r * ldc + c] : 0.0;
      }
  const int npan = (n + 7) >> 3;
  // T of every panel depends on the node factor only: build them all up front
  // (partial G per warp and panel, then warp w forms T of panels w, w+8)
  double* gall = wfin + 8 * TA_KB;            // [panel][warp][8 x 8]
  double* tball = gall + DR_NCB * WARPS * 64;  // [panel][lane][2]
  for (int p = 0; p < npan; ++p) {
    const int pc = 8 * p;
    if (16 * w > pc + 7) continue;  // no nonzero rows of Y_p in this warp
    double xg[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int r = 16 * w + 8 * (k >> 1) + 2 * q + (k & 1), c = pc + g;
      xg[k] = (r < n && c < n) ? __ldg(Yn + (int64_t)r * n + c) : 0.0;
    }
    double G[2] = {0.0, 0.0};
#pragma unroll
    for (int k = 0; k < 4; ++k) dmma(G[0], G[1], xg[k], xg[k]);
    gall[(p * WARPS + w) * 64 + g * 8 + 2 * q] = G[0];
    gall[(p * WARPS + w) * 64 + g * 8 + 2 * q + 1] = G[1];
  }
  __syncthreads();
  for (int p = w; p < npan; p += WARPS) {
    const int pc = 8 * p;
    const int wmax = min(WARPS - 1, (pc + 7) >> 4);
    double G[2] = {0.0, 0.0};
    for (int w2 = 0; w2 <= wmax; ++w2) {
      G[0] += gall[(p * WARPS + w2) * 64 + g * 8 + 2 * q];
      G[1] += gall[(p * WARPS + w2) * 64 + g * 8 + 2 * q + 1];
    }
    DaPanel P;
    P.x[0] = P.x[1] = P.x[2] = P.x[3] = 0.0;
    P.tg = (pc + g < n) ? __ldg(tn + pc + g) : 0.0;
    P.tq0 = (pc + 2 * q < n) ? __ldg(tn + pc + 2 * q) : 0.0;
    P.tq1 = (pc + 2 * q + 1 < n) ? __ldg(tn + pc + 2 * q + 1) : 0.0;
    double tb0, tb1;
    da_form_t_g<TR>(P, G, tb0, tb1);
    tball[p * 64 + 2 * lane] = tb0;
    tball[p * 64 + 2 * lane + 1] = tb1;
  }
  __syncthreads();
  for (int i = 0; i < npan; ++i) {
    const int p = TR ? i : npan - 1 - i;
    const int pc = 8 * p;
    const int wmax = min(WARPS - 1, (pc + 7) >> 4);  // warps holding nonzero rows of Y_p
    const bool active = w <= wmax;
    double x[4], vb[2][2];
    if (active) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int r = 16 * w + 8 * (k >> 1) + 2 * q + (k & 1), c = pc + g;
        x[k] = (r < n && c < n) ? __ldg(Yn + (int64_t)r * n + c) : 0.0;
      }
#pragma unroll
      for (int bb = 0; bb < 2; ++bb)
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          const int r = 16 * w + 8 * bb + g, c = pc + 2 * q + s;
          vb[bb][s] = (r < n && c < n) ? __ldg(Yn + (int64_t)r * n + c) : 0.0;
        }
#pragma unroll
      for (int cb = 0; cb < TA_KB / 8; ++cb) {
        double wa0 = 0.0, wa1 = 0.0, wb0 = 0.0, wb1 = 0.0;
        dmma(wa0, wa1, Cb[cb][0][0], x[0]);
        dmma(wb0, wb1, Cb[cb][1][0], x[2]);
        dmma(wa0, wa1, Cb[cb][0][1], x[1]);
        dmma(wb0, wb1, Cb[cb][1][1], x[3]);
        double* wp = wpart + w * 8 * TA_KB + 8 * cb + g;
        wp[(2 * q) * TA_KB] = wa0 + wb0;
        wp[(2 * q + 1) * TA_KB] = wa1 + wb1;
      }
    }
    __syncthreads();
    {  // W' of column block w
      const double tb0 = tball[p * 64 + 2 * lane], tb1 = tball[p * 64 + 2 * lane + 1];
      double* ca = Ca + (pc + 2 * q) * TA_LDC + 8 * w + g;
      double w0 = ca[0], w1 = ca[TA_LDC];
      for (int w2 = 0; w2 <= wmax; ++w2) {
        const double* wp = wpart + w2 * 8 * TA_KB + 8 * w + g;
        w0 += wp[(2 * q) * TA_KB];
        w1 += wp[(2 * q + 1) * TA_KB];
      }
      double u0 = 0.0, u1 = 0.0;
      dmma(u0, u1, w0, tb0);
      dmma(u0, u1, w1, tb1);
      ca[0] -= u0;
      ca[TA_LDC] -= u1;
      wfin[(2 * q) * TA_KB + 8 * w + g] = u0;
      wfin[(2 * q + 1) * TA_KB + 8 * w + g] = u1;
    }
    __syncthreads();
    if (active) {
#pragma unroll
      for (int cb = 0; cb < TA_KB / 8; ++cb) {
        const double u0 = wfin[(2 * q) * TA_KB + 8 * cb + g];
        const double u1 = wfin[(2 * q + 1) * TA_KB + 8 * cb + g];
#pragma unroll
        for (int bb = 0; bb < 2; ++bb) dmma(Cb[cb][bb][0], Cb[cb][bb][1], -u0, vb[bb][0]);
#pragma unroll
        for (int bb = 0; bb < 2; ++bb) dmma(Cb[cb][bb][0], Cb[cb][bb][1], -u1, vb[bb][1]);
      }
    }
  }
#pragma unroll
  for (int cb = 0; cb < TA_KB / 8; ++cb)
#pragma unroll
    for (int bb = 0; bb < 2; ++bb)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = 16 * w + 8 * bb + 2 * q + e, c = 8 * cb + g;
        if (r < n && c < ncb) Cbg[(int64_t)r * ldc + c] = Cb[cb][bb][e];
      }
  __syncthreads();
  for (int idx = threadIdx.x; idx < n * TA_KB; idx += THREADS) {
    const int r = idx / TA_KB, c = idx - r * TA_KB;
    if (c < ncb) Cag[(int64_t)r * ldc + c] = Ca[r * TA_LDC + c];
  }
}

// ---------------------------------------------------------------------------
// DMMA tree factor: the STACKED combine [R_a; R_b] -> R, node Y / tau
// (qr_stacked_triangles, q = 2, householder.py:263-294) for n <= 64 with the
// node factor kept (explicit / implicit Q).  One CTA per event; warp w owns
// column block w (8 columns) of R_b in registers -- all NP rows as NG 16-row
// groups in the DMMA accumulator layout of k_leaf_dmma -- and of the pivot
// rows R_a (shared memory).  Panel p (8 reflectors) is factored Level-2 by the
// warp that owns block p (dr_gen over NG groups), which publishes Y_p and T_p
// (shared memory, version counter); every warp owning a later block then
// applies the panel in compact WY on the tensor cores.  The owner of block p+1
// factors panel p+1 as soon as its own block has panel p applied: the
// critical path is one panel factor + one block update per 8 reflectors
// instead of two CTA barriers per reflector (k_tree_factor).  R_b is treated
// as a dense NP-row block: its zeros below the diagonal stay exactly zero.
// ---------------------------------------------------------------------------
template <int NP>
struct TreeFactorDmmaSmem {
  static constexpr int NCB = NP / 8, LDA = NP + 2, LDY = 9;
  static constexpr size_t doubles =
      (size_t)NP * LDA + (size_t)NCB * NP * LDY + NCB * 64 + NCB * 64 + NCB * 8;
  static constexpr size_t bytes = sizeof(double) * doubles + sizeof(int) * NCB;
};

// dr_gen over NG 16-row groups (the pivot row x0 and the column sums are
// shared by all groups).
template <int I, int NG>
__device__ __forceinline__ void tf_gen(double (&x)[NG][4], double rgi, double* Rrow, double* gs,
                                       double* taus) {
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, q = lane & 3;
  const int src = 4 * I + q;
  double xi[NG][4];
#pragma unroll
  for (int j = 0; j < NG; ++j)
#pragma unroll
    for (int k = 0; k < 4; ++k) xi[j][k] = __shfl_sync(FULL, x[j][k], src);
  const double x0 = __shfl_sync(FULL, rgi, 4 * I);
  double s = 0.0, s2 = 0.0, pd = 0.0, pd2 = 0.0;
#pragma unroll
  for (int j = 0; j < NG; ++j) {
    s = fma(xi[j][0], xi[j][0], s);
    s2 = fma(xi[j][2], xi[j][2], s2);
    s = fma(xi[j][1], xi[j][1], s);
    s2 = fma(xi[j][3], xi[j][3], s2);
    pd = fma(xi[j][0], x[j][0], pd);
    pd2 = fma(xi[j][2], x[j][2], pd2);
    pd = fma(xi[j][1], x[j][1], pd);
    pd2 = fma(xi[j][3], x[j][3], pd2);
  }
  s += s2;
  pd += pd2;
  s += __shfl_xor_sync(FULL, s, 1);
  pd += __shfl_xor_sync(FULL, pd, 1);
  s += __shfl_xor_sync(FULL, s, 2);
  pd += __shfl_xor_sync(FULL, pd, 2);
  double beta, tau, scale, invb;
  house_fast(x0, s, beta, tau, scale, invb);
  const double tw = fma(scale, pd, rgi);
  const double wv = tau * tw;
  const bool upd = g > I;
  const bool own = (g == I);  // owner column: v = scale * x_I in one rounding (see dr_gen)
  const double f = upd ? tw * invb : (own ? scale : 0.0);
#pragma unroll
  for (int j = 0; j < NG; ++j)
#pragma unroll
    for (int k = 0; k < 4; ++k) x[j][k] = fma(f, xi[j][k], own ? 0.0 : x[j][k]);
  double* dst = upd ? Rrow + g : ((g == I) ? Rrow + I : gs + g * 8 + I);
  *dst = upd ? rgi - wv : ((g == I) ? beta : scale * pd);
  taus[I] = tau;
}

template <int NP>
__global__ void __launch_bounds__(THREADS, 1)
k_tree_factor_dmma(double* Rslots, int n, const int* __restrict__ ev, double* Ynode,
                   double* taunode) {
  using SMT = TreeFactorDmmaSmem<NP>;
  constexpr int NG = NP / 16, NCB = SMT::NCB, LDA = SMT::LDA, LDY = SMT::LDY;
  extern __shared__ __align__(16) double sm[];
  double* Ra = sm;                         // pivot rows, NP x LDA
  double* Ys = Ra + NP * LDA;              // [panel][row NP][LDY]
  double* tbs = Ys + NCB * NP * LDY;       // [panel][lane][2]
  double* gss = tbs + NCB * 64;            // [panel][8 x 8]
  double* tss = gss + NCB * 64;            // [panel][8]
  int* ver = reinterpret_cast<int*>(tss + NCB * 8);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int a = ev[3 * blockIdx.x], b = ev[3 * blockIdx.x + 1], id = ev[3 * blockIdx.x + 2];
  const double* Rag = Rslots + (int64_t)a * n * n;
  const double* Rbg = Rslots + (int64_t)b * n * n;
  for (int idx = threadIdx.x; idx < NP * NP; idx += THREADS) {
    const int r = idx / NP, c = idx - r * NP;
    Ra[r * LDA + c] = (r < n && c < n && c >= r) ? Rag[r * n + c] : 0.0;
  }
  if (threadIdx.x < NCB) ver[threadIdx.x] = 0;
  double C[NG][2][2];  // block w of R_b: rows 16 j + 8 bb + 2 q + e, column 8 w + g
#pragma unroll
  for (int j = 0; j < NG; ++j)
#pragma unroll
    for (int bb = 0; bb < 2; ++bb)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = 16 * j + 8 * bb + 2 * q + e, c = 8 * w + g;
        C[j][bb][e] = (w < NCB && r < n && c < n && c >= r) ? Rbg[r * n + c] : 0.0;
      }
  __syncthreads();
  const int npan = (n + 7) >> 3;
  double* Yo = Ynode + (int64_t)id * n * n;
  double* to = taunode + (int64_t)id * n;
  const int pmax = (w < npan) ? w : -1;  // warps past the last panel own padding only
  for (int p = 0; p <= pmax; ++p) {
    const int pc = 8 * p;
    if (p == w) {  // factor panel p (my block)
      double* gs = gss + p * 64;
      double* taus = tss + p * 8;
      double rg[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) rg[i] = Ra[(pc + i) * LDA + pc + g];
      double x[NG][4];
#pragma unroll
      for (int j = 0; j < NG; ++j) {
        x[j][0] = C[j][0][0]; x[j][1] = C[j][0][1]; x[j][2] = C[j][1][0]; x[j][3] = C[j][1][1];
      }
      double* Rrow = Ra + pc * LDA + pc;
      tf_gen<0, NG>(x, rg[0], Rrow, gs, taus);
      tf_gen<1, NG>(x, rg[1], Rrow + LDA, gs, taus);
      tf_gen<2, NG>(x, rg[2], Rrow + 2 * LDA, gs, taus);
      tf_gen<3, NG>(x, rg[3], Rrow + 3 * LDA, gs, taus);
      tf_gen<4, NG>(x, rg[4], Rrow + 4 * LDA, gs, taus);
      tf_gen<5, NG>(x, rg[5], Rrow + 5 * LDA, gs, taus);
      tf_gen<6, NG>(x, rg[6], Rrow + 6 * LDA, gs, taus);
      tf_gen<7, NG>(x, rg[7], Rrow + 7 * LDA, gs, taus);
      double* ys = Ys + p * NP * LDY;
#pragma unroll
      for (int j = 0; j < NG; ++j)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int r = 16 * j + 8 * (k >> 1) + 2 * q + (k & 1);
          ys[r * LDY + g] = x[j][k];
          if (r < n && pc + g < n) Yo[(int64_t)r * n + pc + g] = x[j][k];
        }
      __syncwarp();
      double tb0, tb1;
      dr_form_t(gs, taus, tb0, tb1);
      tbs[p * 64 + 2 * lane] = tb0;
      tbs[p * 64 + 2 * lane + 1] = tb1;
      if (lane < 8 && pc + lane < n) to[pc + lane] = taus[lane];
      dr_signal(ver + p, 1, lane);
    } else {  // apply panel p to my block (w > p)
      dr_wait(ver + p, 1, lane);
      const double* ys = Ys + p * NP * LDY;
      double xv[NG][4], vb[NG][2][2];
#pragma unroll
      for (int j = 0; j < NG; ++j) {
#pragma unroll
        for (int k = 0; k < 4; ++k) xv[j][k] = ys[(16 * j + 8 * (k >> 1) + 2 * q + (k & 1)) * LDY + g];
#pragma unroll
        for (int bb = 0; bb < 2; ++bb)
#pragma unroll
          for (int s = 0; s < 2; ++s) vb[j][bb][s] = ys[(16 * j + 8 * bb + g) * LDY + 2 * q + s];
      }
      const double tb0 = tbs[p * 64 + 2 * lane], tb1 = tbs[p * 64 + 2 * lane + 1];
      double* rp = Ra + (pc + 2 * q) * LDA + 8 * w + g;
      const double ro0 = rp[0], ro1 = rp[LDA];
      double w0 = ro0, w1 = ro1;
#pragma unroll
      for (int j = 0; j < NG; ++j) {
        dmma(w0, w1, C[j][0][0], xv[j][0]);
        dmma(w0, w1, C[j][1][0], xv[j][2]);
        dmma(w0, w1, C[j][0][1], xv[j][1]);
        dmma(w0, w1, C[j][1][1], xv[j][3]);
      }
      double u0 = 0.0, u1 = 0.0;
      dmma(u0, u1, w0, tb0);
      dmma(u0, u1, w1, tb1);
      rp[0] = ro0 - u0;
      rp[LDA] = ro1 - u1;
#pragma unroll
      for (int j = 0; j < NG; ++j) {
        dmma(C[j][0][0], C[j][0][1], -u0, vb[j][0][0]);
        dmma(C[j][1][0], C[j][1][1], -u0, vb[j][1][0]);
        dmma(C[j][0][0], C[j][0][1], -u1, vb[j][0][1]);
        dmma(C[j][1][0], C[j][1][1], -u1, vb[j][1][1]);
      }
    }
  }
  __syncthreads();
  double* Ro = Rslots + (int64_t)a * n * n;
  for (int idx = threadIdx.x; idx < n * n; idx += THREADS) {
    const int r = idx / n, c = idx - r * n;
    Ro[idx] = (c >= r) ? Ra[r * LDA + c] : 0.0;
  }
}

// ---------------------------------------------------------------------------
// DMMA dense first tile (n <= 64): the DENSE QR of a leaf's first H0 rows
// (qr_unblocked, householder.py:128-145; LAPACK layout: R on and above the
// diagonal, V below it) as column-block warps like k_tree_factor_dmma: warp w
// holds column block w of the whole tile (NG = H0/16 row groups) in
// registers; the owner of block p factors panel p Level-2 (dd_gen: the pivot
// row is inside the column, so every sum is masked by row index), publishes V_p
// (unit lower trapezoidal) and T_p, and the owners of later blocks apply
// I - V T^T V^T on the tensor cores.  Replaces k_leaf_dense's two CTA barriers
// per reflector with one panel factor + one block update per 8 reflectors.
// ---------------------------------------------------------------------------
template <int NP>
struct DenseDmmaSmem {
  static constexpr int NCB = NP / 8, H0 = WARPS * Geo<NP>::HD, LDY = 9;
  static constexpr size_t doubles = (size_t)NCB * H0 * LDY + NCB * 64 + NCB * 64 + NCB * 8;
  static constexpr size_t bytes = sizeof(double) * doubles + sizeof(int) * NCB;
};

// Generation I of panel pc (pivot row jr = pc + I) over the NG groups of the
// owner's registers x (lane (g, q): rows 16 J + 8 (k >> 1) + 2 q + (k & 1) of
// column pc + g).  Column I's values are shuffled twice (sums, then update)
// rather than held, to keep the register count down.
template <int I, int NG>
__device__ __forceinline__ void dd_gen(double (&x)[NG][4], int pc, double* gs, double* taus) {
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, q = lane & 3;
  const int src = 4 * I + q, jr = pc + I;
  double s = 0.0, pd = 0.0, x0 = 0.0, xg0 = 0.0;
#pragma unroll
  for (int J = 0; J < NG; ++J)
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int r = 16 * J + 8 * (k >> 1) + 2 * q + (k & 1);
      const double v = __shfl_sync(FULL, x[J][k], src);
      const double vb = r > jr ? v : 0.0;
      s = fma(vb, vb, s);
      pd = fma(vb, x[J][k], pd);
      x0 += r == jr ? v : 0.0;
      xg0 += r == jr ? x[J][k] : 0.0;
    }
  s += __shfl_xor_sync(FULL, s, 1);
  pd += __shfl_xor_sync(FULL, pd, 1);
  x0 += __shfl_xor_sync(FULL, x0, 1);
  xg0 += __shfl_xor_sync(FULL, xg0, 1);
  s += __shfl_xor_sync(FULL, s, 2);
  pd += __shfl_xor_sync(FULL, pd, 2);
  x0 += __shfl_xor_sync(FULL, x0, 2);
  xg0 += __shfl_xor_sync(FULL, xg0, 2);
  double beta, tau, scale;
  house_scalars(x0, s, beta, tau, scale);
  const double invb = (s == 0.0) ? 0.0 : __drcp_rn(beta);
  const double tw = fma(scale, pd, xg0);  // w_g = x[jr][g] + v^T x_g (below jr)
  const bool upd = g > I, own = g == I;
  const double f = upd ? tw * invb : (own ? scale : 0.0);  // below jr
  const double pn = upd ? fma(-tau, tw, xg0) : beta;        // row jr (g >= I)
#pragma unroll
  for (int J = 0; J < NG; ++J)
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int r = 16 * J + 8 * (k >> 1) + 2 * q + (k & 1);
      const double v = __shfl_sync(FULL, x[J][k], src);
      const double nb = fma(f, v, own ? 0.0 : x[J][k]);
      x[J][k] = r > jr ? nb : ((r == jr && g >= I) ? pn : x[J][k]);
    }
  if (g < I) gs[g * 8 + I] = tw;  // G[g][I] = v_g^T v_I
  taus[I] = tau;
}

template <int NP>
__global__ void __launch_bounds__(THREADS, 1)
k_leaf_dense_dmma(const double* __restrict__ A, int64_t lda, int64_t m, int n, int P, int64_t base,
                  double* Y, int64_t ldy, double* tau, int64_t tau_stride, double* Rout, int* flag) {
  using SMD = DenseDmmaSmem<NP>;
  constexpr int NCB = SMD::NCB, H0 = SMD::H0, NG = H0 / 16, LDY = SMD::LDY;
  extern __shared__ __align__(16) double sm[];
  double* Ys = sm;                      // [panel][row H0][LDY]: V_p, unit lower trapezoidal
  double* tbs = Ys + NCB * H0 * LDY;    // [panel][lane][2]
  double* gss = tbs + NCB * 64;         // [panel][8 x 8]
  double* tss = gss + NCB * 64;         // [panel][8]
  int* ver = reinterpret_cast<int*>(tss + NCB * 8);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int leaf = blockIdx.x;
  const int64_t r0 = (int64_t)leaf * base;
  const int64_t b = (leaf == P - 1) ? m - r0 : base;
  const int rows = (int)min64(H0, b);
  double* tl = tau ? tau + (int64_t)leaf * tau_stride : nullptr;
  if (threadIdx.x < NCB) ver[threadIdx.x] = 0;
  bool bad = false;
  double C[NG][4];  // block w: rows 16 J + 8 (k >> 1) + 2 q + (k & 1), column 8 w + g
  const int c = 8 * w + g;
#pragma unroll
  for (int J = 0; J < NG; ++J)
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int r = 16 * J + 8 * (k >> 1) + 2 * q + (k & 1);
      double v = 0.0;
      if (w < NCB && r < rows && c < n) v = A[(r0 + r) * lda + c];
      bad |= !isfinite(v);
      C[J][k] = v;
    }
  __syncthreads();
  const int npan = (n + 7) >> 3;
  const int pmax = (w < npan) ? w : -1;
  for (int p = 0; p <= pmax; ++p) {
    const int pc = 8 * p;
    if (p == w) {  // factor panel p (my block)
      double* gs = gss + p * 64;
      double* taus = tss + p * 8;
      dd_gen<0, NG>(C, pc, gs, taus);
      dd_gen<1, NG>(C, pc, gs, taus);
      dd_gen<2, NG>(C, pc, gs, taus);
      dd_gen<3, NG>(C, pc, gs, taus);
      dd_gen<4, NG>(C, pc, gs, taus);
      dd_gen<5, NG>(C, pc, gs, taus);
      dd_gen<6, NG>(C, pc, gs, taus);
      dd_gen<7, NG>(C, pc, gs, taus);
      double* ys = Ys + p * H0 * LDY;
#pragma unroll
      for (int J = 0; J < NG; ++J)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int r = 16 * J + 8 * (k >> 1) + 2 * q + (k & 1);
          ys[r * LDY + g] = r > pc + g ? C[J][k] : (r == pc + g ? 1.0 : 0.0);
        }
      __syncwarp();
      double tb0, tb1;
      dr_form_t(gs, taus, tb0, tb1);
      tbs[p * 64 + 2 * lane] = tb0;
      tbs[p * 64 + 2 * lane + 1] = tb1;
      if (tl && lane < 8 && pc + lane < n) tl[pc + lane] = taus[lane];
      dr_signal(ver + p, 1, lane);
    } else {  // apply panel p to my block: C -= V (T^T (V^T C))
      dr_wait(ver + p, 1, lane);
      const double* ys = Ys + p * H0 * LDY;
      const double tb0 = tbs[p * 64 + 2 * lane], tb1 = tbs[p * 64 + 2 * lane + 1];
      const int J0 = pc >> 4;  // V_p is zero above row pc
      double w0 = 0.0, w1 = 0.0;
#pragma unroll
      for (int J = 0; J < NG; ++J) {
        if (J < J0) continue;
        double xv[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) xv[k] = ys[(16 * J + 8 * (k >> 1) + 2 * q + (k & 1)) * LDY + g];
        dmma(w0, w1, C[J][0], xv[0]);
        dmma(w0, w1, C[J][2], xv[2]);
        dmma(w0, w1, C[J][1], xv[1]);
        dmma(w0, w1, C[J][3], xv[3]);
      }
      double u0 = 0.0, u1 = 0.0;
      dmma(u0, u1, w0, tb0);
      dmma(u0, u1, w1, tb1);
#pragma unroll
      for (int J = 0; J < NG; ++J) {
        if (J < J0) continue;
        double vb[2][2];
#pragma unroll
        for (int bb = 0; bb < 2; ++bb)
#pragma unroll
          for (int s2 = 0; s2 < 2; ++s2) vb[bb][s2] = ys[(16 * J + 8 * bb + g) * LDY + 2 * q + s2];
        dmma(C[J][0], C[J][1], -u0, vb[0][0]);
        dmma(C[J][2], C[J][3], -u0, vb[1][0]);
        dmma(C[J][0], C[J][1], -u1, vb[0][1]);
        dmma(C[J][2], C[J][3], -u1, vb[1][1]);
      }
    }
  }
  // the tile (R on / above the diagonal, V below) to Y; R to the leaf's slot
  double* Ro = Rout + (int64_t)leaf * n * n;
  if (w < npan) {
#pragma unroll
    for (int J = 0; J < NG; ++J)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int r = 16 * J + 8 * (k >> 1) + 2 * q + (k & 1);
        if (c < n) {
          if (Y && r < rows) Y[(r0 + r) * ldy + c] = C[J][k];
          if (r < n) Ro[r * n + c] = (c >= r) ? C[J][k] : 0.0;
        }
      }
  }
  if (bad && flag) atomicOr(flag, 1);
}
