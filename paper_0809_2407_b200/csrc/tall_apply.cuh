// Leaf Q^T C / Q C for chain leaves with TALL tiles (64 rows per TRI_ON_RECT
// step, the factors k_leaf_tt<64, 1, true> keeps; n in (64, 128]) -- the CAQR
// trailing update (_apply_yt, householder.py:175-186, :209) and the explicit-Q
// / apply_q walk (householder.py:377-404).  Chain tiles only: the dense first
// tile of the leaf is applied by k_leaf_q_dmma (dense_only) before (Q^T) or
// after (Q) this kernel, through the leaf's top n rows of C.
//
// k_leaf_apply_dmma / k_leaf_q_dmma split a leaf's 16-row tiles over the warps
// of a CTA (a warp ring over the shared pivot rows); per 16 rows each warp pays
// the panel's T (14 DMMA) and T^T W (2 of every 10 DMMA per block), so at most
// 73% of the issued FP64 work is the update itself, and the ring's hand-overs
// cap the kernel near 56% of the FP64 peak.  Here the COLUMNS are split: one
// (leaf, 128-column block) per CTA, warp w owns 16 columns (two 8-column blocks)
// and every row of the leaf -- its slice of the pivot rows in shared memory is
// private, so the warps never wait on each other inside a half tile -- and
// walks the tiles in order.  Per 64-row tile, in two halves of 8 panels:
//
//   the half's Y (64 rows x 64 columns) staged in shared memory by cp.async,
//   one half ahead;
//   T of the 8 panels once per CTA (warp w: G = Y_p^T Y_p, 16 DMMA, Neumann
//   product 10), published in shared memory; two barriers per half;
//   per panel and block  W = Cs_p + Y_p^T C (16 DMMA), W' = T^T W (2),
//                        Cs_p -= W', C -= Y_p W' (16)
//   with the fragment loads of Y_p placed one between DMMAs (ta_panel).
//
// 32 of every 34 DMMA are the update.  Measured on the way here (Q^T C, 8 leaves
// of 2048 x 128 on 16256 columns): every warp reading Y_p through L1, 14-16
// TF/s; 8 columns per warp, shared-memory wavefronts at 65% of peak, 17 TF/s;
// 16 columns per warp with the fragment loads in one burst per panel, DMMA pipe
// 65%, 21 TF/s; a ninth producer warp instead of the barriers: three warps on
// one sub-partition cap the kernel at 168 registers (spills), 20 TF/s.
// Included by tsqr_sm100.cu (namespace tsqr) after dmma_apply.cuh and tm_tall.cuh.

constexpr int TLA_H = 64, TLA_K = TLA_H / 4, TLA_W = 8, TLA_KB = 16 * TLA_W;
struct TallApplySmem {
  static constexpr int YLD = 68;                      // Y row stride (doubles): 2-wavefront fragment loads
  static constexpr int YS = 0;                        // [2 halves][64][YLD]
  static constexpr int CS = YS + 2 * TLA_H * YLD;     // [warp][128][16] pivot-row slices
  static constexpr int TBS = CS + TLA_W * 128 * 16;   // [2 halves][8 panels][32 lanes][2]
  static constexpr int doubles = TBS + 2 * 8 * 64;
  static constexpr size_t bytes = sizeof(double) * doubles;
};

__device__ __forceinline__ double ta_lds(const double* p) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"((unsigned)__cvta_generic_to_shared(p)));
  return v;
}
__device__ __forceinline__ void ta_lds2(double& a, double& b, const double* p) {
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(a), "=d"(b)
               : "r"((unsigned)__cvta_generic_to_shared(p)));
}

// One panel on the warp's two blocks.  y holds this panel's fragments on entry and the next
// panel's (from ysn, nullptr: none) on return; vb is this panel's, loaded here.  The shared-
// memory loads are volatile and placed one between DMMAs: issued as a burst (24 per panel)
// they sit in front of the in-order warp's next DMMAs (measured: short_scoreboard + mio
// throttle 26% of the warp time, DMMA pipe 65%).  vb of this panel is loaded under the W
// phase, y of the next panel under the update phase (y is dead by then).
template <int K>
__device__ __forceinline__ void ta_panel(double (&c)[2][K], double (&y)[K], double tb0, double tb1,
                                         double* rp, const double* ysc, const double* ysn, int g,
                                         int q) {
  constexpr int YLD = TallApplySmem::YLD;
  double vb[K / 2][2];
  double ro[2][2], w0[2], w1[2];
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    ro[j][0] = rp[8 * j];
    ro[j][1] = rp[8 * j + 16];
    w0[j] = ro[j][0];
    w1[j] = ro[j][1];
  }
#pragma unroll
  for (int k = 0; k < K; ++k) {
#pragma unroll
    for (int j = 0; j < 2; ++j) dmma(w0[j], w1[j], c[j][k], y[k]);
    if ((k & 1) == 0) ta_lds2(vb[k >> 1][0], vb[k >> 1][1], ysc + (8 * (k >> 1) + g) * YLD + 2 * q);
  }
  double u0[2] = {0.0, 0.0}, u1[2] = {0.0, 0.0};
#pragma unroll
  for (int j = 0; j < 2; ++j) dmma(u0[j], u1[j], w0[j], tb0);
#pragma unroll
  for (int j = 0; j < 2; ++j) dmma(u0[j], u1[j], w1[j], tb1);
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    rp[8 * j] = ro[j][0] - u0[j];
    rp[8 * j + 16] = ro[j][1] - u1[j];
    u0[j] = -u0[j];
    u1[j] = -u1[j];
  }
#pragma unroll
  for (int i = 0; i < K / 2; ++i) {
#pragma unroll
    for (int j = 0; j < 2; ++j) dmma(c[j][2 * i], c[j][2 * i + 1], u0[j], vb[i][0]);
    if (ysn) y[2 * i] = ta_lds(ysn + (8 * i + 2 * q) * YLD + g);
  }
#pragma unroll
  for (int i = 0; i < K / 2; ++i) {
#pragma unroll
    for (int j = 0; j < 2; ++j) dmma(c[j][2 * i], c[j][2 * i + 1], u1[j], vb[i][1]);
    if (ysn) y[2 * i + 1] = ta_lds(ysn + (8 * i + 2 * q + 1) * YLD + g);
  }
}

template <bool TR>
__global__ void __launch_bounds__(TLA_W * 32, 1)
k_tall_apply(const double* __restrict__ Y, int64_t ldy, const double* __restrict__ tau,
             int64_t tau_stride, int64_t m, int n, int P, int64_t base, double* C, int64_t ldc,
             int64_t ncols, const double* __restrict__ S, int64_t lds, int64_t s_slot_rows,
             int zero_init, int h0) {
  using Sm = TallApplySmem;
  constexpr int K = TLA_K, YLD = Sm::YLD;
  extern __shared__ __align__(16) double sm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int leaf = blockIdx.x;
  const int64_t col0 = (int64_t)blockIdx.y * TLA_KB + 16 * w;  // this warp's 16 columns
  const int64_t r0 = (int64_t)leaf * base;
  const int64_t bl = (leaf == P - 1) ? m - r0 : base;
  const int64_t rest = bl - h0;
  const int T = rest > 0 ? (int)((rest + TLA_H - 1) / TLA_H) : 0;  // 0: only S -> C below
  const int npan = (n + 7) >> 3;
  const int nh = npan > 8 ? 2 : 1;  // halves per tile that hold panels
  const int NS = nh * T;            // steps
  const double* tl = tau + (int64_t)leaf * tau_stride;
  const double* Yl = Y + (r0 + h0) * ldy;
  double* Cl = C + r0 * ldc + col0;  // leaf row 0; chain rows from h0
  double* Cw = sm + Sm::CS + w * 128 * 16;
  double2* tbs = reinterpret_cast<double2*>(sm + Sm::TBS);
  const int wcols = (int)min64(16, ncols - col0);  // <= 0: nothing to update (still stages / forms T)
  const bool v16 = ((ldy & 1) == 0) && ((n & 1) == 0) && (((uintptr_t)Y & 15) == 0);
  // step o (walking order) = (tile, half); half h holds panels 8h .. 8h+7
  auto half_of = [&](int o) { return nh == 1 ? 0 : (TR ? (o & 1) : 1 - (o & 1)); };
  auto tile_of = [&](int o) { return TR ? o / nh : T - 1 - o / nh; };
  // Y[tile rows][64 h .. 64 h + 63] -> Ys[o & 1], zero fill below `valid` and right of n
  auto stage = [&](int o) {
    const int t = tile_of(o), c0 = 64 * half_of(o);
    const int64_t row = (int64_t)t * TLA_H;
    const int valid = (int)min64(TLA_H, rest - row);
    const double* Yt = Yl + row * ldy + c0;
    const unsigned sb = (unsigned)__cvta_generic_to_shared(sm + Sm::YS + (o & 1) * TLA_H * YLD);
    if (v16) {
      for (int idx = threadIdx.x; idx < TLA_H * 32; idx += TLA_W * 32) {
        const int r = idx >> 5, c2 = idx & 31;
        const bool ok = r < valid && c0 + 2 * c2 < n;
        cp_async<16>(sb + 8u * (unsigned)(r * YLD + 2 * c2), ok ? Yt + (int64_t)r * ldy + 2 * c2 : Y,
                     ok ? 16u : 0u);
      }
    } else {
      for (int idx = threadIdx.x; idx < TLA_H * 64; idx += TLA_W * 32) {
        const int r = idx >> 6, c = idx & 63;
        const bool ok = r < valid && c0 + c < n;
        cp_async<8>(sb + 8u * (unsigned)(r * YLD + c), ok ? Yt + (int64_t)r * ldy + c : Y, ok ? 8u : 0u);
      }
    }
    cp_async_commit();
  };
  if (NS > 0) stage(0);
  {  // pivot rows: the leaf's top n rows (Q: from the tree's block S when given)
    const double* Sl = (!TR && S) ? S + (int64_t)leaf * s_slot_rows * lds + col0 : nullptr;
    for (int idx = lane; idx < 128 * 16; idx += 32) {
      const int r = idx >> 4, c = idx & 15;
      double v = 0.0;
      if (r < n && c < wcols) v = Sl ? Sl[(int64_t)r * lds + c] : Cl[(int64_t)r * ldc + c];
      Cw[idx] = v;
    }
    __syncwarp();
  }
  double c[2][K];
  for (int o = 0; o < NS; ++o) {
    const int t = tile_of(o), hf = half_of(o);
    const int64_t row = (int64_t)t * TLA_H;  // within the chain rows
    const int valid = (int)min64(TLA_H, rest - row);
    const double* tt = tl + (int64_t)(t + 1) * n;
    const double* Ys = sm + Sm::YS + (o & 1) * TLA_H * YLD;
    double2* tb_t = tbs + (o & 1) * 8 * 32;
    const bool first = (o % nh) == 0, last = (o % nh) == nh - 1;
    const int np_h = min(8, npan - 8 * hf);
    if (wcols > 0 && first) {  // the tile's rows of C (in flight across the barrier)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const int r = 8 * (k >> 1) + 2 * q + (k & 1), cc = 8 * j + g;
          c[j][k] = (!zero_init && r < valid && cc < wcols) ? Cl[(h0 + row + r) * ldc + cc] : 0.0;
        }
    }
    cp_async_wait<0>();
    __syncthreads();  // this half's Y is in; every warp is done with the previous half (the other buffers)
    if (o + 1 < NS) stage(o + 1);
    if (w < np_h) {  // T of panel 8 hf + w
      const int pc = 8 * (8 * hf + w);
      DaPanel Pn;
      double G[2] = {0.0, 0.0}, G2[2] = {0.0, 0.0};
#pragma unroll
      for (int k = 0; k < K; k += 2) {
        const double ya = Ys[(8 * (k >> 1) + 2 * q) * YLD + 8 * w + g];
        const double yb = Ys[(8 * (k >> 1) + 2 * q + 1) * YLD + 8 * w + g];
        dmma(G[0], G[1], ya, ya);
        dmma(G2[0], G2[1], yb, yb);
      }
      G[0] += G2[0];
      G[1] += G2[1];
      Pn.x[0] = Pn.x[1] = Pn.x[2] = Pn.x[3] = 0.0;
      Pn.tg = (pc + g < n) ? __ldg(tt + pc + g) : 0.0;
      Pn.tq0 = (pc + 2 * q < n) ? __ldg(tt + pc + 2 * q) : 0.0;
      Pn.tq1 = (pc + 2 * q + 1 < n) ? __ldg(tt + pc + 2 * q + 1) : 0.0;
      double tb0, tb1;
      da_form_t_g<TR>(Pn, G, tb0, tb1);
      tb_t[w * 32 + lane] = make_double2(tb0, tb1);
    }
    __syncthreads();
    if (wcols <= 0) continue;
    double y[K];
    {
      const double* ys0 = Ys + 8 * (TR ? 0 : np_h - 1);
#pragma unroll
      for (int k = 0; k < K; ++k) y[k] = ys0[(8 * (k >> 1) + 2 * q + (k & 1)) * YLD + g];
    }
    if (np_h == 8) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int pl = TR ? i : 7 - i, p = 8 * hf + pl;
        const double2 tb = tb_t[pl * 32 + lane];
        ta_panel<K>(c, y, tb.x, tb.y, Cw + (8 * p + 2 * q) * 16 + g, Ys + 8 * pl,
                    i < 7 ? Ys + 8 * (TR ? pl + 1 : pl - 1) : nullptr, g, q);
      }
    } else {
      for (int i = 0; i < np_h; ++i) {
        const int pl = TR ? i : np_h - 1 - i, p = 8 * hf + pl;
        const double2 tb = tb_t[pl * 32 + lane];
        ta_panel<K>(c, y, tb.x, tb.y, Cw + (8 * p + 2 * q) * 16 + g, Ys + 8 * pl,
                    i + 1 < np_h ? Ys + 8 * (TR ? pl + 1 : pl - 1) : nullptr, g, q);
      }
    }
    if (last) {
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const int r = 8 * (k >> 1) + 2 * q + (k & 1), cc = 8 * j + g;
          if (r < valid && cc < wcols) Cl[(h0 + row + r) * ldc + cc] = c[j][k];
        }
    }
  }
  __syncwarp();
  if (wcols > 0) {
    for (int idx = lane; idx < n * 16; idx += 32) {
      const int r = idx >> 4, cc = idx & 15;
      if (cc < wcols) Cl[(int64_t)r * ldc + cc] = Cw[idx];
    }
  }
}
