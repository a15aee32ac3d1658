// DMMA warp-ring leaf (NP = 128: 64 < n <= 128, the C3 hot kernel; NP = 64: 32 < n <= 64;
// NP = 32 opt-in), R only or keeping the chain tiles' factors (Q).
//
// The flat chain of triangle-on-rectangle steps of a leaf (Alg. 2,
// PAPER.md:840-866; one step = qr_triangle_on_rect, householder.py:297-332)
// runs as a warp ring like k_leaf_chain -- warp w owns the 16-row tiles
// t = w, w+8, ..., the pivot rows R live in shared memory -- but every tile
// step is BLOCKED: 8-column panels are factored Level-2 inside the warp and
// the trailing update of each panel is the compact-WY product
// (householder.py:175-186 with V = [I; Y])
//
//     W  = R_p,trail + Y^T C          (4 DMMA per 8-column block)
//     W' = T^T W                      (2 DMMA)
//     R_p,trail -= W',  C -= Y W'     (4 DMMA)
//
// on the FP64 tensor cores (mma.m8n8k4.f64); T itself is a Neumann product
// on the tensor cores (dr_form_t).
//
// Register layout: the tile (16 x 128) is held as 16 x 2 blocks of 8 x 8 in
// the DMMA accumulator layout of C^T: lane (g = lane/4, q = lane%4) holds
// C[8 b + 2 q + e][8 cb + g], e = 0, 1.  With the rows of every k-step
// permuted to {2 q + s}, that same register is the A operand of C^T Y and the
// accumulator of C^T -= W'^T Y^T, so the tile never leaves registers.  The
// panel being factored is always register block 0: after each panel the
// blocks shift down by one.
//
// Look-ahead: the Level-2 of panel p+1 (block 1, once panel p has updated
// it) is interleaved generation by generation with panel p's updates of the
// other blocks, so the warp's latency-bound reflector chain and its DMMA work
// overlap.
//
// Pivot rows: R is stored panel-packed in shared memory (panel p = rows
// 8p..8p+7, columns 8p..127, row stride 130 - 8p).  Tile t may factor panel p
// once tile t-1 has (ver[p] == t); tile t-1 publishes ver[p+1] only after its
// update of R_p,trail, so the same counter also releases R_p,trail -- the ring
// of k_leaf_chain at panel granularity.
// Included by tsqr_sm100.cu (namespace tsqr).

constexpr int DR_WARPS = 8;
constexpr int DR_H = 16;            // tile rows per warp
constexpr int DR_NP = 128;          // padded width
constexpr int DR_NCB = DR_NP / 8;   // 8-column blocks
constexpr int DR_SLD = DR_NP + 2;   // staging row stride (doubles): conflict-free fragment loads
constexpr int DR_SCR = 264;         // per-warp scratch: Y^T staging 16 x 12, G 8 x 8, tau 8
// The ring kernel is built for NP = 128 (64 < n <= 128, one CTA per SM) and
// NP = 64 (32 < n <= 64: half the registers and shared memory, two CTAs per SM).
template <int NP = DR_NP>
__host__ __device__ constexpr int dr_ldr(int p) { return NP - 8 * p + 2; }
template <int NP = DR_NP>
__host__ __device__ constexpr int dr_pbase(int p) { return 8 * (p * (NP + 2) - 4 * p * (p - 1)); }
template <int NP = DR_NP>
struct DmmaRingSmem {
  static constexpr int NCB = NP / 8;
  static constexpr int SLD = NP + 2;  // conflict-free fragment loads (SLD = 2 mod 16)
  static constexpr int RP = dr_pbase<NP>(NCB);
  static constexpr int MINB = NP == 128 ? 1 : 2;  // CTAs per SM
  static constexpr size_t doubles = (size_t)RP + DR_WARPS * DR_H * SLD + DR_WARPS * DR_SCR;
  static constexpr size_t bytes = sizeof(double) * doubles + sizeof(int) * 2 * NCB;
};

// Stage tile rows [row0, row0 + valid) of A into the warp's staging buffer
// (cp.async, zero fill below `valid`); V16: 16-byte granules (n, lda even).
template <int NP, bool V16>
__device__ __forceinline__ void dr_issue(double* stage, const double* __restrict__ A, int64_t lda,
                                         int64_t row0, int valid, int n) {
  const int lane = threadIdx.x & 31;
  const unsigned sb = (unsigned)__cvta_generic_to_shared(stage);
  if constexpr (V16) {
    const int cpr = n >> 1;
#pragma unroll 4
    for (int idx = lane; idx < DR_H * NP / 2; idx += 32) {
      const int r = idx / (NP / 2), c2 = idx % (NP / 2);
      if (c2 < cpr) {
        const bool ok = r < valid;
        const double* src = ok ? A + (row0 + r) * lda + 2 * c2 : A;
        cp_async<16>(sb + 8u * (unsigned)(r * (NP + 2) + 2 * c2), src, ok ? 16u : 0u);
      }
    }
  } else {
#pragma unroll 4
    for (int idx = lane; idx < DR_H * NP; idx += 32) {
      const int r = idx / NP, c = idx % NP;
      if (c < n) {
        const bool ok = r < valid;
        const double* src = ok ? A + (row0 + r) * lda + c : A;
        cp_async<8>(sb + 8u * (unsigned)(r * (NP + 2) + c), src, ok ? 8u : 0u);
      }
    }
  }
  cp_async_commit();
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
// the slow collective path -- measured 2.2x slower).
__device__ __forceinline__ void dr_wait(const int* ver, int target, int lane) {
  for (;;) {
    int v = 0;
    if (lane == 0) v = ld_acquire(ver);
    v = __shfl_sync(FULL, v, 0);
    if (v == target) break;
  }
  __syncwarp();  // lane 0's acquire, then the warp barrier orders the other lanes' reads
}
// Publish: the warp barrier orders every lane's prior shared-memory writes before
// lane 0's release store (PTX memory model: bar.warp.sync orders memory among
// its threads, st.release makes what happens-before it visible to the acquirer).
__device__ __forceinline__ void dr_signal(int* ver, int value, int lane) {
  __syncwarp();
  if (lane == 0) st_release(ver, value);
}

// house_gen scalars (householder.py:97-113) for the panel generations, with
// the reciprocal seeded from the rsqrt seed so its MUFU latency overlaps the
// rsqrt Newton steps (two Newton steps from a ~2^-19 seed: full precision),
// plus invb = 1/beta (= -sign(x0) y; 0 when sigma = 0) so that the column
// update factor -scale * tau * t = t / beta needs no product with tau.
__device__ __forceinline__ void house_fast(double x0, double sigma, double& beta, double& tau,
                                           double& scale, double& invb) {
  const double a = fma(x0, x0, sigma);
  const double ax = fabs(x0);
  double y, r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
  const double d0 = fma(a, y, ax);
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d0));
  // one third-order step each from the ~2^-20 MUFU seeds (error e^3 ~ 2^-60;
  // tools/house_acc.cu: nrm within 2.3 ulp, 1/(|x0| + nrm) within 3.5 ulp):
  // y (1 - e)^(-1/2) ~ y (1 + e/2 + 3e^2/8), e = 1 - a y^2; r / (1 - e) ~ r (1 + e + e^2)
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
  invb = z ? 0.0 : (pos ? neg_alu(y) : y);
}

// Sum over the four lanes (g, 0..3) of a column group, result in all four: one DMMA,
// D[g][.] = sum_q A[g][q] * 1 (26 cycles), instead of two shuffle + add rounds (~72 cycles
// on the reflector chain: tools/ttg_probe.cu, 596 -> 519 cycles per generation at 64 rows).
__device__ __forceinline__ double dr_quad_sum(double v) {
  double d0 = 0.0, d1 = 0.0;
  dmma(d0, d1, v, 1.0);
  return d0;
}

// One generation (reflector I of the panel) of the register Level-2, with
// branch-free stores: every lane stores (the four lanes of a column group
// write the same value to the same address), so the look-ahead block stays
// one basic block.  rgi = R[pc+I][pc+g] (preloaded); Rrow = &R[pc+I][pc].
template <int I, bool EXACT = true>
__device__ __forceinline__ void dr_gen(double (&x)[4], double rgi, double* Rrow, double* gs,
                                       double* taus) {
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, q = lane & 3;
  const int src = 4 * I + q;
  double xi[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) xi[k] = __shfl_sync(FULL, x[k], src);
  const double x0 = __shfl_sync(FULL, rgi, 4 * I);
  // p_g = x_I . x_g over the tile; the norm sigma = p_I is the owner column's
  // own dot product (the same products in the same order as a separate sum of
  // squares, so bitwise the same), fetched with one shuffle: 7 FP64
  // instructions fewer per generation on the pipe the DMMAs share
  double pd = xi[0] * x[0], pd2 = xi[2] * x[2];
  pd = fma(xi[1], x[1], pd);
  pd2 = fma(xi[3], x[3], pd2);
  pd += pd2;
  pd = dr_quad_sum(pd);
  const double s = __shfl_sync(FULL, pd, 4 * I);
  double beta, tau, scale, invb;
  house_fast(x0, s, beta, tau, scale, invb);
  const double tw = fma(scale, pd, rgi);  // R[i][g] + v^T x_g
  const double wv = tau * tw;
  const bool upd = g > I;
  // x_g -= scale * wv * x_I for g > I (f = t / beta = -scale tau t).  The owner
  // column becomes v = scale * x_I.  EXACT: fma(scale, x_I, 0), one rounding --
  // kept factors (Q) need it: the one-FMA form x + (scale - 1) x below rounds
  // at eps |x| = eps |v| / scale, and tau (1 + |v|^2) - 2 drifts by ~eps |v|^2 /
  // scale (measured 2.9e-15 on tree nodes, where |v| ~ 1).  R-only leaves take
  // the one-FMA form (1% faster; tiles below a tall R have |v|^2 / scale < 1).
  const bool own = (g == I);
  const double f = upd ? tw * invb : (own ? (EXACT ? scale : scale - 1.0) : 0.0);
#pragma unroll
  for (int k = 0; k < 4; ++k) x[k] = fma(f, xi[k], (EXACT && own) ? 0.0 : x[k]);
  double* dst = upd ? Rrow + g : ((g == I) ? Rrow + I : gs + g * 8 + I);
  *dst = upd ? rgi - wv : ((g == I) ? beta : scale * pd);
  taus[I] = tau;
}

// T^T of the panel on the FP64 tensor cores: with S = striu(G), D = diag(tau)
// and N = D S (nilpotent), T = (I + N)^-1 D (T^-1 = D^-1 + S; equals dlarft's
// recurrence, householder.py:148-164, also when some tau = 0), so
// T^T = D P(M), M = N^T, P(M) = (I - M)(I + M^2)(I + M^4): five m8n8k4 pairs
// instead of the sequential recurrence.  Returns tb[s] = T[2q+s][g], the B
// operand of W'^T = W^T T.  Accumulator layout A: lane (g,q) holds X[g][2q+e];
// B form: X[2q+s][g] (= the accumulator layout of X^T).
__device__ __forceinline__ void dr_form_t(const double* gs, const double* taus, double& tb0,
                                           double& tb1) {
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, q = lane & 3;
  const double tg = taus[g];
  double MA[2], MB[2];
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const int c = 2 * q + e;
    MA[e] = (c < g) ? taus[c] * gs[c * 8 + g] : 0.0;  // M[g][c] = tau_c G[c][g]
    MB[e] = (g < c) ? tg * gs[g * 8 + c] : 0.0;       // M[c][g] = tau_g G[g][c]
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
  tb0 = tg * PA[0];
  tb1 = tg * PA[1];
}

// Compact-WY update (householder.py:175-186, V = [I; Y]) of one 8-column
// block (registers Cb = C[cb][.][.]) by the panel: x = Y as the B operand of
// C^T Y, vb = Y in the B layout of Y^T, tb = T in the B layout of W^T T; the
// block's pivot rows R_p,trail at rp (row stride ldr).
__device__ __forceinline__ void dr_upd(double (&Cb)[2][2], const double (&x)[4],
                                       const double (&vb)[2][2], double tb0, double tb1,
                                       double* rp, int ldr) {
  const double ro0 = rp[0], ro1 = rp[ldr];
  // one accumulation chain seeded with R_p,trail: no FP64 adds on the pipe
  double w0 = ro0, w1 = ro1;
  dmma(w0, w1, Cb[0][0], x[0]);
  dmma(w0, w1, Cb[1][0], x[2]);
  dmma(w0, w1, Cb[0][1], x[1]);
  dmma(w0, w1, Cb[1][1], x[3]);
  double u0 = 0.0, u1 = 0.0;
  dmma(u0, u1, w0, tb0);
  dmma(u0, u1, w1, tb1);
  rp[0] = ro0 - u0;
  rp[ldr] = ro1 - u1;
  dmma(Cb[0][0], Cb[0][1], -u0, vb[0][0]);
  dmma(Cb[1][0], Cb[1][1], -u0, vb[1][0]);
  dmma(Cb[0][0], Cb[0][1], -u1, vb[0][1]);
  dmma(Cb[1][0], Cb[1][1], -u1, vb[1][1]);
}

template <int NP, bool V16, bool Q>
__global__ void __launch_bounds__(DR_WARPS * 32, DmmaRingSmem<NP>::MINB)
k_leaf_dmma(const double* __restrict__ A, int64_t lda, int64_t m, int n, int P, int64_t base,
            double* Y, int64_t ldy, double* tau, int64_t tau_stride, double* Rio, int* flag,
            int h0, double* Tout = nullptr) {
  // Tout (nullable, with Y): every chain tile's panel T, as the apply kernels want it
  // (tb[s] = T[2q+s][g] per lane), at ((leaf * tau_stride / n + t + 1) * 16 + p) * 64 + 2 * lane:
  // the CAQR trailing update then reads 512 bytes per tile panel instead of rebuilding T
  // (14 of its 174 DMMAs) in every 128-column CTA.
  // h0 = 0: R only, the chain starts from R = 0 at the leaf's first row.
  // h0 > 0: the chain continues from the leaf's R slot after a dense first tile of h0 rows
  // (k_leaf_dense); Y / tau (nullable) receive each chain tile's TRI_ON_RECT factor in the
  // layout of k_leaf_chain<128, 16> (tile t: Y rows h0 + 16t.., tau at (t + 1) * n).
  // Y may alias A (tile rows are staged before they are overwritten).
  using SM = DmmaRingSmem<NP>;
  constexpr int NCB = SM::NCB, SLD = SM::SLD;
  extern __shared__ __align__(16) double sm[];
  double* Rp = sm;
  double* stage_all = Rp + SM::RP;
  double* scr_all = stage_all + DR_WARPS * DR_H * SLD;
  int* ver = reinterpret_cast<int*>(scr_all + DR_WARPS * DR_SCR);  // one counter per panel
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, q = lane & 3;
  const int leaf = blockIdx.x;
  const int64_t r0 = (int64_t)leaf * base;
  const int64_t b = (leaf == P - 1) ? m - r0 : base;
  const int64_t rest = b - h0;
  if (rest <= 0) return;  // the dense tile was the whole leaf: R is already in its slot
  const int T = (int)((rest + DR_H - 1) / DR_H);
  const int npan = (n + 7) >> 3;
  double* Rl = Rio + (int64_t)leaf * n * n;
  for (int i = threadIdx.x; i < SM::RP; i += DR_WARPS * 32) {
    double v = 0.0;
    if (Q || h0) {  // panel-packed index -> (r, c)
      int pp = 0;
      while (pp + 1 < NCB && dr_pbase<NP>(pp + 1) <= i) ++pp;
      const int off = i - dr_pbase<NP>(pp), ld = dr_ldr<NP>(pp);
      const int r = 8 * pp + off / ld, c = 8 * pp + off % ld;
      if (r < n && c < n && c >= r) v = Rl[r * n + c];
    }
    Rp[i] = v;
  }
  double* tl = tau ? tau + (int64_t)leaf * tau_stride : nullptr;
  if (threadIdx.x < 2 * NCB) ver[threadIdx.x] = 0;
  double* stage = stage_all + w * DR_H * SLD;
  double* vs = scr_all + w * DR_SCR;  // 16 x 12
  double* gs = vs + 192;
  double* taus = gs + 64;
  __syncthreads();
  bool bad = false;
  if (w < T) {
    const int64_t row = r0 + h0 + (int64_t)w * DR_H;
    dr_issue<NP, V16>(stage, A, lda, row, (int)min64(DR_H, r0 + b - row), n);
  }
  DR_TICK(k0_);
  for (int t = w; t < T; t += DR_WARPS) {
    cp_async_wait<0>();
    __syncwarp();
    double C[NCB][2][2];  // [column block][row block][e]
#pragma unroll
    for (int cb = 0; cb < NCB; ++cb)
#pragma unroll
      for (int bb = 0; bb < 2; ++bb)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = 8 * cb + g;
          double v = stage[(8 * bb + 2 * q + e) * SLD + c];
          v = (c < n) ? v : 0.0;
          C[cb][bb][e] = v;
        }
    __syncwarp();
    if (t + DR_WARPS < T) {
      const int64_t row = r0 + h0 + (int64_t)(t + DR_WARPS) * DR_H;
      dr_issue<NP, V16>(stage, A, lda, row, (int)min64(DR_H, r0 + b - row), n);
    }
    const int64_t trow = r0 + h0 + (int64_t)t * DR_H;  // this tile's first row
    const int tvalid = (int)min64(DR_H, r0 + b - trow);
    // ---- prologue: L2 of panel 0 ----
    double x[4], rg[8];
    DR_TICK(c0_);
    dr_wait(ver, t, lane);
    {
      const int l0 = dr_ldr<NP>(0);
#pragma unroll
      for (int i = 0; i < 8; ++i) rg[i] = Rp[i * l0 + g];
      x[0] = C[0][0][0]; x[1] = C[0][0][1]; x[2] = C[0][1][0]; x[3] = C[0][1][1];
      dr_gen<0, Q>(x, rg[0], Rp, gs, taus);
      dr_gen<1, Q>(x, rg[1], Rp + l0, gs, taus);
      dr_gen<2, Q>(x, rg[2], Rp + 2 * l0, gs, taus);
      dr_gen<3, Q>(x, rg[3], Rp + 3 * l0, gs, taus);
      dr_gen<4, Q>(x, rg[4], Rp + 4 * l0, gs, taus);
      dr_gen<5, Q>(x, rg[5], Rp + 5 * l0, gs, taus);
      dr_gen<6, Q>(x, rg[6], Rp + 6 * l0, gs, taus);
      dr_gen<7, Q>(x, rg[7], Rp + 7 * l0, gs, taus);
    }
    DR_TICK(c1_);
    DR_ADD(0, c0_, c1_);
    for (int p = 0; p < npan; ++p) {
      const int ldr = dr_ldr<NP>(p);
      double* Rpan = Rp + dr_pbase<NP>(p);
      DR_TICK(c2_);
      // L2(p) stored R_pp, G and tau as it went; publish R_pp
      dr_signal(ver + p, t + 1, lane);  // (__syncwarp first: gs / taus visible)
      if (Q) {  // the tile's factor for panel p: Y (= x, rows 8b+2q+e, column 8p+g) and tau
        const int c = 8 * p + g;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int tr = 8 * (k >> 1) + 2 * q + (k & 1);
          if (tr < tvalid && c < n) Y[(trow + tr) * ldy + c] = x[k];
        }
        if (lane < 8 && 8 * p + lane < n) tl[(int64_t)(t + 1) * n + 8 * p + lane] = taus[lane];
      }
      const int nl = npan - p;            // live register blocks 0 .. nl-1
      if (nl > 1) {
        double vb[2][2], tb0, tb1;
        // Y^T in the B layout of C^T -= W'^T Y^T, and T
#pragma unroll
        for (int k = 0; k < 4; ++k) vs[(8 * (k >> 1) + 2 * q + (k & 1)) * 12 + g] = x[k];
        __syncwarp();
        dr_form_t(gs, taus, tb0, tb1);
        if (Q && Tout)
          reinterpret_cast<double2*>(Tout)[((int64_t)(leaf * (tau_stride / n) + t + 1) * 16 + p) * 32 + lane] =
              make_double2(tb0, tb1);
#pragma unroll
        for (int bb = 0; bb < 2; ++bb)
#pragma unroll
          for (int s = 0; s < 2; ++s) vb[bb][s] = vs[(8 * bb + g) * 12 + 2 * q + s];
        DR_TICK(c3_);
        DR_ADD(1, c2_, c3_);
        // one wait covers both R_{p+1,p+1} and R_p,trail: tile t-1 publishes
        // ver[p+1] (after its L2(p+1)) only once its update of R_p,trail is done
        // (program order + release), so no separate counter is needed for it
        dr_wait(ver + p + 1, t, lane);
        double* rrow = Rpan + (2 * q) * ldr + g;
        // block 1 (the next panel's columns) first: it feeds L2(p+1)
        dr_upd(C[1], x, vb, tb0, tb1, rrow + 8, ldr);
        __syncwarp();  // vb reads done before the next panel's vs writes
        DR_TICK(c4_);
        DR_ADD(2, c3_, c4_);
        // ---- look-ahead block: L2(p+1) || blocks 2 .. nl-1 by panel p ----
        // (interleaved in the source: ptxas keeps this order at this register
        // pressure, so the update DMMAs run in the shadow of the reflector chain)
        const int ldr1 = dr_ldr<NP>(p + 1);
        double* Rpan1 = Rp + dr_pbase<NP>(p + 1);
#pragma unroll
        for (int i = 0; i < 8; ++i) rg[i] = Rpan1[i * ldr1 + g];
        double xn[4] = {C[1][0][0], C[1][0][1], C[1][1][0], C[1][1][1]};
#define DR_UPD(CB) \
  if constexpr ((CB) < NCB) { if ((CB) < nl) dr_upd(C[CB], x, vb, tb0, tb1, rrow + 8 * (CB), ldr); }
        dr_gen<0, Q>(xn, rg[0], Rpan1, gs, taus);
        DR_UPD(2); DR_UPD(3);
        dr_gen<1, Q>(xn, rg[1], Rpan1 + ldr1, gs, taus);
        DR_UPD(4); DR_UPD(5);
        dr_gen<2, Q>(xn, rg[2], Rpan1 + 2 * ldr1, gs, taus);
        DR_UPD(6); DR_UPD(7);
        dr_gen<3, Q>(xn, rg[3], Rpan1 + 3 * ldr1, gs, taus);
        DR_UPD(8); DR_UPD(9);
        dr_gen<4, Q>(xn, rg[4], Rpan1 + 4 * ldr1, gs, taus);
        DR_UPD(10); DR_UPD(11);
        dr_gen<5, Q>(xn, rg[5], Rpan1 + 5 * ldr1, gs, taus);
        DR_UPD(12); DR_UPD(13);
        dr_gen<6, Q>(xn, rg[6], Rpan1 + 6 * ldr1, gs, taus);
        DR_UPD(14); DR_UPD(15);
        dr_gen<7, Q>(xn, rg[7], Rpan1 + 7 * ldr1, gs, taus);
#undef DR_UPD
#pragma unroll
        for (int k = 0; k < 4; ++k) x[k] = xn[k];
        DR_TICK(c5_);
        DR_ADD(3, c4_, c5_);
      }
      if (Q && Tout && nl <= 1) {  // the last panel has no trailing block here; the update needs its T
        double tb0, tb1;
        __syncwarp();
        dr_form_t(gs, taus, tb0, tb1);
        reinterpret_cast<double2*>(Tout)[((int64_t)(leaf * (tau_stride / n) + t + 1) * 16 + p) * 32 + lane] =
            make_double2(tb0, tb1);
        __syncwarp();
      }
      // shift the register blocks: the next panel becomes block 0
#pragma unroll
      for (int cb = 0; cb + 1 < NCB; ++cb)
#pragma unroll
        for (int bb = 0; bb < 2; ++bb) {
          C[cb][bb][0] = C[cb + 1][bb][0];
          C[cb][bb][1] = C[cb + 1][bb][1];
        }
    }
  }
  DR_TICK(k1_);
  DR_ADD(5, k0_, k1_);
  __syncthreads();
  // NaN / Inf anywhere in the leaf reaches R (every entry enters a column norm
  // or a dot product, and non-finite values never become finite again), so R is
  // checked once instead of every input element on the FP64 pipe
  for (int idx = threadIdx.x; idx < n * n; idx += DR_WARPS * 32) {
    const int r = idx / n, c = idx - r * n;
    const int p = r >> 3;
    const double v = (c >= r) ? Rp[dr_pbase<NP>(p) + (r & 7) * dr_ldr<NP>(p) + (c - 8 * p)] : 0.0;
    bad |= !isfinite(v);
    Rl[idx] = v;
  }
  if (bad && flag) atomicOr(flag, 1);
}
