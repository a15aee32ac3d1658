// DMMA tree factor for 64 < n <= 128: the STACKED combine [R_a; R_b] -> R with the node
// factor kept (qr_stacked_triangles, q = 2, householder.py:263-294), the column-block scheme
// of k_tree_factor_dmma (dmma_apply.cuh) with 16 warps.
//
// k_tree_factor<128> sweeps the 128 columns with the whole CTA, two barriers per reflector:
// 161 us per node (2460 cycles per column), and CAQR pays four or five such levels per panel
// on its critical path.  Here warp w owns column block w (8 columns) of R_b in registers --
// only its rows 0 .. 8w+7, R_b is upper triangular and stays so -- and of the pivot rows R_a
// (shared memory, panel-packed like the leaf kernels).  Panel p (8 reflectors over R_a's row
// and rows 0 .. 8p+7 of R_b) is factored Level-2 by warp p: the owner column goes to the other
// column groups through shared memory, the column-group sums run on one DMMA (dr_quad_sum);
// the warp publishes Y_p (triangular storage: only rows <= 8p+7) and T_p, and every warp that
// owns a later block applies the panel in compact WY on the tensor cores, block p+1 first
// (its owner then starts panel p+1).  Critical path: one panel factor + one block update per 8
// reflectors.
// Included by tsqr_sm100.cu (namespace tsqr) after tm_tall.cuh.

constexpr int TF_W = 16;  // warps = column blocks
#ifdef TF_PROBE
__device__ unsigned long long g_tf_cycles[8];
#define TF_TICK(v) const long long v = clock64()
#define TF_ADD(i, a, b) if (lane == 0 && blockIdx.x == 0) atomicAdd(&g_tf_cycles[i], (unsigned long long)((b) - (a)))
#else
#define TF_TICK(v)
#define TF_ADD(i, a, b)
#endif
struct TreeFactor128Smem {
  static constexpr int LDY = 9;
  static constexpr int RA = 0;                               // panel-packed pivot rows
  static constexpr int YS = RA + dr_pbase<128>(16);          // panel p: rows 0 .. 8p+7, [row][LDY]
  static constexpr int TBS = YS + LDY * 8 * (16 * 17 / 2);   // [panel][lane][2]
  static constexpr int GSS = TBS + 16 * 64;                  // [panel][8 x 8]
  static constexpr int TSS = GSS + 16 * 64;                  // [panel][8]
  static constexpr int XS = TSS + 16 * 8;                    // [2][128] owner column of a generation
  static constexpr int doubles = XS + 2 * 128;
  static constexpr size_t bytes = sizeof(double) * doubles + sizeof(int) * 16;
  __host__ __device__ static constexpr int ys_off(int p) { return LDY * 8 * (p * (p + 1) / 2); }
};

// Generation I of a panel over ng 16-row groups (warp-uniform count): dr_gen's arithmetic in
// the EXACT form (kept factors).  x[j][k]: row 16j + 8(k >> 1) + 2q + (k & 1), column g.  The
// owner column is read from shared memory twice (sums, then update) instead of held.
template <int I>
__device__ __forceinline__ void tf128_gen(double (&x)[8][4], int ng, double* Rrow, double* gs,
                                          double* taus, double* xs) {
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, q = lane & 3;
  double2* buf = reinterpret_cast<double2*>(xs + (I & 1) * 128) + q;  // row pair (2q, 2q+1) of a block
  if (g == I) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (j < ng) {
        buf[8 * j] = make_double2(x[j][0], x[j][1]);
        buf[8 * j + 4] = make_double2(x[j][2], x[j][3]);
      }
  }
  const double x0 = Rrow[I], rgi = Rrow[g];
  __syncwarp();
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
  for (int j = 0; j < 8; ++j)
    if (j < ng) {
      const double2 t0 = buf[8 * j], t1 = buf[8 * j + 4];
      a0 = fma(t0.x, x[j][0], a0);
      a1 = fma(t0.y, x[j][1], a1);
      a2 = fma(t1.x, x[j][2], a2);
      a3 = fma(t1.y, x[j][3], a3);
    }
  const double pd = dr_quad_sum((a0 + a1) + (a2 + a3));
  const double s = __shfl_sync(FULL, pd, 4 * I);
  double beta, tau, scale, invb;
  house_fast(x0, s, beta, tau, scale, invb);
  const double tw = fma(scale, pd, rgi);
  const double wv = tau * tw;
  const bool upd = g > I, own = (g == I);
  const double f = upd ? tw * invb : (own ? scale : 0.0);
#pragma unroll
  for (int j = 0; j < 8; ++j)
    if (j < ng) {
      const double2 t0 = buf[8 * j], t1 = buf[8 * j + 4];
      x[j][0] = fma(f, t0.x, own ? 0.0 : x[j][0]);
      x[j][1] = fma(f, t0.y, own ? 0.0 : x[j][1]);
      x[j][2] = fma(f, t1.x, own ? 0.0 : x[j][2]);
      x[j][3] = fma(f, t1.y, own ? 0.0 : x[j][3]);
    }
  double* dst = upd ? Rrow + g : (own ? Rrow + I : gs + g * 8 + I);
  *dst = upd ? rgi - wv : (own ? beta : scale * pd);
  taus[I] = tau;
}

__global__ void __launch_bounds__(TF_W * 32, 1)
k_tree_factor_dmma128(double* Rslots, int n, const int* __restrict__ ev, double* Ynode,
                      double* taunode) {
  using Sm = TreeFactor128Smem;
  constexpr int LDY = Sm::LDY;
  extern __shared__ __align__(16) double sm[];
  double* Ra = sm + Sm::RA;
  double* tbs = sm + Sm::TBS;
  double* gss = sm + Sm::GSS;
  double* tss = sm + Sm::TSS;
  double* xs = sm + Sm::XS;
  int* ver = reinterpret_cast<int*>(sm + Sm::doubles);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int a = ev[3 * blockIdx.x], b = ev[3 * blockIdx.x + 1], id = ev[3 * blockIdx.x + 2];
  const double* Rag = Rslots + (int64_t)a * n * n;
  const double* Rbg = Rslots + (int64_t)b * n * n;
  {  // R_a -> the panel-packed pivot rows (row r of panel r >> 3: columns 8 (r >> 3) .. 127), cp.async
    const unsigned sb = (unsigned)__cvta_generic_to_shared(Ra);
    for (int idx = threadIdx.x; idx < 128 * 128; idx += TF_W * 32) {
      const int r = idx >> 7, c = idx & 127, pn = r >> 3;
      if (c >= 8 * pn) {
        const bool ok = r < n && c < n && c >= r;
        cp_async<8>(sb + 8u * (unsigned)(dr_pbase<128>(pn) + (r & 7) * dr_ldr<128>(pn) + (c - 8 * pn)),
                    ok ? Rag + r * n + c : Rag, ok ? 8u : 0u);
      }
    }
    cp_async_commit();
  }
  if (threadIdx.x < 16) ver[threadIdx.x] = 0;
  // block w of R_b: rows 0 .. 8w+7 (groups 0 .. w/2), column 8w + g
  const int ngw = (w >> 1) + 1;
  double C[8][4];
#pragma unroll
  for (int j = 0; j < 8; ++j)
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int r = 16 * j + 8 * (k >> 1) + 2 * q + (k & 1), c = 8 * w + g;
      C[j][k] = (j < ngw && r < n && c < n && c >= r) ? Rbg[r * n + c] : 0.0;
    }
  cp_async_wait<0>();
  __syncthreads();
  TF_TICK(k0_);
  const int npan = (n + 7) >> 3;
  double* Yo = Ynode + (int64_t)id * n * n;
  double* to = taunode + (int64_t)id * n;
  const int pmax = (w < npan) ? w : -1;  // warps past the last panel own padding only
  for (int p = 0; p <= pmax; ++p) {
    const int pc = 8 * p;
    const int ngp = (p >> 1) + 1;  // groups holding rows 0 .. 8p+7
    const int ldr = dr_ldr<128>(p);
    double* Rpan = Ra + dr_pbase<128>(p);
    double* ys = sm + Sm::YS + Sm::ys_off(p);
    if (p == w) {  // factor panel p (my block)
      double* gs = gss + p * 64;
      double* taus = tss + p * 8;
      TF_TICK(t0_);
      tf128_gen<0>(C, ngp, Rpan, gs, taus, xs);
      tf128_gen<1>(C, ngp, Rpan + ldr, gs, taus, xs);
      tf128_gen<2>(C, ngp, Rpan + 2 * ldr, gs, taus, xs);
      tf128_gen<3>(C, ngp, Rpan + 3 * ldr, gs, taus, xs);
      tf128_gen<4>(C, ngp, Rpan + 4 * ldr, gs, taus, xs);
      tf128_gen<5>(C, ngp, Rpan + 5 * ldr, gs, taus, xs);
      tf128_gen<6>(C, ngp, Rpan + 6 * ldr, gs, taus, xs);
      tf128_gen<7>(C, ngp, Rpan + 7 * ldr, gs, taus, xs);
      TF_TICK(t1_);
      TF_ADD(0, t0_, t1_);
#pragma unroll
      for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int r = 16 * j + 8 * (k >> 1) + 2 * q + (k & 1);
          if (r < 8 * p + 8) ys[r * LDY + g] = C[j][k];  // (the node's Y goes out at the end, from here)
        }
      __syncwarp();
      double tb0, tb1;
      dr_form_t(gs, taus, tb0, tb1);
      tbs[p * 64 + 2 * lane] = tb0;
      tbs[p * 64 + 2 * lane + 1] = tb1;
      if (lane < 8 && pc + lane < n) to[pc + lane] = taus[lane];
      dr_signal(ver + p, 1, lane);
      TF_TICK(t2_);
      TF_ADD(1, t1_, t2_);
    } else {  // apply panel p to my block (w > p): Y_p is zero below row 8p+7
      // the next panel's owner polls; the other 14 warps back off (their spin loops --
      // LDS + SHFL + branch -- otherwise share the sub-partitions with the owner's chain)
      if (w != p + 1) {
        for (;;) {
          int v = 0;
          if (lane == 0) v = ld_acquire(ver + p);
          v = __shfl_sync(FULL, v, 0);
          if (v == 1) break;
          __nanosleep(200);
        }
        __syncwarp();
      } else {
        dr_wait(ver + p, 1, lane);
      }
      TF_TICK(t3_);
      const double tb0 = tbs[p * 64 + 2 * lane], tb1 = tbs[p * 64 + 2 * lane + 1];
      double* rp = Rpan + (2 * q) * ldr + 8 * (w - p) + g;
      const double ro0 = rp[0], ro1 = rp[ldr];
      double w0 = ro0, w1 = ro1, v0 = 0.0, v1 = 0.0;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j < ngp) {
#pragma unroll
          for (int k = 0; k < 4; k += 2) {
            const int r0 = 16 * j + 8 * (k >> 1) + 2 * q;
            const double y0 = (r0 < 8 * p + 8) ? ys[r0 * LDY + g] : 0.0;
            const double y1 = (r0 < 8 * p + 8) ? ys[(r0 + 1) * LDY + g] : 0.0;
            dmma(w0, w1, C[j][k], y0);
            dmma(v0, v1, C[j][k + 1], y1);
          }
        }
      w0 += v0;
      w1 += v1;
      double u0 = 0.0, u1 = 0.0;
      dmma(u0, u1, w0, tb0);
      dmma(u0, u1, w1, tb1);
      rp[0] = ro0 - u0;
      rp[ldr] = ro1 - u1;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j < ngp) {
#pragma unroll
          for (int bb = 0; bb < 2; ++bb) {
            const int r = 16 * j + 8 * bb + g;
            const bool in = r < 8 * p + 8;
            const double vb0 = in ? ys[r * LDY + 2 * q] : 0.0;
            const double vb1 = in ? ys[r * LDY + 2 * q + 1] : 0.0;
            dmma(C[j][2 * bb], C[j][2 * bb + 1], -u0, vb0);
            dmma(C[j][2 * bb], C[j][2 * bb + 1], -u1, vb1);
          }
        }
      TF_TICK(t4_);
      if (w == p + 1) TF_ADD(2, t3_, t4_);
    }
  }
  __syncthreads();
  TF_TICK(k1_);
  if (w == 0) TF_ADD(3, k0_, k1_);
  double* Ro = Rslots + (int64_t)a * n * n;
  for (int idx = threadIdx.x; idx < n * n; idx += TF_W * 32) {
    const int r = idx / n, c = idx - r * n;
    const int pn = r >> 3, pcn = c >> 3;
    Ro[idx] = (c >= r) ? Ra[dr_pbase<128>(pn) + (r & 7) * dr_ldr<128>(pn) + (c - 8 * pn)] : 0.0;
    // node Y, coalesced (32 scattered stores per lane from the panel owner cost 2.5 K cycles
    // per panel on the chain): Y_p is zero below row 8p+7
    Yo[idx] = (r < 8 * pcn + 8) ? sm[Sm::YS + Sm::ys_off(pcn) + r * LDY + (c & 7)] : 0.0;
  }
}
