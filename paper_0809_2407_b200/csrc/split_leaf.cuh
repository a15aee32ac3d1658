// Split-role warp ring leaf (k_leaf_split): the C3 R-only leaf (64 < n <= 128).
//
// Same flat chain and 16-row tiles as k_leaf_dmma (Alg. 2, PAPER.md:840-866;
// each tile step is qr_triangle_on_rect, householder.py:297-332, blocked in
// 8-column panels with compact-WY updates, householder.py:175-186), but the
// two kinds of work of a tile run in DIFFERENT warps:
//
//   generation warp g (8 of them, tiles t = g, g + 8, ...): holds only the
//     current 16 x 8 panel block of its tile in registers and runs the
//     latency-bound reflector chain (dr_gen), then T (dr_form_t) and the
//     update of the next panel's block (dr_upd), i.e. everything on the
//     tile's critical path;
//   update warp u (8, paired with generation warp u): applies panel p to the
//     tile's other trailing blocks (dr_upd on fragments loaded from and stored
//     back to shared memory) one panel behind.
//
// In k_leaf_dmma one warp interleaves both, and every DMMA it issues sits in
// front of its own next dependent DFMA on the shared FP64 pipe; here the chain
// warps carry no bulk DMMA work, so 8 chains run at their latency while the
// update warps fill the pipe.  Tiles live in shared memory (8 slots of 16
// rows), R panel-packed as in k_leaf_dmma.
//
// Synchronisation (acquire/release counters, warp-uniform spins):
//   ver_pp[p]  tile t-1 finished panel p's generations (R_pp final)
//   ver_p1[p]  tile t-1 finished U(p, p+1) (R_p,p+1 final)       [gen warps]
//   ver_u[p]   tile t-1 finished U(p, >= p+2) (R_p,>=p+2 final)  [update warps]
//   yrdy[s]    slot s: Y_p and T_p published (job = 16 * local tile + p)
//   ufirst[s]  slot s: U(p, p+2) stored (the next handoff's block)
// Included by tsqr_sm100.cu (namespace tsqr), after dmma_ring.cuh.

constexpr int SP_G = 8;                    // generation warps = tiles in flight
constexpr int SP_THREADS = 2 * SP_G * 32;  // + one update warp per slot
constexpr int SP_H = 16;                   // tile rows
constexpr int SP_LD = 132;                 // tile row stride (doubles): 2-wavefront fragments

#ifdef SP_PROBE
__device__ unsigned long long g_sp_cycles[16];
#define SP_TICK(v) const long long v = clock64()
#define SP_ADD(i, a, b) \
  if (lane == 0 && blockIdx.x == 0) atomicAdd(&g_sp_cycles[i], (unsigned long long)((b) - (a)))
#else
#define SP_TICK(v)
#define SP_ADD(i, a, b)
#endif

struct SpSmem {  // offsets in doubles, then ints
  static constexpr int R = 0;
  static constexpr int TILE = R + dr_pbase<128>(16);
  static constexpr int TB = TILE + SP_G * SP_H * SP_LD;  // [slot][2 parities][32][2]
  static constexpr int GS = TB + SP_G * 2 * 64;          // [slot][72]: G 8 x 8, tau 8
  static constexpr int doubles = GS + SP_G * 72;
  static constexpr int NCNT = 3 * 16 + 2 * SP_G;
  static constexpr size_t bytes = sizeof(double) * doubles + sizeof(int) * NCNT;
};

__device__ __forceinline__ void sp_wait_ge(const int* c, int target, int lane) {
  for (;;) {
    int v = 0;
    if (lane == 0) v = ld_acquire(c);
    v = __shfl_sync(FULL, v, 0);
    if (v >= target) break;
  }
  __syncwarp();
}

// fragments of a 16 x 8 block (columns 8b..8b+7) of a tile slot, in the DMMA
// accumulator layout of C^T: x[k] = tile[8 (k >> 1) + 2q + (k & 1)][8b + g]
__device__ __forceinline__ void sp_load(double (&x)[4], const double* slot, int b, int g, int q) {
#pragma unroll
  for (int k = 0; k < 4; ++k) x[k] = slot[(8 * (k >> 1) + 2 * q + (k & 1)) * SP_LD + 8 * b + g];
}
__device__ __forceinline__ void sp_store(const double (&x)[4], double* slot, int b, int g, int q) {
#pragma unroll
  for (int k = 0; k < 4; ++k) slot[(8 * (k >> 1) + 2 * q + (k & 1)) * SP_LD + 8 * b + g] = x[k];
}
// Y^T in the B layout: vb[bb][s] = Y[8 bb + g][2q + s]
__device__ __forceinline__ void sp_load_vb(double (&vb)[2][2], const double* slot, int p, int g, int q) {
#pragma unroll
  for (int bb = 0; bb < 2; ++bb)
#pragma unroll
    for (int s = 0; s < 2; ++s) vb[bb][s] = slot[(8 * bb + g) * SP_LD + 8 * p + 2 * q + s];
}
__device__ __forceinline__ void sp_upd(double (&x)[4], const double (&y)[4], const double (&vb)[2][2],
                                       double tb0, double tb1, double* rp, int ldr) {
  double C[2][2] = {{x[0], x[1]}, {x[2], x[3]}};
  dr_upd(C, y, vb, tb0, tb1, rp, ldr);
  x[0] = C[0][0]; x[1] = C[0][1]; x[2] = C[1][0]; x[3] = C[1][1];
}

template <bool V16>
__global__ void __launch_bounds__(SP_THREADS, 1)
k_leaf_split(const double* __restrict__ A, int64_t lda, int64_t m, int n, int P, int64_t base,
             double* Rio, int* flag) {
  extern __shared__ __align__(16) double sm[];
  double* Rp = sm + SpSmem::R;
  int* cnt = reinterpret_cast<int*>(sm + SpSmem::doubles);
  int* ver_pp = cnt;
  int* ver_p1 = cnt + 16;
  int* ver_u = cnt + 32;
  int* yrdy = cnt + 48;
  int* ufirst = yrdy + SP_G;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, q = lane & 3;
  const int leaf = blockIdx.x;
  const int64_t r0 = (int64_t)leaf * base;
  const int64_t b = (leaf == P - 1) ? m - r0 : base;
  const int T = (int)((b + SP_H - 1) / SP_H);
  const int npan = (n + 7) >> 3;
  for (int i = threadIdx.x; i < SpSmem::TILE; i += SP_THREADS) Rp[i] = 0.0;  // R only: R = 0
  for (int i = threadIdx.x; i < SpSmem::NCNT; i += SP_THREADS) cnt[i] = 0;
  __syncthreads();
  const int s = w & (SP_G - 1);
  double* slot = sm + SpSmem::TILE + s * SP_H * SP_LD;
  double2* tbs = reinterpret_cast<double2*>(sm + SpSmem::TB + s * 128);
  if (w < SP_G) {
    // ============================ generation warp ============================
    double* gs = sm + SpSmem::GS + s * 72;
    double* taus = gs + 64;
    const unsigned sb = (unsigned)__cvta_generic_to_shared(slot);
    auto prefetch = [&](int t) {
      if (t >= T) return;
      const int64_t row = r0 + (int64_t)t * SP_H;
      const int rows = (int)min64(SP_H, r0 + b - row);
      const int lpr = (n * 8 + 127) / 128;
      for (int i = lane; i < rows * lpr; i += 32) {
        const double* a = A + (row + i / lpr) * lda + (i % lpr) * 16;
        asm volatile("prefetch.global.L2 [%0];" :: "l"(a));
      }
    };
    prefetch(s);
    int lt = 0;
    SP_TICK(k0_);
    for (int t = s; t < T; t += SP_G, ++lt) {
      SP_TICK(l0_);
      // tile rows into the slot (zero fill: short last tile, padded columns)
      {
        const int64_t row0 = r0 + (int64_t)t * SP_H;
        const int valid = (int)min64(SP_H, r0 + b - row0);
        if constexpr (V16) {
          for (int idx = lane; idx < SP_H * 64; idx += 32) {
            const int r = idx >> 6, c2 = idx & 63;
            const bool ok = r < valid && 2 * c2 < n;
            cp_async<16>(sb + 8u * (unsigned)(r * SP_LD + 2 * c2), ok ? A + (row0 + r) * lda + 2 * c2 : A,
                         ok ? 16u : 0u);
          }
        } else {
          for (int idx = lane; idx < SP_H * 128; idx += 32) {
            const int r = idx >> 7, c = idx & 127;
            const bool ok = r < valid && c < n;
            cp_async<8>(sb + 8u * (unsigned)(r * SP_LD + c), ok ? A + (row0 + r) * lda + c : A,
                        ok ? 8u : 0u);
          }
        }
        cp_async_commit();
        cp_async_wait<0>();
        __syncwarp();
        __threadfence_block();
      }
      prefetch(t + SP_G);
      SP_TICK(l1_);
      SP_ADD(6, l0_, l1_);
      double x[4];
      sp_load(x, slot, 0, g, q);
      for (int p = 0; p < npan; ++p) {
        const int job = lt * 16 + p;
        const int ldr = dr_ldr<128>(p);
        double* Rpan = Rp + dr_pbase<128>(p);
        double rg[8];
        SP_TICK(a0_);
        dr_wait(ver_pp + p, t, lane);
        SP_TICK(a1_);
        SP_ADD(0, a0_, a1_);
#pragma unroll
        for (int i = 0; i < 8; ++i) rg[i] = Rpan[i * ldr + g];
        dr_gen<0, false>(x, rg[0], Rpan, gs, taus);
        dr_gen<1, false>(x, rg[1], Rpan + ldr, gs, taus);
        dr_gen<2, false>(x, rg[2], Rpan + 2 * ldr, gs, taus);
        dr_gen<3, false>(x, rg[3], Rpan + 3 * ldr, gs, taus);
        dr_gen<4, false>(x, rg[4], Rpan + 4 * ldr, gs, taus);
        dr_gen<5, false>(x, rg[5], Rpan + 5 * ldr, gs, taus);
        dr_gen<6, false>(x, rg[6], Rpan + 6 * ldr, gs, taus);
        dr_gen<7, false>(x, rg[7], Rpan + 7 * ldr, gs, taus);
        dr_signal(ver_pp + p, t + 1, lane);  // R_pp final (warp barrier, then release)
        SP_TICK(a2_);
        SP_ADD(1, a1_, a2_);
        if (p + 1 >= npan) break;
        // Y_p into the slot's block p (the update warp's operand), T_p
        sp_store(x, slot, p, g, q);
        __syncwarp();
        double vb[2][2], tb0, tb1;
        sp_load_vb(vb, slot, p, g, q);
        dr_form_t(gs, taus, tb0, tb1);
        tbs[(p & 1) * 32 + lane] = make_double2(tb0, tb1);
        dr_signal(yrdy + s, job + 1, lane);
        SP_TICK(a3_);
        SP_ADD(2, a2_, a3_);
        // handoff: block p+1, updated by panel p-1 in the update warp, then by
        // panel p here (it is the next panel, on the critical path)
        if (p >= 1) sp_wait_ge(ufirst + s, job, lane);
        SP_TICK(a4_);
        SP_ADD(3, a3_, a4_);
        double c1[4];
        sp_load(c1, slot, p + 1, g, q);
        dr_wait(ver_p1 + p, t, lane);
        SP_TICK(a5_);
        SP_ADD(4, a4_, a5_);
        sp_upd(c1, x, vb, tb0, tb1, Rpan + 2 * q * ldr + 8 + g, ldr);
        dr_signal(ver_p1 + p, t + 1, lane);
        SP_TICK(a6_);
        SP_ADD(5, a5_, a6_);
#pragma unroll
        for (int k = 0; k < 4; ++k) x[k] = c1[k];
      }
    }
    SP_TICK(k1_);
    SP_ADD(7, k0_, k1_);
  } else {
    // ============================== update warp ==============================
    int lt = 0;
    for (int t = s; t < T; t += SP_G, ++lt) {
      for (int p = 0; p + 2 < npan; ++p) {
        const int job = lt * 16 + p;
        const int ldr = dr_ldr<128>(p);
        double* Rpan = Rp + dr_pbase<128>(p);
        SP_TICK(u0_);
        sp_wait_ge(yrdy + s, job + 1, lane);
        SP_TICK(u1_);
        SP_ADD(8, u0_, u1_);
        double y[4], vb[2][2];
        sp_load(y, slot, p, g, q);
        sp_load_vb(vb, slot, p, g, q);
        const double2 tb = tbs[(p & 1) * 32 + lane];
        dr_wait(ver_u + p, t, lane);
        SP_TICK(u2_);
        SP_ADD(9, u1_, u2_);
        double* rrow = Rpan + 2 * q * ldr + g;
        int bb = p + 2;
#ifdef SP_NOUPD
        bb = npan;  // probe only: skip the trailing updates (wrong R)
        dr_signal(ufirst + s, job + 1, lane);
#endif
        // two blocks at a time: independent DMMA chains side by side
        for (; bb + 1 < npan; bb += 2) {
          double c0[4], c1[4];
          sp_load(c0, slot, bb, g, q);
          sp_load(c1, slot, bb + 1, g, q);
          double C0[2][2] = {{c0[0], c0[1]}, {c0[2], c0[3]}};
          double C1[2][2] = {{c1[0], c1[1]}, {c1[2], c1[3]}};
          double* rp0 = rrow + 8 * (bb - p);
          double* rp1 = rp0 + 8;
          const double ra0 = rp0[0], ra1 = rp0[ldr], rb0 = rp1[0], rb1 = rp1[ldr];
          double wa0 = ra0, wa1 = ra1, wb0 = rb0, wb1 = rb1;
          dmma(wa0, wa1, C0[0][0], y[0]);
          dmma(wb0, wb1, C1[0][0], y[0]);
          dmma(wa0, wa1, C0[1][0], y[2]);
          dmma(wb0, wb1, C1[1][0], y[2]);
          dmma(wa0, wa1, C0[0][1], y[1]);
          dmma(wb0, wb1, C1[0][1], y[1]);
          dmma(wa0, wa1, C0[1][1], y[3]);
          dmma(wb0, wb1, C1[1][1], y[3]);
          double ua0 = 0.0, ua1 = 0.0, ub0 = 0.0, ub1 = 0.0;
          dmma(ua0, ua1, wa0, tb.x);
          dmma(ub0, ub1, wb0, tb.x);
          dmma(ua0, ua1, wa1, tb.y);
          dmma(ub0, ub1, wb1, tb.y);
          rp0[0] = ra0 - ua0;
          rp0[ldr] = ra1 - ua1;
          rp1[0] = rb0 - ub0;
          rp1[ldr] = rb1 - ub1;
          dmma(C0[0][0], C0[0][1], -ua0, vb[0][0]);
          dmma(C1[0][0], C1[0][1], -ub0, vb[0][0]);
          dmma(C0[1][0], C0[1][1], -ua0, vb[1][0]);
          dmma(C1[1][0], C1[1][1], -ub0, vb[1][0]);
          dmma(C0[0][0], C0[0][1], -ua1, vb[0][1]);
          dmma(C1[0][0], C1[0][1], -ub1, vb[0][1]);
          dmma(C0[1][0], C0[1][1], -ua1, vb[1][1]);
          dmma(C1[1][0], C1[1][1], -ub1, vb[1][1]);
          c0[0] = C0[0][0]; c0[1] = C0[0][1]; c0[2] = C0[1][0]; c0[3] = C0[1][1];
          c1[0] = C1[0][0]; c1[1] = C1[0][1]; c1[2] = C1[1][0]; c1[3] = C1[1][1];
          sp_store(c0, slot, bb, g, q);
          sp_store(c1, slot, bb + 1, g, q);
          if (bb == p + 2) dr_signal(ufirst + s, job + 1, lane);
        }
        if (bb < npan) {
          double c0[4];
          sp_load(c0, slot, bb, g, q);
          sp_upd(c0, y, vb, tb.x, tb.y, rrow + 8 * (bb - p), ldr);
          sp_store(c0, slot, bb, g, q);
          if (bb == p + 2) dr_signal(ufirst + s, job + 1, lane);
        }
        dr_signal(ver_u + p, t + 1, lane);
        SP_TICK(u3_);
        SP_ADD(10, u2_, u3_);
      }
    }
  }
  __syncthreads();
  // NaN / Inf anywhere in the leaf reaches R (see k_leaf_dmma)
  bool bad = false;
  double* Rl = Rio + (int64_t)leaf * n * n;
  for (int idx = threadIdx.x; idx < n * n; idx += SP_THREADS) {
    const int r = idx / n, c = idx - r * n;
    const int p = r >> 3;
    const double v = (c >= r) ? Rp[dr_pbase<128>(p) + (r & 7) * dr_ldr<128>(p) + (c - 8 * p)] : 0.0;
    bad |= !isfinite(v);
    Rl[idx] = v;
  }
  if (bad && flag) atomicOr(flag, 1);
}
