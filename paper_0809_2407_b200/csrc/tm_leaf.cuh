// Split-role ring with the tiles in tensor memory (k_leaf_tm): the C3 R-only
// leaf (64 < n <= 128), 12 or 16 tiles in flight instead of 8.
//
// k_leaf_split (split_leaf.cuh) showed that with the reflector chains in
// their own warps the leaf is bound by how many 16-row tiles are in flight:
// each tile's 128 generations form one latency chain, and 8 tiles is what
// shared memory holds next to R.  Here the tiles live in TMEM (256 KB per SM,
// otherwise unused by an FP64 kernel): tile s is 16 rows x 128 columns = 128
// 32-bit TMEM columns of the 32 lanes of sub-partition s % 4 -- exactly the
// lane-private fragment layout of the DMMA accumulators (lane (g, q) holds
// rows 8b + 2q + e of column 8cb + g), so a block moves with one
// tcgen05.ld / tcgen05.st .32x32b.x8 per lane.
//
//   G = 12 or 16 generation warps (3 or 4 per sub-partition): tile s's
//      reflector chain (dr_gen), T, and the next panel's block (dr_upd), as in
//      k_leaf_split;
//   8 update warps (2 per sub-partition): the other trailing blocks of the
//      tiles of their sub-partition (update warp G + k serves slots k, k + 4,
//      update warp G + 4 + k slots k + 8, k + 12), polling their slots.
//
// Y_p and T_p of a slot go through shared memory (the B layout of Y^T needs
// other lanes' values); the ring counters are those of k_leaf_split.  TMEM
// hand-offs: producer tcgen05.st, tcgen05.wait::st, tcgen05.fence::
// before_thread_sync, warp barrier, release store; consumer acquire load,
// warp barrier, tcgen05.fence::after_thread_sync, tcgen05.ld, wait::ld.
// Included by tsqr_sm100.cu (namespace tsqr), after split_leaf.cuh.

constexpr int TM_U = 8;  // update warps (2 per sub-partition)
#ifndef TM_GEN
#define TM_GEN dr_gen_nx
#endif
template <int TM_G>      // generation warps = tiles in flight: 12 or 16 (TMEM holds 16)
struct TmCfg {
  static constexpr int THREADS = (TM_G + TM_U) * 32;
};

template <int TM_G>
struct TmSmem {  // offsets in doubles, then ints
  static constexpr int R = 0;
  static constexpr int YS = R + dr_pbase<128>(16);  // [slot][2 parities][16 x 8] Y_p
  static constexpr int TB = YS + TM_G * 2 * 128;     // [slot][2 parities][32][2] T
  static constexpr int GS = TB + TM_G * 2 * 64;      // [slot][72] G, tau
  static constexpr int STG = GS + TM_G * 72;         // [slot][16 x 8] next tile's block p
  static constexpr int doubles = STG + TM_G * 128;
  static constexpr int NCNT = 3 * 16 + 2 * TM_G + 4;
  static constexpr size_t bytes = sizeof(double) * doubles + sizeof(int) * NCNT;
};

__device__ __forceinline__ void tm_ld_issue(uint32_t (&r)[8], uint32_t taddr) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                 "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tm_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tm_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tm_unpack(double (&x)[4], const uint32_t (&r)[8]) {
#pragma unroll
  for (int k = 0; k < 4; ++k) x[k] = __hiloint2double((int)r[2 * k + 1], (int)r[2 * k]);
}
__device__ __forceinline__ void tm_st(uint32_t taddr, const double (&x)[4]) {
  uint32_t r[8];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    r[2 * k] = (uint32_t)__double2loint(x[k]);
    r[2 * k + 1] = (uint32_t)__double2hiint(x[k]);
  }
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};"
               :: "r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]),
                  "r"(r[6]), "r"(r[7])
               : "memory");
}
__device__ __forceinline__ void tm_ld(double (&x)[4], uint32_t taddr) {
  uint32_t r[8];
  tm_ld_issue(r, taddr);
  tm_ld_wait();
  tm_unpack(x, r);
}

template <int I>
__device__ __forceinline__ void dr_gen_nx(double (&x)[4], double rgi, double* Rrow, double* gs,
                                          double* taus) {
  dr_gen<I, false>(x, rgi, Rrow, gs, taus);
}

// Y_p of a slot in shared memory, natural 16 x 8 layout: the B operand of
// C^T Y (fragment layout) and of Y^T (vb)
__device__ __forceinline__ void tm_y_store(double* ys, const double (&x)[4], int g, int q) {
#pragma unroll
  for (int k = 0; k < 4; ++k) ys[(8 * (k >> 1) + 2 * q + (k & 1)) * 8 + g] = x[k];
}
__device__ __forceinline__ void tm_y_load(const double* ys, double (&y)[4], double (&vb)[2][2], int g,
                                          int q) {
#pragma unroll
  for (int k = 0; k < 4; ++k) y[k] = ys[(8 * (k >> 1) + 2 * q + (k & 1)) * 8 + g];
#pragma unroll
  for (int bb = 0; bb < 2; ++bb)
#pragma unroll
    for (int s = 0; s < 2; ++s) vb[bb][s] = ys[(8 * bb + g) * 8 + 2 * q + s];
}

template <int TM_G>
__global__ void __launch_bounds__(TmCfg<TM_G>::THREADS, 1)
k_leaf_tm(const double* __restrict__ A, int64_t lda, int64_t m, int n, int P, int64_t base,
          double* Rio, int* flag) {
  using TmSmem = TmSmem<TM_G>;
  constexpr int TM_THREADS = TmCfg<TM_G>::THREADS;
  extern __shared__ __align__(16) double sm[];
  double* Rp = sm + TmSmem::R;
  int* cnt = reinterpret_cast<int*>(sm + TmSmem::doubles);
  int* ver_pp = cnt;
  int* ver_p1 = cnt + 16;
  int* ver_u = cnt + 32;
  int* yrdy = cnt + 48;
  int* ufirst = yrdy + TM_G;
  uint32_t* tbase_s = reinterpret_cast<uint32_t*>(ufirst + TM_G);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, q = lane & 3;
  const int leaf = blockIdx.x;
  const int64_t r0 = (int64_t)leaf * base;
  const int64_t b = (leaf == P - 1) ? m - r0 : base;
  const int T = (int)((b + SP_H - 1) / SP_H);
  const int npan = (n + 7) >> 3;
  for (int i = threadIdx.x; i < TmSmem::YS; i += TM_THREADS) Rp[i] = 0.0;  // R only: R = 0
  for (int i = threadIdx.x; i < 3 * 16 + 2 * TM_G; i += TM_THREADS) cnt[i] = 0;
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;"
                 :: "r"((unsigned)__cvta_generic_to_shared(tbase_s)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tm_fence_before();
  __syncthreads();
  tm_fence_after();
  const uint32_t tbase = *tbase_s;
  const int sp = w & 3;  // SM sub-partition = TMEM lane quarter
  auto taddr = [&](int s, int blk) -> uint32_t {
    return tbase + ((uint32_t)(32 * (s & 3)) << 16) + (uint32_t)((s >> 2) * 128 + 8 * blk);
  };
  if (w < TM_G) {
    // ============================ generation warp ============================
    const int s = w;
    double* gs = sm + TmSmem::GS + s * 72;
    double* taus = gs + 64;
    double2* tbs = reinterpret_cast<double2*>(sm + TmSmem::TB + s * 128);
    double* stg = sm + TmSmem::STG + s * 128;
    const bool v16 = ((lda & 1) == 0) && ((n & 1) == 0) && (((uintptr_t)A & 15) == 0);
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
    for (int t = s; t < T; t += TM_G, ++lt) {
      SP_TICK(l0_);
      // tile t: block 0 into registers, blocks 1.. into the slot's TMEM columns.
      // The slot's first tile is loaded here; every later tile was staged
      // block by block during the previous tile (panel p moves block p, dead by
      // then, through shared memory by cp.async), so only block 0 is read back.
      // Loading the next tile from the update warps measured slower (52.8 ms).
      const int64_t row0 = r0 + (int64_t)t * SP_H;
      double x[4];
      if (lt > 0) tm_ld(x, taddr(s, 0));
#pragma unroll 1
      for (int blk = 0; blk < (lt > 0 ? 0 : 16); ++blk) {
        double v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int64_t row = row0 + 8 * (k >> 1) + 2 * q + (k & 1);
          const int col = 8 * blk + g;
          v[k] = (row < r0 + b && col < n) ? __ldg(A + row * lda + col) : 0.0;
        }
        if (blk == 0) {
#pragma unroll
          for (int k = 0; k < 4; ++k) x[k] = v[k];
        } else {
          tm_st(taddr(s, blk), v);
        }
      }
      tm_st_wait();
      tm_fence_before();  // published by the first yrdy release below
      prefetch(t + TM_G);
      SP_TICK(l1_);
      SP_ADD(6, l0_, l1_);
      const bool more = t + TM_G < T;
      const int64_t nrow0 = r0 + (int64_t)(t + TM_G) * SP_H;
      const int nvalid = more ? (int)min64(SP_H, r0 + b - nrow0) : 0;
      for (int p = 0; p < npan; ++p) {
        const int job = lt * 16 + p;
        const int ldr = dr_ldr<128>(p);
        double* Rpan = Rp + dr_pbase<128>(p);
        double rg[8];
        if (more) {  // next tile's block p -> shared stage (lands during this panel)
          const unsigned sb = (unsigned)__cvta_generic_to_shared(stg);
          if (v16) {
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const int x2 = lane + 32 * i, r = x2 >> 2, c2 = x2 & 3;
              const bool ok = r < nvalid && 8 * p + 2 * c2 < n;
              cp_async<16>(sb + 8u * (unsigned)(r * 8 + 2 * c2),
                           ok ? A + (nrow0 + r) * lda + 8 * p + 2 * c2 : A, ok ? 16u : 0u);
            }
          } else {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int x1 = lane + 32 * i, r = x1 >> 3, c = x1 & 7;
              const bool ok = r < nvalid && 8 * p + c < n;
              cp_async<8>(sb + 8u * (unsigned)(r * 8 + c), ok ? A + (nrow0 + r) * lda + 8 * p + c : A,
                          ok ? 8u : 0u);
            }
          }
          cp_async_commit();
        }
        SP_TICK(a0_);
        dr_wait(ver_pp + p, t, lane);
        SP_TICK(a1_);
        SP_ADD(0, a0_, a1_);
#pragma unroll
        for (int i = 0; i < 8; ++i) rg[i] = Rpan[i * ldr + g];
        TM_GEN<0>(x, rg[0], Rpan, gs, taus);
        TM_GEN<1>(x, rg[1], Rpan + ldr, gs, taus);
        TM_GEN<2>(x, rg[2], Rpan + 2 * ldr, gs, taus);
        TM_GEN<3>(x, rg[3], Rpan + 3 * ldr, gs, taus);
        TM_GEN<4>(x, rg[4], Rpan + 4 * ldr, gs, taus);
        TM_GEN<5>(x, rg[5], Rpan + 5 * ldr, gs, taus);
        TM_GEN<6>(x, rg[6], Rpan + 6 * ldr, gs, taus);
        TM_GEN<7>(x, rg[7], Rpan + 7 * ldr, gs, taus);
        dr_signal(ver_pp + p, t + 1, lane);
        if (more) {  // TMEM block p is dead (read by the hand-off of panel p-1): stage it
          cp_async_wait<0>();
          __syncwarp();
          double v[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) v[k] = stg[(8 * (k >> 1) + 2 * q + (k & 1)) * 8 + g];
          __syncwarp();
          tm_st(taddr(s, p), v);
        }
        SP_TICK(a2_);
        SP_ADD(1, a1_, a2_);
        if (p + 1 >= npan) break;
        double* ys = sm + TmSmem::YS + (s * 2 + (p & 1)) * 128;
        tm_y_store(ys, x, g, q);
        __syncwarp();
        double yv[4], vb[2][2], tb0, tb1;
        tm_y_load(ys, yv, vb, g, q);
        dr_form_t(gs, taus, tb0, tb1);
        tbs[(p & 1) * 32 + lane] = make_double2(tb0, tb1);
        dr_signal(yrdy + s, job + 1, lane);
        SP_TICK(a3_);
        SP_ADD(2, a2_, a3_);
        // hand-off: block p+1 (panel p-1 applied by the update warp), panel p here
        if (p >= 1) sp_wait_ge(ufirst + s, job, lane);
        SP_TICK(a4_);
        SP_ADD(3, a3_, a4_);
        tm_fence_after();
        double c1[4];
        tm_ld(c1, taddr(s, p + 1));
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
    const int u = w - TM_G;  // 0..7; sub-partition u & 3
    int slot[2], nsl = 0;  // slots of this sub-partition: update warp u serves the (u / 4)-th pair
    for (int i = 0; i < 2; ++i) {
      const int s2 = sp + 4 * (2 * (u >> 2) + i);
      if (s2 < TM_G) slot[nsl++] = s2;
    }
    int tt[2], lt[2], pp[2];
    for (int i = 0; i < nsl; ++i) {
      tt[i] = slot[i];
      lt[i] = 0;
      pp[i] = 0;
    }
    auto advance = [&](int i) {
      if (++pp[i] + 2 >= npan) {
        pp[i] = 0;
        ++lt[i];
        tt[i] += TM_G;
      }
    };
    if (npan < 3) nsl = 0;  // no trailing blocks beyond the next panel's
    for (;;) {
      bool any = false, did = false;
      for (int i = 0; i < nsl; ++i) {
        if (tt[i] >= T) continue;
        any = true;
        const int s = slot[i], t = tt[i], p = pp[i];
        const int job = lt[i] * 16 + p;
        int ready = 0;
        if (lane == 0) ready = (ld_acquire(yrdy + s) >= job + 1) && (ld_acquire(ver_u + p) == t);
        ready = __shfl_sync(FULL, ready, 0);
        if (!ready) continue;
        __syncwarp();
        tm_fence_after();
        did = true;
        SP_TICK(u0_);
        const int ldr = dr_ldr<128>(p);
        double* Rpan = Rp + dr_pbase<128>(p);
        double y[4], vb[2][2];
        tm_y_load(sm + TmSmem::YS + (s * 2 + (p & 1)) * 128, y, vb, g, q);
        const double2 tb = reinterpret_cast<const double2*>(sm + TmSmem::TB + s * 128)[(p & 1) * 32 + lane];
        double* rrow = Rpan + 2 * q * ldr + g;
        for (int bb = p + 2; bb < npan; ++bb) {
          double c[4];
          tm_ld(c, taddr(s, bb));
          sp_upd(c, y, vb, tb.x, tb.y, rrow + 8 * (bb - p), ldr);
          tm_st(taddr(s, bb), c);
          if (bb == p + 2) {
            tm_st_wait();
            tm_fence_before();
            dr_signal(ufirst + s, job + 1, lane);
          }
        }
        tm_st_wait();
        dr_signal(ver_u + p, t + 1, lane);
        SP_TICK(u1_);
        SP_ADD(10, u0_, u1_);
        advance(i);
      }
      if (!any) break;
      if (!did) __nanosleep(64);
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
  for (int idx = threadIdx.x; idx < n * n; idx += TM_THREADS) {
    const int r = idx / n, c = idx - r * n;
    const int pn = r >> 3;
    const double v = (c >= r) ? Rp[dr_pbase<128>(pn) + (r & 7) * dr_ldr<128>(pn) + (c - 8 * pn)] : 0.0;
    bad |= !isfinite(v);
    Rl[idx] = v;
  }
  if (bad && flag) atomicOr(flag, 1);
}
