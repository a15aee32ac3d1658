// Blocked tall-tile leaf (R only, n <= 128): the flat chain of triangle-on-
// rectangle steps (Alg. 2, householder.py:297-332) with 128-row tiles held in
// shared memory and the trailing update of each 16-column panel done as a
// compact-WY product on the FP64 tensor cores (mma.m8n8k4.f64):
//
//   panel p (warp 0):  Level-2 QR of [R_pp; C_p] -> Y_p (128 x 16), tau_p
//   G = Y^T Y, T (dlarft, V = [I; Y] so V^T V = I + G)            (warp 1)
//   W  = R_p,trail + Y^T C_trail                                    (DMMA)
//   W' = T^T W;  R_p,trail -= W';  C_trail -= Y W'                  (DMMA)
//
// One reflector generation now serves 128 rows (the ring serves 16), and the
// rank-16 updates run as tensor-core GEMMs instead of rank-1 DFMA sweeps.
// Included by tsqr_sm100.cu (namespace tsqr).

constexpr int BL_T = 128;          // tile rows
constexpr int BL_PW = 16;          // panel width
constexpr int BL_LD = 132;         // tile row stride (doubles)
constexpr int BL_RPK = 128 * 129 / 2;
constexpr int BL_WLD = 128;        // W row stride
struct BlockedSmem {
  static constexpr size_t doubles = (size_t)BL_RPK + BL_T * BL_LD + 16 * BL_WLD + 2 * 256 + 2 * 256 + 2 * 16;
  static constexpr size_t bytes = sizeof(double) * doubles;
};

__device__ __forceinline__ int bl_pk(int j, int c) { return j * 128 - (j * (j - 1)) / 2 + (c - j); }


__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(FULL, x, o);
  return x;
}

// Warp 0: Level-2 factorisation of panel p (columns pc .. pc+15) of the tile
// against the pivot rows R[pc .. pc+15] (packed, shared).  Lane l owns tile
// rows l, l+32, l+64, l+96.  On return the panel columns of Ct hold Y.
__device__ __forceinline__ void bl_panel(double* Ct, double* Rp, double* Tau, int pc, int n) {
  const int lane = threadIdx.x & 31;
  double X[4][16];
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int c = 0; c < 16; ++c) X[k][c] = Ct[(lane + 32 * k) * BL_LD + pc + c];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    // columns >= n are zero: sigma = x0 = 0 gives tau = 0 (an identity reflector),
    // so no data-dependent exit is needed (it would stop the full unroll)
    const int j = pc + i;
    double s = X[0][i] * X[0][i];
    s = fma(X[1][i], X[1][i], s);
    s = fma(X[2][i], X[2][i], s);
    s = fma(X[3][i], X[3][i], s);
    s = warp_sum(s);
    const double x0 = Rp[bl_pk(j, j)];
    double beta, tau, scale;
    house_lean(x0, s, beta, tau, scale);
    double v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = X[k][i] * scale;
    // (constant trip counts with a c > i guard: an i-dependent bound would keep
    // these loops rolled and push X / d into local memory)
    double d[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      double t = 0.0;
      if (c > i) {
        t = v[0] * X[0][c];
        t = fma(v[1], X[1][c], t);
        t = fma(v[2], X[2][c], t);
        t = fma(v[3], X[3][c], t);
      }
      d[c] = t;
    }
    // transposing butterfly: 16 partial sums x 32 lanes -> lane l holds the
    // full sum of column cl = 8 b4 + 4 b3 + 2 b2 + b1 (bits of l), 16 shuffles
    double r8[8], r4[4], r2[2];
    {
      const bool h = lane & 16;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const double snd = h ? d[k] : d[k + 8], kp = h ? d[k + 8] : d[k];
        r8[k] = kp + __shfl_xor_sync(FULL, snd, 16);
      }
    }
    {
      const bool h = lane & 8;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const double snd = h ? r8[k] : r8[k + 4], kp = h ? r8[k + 4] : r8[k];
        r4[k] = kp + __shfl_xor_sync(FULL, snd, 8);
      }
    }
    {
      const bool h = lane & 4;
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const double snd = h ? r4[k] : r4[k + 2], kp = h ? r4[k + 2] : r4[k];
        r2[k] = kp + __shfl_xor_sync(FULL, snd, 4);
      }
    }
    double r1;
    {
      const bool h = lane & 2;
      const double snd = h ? r2[0] : r2[1], kp = h ? r2[1] : r2[0];
      r1 = kp + __shfl_xor_sync(FULL, snd, 2);
    }
    r1 += __shfl_xor_sync(FULL, r1, 1);
    const int cl = ((lane >> 1) & 8) | ((lane >> 1) & 4) | ((lane >> 1) & 2) | ((lane >> 1) & 1);
    // the owner of column cl forms q = tau (R[j][c] + d) and updates R; one
    // shuffle per live column hands q to every lane for its rank-1 update
    double qmine = 0.0;
    {
      const bool live = (cl > i) && (pc + cl) < n;
      const double r = live ? Rp[bl_pk(j, pc + cl)] : 0.0;
      qmine = (cl > i) ? tau * (r + r1) : 0.0;
      if (live && !(lane & 1)) Rp[bl_pk(j, pc + cl)] = r - qmine;
    }
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      if (c <= i) continue;
      const int src = ((c & 8) << 1) | ((c & 4) << 1) | ((c & 2) << 1) | ((c & 1) << 1);
      const double q = __shfl_sync(FULL, qmine, src);
#pragma unroll
      for (int k = 0; k < 4; ++k) X[k][c] = fma(-v[k], q, X[k][c]);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) X[k][i] = v[k];
    if (lane == 0) {
      Rp[bl_pk(j, j)] = beta;
      Tau[i] = tau;
    }
  }
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int c = 0; c < 16; ++c) Ct[(lane + 32 * k) * BL_LD + pc + c] = X[k][c];
}

// Warp 1: G = Y^T Y (DMMA) and the compact-WY T (dlarft forward, columnwise,
// householder.py:148-164 with V = [I; Y]).  T is 16 x 16 row-major.
__device__ __forceinline__ void bl_form_t(const double* Ct, const double* Tau, double* G, double* T,
                                          int pc) {
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, q = lane & 3;
  double acc[2][2][2] = {};
#pragma unroll 4
  for (int k0 = 0; k0 < BL_T; k0 += 4) {
    const double* row = Ct + (k0 + q) * BL_LD + pc;
    const double a0 = row[g], a1 = row[8 + g];  // A[m][k] = Y[k][m], m = g (+8)
    dmma(acc[0][0][0], acc[0][0][1], a0, a0);
    dmma(acc[0][1][0], acc[0][1][1], a0, a1);
    dmma(acc[1][0][0], acc[1][0][1], a1, a0);
    dmma(acc[1][1][0], acc[1][1][1], a1, a1);
  }
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      G[(8 * mt + g) * 16 + 8 * nt + 2 * q] = acc[mt][nt][0];
      G[(8 * mt + g) * 16 + 8 * nt + 2 * q + 1] = acc[mt][nt][1];
    }
  __syncwarp();
  // T[l][i] = -tau_i * sum_{l <= s < i} T[l][s] G[s][i]; lane l (< 16) owns
  // row l of T in registers, G's column i is a broadcast load
  double Tr[16];
  const int l = lane & 15;
#pragma unroll
  for (int c = 0; c < 16; ++c) Tr[c] = (c == l) ? Tau[l] : 0.0;
#pragma unroll
  for (int i = 1; i < 16; ++i) {
    double z = 0.0;
#pragma unroll
    for (int s2 = 0; s2 < 16; ++s2)
      if (s2 < i) z = fma(Tr[s2], G[s2 * 16 + i], z);  // Tr[s2] = 0 for s2 < l
    if (l < i) Tr[i] = -Tau[i] * z;
  }
  if (lane < 16) {
#pragma unroll
    for (int c = 0; c < 16; ++c) T[lane * 16 + c] = Tr[c];
  }
}

__device__ __forceinline__ void bl_bar_sync(int id, int cnt) {
  asm volatile("bar.sync %0, %1;" :: "r"(id), "r"(cnt) : "memory");
}
__device__ __forceinline__ void bl_bar_arrive(int id, int cnt) {
  asm volatile("bar.arrive %0, %1;" :: "r"(id), "r"(cnt) : "memory");
}

// W' = T^T W, R_p,trail -= W', C -= Y W' for one 8-column tile (update warps)
__device__ __forceinline__ void bl_apply_tile(double* Ct, double* Rp, double* Ws, const double* T,
                                              int pc, int c0, int n) {
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, q4 = lane & 3;
  double wp[2][2] = {};
#pragma unroll
  for (int k0 = 0; k0 < 16; k0 += 4) {
    const double bfr = Ws[(k0 + q4) * BL_WLD + c0 + g];
    dmma(wp[0][0], wp[0][1], T[(k0 + q4) * 16 + g], bfr);
    dmma(wp[1][0], wp[1][1], T[(k0 + q4) * 16 + 8 + g], bfr);
  }
  __syncwarp();
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int i = 8 * mt + g, c = c0 + 2 * q4 + e;
      Ws[i * BL_WLD + c] = wp[mt][e];
      if (c < n) Rp[bl_pk(pc + i, c)] -= wp[mt][e];
    }
  __syncwarp();
  double bw[4];
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) bw[ks] = Ws[(4 * ks + q4) * BL_WLD + c0 + g];
#pragma unroll 2
  for (int mt = 0; mt < BL_T / 8; ++mt) {
    double* crow = Ct + (8 * mt + g) * BL_LD + c0 + 2 * q4;
    double d0 = crow[0], d1 = crow[1];
    const double* yrow = Ct + (8 * mt + g) * BL_LD + pc;
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) dmma(d0, d1, -yrow[4 * ks + q4], bw[ks]);
    crow[0] = d0;
    crow[1] = d1;
  }
}

// W = R_p,trail + Y^T C for one 8-column tile (update warps)
__device__ __forceinline__ void bl_w_tile(const double* Ct, const double* Rp, double* Ws, int pc,
                                          int c0) {
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, q4 = lane & 3;
  double acc[2][2];
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int c = c0 + 2 * q4 + e;
      acc[mt][e] = (c < 128) ? Rp[bl_pk(pc + 8 * mt + g, c)] : 0.0;
    }
#pragma unroll 4
  for (int k0 = 0; k0 < BL_T; k0 += 4) {
    const double* row = Ct + (k0 + q4) * BL_LD;
    const double bfr = row[c0 + g];
    dmma(acc[0][0], acc[0][1], row[pc + g], bfr);
    dmma(acc[1][0], acc[1][1], row[pc + 8 + g], bfr);
  }
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int e = 0; e < 2; ++e) Ws[(8 * mt + g) * BL_WLD + c0 + 2 * q4 + e] = acc[mt][e];
}

// Warp-specialised schedule (8 warps): warp 0 factors the panels; warps 1-7
// own the 8-column tiles c0 = 8 u (u = 0..15) with owner 1 + u % 7 and apply
// each panel's WY update, the tiles of the next panel first, so warp 0 can
// factor panel p+1 while the rest of panel p's update runs (named barriers:
// 1 = Y_p ready, 2 = T_p and W ready among the update warps, 3 = panel p+1's
// columns updated).  G and T are double-buffered by panel parity.
#ifdef BL_PROBE
__device__ unsigned long long g_bl_cycles[4];
#define BL_TICK(v) const long long v = clock64()
#define BL_ADD(i, a, b) if ((threadIdx.x & 31) == 0 && blockIdx.x == 0) atomicAdd(&g_bl_cycles[i], (unsigned long long)((b) - (a)))
#else
#define BL_TICK(v)
#define BL_ADD(i, a, b)
#endif
// Warp 4 shares warp 0's scheduler (warp w runs on sub-partition w % 4): it
// owns no tiles, so the panel factorisation has that FP64 pipe to itself.
__device__ __forceinline__ int bl_owner(int u) {
  constexpr int own[6] = {1, 2, 3, 5, 6, 7};
  return own[u % 6];
}
__global__ void __launch_bounds__(256, 1)
k_leaf_blocked(const double* __restrict__ A, int64_t lda, int64_t m, int n, int P, int64_t base,
               double* Rio, int* flag) {
  extern __shared__ __align__(16) double sm[];
  double* Rp = sm;
  double* Ct = Rp + BL_RPK;
  double* Ws = Ct + BL_T * BL_LD;
  double* Gb = Ws + 16 * BL_WLD;   // 2 x 256
  double* Tb = Gb + 512;           // 2 x 256
  double* Taub = Tb + 512;         // 2 x 16
  const int w = threadIdx.x >> 5;
  const int leaf = blockIdx.x;
  const int64_t r0 = (int64_t)leaf * base;
  const int64_t b = (leaf == P - 1) ? m - r0 : base;
  for (int i = threadIdx.x; i < BL_RPK; i += 256) Rp[i] = 0.0;
  bool bad = false;
  const int tiles = (int)((b + BL_T - 1) / BL_T);
  const int npan = (n + BL_PW - 1) / BL_PW;
  const int nut = (n + 7) >> 3;  // 8-column tiles of the matrix
  for (int t = 0; t < tiles; ++t) {
    const int64_t row0 = r0 + (int64_t)t * BL_T;
    const int valid = (int)min64((int64_t)BL_T, r0 + b - row0);
    __syncthreads();  // previous tile fully consumed
    for (int idx = threadIdx.x; idx < BL_T * 128; idx += 256) {
      const int r = idx >> 7, c = idx & 127;
      double x = 0.0;
      if (r < valid && c < n) {
        x = __ldg(A + (row0 + r) * lda + c);
        bad |= !isfinite(x);
      }
      Ct[r * BL_LD + c] = x;
    }
    __syncthreads();
    if (w == 0) {
      for (int p = 0; p < npan; ++p) {
        if (p > 0) bl_bar_sync(3, 256);  // panel p's columns carry panel p-1's update
        BL_TICK(a_);
        bl_panel(Ct, Rp, Taub + 16 * (p & 1), BL_PW * p, n);
        BL_TICK(b_);
        BL_ADD(0, a_, b_);
        bl_bar_arrive(1, 256);           // Y_p, tau_p, R_pp ready
      }
    } else {
      for (int p = 0; p < npan; ++p) {
        const int pc = BL_PW * p;
        bl_bar_sync(1, 256);
        BL_TICK(a_);
        const int u_lo = (pc + BL_PW) >> 3;  // first trailing 8-column tile
        if (u_lo >= nut) continue;            // last panel: nothing to update
        double* G = Gb + 256 * (p & 1);
        double* T = Tb + 256 * (p & 1);
        if (w == 1) bl_form_t(Ct, Taub + 16 * (p & 1), G, T, pc);
        for (int u = u_lo; u < nut; ++u)
          if (bl_owner(u) == w) bl_w_tile(Ct, Rp, Ws, pc, 8 * u);
        bl_bar_sync(2, 224);                  // T_p and every W tile ready
        BL_TICK(b_);
        BL_ADD(1, a_, b_);
        // the next panel's two tiles first, then release warp 0
        for (int u = u_lo; u < u_lo + 2 && u < nut; ++u)
          if (bl_owner(u) == w) bl_apply_tile(Ct, Rp, Ws, T, pc, 8 * u, n);
        if (p + 1 < npan) bl_bar_arrive(3, 256);
        for (int u = u_lo + 2; u < nut; ++u)
          if (bl_owner(u) == w) bl_apply_tile(Ct, Rp, Ws, T, pc, 8 * u, n);
        BL_TICK(c_);
        BL_ADD(2, b_, c_);
      }
    }
  }
  __syncthreads();
  double* Rl = Rio + (int64_t)leaf * n * n;
  for (int idx = threadIdx.x; idx < n * n; idx += 256) {
    const int r = idx / n, c = idx - r * n;
    Rl[idx] = (c >= r) ? Rp[bl_pk(r, c)] : 0.0;
  }
  if (bad && flag) atomicOr(flag, 1);
}
