// Column-parallel DMMA tree apply for 64 < n <= 128: [C_a; C_b] <- Q_node^T [C_a; C_b] (TR) or
// Q_node [C_a; C_b] for a STACKED node (qr_stacked_triangles, q = 2: reflector j = [e_j;
// Y[0..j][j]], householder.py:263-294, 335-374) -- the CAQR tree-level update and the tree walk
// of explicit Q / apply_q.
//
// k_tree_apply_dmma splits the ROWS of C_b over the warps: per 8-reflector panel the partial
// W = Y^T C_b of every warp meets in shared memory, two CTA barriers per panel, 42-50 us per
// level even for a single node (CAQR pays four or five such levels per panel on its critical
// path, and 13% of the C5 step in the trailing updates).  Here the COLUMNS are split: one
// (event, 64-column block) per CTA, warp w owns 8 columns of both C_a and C_b in registers
// (128 + 128 rows), so after the prologue -- the node's Y staged in shared memory (triangular:
// panel p has rows 0 .. 8p+7) and the 16 T_p formed once per CTA, two barriers in all -- the
// warps never meet again.  The panel loop is fully unrolled: panel p touches rows 0 .. 8p+7 of
// C_b only (4p + 6 DMMAs).
// Included by tsqr_sm100.cu (namespace tsqr) after tree_factor128.cuh.

constexpr int TAC_KB = 64;
struct TreeApplyCpSmem {
  static constexpr int LDY = 9;
  static constexpr int YS = 0;                               // panel p: rows 0 .. 8p+7, [row][LDY]
  static constexpr int TBS = YS + LDY * 8 * (16 * 17 / 2);   // [panel][lane][2]
  static constexpr int doubles = TBS + 16 * 64;
  static constexpr size_t bytes = sizeof(double) * doubles;
  __host__ __device__ static constexpr int ys_off(int p) { return LDY * 8 * (p * (p + 1) / 2); }
};

// panel P of the node on this warp's 8 columns; Ca / Cb: rows 16j + 8(k >> 1) + 2q + (k & 1)
template <int P>
__device__ __forceinline__ void tac_panel(double (&Ca)[8][4], double (&Cb)[8][4], const double* sm,
                                          int lane, int g, int q) {
  using Sm = TreeApplyCpSmem;
  constexpr int LDY = Sm::LDY;
  const double* ys = sm + Sm::YS + Sm::ys_off(P);
  const double tb0 = sm[Sm::TBS + P * 64 + 2 * lane], tb1 = sm[Sm::TBS + P * 64 + 2 * lane + 1];
  constexpr int JP = P >> 1, KP = 2 * (P & 1);  // the pivot rows 8P + 2q + e live in Ca[JP][KP + e]
  double w0 = Ca[JP][KP], w1 = Ca[JP][KP + 1], v0 = 0.0, v1 = 0.0;
#pragma unroll
  for (int rb = 0; rb <= P; ++rb) {  // 8-row blocks 0 .. P of C_b
    const double y0 = ys[(8 * rb + 2 * q) * LDY + g], y1 = ys[(8 * rb + 2 * q + 1) * LDY + g];
    dmma(w0, w1, Cb[rb >> 1][2 * (rb & 1)], y0);
    dmma(v0, v1, Cb[rb >> 1][2 * (rb & 1) + 1], y1);
  }
  w0 += v0;
  w1 += v1;
  double u0 = 0.0, u1 = 0.0;
  dmma(u0, u1, w0, tb0);
  dmma(u0, u1, w1, tb1);
  Ca[JP][KP] -= u0;
  Ca[JP][KP + 1] -= u1;
#pragma unroll
  for (int rb = 0; rb <= P; ++rb) {
    const double vb0 = ys[(8 * rb + g) * LDY + 2 * q], vb1 = ys[(8 * rb + g) * LDY + 2 * q + 1];
    dmma(Cb[rb >> 1][2 * (rb & 1)], Cb[rb >> 1][2 * (rb & 1) + 1], -u0, vb0);
    dmma(Cb[rb >> 1][2 * (rb & 1)], Cb[rb >> 1][2 * (rb & 1) + 1], -u1, vb1);
  }
}

template <bool TR>
__global__ void __launch_bounds__(THREADS, 1)
k_tree_apply_cp(const double* __restrict__ Ynode, const double* __restrict__ taunode, int n,
                const int* __restrict__ ev, double* C, int64_t ldc, int64_t slot_rows,
                int64_t ncols, int zero_partner) {
  using Sm = TreeApplyCpSmem;
  constexpr int LDY = Sm::LDY;
  extern __shared__ __align__(16) double sm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int a = ev[3 * blockIdx.x], b = ev[3 * blockIdx.x + 1], id = ev[3 * blockIdx.x + 2];
  const int64_t col0 = (int64_t)blockIdx.y * TAC_KB + 8 * w;
  const int wc = (int)min64(8, ncols - col0);  // this warp's columns (<= 0: none)
  double* Cag = C + (int64_t)a * slot_rows * ldc + col0;
  double* Cbg = C + (int64_t)b * slot_rows * ldc + col0;
  const double* Yn = Ynode + (int64_t)id * n * n;
  const double* tn = taunode + (int64_t)id * n;
  const int npan = (n + 7) >> 3;
  // the two operands' rows of this warp's columns (in flight under the prologue)
  double Ca[8][4], Cb[8][4];
#pragma unroll
  for (int j = 0; j < 8; ++j)
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int r = 16 * j + 8 * (k >> 1) + 2 * q + (k & 1);
      const bool in = r < n && g < wc;
      Ca[j][k] = in ? Cag[(int64_t)r * ldc + g] : 0.0;
      Cb[j][k] = (in && !zero_partner) ? Cbg[(int64_t)r * ldc + g] : 0.0;
    }
  // node Y -> shared memory, triangular (column c of panel p = c >> 3 has rows 0 .. 8p+7):
  // 8-byte cp.async, all in flight at once (a load-then-store loop spent ~15 us of the
  // kernel's 31 here on L2 latency)
  {
    const unsigned sb = (unsigned)__cvta_generic_to_shared(sm + Sm::YS);
    for (int idx = threadIdx.x; idx < 128 * 128; idx += THREADS) {
      const int r = idx >> 7, c = idx & 127, p = c >> 3;
      if (r < 8 * p + 8) {
        const bool ok = r < n && c < n;
        cp_async<8>(sb + 8u * (unsigned)(Sm::ys_off(p) + r * LDY + (c & 7)), ok ? Yn + (int64_t)r * n + c : Yn,
                    ok ? 8u : 0u);
      }
    }
    cp_async_commit();
    cp_async_wait<0>();
  }
  __syncthreads();
  for (int p = w; p < 16; p += WARPS) {  // T of panels w, w + 8
    const int pc = 8 * p;
    const double* ys = sm + Sm::YS + Sm::ys_off(p);
    double G[2] = {0.0, 0.0}, G2[2] = {0.0, 0.0};
    for (int rb = 0; rb <= p; ++rb) {
      const double y0 = ys[(8 * rb + 2 * q) * LDY + g], y1 = ys[(8 * rb + 2 * q + 1) * LDY + g];
      dmma(G[0], G[1], y0, y0);
      dmma(G2[0], G2[1], y1, y1);
    }
    G[0] += G2[0];
    G[1] += G2[1];
    DaPanel Pn;
    Pn.x[0] = Pn.x[1] = Pn.x[2] = Pn.x[3] = 0.0;
    Pn.tg = (pc + g < n) ? __ldg(tn + pc + g) : 0.0;
    Pn.tq0 = (pc + 2 * q < n) ? __ldg(tn + pc + 2 * q) : 0.0;
    Pn.tq1 = (pc + 2 * q + 1 < n) ? __ldg(tn + pc + 2 * q + 1) : 0.0;
    double tb0, tb1;
    da_form_t_g<TR>(Pn, G, tb0, tb1);
    sm[Sm::TBS + p * 64 + 2 * lane] = tb0;
    sm[Sm::TBS + p * 64 + 2 * lane + 1] = tb1;
  }
  __syncthreads();
  if (wc <= 0) return;
#define TAC_P(PV) if (PV < npan) tac_panel<PV>(Ca, Cb, sm, lane, g, q);
  if (TR) {
    TAC_P(0) TAC_P(1) TAC_P(2) TAC_P(3) TAC_P(4) TAC_P(5) TAC_P(6) TAC_P(7)
    TAC_P(8) TAC_P(9) TAC_P(10) TAC_P(11) TAC_P(12) TAC_P(13) TAC_P(14) TAC_P(15)
  } else {
    TAC_P(15) TAC_P(14) TAC_P(13) TAC_P(12) TAC_P(11) TAC_P(10) TAC_P(9) TAC_P(8)
    TAC_P(7) TAC_P(6) TAC_P(5) TAC_P(4) TAC_P(3) TAC_P(2) TAC_P(1) TAC_P(0)
  }
#undef TAC_P
#pragma unroll
  for (int j = 0; j < 8; ++j)
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int r = 16 * j + 8 * (k >> 1) + 2 * q + (k & 1);
      if (r < n && g < wc) {
        Cag[(int64_t)r * ldc + g] = Ca[j][k];
        Cbg[(int64_t)r * ldc + g] = Cb[j][k];
      }
    }
}
