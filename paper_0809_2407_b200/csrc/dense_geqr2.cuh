// General-shape kernels of the kernel-level API (householder.py, any m x n):
//
//   k_geqr2   qr_unblocked (householder.py:128-145) in place, LAPACK layout:
//             R on and above the diagonal, v_j below it (v_j[0] = 1 implicit),
//             tau.  Column sweep with house_gen's scalars (:89-114, IEEE
//             sqrt and division as in house_scalars) and _update_columns
//             (:117-125), skipped when tau = 0 (:142).  One CTA of 1024
//             threads, A in global memory: lanes take 32 consecutive
//             columns of a row (coalesced), warps stride the rows.  The
//             single-block kernels (<= 128 rows, shared memory) cover the
//             small shapes; this one has no shape limit and is the base of
//             qr_unblocked / qr_blocked panels / qr_recursive leaves beyond
//             them.  Exact zeros stay exact zeros, so on a stacked matrix of
//             triangles (or [R; B]) it produces the structured reflectors of
//             qr_stacked_triangles / qr_triangle_on_rect (:263-332).
//   k_form_t  form_t (householder.py:148-164): T[j][j] = tau_j and
//             T[:j, j] = -tau_j T[:j, :j] G[:j, j] with G = Y^T Y (the Gram is
//             one library GEMM on the Python side), nothing when tau_j = 0.
//             One CTA; threads over rows of T, columns in sequence.
// Included by tsqr_sm100.cu (namespace tsqr).

constexpr int GQ_THREADS = 1024;
constexpr int GQ_WARPS = GQ_THREADS / 32;

__global__ void __launch_bounds__(GQ_THREADS, 1)
k_geqr2(double* __restrict__ A, int64_t lda, int64_t m, int n, double* __restrict__ tau, int* flag) {
  __shared__ double red[GQ_WARPS][33];
  __shared__ double wv[32];
  __shared__ double sc[3];  // beta, tau, scale
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int kmax = (int)min64(m, n);
  bool bad = false;
  for (int j = 0; j < kmax; ++j) {
    // sigma = ||A[j+1:, j]||^2, fixed-order reduction (warps, then warp 0)
    double s = 0.0;
    for (int64_t i = j + 1 + tid; i < m; i += GQ_THREADS) {
      const double x = A[i * lda + j];
      bad |= !isfinite(x);
      s = fma(x, x, s);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
    if (lane == 0) red[w][32] = s;
    __syncthreads();
    if (w == 0) {
      double t = red[lane][32];
#pragma unroll
      for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(FULL, t, o);
      if (lane == 0) {
        const double x0 = A[(int64_t)j * lda + j];
        bad |= !isfinite(x0);
        double beta, tj, scale;
        house_scalars(x0, t, beta, tj, scale);
        sc[0] = beta;
        sc[1] = tj;
        sc[2] = scale;
        tau[j] = tj;
      }
    }
    __syncthreads();
    const double beta = sc[0], tj = sc[1], scale = sc[2];
    for (int64_t i = j + 1 + tid; i < m; i += GQ_THREADS) A[i * lda + j] *= scale;  // v below the diagonal
    if (tid == 0) A[(int64_t)j * lda + j] = beta;
    __syncthreads();
    if (tj == 0.0) continue;
    // trailing update, 32 columns per pass: w_c = A[j][c] + v^T A[j+1:, c]
    for (int c0 = j + 1; c0 < n; c0 += 32) {
      const int c = c0 + lane;
      const bool live = c < n;
      double part = 0.0;
      for (int64_t i = j + 1 + w; i < m; i += GQ_WARPS)
        part = fma(A[i * lda + j], live ? A[i * lda + c] : 0.0, part);
      red[w][lane] = part;
      __syncthreads();
      if (w == 0) {
        double t = live ? A[(int64_t)j * lda + c] : 0.0;
        for (int k = 0; k < GQ_WARPS; ++k) t += red[k][lane];
        const double q = tj * t;
        wv[lane] = q;
        if (live) A[(int64_t)j * lda + c] -= q;
      }
      __syncthreads();
      const double q = wv[lane];
      if (live)
        for (int64_t i = j + 1 + w; i < m; i += GQ_WARPS) A[i * lda + c] = fma(-q, A[i * lda + j], A[i * lda + c]);
      __syncthreads();
    }
  }
  if (bad && flag) atomicOr(flag, 1);
}

__global__ void __launch_bounds__(1024, 1)
k_form_t(const double* __restrict__ G, int64_t ldg, int n, const double* __restrict__ tau,
         double* __restrict__ T, int64_t ldt) {
  for (int64_t idx = threadIdx.x; idx < (int64_t)n * n; idx += blockDim.x) T[(idx / n) * ldt + idx % n] = 0.0;
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    const double tj = tau[j];
    if (tj != 0.0) {
      for (int i = threadIdx.x; i < j; i += blockDim.x) {
        double z = 0.0;
        for (int k = i; k < j; ++k) z = fma(T[(int64_t)i * ldt + k], G[(int64_t)k * ldg + j], z);
        T[(int64_t)i * ldt + j] = -tj * z;
      }
    }
    if (threadIdx.x == 0) T[(int64_t)j * ldt + j] = tj;
    __syncthreads();
  }
}

// Unblocked Cholesky G = R^T R (upper R, in place in the upper triangle) for
// CholeskyQR ("our own unblocked kernel with failure
// detection at nonpositive pivots").  One CTA; info = j + 1 for the first
// pivot j that is not positive (the factorization stops there), 0 on success.
__global__ void __launch_bounds__(1024, 1)
k_cholesky(double* __restrict__ G, int64_t ldg, int n, int* info) {
  __shared__ double piv;
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    if (threadIdx.x == 0) {
      const double d = G[(int64_t)j * ldg + j];
      if (!(d > 0.0)) {  // nonpositive or NaN pivot
        bad = j + 1;
      } else {
        piv = sqrt(d);
        G[(int64_t)j * ldg + j] = piv;
      }
    }
    __syncthreads();
    if (bad) break;
    const double inv = 1.0 / piv;
    for (int c = j + 1 + threadIdx.x; c < n; c += blockDim.x) G[(int64_t)j * ldg + c] *= inv;
    __syncthreads();
    // trailing update of the upper triangle: G[r][c] -= R[j][r] R[j][c], j < r <= c
    for (int64_t idx = threadIdx.x; idx < (int64_t)(n - j - 1) * (n - j - 1); idx += blockDim.x) {
      const int r = j + 1 + (int)(idx / (n - j - 1)), c = j + 1 + (int)(idx % (n - j - 1));
      if (c >= r) G[(int64_t)r * ldg + c] -= G[(int64_t)j * ldg + r] * G[(int64_t)j * ldg + c];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *info = bad;
}
