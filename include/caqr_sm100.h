/* caqr_sm100.h -- C-ABI of libcaqr_sm100.so, the B200 (sm_100a) FP64 TSQR/CAQR
 * hot path of arXiv:0809.2407.
 *
 * All matrix pointers are DEVICE pointers to row-major (C-order) float64 data
 * with an explicit leading dimension in elements (the reference's in-memory
 * convention, pkg/src/caqr/core.py:3-5).  All calls are asynchronous on the
 * given cudaStream_t (passed as void*), re-entrant across streams/devices,
 * and allocate no device memory: the caller owns every buffer.
 * Return value: 0 ok, 1 bad argument, 2 non-finite input, 3 CUDA error,
 * 4 communication error; tsqr_last_error() describes the last failure of the
 * calling thread.
 *
 * Reference interfaces replaced (the reference is numpy-only; these are the
 * kernels its Python API would bind through ctypes):
 *
 *   tsqr_f64_leaf_factor       <- qr_unblocked per leaf block
 *                                 (pkg/src/caqr/householder.py:128-145) composed
 *                                 with qr_triangle_on_rect (:297-332) as the
 *                                 flat in-leaf chain of Alg. 2;
 *                                 leaf blocks follow BlockRowLayout (core.py:36-61)
 *   tsqr_f64_tree_factor_level <- qr_stacked_triangles, q = 2 (householder.py:263-294)
 *                                 for every CombineEvent of one level of
 *                                 ReductionTree.schedule() (trees.py:146-152)
 *   tsqr_f64_tree_apply_level  <- apply_q / apply_qt on a STACKED factor
 *                                 (householder.py:377-396, row set :65-70), the
 *                                 inner-product update of apply_qt_structured (:335-374)
 *   tsqr_f64_leaf_apply        <- apply_q / apply_qt / explicit_q on a leaf
 *                                 (householder.py:377-404) and the compact-WY
 *                                 trailing update _apply_yt(transpose=True) (:175-186)
 *   tsqr_f64_block_factor      <- qr_unblocked (mode 0) / qr_triangle_on_rect
 *                                 (mode 2) on blocks of <= 128 rows
 *   tsqr_f64_block_apply       <- apply_q / apply_qt on those single-block factors
 *   tsqr_f64_geqr2             <- qr_unblocked of any shape (householder.py:128-145)
 *   tsqr_f64_form_t            <- form_t (householder.py:148-164)
 *                                 (householder.py:377-396)
 */
#ifndef CAQR_SM100_H
#define CAQR_SM100_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CAQR_SM100_ABI_VERSION 1

#define CAQR_OK 0
#define CAQR_ERR_ARG 1
#define CAQR_ERR_NONFINITE 2
#define CAQR_ERR_CUDA 3
#define CAQR_ERR_COMM 4

int caqr_sm100_abi_version(void);
const char* tsqr_last_error(void);

/* Kernel geometry for n columns: padded width np (32/64/128), dense first-tile
 * height h0 and chain tile height ht.  Leaf i's implicit Q is its dense tile
 * (rows [0, min(b_i, h0)), LAPACK layout: R above, Y strictly below the
 * diagonal, unit diagonal implicit) followed by ceil((b_i - h0)/ht) chain tiles
 * (TRI_ON_RECT factors whose rectangle V is stored in the tile's rows). */
int tsqr_f64_geometry(int64_t n, int64_t* np, int64_t* h0, int64_t* ht);

/* Factor the P leaves of A (m x n, 1 <= n <= 128): leaf i = rows
 * [i*floor(m/P), ...) with the last leaf absorbing the remainder.
 * R: P x n x n (slot i = leaf i's upper-triangular R).
 * Y (nullable, m x n, ldy) and tau (P x tau_stride, tile t of leaf i at
 * tau[i*tau_stride + t*n]) receive the implicit Q; pass both or neither.
 * flag (nullable, device int): OR-ed with 1 if A holds NaN/Inf. */
int tsqr_f64_leaf_factor(const double* A, int64_t lda, int64_t m, int64_t n, int64_t P,
                         double* Y, int64_t ldy, double* tau, int64_t tau_stride,
                         double* R, int* flag, void* stream);

/* R-only TSQR with the binary reduce tree (trees.py:52-66), everything on
 * device: the leaves of BlockRowLayout(m, n, P), then every tree level.  The
 * root R ends in Rslots[0] (P x n x n workspace; with more leaves than the GPU has CTA or
 * warp slots the rows are dealt to fewer, longer runs, CAQR_TUNE_FUSE below: the same R up to
 * rounding, the other slots are scratch).  tickets: device workspace
 * of P * ceil(log2 P) ints (zeroed by the call; used by the fused-tree narrow
 * path for n <= 8, may be null otherwise). */
int tsqr_f64_r_binary(const double* A, int64_t lda, int64_t m, int64_t n, int64_t P, double* Rslots,
                      int* tickets, int* flag, void* stream);

/* tsqr_f64_r_binary over leaves of `base` rows, the last taking the remainder
 * (m - (P-1) base >= base): one chunk of a larger BlockRowLayout whose base is
 * not m / P of the chunk (streamed / out-of-core TSQR; the
 * chunk's leaves must form whole subtrees of the global binary tree). */
int tsqr_f64_r_binary_rows(const double* A, int64_t lda, int64_t m, int64_t n, int64_t P,
                           int64_t base, double* Rslots, int* tickets, int* flag, void* stream);

/* One R-only combine level (events as in tsqr_f64_tree_factor_level, no node
 * factors kept) with the same arithmetic as tsqr_f64_r_binary's own tree
 * (qr_stacked_triangles, householder.py:263-294; for n <= 8 the narrow
 * path's half-step combine), so a tree split across calls gives the same R. */
int tsqr_f64_r_combine_level(double* Rslots, int64_t n, const int32_t* events, int64_t nev,
                             void* stream);

/* One level of the binary reduce tree: for every event e (int32 triples
 * {receiver, partner, node} in `events`, device memory), QR of
 * [R[receiver]; R[partner]] -> R[receiver]; node factor -> Ynode[node] (n x n
 * upper-triangular lower block of the STACKED Y) and taunode[node] (n). */
int tsqr_f64_tree_factor_level(double* Rslots, int64_t n, const int32_t* events, int64_t nev,
                               double* Ynode, double* taunode, void* stream);

/* [C_a; C_b] <- Q_node^T [C_a; C_b] (transpose=1) or Q_node [C_a; C_b] for the
 * events of one level; C_a = C + receiver*slot_rows*ldc, C_b likewise (n rows
 * each, ncols columns).  zero_partner=1 treats C_b as zero on input. */
int tsqr_f64_tree_apply_level(const double* Ynode, const double* taunode, int64_t n,
                              const int32_t* events, int64_t nev, double* C, int64_t ldc,
                              int64_t slot_rows, int64_t ncols, int transpose, int zero_partner,
                              void* stream);

/* C[leaf rows] <- Q_leaf^T C (transpose=1) or Q_leaf C for every leaf of the
 * factor (Y, tau as written by tsqr_f64_leaf_factor).  For Q only: S (nullable)
 * supplies the leaf's top n rows (leaf i at S + i*s_slot_rows*lds) instead of
 * C's own; zero_init=1 treats the rest of C as zero (explicit-Q formation);
 * tri_skip=1 skips columns known to stay zero (S upper triangular). */
int tsqr_f64_leaf_apply(const double* Y, int64_t ldy, const double* tau, int64_t tau_stride,
                        int64_t m, int64_t n, int64_t P, double* C, int64_t ldc, int64_t ncols,
                        const double* S, int64_t lds, int64_t s_slot_rows, int transpose,
                        int zero_init, int tri_skip, void* stream);

/* The CAQR trailing update with the chain tiles' panel T kept (householder.py:175-186, :209:
 * _apply_yt(transpose=True) with T from form_t, :148-164, instead of rebuilt per call).
 * tsqr_f64_leaf_factor_t is tsqr_f64_leaf_factor (Y, tau required) and also writes, for
 * every chain tile t and 8-column panel p of a leaf, T_p as 32 x 2 doubles at
 * T[((leaf * (tau_stride / n) + t + 1) * 16 + p) * 64 ..]: T needs P * (tau_stride / n) * 1024
 * doubles.  tsqr_f64_leaf_apply_t is tsqr_f64_leaf_apply(transpose = 1) reading that buffer.
 * The buffer is used when tsqr_f64_panel_t_used(n) returns 1 (n in (64, 128] with the default
 * 16-row DMMA ring kernels); otherwise both calls behave like the plain ones and T is ignored. */
int tsqr_f64_panel_t_used(int64_t n);
int tsqr_f64_leaf_factor_t(const double* A, int64_t lda, int64_t m, int64_t n, int64_t P, double* Y,
                           int64_t ldy, double* tau, int64_t tau_stride, double* R, int* flag,
                           double* T, void* stream);
int tsqr_f64_leaf_apply_t(const double* Y, int64_t ldy, const double* tau, int64_t tau_stride,
                          int64_t m, int64_t n, int64_t P, double* C, int64_t ldc, int64_t ncols,
                          const double* T, void* stream);

/* Single-CTA factorization of a block of rows <= 128: mode 0 = DENSE
 * (qr_unblocked: R out, Y m x n LAPACK layout), mode 2 = TRIRECT
 * (qr_triangle_on_rect: R in/out, Y = rectangle), mode 3 = STACKED with q-1
 * lower triangles stacked in A (qr_stacked_triangles: R = top triangle in/out). */
int tsqr_f64_block_factor(const double* A, int64_t lda, int64_t rows, int64_t n, double* R,
                          double* Y, int64_t ldy, double* tau, int mode, int* flag, void* stream);

/* qr_unblocked (householder.py:128-145) of any m x n block, in place in LAPACK
 * layout (R on/above the diagonal, reflectors v_j below it with v_j[0] = 1
 * implicit) plus tau[n]; house_gen scalars (:89-114), update skipped for tau = 0
 * (:142).  Single CTA, no shape limit: the kernel-level API beyond the
 * shared-memory block kernels (qr_unblocked / qr_blocked panels / qr_recursive
 * leaves / house_gen / stacked and triangle-on-rectangle factors). */
int tsqr_f64_geqr2(double* A, int64_t lda, int64_t m, int64_t n, double* tau, int* flag,
                   void* stream);

/* form_t (householder.py:148-164): upper-triangular T (n x n, ldt) from the Gram
 * G = Y^T Y (strict upper part read, ldg) and tau: T[j][j] = tau_j,
 * T[:j, j] = -tau_j T[:j, :j] G[:j, j], skipped when tau_j = 0. */
int tsqr_f64_form_t(const double* G, int64_t ldg, int64_t n, const double* tau, double* T,
                    int64_t ldt, void* stream);

/* Unblocked Cholesky of the Gram G = A^T A in place (upper triangle -> R with
 * G = R^T R) for the CholeskyQR competitor of the stability sweep
 * (SPEC.md:409-415); *info (device int) = j + 1 at the first nonpositive
 * pivot j, 0 on success. */
int tsqr_f64_cholesky(double* G, int64_t ldg, int64_t n, int* info, void* stream);

/* Q C / Q^T C for a single-block factor of tsqr_f64_block_factor: mode 0 =
 * DENSE (C has rows rows), mode 2 = TRIRECT (C = [Ctop (n rows, ldt); C
 * (rows rows)]); rows <= 128. */
int tsqr_f64_block_apply(const double* Y, int64_t ldy, int64_t rows, int64_t n, const double* tau,
                         double* Ctop, int64_t ldt, double* C, int64_t ldc, int64_t ncols, int mode,
                         int transpose, void* stream);

/* Process-wide tuning knobs (not thread-safe; set before launching work).
 * CAQR_TUNE_CHAIN_HT_{32,64,128}: chain tile height for padded width 32/64
 * (16 or 32) and 128 (16 or 24).  It fixes the implicit-Q format: factor and
 * apply calls on the same factor must see the same value. */
#define CAQR_TUNE_CHAIN_HT_32 1
#define CAQR_TUNE_CHAIN_HT_64 2
#define CAQR_TUNE_CHAIN_HT_128 3
/* CAQR_TUNE_NARROW: lane-private chains for n <= 8 when no Q is stored: 0 off, 1 with
 * register prefetch, 2 with cp.async shared-memory stages for 8-column rows (4 rows per
 * step), 3 (default) 8 rows per step for contiguous 16-byte-aligned 8-column rows. */
#define CAQR_TUNE_NARROW 4
/* 5: reserved (retired experimental kernel). */
/* CAQR_TUNE_ZSTART: 1 (default) = R-only leaves (no Y stored) run the chain from
 * R = 0 over all their rows instead of a dense first tile + chain. */
#define CAQR_TUNE_ZSTART 6
/* (key 8 retired: the tall-tile leaf measured slower than the DMMA ring and was removed) */
/* CAQR_TUNE_DMMA: 1 (default) = leaves with n in (64, 128] run the DMMA warp ring
 * (16-row tiles per warp in registers, 8-column Level-2 panels with look-ahead,
 * compact-WY trailing updates on the FP64 tensor cores); 2 = also n in (32, 64] (the NP = 64
 * ring, two CTAs per SM; implicit-Q leaves need CAQR_TUNE_CHAIN_HT_64 = 16); 3 = also n <= 32
 * (NP = 32 ring; no gain on C1); 0 = the rank-1 warp ring. */
#define CAQR_TUNE_DMMA 9
/* CAQR_TUNE_DMMA_APPLY: 1 (default) = Q^T C for leaves with 16-row chain tiles (the CAQR
 * trailing update) runs on the DMMA ring (compact-WY per 8-reflector panel on the FP64 tensor
 * cores): n in (64, 128] on k_leaf_apply_dmma, n <= 64 on k_leaf_q_dmma (for n in (32, 64]:
 * 64-column CTAs, two per SM; 2 = 32-column CTAs, 3 = one CTA per SM); 0 = the
 * reflector-by-reflector warp ring.  n in (64, 128]: 128-column CTAs (the dense first tile
 * column-parallel for leaves of <= 1024 rows); with the kept panel T (tsqr_f64_leaf_apply_t)
 * 64-column CTAs, two per SM, dense first tile column-parallel. */
#define CAQR_TUNE_DMMA_APPLY 10
/* CAQR_TUNE_DMMA_Q: 1 (default) = Q C (explicit Q, apply_q) for leaves with 16-row chain tiles
 * and n <= 128 runs the DMMA ring backward (compact WY per 8-reflector panel, panels in reverse
 * order); for n in (32, 64]: 2 = 32-column CTAs, 3 = one CTA per SM; 0 = the
 * reflector-by-reflector warp ring. */
#define CAQR_TUNE_DMMA_Q 11
/* CAQR_TUNE_DMMA_TREE: Q C / Q^T C of the tree nodes (STACKED factors): 2 (default) =
 * k_tree_apply_cp for n in (64, 128] (column-parallel warps, no barrier in the panel loop) and
 * k_tree_apply_dmma below; 1 = k_tree_apply_dmma for every n (compact WY per 8 reflectors, two
 * CTA barriers per panel); 0 = the reflector-by-reflector k_tree_apply / k_tree_apply_w32. */
#define CAQR_TUNE_DMMA_TREE 12
/* CAQR_TUNE_DMMA_TREE_FACTOR: 1 (default) = the q = 2 node factors (Q kept) for n <= 64 run
 * k_tree_factor_dmma (column-block warps, panels factored Level-2 by the owning warp and
 * applied in compact WY on the FP64 tensor cores); 0 = k_tree_factor / k_tree_factor_w32. */
#define CAQR_TUNE_DMMA_TREE_FACTOR 13
/* CAQR_TUNE_DMMA_DENSE: 1 = the dense first tile of leaves that keep Q, n <= 64, runs
 * k_leaf_dense_dmma (column-block warps, masked Level-2 panels, compact-WY updates on the FP64
 * tensor cores; parity-tested but slower: one warp per panel serialises the tall tile);
 * 0 (default) = the CTA sweep k_leaf_dense. */
#define CAQR_TUNE_DMMA_DENSE 14
/* CAQR_TUNE_CC: R-only leaves with n in (64, 128]: 5 (default) = the split-role ring with
 * 4 tall tiles of 64 rows held in tensor memory (k_leaf_tt<64, 1>), 6 = 8 tiles of 32 rows,
 * 4 = 16 tiles of 16 rows in tensor memory (k_leaf_tm<16>), 3 = the same with 12 tiles,
 * 2 = the split-role ring with 8 tiles in shared memory, 0 = the DMMA warp ring. */
#define CAQR_TUNE_CC 15
/* CAQR_TUNE_FUSE: R-only binary-tree TSQR with n in (64, 128] and more than `value` leaves:
 * the rows are dealt to at most `value` CTAs (default 148, one per SM) in runs of whole 64-row
 * tiles, each CTA chaining its run into one R (flat tree inside a CTA, binary tree across
 * CTAs); 0 = one CTA and one tree leaf per leaf. */
#define CAQR_TUNE_FUSE 16
/* CAQR_TUNE_NARROW_PF: how many 256-row steps ahead k_leaf_narrow8 prefetches into L2
 * (default 1: measured 1.46 ms at C4 against 1.62 / 1.99 ms for 2 / 3 steps, whose lines are
 * evicted again before they are read; 0 = no prefetch, 1.56 ms). */
#define CAQR_TUNE_NARROW_PF 17
int caqr_tune(int key, int value);

/* FP64 pipe microbenchmark (mode 0 DFMA, 1 DMMA m8n8k4). */
int caqr_f64_peak_probe(double* scratch, int mode, int iters, int blocks, void* stream);

/* Transpose-on-load: rows x cols column-major src (column c at src + c*ld_src,
 * the MAT1 on-disk order, pkg/src/caqr/matio.py:1-10) into row-major dst
 * (row r at dst + r*ld_dst), as read_mat1's reshape(order="F") (:43-51)
 * followed by the C-order layout the kernels use. */
int tsqr_f64_colmajor_to_rowmajor(const double* src, int64_t ld_src, int64_t rows, int64_t cols,
                                  double* dst, int64_t ld_dst, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* CAQR_SM100_H */
