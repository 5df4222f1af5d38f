/*
 * skelb200 -- C ABI of the B200-native (sm_100a) level-batched recursive
 * skeletonization kernels (arXiv 2001.11619 hot path).
 *
 * The reference package (skelsolve, pure Python) has no FFI: its hot path calls
 * NumPy ufuncs and SciPy LAPACK per box.  Each entry point below replaces one of
 * those per-box call sites with ONE batched call over all boxes of a quadtree
 * level, and cites the reference file:line it replaces (paths relative to
 * /root/reference/pkg/src/skelsolve/).  The Python drop-in (package
 * paper_2001_11619_b200, module skel.py) binds these through ctypes exactly
 * as shown in INTEGRATION.md.
 *
 * Conventions
 *  - All double/int pointers inside descriptors are DEVICE pointers unless a
 *    parameter is documented as host memory.  Descriptor arrays themselves
 *    (SkbGemm*, SkbMat*, int64_t* lists of per-box sizes) are HOST memory; the
 *    library uploads them stream-ordered.
 *  - Matrices are fp64 row-major (NumPy C order) unless noted; stacks for the
 *    ID are column-major per box (each stack column contiguous).
 *  - stream is a cudaStream_t passed as void*.  Calls are stream-ordered and
 *    asynchronous; scratch is allocated with cudaMallocAsync on that stream.
 *  - Return value: 0 = OK, < 0 = -(cudaError_t), > 0 = argument error.
 *  - Numerical conditions (zero pivots, pivot ratios, ranks) are reported in
 *    per-box output arrays, never as return codes; results are deterministic
 *    and independent of batch composition (no float atomics).
 */
#ifndef SKELB200_H
#define SKELB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* D = alpha * op(A) * op(B) + beta * C, op(A) m x k, op(B) k x n, row-major.
 * transA == 0: A stored m x k (A[i*lda+p]); transA == 1: A stored k x m.
 * transB == 0: B stored k x n;              transB == 1: B stored n x k.
 * C may alias D.  beta == 0 never reads C.                                 */
typedef struct SkbGemm {
  const double* A;
  const double* B;
  const double* C;
  double* D;
  int64_t m, n, k;
  int64_t lda, ldb, ldc, ldd;
  double alpha, beta;
  int32_t transA, transB;
  int64_t tile_begin; /* filled by the library */
} SkbGemm;

/* A dense row-major matrix view. */
typedef struct SkbMat {
  double* ptr;
  int64_t rows, cols, ld;
} SkbMat;

int skb_version(void);

/* Live per-kernel-family timing with CUDA events on the launching stream
 * (families: 0 assemble, 1 geqrf, 2 qrcp, 3 id_T, 4 gemm, 5 getrf, 6 trsm,
 * 7 data movement).  skb_prof_read fills 8-entry arrays (ms summed over
 * launches, launch counts, flops/bytes registered via skb_prof_add and by the
 * GEMM itself) and optionally resets.  Off by default (zero overhead).      */
int skb_prof_enable(int32_t on);

/* CUDA-graph capture sessions: between begin and end, descriptor uploads are
 * staged through a pinned arena (allocated by begin, before the capture starts)
 * kept alive until skb_capture_release(id)
 * (id returned by skb_capture_end), so a captured graph can be replayed.     */
int skb_capture_begin(int64_t arena_bytes);
int skb_capture_end(void);
int skb_capture_release(int32_t session);

/* Host -> device copy of a small host block (level descriptors, index lists)
 * on `stream`, staged through the library's pinned ring (per-stream events
 * guard slot reuse) or, inside a capture session, its arena.  The host block
 * may be reused as soon as the call returns.  Replaces the implicit uploads
 * of the reference's NumPy arrays (skel.py:293-338 operate on host arrays).  */
int skb_h2d(const void* host, int64_t bytes, void* dev, void* stream);
int skb_prof_add(int32_t family, double flops, double bytes);
int skb_prof_read(double* ms_out, int64_t* count_out, double* flops_out, double* bytes_out,
                  int32_t reset);

/* Grouped fp64 GEMM on DMMA (mma.sync m8n8k4 f64) tiles.
 * Replaces the NumPy '@' products of skel.py:321-334, 389-396, 140-163,
 * 182, 188, 199-201, 214-215.                                               */
int skb_gemm_grouped(SkbGemm* probs, int64_t nprob, void* stream);

/* (a) ID stacks of a level batch, column-major per box with ld = rows_b,
 * rows_b = 2*nF_b + 6*P + 2, row blocks [K_in; P_in; n_in; K_out^T; P_out; n_out].
 * Replaces kernels.eval_block_pair (kernels.py:133-160), proxy_block_incoming
 * (kernels.py:307-321), proxy_block_outgoing (kernels.py:328-346),
 * nullspace_capture_rows (kernels.py:355-371) and the vstack at skel.py:306-314.
 * pos/nrm: (N,2); w: (N,); act/far: CSR DOF lists per box (device);
 * ppts/pnrm: (nbox,P,2) proxy points and radial normals; pw: (nbox,) weights;
 * stack_off: (nbox,) element offsets into stack.  FMA contraction is off so
 * entries follow NumPy's rounding order.                                    */
int skb_assemble_stack(const double* pos, const double* nrm, const double* w, int64_t nbox,
                       const int64_t* act_off, const int64_t* act, const int64_t* far_off,
                       const int64_t* far, const double* ppts, const double* pnrm,
                       const double* pw, int32_t P, const int64_t* stack_off, double* stack,
                       int64_t max_cols, int64_t max_items, void* stream);

/* (a) Self blocks E_b = A[active_b, active_b] (kernels.eval_block, kernels.py:89-130)
 * with children's Schur-complemented skeleton blocks on the diagonal
 * (_Compressor.self_block, skel.py:282-291), written in permuted order:
 * E_out[i][j] = E[perm[i]][perm[j]] (perm == NULL -> identity).
 * child_off: (nbox*5) active offsets of up to 4 children, -1 terminated;
 * child_xss: (nbox*4) device addresses of child Xss blocks (row-major k_c x k_c).
 * E_out: E_off[b] element offset, row stride E_ld[b].                       */
int skb_assemble_self(const double* pos, const double* nrm, const double* w, const double* kappa,
                      int64_t nbox, const int64_t* act_off, const int64_t* act,
                      const int64_t* perm_off, const int32_t* perm,
                      const int64_t* child_off, const int64_t* child_xss,
                      double* E, const int64_t* E_off, const int64_t* E_ld,
                      int64_t max_n, void* stream);

/* Laplace-Neumann variants (SystemSpec(LAPLACE): one DOF per node): ID stack
 * of rows 2 nF + 2 P + 2 (kernels.py:161-168, 322-325, 347-352, 368-370;
 * pnrm unused) and self blocks of the adjoint double layer with the +1
 * completion and the kappa / (4 pi) same-node limit (kernels.py:119-125).    */
int skb_assemble_stack_lap(const double* pos, const double* nrm, const double* w, int64_t nbox,
                           const int64_t* act_off, const int64_t* act, const int64_t* far_off,
                           const int64_t* far, const double* ppts, const double* pnrm,
                           const double* pw, int32_t P, const int64_t* stack_off, double* stack,
                           int64_t max_cols, int64_t max_items, void* stream);
int skb_assemble_self_lap(const double* pos, const double* nrm, const double* w,
                          const double* kappa, int64_t nbox, const int64_t* act_off,
                          const int64_t* act, const int64_t* perm_off, const int32_t* perm,
                          const int64_t* child_off, const int64_t* child_xss, double* E,
                          const int64_t* E_off, const int64_t* E_ld, int64_t max_n, void* stream);

/* (d) Stokeslet/rotlet columns H (nd x 3p) and weighted rigid-body functionals
 * Psi (nd x 3p) -- kernels.stokeslet_rotlet_columns (kernels.py:201-223) and
 * build_augmentation (kernels.py:226-246).  curve_off: (p+2,) node offsets.  */
int skb_assemble_aug(const double* pos, const double* w, int64_t n_nodes,
                     const double* hole_centers, int64_t n_holes, const int64_t* curve_off_host,
                     double* H, double* Psi, void* stream);

/* (b) Batched unpivoted Householder QR (LAPACK dgeqrf semantics, blocked
 * compact-WY, panel width 32) of column-major matrices A_b (m_b x n_b, lda_b):
 * the R factor lands in the upper triangle, the strictly lower triangle of the
 * leading min(m,n) rows is zeroed on exit (R ready for QRCP).
 * Replaces the pre-reduction sla.qr(A, mode="r") at dense.py:56-59.
 * m, n, lda, A: HOST arrays of length nbox (A as device addresses).          */
int skb_geqrf_batched(int64_t nbox, const int64_t* m, const int64_t* n, const int64_t* lda,
                      const int64_t* A, void* stream);

/* (b) Batched column-pivoted QR + interpolative decomposition with LAPACK
 * dgeqp3/dlaqp2 pivot semantics (largest partial column norm, lowest index on
 * ties, dlaqp2 norm downdating with recompute at sqrt(eps)) and the rank
 * k = #{|R_jj| > tol*|R_00|} (dense.py:65-68).  Stops once every remaining
 * partial norm is below the rank threshold (and at least kmin_b steps done).
 * Lazy pivoting: columns are not moved; perm[i] is the column chosen at step i,
 * perm[k..] lists the redundant columns (pivots past k, then the unchosen ones
 * ascending) and R(i, perm[j]) stays in A[perm[j]][i].  Large boxes are
 * spread over up to 32 co-resident CTAs (cooperative launch).
 * Replaces sla.qr(..., pivoting=True) + rank_for_tol (dense.py:48-68).
 * Host arrays: m, n, lda, A (device addresses), kmin.
 * Device outputs: perm (int32, perm_off[b] offsets), k_out (int32 per box),
 * diag (|R_jj|, at perm_off[b]), min_gap (double per box, smallest relative
 * gap between the pivot norm and the runner-up over the first k steps).     */
int skb_qrcp_id_batched(int64_t nbox, const int64_t* m, const int64_t* n, const int64_t* lda,
                        const int64_t* A, const int64_t* kmin, double tol,
                        const int64_t* perm_off_host, int32_t* perm, double* diag,
                        int32_t* k_out, int32_t* steps_out, double* min_gap, void* stream);

/* (b) T = R11^-1 R12 per box after skb_qrcp_id_batched (dense.py:77): gathers
 * the lazily pivoted R11 (k x k) / R12 (k x (n-k)) from the column-major A_b
 * via the device perm_b and solves in place into row-major T_b (k x (n-k)).
 * A, lda, k, n, perm_dev (device int32 addresses), T: HOST arrays.            */
int skb_id_T_batched(int64_t nbox, const int64_t* A, const int64_t* lda, const int64_t* k,
                     const int64_t* n, const int64_t* perm_dev, const int64_t* T, void* stream);

/* Batched 2-D copy: dst_b[i][j] = src_b[i][j] (trans == 0) or src_b[j][i]
 * (trans == 1, src stored cols x rows), for i < rows_b, j < cols_b.
 * dst/src: HOST arrays of SkbMat (device pointers; rows/cols of dst used). */
int skb_copy2d_batched(int64_t nbox, const SkbMat* dst, const SkbMat* src, int32_t trans,
                       void* stream);

/* (c) Batched LU with partial pivoting of row-major n_b x n_b matrices (in
 * place), LAPACK dgetrf semantics (largest |a| in the column, first on ties),
 * blocked (panel 64; trailing update on the grouped DMMA GEMM).  ipiv: 0-based
 * row interchanges (int32).  info_out[b] = first exact zero pivot index or -1;
 * ratio_out[b] = min|u_ii| / max|u_ii| (1.0 for n == 0).
 * Replaces sla.lu_factor + pivot_ratio (dense.py:113-127).
 * a: HOST array of SkbMat (square); ipiv: HOST array of device int32 addrs.  */
int skb_getrf_batched(int64_t nbox, const SkbMat* a, const int64_t* ipiv, int32_t* info_out,
                      double* ratio_out, void* stream);

/* (c) Batched LU solve B_b <- A_b^-1 B_b with factors from skb_getrf_batched
 * (trans == 0) -- sla.lu_solve, dense.py:129-135.  b: HOST SkbMat array,
 * rows must equal the LU order.                                             */
int skb_getrs_batched(int64_t nbox, const SkbMat* lu, const int64_t* ipiv, const SkbMat* b,
                      void* stream);

/* Row gather/scatter by DOF lists: the NumPy fancy indexing x[dofs] of
 * skel.py:140-163, 180-221, 384-396.  For box b, local row i < cnt_b:
 *   gather : dst[dst_off[b] + i*dst_ld[b] + c] = src[idx[i]*src_ld + col[c]]
 *   scatter: dst[idx[i]*dst_ld_g + col[c]] = src[src_off[b] + i*src_ld[b] + c]
 * for c < ncol_b; col == NULL means col[c] = c.  idx lists are CSR (idx_off,
 * idx); col lists CSR (col_off, col) or NULL with ncol uniform (ncols).
 * Device arrays throughout; max_rows/max_cols (host scalars) size the grid.
 * accumulate != 0 in scatter adds instead of storing (alpha * src).         */
int skb_gather_rows(int64_t nbox, const int64_t* idx_off, const int64_t* idx,
                    const int64_t* col_off, const int64_t* col, int64_t ncols,
                    const double* src, int64_t src_ld, double* dst, const int64_t* dst_off,
                    const int64_t* dst_ld, int64_t max_rows, int64_t max_cols, void* stream);
int skb_scatter_rows(int64_t nbox, const int64_t* idx_off, const int64_t* idx,
                     const int64_t* col_off, const int64_t* col, int64_t ncols,
                     const double* src, const int64_t* src_off, const int64_t* src_ld,
                     double* dst, int64_t dst_ld, int32_t accumulate, double alpha,
                     int64_t max_rows, int64_t max_cols, void* stream);

/* (d) Deterministic accumulation of per-box Schur partials into the q x q
 * augmentation corner (skel.py:396: schur += PsiV[rd]^T w, box order kept):
 *   schur[row][c] += sum over contributions t of row (CSR row_off/contrib, in
 *   box order) of part[contrib[t] + c], c < q.                              */
int skb_schur_accumulate(int64_t q, const int64_t* row_off, const int64_t* contrib,
                         const double* part, double* schur, void* stream);

/* Column-sparse, compensated Psi^T z (skel.py:182 corr = lam - PsiV[nonroot]^T x,
 * skel.py:142 bottom = PsiV^T y - lam): PsiV rows are nonzero only in the hole
 * columns of the box that eliminated them, so column c sums over its row list
 * (CSR col_off/rows, list order) with TwoSum/TwoProduct (double-double) accuracy:
 *   out[c][j] = C[c][j] + alpha * sum_t psi[rows[t]][c] * z[rows[t]][j].        */
int skb_psi_dot(int64_t q, const int64_t* col_off, const int64_t* rows, const double* psi,
                int64_t ldp, const double* z, int64_t ldz, int64_t nrhs, const double* C,
                int64_t ldc, double alpha, double* out, int64_t ldo, void* stream);

/* Deterministic split-K reduction: D[e] = C[e] + alpha * sum_p parts[p*stride + e]
 * (fixed order; C may be NULL) for e < count -- the second pass of the split-K
 * products with K = 2N (PsiV^T x of skel.py:182).                              */
int skb_sum_partials(int64_t count, int32_t nparts, const double* parts, int64_t stride,
                     const double* C, double alpha, double* D, void* stream);

/* Fill dst (n x n, ld) with diag_val*I + scale*src (src may be NULL). */
int skb_diag_fill(int64_t n, double* dst, int64_t ld, double diag_val, const double* src,
                  int64_t src_ld, double scale, void* stream);

/* Exact augmented system product y = M x by direct summation (reference
 * kernels.system_matvec, kernels.py:393-414): y[:2N] = (-1/2 I + D + N) mu + H lam,
 * y[2N:] = Psi^T mu - lam.  x, y: (2N + 3p) x nrhs row-major; curve_off_dev:
 * device int64 node offsets of the p+2 curve boundaries.  Residual oracle for
 * the large configurations.                           */
int skb_system_matvec(const double* pos, const double* nrm, const double* w, const double* kappa,
                      int64_t n_nodes, const double* hole_centers, int64_t n_holes,
                      const int64_t* curve_off_dev, const double* x, int64_t nrhs, double* y,
                      void* stream);
/* Field at interior targets from a solve() output, out (2m x nrhs) row-major:
 * u = D mu + H lam (reference evaluate_interior skel.py:537-564,
 * eval_forward_block kernels.py:171-198).  x: (2N + 3p) x nrhs row-major.    */
/* Laplace-Neumann exact operator y = (-1/2 I + K' + 1 w^T) mu (kernels.py:
 * 119-125 summed over all nodes) and interior field u = -S mu (kernels.py:
 * 193-194); x: N x nrhs, y: N x nrhs, out: m x nrhs (row-major).            */
int skb_system_matvec_lap(const double* pos, const double* nrm, const double* w,
                          const double* kappa, int64_t n_nodes, const double* x, int64_t nrhs,
                          double* y, void* stream);
int skb_eval_interior_lap(const double* pos, const double* w, int64_t n_nodes, const double* x,
                          int64_t nrhs, const double* targets, int64_t m, double* out, void* stream);
int skb_eval_interior(const double* pos, const double* nrm, const double* w, int64_t n_nodes,
                      const double* hole_centers, int64_t n_holes, const double* x, int64_t nrhs,
                      const double* targets, int64_t m, double* out, void* stream);
/* Boundary.point_in_domain (reference geometry.py:179-192): winding numbers of
 * the node polylines (curve_off: ncurves + 1 node offsets, device) and
 * nearest-node distance > 1e-12; inside[m] = 1 / 0.                           */
int skb_point_in_domain(const double* pos, const int64_t* curve_off_dev, int64_t ncurves,
                        const double* targets, int64_t m, uint8_t* inside, void* stream);

/* dst[idx[i]*ld + c] = value for i < nidx, c < ncols (the nonroot mask of
 * skel.py:181-188 applied by zeroing root rows of a copy). unused: NULL.    */
int skb_fill_rows(int64_t nidx, const int64_t* idx, double* dst, int64_t ld, const void* unused,
                  int64_t ncols, double value, void* stream);

/* ---- level-granular entry points (csrc/level.cu) ---------------------------
 * One call per quadtree level; descriptor arrays are HOST memory, matrices
 * device.  Per-box factor addresses (uint64) as laid out by the caller.      */

/* (c) of compress_box for a level batch (skel.py:316-338): T = R11^-1 R12 from
 * the QRCP'd stacks A (lda), permuted self blocks E with the children's Xss
 * (child_off/child_xss: nbox x 5, as skb_assemble_self), X_sr, X_rs, X_rr
 * (grouped DMMA GEMMs), LU(X_rr) with pivot ratio (info_dev/ratio_dev, as
 * skb_getrf_batched), X_rs_div = X_rr^-1 X_rs and Xss_mod = E_SS - X_sr X_rs_div.
 * nB, k, act_off: host; act_off_dev/act_dev/perm_dev: the level's device CSR
 * active lists and QRCP permutations.                                         */
int skb_level_schur(int64_t nbox, const int64_t* nB, const int64_t* k,
                    const int64_t* act_off, const double* pos, const double* nrm,
                    const double* w, const double* kappa, const int64_t* act_off_dev,
                    const int64_t* act_dev, const int32_t* perm_dev, const int64_t* A,
                    const int64_t* lda, const int64_t* child_off,
                    const uint64_t* child_xss, const uint64_t* T, const uint64_t* Xrr,
                    const uint64_t* LU, const uint64_t* Xsr, const uint64_t* Xrsdiv,
                    const uint64_t* Xss, const uint64_t* ipiv, int32_t* info_dev,
                    double* ratio_dev, int32_t pde, void* stream);   /* pde 0 Stokes, 1 Laplace */

/* (d) augmentation sweep of one level (_finish_top, skel.py:384-396): on the
 * (2N x q) UH / PsiV / UH_div, UH_R -= T^T UH_S; w = X_rr^-1 UH_R;
 * UH_S -= X_sr w; UH_div_R = w; PsiV_R -= T^T PsiV_S; PsiV_S -= X_rs_div^T PsiV_R
 * (PsiV restricted to the box's hole columns cols, host CSR cols_off/cols and
 * the same lists on the device c_off/c) and the deterministic (box order)
 * accumulation schur += PsiV_R^T w.  sd/rd: device CSR skeleton/redundant DOFs. */
int skb_level_aug(int64_t nbox, const int64_t* k, const int64_t* r, int64_t q,
                  const int64_t* cols_off, const int64_t* cols, const int64_t* sd_off,
                  const int64_t* sd, const int64_t* rd_off, const int64_t* rd,
                  const int64_t* c_off, const int64_t* c, const uint64_t* T, const uint64_t* LU,
                  const uint64_t* Xsr, const uint64_t* Xrsdiv, const uint64_t* ipiv, double* UH,
                  double* PsiV, double* UH_div, double* schur, double* stash, const int64_t* st_us,
                  const int64_t* st_ps, const int64_t* st_sp, int32_t acc, void* stream);
/* Accumulate one level's stored Schur parts (stash + st_sp) into schur, in
 * skb_level_aug's order (skel.py:396).                                       */
int skb_level_schur_acc(int64_t nbox, const int64_t* cols_off, const int64_t* cols, int64_t q,
                        const double* stash, const int64_t* st_sp, double* schur, void* stream);
/* update(): incremental _finish_top.  The sweep of a
 * level restricted to the changed augmentation columns qc (host list) for
 * boxes whose factors were reused; updates UH / UH_div rows, the stored
 * outgoing UH_S and Schur parts at those columns.                            */
int skb_level_aug_narrow(int64_t nbox, const int64_t* k, const int64_t* r, int64_t q, int64_t nqc,
                         const int64_t* qc, const int64_t* cols_off, const int64_t* sd_off,
                         const int64_t* sd, const int64_t* rd_off, const int64_t* rd,
                         const int64_t* c_off, const int64_t* c, const uint64_t* T,
                         const uint64_t* LU, const uint64_t* Xsr, const uint64_t* ipiv, double* UH,
                         const double* PsiV, double* UH_div, double* stash, const int64_t* st_us,
                         const int64_t* st_sp, void* stream);
/* Stored outgoing skeleton rows of reused boxes (us: k x q, ps: k x nc per
 * box, device addresses) back into UH (columns with qmask 0) and PsiV.       */
int skb_restore_rows(int64_t nbox, const int64_t* sd_off, const int64_t* sd, int64_t max_k,
                     const int64_t* c_off, const int64_t* c, const uint64_t* us, const uint64_t* ps,
                     const uint8_t* qmask_dev, int64_t q, double* UH, double* PsiV, void* stream);
/* One level of update()'s incremental sweep (reused boxes: copy + narrow +
 * restore under a dirty parent; dirty boxes: full; then accumulation), all
 * descriptor arrays on the host.                                             */
int skb_level_aug_update(int64_t nbox, const int64_t* k, const int64_t* r, int64_t q,
                         const int64_t* cols_off, const int64_t* cols, const int64_t* sd_off,
                         const int64_t* sd, const int64_t* rd_off, const int64_t* rd,
                         const uint8_t* dirty, const uint8_t* parent_dirty, const uint64_t* T,
                         const uint64_t* LU, const uint64_t* Xsr, const uint64_t* Xrsdiv,
                         const uint64_t* ipiv, const uint64_t* old_us, const uint64_t* old_ps,
                         const uint64_t* old_sp, int64_t nqc, const int64_t* qc,
                         const uint8_t* qmask_dev, double* UH, double* PsiV, double* UH_div,
                         double* schur, double* stash, const int64_t* st_us, const int64_t* st_ps,
                         const int64_t* st_sp, void* stream);
/* dst rows idx (n) and columns qc (nqc) <- src, both nrows x ncols row-major. */
int skb_copy_rows_cols(int64_t n, const int64_t* idx_dev, int64_t nqc, const int64_t* qc_dev,
                       int64_t nrows, int64_t ncols, const double* src, double* dst, void* stream);

/* ---- native level engine (csrc/engine.cu) ----------------------------------
 * The compression chain of factor() (skel.py:443-449 over compress_box
 * skel.py:293-316: assign_internal_actives, far_dofs, proxy rings, ID stack,
 * Householder pre-reduction, QRCP, skeletons) runs level by level on a host
 * thread of the library; the caller consumes finished levels.
 * tree = {center, hw, neighbours, lev, ix, iy, children (nbox x 4), level_start,
 * is_leaf (uint8)}; store = {big, a_start, a_len, s_start, s_len, fill} (int64,
 * big of capacity cap; leaf actives pre-filled, the engine appends);
 * geo = {px, py (host), pos, nrm, w (device), cs (P x 2 host)}.  Levels depth
 * down to lev_lo; max_level_ints bounds one level's (perm, k, steps, gap).   */
int skb_engine_start(const void* const* tree, int64_t depth, const double* root, double factor,
                     int64_t* const* store, int64_t cap, const double* const* geo, int64_t P,
                     double tol, void* stream, int64_t lev_lo, int64_t max_level_ints,
                     int32_t pde, int64_t* handle);   /* pde 0 Stokes, 1 Laplace */
/* Block until level L is done: sizes = {rc, B, na, box0, o_int, o_act, h2d bytes,
 * d2h bytes}; ptrs =
 * {act_off, act, rows, A, m_q, perm, k, steps, gap (host), stack, dbuf, dup
 * (device), event, idx (host: the compressed boxes)}.  Host arrays stay valid until skb_engine_free.          */
int skb_engine_wait(int64_t handle, int64_t L, int64_t* sizes, int64_t* ptrs);
/* Update mode (start with lev_lo <= 0 = deferred): recompress only the boxes
 * with todo[i] != 0; clean boxes take their skeleton from clean_off/clean_skel
 * (CSR over all boxes).  skb_engine_go starts a deferred engine.  In update
 * mode sizes[1] counts the recompressed boxes and ptrs[13] lists them.       */
int skb_engine_set_update(int64_t handle, const uint8_t* todo, const int64_t* clean_off,
                          const int64_t* clean_skel);
int skb_engine_go(int64_t handle);
/* Update mode for the native level driver: the clean boxes' skeletons are read
 * from the previous factorization's level table, int64 [levels][21], row =
 * {B, code (ix * 2^level + iy, ascending), act_off, act, perm (int32), k,
 * T, X_rr, LU, X_sr, X_rs_div, Xss (uint64 per box), ipiv, info, ratio, stash
 * (device address), st_us, st_ps, st_sp, gap, steps}; host arrays of the caller. */
int skb_engine_set_update_table(int64_t handle, const uint8_t* todo, const int64_t* old_table);
/* Grow the engine's stream-ordered pool and the default pool to the given
 * reserved sizes now (no pool growth inside a later level pipeline).         */
int skb_pool_prewarm(int64_t engine_bytes, int64_t default_bytes);
/* Native level driver: the consumer side of the level loop (run_level
 * skel.py:340-361, compress_box (c) skel.py:316-338, the _finish_top sweep
 * skel.py:384-396) on the calling thread.  Per level: wait for the engine,
 * X_RR pivot check of the level below (100 = a box must migrate, the caller
 * re-runs on its Python path), merge with the clean boxes of the previous
 * factorization (101 = no twin, 102 = active set changed), factor storage,
 * skb_level_schur, acknowledge, augmentation sweep of the level below
 * (skb_level_aug, or skb_level_aug_update when cfg[18]), level lists on the
 * device.  cfg (int64 x 24) = {level stream, sweep stream, curvature (device),
 * q, npairs, pair_box, pair_curve ((box, curve) membership, sorted by box),
 * parent, UH, PsiV, UH_div, schur (device), update, dirty mask (uint8 per box),
 * nqc, qc (host), qmask (device), previous level table, incremental sweep,
 * xss (uint64 per box, host, filled)}.                                        */
int skb_drv_run(int64_t engine, const int64_t* cfg, double pivot_ratio_floor, int64_t* handle);
/* Arrays of one level (valid until skb_drv_free): sizes (int64 x 24) = {B, na,
 * nnew, nsd, nrd, ncols, slab, slab bytes, stash, stash bytes, desc, desc bytes,
 * offsets of {sd_off, sd, rd_off, rd, c_off, c} in desc (int64 units), total
 * h2d bytes, total d2h bytes}; ptrs (int64 x 32) = {idx, code, act_off, act, perm
 * (int32), k, steps, gap, info, ratio, clean_pos, T, X_rr, LU, X_sr, X_rs_div,
 * Xss, ipiv, sd_off, sd, rd_off, rd, cols_off, cols, st_us, st_ps, st_sp,
 * new_pos}.  The device allocations (skb_dev_alloc pool) become the caller's. */
/* Wait for every level's X_RR pivot info (skb_drv_run only polls it): 0, or 100
 * = a box must migrate.  Call before skb_drv_level.                           */
int skb_drv_resolve(int64_t handle);
int skb_drv_level(int64_t handle, int64_t lev, int64_t* sizes, int64_t* ptrs);
int skb_drv_free(int64_t handle);
/* stream waits for level L's compression */
int skb_engine_stream_wait(int64_t handle, int64_t L, void* stream);
/* free level L's device buffers, stream-ordered on stream */
int skb_engine_release(int64_t handle, int64_t L, void* stream);
/* the caller has enqueued level L's Schur stage; lead >= 0 limits how many
 * levels the engine may run ahead of the acknowledged level               */
int skb_engine_ack(int64_t handle, int64_t L);
int skb_engine_set_lead(int64_t handle, int64_t lead);
/* stop after the current level and join the engine thread */
int skb_engine_stop(int64_t handle);
int skb_engine_free(int64_t handle, void* stream);
/* Factor storage from a process-wide stream-ordered pool (no implicit device
 * synchronisation when it grows); freed stream-ordered.                      */
int skb_dev_alloc(int64_t bytes, void* stream, uint64_t* out);
int skb_dev_free(uint64_t ptr, void* stream);
/* Synchronous device -> host copy of raw bytes (factor inspection). */
int skb_d2h(void* host, const void* dev, int64_t bytes);
/* Debug (SKB_ENGINE_SNAP=<level>): host copy of the snapshot `which` of that
 * level's ID stacks (0 after assembly, 1 after pre-reduction, 2 after QRCP);
 * returns the element count, -1 when no snapshot was taken.                  */
int64_t skb_debug_snap(int32_t which, double* host, int64_t n_host);

/* ---- native host runtime (host arrays, no device; csrc/host.cpp) ---------
 * Per-level bookkeeping the reference does per box in Python.  Tree arrays as
 * in tree.py: center (nbox x 2), hw, neighbours (nbox x 8, -1 = none, sorted
 * keys), lev/ix/iy, is_leaf (uint8), level_start (depth + 2);
 * root = {cx, cy, half width}.                                               */

/* Host allocator tuning (called once at load): large freed blocks stay in the
 * heap instead of being unmapped, so per-level host arrays do not page-fault. */
int skb_host_init(void);

/* F_int of each box idx[b] (reference _Compressor.far_dofs, skel.py:258-280 with
 * Tree.colleagues tree.py:70-81, Tree.shallow_leaves_near tree.py:83-99 and
 * proxy_radius tree.py:158-160): active DOFs (segments big[a_start[j]..+a_len[j]])
 * of the colleagues then the coarser leaves meeting the proxy disc, kept where
 * the node lies strictly inside the disc.  far_off: nb + 1.  Returns 1 with
 * *need = required length when cap is too small.                            */
int skb_host_far_lists(int64_t nb, const int64_t* idx, const double* center, const double* hw,
                       const int64_t* nbr, const int64_t* lev, const int64_t* ix,
                       const int64_t* iy, const uint8_t* is_leaf, const int64_t* level_start,
                       int64_t depth, const double* root, double factor, const int64_t* big,
                       const int64_t* a_start, const int64_t* a_len, const double* px,
                       const double* py, int64_t* far_off, int64_t* far, int64_t cap,
                       int64_t* need, int32_t dof_shift);   /* node = dof >> dof_shift */

/* Proxy rings (kernels.py:263-273): pts = centre + r_p (cos, sin)(2 pi j / P),
 * radial normals about the ring centroid (kernels.py:340-342), weights
 * 2 pi r_p / P.  cs: P x 2 (cos, sin); pts, pn: nb x P x 2; pw: nb.          */
/* Leaf active sets (skel.py:243-249) appended to `big` level by level; returns
 * the fill (or -1: capacity).                                                */
int64_t skb_host_leaf_actives(int64_t nbox, int64_t depth, const int64_t* lev, const uint8_t* is_leaf,
                              const int64_t* node_start, const int64_t* node_cnt,
                              const int64_t* level_nodes, const int64_t* level_nodes_off,
                              const int64_t* level_start, int64_t dpn, int64_t* big, int64_t cap,
                              int64_t* a_start, int64_t* a_len);
int skb_host_proxies(int64_t nb, const int64_t* idx, const double* center, const double* hw,
                     double factor, int64_t P, const double* cs, double* pts, double* pn,
                     double* pw);

/* Adaptive quadtree (reference build_tree, tree.py:110-155): root {cx, cy,
 * half width}; split while a box holds more than leaf_cap nodes (depth <
 * max_depth), east = x >= cx, north = y >= cy, empty children pruned, boxes of
 * a level sorted by key.  Returns an opaque handle; skb_tree_sizes gives
 * {nbox, depth, level-node entries}; skb_tree_export copies the flat arrays
 * (tree.py layout: children nbox x 4 compacted in SW, SE, NW, NE order,
 * neighbours nbox x 8, level_nodes concatenated with level_nodes_off,
 * node_leaf N); skb_tree_free releases the handle.                          */
int skb_tree_build(const double* pos, int64_t N, int64_t leaf_cap, int64_t max_depth,
                   const double* root, int64_t* handle);
int skb_tree_sizes(int64_t handle, int64_t* sizes);
int skb_tree_export(int64_t handle, int64_t* level_start, int64_t* lev, int64_t* ix, int64_t* iy,
                    int64_t* parent, double* center, double* hw, int64_t* children,
                    int64_t* nchild, int64_t* node_start, int64_t* node_cnt, int64_t* level_nodes,
                    int64_t* level_nodes_off, int64_t* nbr, int64_t* node_leaf);
int skb_tree_free(int64_t handle);

/* Dirty boxes of a local update (reference update skel.py:476-491 with
 * ownership_changed tree.py:251-270, _mark_disc_hits tree.py:215-236 and
 * _dirty_closure skel.py:517-534).  Trees passed as 11 flat arrays {level_start,
 * lev, ix, iy, parent, node_start, node_cnt, level_nodes, level_nodes_off,
 * neighbours, node_leaf}; pts: moved positions (old and new, npts x 2);
 * mod_new: moved nodes (new numbering).  out_mask: new-tree boxes.          */
int skb_dirty_set(const int64_t* const* new_arrays, const double* new_center, int64_t new_depth,
                  const int64_t* const* old_arrays, int64_t old_depth, const double* root,
                  const int64_t* old_to_new, const double* pts, int64_t npts,
                  const int64_t* mod_new, int64_t nmod, double proxy_factor, uint8_t* out_mask);

#ifdef __cplusplus
}
#endif

#endif /* SKELB200_H */
