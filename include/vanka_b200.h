/*
 * vanka_b200.h — C ABI of the B200-native Vanka / multigrid hot path.
 *
 * Plain C types only (pointers, sizes, opaque handles, int status).  Every
 * entry point names the reference interface it replaces (file:line under
 * /root/reference/pkg/src/stokesmg/); see INTEGRATION.md for the ctypes
 * binding the reference package would add.
 *
 * Conventions
 *   - status: 0 ok; VK_ERR_* (< 0) argument / CUDA / allocation error, with a
 *     message from vk_last_error(); factor reports per-patch singularity in
 *     its status array and returns VK_SINGULAR (> 0).
 *   - handles own their device memory; vectors are caller-owned DEVICE
 *     pointers (fp64) unless the name says host.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default);
 *     all vector calls are asynchronous and stream-ordered, capturable in a
 *     CUDA graph (no allocation, no host sync).
 *   - array inputs to *_create / *_build may be host or device pointers
 *     (copied with cudaMemcpyDefault).
 */
#ifndef VANKA_B200_H
#define VANKA_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define VK_API __attribute__((visibility("default")))
#else
#define VK_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define VK_OK 0
#define VK_SINGULAR 1
#define VK_ERR_ARG (-1)
#define VK_ERR_CUDA (-2)
#define VK_ERR_ALLOC (-3)
#define VK_ERR_UNSUPPORTED (-4)

/* per-patch factor status (reference sparsela.py:76-83) */
#define VK_PATCH_OK 0
#define VK_PATCH_ZERO_ROW 1      /* "matrix has an all-zero row"            */
#define VK_PATCH_SMALL_PIVOT 2   /* "pivot below 1e-12 of its row magnitude" */

/* weighting (reference vanka.py:25) */
#define VK_WEIGHT_INVMULT 0
#define VK_WEIGHT_UNIT 1

/* gather epilogues for vk_patches_apply (reference vanka.py:142-148 and the
 * damped update of mg.py:268-271) */
#define VK_APPLY_OUT 0           /* out  = sum_i R_i^T W_i A_i^-1 R_i r        */
#define VK_APPLY_XSET 1          /* x    = scale * out        (x was zero)     */
#define VK_APPLY_XADD 2          /* x    = x + scale * out                     */

typedef struct vk_csr_s* vk_csr_t;
typedef struct vk_patches_s* vk_patches_t;

VK_API const char* vk_last_error(void);
VK_API int vk_version(void);
VK_API int vk_device_sync(void);

/* ---------------- matrices: scipy.sparse.csr_matrix on the device ---------
 * replaces the CSR the reference builds in assembly.py:288-332 / mg.py:159-167
 * (consumed by sparsela.py:45-47, mg.py:41-45). */
VK_API int vk_csr_create(const int32_t* indptr, const int32_t* indices, const double* data,
                  int32_t nrows, int32_t ncols, int64_t nnz, vk_csr_t* out);
/* transpose (masked.T for restriction, mg.py:44-45), deterministic order */
VK_API int vk_csr_transpose(vk_csr_t a, vk_csr_t* out);
VK_API int vk_csr_info(vk_csr_t a, int32_t* nrows, int32_t* ncols, int64_t* nnz);
VK_API int vk_csr_destroy(vk_csr_t a);
/* copy a CSR to HOST arrays (any may be NULL): indptr[nrows+1], indices[nnz],
 * data[nnz] (scipy layout, sorted indices) */
VK_API int vk_csr_export(vk_csr_t a, int32_t* indptr, int32_t* indices, double* data);
/* max |a_ij| over the stored entries (the coarse shift of mg.py:231) */
VK_API int vk_csr_max_abs(vk_csr_t a, double* out_host);

/* ---------------- SpMV (K5/K6) ---------------------------------------------
 * y = alpha*A x + beta*y   : sparsela.spmv (sparsela.py:45-47), prolong
 *                            (mg.py:41-42, with beta=1 for x + P e, mg.py:296)
 * r = b - A x              : residual at mg.py:270, 294 */
VK_API int vk_spmv(vk_csr_t a, const double* x, double* y, double alpha, double beta, void* stream);
VK_API int vk_residual(vk_csr_t a, const double* b, const double* x, double* r, void* stream);
/* fused V-cycle transfer units (one cooperative launch each, a grid barrier
 * between the two SpMVs; every row summed exactly as vk_spmv / vk_residual,
 * so bit-identical to the two separate calls):
 *   vk_residual_restrict: r = b - A x, then rc = PT r      (mg.py:294-295)
 *   vk_prolong_residual:  x = x + P xc, then r = b - A x   (mg.py:296-297 and
 *                         the first residual of post-smoothing, mg.py:270) */
VK_API int vk_residual_restrict(vk_csr_t a, const double* b, const double* x, double* r,
                                vk_csr_t pt, double* rc, void* stream);
VK_API int vk_prolong_residual(vk_csr_t p, const double* xc, double* x, vk_csr_t a,
                               const double* b, double* r, void* stream);

/* ---------------- patches (K1-K4) ------------------------------------------
 * vk_patches_build replaces vanka.build_patches_taylor_hood /
 * build_patches_hdiv_extended / _finish (vanka.py:49-126).  Candidate patch
 * p (in reference order: dim, entity index) owns the cells
 * ent2cell[ent2cell_ptr[p] : ent2cell_ptr[p+1]] and the pressure DoFs
 * pdofs[pdof_ptr[p] : pdof_ptr[p+1]] (already offset).  Velocity DoFs =
 * sorted unique union of cell_dofs over those cells minus constrained
 * (constrained[d] != 0).  Empty candidates are dropped (vanka.py:64-65). */
VK_API int vk_patches_build(const int32_t* cell_dofs, int32_t ncells, int32_t nloc,
                     const int32_t* ent2cell_ptr, const int32_t* ent2cell,
                     int32_t ncand, const int32_t* pdof_ptr, const int32_t* pdofs,
                     const uint8_t* constrained, int32_t ndof, int32_t weighting,
                     vk_patches_t* out);
/* patch set from explicit lists (reference Patch/PatchSet built by hand,
 * vanka.py:28-46): offsets[npatch+1] (int64), indices[offsets[npatch]],
 * num_velocity[npatch], weights[offsets[npatch]] (NULL = all ones);
 * multiplicity is recomputed by counting. */
VK_API int vk_patches_from_lists(const int64_t* offsets, const int32_t* indices,
                          const int32_t* num_velocity, const double* weights,
                          int32_t npatch, int32_t ndof, vk_patches_t* out);
/* sizes: number of kept patches, total patch entries (sum s), max patch size */
VK_API int vk_patches_info(vk_patches_t h, int32_t* npatch, int64_t* total, int32_t* smax);
/* bit-exact export to HOST arrays (any may be NULL): offsets[npatch+1],
 * indices[total], num_velocity[npatch], weights[total], multiplicity[ndof],
 * cand_of_patch[npatch] (candidate index of each kept patch) */
VK_API int vk_patches_export(vk_patches_t h, int64_t* offsets, int32_t* indices,
                      int32_t* num_velocity, double* weights, double* multiplicity,
                      int32_t* cand_of_patch);
/* general dense extraction A[rows, cols] (sparsela.extract_submatrix,
 * sparsela.py:50-60) into a DEVICE row-major nrows x ncols array; rows/cols
 * are DEVICE int32 lists, sorted and duplicate-free (checked by the caller). */
VK_API int vk_extract(vk_csr_t a, const int32_t* rows, int32_t nrows, const int32_t* cols,
                      int32_t ncols, double* out_dev, void* stream);
/* extract dense blocks A[idx, idx] (sparsela.extract_submatrix, sparsela.py:50-60)
 * for patches first..first+count-1 into HOST row-major blocks concatenated in
 * patch order (sum s^2 doubles). */
VK_API int vk_patches_extract(vk_patches_t h, vk_csr_t a, int32_t first, int32_t count,
                       double* blocks_host);
/* extract + batched LU-with-partial-pivoting-equivalent Gauss-Jordan inverse
 * with the reference row-scale guard (vanka.factor_patches, vanka.py:129-139;
 * sparsela.lu_factor, sparsela.py:63-84).  status_host[npatch] (may be NULL)
 * receives VK_PATCH_*; returns VK_SINGULAR if any patch is singular and
 * first_bad (may be NULL) = its index. */
VK_API int vk_patches_factor(vk_patches_t h, vk_csr_t a, int32_t* status_host, int32_t* first_bad);
/* explicit patch inverses to HOST (row-major s x s per patch, concatenated) */
VK_API int vk_patches_export_inverse(vk_patches_t h, int32_t first, int32_t count, double* inv_host);
/* additive sweep (vanka.apply_additive, vanka.py:142-148, + mg.py:268-271):
 * mode VK_APPLY_OUT: out = sum_i R_i^T W_i A_i^{-1} R_i r ; XSET/XADD: see above.
 * Deterministic: contributions summed per DoF in patch order.
 * zbuf: DEVICE buffer of `total` doubles (vk_patches_info) for the weighted
 * local corrections, or NULL for the handle's own.  The handle is immutable
 * after factor, so sweeps of one handle may run concurrently on different
 * streams as long as each passes its own zbuf (and its own out). */
VK_API int vk_patches_apply(vk_patches_t h, const double* r, double* out, double scale,
                     int32_t mode, double* zbuf, void* stream);
/* the two halves of vk_patches_apply, for per-kernel timing:
 * solve: z = W A_i^{-1} R_i r into zbuf (NULL = handle's; K4a);
 * accumulate: per-DoF patch-ordered sum of z + epilogue (K4b). */
VK_API int vk_patches_solve(vk_patches_t h, const double* r, double* zbuf, void* stream);
VK_API int vk_patches_accumulate(vk_patches_t h, const double* zbuf, double* out, double scale,
                                 int32_t mode, void* stream);
/* one preconditioned Chebyshev step of degree mode (mg.py:237-255) with the
 * sweep fused in: acc = apply_additive(r) (K4a + K4b), then in K4b's
 * epilogue, elementwise in the reference's order,
 *   first == 1:  d = acc / c2                 (d = preconditioner(r) / theta)
 *   first == 0:  d = c1 * d + c2 * acc        (c1 = rho_next*rho, c2 = 2 rho_next/delta)
 *   and x = x + d;  first == 2: as 1 but x = d (x was zero: x + d = d).
 * zbuf as for vk_patches_apply. */
VK_API int vk_patches_apply_cheb(vk_patches_t h, const double* r, double* x, double* d,
                                 double c1, double c2, int32_t first, double* zbuf, void* stream);
/* name of the K4a kernel vk_patches_solve launches for this patch set (for
 * profiling tools and the bench line) */
VK_API const char* vk_patches_solve_kernel(vk_patches_t h);
VK_API int vk_patches_destroy(vk_patches_t h);

/* ---------------- dense / vector helpers (FGMRES + V-cycle plumbing) -------
 * sparsela.fgmres (sparsela.py:117-191), coarse_solve (mg.py:274-279),
 * v_cycle bc copy (mg.py:298-300).  Device scalars are single doubles.
 *
 * Reductions take a caller-owned DEVICE scratch of VK_REDUCE_SCRATCH doubles,
 * zero-filled once before its first use (each reduction leaves it ready for
 * the next).  Reductions in flight at the same time (different streams) need
 * distinct scratch buffers; one buffer may serve any number of reductions
 * ordered on one stream (or one CUDA graph). */
#define VK_REDUCE_SCRATCH 320
/* *out_dev = x . y  (deterministic two-level reduction, one launch) */
VK_API int vk_dot(int64_t n, const double* x, const double* y, double* out_dev,
                  double* scratch_dev, void* stream);
/* y = y - (*a_dev) * x */
VK_API int vk_axpy_dev(int64_t n, const double* a_dev, const double* x, double* y, void* stream);
/* Fused modified-Gram-Schmidt step (sparsela.py:160-163): y = y - (*a_dev) * x,
 * then *out_dev = x2 . y (sqrt of it if sqrt_out; x2 may alias y).  The dot
 * uses vk_dot's thread/element mapping and reduction tree, so the result is
 * bit-identical to vk_axpy_dev followed by vk_dot / vk_nrm2. */
VK_API int vk_axpy_dot(int64_t n, const double* a_dev, const double* x, double* y, const double* x2,
                       double* out_dev, int32_t sqrt_out, double* scratch_dev, void* stream);
/* y = y + a * x  (host scalar) */
VK_API int vk_axpy(int64_t n, double a, const double* x, double* y, void* stream);
/* y = x / (*d_dev) */
VK_API int vk_div_dev(int64_t n, const double* x, const double* d_dev, double* y, void* stream);
/* *out_dev = sqrt(x . x) */
VK_API int vk_nrm2(int64_t n, const double* x, double* out_dev, double* scratch_dev,
                   void* stream);
/* x = x - q (q . x) in place (NullspaceProjector, sparsela.py:113-114);
 * scratch_dev: VK_REDUCE_SCRATCH doubles as above */
VK_API int vk_project(int64_t n, const double* q, double* x, double* scratch_dev, void* stream);
/* Chebyshev vector update of degree mode (mg.py:246-254) for a generic
 * operator/preconditioner: first != 0: d = z / c2; else d = c1 d + c2 z;
 * then x = x + d (elementwise, the reference's operation order) */
VK_API int vk_cheb_update(int64_t n, const double* z, double* d, double* x, double c1, double c2,
                          int32_t first, void* stream);
/* dst[idx[k]] = src[idx[k]] */
VK_API int vk_copy_index(int64_t m, const int32_t* idx, const double* src, double* dst, void* stream);
/* y = M x for a dense row-major m x n matrix (coarse inverse apply) */
VK_API int vk_gemv(int32_t m, int32_t n, const double* mat, const double* x, double* y, void* stream);
/* x += sum_k coef_dev[k] * Z[k, :]  (Z row-major count x n): FGMRES update */
VK_API int vk_combine(int64_t n, int32_t count, const double* z, const double* coef_dev,
               double* x, void* stream);
/* dense[rows x cols] (row-major, device) = CSR (coarse operator densify) */
VK_API int vk_csr_to_dense(vk_csr_t a, double* dense, void* stream);

/* ---------------- device assembly ------------------------
 * replaces assembly.py:93-172, 230-285 (operator) and mg.py:127-167
 * (prolongation).  The host passes reference-cell data only; COO entries
 * are written at fixed positions (cell-major / facet-major / in the
 * reference's prolongation loop order) into caller-owned DEVICE buffers
 * keys[] (row * ncols + col) and vals[].
 * vk_assemble_cells: per cell, the velocity block 2 nu (eps u, eps v) and
 *   both divergence blocks -(div v, p) (nv*nv + 2*np*nv entries per cell);
 *   rv/rg: reference velocity basis values / gradients at the nq points
 *   ([nq][nv][2], [nq][nv][2][2]); pv [nq][np]; cell_xy [ncells][3|4][2] in
 *   reference-map vertex order; piola: H(div) contravariant map.
 * vk_assemble_load: per cell, the manufactured-forcing load (assembly.py:
 *   136-172 with the forcing of assembly.py:62-87) as nv (dof, s_i load_i)
 *   pairs (keys[] = dof); reduce them with vk_coo_to_csr (ncols = 1).
 * vk_assemble_facets: per interior edge the (2nv)^2 block of the H(div)
 *   consistency / symmetry / penalty terms (assembly.py:243-267); rv/rg
 *   [6][nq][nv][..] tables per (local edge slot, aligned); info [ne][6] =
 *   c1, c2, slot1, aligned1, slot2, aligned2; geo [ne][5] = t, n1, h_e.
 * vk_prolong_entries: per (parent, child slot) the block (sc/sf) E[cfg]
 *   (mg.py:141-147) in loop order.
 * vk_coo_to_csr: stable sort by (row, col); duplicates summed in generation
 *   order (dup_first = 0) or the first kept (dup_first = 1, mg.py:149-153);
 *   entries with |v| <= drop_abs, in row_drop rows or col_drop columns are
 *   removed; rows flagged in diag_one become identity rows (the buffers then
 *   need n + nrows entries).  Synchronous; *out is a new CSR handle. */
VK_API int vk_assemble_cells(int32_t ncells, int32_t nq, int32_t nv, int32_t np, int32_t quad,
                             int32_t piola, const double* w, const double* pts, const double* rv,
                             const double* rg, const double* pv, const double* cell_xy,
                             const int32_t* vdofs, const double* vscale, const int32_t* pdofs,
                             const double* pscale, int32_t poffset, double viscosity,
                             int64_t ncols, int64_t* keys, double* vals, void* stream);
VK_API int vk_assemble_load(int32_t ncells, int32_t nq, int32_t nv, int32_t quad, int32_t piola,
                            const double* w, const double* pts, const double* rv,
                            const double* cell_xy, const int32_t* vdofs, const double* vscale,
                            double viscosity, int64_t* keys, double* vals, void* stream);
VK_API int vk_assemble_facets(int32_t nedges, int32_t nq, int32_t nv, const double* w,
                              const double* rv, const double* rg, const int32_t* info,
                              const double* geo, const double* cell_xy, const int32_t* vdofs,
                              const double* vscale, double viscosity, double alpha,
                              int64_t ncols, int64_t* keys, double* vals, void* stream);
VK_API int vk_prolong_entries(int32_t nparent, int32_t nf, int32_t nc, const int32_t* children,
                              const int32_t* cfg, const double* tables, const int32_t* cdofs,
                              const double* cscale, const int32_t* fdofs, const double* fscale,
                              int64_t row_off, int64_t col_off, int64_t ncols, int64_t* keys,
                              double* vals, void* stream);
VK_API int vk_coo_to_csr(int64_t n, int64_t* keys, double* vals, int32_t nrows, int32_t ncols,
                         int32_t dup_first, double drop_abs, const uint8_t* row_drop,
                         const uint8_t* col_drop, const uint8_t* diag_one, vk_csr_t* out);

/* ---------------- discretisation-error measurement --------------------------
 * replaces the reference's bench.error_norms (bench.py:95-164) for the
 * manufactured enclosed-flow solution (assembly.py:55-87), called by
 * run_case / stopping_study (bench.py:174-191, 239-301).
 * vk_error_cells: per (cell, quadrature point) of the degree min(2k+4, 20)
 *   rule: w det (|u_h - u|^2 + |grad u_h - grad u|^2), w det (|u|^2 +
 *   |grad u|^2), |div u_h|, p_h and w det into work[5][ncells*nq]; tables and
 *   maps as for vk_assemble_cells, x the solution vector (pressure block at
 *   poffset).
 * vk_error_jump: per (interior edge, point) w_q [u_h . t]^2 / 2 (the
 *   tangential-jump seminorm integrand, bench.py:143-158) into
 *   work[nedges*nq]; rv/info/geo as for vk_assemble_facets.
 * vk_error_reduce: fixed-order single-CTA reduction; out[6] (device) = sum
 *   e2, sum base, max |div|, sum w (p - mean)^2, sum of the jump terms, mean
 *   pressure.  All stream-ordered, asynchronous. */
VK_API int vk_error_cells(int32_t ncells, int32_t nq, int32_t nv, int32_t np, int32_t quad,
                          int32_t piola, const double* w, const double* pts, const double* rv,
                          const double* rg, const double* pv, const double* cell_xy,
                          const int32_t* vdofs, const double* vscale, const int32_t* pdofs,
                          const double* pscale, int32_t poffset, const double* x, double* work,
                          void* stream);
VK_API int vk_error_jump(int32_t nedges, int32_t nq, int32_t nv, const double* w, const double* rv,
                         const int32_t* info, const double* geo, const double* cell_xy,
                         const int32_t* vdofs, const double* vscale, const double* x,
                         double* work, void* stream);
VK_API int vk_error_reduce(int64_t ncq, const double* work, int64_t neq, const double* jump,
                           double* out, void* stream);

/* ---------------- coarse dense operator and its inverse --------------------
 * replaces the reference's coarse factorization (mg.py:228-232:
 * lu_factor(A0.toarray() + shift * np.outer(q, q))), applied per V-cycle as
 * x = M^{-1} b by vk_gemv (mg.py:274-279 applies getrs).
 * vk_coarse_operator: dense row-major M = A0 + shift q q^T, formed exactly as
 * numpy does (fl(a + fl(shift * fl(q_i q_j))), bit-identical).
 * vk_dense_inverse: explicit inverse of a DEVICE row-major n x n matrix by
 * blocked Gauss-Jordan elimination with partial pivoting (LAPACK pivot
 * order); `work` is a DEVICE buffer of vk_dense_inverse_workspace(n) bytes.
 * The reference guard of sparsela.lu_factor (sparsela.py:76-83) applies:
 * returns VK_SINGULAR with *reason = VK_PATCH_ZERO_ROW (all-zero row
 * *singular_at) or VK_PATCH_SMALL_PIVOT (|pivot of column *singular_at| <
 * 1e-12 x its source row's magnitude).  Synchronises `stream`. */
VK_API int vk_coarse_operator(vk_csr_t a, const double* q, double shift, double* dense,
                              void* stream);
VK_API int64_t vk_dense_inverse_workspace(int32_t n);
/* the factorization alone (sparsela.lu_factor, sparsela.py:63-84, for a dense
 * DEVICE matrix): lu = packed L\U (row-major, unit L below the diagonal),
 * ipiv_host[n] (may be NULL) = LAPACK's 0-based swap sequence; same guard,
 * workspace and synchronisation as vk_dense_inverse. */
VK_API int vk_dense_lu(int32_t n, const double* a, double* lu, int32_t* ipiv_host, void* work,
                       int32_t* reason, int32_t* singular_at, void* stream);
VK_API int vk_dense_inverse(int32_t n, const double* a, double* inv, void* work,
                            int32_t* reason, int32_t* singular_at, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* VANKA_B200_H */
