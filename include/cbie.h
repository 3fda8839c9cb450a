/*
 * cbie.h — C-ABI of libcbie.so, the B200 (sm_100a) implementation of the
 * CBIE fill -> ACA -> H-LU hot path of the chebscat reference
 * (arXiv 2408.17116; reference sources /root/reference/pkg/src/chebscat/).
 *
 * Plain C types only: pointers + sizes, no torch / numpy types.  Host arrays
 * belong to the caller and are read/written during the call only.  Device
 * memory belongs to the handles.  Every call is synchronous on return.
 * Return value: 0 on success, else one of the CBIE_E* codes below (the
 * Python shim maps them onto the reference exception hierarchy,
 * errors.py:1-73).  cbie_last_error() gives the message.
 *
 * Index conventions (identical to the reference):
 *   points are patch-major, node flat index k*nu + l (u fastest)   geometry.py:145-155
 *   dof = point*C + component (components interleaved)               assembly.py:41-58
 *   dense outputs are row-major (numpy C order)
 */
#ifndef CBIE_H
#define CBIE_H

#define CBIE_STAR_TABLE 140

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct cbie_ctx cbie_ctx;
typedef struct cbie_hmat cbie_hmat;
typedef struct cbie_hlu cbie_hlu;
typedef struct { double re, im; } cbie_c128;   /* == numpy complex128 */

enum {
  CBIE_OK = 0,
  CBIE_ESINGULAR_DIAGONAL = 1,   /* errors.py:40  SingularDiagonal  */
  CBIE_EDEGENERATE_PATCH = 2,    /* errors.py:8   DegeneratePatch   */
  CBIE_ESINGULAR_POINT = 3,      /* errors.py:28  SingularPoint     */
  CBIE_ECAP_EXCEEDED = 4,        /* errors.py:44  CapExceeded       */
  CBIE_ERANK_OVERFLOW = 5,       /* errors.py:36  RankOverflow      */
  CBIE_ECUDA = 10,
  CBIE_ENCCL = 11,
  CBIE_EOOM = 12,
  CBIE_EINVALID = 13,
  CBIE_ESTATE = 14               /* call made before its prerequisites */
};

enum { CBIE_CHART_SAMPLES = 0, CBIE_CHART_CUBE_SPHERE = 1, CBIE_CHART_STAR = 2 };
enum { CBIE_MFIE_PEC = 0, CBIE_MULLER = 1 };
enum { CBIE_FAR = 0, CBIE_NEAR = 1, CBIE_SELF = 2 };

/* Context on one CUDA device (one process per GPU).
 * Replaces the construction of EntryGenerator (assembly.py:68-95). */
int cbie_create(int device, cbie_ctx** out);
void cbie_destroy(cbie_ctx* ctx);
const char* cbie_last_error(const cbie_ctx* ctx);

/* Number of libcbie kernel launches so far (process-wide counter). */
int64_t cbie_launch_count(void);

/* The context's CUDA stream (cudaStream_t), for event timing by the caller. */
void* cbie_stream(cbie_ctx* ctx);

/* Patch geometry, uniform order nu x nv for all patches.
 *   samples      [npatch][nu][nv][3]   == Patch.samples[l, k, :]   (geometry.py:100-117)
 *   chart_kind   [npatch]              CBIE_CHART_*
 *   chart_params [npatch][8]           cube sphere: radius, face, u_lo, u_hi, v_lo, v_hi
 *                                      (geometry.py:63-68); star: radius, face, u_lo..v_hi
 *   star_coef    [CBIE_STAR_TABLE = 140] star-chart monomial tables for CBIE_CHART_STAR, else
 *                NULL: coefficients of f = sum c_lm Y_lm (l <= 4) and of df/dx, df/dy, df/dz
 *                over the 35 monomials x^a y^b z^c of degree <= 4 (geometry.py star_tables)
 *   cheb_coef    [npatch][6][3][nu][nv] Chebyshev coefficient tensors of the samples
 *                (position, d/du, d/dv, d2/du2, d2/dudv, d2/dv2; Patch.position_coeffs +
 *                deriv_coeffs, geometry.py:137-143, 228-238) or NULL to compute them
 *                natively.  Passing the host's numpy tensors makes interpolated
 *                positions bit-identical to the reference's.
 * Replaces Patch/CubeSphereFace/eval_frames (geometry.py:48-220). */
int cbie_set_geometry(cbie_ctx* ctx, int npatch, int nu, int nv, const double* samples,
                      const int* chart_kind, const double* chart_params, const double* star_coef,
                      const double* cheb_coef);

/* Node frames computed on the device: pos/a_u/a_v [npts][3], sqrt_g [npts]
 * (Patch.node_frames, geometry.py:157-163).  Any pointer may be NULL. */
int cbie_node_frames(cbie_ctx* ctx, double* pos, double* a_u, double* a_v, double* sqrt_g);

/* Formulation and quadrature parameters (kernels.py:31-100, quadrature.py:26-56,
 * solver.py:102-117).  k1/k2 are Medium.k of outer/inner media (k2 ignored for
 * MFIE); row/col scales are the per-component equilibration factors
 * (length C = 2 or 4). */
int cbie_set_formulation(cbie_ctx* ctx, int kind, double omega, cbie_c128 k1, cbie_c128 k2,
                         cbie_c128 eps1, cbie_c128 mu1, cbie_c128 eps2, cbie_c128 mu2,
                         double tau, int grading, int oversample,
                         const cbie_c128* row_scale_c, const cbie_c128* col_scale_c);

/* FAR/NEAR/SELF classification of every (point, patch) pair plus the near
 * pair-block table.  Replaces EntryGenerator._classify_patch_column
 * (assembly.py:106-143) + quadrature.closest_points (quadrature.py:87-140)
 * + the NEAR/SELF branch of _pair_block_compute (assembly.py:191-213). */
int cbie_classify(cbie_ctx* ctx, int64_t* n_near, int64_t* n_self, int64_t* n_fallback);

/* Export of the non-FAR classification records, sorted by (point, patch). */
int cbie_export_classification(cbie_ctx* ctx, int64_t cap, int32_t* point, int32_t* patch,
                               int8_t* tag, double* u, double* v, int8_t* newton_ok);

/* One canonical pair block (C x nu*nv*C, row-major), EntryGenerator.pair_block
 * (assembly.py:146-213). */
int cbie_pair_block(cbie_ctx* ctx, int64_t point, int patch, cbie_c128* out);

/* Sub-block rows x cols (original dof ids) -> out[m][n] row-major.
 * scaled != 0 applies the equilibration (solver.py:127-129).
 * Replaces EntryGenerator.block / row_segment / col_segment / entry
 * (assembly.py:229-271) and EquilibratedGenerator (solver.py:119-129). */
int cbie_fill_block(cbie_ctx* ctx, const int64_t* rows, int64_t m, const int64_t* cols,
                    int64_t n, int scaled, cbie_c128* out);

/* Dense matrix (unscaled), assemble_dense (assembly.py:438-460); CBIE_ECAP_EXCEEDED
 * if N > cap.  out: N x N row-major host buffer. */
int cbie_fill_dense(cbie_ctx* ctx, int64_t cap, cbie_c128* out);

/* Dense path solve_dense (solver.py:178-203) on the device: assemble_dense into HBM,
 * LU with partial pivoting (scipy.linalg.lu_factor / zgetrf, solver.py:186), lu_solve
 * (zgetrs) and the residual |A x - b| / |b| (solver.py:197-198) from the kept matrix.
 *   b, x      [N][nrhs] row-major host arrays
 *   residual  out, may be NULL
 *   lu_out    [N][N] row-major packed L\U (scipy's lu) or NULL; piv_out [N] 0-based
 *             interchanges (scipy's piv) or NULL
 * CBIE_ECAP_EXCEEDED if N > cap; CBIE_ESINGULAR_DIAGONAL on an exactly singular U. */
int cbie_dense_solve(cbie_ctx* ctx, int64_t cap, const cbie_c128* b, int nrhs, cbie_c128* x,
                     double* residual, cbie_c128* lu_out, int32_t* piv_out);

/* H-matrix from host-evaluated leaves (any generator of the reference's protocol, e.g.
 * the reference tests' KernelGen / IdGen / ZeroGen, tests/test_hmatrix.py:9-36, 228-274):
 *   cbie_hmatrix_layout  host only: cluster + block tree of a point cloud
 *                        (build_cluster_tree / build_block_tree, hmatrix.py:82, 344);
 *                        dof_perm [npts*C] (new -> original dof), leaves [nleaf][5]
 *                        (r_lo, r_hi, c_lo, c_hi in permuted points, admissible); NULL ok
 *   cbie_hmatrix_import  data = every leaf's block, row-major m x n over the permuted
 *                        dofs, concatenated in leaf order; dense leaves stored, admissible
 *                        ones compressed on the device (truncated SVD, s > tol s_0) and
 *                        demoted above min(m, n) / 2 (HMatrix._fill_leaf, hmatrix.py:243-264).
 *                        The handle takes cbie_hlu_factor / cbie_hmatvec like a built one. */
/* Host only: the layout of the sharded H-matrix after the exchange (csrc/shard.cu,
 * shard_layout), a pure function of the leaf shapes m[], n[], admissibility adm[],
 * owners (cbie_partition_lpt) and the all-reduced info[2 * leaf] = (rank, demoted):
 * leaf_off [nleaf][3] dense / U / V arena offsets (-1: none), ranges [world][4] each
 * owner's dense range and tail (the spans it broadcasts), total = arena elements. */
int cbie_shard_layout_host(int nleaf, const int* m, const int* n, const uint8_t* adm, const int* owner,
                           const int* info, int world, int64_t* leaf_off, int64_t* ranges, int64_t* total);

/* Move the H-matrix leaf data to pinned host memory mapped into the device address
 * space; the handle stays usable (factor / matvec read it over the host link) and its
 * device memory is released -- for problems whose H-matrix and factors do not fit HBM
 * together (config 5). */
int cbie_hmatrix_offload(cbie_hmat* h);

int cbie_hmatrix_layout(const double* pts, int64_t npts, int C, int n_leaf, double eta, int64_t* dof_perm,
                        int64_t* leaves, int64_t* nleaf);
int cbie_hmatrix_import(cbie_ctx* ctx, const double* pts, int64_t npts, int C, int n_leaf, double eta, double tol,
                        const cbie_c128* data, cbie_hmat** out);

/* H-matrix of the equilibrated system: cluster tree, block tree, dense leaves,
 * batched ACA + recompression, demotion.  Replaces build_hmatrix
 * (solver.py:132-145): build_cluster_tree (hmatrix.py:82), build_block_tree
 * (hmatrix.py:344), HMatrix.fill (hmatrix.py:207-264), aca (352-409),
 * truncate_lowrank (412-426). */
int cbie_hmatrix_build(cbie_ctx* ctx, int n_leaf, double eta, double aca_tol, cbie_hmat** out);
void cbie_hmatrix_destroy(cbie_hmat* h);

/* Tree export: dof_perm[N] (new -> original, ClusterTree.dof_perm), leaves
 * [nleaf][6] = r_lo, r_hi, c_lo, c_hi (point units, permuted order), kind
 * (0 dense, 1 low rank), rank. Pass NULL to query *nleaf only. */
int cbie_hmatrix_tree(cbie_hmat* h, int64_t* dof_perm, int64_t* leaves, int64_t* nleaf);

/* One leaf in permuted local order (row-major): dense -> D[m][n];
 * low rank -> U[m][rank], V[rank][n].  hmatrix.py:96-143 */
int cbie_hmatrix_leaf(cbie_hmat* h, int64_t leaf, int* kind, int* rank, cbie_c128* D_or_U,
                      cbie_c128* V);

/* y = H x for nrhs column vectors in ORIGINAL dof order, x/y [N][nrhs] row-major.
 * HMatrix.matvec (hmatrix.py:267-274). */
int cbie_hmatvec(cbie_hmat* h, const cbie_c128* x, cbie_c128* y, int nrhs);

/* Restarted GMRES on the device H-matvec (gmres / solve_gmres, solver.py:206-307):
 * zero initial guess, restart length `restart`, one re-orthogonalisation pass,
 * complex Givens rotations; b, x [N] in original dof order.  *iterations = inner
 * iterations, *rel_residual = |b - H x| / |b|, *converged = 0 / 1. */
int cbie_gmres(cbie_hmat* h, const cbie_c128* b, double tol, int restart, int max_iters, cbie_c128* x,
               int* iterations, double* rel_residual, int* converged);

/* H-LU of the H-matrix (copy; h unchanged).  hlu_factor (hmatrix.py:827-858). */
int cbie_hlu_factor(cbie_hmat* h, double trunc_tol, cbie_hlu** out);
void cbie_hlu_destroy(cbie_hlu* f);

/* One leaf of the H-LU factors (same layout as cbie_hmatrix_leaf); factored
 * diagonal leaves return LAPACK-style combined L\U in D and 0-based row
 * pivots in piv (may be NULL).  kind: 0 dense, 1 low rank, 2 factored. */
int cbie_hlu_leaf(cbie_hlu* f, int64_t leaf, int* kind, int* rank, cbie_c128* D_or_U,
                  cbie_c128* V, int32_t* piv);

/* x = (LU)^{-1} b, original dof order, [N][nrhs] row-major.
 * HLUFactors.solve (hmatrix.py:807-816). */
int cbie_hlu_solve(cbie_hlu* f, const cbie_c128* b, cbie_c128* x, int nrhs);

/* Far-field radiation sums (postprocess.far_field, postprocess.py:193-212):
 * out[a][t] = sum_n exp(j k rhat_a . pos_n) tab[n][t] over the context's
 * quadrature nodes (cbie_node_frames order); tab [npts][ntab] row-major
 * (ntab <= 8: the w J, w div J [, w M, w div M] tables), rhat [nang][3]. */
int cbie_far_field_sums(cbie_ctx* ctx, const cbie_c128* tab, int ntab, const double* rhat, int nang,
                        double k, cbie_c128* out);

/* Low-rank recompression of host data (truncate_lowrank, hmatrix.py:412-426):
 * U [m][k] row-major, V [k][n] row-major -> Uo [m][*r], Vo [*r][n] (capacity
 * min(m, n, k) rows/cols).  V == NULL: truncated SVD of the dense U [m][n]
 * (hmatrix.py:605-609, k ignored). */
int cbie_lowrank_truncate(cbie_ctx* ctx, const cbie_c128* U, int m, int k, const cbie_c128* V,
                          int n, double tol, int* r, cbie_c128* Uo, cbie_c128* Vo);

/* Development benchmark of the Gram-path recompression kernel (no reference
 * counterpart; tools/trunc_bench.py): nprob synthetic problems U (m x k), Vt (n x k)
 * of numerical rank ~r_true, recompressed reps times on clusters of csize CTAs.
 * ms_out: mean launch time [1]; prof_out: cycle counters [32]; ranks_out [nprob]. */
int cbie_trunc_bench(cbie_ctx* ctx, int m, int n, int k, int r_true, int nprob, double tol, int csize,
                     int reps, float* ms_out, unsigned long long* prof_out, int* ranks_out);

/* ---- multi-GPU fill (one process per GPU, NCCL over NVLink / NVSwitch) ----
 * The reference fills leaves with a thread pool over HMatrix._fill_leaf
 * (hmatrix.py:207-224, 243-264); here each process fills the leaves it owns and
 * the shards are exchanged with ncclBroadcast. */

/* Deterministic LPT partition of n work items (leaves) over `world` owners by
 * cost (largest first, each to the least-loaded owner, ties to the lowest rank).
 * Host-only, no GPU needed. */
void cbie_partition_lpt(const double* cost, int64_t n, int world, int* owner);

/* ncclGetUniqueId into out (cap >= 128 bytes); rank 0 creates it, the caller
 * distributes it (torch.distributed / any side channel). */
int cbie_nccl_unique_id(char* out, int cap);

/* NCCL communicator of this context (rank, world); cbie_dist_finalize drops it. */
int cbie_dist_init(cbie_ctx* ctx, const char* nccl_id, int rank, int world);
void cbie_dist_finalize(cbie_ctx* ctx);

/* cbie_hmatrix_build with leaf sharding: this process fills the leaves the LPT
 * partition gives `rank`; exchange != 0 broadcasts the shards (needs
 * cbie_dist_init with the same rank / world) so every rank holds the complete
 * H-matrix.  exchange == 0 leaves a partial H-matrix (cbie_hmatrix_leaf reports
 * kind -1 for leaves owned elsewhere) -- used to check the shards on one GPU. */
int cbie_hmatrix_build_shard(cbie_ctx* ctx, int n_leaf, double eta, double aca_tol, int rank,
                             int world, int exchange, cbie_hmat** out);

/* Block-row-distributed H-LU (replaces the single-core recursion
 * hlu_factor / _factor, hmatrix.py:827-858): every rank of the cbie_dist_init
 * communicator records the same tape, runs the tasks of the block rows it owns
 * (row clusters dealt cyclically at the first tree level with >= 2 world
 * clusters) and exchanges the factored diagonal blocks / panels its peers read
 * with ncclSend / ncclRecv between dependency levels; at the end every owner
 * broadcasts its factored leaves, so every rank holds complete factors
 * (cbie_hlu_solve / cbie_hlu_leaf as for cbie_hlu_factor).  Collective: every
 * rank calls it with the same complete H-matrix. */
int cbie_hlu_factor_dist(cbie_hmat* h, double trunc_tol, cbie_hlu** out);

/* The same distributed plan executed by `world` virtual ranks inside this
 * process on one GPU (one arena per virtual rank, device copies instead of
 * NCCL) -- checks the ownership / transfer plan without several GPUs. */
int cbie_hlu_factor_emulated(cbie_hmat* h, double trunc_tol, int world, cbie_hlu** out);

/* Host only (no GPU): the distributed H-LU plan of the block structure of the
 * points pts [npts][3] (leaf size n_leaf dofs, admissibility eta), low-rank
 * capacities from an assumed rank min(m, n) / 8.  stats[11] = tasks, messages,
 * transferred buffers, transferred complex elements, write conflicts (always 0:
 * a conflict is an error), dependency levels, block-row tree level, fewest /
 * most tasks of a rank, complex elements of the final factor broadcast,
 * leaves; leaf_owner[nleaf] (may be NULL) = owning rank of every leaf. */
int cbie_hlu_dist_plan_host(const double* pts, int64_t npts, int C, int n_leaf, double eta, int world,
                            int64_t* stats, int32_t* leaf_owner);

/* Timings (CUDA events), counts, flops, bytes as one JSON object.
 * which: 0 = context, 1 = hmatrix, 2 = hlu. */
int cbie_stats_json(const void* handle, int which, char* buf, size_t cap);

#ifdef __cplusplus
}
#endif
#endif /* CBIE_H */
