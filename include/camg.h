/*
 * libcamg — B200-native (sm_100a) saddle-point AMG solve path.
 *
 * C ABI: plain pointers and sizes only.  Vectors passed to the compute entry
 * points are DEVICE pointers (fp64); `stream` is a cudaStream_t passed as
 * void* (NULL = legacy default stream).  Every function returns a status code;
 * camg_last_error() returns the message of the last failure on the calling
 * thread.  Status codes map 1:1 onto the reference exception classes
 * (pkg/src/contactamg/errors.py:4-25).
 *
 * Each entry point names the reference interface it replaces
 * (paths relative to /root/reference/pkg/src/contactamg/).
 */
#ifndef CAMG_H
#define CAMG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CAMG_OK 0
#define CAMG_ERR_DIMENSION 1 /* errors.py:8  DimensionError       */
#define CAMG_ERR_SINGULAR 2  /* errors.py:12 SingularMatrixError  */
#define CAMG_ERR_CONFIG 3    /* errors.py:20 ConfigError          */
#define CAMG_ERR_SETUP 4     /* errors.py:24 SetupError           */
#define CAMG_ERR_CUDA 5      /* CUDA runtime failure (no reference counterpart) */
#define CAMG_ERR_NATIVE 6    /* other native failure */
#define CAMG_ERR_ARG 7       /* invalid argument (ValueError) */

/* block smoother kinds: smoothers.py:25 BLOCK_KINDS */
#define CAMG_UZAWA 0
#define CAMG_BRAESS_SARAZIN 1
#define CAMG_SIMPLE 2
#define CAMG_SIMPLEC 3
/* point smoother kinds: smoothers.py:24 POINT_KINDS (jacobi, sgs, ilu0,
 * direct with the reference's exact semantics; sgs / ilu0 as lexicographic
 * sync-free triangular solves) plus GPU-only variants compared by
 * convergence, never elementwise */
#define CAMG_PT_JACOBI 0
#define CAMG_PT_SGS 1       /* smoothers.py:155-164, 189-191 */
#define CAMG_PT_ILU0 2      /* smoothers.py:80-138, 193-196  */
#define CAMG_PT_DIRECT 3
#define CAMG_PT_CHEBYSHEV 4 /* GPU-only */
#define CAMG_PT_MCGS 5      /* GPU-only multicolour symmetric Gauss-Seidel: predictor on K (node-block
                               colouring, node_block), corrector on S~ (point colouring)      */
#define CAMG_PT_MCILU0 6    /* GPU-only multicolour ILU(0) corrector on S~: the reference ILU(0)
                               (smoothers.py:82-123) on the point-colour permuted S~          */
/* A_hat modes: smoothers.py:26 A_HAT_MODES */
#define CAMG_AHAT_PLAIN 0
#define CAMG_AHAT_ABS_ROWSUM 1
#define CAMG_AHAT_EXACT 2   /* test-scale: S~ = scale (Cz + B2 K^-1 B1) supplied by camg_level_set_schur,
                               A^-1 = K^-1 from camg_level_set_k_lu (smoothers.py:233-236, 272-273) */
/* coarse solvers: hierarchy.py:47 COARSE_SOLVERS */
#define CAMG_COARSE_MERGED_LU 0
#define CAMG_COARSE_BLOCK_SMOOTHER 1

typedef struct camg_csr camg_csr;
typedef struct camg_level camg_level;
typedef struct camg_hierarchy camg_hierarchy;
typedef struct camg_scalar_hierarchy camg_scalar_hierarchy;
typedef struct camg_vcycle_workspace camg_vcycle_workspace;
typedef struct camg_gmres_workspace camg_gmres_workspace;
typedef struct camg_point camg_point;

typedef struct {
  int kind;           /* CAMG_UZAWA .. CAMG_SIMPLEC                 (BlockSmootherConfig.kind)   */
  double alpha;       /*                                            (BlockSmootherConfig.alpha)  */
  int outer_sweeps;   /*                                            (.outer_sweeps)              */
  int a_hat_mode;     /* effective mode (smoothers.py:64-70)        (.a_hat_mode)                */
  int pred_kind;      /* predictor PointSmootherConfig.kind                                      */
  int pred_sweeps;
  double pred_damping;
  int corr_kind;      /* corrector PointSmootherConfig.kind                                      */
  int corr_sweeps;
  double corr_damping;
  int node_block;     /* DOFs per displacement node of the level (uniform contiguous blocks;
                         1 = none): the node colouring of a CAMG_PT_MCGS predictor on K          */
} camg_smoother_cfg;

/* execution paths reported by camg_level_get_info (which kernels a level's
 * smoother runs; several engage only above size thresholds) */
#define CAMG_PATH_NONE 0
#define CAMG_PATH_FUSED 1         /* Jacobi / Chebyshev sweeps fused into the row passes */
#define CAMG_PATH_DENSE_LU 2      /* dense LU solve (direct corrector)                    */
#define CAMG_PATH_COLOUR_CSR 3    /* one launch per colour (and direction), CSR rows      */
#define CAMG_PATH_COLOUR_SELL 4   /* one launch per colour over a colour-ordered block SELL */
#define CAMG_PATH_CTA 5           /* whole sweeps in one CTA                              */
#define CAMG_PATH_CLUSTER 6       /* whole sweeps on one 16-CTA thread-block cluster      */
#define CAMG_PATH_INNER_AMG 7     /* nested preconditioner: scalar AMG V-cycle predictor  */
#define CAMG_PATH_LEX_TRSV 8      /* lexicographic sgs / ilu0: sync-free triangular solves */
#define CAMG_PATH_LAM_FUSED 9     /* whole lambda side of a step (rc, MC-ILU(0) sweep, lambda
                                     update, B1 correction) in one 16-CTA cluster launch     */
#define CAMG_PATH_DENSE_INV 10    /* small S~: the zero-start MC-ILU(0) sweep as one dense GEMV
                                     with the explicit inverse of its factors                */
#define CAMG_PATH_LAM_ENGINE 11   /* whole lambda side of a step (rc, MC-ILU(0) forward /
                                     backward rows, lambda update, B1 correction) in one
                                     sync-free launch with per-row completion flags          */

typedef struct {
  int64_t n_u, n_lam, nnz;     /* merged operator of the level                                   */
  int sell_block;              /* node-block SELL-32 mirror of the [K | B1] rows: block size, 0 = CSR */
  int sell_masked;             /* 1: masked slots (only the union pattern of a slot stored)     */
  int sell_lanes;              /* lanes per block row of a pass: 1, 2 (pairs) or 4              */
  int64_t sell_rows, sell_slices;
  int overlap;                 /* lambda-side chain overlapped with the next [K | B1] pass      */
  int64_t overlap_indep_slices, overlap_dep_slices;
  int pred_path, pred_colors;  /* CAMG_PATH_* of the predictor on K                             */
  int corr_path, corr_colors;  /* CAMG_PATH_* of the corrector on S~                            */
  int transfer_block_rows;     /* P has a br x bc block SELL mirror: br (0 = CSR)               */
  int restrict_block_rows;     /* R = P^T has one: its block rows (0 = CSR)                     */
  int watchdog;                /* 1: a bounded device wait of this level expired (a bug; results
                                  invalid) -- reading it synchronises the device               */
  int sell_shared_values;      /* 1: bit-identical slots of the masked mirror share one stored copy
                                  (CAMG_SELL_DEDUP=0 disables)                                  */
  int64_t sell_value_groups;   /* 32-value groups the mirror stores ...                          */
  int64_t sell_value_groups_full; /* ... and before sharing                                      */
} camg_level_info;

/* ---- library ------------------------------------------------------------ */
const char* camg_last_error(void);
int camg_version(void);
int camg_device_count(int* count);
/* number of kernel launches issued by this library since load (evidence for
 * the bench's gpu_launches field) */
int64_t camg_launch_count(void);

/* ---- matrices: replaces SparseMatrix (sparse.py:24-115) ------------------ */
/* host arrays in, canonical CSR expected (sorted, no duplicates) */
int camg_csr_from_host(int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* rowptr,
                       const int64_t* col, const double* val, camg_csr** out);
/* device arrays in (copied): rowptr int64, col int32 */
int camg_csr_from_device(int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* rowptr,
                         const int32_t* col, const double* val, camg_csr** out);
int camg_csr_destroy(camg_csr* A);
int camg_csr_shape(const camg_csr* A, int64_t* n_rows, int64_t* n_cols, int64_t* nnz);
int camg_csr_to_host(const camg_csr* A, int64_t* rowptr, int64_t* col, double* val);
/* attach a block SELL-32 mirror (node blocks of size bs in {2,3,6}) of the
 * first nrows rows; SpMV / smoother kernels then stream those rows from it */
int camg_csr_attach_blocks(camg_csr* A, int bs, int64_t nrows);
/* same with br x bc blocks over the first ncols_blocked columns */
int camg_csr_attach_rect_blocks(camg_csr* A, int br, int bc, int64_t nrows, int64_t ncols_blocked);
/* 32-value groups the block mirror stores (kept) and would store without sharing
 * bit-identical slots (full); kept < full: shared value groups are in use (sell.cu) */
int camg_csr_value_groups(const camg_csr* A, int64_t* kept, int64_t* full);
/* slots of the masked mirror: out[5] = {slots, lane-uniform (one dense block, shared-value mirrors),
 * linear (block columns c0 + lane, no column index stored), both, uniform but for one or two lanes} */
int camg_csr_slot_stats(const camg_csr* A, int64_t* out);
/* out[5] = {slices of the block mirror, uniform slices: 32 consecutive block rows whose slots are all linear
 * and lane-uniform but for one or two lanes (a structured mesh row and its ends), which the pass runs without
 * descriptor decoding, groups of neighbouring uniform slices run as one work item (two or three block rows
 * per lane, values loaded once), slices with offset-aligned slots (slot j = the block at the slice's j-th
 * column offset, zero blocks where a row has none), pairs of slices with the same exception lanes a mesh-row
 * period apart run as one work item}; CAMG_SELL_USLICE=0 turns the loops off, =1 the grouping,
 * CAMG_SELL_ALIGN=0 the offset alignment, CAMG_SELL_WITEMS=0 / CAMG_SELL_XGROUPS=0 the host-made work items /
 * the exception-lane pairs */
int camg_csr_uniform_slices(const camg_csr* A, int64_t* out);
/* compulsory bytes of one SpMV pass in the matrix's current format */
int camg_csr_stream_bytes(const camg_csr* A, double* bytes);
/* merged saddle operator [[K, B1], [B2, -Cz]] (saddle.py:58-67) */
int camg_csr_saddle_merge(const camg_csr* K, const camg_csr* B1, const camg_csr* B2,
                          const camg_csr* Cz, camg_csr** out);

/* ---- sparse kernels ------------------------------------------------------ */
/* y = alpha*A*x + beta*y            spmv (sparse.py:149-154)                 */
int camg_spmv(const camg_csr* A, double alpha, const double* x, double beta, double* y,
              void* stream);
/* R = A^T, canonical                 sp_transpose (sparse.py:157-158)        */
int camg_transpose(const camg_csr* A, camg_csr** out);
/* C = A*B, canonical, exact zeros dropped, accumulation order of scipy
 *                                    sp_matmul (sparse.py:161-166)           */
int camg_spgemm(const camg_csr* A, const camg_csr* B, camg_csr** out);
/* C = (R*A)*P, canonical             galerkin_triple (sparse.py:169-173)     */
int camg_galerkin(const camg_csr* R, const camg_csr* A, const camg_csr* P, camg_csr** out);
/* d = diag(A) (mode 0) or abs row sums (mode 1), device output
 *                                    extract_diagonal (sparse.py:176-188)    */
int camg_diagonal(const camg_csr* A, int mode, double* d);
/* C = alpha*A + beta*B (same shape), canonical, exact zeros dropped          */
int camg_csr_axpby(double alpha, const camg_csr* A, double beta, const camg_csr* B,
                   camg_csr** out);
/* C = diag(s) * A  (scipy A.multiply(s[:,None])), s device                    */
int camg_csr_scale_rows(const camg_csr* A, const double* s, camg_csr** out);

/* ---- Galerkin setup (transfer.py) --------------------------------------- */
/* one power step of estimate_lambda_max (transfer.py:148-161):
 * w = (A v) / d  (device vectors)                                            */
int camg_power_step(const camg_csr* A, const double* d, const double* v, double* w, void* stream);
/* v = w / s */
int camg_vec_scale_div(int64_t n, const double* w, double s, double* v, void* stream);
/* lambda_max(D^-1 A) of estimate_lambda_max (transfer.py:148-161) with the
 * norms taken on the device (the Python path takes them with numpy on the
 * host, bit-identical to the reference); d = device diag(A) or NULL        */
int camg_lambda_max(const camg_csr* A, const double* d, int iters, double* out);
/* P = P_tent - (omega/lam_max) * (diag(1/d) A) P_tent  (transfer.py:164-183) */
int camg_smooth_prolongator(const camg_csr* P_tent, const camg_csr* A, const double* d,
                            double omega_eff, camg_csr** out);
/* S~ = scale*Cz + scale*(B2 diag(ainv) B1)  (smoothers.py:220-239) */
int camg_schur(const camg_csr* B2, const camg_csr* Cz, const camg_csr* B1, const double* ainv,
               double scale, camg_csr** out);

/* ---- aggregation (host integer work, aggregation.py) --------------------- */
/* node graph of K with cross-body and |v| <= eps*sqrt(|kii kjj|) entries
 * dropped, symmetrised (aggregation.py:127-145, :47-63), returned as a device
 * pattern matrix (fetch with camg_pattern_to_host).                          */
int camg_node_graph(const camg_csr* K, const int64_t* dof_node, int64_t num_nodes,
                    const int8_t* node_body, double eps_drop, camg_csr** graph, int64_t* nnz);
/* sparsity pattern of a device matrix into host int64 arrays (n_rows+1, nnz) */
int camg_pattern_to_host(const camg_csr* A, int64_t* indptr, int64_t* indices);
void camg_free_host(void* p);
/* three-phase greedy aggregation (aggregation.py:186-258), host */
int camg_aggregate_greedy(int64_t n, const int64_t* indptr, const int64_t* indices,
                          int64_t min_size, int64_t* node_to_agg, int64_t* num_aggs,
                          int64_t* roots, int64_t* singletons);
/* Lagrange multiplier aggregation, paper Alg. 1 (aggregation.py:261-303), host.
 * D given as host CSR.                                                        */
int camg_aggregate_lagrange(const int64_t* disp_node_to_agg, int64_t n_rows,
                            const int64_t* d_rowptr, const int64_t* d_col,
                            const double* d_val, const int64_t* slave_dofs,
                            const int64_t* row_node, const int64_t* lm_node_of_lm_dof,
                            int64_t n_lm_dofs, int64_t* lam_node_to_agg, int64_t* num_aggs,
                            int64_t* roots, int64_t* overlaps);

/* tentative prolongator CSR from host QR factors (transfer.py:86-145):
 * groups of aggregates with equal DOF count M; meta[6*g] = {G, M, kk, dof_off,
 * q_off, agg_off}; dofs[dof_off + a*M + i] = DOF i of aggregate a of the
 * group, Q[q_off + (a*M + i)*kk + c], rank/col0 per aggregate (group order).  */
int camg_tentative_csr(int64_t n_dofs, int64_t ncoarse, int64_t ngroups, const int64_t* meta,
                       const int64_t* dofs, int64_t ndofs_total, const double* Q, int64_t nq,
                       const int64_t* rank, const int64_t* col0, int64_t naggs, camg_csr** out);

/* ---- problem generator (device stiffness assembly from a stencil table) -- */
/* table: [27 types][noff][dim][dim] fp64 host; one call per block           */
int camg_assemble_stencil(int dim, const int64_t* grid, int clamp_lo, int clamp_hi,
                          int64_t node_offset, int64_t n_rows_total, const double* table,
                          camg_csr* K_inout, int64_t row_offset);
int camg_stencil_block_counts(int dim, const int64_t* grid, int clamp_lo, int clamp_hi,
                              const double* table, int64_t* nnz_out);
/* Host batched pivoted QR of G aggregate blocks of M x k (block g = rows
 * dofs[g*M .. g*M+M) of the row-major n_dofs x k null space `vecs`), for the
 * tentative prolongator (transfer.py:86-145: scipy.linalg.qr(mode="economic",
 * pivoting=True) per aggregate): LAPACK dgeqp3 + dorgqr from the library at
 * lapack_path (scipy's bundled OpenBLAS: bit-identical to the reference),
 * on nthreads host threads.  Q (G, M, kk), R (G, kk, k), piv (G, k) 0-based
 * in C order, kk = min(M, k); info_out = first block LAPACK rejected, or -1. */
int camg_qr_batch(const char* lapack_path, int64_t G, int M, int k, const double* vecs, int64_t n_dofs,
                  const int64_t* dofs, double* q_out, double* r_out, int64_t* piv_out, int nthreads,
                  int64_t* info_out);
/* The whole tentative prolongator natively (transfer.py:86-145): DOFs of
 * each aggregate (node_to_agg[dof_node[i]]) in ascending order, one LAPACK
 * pivoted QR per aggregate (as camg_qr_batch, bit-identical to the
 * reference), rank |r_ii| > rank_tol |r_00|, coarse null space R P^T rows
 * (coarse_ns: room for na*k rows of k), the CSR of P on the device.
 * rank_out: kept columns per aggregate; errors name the aggregate.       */
int camg_tentative(const char* lapack_path, int64_t n_dofs, int k, const double* vecs, const int64_t* dof_node,
                   const int64_t* node_to_agg, int64_t num_nodes, int64_t na, double rank_tol, int nthreads,
                   camg_csr** P_out, int64_t* rank_out, double* coarse_ns, int64_t* ncoarse);
/* The same with the pivoted QR on the device (tentqr.cu):
 * one warp per aggregate runs LAPACK's dlaqp2 + dorg2r algorithm in shared
 * memory.  Factors equal scipy's to rounding where the pivot order is decided
 * by more than rounding; mathematically tied columns (rotation modes of
 * symmetric aggregates) may come out in another order / sign -- the same
 * coarse space and projector P P^T in another basis.  A GPU variant compared
 * by spanned space and convergence; the bit-identical camg_tentative stays
 * the default (transfer.py: CAMG_TENTATIVE=gpu selects this one).           */
int camg_tentative_device(int64_t n_dofs, int k, const double* vecs, const int64_t* dof_node,
                          const int64_t* node_to_agg, int64_t num_nodes, int64_t na, double rank_tol,
                          camg_csr** P_out, int64_t* rank_out, double* coarse_ns, int64_t* ncoarse);
/* Allocates an empty n_rows x n_cols matrix with nnz slots (filled by
 * camg_assemble_stencil). */
int camg_csr_alloc(int64_t n_rows, int64_t n_cols, int64_t nnz, camg_csr** out);

/* ---- levels, smoothers, V-cycle (smoothers.py, hierarchy.py) ------------- */
/* BlockSmoother(cfg, op) bound to one saddle operator (smoothers.py:253-281) */
int camg_level_create(const camg_csr* K, const camg_csr* B1, const camg_csr* B2,
                      const camg_csr* Cz, const camg_smoother_cfg* cfg, int pre_sweeps,
                      int post_sweeps, camg_level** out);
/* same, borrowing an existing merged operator A = [[K,B1],[B2,-Cz]] (the
 * caller keeps A alive; one copy serves GMRES and the smoother) */
int camg_level_create_shared(camg_csr* A, const camg_csr* K, const camg_csr* B1, const camg_csr* B2,
                             const camg_csr* Cz, const camg_smoother_cfg* cfg, int pre_sweeps,
                             int post_sweeps, camg_level** out);
int camg_level_destroy(camg_level* L);
/* S~ of the bound smoother (copy) */
int camg_level_schur(const camg_level* L, camg_csr** out);
/* merged operator of the level (shared; do not destroy) */
int camg_level_operator(const camg_level* L, const camg_csr** out);
/* dense LU factors of S~ for a `direct` corrector: column-major n x n, 0-based
 * LAPACK pivots (scipy.linalg.lu_factor)                                      */
int camg_level_set_corrector_lu(camg_level* L, int64_t n, const double* lu_colmajor,
                                const int32_t* piv);
/* dense LU factors of K (column-major, 0-based LAPACK pivots): the `direct`
 * predictor (smoothers.py:182-183) and the exact A^-1 of a_hat_mode "exact"
 * (smoothers.py:272-273) */
int camg_level_set_k_lu(camg_level* L, int64_t n, const double* lu_colmajor, const int32_t* piv);
/* replace S~ (a_hat_mode "exact": scale (Cz + B2 K^-1 B1), smoothers.py:233-236)
 * and rebuild the corrector on it (copied)                                    */
int camg_level_set_schur(camg_level* L, const camg_csr* S);
/* segregated transfer (transfer.py:186-188): R = P^T computed on device */
int camg_level_set_transfer(camg_level* L, const camg_csr* P_u, const camg_csr* P_lam);
/* block SELL-32 mirrors for the transfers of a level with uniform node
 * blocks: P rows [0,nu) in bs_fine x bs_coarse blocks over the first
 * ncoarse_u columns, R = P^T rows [0,ncoarse_u) in bs_coarse x bs_fine blocks */
int camg_level_block_transfer(camg_level* L, int bs_fine, int bs_coarse, int64_t ncoarse_u);
/* one fine-level pass of the dominant smoother kernel (mode 1: fused
 * residual + first Jacobi sweep; mode 2: extra Jacobi sweep; mode 3: one
 * multicolour SGS predictor sweep, forward + backward over all colours) on
 * x, b; returns its algorithmic bytes (SURVEY §8(d) CSR model, and the
 * format's).  mode | 0x100 runs the pass through a second mirror of the rows in
 * the streaming layout (no shared value groups; built on first use), mode
 * 0x200 releases that mirror */
int camg_level_fine_pass(camg_level* L, int mode, const double* x, const double* b, void* stream,
                         double* bytes_csr_model, double* bytes_format);
/* BlockSmoother.sweep on merged vectors x, b -> out (smoothers.py:316-326) */
int camg_level_sweep(camg_level* L, const double* x, const double* b, double* out, void* stream);

/* Hierarchy (hierarchy.py:96-120).  Levels are borrowed (caller keeps them alive). */
int camg_hierarchy_create(camg_level** levels, int num_levels, int coarse_solver,
                          camg_hierarchy** out);
/* merged dense LU of the coarsest operator (hierarchy.py:242-249) */
int camg_hierarchy_set_coarse_lu(camg_hierarchy* H, int64_t n, const double* lu_colmajor,
                                 const int32_t* piv);
/* explicit inverse of the coarsest merged operator (row-major n x n, n <=
 * 4096; from the same LU factors): the coarse solve becomes two dense GEMVs
 * with one refinement step, x0 = A^-1 b, x = x0 + A^-1 (b - A x0)
 * (hierarchy.py:110-113 semantics, O(eps cond) like the LU solve)          */
int camg_hierarchy_set_coarse_inverse(camg_hierarchy* H, int64_t n, const double* inv_rowmajor);
/* LU factors (LAPACK dgetrf semantics, partial pivoting) and, up to 4096
 * rows and when `inverse`, the explicit inverse of the coarsest merged
 * operator computed on the device: replaces set_coarse_lu / set_coarse_inverse
 * for hosts without LAPACK (hierarchy.py:242-249)                          */
int camg_hierarchy_coarse_factor(camg_hierarchy* H, int inverse);
/* Hierarchy.solve_coarsest on device vectors (hierarchy.py:108-113)        */
int camg_hierarchy_coarse_solve(camg_hierarchy* H, const double* b, double* x, void* stream);
int camg_hierarchy_destroy(camg_hierarchy* H);
/* one V-cycle from zero: z = M^-1 r  (Hierarchy.apply, hierarchy.py:115-120) */
int camg_vcycle(camg_hierarchy* H, const double* r, double* z, void* stream);
/* Re-entrant application (a built hierarchy may be applied
 * concurrently to independent right-hand sides, each application owning its
 * work vectors; hierarchy.py:115-120).  A workspace owns private copies of
 * every vector a V-cycle writes plus its own CUDA graph and stream; cycles on
 * different workspaces may run concurrently (different caller streams or
 * threads).  camg_vcycle uses the hierarchy's own (default) workspace.       */
int camg_vcycle_workspace_create(camg_hierarchy* H, camg_vcycle_workspace** out);
int camg_vcycle_workspace_destroy(camg_vcycle_workspace* ws);
/* z = M^-1 r on workspace ws (NULL = the default workspace) */
int camg_vcycle_ws(camg_hierarchy* H, camg_vcycle_workspace* ws, const double* r, double* z, void* stream);
/* kernels in one recorded V-cycle graph (-1 before the first camg_vcycle) */
int camg_hierarchy_kernels_per_cycle(camg_hierarchy* H, int64_t* kernels);
/* execution paths and formats a level's smoother uses (see camg_level_info) */
int camg_level_get_info(const camg_level* L, camg_level_info* info);
/* enable/disable CUDA-graph replay of the V-cycle (default on) */
int camg_hierarchy_use_graph(camg_hierarchy* H, int enable);
/* algorithmic bytes of one V-cycle (SURVEY.md §8(d) model) */
int camg_hierarchy_vcycle_bytes(const camg_hierarchy* H, double* bytes_csr_model,
                                double* bytes_format);

/* ---- nested preconditioner (hierarchy.py:289-385) -------------------------- */
/* ScalarHierarchy (hierarchy.py:300-320) from the Python-built levels
 * (build_scalar_hierarchy, :323-363): operators A[0..n-1] (borrowed), transfers
 * P[0..n-2] (copied; R = P^T on device), one point smoother for every
 * non-coarsest level: kind CAMG_PT_JACOBI / CAMG_PT_MCGS (node colouring with
 * node_block[l] DOFs per node) / CAMG_PT_CHEBYSHEV                            */
int camg_scalar_hierarchy_create(int num_levels, const camg_csr* const* A, const camg_csr* const* P,
                                 const int* node_block, int kind, int sweeps, double damping,
                                 camg_scalar_hierarchy** out);
/* dense LU of the coarsest scalar operator (hierarchy.py:356-360) */
int camg_scalar_hierarchy_set_coarse_lu(camg_scalar_hierarchy* H, int64_t n, const double* lu_colmajor,
                                        const int32_t* piv);
/* x = one scalar V-cycle from zero on b (ScalarHierarchy.apply, :317-318) */
int camg_scalar_hierarchy_apply(camg_scalar_hierarchy* H, const double* b, double* x, void* stream);
int camg_scalar_hierarchy_destroy(camg_scalar_hierarchy* H);
/* BlockSmoother(cfg, op, predictor_solver=inner) (smoothers.py:251-278): the
 * level's predictor becomes du = inner(r_u) (NULL restores the configured
 * predictor); inner is borrowed                                              */
int camg_level_set_predictor_solver(camg_level* L, camg_scalar_hierarchy* inner);

/* ---- point smoothers (PointSmoother, smoothers.py:141-199) ---------------- */
/* kind CAMG_PT_JACOBI / SGS / ILU0 / DIRECT bound to a square A (borrowed);
 * sgs / ilu0 keep the reference's lexicographic order (sync-free triangular
 * solves); ilu0 factors on the host in the reference's IKJ order; direct
 * needs camg_point_set_lu.  Zero diagonals raise CAMG_ERR_SINGULAR naming
 * the row (smoothers.py:146-158).                                            */
int camg_point_create(const camg_csr* A, int kind, int sweeps, double damping, camg_point** out);
int camg_point_set_lu(camg_point* P, int64_t n, const double* lu_colmajor, const int32_t* piv);
/* PointSmoother.smooth(x, b) (x NULL = zero start, i.e. .apply(b)) -> out   */
int camg_point_smooth(camg_point* P, const double* x, const double* b, double* out, void* stream);
int camg_point_destroy(camg_point* P);

/* ---- Krylov (krylov.py:45-129) -------------------------------------------- */
/* right-preconditioned GMRES(restart), x0 = 0, CGS2 orthogonalisation.
 * H may be NULL (no preconditioner).  history must hold max_iters+1 values.  */
int camg_gmres(const camg_csr* A, camg_hierarchy* H, const double* b, double* x, double rel_tol,
               int max_iters, int restart, int* iterations, double* history, int* converged,
               void* stream);
/* camg_gmres keeps its Krylov basis (n x (restart+1)) and the stored
 * preconditioned vectors Z (n x restart, when 4 GB remain free) cached per
 * thread for later solves of the same size; this frees that cache.          */
int camg_gmres_release(void);
/* caller-owned GMRES workspace for systems of n rows and restart length
 * `restart` (re-entrant solves); store_z: 1 keep Z (x += Z y at
 * the end of a restart cycle, no extra V-cycle), 0 recompute, -1 keep Z when
 * 4 GB of device memory remain free at each solve                           */
int camg_gmres_workspace_create(int64_t n, int restart, int store_z, camg_gmres_workspace** out);
int camg_gmres_workspace_destroy(camg_gmres_workspace* ws);
/* caller-supplied linear map y = f(x) on device vectors of the solve's
 * length, enqueued on `stream`; returns 0 on success (the solve stops with
 * CAMG_ERR_NATIVE otherwise).  krylov.py:45's `apply_A` / `apply_Minv`
 * callables.                                                                 */
typedef int (*camg_apply_fn)(void* user, const double* x, double* y, void* stream);
/* general form of camg_gmres (krylov.py:45-129) for n unknowns: the operator
 * is the device matrix A or the callback apply_A (exactly one); the
 * preconditioner is a V-cycle of H on the V-cycle workspace vws (NULL = its
 * default), or one block-smoother sweep from zero of level L (the nested
 * preconditioner, hierarchy.py:366-376), or the callback apply_M, or none
 * (at most one).  gws NULL = the per-thread cache.                           */
int camg_gmres_ex(int64_t n, const camg_csr* A, camg_apply_fn apply_A, void* user_A, camg_hierarchy* H,
                  camg_vcycle_workspace* vws, camg_level* L, camg_apply_fn apply_M, void* user_M,
                  camg_gmres_workspace* gws, const double* b, double* x, double rel_tol, int max_iters,
                  int restart, int* iterations, double* history, int* converged, void* stream);

/* ---- dense vector helpers (device) ---------------------------------------- */
int camg_dot(int64_t n, const double* x, const double* y, double* result, void* stream);
int camg_axpy(int64_t n, double alpha, const double* x, double* y, void* stream);

/* reference ilu0_factor (smoothers.py:80-106): ILU(0) of the canonical host
 * CSR (n x n, columns strictly increasing per row) in place: the combined
 * factor values on A's pattern, unit lower diagonal implicit.  Host only (no
 * device work); a missing diagonal or zero pivot -> CAMG_ERR_SINGULAR naming
 * the row. */
int camg_ilu0_factor(int64_t n, const int64_t* rowptr, const int32_t* col, double* val);

#ifdef __cplusplus
}
#endif
#endif /* CAMG_H */
