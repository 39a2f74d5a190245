/* ldgmg_b200.h -- C ABI of the B200-native multigrid V-cycle core.
 *
 * Drop-in boundary for the FP64 block-sparse hot path of the reference
 * (`ldgmg`, arXiv 2412.12506, /root/reference/proj/include/ldgmg/).  The
 * reference has no FFI: its "operator API" is the header-only C++ surface in
 * blockla.hpp / smoothers.hpp / multigrid.hpp.  Every entry point below
 * replaces one of those functions; the replaced signature is cited per entry.
 * The C++ wrapper include/ldgmg_b200.hpp re-exposes them with the reference
 * class names (ldgmg::gpu::{BlockCsr,Smoother,Multigrid}) and maps the status
 * codes back to the reference's exception types.
 *
 * Conventions
 *  - Plain pointers and sizes only; no torch or CUDA types in signatures
 *    (streams are passed as void* = cudaStream_t).
 *  - Host arrays use the reference layouts: BlockCsr ptr/col int32, blocks
 *    row-major (inc/blockla.hpp:73-92); vectors element-major (BlockVec::data,
 *    inc/blockla.hpp:46-58).
 *  - Functions taking `const double* x` / `double* y` without a _host suffix
 *    take DEVICE pointers on the context's device; work is enqueued on the
 *    context stream (asynchronous unless stated).
 *  - Every function returns LDGMG_OK or an error code; ldgmg_last_error()
 *    returns the thread-local message, which repeats the reference's exception
 *    text where one exists (e.g. "spmv: shape mismatch", blockla.hpp:137).
 *  - No CPU fallback: without a visible CUDA device every compute entry point
 *    fails with LDGMG_ERR_CUDA.
 */
#ifndef LDGMG_B200_H
#define LDGMG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LDGMG_B200_ABI_VERSION 1

/* status codes -> reference exception types (include/ldgmg_b200.hpp) */
#define LDGMG_OK 0
#define LDGMG_ERR_INVALID_ARGUMENT 1 /* std::invalid_argument */
#define LDGMG_ERR_RUNTIME 2          /* std::runtime_error    */
#define LDGMG_ERR_LOGIC 3            /* std::logic_error      */
#define LDGMG_ERR_CUDA 4             /* device / driver failure, no device */
#define LDGMG_ERR_NCCL 5             /* collective failure */

/* enum values mirror the reference enums */
enum { LDGMG_SWEEP_FORWARD = 0, LDGMG_SWEEP_REVERSE = 1 };               /* smoothers.hpp:19 */
enum { LDGMG_JACOBI = 0, LDGMG_COLOURED_GS = 1, LDGMG_PROC_BLOCK_GS = 2, /* smoothers.hpp:21 */
       LDGMG_SAI = 3 };
enum { LDGMG_SYSTEM_SCALAR = 0, LDGMG_SYSTEM_STOKES = 1 };              /* ldg_core.hpp:40 */
enum { LDGMG_BC_PERIODIC = 0, LDGMG_BC_DIRICHLET = 1, LDGMG_BC_NEUMANN = 2 }; /* mesh.hpp:28 */
enum { LDGMG_PHASE_SINGLE = 0, /* one phase (PhaseGeometry::single)                        */
       LDGMG_PHASE_BOXES = 1,  /* inner box (lo,hi) + background (harness.hpp:58-64)       */
       LDGMG_PHASE_BALL = 2,   /* centroid inside ball/ellipse (extension A2, re-tested on  */
       LDGMG_PHASE_ELLIPSE = 3 /*   every level)                              */
};

/* SmootherConfig (smoothers.hpp:23-58) */
typedef struct ldgmg_smoother_config {
    int kind;       /* LDGMG_JACOBI ... LDGMG_SAI */
    double omega;   /* damping; coloured GS always runs undamped */
    int partitions; /* processor-block GS only */
    int level;      /* SAI pattern power */
    double zeta;    /* SAI pressure balance weight */
    int cache;      /* SAI least-squares dedupe (bitwise transparent) */
} ldgmg_smoother_config;

/* MultigridConfig (multigrid.hpp:26-36) */
typedef struct ldgmg_mg_config {
    ldgmg_smoother_config smoother;
    int pre, post; /* LDGMG_SWEEP_* */
    int nu1, nu2;
    int bottom_max_elements;
    double bottom_tol;
    int min_depth;
} ldgmg_mg_config;

/* SaiStats (smoothers.hpp:132-138) */
typedef struct ldgmg_sai_stats {
    int rank_deficient_columns;
    int64_t cache_hits, cache_misses;
    int n_shapes;        /* distinct (row blocks, col blocks) local LS shapes */
    int shape_rows[8];   /* first 8 shapes, ascending like std::map */
    int shape_cols[8];
    int shape_count[8];
} ldgmg_sai_stats;

/* Problem description for the built-in host setup (mesh chain + LDG assembly
 * per level).  Mirrors harness.hpp:30-40 plus the BASELINE config knobs.     */
typedef struct ldgmg_problem_spec {
    int kind;          /* LDGMG_SYSTEM_SCALAR / _STOKES */
    int dim;           /* 2 or 3 */
    int n;             /* elements per axis (power of two; any n >= 2 with LDGMG_PROBLEM_ANY_N) */
    int degree;        /* polynomial degree p */
    int bc[6];         /* per side 2*axis+{0 lower,1 upper}: LDGMG_BC_* */
    double beta;       /* <=0: 4 p^2 (library default, ldg_core.hpp:101) */
    double beta_p;     /* Stokes pressure penalty scale */
    double gamma;      /* Stokes form: 0 standard, 1 stress */
    double delta;      /* Stokes time step; <=0 steady */
    int phase_shape;   /* LDGMG_PHASE_* */
    double center[3];  /* ball/ellipse centre, or box lo */
    double radii[3];   /* ball radius in radii[0] / ellipse semi-axes, or box hi */
    double mu_in, mu_out, rho_in, rho_out;
} ldgmg_problem_spec;

typedef struct ldgmg_ctx ldgmg_ctx;
typedef struct ldgmg_bsr ldgmg_bsr;
typedef struct ldgmg_smoother ldgmg_smoother;
typedef struct ldgmg_transfer ldgmg_transfer;
typedef struct ldgmg_mg ldgmg_mg;
typedef struct ldgmg_problem ldgmg_problem;

/* ------------------------------------------------------------------ misc */
const char* ldgmg_last_error(void);
int ldgmg_abi_version(void);
/* Number of kernel launches this process issued (all contexts); counter for
 * bench.py's gpu_launches claim. */
int64_t ldgmg_launch_count(void);

/* --------------------------------------------------------------- context */
int ldgmg_ctx_create(int device, ldgmg_ctx** out);
int ldgmg_ctx_destroy(ldgmg_ctx* ctx);
int ldgmg_ctx_set_stream(ldgmg_ctx* ctx, void* cuda_stream);
void* ldgmg_ctx_stream(ldgmg_ctx* ctx);
int ldgmg_ctx_synchronize(ldgmg_ctx* ctx);
/* device scratch helpers for C callers without their own allocator */
int ldgmg_device_alloc(ldgmg_ctx* ctx, size_t bytes, void** ptr);
int ldgmg_device_free(ldgmg_ctx* ctx, void* ptr);
int ldgmg_copy_h2d(ldgmg_ctx* ctx, void* dst, const void* src, size_t bytes);
int ldgmg_copy_d2h(ldgmg_ctx* ctx, void* dst, const void* src, size_t bytes);

/* ------------------------------------------------------------ BSR (L1)
 * replaces BlockCsr (inc/blockla.hpp:73-92) / BlockBuilder::freeze (:113-132) */
int ldgmg_bsr_upload(ldgmg_ctx* ctx, int brows, int bcols, int row_bs, int col_bs,
                     const int* ptr, const int* col, const double* val, ldgmg_bsr** out);
int ldgmg_bsr_shape(const ldgmg_bsr* A, int* brows, int* bcols, int* row_bs, int* col_bs,
                    int64_t* nnzb);
/* download back to the reference layout (row-major blocks) */
int ldgmg_bsr_download(ldgmg_ctx* ctx, const ldgmg_bsr* A, int* ptr, int* col, double* val);
/* bytes of device memory the operator occupies (values + indices) */
int64_t ldgmg_bsr_device_bytes(const ldgmg_bsr* A);
int ldgmg_bsr_destroy(ldgmg_bsr* A);

/* Block-coordinate text format (replaces dump_block_coo, blockla.hpp:253-268;
 * the load side is the BlockBuilder round trip of tests/test_blockla.cpp:207-230:
 * duplicates summed in file order, ascending columns).  Device variants
 * download / upload; the _host variants touch no GPU.  coo_read_host is
 * two-phase: with ptr == NULL it only reports the shape and nnzb. */
int ldgmg_bsr_dump_coo(ldgmg_ctx* ctx, const ldgmg_bsr* A, const char* path);
int ldgmg_bsr_load_coo(ldgmg_ctx* ctx, const char* path, ldgmg_bsr** out);
int ldgmg_coo_write_host(const char* path, int brows, int bcols, int row_bs, int col_bs, const int* ptr,
                         const int* col, const double* val);
int ldgmg_coo_read_host(const char* path, int* brows, int* bcols, int* row_bs, int* col_bs, int64_t* nnzb,
                        int* ptr, int* col, double* val);

/* Upload a rank-local slice whose column indices are renumbered (owned
 * columns first, then ghost slots): block order inside each row must stay
 * the global ascending order, so columns need not ascend locally.
 * flags: LDGMG_BSR_UNSORTED_COLUMNS. */
#define LDGMG_BSR_UNSORTED_COLUMNS 1
int ldgmg_bsr_upload_ex(ldgmg_ctx* ctx, int brows, int bcols, int row_bs, int col_bs,
                        const int* ptr, const int* col, const double* val, int flags,
                        ldgmg_bsr** out);

/* Batched FP64 GEMM on the tensor cores (mma.sync m8n8k4 DMMA), the kernel
 * behind the SAI setup's least-squares solves (dense_lstsq blockla.hpp:
 * 278-309 -> dgels; its compact-WY trailing updates):
 *   D[b](m, n) = alpha * sum_k A[b](m, k) * B[b](n, k) + beta * D[b](m, n)
 * A(m, k) at A + b*strideA + m*lda + k, B(n, k) at B + b*strideB + n*ldb + k
 * (k contiguous in both), D(m, n) at D + b*strideD + m + n*ldd (column-major);
 * device pointers, batch <= 65535. */
int ldgmg_dgemm_nt_batched(ldgmg_ctx* ctx, int M, int N, int K, double alpha, const double* A, int64_t lda,
                           int64_t strideA, const double* B, int64_t ldb, int64_t strideB, double beta, double* D,
                           int64_t ldd, int64_t strideD, int batch);

/* Values of blocks [first_block, first_block + nblocks) in the reference's
 * layout (row-major blocks, BlockCsr::val order); a matrix uploaded with
 * val == NULL starts from zero blocks.  Streams a BlockBuilder::freeze'd
 * operator (blockla.hpp:113-132) in pieces: the distributed setup fills a
 * rank's rows from several host slices without concatenating them. */
int ldgmg_bsr_set_values(ldgmg_ctx* ctx, ldgmg_bsr* A, int64_t first_block, int64_t nblocks,
                         const double* val);
/* A new matrix with pattern (ptr, col) whose block q is a device-side copy
 * of src's block src_blocks[q] (host int64 array, nnzb entries): a rank's
 * rows of a device-assembled operator with its local column numbering,
 * cut without moving the values through the host. */
int ldgmg_bsr_gather(ldgmg_ctx* ctx, const ldgmg_bsr* src, int brows, int bcols, const int* ptr, const int* col,
                     const int64_t* src_blocks, ldgmg_bsr** out);
/* The first nrows block rows of `base` as a matrix of their own (values
 * shared, not copied; `base` must outlive the view).  Distributed B: the
 * forward sweep's rank rows of a matrix that also stores the ghost rows the
 * transposed sweep needs. */
int ldgmg_bsr_row_prefix_view(ldgmg_ctx* ctx, const ldgmg_bsr* base, int nrows, ldgmg_bsr** out);
/* A transposed VIEW with its own pattern: block q of the result is block
 * perm[q] of `base` read transposed (no copy).  spmv_transpose's scatter
 * order (blockla.hpp:157-176, source rows ascending) is the caller's choice
 * of (ptr, col, perm).  The distributed B^T: a rank's B^T rows (its columns
 * of B) read from the B rows it stores. */
int ldgmg_bsr_transposed_view(ldgmg_ctx* ctx, const ldgmg_bsr* base, int brows, int bcols, const int* ptr,
                              const int* col, const int* perm, ldgmg_bsr** out);

/* Memory-safety net (no reference counterpart): with LDGMG_GUARD_BYTES=G in
 * the environment every library allocation carries G-byte guard zones; the
 * check returns how many zones were overwritten so far (out-of-bounds
 * writes), -1 when guards are off.  live = guarded allocations alive. */
int64_t ldgmg_debug_guard_check(void);
int64_t ldgmg_debug_guard_live(void);

/* replaces spmv(const BlockCsr&, const BlockVec&, BlockVec&)  blockla.hpp:136-154 */
int ldgmg_spmv(ldgmg_ctx* ctx, const ldgmg_bsr* A, const double* x, double* y);
/* replaces spmv_transpose(...)                                 blockla.hpp:157-176 */
int ldgmg_spmv_transpose(ldgmg_ctx* ctx, const ldgmg_bsr* A, const double* x, double* y);
/* r = b - A x (multigrid.hpp:256-258, smoothers.hpp:439-440), fused */
int ldgmg_residual(ldgmg_ctx* ctx, const ldgmg_bsr* A, const double* b, const double* x,
                   double* r);
/* y += A x  (the SAI update x += B r, smoothers.hpp:441-446, as one pass) */
int ldgmg_spmv_add(ldgmg_ctx* ctx, const ldgmg_bsr* A, const double* x, double* y);
/* residual / spmv_add restricted to the block rows `rows` (device int32):
 * the interior / boundary halves of a distributed pass (the interior runs
 * while the ghost layer is in flight); per-row arithmetic is unchanged */
int ldgmg_residual_rows(ldgmg_ctx* ctx, const ldgmg_bsr* A, const double* b, const double* x, double* r,
                        const int* rows, int nrows);
int ldgmg_spmv_add_rows(ldgmg_ctx* ctx, const ldgmg_bsr* A, const double* x, double* y, const int* rows,
                        int nrows);
/* Processor-block GS on one rank (smoothers.hpp:426-436 with partitions =
 * ranks): wavefront schedule of the sequential sweep over the rank's n_own
 * rows (local CSR; columns >= n_own are frozen ghosts).  rows (n_own) and
 * level_ptr (nlevels + 1) may be NULL to query nlevels. */
int ldgmg_pgs_schedule(int n_own, const int* ptr, const int* col, int reverse, int* rows, int* level_ptr,
                       int* nlevels);

/* Block-diagonal relaxation of every row of a (possibly rank-local,
 * rectangular) operator with caller-held factors: x_out[e] = (1-w) x_live[e]
 * + w s o pinv(V, lambda)(s o (b_e - sum_{j != e} A_ej x_src[j]))
 * (smoothers.hpp:496-518).  Row e's diagonal block is the one whose column
 * index equals diag_col_offset + e. */
typedef struct ldgmg_factors ldgmg_factors;
int ldgmg_factors_upload(ldgmg_ctx* ctx, int n, int bs, const double* V, const double* lambda,
                         const double* s, ldgmg_factors** out);
int ldgmg_factors_destroy(ldgmg_factors* F);
int ldgmg_relax(ldgmg_ctx* ctx, const ldgmg_bsr* A, const ldgmg_factors* F, const double* b,
                const double* x_src, const double* x_live, double* x_out, double omega);
/* the same restricted to the block rows `rows` (device int32, nrows entries):
 * one colour phase of coloured GS on a rank's rows */
int ldgmg_relax_rows(ldgmg_ctx* ctx, const ldgmg_bsr* A, const ldgmg_factors* F, const double* b,
                     const double* x_src, const double* x_live, double* x_out, double omega, const int* rows,
                     int nrows);

/* out[i*bs .. i*bs+bs) = x[idx[i]*bs ..]  (ghost-exchange packing; idx on the device) */
/* Kernel projection of a rank's element slice [r0, r1) of an N-element
 * vector in the deterministic fast mode (256 fixed global element ranges, one
 * fixed-tree partial per range; the slice must be a union of ranges, true for
 * contiguous partitions into P | 256 parts).  partials: 256 * ncomp doubles,
 * the slice's ranges written; apply needs all 256 * ncomp (gathered). */
int ldgmg_project_partials(ldgmg_ctx* ctx, const double* v_own, int N, int r0, int r1, int bs, const int* offs,
                           int ncomp, double kval, double* partials);
int ldgmg_project_apply(ldgmg_ctx* ctx, double* v_own, int N, int r0, int r1, int bs, const int* offs, int ncomp,
                        double kval, const double* partials);
int ldgmg_gather_blocks(ldgmg_ctx* ctx, const double* x, const int* idx, int n, int bs, double* out);

/* Partition plan of one level for `nranks` contiguous element ranges
 * [p*N/P, (p+1)*N/P) (partition_ranges, smoothers.hpp:87-94).  Host-only.
 * Phase 1 (local_col / send_idx NULL): sizes.  Phase 2: fills
 *   local_col[nnz_local]   : columns of the owned rows renumbered (owned j -> j-r0,
 *                            ghost j -> n_owned + slot), block order unchanged
 *   ghost_gid[n_ghost]     : global ids of the ghost slots, grouped by owner rank,
 *                            ascending inside each group
 *   recv_count[nranks]     : ghost slots received from each rank (consecutive)
 *   send_count[nranks]     : owned elements each rank needs from us
 *   send_idx[n_send]       : their local (owned) indices, grouped by rank, ascending gid
 * The ghost set of rank p is the column set of its rows (A pattern); the send
 * lists are derived from the other ranks' rows (structurally symmetric or not). */
int ldgmg_partition_level(int N, const int* ptr, const int* col, int nranks, int rank, int* r0,
                          int* r1, int* n_ghost, int* n_send, int* local_col, int* ghost_gid,
                          int* recv_count, int* send_count, int* send_idx);

/* BLAS-1 (blockla.hpp:60-71); dot/norm write one double to *out_host (synchronous) */
int ldgmg_dot(ldgmg_ctx* ctx, int64_t n, const double* a, const double* b, double* out_host);
int ldgmg_axpy(ldgmg_ctx* ctx, int64_t n, double alpha, const double* x, double* y);

/* ------------------------------------------------------- smoothers (L3)
 * replaces Smoother(const System&, const SmootherConfig&, SaiCache*)
 * (smoothers.hpp:377-404).  `system_kind`/`n_velocity` carry the System
 * fields the smoother reads (ldg_core.hpp:44-59).  Setup (diagonal factors,
 * colouring, SAI least squares) runs on the GPU. */
int ldgmg_smoother_create(ldgmg_ctx* ctx, const ldgmg_bsr* A, int system_kind, int n_velocity,
                          const ldgmg_smoother_config* cfg, ldgmg_smoother** out);
/* Drop-in variants: adopt setup computed by the caller's reference objects
 * (factor_diagonal smoothers.hpp:464-494 / build_sai :259-367), host arrays. */
int ldgmg_smoother_create_with_factors(ldgmg_ctx* ctx, const ldgmg_bsr* A,
                                       const ldgmg_smoother_config* cfg, const double* V,
                                       const double* lambda, const double* s,
                                       ldgmg_smoother** out);
int ldgmg_smoother_create_with_sai(ldgmg_ctx* ctx, const ldgmg_bsr* A,
                                   const ldgmg_smoother_config* cfg, const int* Bptr,
                                   const int* Bcol, const double* Bval, ldgmg_smoother** out);
/* replaces Smoother::apply(const BlockVec& b, BlockVec& x, Sweep)  smoothers.hpp:406-450 */
int ldgmg_smoother_apply(ldgmg_ctx* ctx, const ldgmg_smoother* S, const double* b, double* x,
                         int sweep);
/* accessors: colours() / n_colours() / sai_matrix() / sai_stats() (smoothers.hpp:452-461) */
int ldgmg_smoother_colours(const ldgmg_smoother* S, int* colour /* N or NULL */, int* ncolours);
int ldgmg_smoother_sai_nnzb(const ldgmg_smoother* S, int64_t* nnzb);
int ldgmg_smoother_sai_matrix(ldgmg_ctx* ctx, const ldgmg_smoother* S, int* ptr, int* col,
                              double* val);
int ldgmg_smoother_sai_stats(const ldgmg_smoother* S, ldgmg_sai_stats* out);
/* replaces build_sai(System, level, zeta, SaiCache*, SaiStats*) (smoothers.hpp:259-367)
 * on a device operator: B on the pattern of A^level.  `col_mask` (NULL or
 * N ints) restricts the least-squares solves to the columns with a nonzero
 * entry (distributed setup); the other columns of B stay zero. */
int ldgmg_sai_build(ldgmg_ctx* ctx, const ldgmg_bsr* A, int system_kind, int n_velocity, int level,
                    double zeta, int cache, const int* col_mask, ldgmg_bsr** B, ldgmg_sai_stats* stats);
/* per-element diagonal factors V (bs*bs, column-major like Eigen), lambda, s */
int ldgmg_smoother_diag_factors(ldgmg_ctx* ctx, const ldgmg_smoother* S, double* V,
                                double* lambda, double* s);
int ldgmg_smoother_destroy(ldgmg_smoother* S);

/* ---------------------------------------------------- transfers (L4)
 * parent_of/orthant_of from coarsen() (mesh.hpp:412-457); K = the 2^dim
 * injection matrices of build_injection() (multigrid.hpp:212-241), each
 * bs_scalar x bs_scalar row-major. */
int ldgmg_transfer_create(ldgmg_ctx* ctx, int n_fine, int n_coarse, const int* parent_of,
                          const int* orthant_of, int dim, int bs_scalar, int n_comp,
                          const double* K, ldgmg_transfer** out);
/* replaces Multigrid::restrict_residual (multigrid.hpp:127-149); rc overwritten */
int ldgmg_restrict(ldgmg_ctx* ctx, const ldgmg_transfer* T, const double* rf, double* rc);
/* replaces Multigrid::interpolate_add (multigrid.hpp:104-123) */
int ldgmg_interpolate_add(ldgmg_ctx* ctx, const ldgmg_transfer* T, const double* xc, double* xf);
int ldgmg_transfer_destroy(ldgmg_transfer* T);

/* ------------------------------------------------- multigrid hierarchy
 * replaces Multigrid(Mesh, const LevelAssembler&, MultigridConfig)
 * (multigrid.hpp:49-65) given the already assembled level operators.
 * A[l] for l < depth; transfers[l] for l < depth-1.  kernel_* are the System
 * flags of level 0 (ldg_core.hpp:52-53).  When bottom_V/bottom_lambda are NULL
 * the bottom eigendecomposition is computed on the GPU. */
int ldgmg_mg_create(ldgmg_ctx* ctx, int depth, const ldgmg_bsr* const* A,
                    const ldgmg_transfer* const* transfers, int system_kind, int dim, int n_comp,
                    int bs_scalar, int kernel_constants, int kernel_pressure,
                    const ldgmg_mg_config* cfg, const double* bottom_V,
                    const double* bottom_lambda, ldgmg_mg** out);
/* Adopt per-level drop-in smoothers instead of building them (optional). */
int ldgmg_mg_set_smoother(ldgmg_mg* mg, int level, ldgmg_smoother* S);
int ldgmg_mg_smoother(ldgmg_mg* mg, int level, ldgmg_smoother** out);
int ldgmg_mg_depth(const ldgmg_mg* mg);
/* replaces Multigrid::cycle(BlockVec& x, const BlockVec& b)  multigrid.hpp:82-85 */
int ldgmg_mg_cycle(ldgmg_ctx* ctx, ldgmg_mg* mg, double* x, const double* b);
/* the bare recursive v_cycle(0, x, b) (multigrid.hpp:247-264), no kernel
 * projection -- the coarse-grid solve of a mesh-partitioned hierarchy */
int ldgmg_mg_vcycle(ldgmg_ctx* ctx, ldgmg_mg* mg, double* x, const double* b);
/* replaces Multigrid::apply(const BlockVec& b) -> x           multigrid.hpp:90-101 */
int ldgmg_mg_apply(ldgmg_ctx* ctx, ldgmg_mg* mg, const double* b, double* x);
/* Run `ncycles` V-cycles (graph-captured after the first call); x in place. */
int ldgmg_mg_cycles(ldgmg_ctx* ctx, ldgmg_mg* mg, double* x, const double* b, int ncycles);
/* Stationary V-cycle solve from HOST buffers (the end-to-end path):
 * x = 0; repeat cycle until ||b-Ax||/||b|| <= tol or maxit; residual history
 * (relative, one entry per iteration incl. iteration 0) to `history` (maxit+1
 * doubles, may be NULL).  Returns iterations in *iters. */
int ldgmg_mg_solve_host(ldgmg_ctx* ctx, ldgmg_mg* mg, const double* b_host, double* x_host,
                        double tol, int maxit, double* history, int* iters);
/* 1: kernel projection dots in the reference's sequential order (bitwise
 * parity mode); 0 (default): fixed-shape deterministic tree reduction. */
int ldgmg_mg_set_strict_order(ldgmg_mg* mg, int strict);
/* algorithmic DOF-updates and HBM bytes of one V-cycle */
/* build every smoother not set by the caller (otherwise done lazily by the
 * first cycle): the rest of the reference constructor's setup, multigrid.hpp:49-65 */
int ldgmg_mg_setup(ldgmg_ctx* ctx, ldgmg_mg* mg);
int ldgmg_mg_cycle_costs(const ldgmg_mg* mg, double* dof_updates, double* alg_bytes);
int ldgmg_mg_destroy(ldgmg_mg* mg);

/* ------------------------------------------------ Krylov (L5, krylov.hpp)
 * The reference's measurement protocol around the V-cycle.  SolveReport
 * (krylov.hpp:38-47); residuals go to the caller's buffer (capacity >= maxit+1). */
typedef struct ldgmg_solve_report {
    double* residuals;
    int capacity;
    int n_residuals;
    int iterations;
    int converged, breakdown;
    double rho, eta;
    int classification; /* 0 fast, 1 slow, 2 nonconvergent (krylov.hpp:25) */
    int low_confidence;
} ldgmg_solve_report;
enum { LDGMG_KRYLOV_CG = 0, LDGMG_KRYLOV_GMRES = 1 };
/* replaces pcg / gmres_left(A, b, preconditioner(V), tol, maxit)
 * (krylov.hpp:117-251): A = level-0 operator, V = Multigrid::apply; device b, x */
int ldgmg_krylov_solve(ldgmg_ctx* ctx, ldgmg_mg* mg, int kind, const double* b, double* x,
                       double tol, int maxit, ldgmg_solve_report* rep);
/* replaces estimate_eta(S, V, kind, {tol, maxit, seed}) (krylov.hpp:293-306) */
int ldgmg_estimate_eta(ldgmg_ctx* ctx, ldgmg_mg* mg, int kind, uint64_t seed, double tol,
                       int maxit, ldgmg_solve_report* rep);

/* --------------------------------------- built-in host setup (L0/L2)
 * The product's own mesh chain + LDG assembly (the reference's
 * build_uniform/coarsen/assemble_scalar/assemble_stokes, mesh.hpp,
 * ldg_scalar.hpp:83-125, ldg_stokes.hpp:102-280) so the framework runs
 * standalone.  Host C++, multi-threaded. */
int ldgmg_problem_create(const ldgmg_problem_spec* spec, int min_depth, int bottom_max_elements,
                         ldgmg_problem** out);
/* Distributed setup: as ldgmg_problem_create, but every level
 * with >= nranks * min_rows_per_rank elements (except the last) assembles
 * only rank `rank`'s element range [rank*N/P, (rank+1)*N/P) (partition_ranges,
 * smoothers.hpp:87-94) plus `halo_hops` face layers; the other rows are left
 * empty.  Each assembled row is bit-identical to the full assembly. */
int ldgmg_problem_create_partial(const ldgmg_problem_spec* spec, int min_depth, int bottom_max_elements,
                                 int nranks, int rank, int halo_hops, int min_rows_per_rank,
                                 ldgmg_problem** out);
/* 1 when the level was assembled partially (rank rows + halo) */
int ldgmg_problem_level_partial(const ldgmg_problem* P, int level);
/* General form of the two above.  flags: LDGMG_PROBLEM_DEVICE_ASSEMBLY = the
 * level operators are not built on the host; the product records each
 * block's accumulation (accumulate_AtDB products, penalty / coupling blocks,
 * ldg_core.hpp:547-586, ldg_stokes.hpp:149-191) and evaluates it on the GPU,
 * bit-identical to the host assembly (ldgmg_problem_device_operator,
 * ldgmg_mg_create_from_problem).  ldgmg_problem_level_matrix then returns the
 * pattern only (val must be NULL). */
/* LDGMG_PROBLEM_ANY_N = extension A1 (the reference
 * requires a power of two, mesh.hpp:143-149): n may be any count >= 2; the
 * elements are the in-range cells of the bounding power-of-two grid in its
 * Morton order, and coarsening halves n while it is even (48 -> ... -> 3). */
enum { LDGMG_PROBLEM_DEVICE_ASSEMBLY = 1, LDGMG_PROBLEM_ANY_N = 2 };
int ldgmg_problem_create_ex(const ldgmg_problem_spec* spec, int min_depth, int bottom_max_elements, int nranks,
                            int rank, int halo_hops, int min_rows_per_rank, int flags, ldgmg_problem** out);
/* the level operator as a device BSR (device assembly, or upload of the host one) */
int ldgmg_problem_device_operator(ldgmg_ctx* ctx, const ldgmg_problem* P, int level, ldgmg_bsr** out);
int ldgmg_problem_depth(const ldgmg_problem* P);
int ldgmg_problem_level_shape(const ldgmg_problem* P, int level, int* n_elements, int* bs,
                              int64_t* nnzb);
int ldgmg_problem_level_matrix(const ldgmg_problem* P, int level, int* ptr, int* col,
                               double* val);
int ldgmg_problem_level_transfer(const ldgmg_problem* P, int level, int* parent_of,
                                 int* orthant_of);
int ldgmg_problem_info(const ldgmg_problem* P, int* dim, int* n_comp, int* bs_scalar,
                       int* kernel_constants, int* kernel_pressure, int* n_velocity);
int ldgmg_problem_injection(const ldgmg_problem* P, double* K);
/* upload the whole hierarchy and build a GPU multigrid in one call */
int ldgmg_mg_create_from_problem(ldgmg_ctx* ctx, const ldgmg_problem* P,
                                 const ldgmg_mg_config* cfg, ldgmg_mg** out);
int ldgmg_problem_destroy(ldgmg_problem* P);

/* the 2^dim polynomial-injection matrices of build_injection
 * (multigrid.hpp:212-241) for a (dim, degree) tensor Legendre basis,
 * row-major ((p+1)^dim)^2 each; host, no device needed */
int ldgmg_injection_matrices(int dim, int degree, double* K);

/* seeded measurement right-hand side: random_rhs (krylov.hpp:279-287),
 * mt19937_64, u = (rng()>>11)*2^-53, v = 2u-1, host buffer */
int ldgmg_random_rhs(int nblocks, int bs, uint64_t seed, double* out);

#ifdef __cplusplus
}
#endif

#endif /* LDGMG_B200_H */
