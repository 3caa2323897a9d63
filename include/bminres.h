/*
 * bminres.h -- C ABI of the B200-native banded-Lanczos block MINRES hot path.
 *
 * Method: K. M. Soodhalter, "A block MINRES algorithm based on the banded
 * Lanczos method" (arXiv:1301.2102).  "P:L" cites PAPER.md line L.
 *
 * Problem: A (n x n) sparse symmetric indefinite, B (n x p).
 * At iteration j every column x_j^(i) minimises ||b_i - A x|| over
 * x_0^(i) + R(U_j), U_j = the first j banded-Lanczos vectors (eqn.min-resid,
 * P:367-374).  Inputs of Alg. 2: A, B, X_0 (= 0 unless requested),
 * eps (= tol), M (= maxit); the dependence tolerance gamma (= deflation_tol,
 * P:562-570).
 *
 * Conventions for every entry point:
 *  - All floating point is fp64.  Block vectors ("panels") are ROW-MAJOR n x p:
 *    element (row r, column c) at ptr[r*p + c].
 *  - Pointers may be device memory (cudaMalloc / torch CUDA tensors) or host
 *    memory; the library detects which (cudaPointerGetAttributes) and, for host
 *    memory, stages the data through device buffers it owns, copying results
 *    back before returning.  The caller owns A, B, X; the library never frees
 *    them and keeps no pointer to them after a call returns (with
 *    opt.plan_reuse = 1 it compares the col_idx pointer of the next call with
 *    the previous one, never dereferencing it outside a call).
 *  - Calls are synchronous with respect to the host: they return after the work
 *    on the handle's stream is complete.  A handle is not re-entrant; distinct
 *    handles may be used from distinct threads.
 *  - Return codes: >= 0 success (BMINRES_OK / BMINRES_MAXIT), < 0 error; the
 *    message is available from bminres_last_error().  There is no CPU
 *    fallback: without a usable CUDA device bminres_create returns
 *    BMINRES_ECUDA.
 */
#ifndef BMINRES_H
#define BMINRES_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BMINRES_OK 0           /* all columns converged: max_i ||f_j^(i)||/||b_i|| < tol */
#define BMINRES_MAXIT 1        /* j reached maxit first (Alg. 2); X holds X_maxit */
#define BMINRES_EINVAL (-1)    /* bad argument: p out of range, n < p, malformed CSR, tol not finite */
#define BMINRES_ECUDA (-2)     /* CUDA runtime error (message in bminres_last_error) */
#define BMINRES_ENCCL (-3)     /* collective / transport error (world > 1) */
#define BMINRES_ENOMEM (-4)    /* device allocation failed */
#define BMINRES_EPOOL (-5)     /* breakdown with the replacement pool empty, not converged */
#define BMINRES_ESINGULAR_R (-6) /* |r_jj| <= eps_mach*||h_j||: R_j singular, X cannot be updated */
#define BMINRES_EPIVOT (-7)    /* bminres_set_preconditioner: IC(0) pivot <= 0 (row in bminres_last_error) */

#define BMINRES_MAX_P 32       /* block sizes 1..8, 16 and 32 are compiled */
#define BMINRES_MAX_POOL 8

typedef struct bminres_ctx *bminres_handle;

/* Sparse symmetric operator A in CSR, both triangles stored.
 * row_ptr: n_loc+1 int32 offsets into col_idx/values, row_ptr[0] = 0.
 * col_idx: int32 GLOBAL column indices, strictly increasing within a row.
 * values:  fp64.  nnz = row_ptr[n_loc] must be < 2^31.
 * Rows [row_begin, row_begin+n_loc) of the global n x n matrix; at world = 1,
 * row_begin = 0 and n_loc = n. */
typedef struct {
    int64_t n;
    int64_t row_begin;
    int64_t n_loc;
    int64_t nnz;
    const int32_t *row_ptr;
    const int32_t *col_idx;
    const double *values;
} bminres_csr;

typedef struct {
    int32_t device;          /* CUDA device ordinal */
    int32_t rank, world;     /* row partition (world > 1: see "Row-partitioned solves" below) */
    void *stream;            /* cudaStream_t to run on; NULL = a stream the library creates */
    uint64_t seed;           /* random replacement vectors (reading C17), default 0 */
    int32_t pool_size;       /* random vectors kept orthogonal to the basis, 0..8, default 1 */
    int32_t use_x0;          /* 0: X is output only, X_0 = 0 (Alg. 2); 1: X holds X_0 on entry */
    int32_t record_history;  /* 1: keep (iterations+1) x p computed relative residuals */
    int32_t use_graphs;      /* 1: replay each block step as a CUDA graph (default); 0: plain launches */
    int32_t timing;          /* 1: CUDA events around every kernel launch, per-phase totals in stats */
    int32_t split_spmm;      /* p in {8,16,32}: 0 auto (split when the n x p panel is >= 128 MB), 1 always,
                                2 never.  Split: the SpMM A V_k runs alone at full occupancy (K1a) and K1
                                streams its result; same arithmetic, bitwise */
    int32_t policy;          /* dependence policy: 0 = replace the dependent vector by a random one
                                (the paper's choice; default); 1 = block-size reduction
                                ("shrink"): the dependent vector is removed (u_{j+p} = 0),
                                its lane stays removed (A 0 = 0) and its Hessenberg columns
                                are deleted; the panels keep p columns, removed ones zero.  The solve
                                stops (BMINRES_MAXIT unless converged) once every lane is removed */
    int32_t coeff_mode;      /* 0 = the paper's symmetric reuse h_{i,j} = h_{j,i} (default);
                                other values: BMINRES_EINVAL (not built) */
    int32_t plan_reuse;      /* world > 1: 0 = rebuild the halo plan on every solve (default; the library keeps
                                nothing of the caller's CSR between calls); 1 = the caller promises that a
                                solve with the same col_idx pointer, nnz, row_begin, n_loc and n passes the
                                same column indices, and the plan of the previous solve is reused */
    int32_t reserved[3];
} bminres_options;

/* One dependence event: candidate h_{j+p,j} <= gamma * ||A u_j||. */
typedef struct {
    int64_t j;       /* iteration (0 = the start block, eqn.init-QR) */
    int32_t col;     /* 1-based block column ((j-1) mod p)+1, or RHS column at j = 0 */
    int32_t kind;    /* 0 exact (h <= 1e-12*omega), 1 near */
    int32_t action;  /* 1 replaced, 2 replaced + retained, 3 pool exhausted, 4 removed (policy 1),
                        5 removed + retained */
    int32_t pad;
    double ratio;    /* h / omega */
} bminres_event;

#define BMINRES_NPHASE 15  /* spmm (K1), orth (K2), smallqr (K3b), update (K4b), slowpath, start, resid, other,
                              reduce (k_reduce), spmm_fused (K1 with the M/X update of block k-2),
                              split mode (large panels): spmm_av (K1a, A V_k alone), epilogue (K1 streaming
                              A V_k), epilogue_fused (the same with the M/X update of block k-2),
                              update_main (split mode, p >= 16: the M/X update of block k-2 as its own
                              kernel before K1a(k)), prec (preconditioned solves: the two triangular
                              kernels of L^-1 A L^-T, in place of K1a) */

typedef struct {
    int32_t status;           /* return code of the last solve */
    int32_t p;
    int64_t n;
    int64_t iterations;       /* banded iterations j completed (one new basis vector each) */
    int64_t block_steps;      /* operator applications to a block of p vectors */
    int64_t n_events;
    int64_t slow_blocks;      /* block steps that took the column-by-column path */
    int64_t history_len;      /* rows available from bminres_get_history */
    int64_t gpu_launches;     /* kernels this library launched during the last solve */
    double comp_res[BMINRES_MAX_P];   /* final ||T(:,i)||/||b_i|| (eqn.comp-resid) */
    double true_res[BMINRES_MAX_P];   /* final ||b_i - A x_i||/||b_i|| */
    double solve_ms;          /* device time of the whole solve (CUDA events) */
    double loop_ms;           /* device time of the block-step loop only */
    double phase_ms[BMINRES_NPHASE];          /* timing = 1 only */
    int64_t phase_launches[BMINRES_NPHASE];   /* timing = 1 only */
    double bytes_per_block_step;  /* algorithmic bytes model: CSR A + 10 panels */
    double spmm_bytes_per_launch; /* algorithmic bytes of one SpMM launch: CSR A + U_k + U_{k-1} + W */
    /* preconditioned solves (bminres_set_preconditioner): comp_res / history are the transformed
     * system's ||L^-1 (b_i - A x_i)|| / ||L^-1 (b_i - A x0_i)||, prec_true_res the same quantity
     * recomputed from X, and true_res the UNpreconditioned ||b_i - A x_i|| / ||b_i|| */
    double prec_true_res[BMINRES_MAX_P];
    int32_t preconditioned;   /* 1: the last solve ran on L^-1 A L^-T */
    int32_t prec_levels;      /* levels of the forward triangular DAG (the solves' dependency depth) */
} bminres_stats_t;

/* Default options (device 0, world 1, seed 0, pool_size 1, history on, graphs on). */
void bminres_default_options(bminres_options *opt);

/* Create a handle bound to opt->device; allocates nothing panel-sized yet. */
int bminres_create(const bminres_options *opt, bminres_handle *out);

/* Solve A X = B for the p columns of B (Alg. 2, with the readings
 * of DESIGN.md).  B: n_loc x p row-major (read only).  X: n_loc x p row-major
 * (output; input X_0 when opt.use_x0).  p in {1..8, 16, 32}; tol >= 0 finite;
 * maxit >= 0; deflation_tol >= 0 (the paper's gamma; reading C14:
 * relative to ||A u_j||).  Workspace (5 panels, + 1 in split mode, + pool;
 * bminres_workspace_bytes) is allocated on the first call for a given
 * (n_loc, p) and reused.
 * Returns BMINRES_OK, BMINRES_MAXIT or an error code. */
int bminres_solve(bminres_handle h, const bminres_csr *A, const double *B, double *X, int32_t p,
                  double tol, int64_t maxit, double deflation_tol);

/* Statistics of the last solve. */
int bminres_stats(bminres_handle h, bminres_stats_t *out);

/* Copy min(cap, history_len) rows of p doubles (row j = iteration j, j = 0 is
 * the start block) into buf (host memory).  Returns the number of rows copied. */
int64_t bminres_get_history(bminres_handle h, double *buf, int64_t cap);

/* Copy min(cap, n_events) events into buf (host memory).  Returns the count copied. */
int64_t bminres_get_events(bminres_handle h, bminres_event *buf, int64_t cap);

/* Component entry points of the hot path (same kernels the solver runs),
 * exported so each step can be checked on its own. */

/* Y = A X (row a1's SpMM): X, Y n_loc x p row-major (Y rows local,
 * X indexed by global column; at world = 1 both n x n).  Each output row is
 * accumulated over the CSR row in stored order with fma. */
int bminres_spmm(bminres_handle h, const bminres_csr *A, const double *X, double *Y, int32_t p);

/* out[i*stride] = entry of random replacement vector (stream, event) at global
 * row row_begin + i, i < n_loc (reading C17: splitmix64 counter hash, uniform
 * [-1,1)); bitwise reproducible. */
int bminres_random_vector(bminres_handle h, uint64_t seed, uint64_t stream, uint64_t event,
                          int64_t row_begin, int64_t n_loc, double *out, int64_t stride);

/* Upper bound on the device workspace bminres_solve allocates for (n_loc, p, pool_size) on one
 * rank: 5 panels (V_{k-1}, V_k, V_{k+1}, M_{k-1}, M_k), the split-mode A V_k panel when the
 * n_loc x p panel is >= 128 MB (p in {8,16,32}), the pool, 2 column-path scratch panels
 * (allocated on the first breakdown only), partial-sum buffers, the history (<= 8 Mi doubles)
 * and the state.  A row partition adds its halo rows to the three V panels; host-pointer
 * calls add the staged copies of A, B and X. */
size_t bminres_workspace_bytes(int64_t n_loc, int32_t p, int32_t pool_size);

/* ---- Row-partitioned solves (world > 1) ----
 * Rank r passes the contiguous rows [row_begin, row_begin + n_loc) of A (GLOBAL column
 * indices), B and X; ranks are in row order and cover 0..n-1.  Per block step the only
 * exchanges are the halo of the SpMM (the V rows other ranks' CSR rows reference, sent after K2)
 * and one fp64 sum-allreduce after each of the two grid-wide reductions; the small banded QR
 * runs replicated.  A transport must be attached before the first solve: NCCL
 * (bminres_get_unique_id on one rank, the id broadcast by the caller, bminres_init_nccl on every
 * rank; graph-capturable) or host callbacks (bminres_set_comm_callbacks; data staged through
 * host memory, plain launches -- a testing transport).  The allreduce must return bitwise
 * identical sums on every rank (ranks then take identical decisions). */

/* Host callbacks of a transport; every pointer is HOST memory; return 0 on success.
 * allreduce: in-place sum over ranks of count doubles.
 * alltoallv: send holds scount[q] int64 for each rank q (in rank order) -> recv gets rcount[q]
 *            int64 from each rank q (in rank order).
 * exchange:  same layout, doubles. */
typedef struct {
    void *ctx;
    int (*allreduce)(void *ctx, double *buf, int64_t count);
    int (*alltoallv)(void *ctx, const int64_t *send, const int64_t *scount, int64_t *recv, const int64_t *rcount);
    int (*exchange)(void *ctx, const double *send, const int64_t *scount, double *recv, const int64_t *rcount);
} bminres_comm_callbacks;

/* NCCL unique id (128 bytes) for bminres_init_nccl; one rank creates it.  BMINRES_ENCCL if
 * libnccl.so.2 cannot be loaded (dlopen; override the path with BMINRES_NCCL_LIB). */
int bminres_get_unique_id(uint8_t out[128]);

/* Create the handle's NCCL communicator for (opt.rank, opt.world) on its device. */
int bminres_init_nccl(bminres_handle h, const uint8_t id[128]);

/* Attach host-callback transport for (opt.rank, opt.world); cb is copied. */
int bminres_set_comm_callbacks(bminres_handle h, const bminres_comm_callbacks *cb);

/* Halo plan of a row partition (host only; no device, no communication).  offsets[0..world]:
 * global row offsets (rank q owns [offsets[q], offsets[q+1])).  col_idx: this rank's nnz
 * GLOBAL column indices.  Outputs: local_col[nnz] = column index into the extended panel
 * [n_loc own rows | n_halo halo rows]; halo_rows[n_halo] = the global rows of the halo,
 * ascending (hence grouped by owner rank); halo_count[world] = halo rows owned by each rank.
 * Pass halo_rows = NULL to query *n_halo only.  BMINRES_EINVAL on a column outside [0, n). */
int bminres_halo_plan(int32_t world, int32_t rank, const int64_t *offsets, int64_t nnz, const int32_t *col_idx,
                      int32_t *local_col, int64_t *halo_rows, int64_t *n_halo, int64_t *halo_count);

/* Interior rows of a partition (host only): the longest run [*lo, *hi) of this rank's rows whose
 * remapped columns (local_col from bminres_halo_plan; < n_loc = own row) are all local, i.e. whose
 * SpMM rows need no halo row.  In split mode the solver runs these rows' SpMM while the halo of
 * the next basis block is exchanged (overlap), then the rows [0, lo) and [hi, n_loc).
 * row_ptr: n_loc+1 offsets into local_col.  lo = hi = 0 when no row is interior. */
int bminres_interior_rows(int64_t n_loc, const int32_t *row_ptr, const int32_t *local_col, int64_t *lo, int64_t *hi);

/* ---- Preconditioning ----
 * "we precondition with the incomplete Cholesky factors of -L constructed using
 * Matlab's ichol() function with the default settings" (zero fill).  Reading R8: the
 * split form.  With a factor set, bminres_solve runs the method on L^-1 A L^-T with
 * Rhat_0 = L^-1 (B - A X_0) from Yhat_0 = 0 and returns X = X_0 + L^-T Yhat; the stop test and
 * the history use the transformed residuals (relative to ||Rhat_0(:,i)||).  Single rank only. */

/* Compute and keep the IC(0) factor L of M (n x n symmetric positive definite, both triangles,
 * columns strictly increasing per row, every diagonal entry present; host or device pointers;
 * copied -- the caller keeps ownership).  L has the pattern of M's lower triangle and
 * (L L^T)_ik = m_ik on it (the up-looking row algorithm, rows in dependency order on the device).
 * M = NULL removes the factor.  Returns BMINRES_OK, BMINRES_EINVAL (malformed M, world > 1) or
 * BMINRES_EPIVOT (a pivot <= 0: IC(0) does not exist for this M; no factor is kept). */
int bminres_set_preconditioner(bminres_handle h, const bminres_csr *M);

/* The factor's values (host or device buffer) in the order of M's lower-triangle entries (row by
 * row, columns ascending, the diagonal last).  Copies min(cap, nnz_L); returns nnz_L (0: none). */
int64_t bminres_get_preconditioner(bminres_handle h, double *l_values, int64_t cap);

/* Component entry point of the preconditioned operator (device pointers, n x p row-major):
 * mode 0: Y = L^-1 X;  mode 1: Y = L^-T X;  mode 2: Y = L^-1 A L^-T X (A: the n x n operator). */
int bminres_precond_apply(bminres_handle h, const bminres_csr *A, const double *X, double *Y, int32_t p,
                          int32_t mode);

/* Message of the last error on this handle (or the last create error if h is NULL). */
const char *bminres_last_error(bminres_handle h);

/* Release the handle and its workspace. */
void bminres_destroy(bminres_handle h);

#ifdef __cplusplus
}
#endif
#endif /* BMINRES_H */
