/*
 * oracle/bminres_oracle.c -- TEST INFRASTRUCTURE, NOT PART OF THE PRODUCT.
 *
 * A plain, slow, single-thread CPU implementation of banded-Lanczos block
 * MINRES (Soodhalter, arXiv:1301.2102), written from PAPER.md in the paper's
 * per-iteration order and notation.  It exists only to check the CUDA path:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` leg may load it.  It shares no code, header, table or
 * helper with paper_1301_2102_b200/ (the CUDA path), and neither includes the
 * other.
 *
 * Citations: "P:L" = PAPER.md line L; "C<k>" = a reading of SURVEY.md §8(c)'s
 * C-table, restated in DESIGN.md "Readings of the paper".
 *
 *   Start block      eqn.init-QR  F0 = U_p S                       P:353-356, C6, C13
 *   Lanczos step     Alg. 1 with symmetric reuse of
 *                    h_{i,j} = h_{j,i} (Alg. 2) C1-C5
 *   Breakdown        h_{j+p,j} <= tau*||A u_j||                    P:562-570, C14-C16
 *   Replacement      random vector orthogonal to all previous       P:571-577, C17-C18
 *                    Lanczos vectors (pool orthogonalised as each
 *                    new vector is created)
 *   Retention        near-dependent vector kept 2p iterations       P:797-805, C15-C16
 *   Progressive QR   one Householder reflector per column, the      P:424-434, C20
 *                    <=2p previous ones applied first
 *   Transformed RHS  [T;0] -> reflector j -> z_j^T, new tail T      P:450-468, C6
 *   Directions       m_j = (u_j - sum r_ij m_i)/r_jj                eqn.search-dir-comp
 *   Update           X += m_j z_j^T                                 eqn.approx-update
 *   Residual         ||f_j^(i)|| = ||tail(:,i)||                    eqn.comp-resid
 *   Stop             max_i ||tail(:,i)||/||b_i|| < tol or j = maxit Alg. 2, C7, C22
 *   Preconditioning  (f3) IC(0) of an SPD M, split form L^-1 A L^-T  P:1026-1027, reading R8
 *                    (orc_ic0, orc_trsv_lower/upper, orc_solve_prec; pinned in
 *                    tests/test_precond_oracle.py, incl. the paper's Fig. 1 counts P:1034-1035)
 *
 * Parity pins (tests/test_oracle_pins.py): dense least squares over an
 * explicitly built block Krylov basis, p = 1 against SciPy MINRES, the paper's
 * Fig. 3 closed form, exact rational dependence steps, the block-grade stall,
 * the paper's C_{pxp} antidiagonal, the replacement zero patterns
 * of \hat H_8 / \hat R_8, the Lanczos relation, Householder
 * invariants.  The replacement vectors' VALUES follow reading C17 (the paper
 * uses Matlab's mt19937ar): "parity unpinned" for those values.
 */
#define _POSIX_C_SOURCE 199309L   /* clock_gettime (timing instrumentation) */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <float.h>
#include <time.h>

#define ORC_OK 0
#define ORC_MAXIT 1
#define ORC_EINVAL (-1)
#define ORC_ENOMEM (-4)
#define ORC_EPOOL (-5)
#define ORC_ESINGULAR_R (-6)

#define ORC_MAX_P 64

typedef struct {
    int64_t j;      /* iteration at which the candidate was rejected (0 = start block) */
    int32_t col;    /* 1-based: block column ((j-1) mod p)+1, or RHS column at j = 0 */
    int32_t kind;   /* 0 = exact (h <= 1e-12*omega), 1 = near (C15) */
    int32_t action; /* 1 = replaced, 2 = replaced + retained, 3 = pool exhausted,
                       4 = removed (shrink policy), 5 = removed + retained */
    int32_t pad;
    double ratio;   /* h / omega */
} orc_event;

typedef struct {
    int32_t p;
    int32_t pool_size;
    int32_t use_x0;
    int32_t policy;         /* 0 = replacement, 1 = block-size reduction "shrink" */
    double tol;
    double tau;             /* deflation tolerance (the paper's gamma) */
    int64_t maxit;
    uint64_t seed;
    double *history;        /* (history_cap) rows of p doubles; row j = iteration j */
    int64_t history_cap;
    orc_event *events;
    int64_t events_cap;
    int64_t dbg_cap;        /* iterations the dense debug dumps hold; 0 = off */
    double *dbg_U;          /* n x (dbg_cap+p), column-major, u_1 .. */
    double *dbg_H;          /* (dbg_cap+p) x dbg_cap, column-major, \bar H */
    double *dbg_R;          /* dbg_cap x dbg_cap, column-major, R */
    double *dbg_M;          /* n x dbg_cap, column-major, m_1 .. */
    double *dbg_Z;          /* dbg_cap x p, row-major, z_j^T rows */
    double *dbg_S;          /* p x p, row-major, S of eqn.init-QR */
} orc_config;

typedef struct {
    int32_t status;
    int32_t pad;
    int64_t iterations;
    int64_t n_events;
    double true_res[ORC_MAX_P];   /* ||b_i - A x_i|| / ||b_i|| at exit */
    double comp_res[ORC_MAX_P];   /* ||T(:,i)|| / ||b_i|| at exit */
    double start_s;               /* wall seconds: start block + pool (instrumentation only) */
    double loop_s;                /* wall seconds: the iteration loop (instrumentation only) */
} orc_result;

static double wall_s(void) {   /* timing instrumentation; no part of the method */
    struct timespec t;
    clock_gettime(CLOCK_MONOTONIC, &t);
    return (double)t.tv_sec + 1e-9 * (double)t.tv_nsec;
}

/* ---------------- plain vector helpers (n-length loops) ---------------- */

static double dot(int64_t n, const double *a, const double *b) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}

static void axpy(int64_t n, double alpha, const double *x, double *y) {
    for (int64_t i = 0; i < n; ++i) y[i] += alpha * x[i];
}

static double nrm2(int64_t n, const double *x) { return sqrt(dot(n, x, x)); }

static void scal(int64_t n, double alpha, double *x) {
    for (int64_t i = 0; i < n; ++i) x[i] *= alpha;
}

/* y = A x for one vector; each row summed over the CSR row in stored order with fma. */
static void csr_matvec(int64_t n, const int32_t *indptr, const int32_t *indices,
                       const double *data, const double *x, double *y) {
    for (int64_t i = 0; i < n; ++i) {
        double s = 0.0;
        for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k) s = fma(data[k], x[indices[k]], s);
        y[i] = s;
    }
}

/* Y = A X for a row-major n x p block (test helper for the SpMM parity tests). */
void orc_csr_block(int64_t n, const int32_t *indptr, const int32_t *indices, const double *data,
                   int32_t p, const double *X, double *Y) {
    for (int64_t i = 0; i < n; ++i) {
        for (int32_t c = 0; c < p; ++c) {
            double s = 0.0;
            for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k)
                s = fma(data[k], X[(int64_t)indices[k] * p + c], s);
            Y[i * p + c] = s;
        }
    }
}

/* ---------------- random vectors (reading C17; values unpinned) ---------------- */

uint64_t orc_splitmix64(uint64_t x);
static uint64_t splitmix64(uint64_t x) { return orc_splitmix64(x); }
uint64_t orc_splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* uniform[-1,1) entry of random vector (stream, event) at global row `row`. */
double orc_rand_entry(uint64_t seed, uint64_t stream, uint64_t event, uint64_t row) {
    uint64_t key = splitmix64(seed ^ (stream << 56) ^ (event << 32));
    uint64_t x = splitmix64(key ^ row);
    return 2.0 * ((double)(x >> 11) * 0x1.0p-53) - 1.0;
}

static void rand_vector(int64_t n, uint64_t seed, uint64_t stream, uint64_t event, double *v) {
    for (int64_t i = 0; i < n; ++i) v[i] = orc_rand_entry(seed, stream, event, (uint64_t)i);
}

/* ---------------- Householder (LAPACK dlarfg convention, C20) ---------------- */

/* Given x[0..len-1], find v (v[0] = 1), tau, beta with (I - tau v v^T) x = beta e_1. */
void orc_house_gen(int32_t len, const double *x, double *v, double *tau, double *beta) {
    double alpha = x[0];
    double xnorm = 0.0;
    for (int32_t q = 1; q < len; ++q) xnorm += x[q] * x[q];
    xnorm = sqrt(xnorm);
    v[0] = 1.0;
    if (xnorm == 0.0) {
        *tau = 0.0;
        *beta = alpha;
        for (int32_t q = 1; q < len; ++q) v[q] = 0.0;
        return;
    }
    double b = -copysign(hypot(alpha, xnorm), alpha);
    *tau = (b - alpha) / b;
    double s = 1.0 / (alpha - b);
    for (int32_t q = 1; q < len; ++q) v[q] = x[q] * s;
    *beta = b;
}

/* y <- (I - tau v v^T) y */
void orc_house_apply(int32_t len, const double *v, double tau, double *y) {
    double s = 0.0;
    for (int32_t q = 0; q < len; ++q) s += v[q] * y[q];
    s *= tau;
    for (int32_t q = 0; q < len; ++q) y[q] -= s * v[q];
}

/* ---------------- the solver ---------------- */

typedef struct {
    double *vec;
    int64_t expiry;   /* last iteration at which it is still projected out */
} retained_t;

static void record_event(const orc_config *cfg, int64_t *nev, int64_t j, int32_t col, int32_t kind,
                         int32_t action, double ratio) {
    if (cfg->events && *nev < cfg->events_cap) {
        orc_event *e = &cfg->events[*nev];
        e->j = j; e->col = col; e->kind = kind; e->action = action; e->pad = 0; e->ratio = ratio;
    }
    (*nev)++;
}

/* The operator the method is applied to: A itself, or (f3) the split-preconditioned
   L^{-1} A L^{-T} of an IC(0) factor L (see "f3" below). */
typedef struct {
    const int32_t *indptr, *indices;
    const double *data;          /* A in CSR */
    const int32_t *Lp, *Li;      /* NULL = no preconditioner; else L (lower, diagonal last per row) */
    const double *Lx;
    const int32_t *Up, *Ui;      /* L^T in CSR (column i of L as row i, ascending) */
    const double *Ux;
    double *t, *u;               /* n-length scratch */
} orc_op;

static void op_apply(int64_t n, const orc_op *op, const double *x, double *y);

static int solve_core(int64_t n, const orc_op *op, const double *B, double *X, const orc_config *cfg,
                      orc_result *res);

int orc_solve(int64_t n, const int32_t *indptr, const int32_t *indices, const double *data,
              const double *B, double *X, const orc_config *cfg, orc_result *res) {
    orc_op op;
    memset(&op, 0, sizeof(op));
    op.indptr = indptr; op.indices = indices; op.data = data;
    return solve_core(n, &op, B, X, cfg, res);
}

static int solve_core(int64_t n, const orc_op *op, const double *B, double *X, const orc_config *cfg,
                      orc_result *res) {
    const int p = cfg->p;
    memset(res, 0, sizeof(*res));
    if (p < 1 || p > ORC_MAX_P || n < p || !(cfg->tol >= 0.0) || cfg->maxit < 0) {
        res->status = ORC_EINVAL;
        return ORC_EINVAL;
    }
    const double tau = cfg->tau;
    const int64_t W2 = 2 * p + 1;      /* ring size: indices j-p .. j+p are live */
    const int64_t HR = p + 1;          /* subdiagonal cache ring (C_{pxp}) */
    const int64_t pool_cap = cfg->pool_size > 0 ? cfg->pool_size : 0;
    const int64_t dcap = cfg->dbg_cap;
    const int64_t ldH = dcap + p;

    double *Ubuf = calloc((size_t)(W2 * n), sizeof(double));
    double *Mbuf = calloc((size_t)(W2 * n), sizeof(double));
    double *Wblk = calloc((size_t)(p * n), sizeof(double));
    double *w = calloc((size_t)n, sizeof(double));
    double *mj = calloc((size_t)n, sizeof(double));
    double *F = calloc((size_t)(p * n), sizeof(double));   /* F0 columns */
    double *pool = calloc((size_t)((pool_cap > 0 ? pool_cap : 1) * n), sizeof(double));
    retained_t *ret = calloc((size_t)(pool_cap + W2 + 4), sizeof(retained_t));
    int64_t n_ret = 0, ret_cap = pool_cap + W2 + 4;
    double *Vref = calloc((size_t)(W2 * (p + 1)), sizeof(double));
    /* shrink policy: absent[i % W2] = 1 when u_i was removed (u_i = 0, not in the basis);
       indices keep their numbering */
    unsigned char *absent = calloc((size_t)W2, 1);
    const int shrink = cfg->policy == 1;
    double *tauref = calloc((size_t)W2, sizeof(double));
    double *hl = calloc((size_t)(HR * p), sizeof(double));   /* hl[i%HR][t-1] = h_{i+t,i} */
    double *hcol = calloc((size_t)(2 * p + 1), sizeof(double));
    double *work = calloc((size_t)(3 * p + 1), sizeof(double));
    double T[ORC_MAX_P * ORC_MAX_P];   /* tail of \bar Z: T[r*p+c] */
    double S[ORC_MAX_P * ORC_MAX_P];
    double bnorm[ORC_MAX_P];
    double ycol[ORC_MAX_P + 1];
    double z[ORC_MAX_P];
    if (!Ubuf || !Mbuf || !Wblk || !w || !mj || !F || !pool || !ret || !Vref || !tauref || !hl ||
        !hcol || !work || !absent) {
        res->status = ORC_ENOMEM;
        goto done;
    }
#define U(idx) (Ubuf + ((idx) % W2) * n)
#define MV(idx) (Mbuf + ((idx) % W2) * n)

    int64_t nev = 0;
    int status = ORC_MAXIT;
    int64_t j = 0;
    const double t_start = wall_s();

    /* ---- start: F0 = B - A X0 (X0 = 0 unless use_x0; Alg. 2, C6) ---- */
    for (int c = 0; c < p; ++c) {
        double s = 0.0;
        for (int64_t i = 0; i < n; ++i) s += B[i * p + c] * B[i * p + c];
        bnorm[c] = sqrt(s);
    }
    if (!cfg->use_x0) memset(X, 0, sizeof(double) * (size_t)(n * p));
    for (int c = 0; c < p; ++c) {
        double *f = F + (int64_t)c * n;
        for (int64_t i = 0; i < n; ++i) f[i] = X[i * p + c];
        op_apply(n, op, f, w);
        for (int64_t i = 0; i < n; ++i) f[i] = B[i * p + c] - w[i];
    }

    /* ---- thin QR F0 = U_p S, MGS with one re-orthogonalisation, step-0 deflation (C13) ---- */
    memset(S, 0, sizeof(S));
    int64_t nrep0 = 0;
    for (int i = 0; i < p; ++i) {
        double *f = F + (int64_t)i * n;
        double fn0 = nrm2(n, f);
        double *ui = U(i + 1);
        memcpy(ui, f, sizeof(double) * (size_t)n);
        for (int pass = 0; pass < 2; ++pass)
            for (int l = 0; l < i; ++l) {
                double s = dot(n, U(l + 1), ui);
                axpy(n, -s, U(l + 1), ui);
                S[l * p + i] += s;
            }
        double h = nrm2(n, ui);
        if (h <= tau * fn0 && shrink) {
            /* shrink: the dependent start column is removed, u_i = 0 */
            double ratio = fn0 > 0.0 ? h / fn0 : 0.0;
            record_event(cfg, &nev, 0, i + 1, h <= 1e-12 * fn0 ? 0 : 1, 4, ratio);
            S[i * p + i] = 0.0;
            memset(ui, 0, sizeof(double) * (size_t)n);
            absent[(i + 1) % W2] = 1;
        } else if (h <= tau * fn0) {
            double ratio = fn0 > 0.0 ? h / fn0 : 0.0;
            record_event(cfg, &nev, 0, i + 1, h <= 1e-12 * fn0 ? 0 : 1, 1, ratio);
            S[i * p + i] = 0.0;
            rand_vector(n, cfg->seed, 0, (uint64_t)nrep0++, ui);
            for (int pass = 0; pass < 2; ++pass)
                for (int l = 0; l < i; ++l) axpy(n, -dot(n, U(l + 1), ui), U(l + 1), ui);
            scal(n, 1.0 / nrm2(n, ui), ui);
        } else {
            S[i * p + i] = h;
            scal(n, 1.0 / h, ui);
        }
    }
    memcpy(T, S, sizeof(double) * (size_t)(p * p));
    if (cfg->dbg_S) memcpy(cfg->dbg_S, S, sizeof(double) * (size_t)(p * p));
    if (dcap > 0 && cfg->dbg_U)
        for (int i = 1; i <= p; ++i) memcpy(cfg->dbg_U + (int64_t)(i - 1) * n, U(i), sizeof(double) * (size_t)n);

    /* ---- replacement pool: drawn at the start, orthogonalised twice against u_1..u_p (C18) ---- */
    int64_t pool_next = 0;
    for (int64_t q = 0; q < pool_cap; ++q) {
        double *r = pool + q * n;
        rand_vector(n, cfg->seed, 1, (uint64_t)q, r);
        for (int pass = 0; pass < 2; ++pass)
            for (int l = 1; l <= p; ++l) axpy(n, -dot(n, U(l), r), U(l), r);
    }

    /* ---- residual history at j = 0 and the while-test of Alg. 2 (C7) ---- */
    {
        double mx = 0.0;
        for (int c = 0; c < p; ++c) {
            double s = 0.0;
            for (int r = 0; r < p; ++r) s += T[r * p + c] * T[r * p + c];
            double rel = bnorm[c] > 0.0 ? sqrt(s) / bnorm[c] : 0.0;
            if (cfg->history && cfg->history_cap > 0) cfg->history[c] = rel;
            if (rel > mx) mx = rel;
        }
        if (mx < cfg->tol) status = ORC_OK;
    }

    int pool_exhausted = 0;
    int64_t iters = 0;                 /* completed iterations */
    const double t_loop = wall_s();
    res->start_s = t_loop - t_start;
    for (j = 1; status == ORC_MAXIT && j <= cfg->maxit; ++j) {
        const int m = (int)((j - 1) % p);          /* 0-based column within the block (C2) */
        /* block operator application every p iterations (Alg. 2, C2) */
        if (m == 0)
            for (int c = 0; c < p; ++c) op_apply(n, op, U(j + c), Wblk + (int64_t)c * n);
        /* shrink: the basis is exhausted once every index of the window j .. j+p-1 is removed */
        if (shrink) {
            int live = 0;
            for (int64_t i = j; i <= j + p - 1; ++i) live += !absent[i % W2];
            if (!live) break;
        }
        if (shrink && absent[j % W2]) {
            /* u_j was removed: column j of \bar H is deleted -- A u_j = 0, so
               u_{j+p} = 0 is removed too, h_{.,j} = 0; no reflector (identity), R column
               j and m_j are zero, z_j is the tail's first row (zero: the removed row of Z) */
            for (int q = 0; q <= 2 * p; ++q) hcol[q] = 0.0;
            for (int t = 1; t <= p; ++t) hl[(j % HR) * p + (t - 1)] = 0.0;
            double *unew0 = U(j + p);
            memset(unew0, 0, sizeof(double) * (size_t)n);
            absent[(j + p) % W2] = 1;
            if (dcap > 0 && j <= dcap && cfg->dbg_U) memset(cfg->dbg_U + (j + p - 1) * n, 0, sizeof(double) * (size_t)n);
            double *vj0 = Vref + (j % W2) * (p + 1);
            for (int q = 0; q <= p; ++q) vj0[q] = q == 0 ? 1.0 : 0.0;
            tauref[j % W2] = 0.0;
            for (int c = 0; c < p; ++c) {
                z[c] = T[c];
                for (int r = 0; r < p - 1; ++r) T[r * p + c] = T[(r + 1) * p + c];
                T[(p - 1) * p + c] = 0.0;
            }
            memset(MV(j), 0, sizeof(double) * (size_t)n);
            for (int64_t i = 0; i < n; ++i)
                for (int c = 0; c < p; ++c) X[i * p + c] += 0.0 * z[c];
            if (dcap > 0 && j <= dcap && cfg->dbg_Z) memcpy(cfg->dbg_Z + (j - 1) * p, z, sizeof(double) * (size_t)p);
            goto residuals;
        }
        memcpy(w, Wblk + (int64_t)m * n, sizeof(double) * (size_t)n);
        const double omega = nrm2(n, w);           /* raw candidate norm ||A u_j|| (C14) */

        /* hcol[r - (j-p)] = h_{r,j}, rows j-p .. j+p */
        for (int q = 0; q <= 2 * p; ++q) hcol[q] = 0.0;
        /* known coefficients h_{i,j} = h_{j,i}, i = max(1,j-p) .. j-1 (Alg. 2; C1, C4) */
        for (int64_t i = (j - p > 1 ? j - p : 1); i <= j - 1; ++i) {
            double hij = hl[(i % HR) * p + (j - i - 1)];
            hcol[i - (j - p)] = hij;
            axpy(n, -hij, U(i), w);
        }
        /* new coefficients by MGS, i = j .. j+p-1 (Alg. 1; Alg. 2; C1, C4) */
        for (int64_t i = j; i <= j + p - 1; ++i) {
            double hij = dot(n, U(i), w);
            hcol[i - (j - p)] = hij;
            axpy(n, -hij, U(i), w);
        }
        /* retained near-dependent vectors (C15-C16) */
        for (int64_t q = 0; q < n_ret; ++q)
            if (ret[q].expiry >= j) axpy(n, -dot(n, ret[q].vec, w), ret[q].vec, w);
        double h = nrm2(n, w);
        double hjp;
        double *unew = U(j + p);
        absent[(j + p) % W2] = 0;
        if (h <= tau * omega) {
            /* breakdown: candidate dependent */
            int kind = h <= 1e-12 * omega ? 0 : 1;
            int action = 1;
            if (kind == 1) {       /* retain w/h for orthogonalisation until step j+2p (C16) */
                if (n_ret == ret_cap) {
                    /* drop an expired slot */
                    int64_t k = 0;
                    for (int64_t q = 0; q < n_ret; ++q)
                        if (ret[q].expiry >= j) ret[k++] = ret[q]; else free(ret[q].vec);
                    n_ret = k;
                }
                double *v = malloc(sizeof(double) * (size_t)n);
                if (!v) { status = ORC_ENOMEM; break; }
                for (int64_t i = 0; i < n; ++i) v[i] = w[i] / h;
                ret[n_ret].vec = v;
                ret[n_ret].expiry = j + 2 * p;
                n_ret++;
                action = 2;
            }
            if (shrink) {
                /* block-size reduction: u_{j+p} = 0 is not added to the basis */
                memset(unew, 0, sizeof(double) * (size_t)n);
                absent[(j + p) % W2] = 1;
                action = kind == 1 ? 5 : 4;
            } else if (pool_next < pool_cap) {
                /* replacement: pool vector, already orthogonal to u_1..u_{j+p-1}
                   (P:718-721); orthogonalised twice more against retained + window, normalised */
                double *r = pool + pool_next * n;
                pool_next++;
                memcpy(unew, r, sizeof(double) * (size_t)n);
                for (int pass = 0; pass < 2; ++pass) {
                    for (int64_t q = 0; q < n_ret; ++q)
                        if (ret[q].expiry >= j) axpy(n, -dot(n, ret[q].vec, unew), ret[q].vec, unew);
                    for (int64_t i = (j - p > 1 ? j - p : 1); i <= j + p - 1; ++i)
                        axpy(n, -dot(n, U(i), unew), U(i), unew);
                }
                scal(n, 1.0 / nrm2(n, unew), unew);
            } else {
                memset(unew, 0, sizeof(double) * (size_t)n);
                pool_exhausted = 1;
                action = 3;
            }
            record_event(cfg, &nev, j, m + 1, kind, action, omega > 0.0 ? h / omega : 0.0);
            hjp = 0.0;                              /* h_{j+p,j} := 0 */
        } else {
            for (int64_t i = 0; i < n; ++i) unew[i] = w[i] / h;   /* Alg. 1 */
            hjp = h;
        }
        hcol[2 * p] = hjp;
        /* cache h_{j+1..j+p, j}: the C_{pxp} queue */
        for (int t = 1; t <= p; ++t) hl[(j % HR) * p + (t - 1)] = hcol[p + t];
        /* pool vectors orthogonalised against each new Lanczos vector */
        for (int64_t q = pool_next; q < pool_cap; ++q) {
            double *r = pool + q * n;
            axpy(n, -dot(n, unew, r), unew, r);
        }
        if (dcap > 0 && j <= dcap) {
            if (cfg->dbg_U) memcpy(cfg->dbg_U + (j + p - 1) * n, unew, sizeof(double) * (size_t)n);
            if (cfg->dbg_H)
                for (int64_t r = (j - p > 1 ? j - p : 1); r <= j + p; ++r)
                    cfg->dbg_H[(r - 1) + (j - 1) * ldH] = hcol[r - (j - p)];
        }

        /* ---- progressive QR of \bar H_j (Alg. 2; C8) ---- */
        const int64_t base = j - 2 * p;   /* work[r - base] = entry in row r */
        double hn = 0.0;
        for (int q = 0; q <= 3 * p; ++q) work[q] = 0.0;
        for (int64_t r = (j - p > 1 ? j - p : 1); r <= j + p; ++r) {
            work[r - base] = hcol[r - (j - p)];
            hn += hcol[r - (j - p)] * hcol[r - (j - p)];
        }
        hn = sqrt(hn);
        for (int64_t i = (j - 2 * p > 1 ? j - 2 * p : 1); i <= j - 1; ++i)
            orc_house_apply(p + 1, Vref + (i % W2) * (p + 1), tauref[i % W2], work + (i - base));
        double beta, tj;
        double *vj = Vref + (j % W2) * (p + 1);
        orc_house_gen(p + 1, work + 2 * p, vj, &tj, &beta);
        tauref[j % W2] = tj;
        work[2 * p] = beta;
        for (int q = 1; q <= p; ++q) work[2 * p + q] = 0.0;
        if (dcap > 0 && j <= dcap && cfg->dbg_R)
            for (int64_t r = (j - 2 * p > 1 ? j - 2 * p : 1); r <= j; ++r)
                cfg->dbg_R[(r - 1) + (j - 1) * dcap] = work[r - base];
        if (fabs(beta) <= DBL_EPSILON * hn) { status = ORC_ESINGULAR_R; break; }

        /* ---- reflector j applied to [T; 0]: row 1 -> z_j^T, rows 2..p+1 -> new tail (C6) ---- */
        for (int c = 0; c < p; ++c) {
            for (int r = 0; r < p; ++r) ycol[r] = T[r * p + c];
            ycol[p] = 0.0;
            orc_house_apply(p + 1, vj, tj, ycol);
            z[c] = ycol[0];
            for (int r = 0; r < p; ++r) T[r * p + c] = ycol[r + 1];
        }

        /* ---- search direction (eqn.search-dir-comp; Alg. 2) ---- */
        memcpy(mj, U(j), sizeof(double) * (size_t)n);
        for (int64_t i = (j - 2 * p > 1 ? j - 2 * p : 1); i <= j - 1; ++i)
            axpy(n, -work[i - base], MV(i), mj);
        scal(n, 1.0 / beta, mj);
        memcpy(MV(j), mj, sizeof(double) * (size_t)n);

        /* ---- X_j = X_{j-1} + m_j z_j^T (eqn.approx-update) ---- */
        for (int64_t i = 0; i < n; ++i)
            for (int c = 0; c < p; ++c) X[i * p + c] += mj[i] * z[c];
        if (dcap > 0 && j <= dcap) {
            if (cfg->dbg_M) memcpy(cfg->dbg_M + (j - 1) * n, mj, sizeof(double) * (size_t)n);
            if (cfg->dbg_Z) memcpy(cfg->dbg_Z + (j - 1) * p, z, sizeof(double) * (size_t)p);
        }

        /* ---- computed residuals (eqn.comp-resid) and the stop test (C7) ---- */
    residuals:;
        double mx = 0.0;
        for (int c = 0; c < p; ++c) {
            double s = 0.0;
            for (int r = 0; r < p; ++r) s += T[r * p + c] * T[r * p + c];
            double rel = bnorm[c] > 0.0 ? sqrt(s) / bnorm[c] : 0.0;
            if (cfg->history && j < cfg->history_cap) cfg->history[j * p + c] = rel;
            if (rel > mx) mx = rel;
        }
        iters = j;
        if (mx < cfg->tol) { status = ORC_OK; break; }
        if (pool_exhausted) { status = ORC_EPOOL; break; }   /* C18 */
    }
    res->loop_s = wall_s() - t_loop;
    res->iterations = iters;
    res->status = status;
    res->n_events = nev;

    /* ---- exit: computed and true residuals ---- */
    for (int c = 0; c < p; ++c) {
        double s = 0.0;
        for (int r = 0; r < p; ++r) s += T[r * p + c] * T[r * p + c];
        res->comp_res[c] = bnorm[c] > 0.0 ? sqrt(s) / bnorm[c] : 0.0;
        for (int64_t i = 0; i < n; ++i) w[i] = X[i * p + c];
        op_apply(n, op, w, mj);
        double t = 0.0;
        for (int64_t i = 0; i < n; ++i) {
            double d = B[i * p + c] - mj[i];
            t += d * d;
        }
        res->true_res[c] = bnorm[c] > 0.0 ? sqrt(t) / bnorm[c] : 0.0;
    }

done:
    if (ret) for (int64_t q = 0; q < n_ret; ++q) free(ret[q].vec);
    free(Ubuf); free(Mbuf); free(Wblk); free(w); free(mj); free(F); free(pool); free(ret);
    free(Vref); free(tauref); free(hl); free(hcol); free(work); free(absent);
#undef U
#undef MV
    return res->status;
}

/* ====================================================================================
 * f3: split preconditioning with an incomplete Cholesky factor.
 *
 * "we precondition with the incomplete Cholesky factors of -L constructed
 * using Matlab's ichol() function with the default settings" -- the default is the
 * zero-fill factorisation IC(0): L lower triangular with the sparsity pattern of the
 * lower triangle of M, and (L L^T)_{ik} = m_{ik} for every (i, k) in that pattern.  The
 * paper does not state how the factor enters MINRES; reading R8: the split
 * (two-sided) form, which keeps the operator symmetric:
 *
 *     Ahat = L^{-1} A L^{-T},   Rhat_0 = L^{-1} (B - A X_0),   Ahat Yhat = Rhat_0, Yhat_0 = 0,
 *     X = X_0 + L^{-T} Yhat,
 *
 * i.e. the unpreconditioned method above (solve_core) run on the transformed system; its
 * residual norms are ||L^{-1}(b_i - A x_i)|| relative to ||L^{-1}(b_i - A x0_i)||.
 * ==================================================================================== */

/* IC(0) of the symmetric matrix M (both triangles stored, columns ascending per row).
 * Row-oriented ("up-looking") definition, row i in order:
 *   l_ik = (m_ik - sum_{j<k, j in pat(i) and pat(k)} l_ij l_kj) / l_kk     (k < i in pat(i), ascending)
 *   l_ii = sqrt(m_ii - sum_{k<i} l_ik^2)
 * (sums in ascending j, each term subtracted with fma).  Output: L in CSR (Lp: n+1, Li/Lx: the lower
 * entries of M in M's order, the diagonal last in each row).  Returns 0, ORC_EINVAL (missing diagonal),
 * or -7 with *bad_row = the row whose pivot is <= 0 (IC(0) breakdown). */
int orc_ic0(int64_t n, const int32_t *indptr, const int32_t *indices, const double *data,
            int32_t *Lp, int32_t *Li, double *Lx, int64_t *bad_row) {
    int64_t nz = 0;
    Lp[0] = 0;
    for (int64_t i = 0; i < n; ++i) {
        for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k)
            if (indices[k] <= i) { Li[nz] = indices[k]; Lx[nz] = data[k]; ++nz; }
        Lp[i + 1] = (int32_t)nz;
        if (nz == Lp[i] || Li[nz - 1] != i) { if (bad_row) *bad_row = i; return ORC_EINVAL; }
    }
    for (int64_t i = 0; i < n; ++i) {
        const int64_t e0 = Lp[i], ed = Lp[i + 1] - 1;   /* ed = the diagonal */
        for (int64_t e = e0; e < ed; ++e) {
            const int64_t k = Li[e];
            double s = Lx[e];                             /* m_ik */
            /* sum over j < k in pat(i) and pat(k): merge row i (entries before e) with row k */
            int64_t a = e0, b = Lp[k];
            const int64_t bend = Lp[k + 1] - 1;           /* row k's off-diagonal entries */
            while (a < e && b < bend) {
                if (Li[a] < Li[b]) ++a;
                else if (Li[a] > Li[b]) ++b;
                else { s = fma(-Lx[a], Lx[b], s); ++a; ++b; }
            }
            Lx[e] = s / Lx[Lp[k + 1] - 1];                /* / l_kk */
        }
        double d = Lx[ed];                                /* m_ii */
        for (int64_t e = e0; e < ed; ++e) d = fma(-Lx[e], Lx[e], d);
        if (!(d > 0.0)) { if (bad_row) *bad_row = i; return -7; }
        Lx[ed] = sqrt(d);
    }
    return 0;
}

/* y = L^{-1} b: forward substitution, row i ascending, y_i = (b_i - sum_{j<i} l_ij y_j) / l_ii. */
void orc_trsv_lower(int64_t n, const int32_t *Lp, const int32_t *Li, const double *Lx, const double *b,
                    double *y) {
    for (int64_t i = 0; i < n; ++i) {
        double s = b[i];
        for (int64_t e = Lp[i]; e < Lp[i + 1] - 1; ++e) s = fma(-Lx[e], y[Li[e]], s);
        y[i] = s / Lx[Lp[i + 1] - 1];
    }
}

/* z = L^{-T} v: backward substitution on U = L^T (row i of U = column i of L, the diagonal FIRST),
   row i descending, z_i = (v_i - sum_{j>i} l_ji z_j) / l_ii, sum in ascending j. */
void orc_trsv_upper(int64_t n, const int32_t *Up, const int32_t *Ui, const double *Ux, const double *v,
                    double *z) {
    for (int64_t i = n - 1; i >= 0; --i) {
        double s = v[i];
        for (int64_t e = Up[i] + 1; e < Up[i + 1]; ++e) s = fma(-Ux[e], z[Ui[e]], s);
        z[i] = s / Ux[Up[i]];
    }
}

/* U = L^T as CSR (plain counting transpose; rows of U ascending in column). */
static int transpose_lower(int64_t n, const int32_t *Lp, const int32_t *Li, const double *Lx,
                           int32_t **Up, int32_t **Ui, double **Ux) {
    const int64_t nz = Lp[n];
    *Up = calloc((size_t)(n + 1), sizeof(int32_t));
    *Ui = malloc(sizeof(int32_t) * (size_t)(nz > 0 ? nz : 1));
    *Ux = malloc(sizeof(double) * (size_t)(nz > 0 ? nz : 1));
    int32_t *fill = calloc((size_t)(n + 1), sizeof(int32_t));
    if (!*Up || !*Ui || !*Ux || !fill) { free(fill); return ORC_ENOMEM; }
    for (int64_t e = 0; e < nz; ++e) (*Up)[Li[e] + 1]++;
    for (int64_t i = 0; i < n; ++i) (*Up)[i + 1] += (*Up)[i];
    for (int64_t i = 0; i < n; ++i)          /* rows of L ascending -> each U row ascending in column */
        for (int64_t e = Lp[i]; e < Lp[i + 1]; ++e) {
            const int64_t c = Li[e];
            const int64_t d = (*Up)[c] + fill[c]++;
            (*Ui)[d] = (int32_t)i;
            (*Ux)[d] = Lx[e];
        }
    free(fill);
    return 0;
}

/* y = op x: A x, or L^{-1} (A (L^{-T} x)) -- the three steps in that order. */
static void op_apply(int64_t n, const orc_op *op, const double *x, double *y) {
    if (!op->Lp) {
        csr_matvec(n, op->indptr, op->indices, op->data, x, y);
        return;
    }
    orc_trsv_upper(n, op->Up, op->Ui, op->Ux, x, op->t);
    csr_matvec(n, op->indptr, op->indices, op->data, op->t, op->u);
    orc_trsv_lower(n, op->Lp, op->Li, op->Lx, op->u, y);
}

/* Y = op X for a row-major n x p block (test helper). */
void orc_prec_op_block(int64_t n, const int32_t *indptr, const int32_t *indices, const double *data,
                       const int32_t *Lp, const int32_t *Li, const double *Lx, int32_t p, const double *X,
                       double *Y) {
    orc_op op;
    memset(&op, 0, sizeof(op));
    op.indptr = indptr; op.indices = indices; op.data = data;
    op.Lp = Lp; op.Li = Li; op.Lx = Lx;
    double *x = malloc(sizeof(double) * (size_t)n), *y = malloc(sizeof(double) * (size_t)n);
    op.t = malloc(sizeof(double) * (size_t)n);
    op.u = malloc(sizeof(double) * (size_t)n);
    int32_t *Up = NULL, *Ui = NULL;
    double *Ux = NULL;
    if (x && y && op.t && op.u && transpose_lower(n, Lp, Li, Lx, &Up, &Ui, &Ux) == 0) {
        op.Up = Up; op.Ui = Ui; op.Ux = Ux;
        for (int32_t c = 0; c < p; ++c) {
            for (int64_t i = 0; i < n; ++i) x[i] = X[i * p + c];
            op_apply(n, &op, x, y);
            for (int64_t i = 0; i < n; ++i) Y[i * p + c] = y[i];
        }
    }
    free(x); free(y); free(op.t); free(op.u); free(Up); free(Ui); free(Ux);
}

/* The preconditioned solve (reading R8): Rhat_0 = L^{-1}(B - A X_0), solve_core on
   (L^{-1} A L^{-T}, Rhat_0) from Yhat_0 = 0, X = X_0 + L^{-T} Yhat.  res->comp_res / ->true_res
   are the core's (preconditioned: relative to ||Rhat_0(:,i)||); ptrue_res[i] (p entries, may be NULL)
   receives the unpreconditioned ||b_i - A x_i|| / ||b_i||. */
int orc_solve_prec(int64_t n, const int32_t *indptr, const int32_t *indices, const double *data,
                   const int32_t *Lp, const int32_t *Li, const double *Lx, const double *B, double *X,
                   const orc_config *cfg, orc_result *res, double *ptrue_res) {
    const int p = cfg->p;
    memset(res, 0, sizeof(*res));
    if (p < 1 || p > ORC_MAX_P || n < p) { res->status = ORC_EINVAL; return ORC_EINVAL; }
    orc_op op;
    memset(&op, 0, sizeof(op));
    op.indptr = indptr; op.indices = indices; op.data = data;
    op.Lp = Lp; op.Li = Li; op.Lx = Lx;
    int32_t *Up = NULL, *Ui = NULL;
    double *Ux = NULL;
    double *Bh = calloc((size_t)(n * p), sizeof(double));
    double *Yh = calloc((size_t)(n * p), sizeof(double));
    double *a = malloc(sizeof(double) * (size_t)n), *b = malloc(sizeof(double) * (size_t)n);
    op.t = malloc(sizeof(double) * (size_t)n);
    op.u = malloc(sizeof(double) * (size_t)n);
    int st = ORC_ENOMEM;
    if (!Bh || !Yh || !a || !b || !op.t || !op.u || transpose_lower(n, Lp, Li, Lx, &Up, &Ui, &Ux) != 0) {
        res->status = ORC_ENOMEM;
        goto out;
    }
    op.Up = Up; op.Ui = Ui; op.Ux = Ux;
    if (!cfg->use_x0) memset(X, 0, sizeof(double) * (size_t)(n * p));
    for (int c = 0; c < p; ++c) {        /* Rhat_0(:,c) = L^{-1} (b_c - A x0_c) */
        for (int64_t i = 0; i < n; ++i) a[i] = X[i * p + c];
        csr_matvec(n, indptr, indices, data, a, b);
        for (int64_t i = 0; i < n; ++i) a[i] = B[i * p + c] - b[i];
        orc_trsv_lower(n, Lp, Li, Lx, a, b);
        for (int64_t i = 0; i < n; ++i) Bh[i * p + c] = b[i];
    }
    orc_config c2 = *cfg;
    c2.use_x0 = 0;
    st = solve_core(n, &op, Bh, Yh, &c2, res);
    if (st == ORC_EINVAL || st == ORC_ENOMEM) goto out;
    for (int c = 0; c < p; ++c) {        /* X = X_0 + L^{-T} Yhat; unpreconditioned true residual */
        for (int64_t i = 0; i < n; ++i) a[i] = Yh[i * p + c];
        orc_trsv_upper(n, Up, Ui, Ux, a, b);
        for (int64_t i = 0; i < n; ++i) X[i * p + c] += b[i];
        for (int64_t i = 0; i < n; ++i) a[i] = X[i * p + c];
        csr_matvec(n, indptr, indices, data, a, b);
        double t = 0.0, bn = 0.0;
        for (int64_t i = 0; i < n; ++i) {
            const double d = B[i * p + c] - b[i];
            t += d * d;
            bn += B[i * p + c] * B[i * p + c];
        }
        if (ptrue_res) ptrue_res[c] = bn > 0.0 ? sqrt(t) / sqrt(bn) : 0.0;
    }
out:
    free(Up); free(Ui); free(Ux); free(Bh); free(Yh); free(a); free(b); free(op.t); free(op.u);
    return res->status;
}
