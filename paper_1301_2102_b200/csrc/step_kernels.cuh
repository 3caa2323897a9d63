// step_kernels.cuh -- sm_100a kernels of one block step of banded-Lanczos block MINRES.
//
// The basis is kept as U_k = V_k Tr_k (V_k = the unnormalised W'_{k-1}, Tr_k = C_{k-1}^{-1});
// every p x p factor is folded into a per-CTA combined matrix, so rows only see V.
// main branch (critical path), block k:
//   K1  k1_spmm     W = (A V_k) Tr_k = A U_k; ||A u_j||; W -= V_{k-1} (Tr_{k-1} C_{k-1}^T);
//                   G = Tr_k^T (V_k^T W) = U_k^T W   (row a1; Alg. 2)
//   K2  k2_orth     pool r_q -= V_k (Tr_k coef_{k-1}); W' = W - V_k (Tr_k G_s);
//                   W'^T W'; r_q^T W'; last CTA: Cholesky W' = U_{k+1} C_k, breakdown test
//                   h_{j+p,j} <= tau ||A u_j||, Tr_{k+1} = C_k^{-1}, pool coefficients
//                   (rows a2/a3/a5; Alg. 1); W' stays as V_{k+1}
// side branch, block k (runs beside the main branch of block k+1):
//   K3b k3b_smallqr one warp: p Hessenberg columns, <= 2p Householder reflectors each,
//                   z_j, residuals, stop test, direction matrices (row a4; P:424-468,
//                   Alg. 2)
//   K4b k4b_update  M_k = V_k (Tr_k R_kk^{-1}) - M_{k-2}R_{k-2,k}R_kk^{-1} - M_{k-1}R_{k-1,k}R_kk^{-1};
//                   X += M_k Z_k
//                   (row a5; eqn.search-dir-comp, eqn.approx-update)
//
// Panels are row-major n x p fp64.  A warp splits a panel row over LANES lanes of VEC
// (=2 -> 16-byte) chunks, RPW rows per warp instruction.
#pragma once
#include <cfloat>

#include "common.cuh"

namespace bmr {

// ------------------------------------------------------------------ K1: SpMM + epilogue

struct K1Args {
    const int* rowptr;
    const int* col;
    const double* val;
    const double* X;      // V_k (gathered by global column); plain mode: the SpMM input
    const double* Vprev;  // V_{k-1}
    double* Y;            // W (written into the V slot of block k+1); plain mode: the output
    long long n;
    DevState* st;
    double* part;
    int par;              // k mod 2
    int sk;               // k mod 3
    int tpw;              // row groups (tiles of RPW rows) per warp, contiguous
    // fused M/X update of block k-2 (DMMA K1 only, graph mode): Y holds V_{k-2} on entry
    int fuse;             // 1: apply the update of block k-2 before the SpMM
    double* Mk2;          // M slot k mod 2: M_{k-4} in, M_{k-2} out
    const double* Mk1;    // M slot (k+1) mod 2: M_{k-3}
    double* Xs;           // solution panel
    // split mode (k1_dmma<P, true>): A V_k was computed by k1a_spmm into AV; K1 stages its rows
    const double* AV;
    int xdefer;           // fused update: X updates deferred in pairs
    // K1a only (row partitions, halo overlap): the rows processed are r0 + v (+ gap once v >= gap_at)
    // for v < nrows; nrows < 0: all n rows
    long long r0 = 0, nrows = -1, gap_at = -1, gap = 0;
    int dyn = 0;          // K1a: CTA chunks taken from st->k1a_ctr[dyn - 1] in order (0: static round robin)
    int ku = 0;           // K1a: row groups per warp per CTA chunk (0: K1aCfg<P>::KU)
};

template <int P>
constexpr int k1_min_blocks() { return P <= 8 ? 3 : 1; }

template <int P>
struct K1Smem {   // dynamic shared memory of the epilogue variant
    static constexpr size_t bytes =
        sizeof(double) * (2 * P * P + (NT / 32) * 3 * PC<P>::RPW * PC<P>::RS + P * P + P + prologue_scratch<P>());
};

// C = A^T B for P x P row-major (leading dimensions lda/ldb/ldc), all threads of the CTA.
template <int P>
__device__ __forceinline__ void cta_matmul_tn(const double* Am, int lda, const double* Bm, int ldb, double* Cm,
                                              int ldc, bool transB = false) {
    for (int t = threadIdx.x; t < P * P; t += blockDim.x) {
        const int r = t / P, c = t % P;
        double s = 0.0;
        for (int i = 0; i < P; ++i) s = fma(Am[i * lda + r], transB ? Bm[c * ldb + i] : Bm[i * ldb + c], s);
        Cm[r * ldc + c] = s;
    }
}
// C = A B
template <int P>
__device__ __forceinline__ void cta_matmul_nn(const double* Am, int lda, const double* Bm, int ldb, double* Cm,
                                              int ldc, bool transB = false) {
    for (int t = threadIdx.x; t < P * P; t += blockDim.x) {
        const int r = t / P, c = t % P;
        double s = 0.0;
        for (int i = 0; i < P; ++i) s = fma(Am[r * lda + i], transB ? Bm[c * ldb + i] : Bm[i * ldb + c], s);
        Cm[r * ldc + c] = s;
    }
}

// W = A X.  Each row's sum runs over its CSR entries in stored order with fma (bitwise equal
// to the oracle's product in plain mode); the entries of a row are fetched CH at a time (all
// column indices, then all gathers) so that a lane has CH independent loads in flight.
template <int P, bool EPI>
__global__ void __launch_bounds__(NT, k1_min_blocks<P>()) k1_spmm(K1Args a) {
    using C = PC<P>;
    constexpr int VEC = C::VEC, LANES = C::LANES, LP = C::LP, RPW = C::RPW, WARPS = NT / 32;
    constexpr int E = P * P + P;
    constexpr int CH = 4;
    DevState* st = a.st;
    if constexpr (EPI) {
        pdl_trigger();
        pdl_wait();
        if (!st->run_main) return;
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int sub = lane % LP, rsub = lane / LP;
    const bool act = sub < LANES;
    const int c0 = sub * VEC;
    constexpr int RS = C::RS;
    constexpr int SR = EPI ? RPW * RS : 2;
    extern __shared__ __align__(16) double dyn1[];
    double* sTk = dyn1;                  // Tr_k
    double* sD = sTk + P * P;            // Tr_{k-1} C_{k-1}^T
    double(*sRow)[3][SR] = reinterpret_cast<double(*)[3][SR]>(sD + P * P);   // A V_k, V_k, V_{k-1} rows
    double* sAcc = sD + P * P + WARPS * 3 * SR;
    double* sScr = sAcc + (EPI ? E : 1);
    bool has_prev = false;
    if constexpr (EPI) {
        has_prev = st->k_main > 1;
        if (!k1_prologue<P>(st, a.par, a.sk, sTk, sD, sScr)) return;
    }
    double g[EPI ? P : 1][VEC];
    double om[VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
        om[v] = 0.0;
#pragma unroll
        for (int b = 0; b < (EPI ? P : 1); ++b) g[b][v] = 0.0;
    }
    const long long stride = (long long)gridDim.x * WARPS * RPW;
    for (long long base = ((long long)blockIdx.x * WARPS + warp) * RPW; base < a.n; base += stride) {
        const long long i = base + rsub;
        const bool valid = act && i < a.n;
        double u[VEC], up[VEC], acc[VEC];
#pragma unroll
        for (int v = 0; v < VEC; ++v) u[v] = up[v] = acc[v] = 0.0;
        int k0 = 0, k1 = 0;
        if (valid) {
            k0 = __ldg(a.rowptr + i);
            k1 = __ldg(a.rowptr + i + 1);
            if constexpr (EPI) {
                ldv<VEC>(a.X + i * P + c0, u);
                if (has_prev) ldv<VEC>(a.Vprev + i * P + c0, up);
            }
        }
        // (f3, preconditioned solves: A V_k is L^-1 A L^-T V_k, computed into AV by prec_kernels.cuh)
        if (EPI && a.AV) {
            if (valid) ldv<VEC>(a.AV + i * P + c0, acc);
            k1 = k0;
        }
        for (int kb = k0; kb < k1; kb += CH) {
            int cc[CH];
            double av[CH];
            double xv[CH][VEC];
#pragma unroll
            for (int t = 0; t < CH; ++t) {
                const bool pr = kb + t < k1;
                cc[t] = pr ? __ldg(a.col + kb + t) : -1;
                av[t] = pr ? __ldg(a.val + kb + t) : 0.0;
            }
#pragma unroll
            for (int t = 0; t < CH; ++t) {
                if (cc[t] >= 0) {
                    ldv<VEC>(a.X + (long long)cc[t] * P + c0, xv[t]);
                } else {
#pragma unroll
                    for (int v = 0; v < VEC; ++v) xv[t][v] = 0.0;
                }
            }
#pragma unroll
            for (int t = 0; t < CH; ++t)
                if (cc[t] >= 0) {
#pragma unroll
                    for (int v = 0; v < VEC; ++v) acc[v] = fma(av[t], xv[t][v], acc[v]);
                }
        }
        if constexpr (EPI) {
            double* rA = sRow[warp][0] + rsub * RS;
            double* rU = sRow[warp][1] + rsub * RS;
            double* rP = sRow[warp][2] + rsub * RS;
            if (act) {
#pragma unroll
                for (int v = 0; v < VEC; ++v) {
                    rA[c0 + v] = acc[v];
                    rU[c0 + v] = u[v];
                    rP[c0 + v] = up[v];
                }
            }
            __syncwarp();
            if (valid) {
                // W = (A V_k) Tr_k = A U_k: the raw candidates, ||A u_j|| (C14)
                double w[VEC];
#pragma unroll
                for (int v = 0; v < VEC; ++v) w[v] = 0.0;
#pragma unroll
                for (int b = 0; b < P; ++b) {
                    const double x = rA[b];
#pragma unroll
                    for (int v = 0; v < VEC; ++v) w[v] = fma(x, sTk[b * P + c0 + v], w[v]);
                }
#pragma unroll
                for (int v = 0; v < VEC; ++v) om[v] = fma(w[v], w[v], om[v]);
                if (has_prev) {
                    // W -= U_{k-1} C_{k-1}^T = V_{k-1} D  (h_{i,j} = h_{j,i})
#pragma unroll
                    for (int b = 0; b < P; ++b) {
                        const double x = rP[b];
#pragma unroll
                        for (int v = 0; v < VEC; ++v) w[v] = fma(-x, sD[b * P + c0 + v], w[v]);
                    }
                }
                // (V_k^T W)(b,m) += V_k(i,b) W(i,m)
#pragma unroll
                for (int b = 0; b < P; ++b) {
                    const double x = rU[b];
#pragma unroll
                    for (int v = 0; v < VEC; ++v) g[b][v] = fma(x, w[v], g[b][v]);
                }
#pragma unroll
                for (int v = 0; v < VEC; ++v) acc[v] = w[v];
            }
            __syncwarp();
        }
        if (valid) stv<VEC>(a.Y + i * P + c0, acc);
    }
    if constexpr (EPI) {
#pragma unroll
        for (int o = LP; o < 32; o <<= 1) {
#pragma unroll
            for (int v = 0; v < VEC; ++v) {
                om[v] += __shfl_xor_sync(FULL, om[v], o);
#pragma unroll
                for (int b = 0; b < P; ++b) g[b][v] += __shfl_xor_sync(FULL, g[b][v], o);
            }
        }
        for (int t = 0; t < WARPS; ++t) {
            if (warp == t && rsub == 0 && act) {
#pragma unroll
                for (int v = 0; v < VEC; ++v) {
#pragma unroll
                    for (int b = 0; b < P; ++b) {
                        const int e = b * P + c0 + v;
                        sAcc[e] = (t ? sAcc[e] : 0.0) + g[b][v];
                    }
                    const int e = P * P + c0 + v;
                    sAcc[e] = (t ? sAcc[e] : 0.0) + om[v];
                }
            }
            __syncthreads();
        }
        cluster_partials(sAcc, E, st->part1);   // reduce1, then K2 forms G = Tr_k^T (V_k^T W)
    }
}

// ------------------------------------------------------------------ K2: W' = W - U_k G_s, Grams, C_k

struct K2Args {
    double* W;            // W in, W' out (the V slot of block k+1)
    const double* V;      // V_k
    double* pool;         // n x pool_cap row-major
    long long n;
    DevState* st;
    double* part;
    int par;              // k mod 2
    int sk;               // k mod 3
    int tpw;              // row groups per warp, contiguous
};

constexpr int NSTAGE = 4;   // cp.async pipeline depth of the streaming panel kernels

template <int P>
struct K2Smem {
    static constexpr int LD = P + 1;
    static constexpr int TILE = PC<P>::RPW * PC<P>::RS;  // one row group of one panel (padded rows)
    static constexpr int RQ = PC<P>::RPW * MAXQ;         // pool values of one row group
    static constexpr int pipe = (NT / 32) * NSTAGE * (2 * TILE + RQ);
    static constexpr int loop = 2 * P * P + P * MAXQ + pipe + P * P + MAXQ * P;
    static constexpr int tail = 3 * P * P + P * MAXQ + prologue_scratch<P>();
    static constexpr size_t bytes = sizeof(double) * (loop + tail);
};

template <int P>
__global__ void __launch_bounds__(NT, P <= 8 ? 2 : 1) k2_orth(K2Args a) {
    using C = PC<P>;
    constexpr int VEC = C::VEC, LANES = C::LANES, LP = C::LP, RPW = C::RPW, WARPS = NT / 32;
    DevState* st = a.st;
    if (!st->run_main) {
        k2_stopped(st);
        return;
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int sub = lane % LP, rsub = lane / LP;
    const bool act = sub < LANES;
    const int c0 = sub * VEC;
    pdl_trigger();
    pdl_wait();
    const int Q = st->q_live, qf = st->q_first, qc = st->pool_cap;
    const int E = P * P + Q * P;
    using SM = K2Smem<P>;
    constexpr int TILE = SM::TILE, RQ = SM::RQ;
    extern __shared__ __align__(16) double dyn2[];
    double* sE = dyn2;                 // Tr_k G_s
    double* sTk = sE + P * P;          // Tr_k
    double* sF = sTk + P * P;          // Tr_k coef_{k-1} (P x MAXQ)
    double* sPipe = sF + P * MAXQ;     // per warp: NSTAGE x {W tile, V tile, pool values}
    double* sAcc = sPipe + SM::pipe;
    double* sTail = sAcc + P * P + MAXQ * P;
    {
        // G = Tr_k^T (V_k^T W) from K1's partials; G_s: lower triangle mirrored (the paper
        // computes h_{i,j} for i >= j)
        double* sGs = sTail;
        double* sCo = sTail + P * P;
        double* sG = sCo + P * MAXQ;
        k2_prologue<P>(st, a.par, a.sk, sG, sTk, sG + P * P);
        const double* Co = st->coef[a.par ^ 1];
        for (int t = threadIdx.x; t < P * P; t += NT) {
            const int r = t / P, c = t % P;
            sGs[t] = r >= c ? sG[r * P + c] : sG[c * P + r];
        }
        for (int t = threadIdx.x; t < P * MAXQ; t += NT) sCo[t] = Co[t];
        __syncthreads();
        cta_matmul_nn<P>(sTk, P, sGs, P, sE, P);
        for (int t = threadIdx.x; t < P * MAXQ; t += NT) {
            const int r = t / MAXQ, q = t % MAXQ;
            double s = 0.0;
            for (int i = 0; i < P; ++i) s = fma(sTk[r * P + i], sCo[i * MAXQ + q], s);
            sF[t] = s;
        }
        __syncthreads();
    }
    double g[P][VEC], pq[MAXQ][VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
#pragma unroll
        for (int b = 0; b < P; ++b) g[b][v] = 0.0;
#pragma unroll
        for (int q = 0; q < MAXQ; ++q) pq[q][v] = 0.0;
    }
    // NSTAGE-deep cp.async pipeline over this warp's row groups (grid-strided)
    constexpr int RS = C::RS;
    double* wb = sPipe + warp * NSTAGE * (2 * TILE + RQ);
    const long long t0 = (long long)blockIdx.x * WARPS + warp, ts = (long long)gridDim.x * WARPS;
    const long long ntiles = (a.n + RPW - 1) / RPW;
    auto issue = [&](long long it, int slot) {
        const long long t = t0 + it * ts;
        const long long i = t * RPW + rsub;
        const bool ok = act && t < ntiles && i < a.n;
        const long long ic = ok ? i : 0;
        double* sl = wb + slot * (2 * TILE + RQ);
        if (act) {   // idle lanes (p/VEC not a power of two) must not touch the next row's slots
            cp_async_vec<VEC>(sl + rsub * RS + c0, a.W + ic * P + c0, ok);
            cp_async_vec<VEC>(sl + TILE + rsub * RS + c0, a.V + ic * P + c0, ok);
            if (sub == 0)
                for (int q = 0; q < Q; ++q) cp_async8(sl + 2 * TILE + rsub * MAXQ + q, a.pool + ic * qc + qf + q, ok);
        }
        cp_commit();
    };
#pragma unroll
    for (int s = 0; s < NSTAGE - 1; ++s) issue(s, s);
    for (long long it = 0; t0 + it * ts < ntiles; ++it) {
        issue(it + NSTAGE - 1, (int)((it + NSTAGE - 1) % NSTAGE));
        cp_wait<NSTAGE - 1>();
        __syncwarp();
        double* sl = wb + (int)(it % NSTAGE) * (2 * TILE + RQ);
        double* tw = sl + rsub * RS;
        const double* tv = sl + TILE + rsub * RS;
        const double* tr = sl + 2 * TILE + rsub * MAXQ;
        const long long i = (t0 + it * ts) * RPW + rsub;
        const bool valid = act && i < a.n;
        double w[VEC], r[MAXQ];
#pragma unroll
        for (int v = 0; v < VEC; ++v) w[v] = tw[c0 + v];
#pragma unroll
        for (int q = 0; q < MAXQ; ++q) r[q] = (q < Q) ? tr[q] : 0.0;
        if (valid) {
            // pool r_q -= U_k coef_{k-1}(:,q) = V_k F(:,q)   (orthogonal to the newest block)
            if (Q > 0) {
#pragma unroll
                for (int b = 0; b < P; ++b) {
                    const double x = tv[b];
#pragma unroll
                    for (int q = 0; q < MAXQ; ++q)
                        if (q < Q) r[q] = fma(-x, sF[b * MAXQ + q], r[q]);
                }
                if (sub == 0) {
#pragma unroll
                    for (int q = 0; q < MAXQ; ++q)
                        if (q < Q) a.pool[i * qc + qf + q] = r[q];
                }
            }
            // W' = W - U_k G_s = W - V_k (Tr_k G_s)
#pragma unroll
            for (int b = 0; b < P; ++b) {
                const double x = tv[b];
#pragma unroll
                for (int v = 0; v < VEC; ++v) w[v] = fma(-x, sE[b * P + c0 + v], w[v]);
            }
            stv<VEC>(a.W + i * P + c0, w);
        }
        __syncwarp();
        if (act) {
#pragma unroll
            for (int v = 0; v < VEC; ++v) tw[c0 + v] = valid ? w[v] : 0.0;
        }
        __syncwarp();
        if (valid) {
#pragma unroll
            for (int b = 0; b < P; ++b) {
                const double x = tw[b];
#pragma unroll
                for (int v = 0; v < VEC; ++v) g[b][v] = fma(x, w[v], g[b][v]);
            }
#pragma unroll
            for (int q = 0; q < MAXQ; ++q) {
                if (q < Q) {
#pragma unroll
                    for (int v = 0; v < VEC; ++v) pq[q][v] = fma(r[q], w[v], pq[q][v]);
                }
            }
        }
        __syncwarp();
    }
    cp_wait<0>();
#pragma unroll
    for (int o = LP; o < 32; o <<= 1) {
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
#pragma unroll
            for (int b = 0; b < P; ++b) g[b][v] += __shfl_xor_sync(FULL, g[b][v], o);
#pragma unroll
            for (int q = 0; q < MAXQ; ++q)
                if (q < Q) pq[q][v] += __shfl_xor_sync(FULL, pq[q][v], o);
        }
    }
    for (int t = 0; t < WARPS; ++t) {
        if (warp == t && rsub == 0 && act) {
#pragma unroll
            for (int v = 0; v < VEC; ++v) {
#pragma unroll
                for (int b = 0; b < P; ++b) {
                    const int e = b * P + c0 + v;
                    sAcc[e] = (t ? sAcc[e] : 0.0) + g[b][v];
                }
#pragma unroll
                for (int q = 0; q < MAXQ; ++q) {
                    if (q < Q) {
                        const int e = P * P + q * P + c0 + v;
                        sAcc[e] = (t ? sAcc[e] : 0.0) + pq[q][v];
                    }
                }
            }
        }
        __syncthreads();
    }
    cluster_partials(sAcc, E, st->part2[a.par]);   // reduce2, then K1(k+1) and K3b(k) factor W'
}

// ------------------------------------------------------------------ K3b: small banded QR (side)
//
// 128 threads stage the state into shared memory with independent loads, warp 0 runs the
// serial chain from shared memory only, and all threads store the results.

constexpr int K3T = 128;

template <int P>
struct K3Smem {
    static constexpr int LD = P + 1, W2 = 2 * P + 1;
    static constexpr int nA = P * LD;
    static constexpr int nH = 4 * P * LD;
    // accumulated Householder (f2): one 2p x 2p block matrix (ld 2p+1), this block's p reflectors
    // (v: p+1, tau), a 2p x p product scratch
    static constexpr int LDQ = 2 * P + 1;
    static constexpr int nV = 2 * P * LDQ + P * (P + 2) + 2 * P * P;
    static constexpr int rest = nH + nV + 4 * P + P * P;
    static constexpr int scr = 8 * P * P + 2 * MAXQ * P + P + 8;   // prologue scratch (reuses sH..)
    static constexpr int doubles = 6 * nA + (rest > scr ? rest : scr);
    static constexpr size_t bytes = sizeof(double) * doubles;
};

template <int P>
__global__ void __launch_bounds__(K3T) k3b_smallqr(DevState* st) {
    using S = K3Smem<P>;
    constexpr int LD = S::LD;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    unsigned long long* tr = trace_begin(st, TR_K3B);
    __shared__ long long s_k, s_jd, s_maxit, s_hcap;
    __shared__ double s_tol;
    __shared__ int s_valid, s_stop_after, s_mlast, s_stop, s_given;
    __shared__ volatile int s_ready, s_done;   // phase B -> Q_k accumulation: reflectors published
    __shared__ unsigned s_am_k, s_am_k1;   // shrink policy: removed lanes of blocks k and k+1
    if (tid == 0) {
        const long long k = st->k_side;
        s_am_k = absent_mask(st, k, P);
        s_am_k1 = absent_mask(st, k + 1, P);
        s_valid = (k < st->stop_side_at) && (k < st->bd_at);
        s_given = st->given_blk == k;
        s_k = k;
        s_jd = st->j_done;
        s_maxit = st->maxit;
        s_hcap = st->hist ? st->hist_cap : 0;
        s_tol = st->tol;
        s_stop_after = st->stop_after;
        if (!s_valid) st->side_go = 0;
        s_ready = 0;
        s_done = 0;
    }
    __syncthreads();
    if (!s_valid) return;
    extern __shared__ __align__(16) double dyn3[];
    double* sC = dyn3;            // C_k
    double* sT = sC + S::nA;      // tail of \bar Z
    double* sZ = sT + S::nA;      // Z_k
    double* sI = sZ + S::nA;      // R_kk^{-1}
    double* sG = sI + S::nA;      // G (K1)
    double* sCp = sG + S::nA;     // C_{k-1}
    double* sH = sCp + S::nA;     // the block's p Hessenberg columns, global-row frame (4p rows)
    double* sQ = sH + S::nH;                   // an accumulated block reflector Q_b (2p x 2p, ld LDQ)
    double* sVb = sQ + 2 * P * S::LDQ;         // this block's reflectors: v (p+1) + tau each
    double* sTmp = sVb + P * (P + 2);          // 2p x p product scratch
    double* sHn = sQ + S::nV;     // ||h_j||
    double* sBeta = sHn + P;      // 1 / ||b_i||
    double* sRes = sBeta + P;     // residuals of the last completed iteration
    double* sHist = sRes + P;     // residual rows of this block (P x P)
    double* sRd = sHist + P * P;  // 1 / r_jj of this block's columns
    const long long k = s_k, j0 = s_jd + 1, maxit = s_maxit;
    const int par = (int)(k & 1);
    {
        // C_k: factor W'^T W' from K2(k)'s partials (as K1(k+1) does), or the host's C_k
        double* scr = sH;   // scratch (the Hessenberg frame is filled later)
        double* sCc = scr + prologue_scratch<P>();
        bool bad = false;
        if (s_given) {
            load_pp<P>(sCc, st->Ck[par]);
        } else if (st->red2_fac && st->fac_blk == k) {
            // reduce2 (k_red2f / k_fac2) already factored these totals with the same code
            // (factor_block): its C_k, bitwise what this CTA would compute (p = 16: 6.7 -> ~1 us)
            bad = st->fac_bad != 0;
            if (!bad) load_pp<P>(sCc, st->Ck[par]);
        } else {
            const int Q = st->q_live;
            double* sRed = scr;
            double* sOm = scr + P * P + MAXQ * P;
            for (int t = tid; t < P * P + Q * P; t += K3T) sRed[t] = st->red2[par][t];
            for (int t = tid; t < P; t += K3T) sOm[t] = st->om2[par][t];
            __syncthreads();
            bad = factor_block<P>(sRed, sOm, sRed + P * P, Q, st->tau, sCc, sOm + P, sOm + P + P * P,
                                  absent_mask(st, k + 1, P));
        }
        if (bad) {   // breakdown of block k: the host runs the column path, then re-runs this block
            if (tid == 0) {
                st->side_go = 0;
                publish_breakdown(st, k, true);   // (to the host; the main branch finds it itself)
            }
            return;
        }
        for (int t = tid; t < P * P; t += K3T) sC[(t / P) * LD + t % P] = sCc[t];
        // the scratch (sCc included) overlaps the reflector ring and the frame loaded next
        __syncthreads();
    }
    trace_pt(tr, 2);
    for (int t = tid; t < P * P; t += K3T) {
        const int r = t / P, c = t % P, g = r * MAXP + c, s = r * LD + c;
        sT[s] = st->T[g];
        sG[s] = st->G[par][g];
        sCp[s] = st->CprevS[g];
        sZ[s] = 0.0;
    }
    for (int t = tid; t < P; t += K3T) {
        sBeta[t] = st->beta[t] > 0.0 ? 1.0 / st->beta[t] : 0.0;   // 1 / ||b_i|| (0: converged at j = 0)
        sRes[t] = st->res[t];
    }
    __syncthreads();

    // ---- the p new columns of \bar H in the frame of global rows (k-3)p+1 .. (k+1)p
    //      (symmetric reuse P:923-945)
    if (warp == 0 && lane < P) {
        const int m = lane;
        double hn = 0.0;
        for (int r = 0; r < P; ++r) sH[r * LD + m] = 0.0;
        for (int mp = 0; mp < P; ++mp) {
            const double cv = (k > 1 && mp >= m) ? sCp[m * LD + mp] : 0.0;
            sH[(P + mp) * LD + m] = cv;
            const double gv = mp >= m ? sG[mp * LD + m] : sG[m * LD + mp];
            sH[(2 * P + mp) * LD + m] = gv;
            const double ck = mp <= m ? sC[mp * LD + m] : 0.0;
            sH[(3 * P + mp) * LD + m] = ck;
            hn = fma(cv, cv, fma(gv, gv, fma(ck, ck, hn)));
        }
        sHn[m] = sqrt(hn);
    }
    // ---- phase A (accumulated Householder): the reflectors
    //      of the previous two blocks, i = (k-3)p+1 .. (k-1)p in increasing order, applied to the p new
    //      columns as two dense products -- Q_{k-2} (block k-2's p reflectors accumulated, acting on
    //      frame rows 0 .. 2p-1) then Q_{k-1} (rows p .. 3p-1) -- by all threads, instead of 2p
    //      reflector applications in a serial chain per column
    for (int b = 2; b >= 1; --b) {
        if (k - b < 1) continue;   // (blocks before the first do not exist)
        const double* Qg = st->Qacc[(k - b) & 1];
        for (int t = tid; t < 4 * P * P; t += K3T) sQ[(t / (2 * P)) * S::LDQ + t % (2 * P)] = Qg[(t / (2 * P)) * (2 * MAXP) + t % (2 * P)];
        __syncthreads();
        const int r0 = (2 - b) * P;   // frame rows r0 .. r0 + 2p - 1
        for (int e = tid; e < 2 * P * P; e += K3T) {
            const int i = e / P, c = e % P;
            double acc = 0.0;
#pragma unroll 8
            for (int t = 0; t < 2 * P; ++t) acc = fma(sQ[i * S::LDQ + t], sH[(r0 + t) * LD + c], acc);
            sTmp[e] = acc;
        }
        __syncthreads();
        for (int e = tid; e < 2 * P * P; e += K3T) sH[(r0 + e / P) * LD + e % P] = sTmp[e];
        __syncthreads();
    }
    trace_pt(tr, 4);

    if (warp == 0) {
        const double tol = s_tol;
        // ---- phase B: generate reflector j, apply it to the later columns and to [T; 0]
        //      (row 1 -> z_j^T), residuals, stop test (Alg. 2)
        // 1 converged, 2 maxit, 3 singular R, 4 pool exhausted, 5 basis exhausted (shrink)
        int m_last = -1, stop = 0;
#ifdef K3B_PROF
        long long pc[6] = {0, 0, 0, 0, 0, 0};
        long long pt0 = clock64();
#define K3P(i) { const long long t_ = clock64(); pc[i] += t_ - pt0; pt0 = t_; }
#else
#define K3P(i)
#endif
        if constexpr (P <= 16) {
            const unsigned am_k = s_am_k, am_k1 = s_am_k1;
            // The chain runs in registers: lane c (< p) holds column c of the frame rows 2p .. 4p-1
            // (hc; reflector m acts on rows 2p+m .. 3p+m) and, for p <= 16, column c of the tail T (tc);
            // each reflector is broadcast from its pivot lane by shuffles.  (Through shared memory every
            // column update waited on the previous store: 1.8k cycles per reflector at p = 16.)
            constexpr bool TREG = P <= 16;
            const int c = lane;
            const bool cl = lane < P;
            double hc[2 * P];
    #pragma unroll
            for (int r = 0; r < 2 * P; ++r) hc[r] = cl ? sH[(2 * P + r) * LD + c] : 0.0;
            double tc[TREG ? P : 1];
            if constexpr (TREG) {
    #pragma unroll
                for (int q = 0; q < P; ++q) tc[q] = cl ? sT[q * LD + c] : 0.0;
            }
            const double bet_c = cl ? sBeta[c] : 0.0;
            // The window of reflector m (frame rows 2p+m .. 3p+m) is always hc[0 .. p]: after each
            // reflector row m is final -- stored -- and the column shifts up by one row.  So the
            // reflector loop indexes the registers with compile-time offsets only and stays a loop
            // (fully unrolled it was 19k instructions, fetched cold on every launch: config 3's K3b
            // took 86 us instead of 37)
            int sh = 0;   // rows stored (and shifted out)
    #pragma unroll 1
            for (int m = 0; m < P; ++m) {
                const long long j = j0 + m;
                if (j > maxit) {
                    stop = 2;
                    break;
                }
                // shrink: every index of the window j .. j+p-1 removed -> the basis is exhausted
                // (lanes >= m of this block, lanes < m of the next)
                if (am_k | am_k1) {
                    const unsigned all = P >= 32 ? 0xffffffffu : ((1u << P) - 1u);
                    const unsigned lo = m >= 32 ? 0xffffffffu : ((1u << m) - 1u);
                    if ((((am_k & ~lo) | (am_k1 & lo)) & all) == all) {
                        stop = 5;
                        break;
                    }
                }
                // shrink: u_j removed -> column j of \bar H is deleted: identity reflector,
                // R column zero (placeholder 1 on the diagonal for R_kk^{-1}), z_j = the tail's first
                // (zero) row, m_j = 0
                const bool gone = (am_k >> m) & 1u;
                // pivot column m (lane m): alpha = row 2p+m, x = rows 2p+m+1 .. 3p+m
                double x2a = 0.0, x2b = 0.0;
    #pragma unroll
                for (int q = 1; q <= P; ++q) {
                    if (q & 1)
                        x2a = fma(hc[q], hc[q], x2a);
                    else
                        x2b = fma(hc[q], hc[q], x2b);
                }
                const double alpha = __shfl_sync(FULL, hc[0], m);
                const double x2 = __shfl_sync(FULL, x2a + x2b, m);
                K3P(0)
                // dlarfg (C20): beta = -sign(alpha) ||(alpha, x)||, tau = (beta - alpha)/beta,
                // v = x/(alpha - beta); one reciprocal 1/(beta (alpha - beta)) serves both quotients
                double tj, beta, scl, rbeta;   // (rbeta = 1 / beta)
                if (gone) {
                    tj = 0.0;
                    beta = 1.0;
                    scl = 0.0;
                    rbeta = 1.0;
                } else if (x2 == 0.0) {   // (||x|| = 0)
                    tj = 0.0;
                    beta = alpha;
                    scl = 0.0;
                    rbeta = 1.0 / beta;
                } else {
                    beta = -copysign(sqrt(fma(alpha, alpha, x2)), alpha);
                    const double s = alpha - beta;
                    const double inv = 1.0 / (beta * s);
                    tj = -s * s * inv;
                    scl = beta * inv;
                    rbeta = s * inv;
                }
                if (!gone && fabs(beta) <= DBL_EPSILON * sHn[m]) {
                    stop = 3;
                    break;
                }
                K3P(1)
                double vq[P + 1];   // v = (1, x scl)
                vq[0] = 1.0;
    #pragma unroll
                for (int q = 1; q <= P; ++q) vq[q] = __shfl_sync(FULL, hc[q], m) * scl;
                if (lane == 0) {
                    sRd[m] = rbeta;   // 1 / r_jj for R_kk^{-1}
                    double* vj = sVb + m * (P + 2);
    #pragma unroll
                    for (int q = 0; q <= P; ++q) vj[q] = vq[q];
                    vj[P + 1] = tj;
                    __threadfence_block();
                    s_ready = m + 1;   // (warps 1-3 accumulate Q_k meanwhile)
                }
                K3P(2)
                double rel = 0.0, rel2 = 0.0;
                if (cl) {
                    if (c > m) {   // later columns of this block
                        double sp[4] = {0.0, 0.0, 0.0, 0.0};
    #pragma unroll
                        for (int q = 0; q <= P; ++q) sp[q & 3] = fma(vq[q], hc[q], sp[q & 3]);
                        const double s = ((sp[0] + sp[1]) + (sp[2] + sp[3])) * tj;
    #pragma unroll
                        for (int q = 0; q <= P; ++q) hc[q] = fma(-s, vq[q], hc[q]);
                    } else if (c == m) {   // the pivot column becomes (beta, 0, ..., 0)
                        hc[0] = beta;
    #pragma unroll
                        for (int q = 1; q <= P; ++q) hc[q] = 0.0;
                    }
                    // [T; 0] -> reflector j -> z_j^T = row 0, new tail = rows 1..p
                    double s0 = 0.0, s1 = 0.0, r2a = 0.0, r2b = 0.0, tl;
                    if constexpr (TREG) {
                        double sp[4] = {0.0, 0.0, 0.0, 0.0};
    #pragma unroll
                        for (int q = 0; q < P; ++q) sp[q & 3] = fma(vq[q], tc[q], sp[q & 3]);
                        const double s = ((sp[0] + sp[1]) + (sp[2] + sp[3])) * tj;
                        sZ[m * LD + c] = tc[0] - s;
    #pragma unroll
                        for (int q = 0; q < P - 1; ++q) {
                            tc[q] = fma(-s, vq[q + 1], tc[q + 1]);
                            if (q & 1)
                                r2b = fma(tc[q], tc[q], r2b);
                            else
                                r2a = fma(tc[q], tc[q], r2a);
                        }
                        tl = -s * vq[P];
                        tc[P - 1] = tl;
                    } else {
    #pragma unroll
                        for (int q = 0; q < P; ++q) {
                            if (q & 1)
                                s1 = fma(vq[q], sT[q * LD + c], s1);
                            else
                                s0 = fma(vq[q], sT[q * LD + c], s0);
                        }
                        const double s = (s0 + s1) * tj;
                        sZ[m * LD + c] = sT[c] - s;
    #pragma unroll
                        for (int q = 0; q < P - 1; ++q) {
                            const double tv = fma(-s, vq[q + 1], sT[(q + 1) * LD + c]);
                            sT[q * LD + c] = tv;
                            if (q & 1)
                                r2b = fma(tv, tv, r2b);
                            else
                                r2a = fma(tv, tv, r2a);
                        }
                        tl = -s * vq[P];
                        sT[(P - 1) * LD + c] = tl;
                    }
                    const double r2 = fma(tl, tl, r2a + r2b);
                    rel2 = r2 * bet_c * bet_c;   // (the stop test on squares: no sqrt on the chain)
                    rel = sqrt(r2) * bet_c;
                    sRes[c] = rel;
                    sHist[m * P + c] = rel;
                }
                // row m of every column is final: store it, shift the window up
                if (cl) sH[(2 * P + m) * LD + c] = hc[0];
    #pragma unroll
                for (int r = 0; r < 2 * P - 1; ++r) hc[r] = hc[r + 1];
                hc[2 * P - 1] = 0.0;
                sh = m + 1;
                const double mx2 = warp_max(rel2);
                K3P(3)
                m_last = m;
                if (mx2 < tol * tol) {
                    stop = 1;
                    break;
                }
                if (s_stop_after > 0 && m == s_stop_after - 1) {
                    stop = 4;
                    break;
                }
            }
            if (cl) {
    #pragma unroll
                for (int r = 0; r < 2 * P; ++r)
                    if (sh + r < 2 * P) sH[(2 * P + sh + r) * LD + c] = hc[r];
                if constexpr (TREG) {
    #pragma unroll
                    for (int q = 0; q < P; ++q) sT[q * LD + c] = tc[q];
                }
            }
            __syncwarp();
            K3P(4)
            // ---- Ainv = R_kk^{-1} (columns past m_last: identity) (eqn.search-dir-comp):
            //      column l of the back substitution in registers (lane l), in the same FMA order
            if (cl) {
                const int l = lane;
                double ic[P];
    #pragma unroll
                for (int r = P - 1; r >= 0; --r) {
                    double s = (r == l) ? 1.0 : 0.0;
                    if (l <= m_last && r <= l) {
    #pragma unroll
                        for (int c2 = r + 1; c2 < P; ++c2)
                            if (c2 <= l) s = fma(-sH[(2 * P + r) * LD + c2], ic[c2], s);
                        ic[r] = s * sRd[r];
                    } else {
                        ic[r] = s;
                    }
                    sI[r * LD + l] = ic[r];
                }
            }
        } else {
            const unsigned am_k = s_am_k, am_k1 = s_am_k1;
            for (int m = 0; m < P; ++m) {
                const long long j = j0 + m;
                if (j > maxit) {
                    stop = 2;
                    break;
                }
                // shrink: every index of the window j .. j+p-1 removed -> the basis is exhausted
                // (lanes >= m of this block, lanes < m of the next)
                if (am_k | am_k1) {
                    const unsigned all = P >= 32 ? 0xffffffffu : ((1u << P) - 1u);
                    const unsigned lo = m >= 32 ? 0xffffffffu : ((1u << m) - 1u);
                    if ((((am_k & ~lo) | (am_k1 & lo)) & all) == all) {
                        stop = 5;
                        break;
                    }
                }
                // shrink: u_j removed -> column j of \bar H is deleted: identity reflector,
                // R column zero (placeholder 1 on the diagonal for R_kk^{-1}), z_j = the tail's first
                // (zero) row, m_j = 0
                const bool gone = (am_k >> m) & 1u;
                const int o = 2 * P + m;
                const double alpha = sH[o * LD + m];
                double x2 = 0.0;
                for (int q = 1 + lane; q <= P; q += 32) x2 = fma(sH[(o + q) * LD + m], sH[(o + q) * LD + m], x2);
                x2 = warp_sum(x2);
                K3P(0)
                // dlarfg (C20): beta = -sign(alpha) ||(alpha, x)||, tau = (beta - alpha)/beta,
                // v = x/(alpha - beta); one reciprocal 1/(beta (alpha - beta)) serves both quotients
                double tj, beta, scl, rbeta;   // (rbeta = 1 / beta)
                if (gone) {
                    tj = 0.0;
                    beta = 1.0;
                    scl = 0.0;
                    rbeta = 1.0;
                } else if (x2 == 0.0) {   // (||x|| = 0)
                    tj = 0.0;
                    beta = alpha;
                    scl = 0.0;
                    rbeta = 1.0 / beta;
                } else {
                    beta = -copysign(sqrt(fma(alpha, alpha, x2)), alpha);
                    const double s = alpha - beta;
                    const double inv = 1.0 / (beta * s);
                    tj = -s * s * inv;
                    scl = beta * inv;
                    rbeta = s * inv;
                }
                if (!gone && fabs(beta) <= DBL_EPSILON * sHn[m]) {
                    stop = 3;
                    break;
                }
                if (lane == 0) sRd[m] = rbeta;   // 1 / r_jj for R_kk^{-1}
                K3P(1)
                double* vj = sVb + m * (P + 2);
                for (int q = lane; q <= P; q += 32) vj[q] = (q == 0) ? 1.0 : sH[(o + q) * LD + m] * scl;
                if (lane == 0) vj[P + 1] = tj;
                __syncwarp();
                if (lane == 0) {
                    __threadfence_block();
                    s_ready = m + 1;   // (warps 1-3 accumulate Q_k meanwhile)
                }
                for (int q = lane; q <= P; q += 32) sH[(o + q) * LD + m] = (q == 0) ? beta : 0.0;
                double rel = 0.0;
                K3P(2)
                if (lane < P) {
                    const int c = lane;
                    // (the serial chain of this loop bounds K3b: each dot product runs as two interleaved
                    // partial sums -- half the dependent FMA latency per reflector)
                    if (c > m) {   // later columns of this block
                        double* h = sH + o * LD + c;
                        double s0 = 0.0, s1 = 0.0;
    #pragma unroll
                        for (int q = 0; q <= P; q += 2) {
                            s0 = fma(vj[q], h[q * LD], s0);
                            if (q + 1 <= P) s1 = fma(vj[q + 1], h[(q + 1) * LD], s1);
                        }
                        const double s = (s0 + s1) * tj;
    #pragma unroll
                        for (int q = 0; q <= P; ++q) h[q * LD] = fma(-s, vj[q], h[q * LD]);
                    }
                    // [T; 0] -> reflector j -> z_j^T = row 0, new tail = rows 1..p
                    double s0 = 0.0, s1 = 0.0;
    #pragma unroll
                    for (int q = 0; q < P; q += 2) {
                        s0 = fma(vj[q], sT[q * LD + c], s0);
                        if (q + 1 < P) s1 = fma(vj[q + 1], sT[(q + 1) * LD + c], s1);
                    }
                    const double s = (s0 + s1) * tj;
                    sZ[m * LD + c] = sT[c] - s;
                    double r2a = 0.0, r2b = 0.0;
    #pragma unroll
                    for (int q = 0; q < P - 1; ++q) {
                        const double tv = fma(-s, vj[q + 1], sT[(q + 1) * LD + c]);
                        sT[q * LD + c] = tv;
                        if (q & 1)
                            r2b = fma(tv, tv, r2b);
                        else
                            r2a = fma(tv, tv, r2a);
                    }
                    const double tl = -s * vj[P];
                    sT[(P - 1) * LD + c] = tl;
                    const double r2 = fma(tl, tl, r2a + r2b);
                    rel = sqrt(r2) * sBeta[c];
                    sRes[c] = rel;
                    sHist[m * P + c] = rel;
                }
                const double mx = warp_max(rel);
                K3P(3)
                m_last = m;
                if (mx < tol) {
                    stop = 1;
                    break;
                }
                if (s_stop_after > 0 && m == s_stop_after - 1) {
                    stop = 4;
                    break;
                }
                __syncwarp();
            }
            __syncwarp();
            K3P(4)
            // ---- Ainv = R_kk^{-1} (columns past m_last: identity) (eqn.search-dir-comp)
            if (lane < P) {
                const int l = lane;
                for (int r = P - 1; r >= 0; --r) {
                    double s = (r == l) ? 1.0 : 0.0;
                    if (l <= m_last && r <= l) {
                        for (int c = r + 1; c <= l; ++c) s = fma(-sH[(2 * P + r) * LD + c], sI[c * LD + l], s);
                        sI[r * LD + l] = s * sRd[r];
                    } else {
                        sI[r * LD + l] = s;
                    }
                }
            }
        }
        K3P(5)
#ifdef K3B_PROF
        if (lane == 0 && tr)
            for (int i = 0; i < 6; ++i) tr[TRACE_PTS + i] = (unsigned long long)pc[i];   // (CTA 1's unused slot)
#endif
        if (lane == 0) {
            s_mlast = m_last;
            s_stop = stop;
            __threadfence_block();
            s_done = 1;
        }
    } else {
        // ---- Q_k = H_{kp} ... H_{(k-1)p+1} on the block's 2p rows (f2), accumulated by warps 1-3 while
        //      warp 0 generates the reflectors: the action of this block's reflectors (those
        //      generated before a stop) for phase A of blocks k+1 and k+2; column c of Q_k is e_c with
        //      the reflectors applied in order.  TPC consecutive lanes per column, each summing and
        //      updating the rows t = sub (mod TPC) of a reflector's p+1, the partial dots combined by
        //      xor shuffles inside the group
        constexpr int TPC0 = (K3T - 32) / (2 * P);
        constexpr int TPC = TPC0 >= 32 ? 32 : TPC0 >= 16 ? 16 : TPC0 >= 8 ? 8 : TPC0 >= 4 ? 4 : TPC0 >= 2 ? 2 : 1;
        static_assert((K3T - 32) / TPC >= 2 * P, "one pass over the columns");
        const int ct = tid - 32, c = ct / TPC, sub = ct % TPC;
        const bool live = c < 2 * P;
        double* q = sQ + (live ? c : 0);   // column c (stride LDQ; phase A is done with sQ)
        if (live)
            for (int r = sub; r < 2 * P; r += TPC) q[r * S::LDQ] = r == c ? 1.0 : 0.0;
        __syncwarp();
        for (int m = 0; m < P; ++m) {   // reflector m acts on block rows m .. m+p
            while (s_ready <= m && !s_done) __nanosleep(32);
            if (s_ready <= m) break;   // (warp 0 stopped before generating reflector m)
            __threadfence_block();
            const double* v = sVb + m * (P + 2);
            double sd = 0.0;
            if (live)
#pragma unroll
                for (int t = sub; t <= P; t += TPC) sd = fma(v[t], q[(m + t) * S::LDQ], sd);
#pragma unroll
            for (int o = 1; o < TPC; o <<= 1) sd += __shfl_xor_sync(FULL, sd, o);
            sd *= v[P + 1];
            if (live)
#pragma unroll
                for (int t = sub; t <= P; t += TPC) q[(m + t) * S::LDQ] = fma(-sd, v[t], q[(m + t) * S::LDQ]);
            __syncwarp();
        }
        if (live) {
            double* Qg = st->Qacc[k & 1];
            for (int r = sub; r < 2 * P; r += TPC) Qg[r * (2 * MAXP) + c] = q[r * S::LDQ];
        }
    }
    __syncthreads();
    trace_pt(tr, 3);
    const int m_last = s_mlast, stop = s_stop;
    // ---- stores (all threads): B1 = R_{k-1,k} Ainv, B2 = R_{k-2,k} Ainv, side state for block k+1
    for (int t = tid; t < P * P; t += K3T) {
        const int a2 = t / P, l = t % P, g = a2 * MAXP + l;
        double s1 = 0.0, s2 = 0.0;
        for (int b = 0; b <= m_last; ++b) {
            s1 = fma(sH[(P + a2) * LD + b], sI[b * LD + l], s1);
            if (a2 >= b) s2 = fma(sH[a2 * LD + b], sI[b * LD + l], s2);
        }
        st->B1[par][g] = s1;
        st->B2[par][g] = s2;
        st->Ainv[par][g] = sI[a2 * LD + l];
        st->Z[par][g] = sZ[a2 * LD + l];
        st->Zh[k % 3][g] = sZ[a2 * LD + l];
        st->T[g] = sT[a2 * LD + l];
        st->CprevS[g] = sC[a2 * LD + l];
    }
    if constexpr (P % 8 == 0) {
        // the update's factors in the DMMA fragment order (dmma_update loads them as they are):
        // Tr_k Ainv in cta_matmul_nn's arithmetic order, -B2, -B1, Z_k
        __syncthreads();   // B1 / B2 / Ainv of this block are in st
        const double* Tk = st->Tr[k % 3];
        for (int t = tid; t < P * P; t += K3T) {
            const int blk = t / 32, l = t % 32, kc = blk / (P / 8), nc = blk % (P / 8);
            const int r = kc * 4 + l % 4, c = nc * 8 + l / 4, g = r * MAXP + c;
            double s = 0.0;
            for (int i = 0; i < P; ++i) s = fma(Tk[r * MAXP + i], st->Ainv[par][i * MAXP + c], s);
            st->uf[par][0][t] = s;
            st->uf[par][1][t] = -st->B2[par][g];
            st->uf[par][2][t] = -st->B1[par][g];
            st->ufz[k % 3][t] = st->Zh[k % 3][g];
        }
    }
    trace_pt(tr, 6);
    trace_pt(tr, 7);
    for (int t = tid; t < P; t += K3T) st->res[t] = sRes[t];
    if (s_hcap > 0)
        for (int t = tid; t < (m_last + 1) * P; t += K3T) {
            const long long j = j0 + t / P;
            if (j < s_hcap) st->hist[j * P + t % P] = sHist[t];
        }
    if (tid == 0) {
        const long long jd = s_jd + (m_last + 1);
        st->j_done = jd;
        st->side_go = m_last >= 0 ? 1 : 0;
        if (m_last >= 0) st->k_side = k + 1;
        int status = 1;
        bool end = false;
        if (stop == 1) { status = 0; end = true; }
        else if (stop == 2 || stop == 5) { status = 1; end = true; }
        else if (stop == 3) { status = -6; end = true; }
        else if (stop == 4) { status = -5; end = true; }
        else if (jd >= maxit) { status = 1; end = true; }
        st->status = status;
        if (end) st->stop_side_at = k + 1;
        st->hflags->status = status;
        st->hflags->j_done = jd;
        st->hflags->k_side = st->k_side;
        if (end) {
            st->hflags->stop_blk = k;
            st->hflags->side_done = 1;
        }
        __threadfence_system();
    }
    trace_pt(tr, 5);
}

// ------------------------------------------------------------------ K4b: directions and X (side)

struct K4bArgs {
    const double* U;      // V_k (U_k = V_k Tr_k)
    double* M2;           // M_{k-2} in, M_k out
    const double* M1;     // M_{k-1}
    double* X;
    long long n;
    DevState* st;
    int sk;               // k mod 3
    int tpw;              // row groups per warp, contiguous
    int par;              // k mod 2 (K3b output buffer)
    int force;            // 1: apply regardless of side_go (host flush of a pending update)
    long long blk;        // k (recorded in upd_last; 0: not recorded)
    // X update mode (DMMA update only): 0 X += M_k Z_k; 1 defer it
    // (no X traffic); 2 X += M_{k-1} Z_{k-1} + M_k Z_k (the deferred pair, in that order -- bitwise
    // the two single updates); 3 X += M_k Z_k alone with M2 holding M_k (host flush)
    int xmode;
    long long zb;         // k for the Zh slots (xmode != 0)
};

template <int P>
struct K4bSmem {
    static constexpr int TILE = PC<P>::RPW * PC<P>::RS;
    static constexpr int pipe = (NT / 32) * NSTAGE * 4 * TILE;   // V, M_{k-2}, M_{k-1}, X tiles
    static constexpr size_t bytes = sizeof(double) * (4 * P * P + pipe);
};

template <int P>
__global__ void __launch_bounds__(NT) k4b_update(K4bArgs a) {
    using C = PC<P>;
    constexpr int VEC = C::VEC, LANES = C::LANES, LP = C::LP, RPW = C::RPW, WARPS = NT / 32;
    constexpr int TILE = K4bSmem<P>::TILE;
    DevState* st = a.st;
    if (!a.force && !st->side_go) return;
    if (a.blk > 0 && blockIdx.x == 0 && threadIdx.x == 0) st->upd_last = a.blk;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int sub = lane % LP, rsub = lane / LP;
    const bool act = sub < LANES;
    const int c0 = sub * VEC;
    extern __shared__ __align__(16) double dyn4[];
    double* sAi = dyn4;
    double* sB1 = sAi + P * P;
    double* sB2 = sB1 + P * P;
    double* sZ = sB2 + P * P;
    double* sPipe = sZ + P * P;
    {
        // sAi = Tr_k R_kk^{-1} (built in sZ's space first)
        double* sT = sAi;
        double* sR = sB1;
        const double* Tk = st->Tr[a.sk];
        for (int t = threadIdx.x; t < P * P; t += NT) {
            const int g = (t / P) * MAXP + t % P;
            sT[t] = Tk[g];
            sR[t] = st->Ainv[a.par][g];
        }
        __syncthreads();
        cta_matmul_nn<P>(sT, P, sR, P, sZ, P);
        __syncthreads();
        for (int t = threadIdx.x; t < P * P; t += NT) {
            const int g = (t / P) * MAXP + t % P;
            sAi[t] = sZ[t];
            sB1[t] = st->B1[a.par][g];
            sB2[t] = st->B2[a.par][g];
        }
        __syncthreads();
        for (int t = threadIdx.x; t < P * P; t += NT) sZ[t] = st->Z[a.par][(t / P) * MAXP + t % P];
        __syncthreads();
    }
    constexpr int RS = C::RS;
    double* wb = sPipe + warp * NSTAGE * 4 * TILE;
    const long long t0 = (long long)blockIdx.x * WARPS + warp, ts = (long long)gridDim.x * WARPS;
    const long long ntiles = (a.n + RPW - 1) / RPW;
    auto issue = [&](long long it, int slot) {
        const long long t = t0 + it * ts;
        const long long i = t * RPW + rsub;
        const bool ok = act && t < ntiles && i < a.n;
        const long long ic = (ok ? i : 0) * P + c0;
        double* sl = wb + slot * 4 * TILE + rsub * RS + c0;
        if (act) {   // idle lanes must not touch the next row's slots
            cp_async_vec<VEC>(sl, a.U + ic, ok);
            cp_async_vec<VEC>(sl + TILE, a.M2 + ic, ok);
            cp_async_vec<VEC>(sl + 2 * TILE, a.M1 + ic, ok);
            cp_async_vec<VEC>(sl + 3 * TILE, a.X + ic, ok);
        }
        cp_commit();
    };
#pragma unroll
    for (int s = 0; s < NSTAGE - 1; ++s) issue(s, s);
    for (long long it = 0; t0 + it * ts < ntiles; ++it) {
        issue(it + NSTAGE - 1, (int)((it + NSTAGE - 1) % NSTAGE));
        cp_wait<NSTAGE - 1>();
        __syncwarp();
        double* sl = wb + (int)(it % NSTAGE) * 4 * TILE + rsub * RS;
        const double* tv = sl;
        double* tm2 = sl + TILE;
        const double* tm1 = sl + 2 * TILE;
        const double* tx = sl + 3 * TILE;
        const long long i = (t0 + it * ts) * RPW + rsub;
        const bool valid = act && i < a.n;
        // M_k = U_k R_kk^{-1} - M_{k-2} B2 - M_{k-1} B1   (eqn.search-dir-comp)
        double mk[VEC];
#pragma unroll
        for (int v = 0; v < VEC; ++v) mk[v] = 0.0;
#pragma unroll
        for (int b = 0; b < P; ++b) {
            const double xu = tv[b], x2 = tm2[b], x1 = tm1[b];
#pragma unroll
            for (int v = 0; v < VEC; ++v) {
                const int m = c0 + v;
                mk[v] = fma(xu, sAi[b * P + m], mk[v]);
                mk[v] = fma(-x2, sB2[b * P + m], mk[v]);
                mk[v] = fma(-x1, sB1[b * P + m], mk[v]);
            }
        }
        __syncwarp();
        if (act) {
#pragma unroll
            for (int v = 0; v < VEC; ++v) tm2[c0 + v] = mk[v];
        }
        if (valid) stv<VEC>(a.M2 + i * P + c0, mk);
        __syncwarp();
        if (valid) {
            // X += M_k Z_k   (eqn.approx-update)
            double x[VEC];
#pragma unroll
            for (int v = 0; v < VEC; ++v) x[v] = tx[c0 + v];
#pragma unroll
            for (int b = 0; b < P; ++b) {
                const double xm = tm2[b];
#pragma unroll
                for (int v = 0; v < VEC; ++v) x[v] = fma(xm, sZ[b * P + c0 + v], x[v]);
            }
            stv<VEC>(a.X + i * P + c0, x);
        }
        __syncwarp();
    }
    cp_wait<0>();
}

}  // namespace bmr
