// step_kernels.cuh -- sm_100a kernels of one block step of banded-Lanczos block MINRES.
//
// main branch (critical path), block k:
//   K1  k1_spmm     W = A U_k; ||A u_j||; W -= U_{k-1} C_{k-1}^T; G = U_k^T W
//                   (row a1; Alg. 2; symmetric reuse P:270-272)
//   K2  k2_orth     W' = W - U_k G_s; W'^T W'; r_q^T W'; last CTA: Cholesky W' = U_{k+1} C_k,
//                   breakdown test h_{j+p,j} <= tau ||A u_j||, C_k^{-1}, pool coefficients
//                   (rows a2/a3; Alg. 1)
//   K4a k4a_basis   U_{k+1} = W' C_k^{-1}; pool r_q -= U_{k+1} coef
// side branch, block k (runs beside the main branch of block k+1):
//   K3b k3b_smallqr one warp: p Hessenberg columns, <= 2p Householder reflectors each,
//                   z_j, residuals, stop test, direction matrices (row a4; P:424-468,
//                   Alg. 2)
//   K4b k4b_update  M_k = (U_k - M_{k-2}R_{k-2,k} - M_{k-1}R_{k-1,k})R_kk^{-1}; X += M_k Z_k
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
    const double* X;      // U_k (gathered by global column)
    const double* Uprev;  // U_{k-1}
    double* Y;            // W
    long long n;
    DevState* st;
    double* part;
    int par;              // k mod 2
};

template <int P>
constexpr int k1_min_blocks() { return P <= 8 ? 3 : 1; }

// W = A X.  Each row's sum runs over its CSR entries in stored order with fma (bitwise equal
// to the oracle's product); the entries of a row are fetched CH at a time (all column
// indices, then all gathers) so that a lane has CH independent loads in flight.
template <int P, bool EPI>
__global__ void __launch_bounds__(NT, k1_min_blocks<P>()) k1_spmm(K1Args a) {
    using C = PC<P>;
    constexpr int VEC = C::VEC, LANES = C::LANES, LP = C::LP, RPW = C::RPW, WARPS = NT / 32;
    constexpr int E = P * P + P;
    constexpr int CH = P <= 8 ? 4 : 4;
    DevState* st = a.st;
    if constexpr (EPI) {
        if (!st->run_main) return;
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int sub = lane % LP, rsub = lane / LP;
    const bool act = sub < LANES;
    const int c0 = sub * VEC;
    __shared__ double sC[EPI ? P * P : 1];
    __shared__ __align__(16) double sU[WARPS][EPI ? RPW * P : 2];
    __shared__ __align__(16) double sV[WARPS][EPI ? RPW * P : 2];
    __shared__ double sAcc[EPI ? E : 1];
    bool has_prev = false;
    if constexpr (EPI) {
        has_prev = st->k_main > 1;
        const double* Cp = st->Ck[a.par ^ 1];   // C_{k-1}
        for (int t = threadIdx.x; t < P * P; t += NT) sC[t] = Cp[(t / P) * MAXP + t % P];
        __syncthreads();
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
                if (has_prev) ldv<VEC>(a.Uprev + i * P + c0, up);
            }
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
            if (act) {
#pragma unroll
                for (int v = 0; v < VEC; ++v) {
                    sU[warp][rsub * P + c0 + v] = u[v];
                    sV[warp][rsub * P + c0 + v] = up[v];
                }
            }
            __syncwarp();
            if (valid) {
#pragma unroll
                for (int v = 0; v < VEC; ++v) om[v] = fma(acc[v], acc[v], om[v]);
                if (has_prev) {
                    // W(:,m) -= sum_b U_{k-1}(:,b) C_{k-1}(m,b)  (h_{i,j} = h_{j,i})
#pragma unroll
                    for (int b = 0; b < P; ++b) {
                        const double x = sV[warp][rsub * P + b];
#pragma unroll
                        for (int v = 0; v < VEC; ++v) acc[v] = fma(-x, sC[(c0 + v) * P + b], acc[v]);
                    }
                }
                // G(b,m) += U_k(i,b) W(i,m)
#pragma unroll
                for (int b = 0; b < P; ++b) {
                    const double x = sU[warp][rsub * P + b];
#pragma unroll
                    for (int v = 0; v < VEC; ++v) g[b][v] = fma(x, acc[v], g[b][v]);
                }
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
        cluster_reduce(sAcc, E, P, a.part, st->G[a.par], st->om2[a.par], &st->cnt1);
    }
}

// ------------------------------------------------------------------ K2: W' = W - U_k G_s, Grams, C_k

struct K2Args {
    double* W;
    const double* U;      // U_k
    const double* pool;   // n x pool_cap row-major
    long long n;
    DevState* st;
    double* part;
    int par;
};

// Cholesky W'^T W' = C_k^T C_k (right-looking, warp 0 of the CTA holding the totals), the
// breakdown / cancellation test, C_k^{-1} and the pool coefficients.  Returns false on a
// breakdown (the main branch stops at this block and the host runs the column path).
template <int P>
struct K2Smem {
    static constexpr int LD = P + 1;
    static constexpr int loop = P * P + 2 * (NT / 32) * PC<P>::RPW * P + P * P + MAXQ * P;
    static constexpr int tail = 3 * P * LD + 2 * P;
    static constexpr size_t bytes = sizeof(double) * (loop + tail);
};

template <int P>
__device__ bool k3a_factor(DevState* st, int par, double* scratch) {
    constexpr int LD = P + 1;
    double* sA = scratch;
    double* sC = sA + P * LD;
    double* sCi = sC + P * LD;
    double* sD = sCi + P * LD;
    double* sOm = sD + P;
    __shared__ int s_bad;
    const int tid = threadIdx.x, lane = tid & 31;
    for (int t = tid; t < P * P; t += NT) {
        const int r = t / P, c = t % P;
        sA[r * LD + c] = st->Gram2[r * MAXP + c];
        sC[r * LD + c] = 0.0;
    }
    for (int t = tid; t < P; t += NT) {
        sD[t] = st->Gram2[t * MAXP + t];
        sOm[t] = st->om2[par][t];
    }
    __syncthreads();
    if (tid < 32) {
        const double tau = st->tau;
        bool bad = false;
        for (int m = 0; m < P; ++m) {
            const double d = sA[m * LD + m];
            // breakdown: h_{j+p,j}^2 = d <= tau^2 ||A u_j||^2; cancellation guard: the pivot kept
            // < 1e-4 of ||w'_m||^2 (more than 4 digits lost) -> column path
            if (!(d > tau * tau * sOm[m]) || !(d >= 1e-4 * sD[m])) {
                bad = true;
                break;
            }
            const double cmm = sqrt(d);
            const double rc = 1.0 / cmm;
            for (int c = m + lane; c < P; c += 32) sC[m * LD + c] = (c == m) ? cmm : sA[m * LD + c] * rc;
            __syncwarp();
            // trailing update A(r,c) -= C(m,r) C(m,c), m < r <= c
            for (int t = lane; t < P * P; t += 32) {
                const int r = t / P, c = t % P;
                if (r > m && c >= r) sA[r * LD + c] = fma(-sC[m * LD + r], sC[m * LD + c], sA[r * LD + c]);
            }
            __syncwarp();
        }
        if (lane == 0) s_bad = bad;
        if (!bad && lane < P) {
            // column `lane` of C_k^{-1} (back substitution)
            const int l = lane;
            for (int r = P - 1; r >= 0; --r) {
                double s = (r == l) ? 1.0 : 0.0;
                for (int c = r + 1; c <= l; ++c) s = fma(-sC[r * LD + c], sCi[c * LD + l], s);
                sCi[r * LD + l] = (r <= l) ? s / sC[r * LD + r] : 0.0;
            }
        }
        const int Q = st->q_live;
        if (!bad && lane < Q) {
            // coef(:,q) = C_k^{-T} (W'^T r_q) = U_{k+1}^T r_q
            double y[P];
#pragma unroll
            for (int m = 0; m < P; ++m) {
                double s = st->pdot[lane * MAXP + m];
#pragma unroll
                for (int i = 0; i < m; ++i) s = fma(-sC[i * LD + m], y[i], s);
                y[m] = s / sC[m * LD + m];
                st->coef[par][m * MAXQ + lane] = y[m];
            }
        }
    }
    __syncthreads();
    if (s_bad) {
        if (tid == 0) {
            st->need_slow = 1;
            st->run_main = 0;
            st->bd_at = st->k_main;
            st->hflags->bd_at = st->k_main;
            st->hflags->need_slow = 1;
            __threadfence_system();
        }
        return false;
    }
    for (int t = tid; t < P * P; t += NT) {
        const int r = t / P, c = t % P;
        st->Ck[par][r * MAXP + c] = sC[r * LD + c];
        st->Cinv[par][r * MAXP + c] = sCi[r * LD + c];
    }
    if (tid == 0) {
        st->k_main = st->k_main + 1;
        st->hflags->k_main = st->k_main;
    }
    return true;
}

template <int P>
__global__ void __launch_bounds__(NT, P <= 8 ? 2 : 1) k2_orth(K2Args a) {
    using C = PC<P>;
    constexpr int VEC = C::VEC, LANES = C::LANES, LP = C::LP, RPW = C::RPW, WARPS = NT / 32;
    DevState* st = a.st;
    if (!st->run_main) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int sub = lane % LP, rsub = lane / LP;
    const bool act = sub < LANES;
    const int c0 = sub * VEC;
    const int Q = st->q_live, qf = st->q_first, qc = st->pool_cap;
    const int E = P * P + Q * P;
    extern __shared__ __align__(16) double dyn2[];
    double* sG = dyn2;
    double(*sU)[RPW * P] = reinterpret_cast<double(*)[RPW * P]>(sG + P * P);
    double(*sW)[RPW * P] = reinterpret_cast<double(*)[RPW * P]>(sG + P * P + WARPS * RPW * P);
    double* sAcc = sG + P * P + 2 * WARPS * RPW * P;
    double* sTail = sAcc + P * P + MAXQ * P;
    // G_s: lower triangle of G mirrored (the paper computes h_{i,j} for i >= j)
    const double* Gp = st->G[a.par];
    for (int t = threadIdx.x; t < P * P; t += NT) {
        const int r = t / P, c = t % P;
        sG[t] = r >= c ? Gp[r * MAXP + c] : Gp[c * MAXP + r];
    }
    __syncthreads();
    double g[P][VEC], pq[MAXQ][VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
#pragma unroll
        for (int b = 0; b < P; ++b) g[b][v] = 0.0;
#pragma unroll
        for (int q = 0; q < MAXQ; ++q) pq[q][v] = 0.0;
    }
    const long long stride = (long long)gridDim.x * WARPS * RPW;
    for (long long base = ((long long)blockIdx.x * WARPS + warp) * RPW; base < a.n; base += stride) {
        const long long i = base + rsub;
        const bool valid = act && i < a.n;
        double w[VEC], u[VEC], r[MAXQ];
#pragma unroll
        for (int v = 0; v < VEC; ++v) w[v] = u[v] = 0.0;
        if (valid) {
            ldc<VEC>(a.W + i * P + c0, w);
            ldv<VEC>(a.U + i * P + c0, u);
#pragma unroll
            for (int q = 0; q < MAXQ; ++q)
                if (q < Q) r[q] = a.pool[i * qc + qf + q];
        }
        if (act) {
#pragma unroll
            for (int v = 0; v < VEC; ++v) sU[warp][rsub * P + c0 + v] = u[v];
        }
        __syncwarp();
        if (valid) {
#pragma unroll
            for (int b = 0; b < P; ++b) {
                const double x = sU[warp][rsub * P + b];
#pragma unroll
                for (int v = 0; v < VEC; ++v) w[v] = fma(-x, sG[b * P + c0 + v], w[v]);
            }
            stv<VEC>(a.W + i * P + c0, w);
        }
        if (act) {
#pragma unroll
            for (int v = 0; v < VEC; ++v) sW[warp][rsub * P + c0 + v] = valid ? w[v] : 0.0;
        }
        __syncwarp();
        if (valid) {
#pragma unroll
            for (int b = 0; b < P; ++b) {
                const double x = sW[warp][rsub * P + b];
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
    if (cluster_reduce(sAcc, E, P, a.part, st->Gram2, st->pdot, &st->cnt2)) k3a_factor<P>(st, a.par, sTail);
}

// ------------------------------------------------------------------ K4a: U_{k+1} = W' C_k^{-1}

struct K4aArgs {
    const double* W;      // W' (or the materialised U_{k+1} when given_main)
    double* Unext;        // U_{k+1} (the slot of U_{k-1})
    double* pool;
    long long n;
    DevState* st;
    int par;
};

template <int P>
__global__ void __launch_bounds__(NT) k4a_basis(K4aArgs a) {
    using C = PC<P>;
    constexpr int VEC = C::VEC, LANES = C::LANES, LP = C::LP, RPW = C::RPW, WARPS = NT / 32;
    constexpr int RG = 2;
    DevState* st = a.st;
    if (!st->run_main) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int sub = lane % LP, rsub = lane / LP;
    const bool act = sub < LANES;
    const int c0 = sub * VEC;
    const bool given = st->given_main != 0;
    const int Q = given ? 0 : st->q_live, qf = st->q_first, qc = st->pool_cap;
    __shared__ double sCi[P * P];
    __shared__ double sCo[P * MAXQ];
    __shared__ __align__(16) double sRow[WARPS][RG][RPW * P];
    for (int t = threadIdx.x; t < P * P; t += NT) sCi[t] = st->Cinv[a.par][(t / P) * MAXP + t % P];
    for (int t = threadIdx.x; t < P * MAXQ; t += NT) sCo[t] = st->coef[a.par][t];
    __syncthreads();
    const long long stride = (long long)gridDim.x * WARPS * RPW * RG;
    for (long long base = ((long long)blockIdx.x * WARPS + warp) * RPW * RG; base < a.n; base += stride) {
        double w[RG][VEC];
        bool valid[RG];
#pragma unroll
        for (int g = 0; g < RG; ++g) {
            const long long i = base + g * RPW + rsub;
            valid[g] = act && i < a.n;
#pragma unroll
            for (int v = 0; v < VEC; ++v) w[g][v] = 0.0;
            if (valid[g]) ldc<VEC>(a.W + i * P + c0, w[g]);
            if (act) {
#pragma unroll
                for (int v = 0; v < VEC; ++v) sRow[warp][g][rsub * P + c0 + v] = w[g][v];
            }
        }
        __syncwarp();
        double un[RG][VEC];
#pragma unroll
        for (int g = 0; g < RG; ++g) {
#pragma unroll
            for (int v = 0; v < VEC; ++v) un[g][v] = given ? w[g][v] : 0.0;
            if (!given) {
#pragma unroll
                for (int b = 0; b < P; ++b) {
                    const double xw = sRow[warp][g][rsub * P + b];
#pragma unroll
                    for (int v = 0; v < VEC; ++v) un[g][v] = fma(xw, sCi[b * P + c0 + v], un[g][v]);
                }
            }
        }
        __syncwarp();
#pragma unroll
        for (int g = 0; g < RG; ++g) {
            const long long i = base + g * RPW + rsub;
            if (valid[g]) stv<VEC>(a.Unext + i * P + c0, un[g]);
            if (act) {
#pragma unroll
                for (int v = 0; v < VEC; ++v) sRow[warp][g][rsub * P + c0 + v] = un[g][v];
            }
        }
        if (Q > 0) {
            __syncwarp();
#pragma unroll
            for (int g = 0; g < RG; ++g) {
                const long long i = base + g * RPW + rsub;
                if (valid[g])
                    for (int q = sub; q < Q; q += LANES) {
                        double r = a.pool[i * qc + qf + q];
                        for (int b = 0; b < P; ++b) r = fma(-sRow[warp][g][rsub * P + b], sCo[b * MAXQ + q], r);
                        a.pool[i * qc + qf + q] = r;
                    }
            }
        }
        __syncwarp();
    }
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
    static constexpr int nV = W2 * (P + 2);
    static constexpr int doubles = 6 * nA + nH + nV + 3 * P + P * P;
    static constexpr size_t bytes = sizeof(double) * doubles;
};

template <int P>
__global__ void __launch_bounds__(K3T) k3b_smallqr(DevState* st) {
    using S = K3Smem<P>;
    constexpr int W2 = S::W2, LD = S::LD;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    __shared__ long long s_k, s_jd, s_maxit, s_hcap;
    __shared__ double s_tol;
    __shared__ int s_valid, s_stop_after, s_mlast, s_stop;
    if (tid == 0) {
        const long long k = st->k_side;
        s_valid = (k < st->stop_side_at) && (k < st->bd_at);
        s_k = k;
        s_jd = st->j_done;
        s_maxit = st->maxit;
        s_hcap = st->hist ? st->hist_cap : 0;
        s_tol = st->tol;
        s_stop_after = st->stop_after;
        if (!s_valid) st->side_go = 0;
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
    double* sV = sH + S::nH;      // reflector ring: v (p+1) + tau per slot
    double* sHn = sV + S::nV;     // ||h_j||
    double* sBeta = sHn + P;      // ||b_i||
    double* sRes = sBeta + P;     // residuals of the last completed iteration
    double* sHist = sRes + P;     // residual rows of this block (P x P)
    const long long k = s_k, j0 = s_jd + 1, maxit = s_maxit;
    const int par = (int)(k & 1);
    for (int t = tid; t < P * P; t += K3T) {
        const int r = t / P, c = t % P, g = r * MAXP + c, s = r * LD + c;
        sC[s] = st->Ck[par][g];
        sT[s] = st->T[g];
        sG[s] = st->G[par][g];
        sCp[s] = st->CprevS[g];
        sZ[s] = 0.0;
    }
    for (int t = tid; t < W2 * (P + 1); t += K3T) {
        const int s = t / (P + 1), q = t % (P + 1);
        sV[s * (P + 2) + q] = st->rv[s * (MAXP + 1) + q];
    }
    for (int s = tid; s < W2; s += K3T) sV[s * (P + 2) + P + 1] = st->rtau[s];
    for (int t = tid; t < P; t += K3T) {
        sBeta[t] = st->beta[t];
        sRes[t] = st->res[t];
    }
    __syncthreads();

    if (warp == 0) {
        const double tol = s_tol;
        // ---- the p new columns of \bar H in the frame of global rows (k-3)p+1 .. (k+1)p
        //      (symmetric reuse P:923-945)
        if (lane < P) {
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
            // phase A: reflectors i = (k-3)p+1 .. (k-1)p (previous two blocks), increasing i;
            // frame offset o = i - ((k-3)p+1) touches rows o .. o+p
            const long long base = (k - 3) * P + 1;
            int slot = (int)(((base % W2) + W2) % W2);
            for (int o = 0; o < 2 * P; ++o, slot = (slot + 1 == W2 ? 0 : slot + 1)) {
                if (base + o < 1) continue;
                const double* v = sV + slot * (P + 2);
                const double t = v[P + 1];
                double* h = sH + o * LD + m;
                double s = 0.0;
#pragma unroll
                for (int q = 0; q <= P; ++q) s = fma(v[q], h[q * LD], s);
                s *= t;
#pragma unroll
                for (int q = 0; q <= P; ++q) h[q * LD] = fma(-s, v[q], h[q * LD]);
            }
        }
        __syncwarp();

        // ---- phase B: generate reflector j, apply it to the later columns and to [T; 0]
        //      (row 1 -> z_j^T), residuals, stop test (Alg. 2)
        int m_last = -1, stop = 0;  // 1 converged, 2 maxit, 3 singular R, 4 pool exhausted
        int slot = (int)(j0 % W2);
        for (int m = 0; m < P; ++m, slot = (slot + 1 == W2 ? 0 : slot + 1)) {
            const long long j = j0 + m;
            if (j > maxit) {
                stop = 2;
                break;
            }
            const int o = 2 * P + m;
            const double alpha = sH[o * LD + m];
            double x2 = 0.0;
            for (int q = 1 + lane; q <= P; q += 32) x2 = fma(sH[(o + q) * LD + m], sH[(o + q) * LD + m], x2);
            x2 = warp_sum(x2);
            const double xnorm = sqrt(x2);
            double tj, beta, scl;
            if (xnorm == 0.0) {
                tj = 0.0;
                beta = alpha;
                scl = 0.0;
            } else {
                beta = -copysign(hypot(alpha, xnorm), alpha);
                tj = (beta - alpha) / beta;
                scl = 1.0 / (alpha - beta);
            }
            if (fabs(beta) <= DBL_EPSILON * sHn[m]) {
                stop = 3;
                break;
            }
            double* vj = sV + slot * (P + 2);
            for (int q = lane; q <= P; q += 32) vj[q] = (q == 0) ? 1.0 : sH[(o + q) * LD + m] * scl;
            if (lane == 0) vj[P + 1] = tj;
            __syncwarp();
            for (int q = lane; q <= P; q += 32) sH[(o + q) * LD + m] = (q == 0) ? beta : 0.0;
            double rel = 0.0;
            if (lane < P) {
                const int c = lane;
                if (c > m) {   // later columns of this block
                    double* h = sH + o * LD + c;
                    double s = 0.0;
#pragma unroll
                    for (int q = 0; q <= P; ++q) s = fma(vj[q], h[q * LD], s);
                    s *= tj;
#pragma unroll
                    for (int q = 0; q <= P; ++q) h[q * LD] = fma(-s, vj[q], h[q * LD]);
                }
                // [T; 0] -> reflector j -> z_j^T = row 0, new tail = rows 1..p
                double s = 0.0;
#pragma unroll
                for (int q = 0; q < P; ++q) s = fma(vj[q], sT[q * LD + c], s);
                s *= tj;
                sZ[m * LD + c] = sT[c] - s;
                double r2 = 0.0;
#pragma unroll
                for (int q = 0; q < P - 1; ++q) {
                    const double tv = fma(-s, vj[q + 1], sT[(q + 1) * LD + c]);
                    sT[q * LD + c] = tv;
                    r2 = fma(tv, tv, r2);
                }
                const double tl = -s * vj[P];
                sT[(P - 1) * LD + c] = tl;
                r2 = fma(tl, tl, r2);
                const double b = sBeta[c];
                rel = b > 0.0 ? sqrt(r2) / b : 0.0;
                sRes[c] = rel;
                sHist[m * P + c] = rel;
            }
            const double mx = warp_max(rel);
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
        // ---- Ainv = R_kk^{-1} (columns past m_last: identity) (eqn.search-dir-comp)
        if (lane < P) {
            const int l = lane;
            for (int r = P - 1; r >= 0; --r) {
                double s = (r == l) ? 1.0 : 0.0;
                if (l <= m_last && r <= l) {
                    for (int c = r + 1; c <= l; ++c) s = fma(-sH[(2 * P + r) * LD + c], sI[c * LD + l], s);
                    sI[r * LD + l] = s / sH[(2 * P + r) * LD + r];
                } else {
                    sI[r * LD + l] = s;
                }
            }
        }
        if (lane == 0) {
            s_mlast = m_last;
            s_stop = stop;
        }
    }
    __syncthreads();
    const int m_last = s_mlast, stop = s_stop;
    // ---- stores (all threads): B1 = R_{k-1,k} Ainv, B2 = R_{k-2,k} Ainv, side state for block k+1
    for (int t = tid; t < P * P; t += K3T) {
        const int a2 = t / P, l = t % P, g = a2 * MAXP + l;
        double s1 = 0.0, s2 = 0.0;
        for (int b = 0; b <= m_last; ++b) {
            s1 = fma(sH[(P + a2) * LD + b], sI[b * LD + l], s1);
            if (a2 >= b) s2 = fma(sH[a2 * LD + b], sI[b * LD + l], s2);
        }
        st->B1[g] = s1;
        st->B2[g] = s2;
        st->Ainv[g] = sI[a2 * LD + l];
        st->Z[g] = sZ[a2 * LD + l];
        st->T[g] = sT[a2 * LD + l];
        st->CprevS[g] = sC[a2 * LD + l];
    }
    for (int t = tid; t < W2 * (P + 1); t += K3T) {
        const int s = t / (P + 1), q = t % (P + 1);
        st->rv[s * (MAXP + 1) + q] = sV[s * (P + 2) + q];
    }
    for (int s = tid; s < W2; s += K3T) st->rtau[s] = sV[s * (P + 2) + P + 1];
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
        else if (stop == 2) { status = 1; end = true; }
        else if (stop == 3) { status = -6; end = true; }
        else if (stop == 4) { status = -5; end = true; }
        else if (jd >= maxit) { status = 1; end = true; }
        st->status = status;
        if (end) st->stop_side_at = k + 1;
        st->hflags->status = status;
        st->hflags->j_done = jd;
        st->hflags->k_side = st->k_side;
        if (end) st->hflags->side_done = 1;
        __threadfence_system();
    }
}

// ------------------------------------------------------------------ K4b: directions and X (side)

struct K4bArgs {
    const double* U;      // U_k
    double* M2;           // M_{k-2} in, M_k out
    const double* M1;     // M_{k-1}
    double* X;
    long long n;
    DevState* st;
};

template <int P>
struct K4bSmem {
    static constexpr size_t bytes = sizeof(double) * (4 * P * P + (NT / 32) * 2 * 3 * PC<P>::RPW * P);
};

template <int P>
__global__ void __launch_bounds__(NT) k4b_update(K4bArgs a) {
    using C = PC<P>;
    constexpr int VEC = C::VEC, LANES = C::LANES, LP = C::LP, RPW = C::RPW, WARPS = NT / 32;
    constexpr int RG = 2;
    DevState* st = a.st;
    if (!st->side_go) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int sub = lane % LP, rsub = lane / LP;
    const bool act = sub < LANES;
    const int c0 = sub * VEC;
    extern __shared__ __align__(16) double dyn4[];
    double* sAi = dyn4;
    double* sB1 = sAi + P * P;
    double* sB2 = sB1 + P * P;
    double* sZ = sB2 + P * P;
    double(*sRow)[RG][3][RPW * P] = reinterpret_cast<double(*)[RG][3][RPW * P]>(sZ + P * P);
    for (int t = threadIdx.x; t < P * P; t += NT) {
        const int g = (t / P) * MAXP + t % P;
        sAi[t] = st->Ainv[g];
        sB1[t] = st->B1[g];
        sB2[t] = st->B2[g];
        sZ[t] = st->Z[g];
    }
    __syncthreads();
    const long long stride = (long long)gridDim.x * WARPS * RPW * RG;
    for (long long base = ((long long)blockIdx.x * WARPS + warp) * RPW * RG; base < a.n; base += stride) {
        double u[RG][VEC], m2[RG][VEC], m1[RG][VEC], x[RG][VEC];
        bool valid[RG];
#pragma unroll
        for (int g = 0; g < RG; ++g) {
            const long long i = base + g * RPW + rsub;
            valid[g] = act && i < a.n;
#pragma unroll
            for (int v = 0; v < VEC; ++v) u[g][v] = m2[g][v] = m1[g][v] = x[g][v] = 0.0;
            if (valid[g]) {
                ldv<VEC>(a.U + i * P + c0, u[g]);
                ldc<VEC>(a.M2 + i * P + c0, m2[g]);
                ldc<VEC>(a.M1 + i * P + c0, m1[g]);
                ldc<VEC>(a.X + i * P + c0, x[g]);
            }
        }
#pragma unroll
        for (int g = 0; g < RG; ++g) {
            if (act) {
#pragma unroll
                for (int v = 0; v < VEC; ++v) {
                    sRow[warp][g][0][rsub * P + c0 + v] = u[g][v];
                    sRow[warp][g][1][rsub * P + c0 + v] = m2[g][v];
                    sRow[warp][g][2][rsub * P + c0 + v] = m1[g][v];
                }
            }
        }
        __syncwarp();
        double mk[RG][VEC];
#pragma unroll
        for (int g = 0; g < RG; ++g) {
#pragma unroll
            for (int v = 0; v < VEC; ++v) mk[g][v] = 0.0;
#pragma unroll
            for (int b = 0; b < P; ++b) {
                const double xu = sRow[warp][g][0][rsub * P + b];
                const double x2 = sRow[warp][g][1][rsub * P + b];
                const double x1 = sRow[warp][g][2][rsub * P + b];
#pragma unroll
                for (int v = 0; v < VEC; ++v) {
                    const int m = c0 + v;
                    mk[g][v] = fma(xu, sAi[b * P + m], mk[g][v]);
                    mk[g][v] = fma(-x2, sB2[b * P + m], mk[g][v]);
                    mk[g][v] = fma(-x1, sB1[b * P + m], mk[g][v]);
                }
            }
        }
        __syncwarp();
#pragma unroll
        for (int g = 0; g < RG; ++g) {
            const long long i = base + g * RPW + rsub;
            if (valid[g]) stv<VEC>(a.M2 + i * P + c0, mk[g]);
            if (act) {
#pragma unroll
                for (int v = 0; v < VEC; ++v) sRow[warp][g][0][rsub * P + c0 + v] = mk[g][v];
            }
        }
        __syncwarp();
#pragma unroll
        for (int g = 0; g < RG; ++g) {
            const long long i = base + g * RPW + rsub;
            if (valid[g]) {
#pragma unroll
                for (int b = 0; b < P; ++b) {
                    const double xm = sRow[warp][g][0][rsub * P + b];
#pragma unroll
                    for (int v = 0; v < VEC; ++v) x[g][v] = fma(xm, sZ[b * P + c0 + v], x[g][v]);
                }
                stv<VEC>(a.X + i * P + c0, x[g]);
            }
        }
        __syncwarp();
    }
}

}  // namespace bmr
