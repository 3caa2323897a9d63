// kernels.cuh -- sm_100a kernels of one block step of banded-Lanczos block MINRES.
//
//   K1 k1_spmm     W = A U_k; raw norms ||A u_j||; W -= U_{k-1} C_{k-1}^T; G = U_k^T W
//                  (rows a1 of DESIGN.md; Alg. 2; symmetric reuse P:270-272)
//   K2 k2_orth     W' = W - U_k G_s; W'^T W'; r_q^T W'             (row a2/a3; Alg. 1)
//   K3 k3_smallqr  one warp: Cholesky W' = U_{k+1} C_k, breakdown test h_{j+p,j} <= tau ||A u_j||,
//                  p Hessenberg columns, <= 2p Householder reflectors each, z_j, residuals, stop
//                  (row a3/a4; Alg. 2)
//   K4 k4_update   U_{k+1} = W' C_k^{-1}; M_k = (U_k - M_{k-2}R_{k-2,k} - M_{k-1}R_{k-1,k})R_kk^{-1};
//                  X += M_k Z_k; pool r_q -= U_{k+1} coef           (row a5; eqn.search-dir-comp
//                  P:436-448, eqn.approx-update, pool P:718-721)
//
// Panels are row-major n x p fp64.  A warp splits a panel row over LANES lanes of VEC
// (=2 -> 16-byte) chunks, RPW rows per warp-instruction, so one warp instruction touches
// RPW*p*8 contiguous bytes.  Reductions are deterministic: registers -> warp shuffles in a
// fixed tree -> CTA in fixed warp order -> per-CTA partials -> the last CTA sums them in
// CTA order (no floating-point atomics).
#pragma once
#include <cfloat>
#include <cstdint>
#include "common.cuh"

namespace bmr {

constexpr unsigned FULL = 0xffffffffu;
constexpr int NT = 256;  // threads of the panel kernels

// ------------------------------------------------------------------ small helpers

template <int VEC>
__device__ __forceinline__ void ldv(const double* p, double (&r)[VEC]) {
    if constexpr (VEC == 2) {
        double2 t = __ldg(reinterpret_cast<const double2*>(p));
        r[0] = t.x;
        r[1] = t.y;
    } else {
        r[0] = __ldg(p);
    }
}
// coherent load (data written earlier in the same kernel by this thread, or by a previous kernel)
template <int VEC>
__device__ __forceinline__ void ldc(const double* p, double (&r)[VEC]) {
    if constexpr (VEC == 2) {
        double2 t = *reinterpret_cast<const double2*>(p);
        r[0] = t.x;
        r[1] = t.y;
    } else {
        r[0] = *p;
    }
}
template <int VEC>
__device__ __forceinline__ void stv(double* p, const double (&r)[VEC]) {
    if constexpr (VEC == 2) {
        *reinterpret_cast<double2*>(p) = make_double2(r[0], r[1]);
    } else {
        *p = r[0];
    }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(FULL, v, o));
    return v;
}

// Last-CTA reduction of entry-major partials part[e*nb + b] (b = CTA) into two
// destinations: entries e < P*P go to outA[(e/P)*MAXP + e%P], the rest to
// outB[((e-P*P)/P)*MAXP + (e-P*P)%P].  Deterministic: every entry is summed by one
// warp over b in a fixed lane-strided order and a fixed shuffle tree.
__device__ __forceinline__ void last_cta_reduce(const double* part, int nb, int E, int P, double* outA,
                                                double* outB, unsigned* cnt) {
    __shared__ int s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(cnt, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int e = warp; e < E; e += nw) {
        double s = 0.0;
        for (int b = lane; b < nb; b += 32) s += __ldcg(part + (size_t)e * nb + b);
        s = warp_sum(s);
        if (lane == 0) {
            if (e < P * P)
                outA[(e / P) * MAXP + e % P] = s;
            else
                outB[((e - P * P) / P) * MAXP + (e - P * P) % P] = s;
        }
    }
    if (threadIdx.x == 0) *cnt = 0u;
}

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
    int nb;
};

template <int P, bool EPI>
__global__ void __launch_bounds__(NT) k1_spmm(K1Args a) {
    using C = PC<P>;
    constexpr int VEC = C::VEC, LANES = C::LANES, LP = C::LP, RPW = C::RPW, WARPS = NT / 32;
    constexpr int E = P * P + P;
    DevState* st = a.st;
    if constexpr (EPI) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            st->k4_pending = 0;
            st->slow_given = 0;
        }
        if (!st->run) return;
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
        has_prev = st->k > 1;
        for (int t = threadIdx.x; t < P * P; t += NT) sC[t] = st->Cprev[(t / P) * MAXP + t % P];
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
        double acc[VEC];
#pragma unroll
        for (int v = 0; v < VEC; ++v) acc[v] = 0.0;
        if (valid) {
            const int k0 = __ldg(a.rowptr + i), k1 = __ldg(a.rowptr + i + 1);
            for (int kk = k0; kk < k1; ++kk) {
                const int c = __ldg(a.col + kk);
                const double av = __ldg(a.val + kk);
                double x[VEC];
                ldv<VEC>(a.X + (long long)c * P + c0, x);
#pragma unroll
                for (int v = 0; v < VEC; ++v) acc[v] = fma(av, x[v], acc[v]);
            }
        }
        if constexpr (EPI) {
            double u[VEC], up[VEC];
#pragma unroll
            for (int v = 0; v < VEC; ++v) u[v] = up[v] = 0.0;
            if (valid) {
                ldv<VEC>(a.X + i * P + c0, u);
                if (has_prev) ldv<VEC>(a.Uprev + i * P + c0, up);
            }
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
        for (int e = threadIdx.x; e < E; e += NT) a.part[(size_t)e * a.nb + blockIdx.x] = sAcc[e];
        last_cta_reduce(a.part, a.nb, E, P, st->G, st->om2, &st->cnt1);
    }
}

// ------------------------------------------------------------------ K2: W' = W - U_k G_s, Grams

struct K2Args {
    double* W;
    const double* U;      // U_k
    const double* pool;   // n x pool_cap row-major
    long long n;
    DevState* st;
    double* part;
    int nb;
};

template <int P>
__global__ void __launch_bounds__(NT) k2_orth(K2Args a) {
    using C = PC<P>;
    constexpr int VEC = C::VEC, LANES = C::LANES, LP = C::LP, RPW = C::RPW, WARPS = NT / 32;
    DevState* st = a.st;
    if (!st->run) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int sub = lane % LP, rsub = lane / LP;
    const bool act = sub < LANES;
    const int c0 = sub * VEC;
    const int Q = st->q_live, qf = st->q_first, qc = st->pool_cap;
    const int E = P * P + Q * P;
    __shared__ double sG[P * P];
    __shared__ __align__(16) double sU[WARPS][RPW * P];
    __shared__ __align__(16) double sW[WARPS][RPW * P];
    __shared__ double sAcc[P * P + MAXQ * P];
    // G_s: lower triangle of G mirrored (the paper computes h_{i,j} for i >= j)
    for (int t = threadIdx.x; t < P * P; t += NT) {
        const int r = t / P, c = t % P;
        sG[t] = r >= c ? st->G[r * MAXP + c] : st->G[c * MAXP + r];
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
        double w[VEC], u[VEC];
#pragma unroll
        for (int v = 0; v < VEC; ++v) w[v] = u[v] = 0.0;
        if (valid) {
            ldc<VEC>(a.W + i * P + c0, w);
            ldv<VEC>(a.U + i * P + c0, u);
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
                    const double r = a.pool[i * qc + qf + q];
#pragma unroll
                    for (int v = 0; v < VEC; ++v) pq[q][v] = fma(r, w[v], pq[q][v]);
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
    for (int e = threadIdx.x; e < E; e += NT) a.part[(size_t)e * a.nb + blockIdx.x] = sAcc[e];
    last_cta_reduce(a.part, a.nb, E, P, st->Gram2, st->pdot, &st->cnt2);
}

// ------------------------------------------------------------------ K3: small banded QR (one warp)

template <int P>
__global__ void __launch_bounds__(32) k3_smallqr(DevState* st) {
    if (!st->run) return;
    constexpr int W2 = 2 * P + 1;
    constexpr int LD = P + 1;
    const int lane = threadIdx.x;
    extern __shared__ __align__(16) double dyn3[];
    double* sA = dyn3;                   // W'^T W'
    double* sC = sA + P * LD;            // C_k
    double* sT = sC + P * LD;            // tail of \bar Z
    double* sZ = sT + P * LD;            // Z_k
    double* sI = sZ + P * LD;            // C_k^{-1}, then R_kk^{-1}
    double* sH = sI + P * LD;            // the block's p Hessenberg columns, global-row frame (4p rows)
    double* sV = sH + 4 * P * LD;        // reflector ring: v (p+1) + tau per slot
    double* sHn = sV + W2 * (P + 2);
    const long long k = st->k;
    const long long j0 = st->j_done + 1;
    const long long maxit = st->maxit;
    const bool given = st->slow_given != 0;
    const double tau = st->tau, tol = st->tol;
    const int stop_after = st->stop_after;   // host column path: pool exhausted at column stop_after-1

    for (int t = lane; t < P * P; t += 32) {
        const int r = t / P, c = t % P;
        sA[r * LD + c] = st->Gram2[r * MAXP + c];
        sC[r * LD + c] = given ? st->Ck[r * MAXP + c] : 0.0;
        sT[r * LD + c] = st->T[r * MAXP + c];
        sZ[r * LD + c] = 0.0;
    }
    for (int t = lane; t < W2 * (P + 1); t += 32) {
        const int s = t / (P + 1), q = t % (P + 1);
        sV[s * (P + 2) + q] = st->rv[s * (MAXP + 1) + q];
    }
    for (int s = lane; s < W2; s += 32) sV[s * (P + 2) + P + 1] = st->rtau[s];
    __syncwarp();

    // ---- 1. new-block factor W' = U_{k+1} C_k by Cholesky of W'^T W'; its diagonal is
    //         h_{j+p,j}; breakdown if h_{j+p,j} <= tau ||A u_j||
    if (!given) {
        bool bad = false;
        for (int m = 0; m < P; ++m) {
            double d = sA[m * LD + m];
            for (int i = 0; i < m; ++i) d -= sC[i * LD + m] * sC[i * LD + m];
            const double om2 = st->om2[m];
            // cancellation guard: the pivot lost > 4 decimal digits of ||w'_m||^2 -> column path
            if (!(d > tau * tau * om2) || !(d >= 1e-4 * sA[m * LD + m])) {
                bad = true;
                break;
            }
            const double cmm = sqrt(d);
            if (lane == m) sC[m * LD + m] = cmm;
            if (lane > m && lane < P) {
                double s = sA[m * LD + lane];
                for (int i = 0; i < m; ++i) s -= sC[i * LD + m] * sC[i * LD + lane];
                sC[m * LD + lane] = s / cmm;
            }
            __syncwarp();
        }
        if (bad) {
            if (lane == 0) {
                st->need_slow = 1;
                st->run = 0;
                st->hflags->need_slow = 1;
                st->hflags->run = 0;
                __threadfence_system();
            }
            return;
        }
        // C_k^{-1} (column lane), and coef = C_k^{-T} (W'^T r_q) = U_{k+1}^T r_q
        if (lane < P) {
            const int l = lane;
            // back substitution for column l of the inverse, written into sI temporarily
            for (int r = P - 1; r >= 0; --r) {
                double s = (r == l) ? 1.0 : 0.0;
                for (int c = r + 1; c < P; ++c) s -= sC[r * LD + c] * sI[c * LD + l];
                sI[r * LD + l] = (r <= l) ? s / sC[r * LD + r] : 0.0;
            }
        }
        __syncwarp();
        for (int t = lane; t < P * P; t += 32) {
            const int r = t / P, c = t % P;
            st->Cinv[r * MAXP + c] = sI[r * LD + c];
            st->Ck[r * MAXP + c] = sC[r * LD + c];
        }
        const int Q = st->q_live;
        if (lane < Q) {
            double y[P];
#pragma unroll
            for (int m = 0; m < P; ++m) {
                double s = st->pdot[lane * MAXP + m];
#pragma unroll
                for (int i = 0; i < m; ++i) s -= sC[i * LD + m] * y[i];
                y[m] = s / sC[m * LD + m];
                st->coef[m * MAXQ + lane] = y[m];
            }
        }
        __syncwarp();
    }

    // ---- 2. the p new columns of \bar H in the frame of global rows (k-3)p+1 .. (k+1)p
    //         (Appendix B of SURVEY / DESIGN.md "Assembly map"; symmetric reuse P:923-945)
    if (lane < P) {
        const int m = lane;
        for (int r = 0; r < 4 * P; ++r) sH[r * LD + m] = 0.0;
        if (k > 1)
            for (int mp = m; mp < P; ++mp) sH[(P + mp) * LD + m] = st->Cprev[m * MAXP + mp];
        for (int mp = 0; mp < P; ++mp) {
            const double gv = mp >= m ? st->G[mp * MAXP + m] : st->G[m * MAXP + mp];
            sH[(2 * P + mp) * LD + m] = gv;
        }
        for (int mp = 0; mp <= m; ++mp) sH[(3 * P + mp) * LD + m] = sC[mp * LD + m];
        double hn = 0.0;
        for (int r = 0; r < 4 * P; ++r) hn += sH[r * LD + m] * sH[r * LD + m];
        sHn[m] = sqrt(hn);
        // phase A: reflectors i = (k-3)p+1 .. (k-1)p (previous two blocks), increasing i;
        // frame offset o = i - ((k-3)p+1) touches rows o .. o+p
        const long long base = (k - 3) * P + 1;
        for (int o = 0; o < 2 * P; ++o) {
            const long long i = base + o;
            if (i < 1) continue;
            const double* v = sV + (int)(i % W2) * (P + 2);
            const double t = v[P + 1];
            double s = 0.0;
            for (int q = 0; q <= P; ++q) s += v[q] * sH[(o + q) * LD + m];
            s *= t;
            for (int q = 0; q <= P; ++q) sH[(o + q) * LD + m] -= s * v[q];
        }
    }
    __syncwarp();

    // ---- 3. phase B: column by column, generate reflector j, apply it to the later columns
    //         and to [T; 0] (row 1 -> z_j^T), residuals, stop test (Alg. 2)
    int m_last = -1;
    int stop = 0;  // 1 converged, 2 maxit, 3 singular R, 4 pool exhausted
    for (int m = 0; m < P; ++m) {
        const long long j = j0 + m;
        if (j > maxit) {
            stop = 2;
            break;
        }
        const int o = 2 * P + m;
        // Householder vector of rows o..o+P (LAPACK dlarfg convention)
        const double alpha = sH[o * LD + m];
        double x2 = 0.0;
        for (int q = 1 + lane; q <= P; q += 32) x2 += sH[(o + q) * LD + m] * sH[(o + q) * LD + m];
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
        double* vj = sV + (int)(j % W2) * (P + 2);
        __syncwarp();
        for (int q = lane; q <= P; q += 32) vj[q] = (q == 0) ? 1.0 : sH[(o + q) * LD + m] * scl;
        if (lane == 0) vj[P + 1] = tj;
        __syncwarp();
        if (lane == 0) {
            sH[o * LD + m] = beta;
            for (int q = 1; q <= P; ++q) sH[(o + q) * LD + m] = 0.0;
        }
        if (fabs(beta) <= DBL_EPSILON * sHn[m]) {
            stop = 3;
            break;
        }
        __syncwarp();
        if (lane < P) {
            const int c = lane;
            if (c > m) {   // later columns of this block
                double s = 0.0;
                for (int q = 0; q <= P; ++q) s += vj[q] * sH[(o + q) * LD + c];
                s *= tj;
                for (int q = 0; q <= P; ++q) sH[(o + q) * LD + c] -= s * vj[q];
            }
            // [T; 0] -> reflector j -> z_j^T = row 0, new tail = rows 1..p
            double s = 0.0;
            for (int q = 0; q < P; ++q) s += vj[q] * sT[q * LD + c];
            s *= tj;
            double z = sT[c] - s;   // q = 0
            for (int q = 0; q < P - 1; ++q) sT[q * LD + c] = sT[(q + 1) * LD + c] - s * vj[q + 1];
            sT[(P - 1) * LD + c] = -s * vj[P];
            sZ[m * LD + c] = z;
        }
        __syncwarp();
        double rel = 0.0;
        if (lane < P) {
            double s = 0.0;
            for (int q = 0; q < P; ++q) s += sT[q * LD + lane] * sT[q * LD + lane];
            const double b = st->beta[lane];
            rel = b > 0.0 ? sqrt(s) / b : 0.0;
            st->res[lane] = rel;
            if (st->hist && j < st->hist_cap) st->hist[j * P + lane] = rel;
        }
        const double mx = warp_max(rel);
        m_last = m;
        if (mx < tol) {
            stop = 1;
            break;
        }
        if (stop_after > 0 && m == stop_after - 1) {
            stop = 4;
            break;
        }
    }
    __syncwarp();

    // ---- 4. direction-update matrices: Ainv = R_kk^{-1}; B1 = R_{k-1,k} Ainv; B2 = R_{k-2,k} Ainv
    //         (eqn.search-dir-comp), columns past m_last masked
    if (lane < P) {
        const int l = lane;
        for (int r = P - 1; r >= 0; --r) {
            double s = (r == l) ? 1.0 : 0.0;
            if (l <= m_last && r <= l) {
                for (int c = r + 1; c <= l; ++c) s -= sH[(2 * P + r) * LD + c] * sI[c * LD + l];
                sI[r * LD + l] = s / sH[(2 * P + r) * LD + r];
            } else {
                sI[r * LD + l] = s;   // identity column (or zero above/below)
            }
        }
    }
    __syncwarp();
    if (lane < P) {
        const int l = lane;
        for (int a = 0; a < P; ++a) {
            double s1 = 0.0, s2 = 0.0;
            for (int b = 0; b <= m_last; ++b) {
                s1 += sH[(P + a) * LD + b] * sI[b * LD + l];
                if (a >= b) s2 += sH[a * LD + b] * sI[b * LD + l];
            }
            st->B1[a * MAXP + l] = s1;
            st->B2[a * MAXP + l] = s2;
            st->Ainv[a * MAXP + l] = sI[a * LD + l];
            st->Z[a * MAXP + l] = sZ[a * LD + l];
            st->T[a * MAXP + l] = sT[a * LD + l];
            st->Cprev[a * MAXP + l] = sC[a * LD + l];
        }
    }
    for (int t = lane; t < W2 * (P + 1); t += 32) {
        const int s = t / (P + 1), q = t % (P + 1);
        st->rv[s * (MAXP + 1) + q] = sV[s * (P + 2) + q];
    }
    for (int s = lane; s < W2; s += 32) st->rtau[s] = sV[s * (P + 2) + P + 1];
    __syncwarp();
    if (lane == 0) {
        const long long jd = st->j_done + (m_last + 1);
        st->j_done = jd;
        if (m_last >= 0) st->k = k + 1;
        int status = 1;
        bool end = false;
        if (stop == 1) { status = 0; end = true; }
        else if (stop == 2) { status = 1; end = true; }
        else if (stop == 3) { status = -6; end = true; }
        else if (stop == 4) { status = -5; end = true; }
        else if (jd >= maxit) { status = 1; end = true; }
        st->status = status;
        st->need_slow = 0;
        if (end) {
            st->run = 0;
            st->k4_pending = m_last >= 0 ? 1 : 0;
        }
        st->hflags->status = status;
        st->hflags->j_done = jd;
        st->hflags->k = st->k;
        st->hflags->need_slow = 0;
        st->hflags->run = end ? 0 : 1;
        __threadfence_system();
    }
}

// ------------------------------------------------------------------ K4: basis, directions, X

struct K4Args {
    const double* W;      // W' (or materialised U_{k+1} when slow_given)
    const double* U;      // U_k
    double* Unext;        // U_{k+1} (the slot of U_{k-1})
    double* M2;           // M_{k-2} in, M_k out
    const double* M1;     // M_{k-1}
    double* X;
    double* pool;
    long long n;
    DevState* st;
};

template <int P>
__global__ void __launch_bounds__(NT) k4_update(K4Args a) {
    using C = PC<P>;
    constexpr int VEC = C::VEC, LANES = C::LANES, LP = C::LP, RPW = C::RPW, WARPS = NT / 32;
    DevState* st = a.st;
    if (!(st->run || st->k4_pending)) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int sub = lane % LP, rsub = lane / LP;
    const bool act = sub < LANES;
    const int c0 = sub * VEC;
    const bool given = st->slow_given != 0;
    const int Q = given ? 0 : st->q_live, qf = st->q_first, qc = st->pool_cap;
    extern __shared__ __align__(16) double dyn[];
    double* sCi = dyn;                 // C_k^{-1}
    double* sAi = sCi + P * P;         // R_kk^{-1}
    double* sB1 = sAi + P * P;
    double* sB2 = sB1 + P * P;
    double* sZ = sB2 + P * P;
    double* sCo = sZ + P * P;          // coef (P x MAXQ)
    double* sRow = sCo + P * MAXQ;     // per-warp staging: 6 rows-sets of RPW*P
    for (int t = threadIdx.x; t < P * P; t += NT) {
        const int r = t / P, c = t % P;
        sCi[t] = st->Cinv[r * MAXP + c];
        sAi[t] = st->Ainv[r * MAXP + c];
        sB1[t] = st->B1[r * MAXP + c];
        sB2[t] = st->B2[r * MAXP + c];
        sZ[t] = st->Z[r * MAXP + c];
    }
    for (int t = threadIdx.x; t < P * MAXQ; t += NT) sCo[t] = st->coef[(t / MAXQ) * MAXQ + t % MAXQ];
    __syncthreads();
    double* sW = sRow + warp * 6 * RPW * P;
    double* sU = sW + RPW * P;
    double* sM2 = sU + RPW * P;
    double* sM1 = sM2 + RPW * P;
    double* sUn = sM1 + RPW * P;
    double* sMk = sUn + RPW * P;
    const long long stride = (long long)gridDim.x * WARPS * RPW;
    for (long long base = ((long long)blockIdx.x * WARPS + warp) * RPW; base < a.n; base += stride) {
        const long long i = base + rsub;
        const bool valid = act && i < a.n;
        double w[VEC], u[VEC], m2[VEC], m1[VEC];
#pragma unroll
        for (int v = 0; v < VEC; ++v) w[v] = u[v] = m2[v] = m1[v] = 0.0;
        if (valid) {
            ldc<VEC>(a.W + i * P + c0, w);
            ldv<VEC>(a.U + i * P + c0, u);
            ldc<VEC>(a.M2 + i * P + c0, m2);
            ldc<VEC>(a.M1 + i * P + c0, m1);
        }
        const int ro = rsub * P;
        if (act) {
#pragma unroll
            for (int v = 0; v < VEC; ++v) {
                sW[ro + c0 + v] = w[v];
                sU[ro + c0 + v] = u[v];
                sM2[ro + c0 + v] = m2[v];
                sM1[ro + c0 + v] = m1[v];
            }
        }
        __syncwarp();
        double un[VEC], mk[VEC];
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
            un[v] = given ? w[v] : 0.0;
            mk[v] = 0.0;
        }
        if (valid) {
#pragma unroll
            for (int b = 0; b < P; ++b) {
                const double xw = sW[ro + b], xu = sU[ro + b], x2 = sM2[ro + b], x1 = sM1[ro + b];
#pragma unroll
                for (int v = 0; v < VEC; ++v) {
                    const int m = c0 + v;
                    if (!given) un[v] = fma(xw, sCi[b * P + m], un[v]);
                    mk[v] = fma(xu, sAi[b * P + m], mk[v]);
                    mk[v] = fma(-x2, sB2[b * P + m], mk[v]);
                    mk[v] = fma(-x1, sB1[b * P + m], mk[v]);
                }
            }
            stv<VEC>(a.Unext + i * P + c0, un);
            stv<VEC>(a.M2 + i * P + c0, mk);
        }
        if (act) {
#pragma unroll
            for (int v = 0; v < VEC; ++v) {
                sUn[ro + c0 + v] = un[v];
                sMk[ro + c0 + v] = mk[v];
            }
        }
        __syncwarp();
        if (valid) {
            double x[VEC];
            ldc<VEC>(a.X + i * P + c0, x);
#pragma unroll
            for (int b = 0; b < P; ++b) {
                const double xm = sMk[ro + b];
#pragma unroll
                for (int v = 0; v < VEC; ++v) x[v] = fma(xm, sZ[b * P + c0 + v], x[v]);
            }
            stv<VEC>(a.X + i * P + c0, x);
            for (int q = sub; q < Q; q += LANES) {
                double r = a.pool[i * qc + qf + q];
                for (int b = 0; b < P; ++b) r = fma(-sUn[ro + b], sCo[b * MAXQ + q], r);
                a.pool[i * qc + qf + q] = r;
            }
        }
        __syncwarp();
    }
}

// ------------------------------------------------------------------ generic column kernels
// (start block, column-by-column path, norms).  Rare or once per solve.

constexpr int MAXREF = 80;
struct VecRef {
    const double* p;
    long long stride;
};

// out[k] = sum_i v_k[i] * t[i], k < K (deterministic)
struct DotArgs {
    VecRef v[MAXREF];
    int K;
    const double* t;
    long long ts;
    long long n;
    double* part;
    int nb;
    double* out;
    unsigned* cnt;
};

__global__ void __launch_bounds__(256) k_dots(DotArgs a) {
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    __shared__ double sred[8][33];
    for (int k0 = 0; k0 < a.K; k0 += 32) {
        const int k = k0 + tx;
        double s = 0.0;
        if (k < a.K) {
            const double* vp = a.v[k].p;
            const long long vs = a.v[k].stride;
            for (long long i = (long long)blockIdx.x * 8 + ty; i < a.n; i += (long long)gridDim.x * 8)
                s = fma(vp[i * vs], a.t[i * a.ts], s);
        }
        sred[ty][tx] = s;
        __syncthreads();
        if (ty == 0 && k < a.K) {
            double r = 0.0;
            for (int y = 0; y < 8; ++y) r += sred[y][tx];
            a.part[(size_t)k * a.nb + blockIdx.x] = r;
        }
        __syncthreads();
    }
    __shared__ int s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(a.cnt, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    for (int e = ty; e < a.K; e += 8) {
        double s = 0.0;
        for (int b = tx; b < a.nb; b += 32) s += __ldcg(a.part + (size_t)e * a.nb + b);
        s = warp_sum(s);
        if (tx == 0) a.out[e] = s;
    }
    if (threadIdx.x == 0) *a.cnt = 0u;
}

// t[i] = scale * (t[i] - sum_k c_k v_k[i]); c_k from cdev (times csign) if non-null else cval
struct AxpyArgs {
    VecRef v[MAXREF];
    double cval[MAXREF];
    const double* cdev;
    double csign;
    int K;
    double* t;
    long long ts;
    long long n;
    const double* scale_dev;   // if non-null: scale = 1/sqrt(*scale_dev) (normalisation)
    double scale;
};

__global__ void __launch_bounds__(256) k_axpy(AxpyArgs a) {
    __shared__ double sc[MAXREF];
    for (int k = threadIdx.x; k < a.K; k += blockDim.x) sc[k] = a.cdev ? a.csign * a.cdev[k] : a.cval[k];
    __syncthreads();
    const double scale = a.scale_dev ? 1.0 / sqrt(*a.scale_dev) : a.scale;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += (long long)gridDim.x * blockDim.x) {
        double t = a.t[i * a.ts];
        for (int k = 0; k < a.K; ++k) t = fma(-sc[k], a.v[k].p[i * a.v[k].stride], t);
        a.t[i * a.ts] = scale == 0.0 ? 0.0 : t * scale;
    }
}

__device__ __forceinline__ unsigned long long splitmix64(unsigned long long x) {
    unsigned long long z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// random replacement vector (reading C17): integer hash, one exact scaling -> bitwise reproducible
__global__ void k_rand(double* out, long long stride, long long n, long long row_begin, unsigned long long seed,
                       unsigned long long stream, unsigned long long event) {
    const unsigned long long key = splitmix64(seed ^ (stream << 56) ^ (event << 32));
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const unsigned long long x = splitmix64(key ^ (unsigned long long)(row_begin + i));
        out[i * stride] = 2.0 * ((double)(x >> 11) * 0x1.0p-53) - 1.0;
    }
}

// out[c] = sum_i (X[i,c] - Y[i,c])^2 for a row-major n x P panel pair (Y may be null)
__global__ void __launch_bounds__(256) k_colsq(const double* X, const double* Y, long long n, int P, double* part,
                                               int nb, double* out, unsigned* cnt) {
    __shared__ double sred[256];
    const int R = 256 / P;
    const int c = threadIdx.x % P, r0 = threadIdx.x / P;
    double s = 0.0;
    if (r0 < R) {
        for (long long i = (long long)blockIdx.x * R + r0; i < n; i += (long long)gridDim.x * R) {
            const double d = X[i * P + c] - (Y ? Y[i * P + c] : 0.0);
            s = fma(d, d, s);
        }
    }
    sred[threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.x < P) {
        double r = 0.0;
        for (int y = 0; y < R; ++y) r += sred[y * P + threadIdx.x];
        part[(size_t)threadIdx.x * nb + blockIdx.x] = r;
    }
    __shared__ int s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(cnt, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int e = warp; e < P; e += 8) {
        double t = 0.0;
        for (int b = lane; b < nb; b += 32) t += __ldcg(part + (size_t)e * nb + b);
        t = warp_sum(t);
        if (lane == 0) out[e] = t;
    }
    if (threadIdx.x == 0) *cnt = 0u;
}

// Y = B - Y (row-major panels, same shape)
__global__ void k_sub_from(const double* B, double* Y, long long total) {
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x)
        Y[e] = B[e] - Y[e];
}

}  // namespace bmr
