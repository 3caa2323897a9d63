// row_kernels.cuh -- thread-per-row panel kernels for block sizes p <= 8 (a panel row is at
// most 64 B): one thread owns one row of a 128-row CTA tile, the tiles stream through shared
// memory by TMA bulk copies (cp.async.bulk, one elected thread, mbarrier completion), and the
// p x p row-local products run on the fp64 CUDA cores from registers.  Compared with the
// warp-tiled DMMA kernels this issues ~5x fewer instructions per row and keeps the loads
// in flight without registers (the kernels are latency/issue bound, not flop bound).
#pragma once
#include "common.cuh"
#include "step_kernels.cuh"

namespace bmr {

constexpr int RT = 128;   // rows per CTA tile = threads per CTA
constexpr int RNS = 2;    // TMA pipeline stages (2 stages x 3 CTAs/SM measured best: 117k vs 116k it/s with 4 x 2)

// bytes of `rows` panel rows of p doubles, rounded up to the 16-byte granule of cp.async.bulk
// (workspace panels carry >= 16 B of slack past row n-1 for the odd-p round-up)
__host__ __device__ __forceinline__ unsigned bulk_bytes(long long rows, int p) {
    return (unsigned)((rows * p * 8 + 15) & ~15ll);
}

// p = 8: a thread's row is 64 B, so the 32 rows a warp reads in one instruction fall on two
// 16-byte bank groups (16-way conflict).  The chunk order is rotated by (lane >> 1) & 3: in each
// instruction lanes 0..7 touch 8 distinct bank groups (4 wavefronts, the minimum for 16-byte
// accesses), and the chunks are put back in place with selects (no dynamic register indexing).
__device__ __forceinline__ double2 sel4(const double2 (&t)[4], int k) {
    double2 x = t[3];
    x = k == 2 ? t[2] : x;
    x = k == 1 ? t[1] : x;
    x = k == 0 ? t[0] : x;
    return x;
}
template <int P>
__device__ __forceinline__ void row_ld(const double* s, double (&r)[P]) {
    if constexpr (P == 8) {
        const int rot = (threadIdx.x >> 1) & 3;
        double2 t[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) t[c] = *reinterpret_cast<const double2*>(s + 2 * ((c + rot) & 3));
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const double2 x = sel4(t, (j - rot) & 3);
            r[2 * j] = x.x;
            r[2 * j + 1] = x.y;
        }
    } else if constexpr (P % 2 == 0) {
#pragma unroll
        for (int c = 0; c < P / 2; ++c) {
            const double2 v = *reinterpret_cast<const double2*>(s + 2 * c);
            r[2 * c] = v.x;
            r[2 * c + 1] = v.y;
        }
    } else {
#pragma unroll
        for (int c = 0; c < P; ++c) r[c] = s[c];
    }
}
template <int P>
__device__ __forceinline__ void row_st(double* s, const double (&r)[P]) {
    if constexpr (P == 8) {   // rotated chunk order (see row_ld)
        const int rot = (threadIdx.x >> 1) & 3;
        double2 t[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) t[j] = make_double2(r[2 * j], r[2 * j + 1]);
#pragma unroll
        for (int c = 0; c < 4; ++c) *reinterpret_cast<double2*>(s + 2 * ((c + rot) & 3)) = sel4(t, (c + rot) & 3);
    } else if constexpr (P % 2 == 0) {
#pragma unroll
        for (int c = 0; c < P / 2; ++c) *reinterpret_cast<double2*>(s + 2 * c) = make_double2(r[2 * c], r[2 * c + 1]);
    } else {
#pragma unroll
        for (int c = 0; c < P; ++c) s[c] = r[c];
    }
}

// ------------------------------------------------------------------ K2 (rows a2/a3, block k)
//
// pool r_q -= U_k coef_{k-1}(:, q); W' = W - U_k G_s = W - V_k (Tr_k G_s)
// (Alg. 1 P:288-291 in block form, G_s = lower triangle of G mirrored);
// partial W'^T W' and r_q^T W' -> cluster partials (the Cholesky W' = U_{k+1} C_k is taken by
// the consumers, K1(k+1) and K3b(k)).
constexpr int K2R_QMAX = 2;   // pool columns handled in registers (larger pools: DMMA / warp kernels)

template <int P>
struct K2RSmem {
    static constexpr int TILE = RT * P + 2;             // doubles of one panel tile (+ odd-p round-up)
    static constexpr int TQ = RT * K2R_QMAX + 2;        // pool tile (row stride pool_cap <= K2R_QMAX)
    static constexpr int STAGE = 2 * TILE + TQ;
    static constexpr int E = P * P + K2R_QMAX * P;
    static constexpr int red = (RT / 32) * 64;
    static constexpr int tail = 4 * P * P + P * MAXQ + prologue_scratch<P>();
    static constexpr size_t bytes =
        sizeof(double) * (RNS * STAGE + P * P + P * MAXQ + (red > tail ? red : tail) + E) + 8 * RNS + 16;
};

template <int P>
__global__ void __launch_bounds__(RT, 3) k2_row(K2Args a) {
    using S = K2RSmem<P>;
    constexpr int NG = P * (P + 1) / 2;
    DevState* st = a.st;
    unsigned long long* tr = trace_begin(st, TR_K2);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int Q = st->q_live, qf = st->q_first, qc = st->pool_cap;
    const int E = P * P + Q * P;
    extern __shared__ __align__(128) double dynr2[];
    double* stage0 = dynr2;                         // RNS x {W tile, V tile, pool tile}
    double* sE = stage0 + RNS * S::STAGE;           // -(Tr_k G_s)
    double* sF = sE + P * P;                        // -(Tr_k coef_{k-1}), P x MAXQ
    double* sTail = sF + P * MAXQ;                  // prologue scratch, then the per-warp partials
    double* sAcc = sTail + (S::red > S::tail ? S::red : S::tail);
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(sAcc + S::E);
    const long long ntiles = (a.n + RT - 1) / RT;
    const long long my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const bool pool_on = Q > 0;
    auto issue = [&](long long it) {   // thread 0: TMA loads of local tile `it` into its stage
        if (it >= my_tiles) return;
        const int s = (int)(it % RNS);
        const long long row0 = (blockIdx.x + it * gridDim.x) * RT;
        const long long rows = a.n - row0 < RT ? a.n - row0 : RT;
        double* sl = stage0 + s * S::STAGE;
        const unsigned bp = bulk_bytes(rows, P), bq = pool_on ? bulk_bytes(rows, qc) : 0u;
        mbar_expect_tx(&bar[s], 2 * bp + bq);
        bulk_g2s(sl, a.W + row0 * P, bp, &bar[s]);
        bulk_g2s(sl + S::TILE, a.V + row0 * P, bp, &bar[s]);
        if (pool_on) bulk_g2s(sl + 2 * S::TILE, a.pool + row0 * qc, bq, &bar[s]);
    };
    if (tid == 0) {
        for (int s = 0; s < RNS; ++s) mbar_init(&bar[s], 1);
        mbar_fence_init();
    }
    __syncthreads();
    if (tid == 0)
        for (int s = 0; s < RNS - 1; ++s) issue(s);   // W (K1 completed before reduce1) streams in
    trace_pt(tr, 1);
    pdl_wait();   // red1 (reduce1) is ready
    // stopped main branch (read after the wait: uniform over the launch, see publish_breakdown);
    // the prefetched stages land before the CTA exits
    if (!st->run_main) {
        for (int s = 0; s < RNS - 1; ++s)
            if (s < my_tiles) mbar_wait(&bar[s], 0u);
        k2_stopped(st);
        return;
    }
    trace_pt(tr, 2);
    {
        // G = Tr_k^T (V_k^T W) from K1's partials; E = -(Tr_k G_s), F = -(Tr_k coef_{k-1})
        double* sGs = sTail;
        double* sTk = sTail + P * P;
        double* sG = sTail + 3 * P * P;
        double* sCo = sTail + 4 * P * P;
        double* sScr = sCo + P * MAXQ;
        const double* Co = st->coef[a.par ^ 1];
        for (int t = tid; t < P * MAXQ; t += RT) sCo[t] = Co[t];
        k2_prologue<P>(st, a.par, a.sk, sG, sTk, sScr);
        for (int t = tid; t < P * P; t += RT) {
            const int r = t / P, c = t % P;
            sGs[t] = r >= c ? sG[r * P + c] : sG[c * P + r];
        }
        __syncthreads();
        for (int t = tid; t < P * P; t += RT) {
            const int r = t / P, c = t % P;
            double s = 0.0;
            for (int i = 0; i < P; ++i) s = fma(sTk[r * P + i], sGs[i * P + c], s);
            sE[t] = -s;
        }
        for (int t = tid; t < P * MAXQ; t += RT) {
            const int r = t / MAXQ, q = t % MAXQ;
            double s = 0.0;
            if (q < Q)
                for (int i = 0; i < P; ++i) s = fma(sTk[r * P + i], sCo[i * MAXQ + q], s);
            sF[t] = -s;
        }
        __syncthreads();
    }
    trace_pt(tr, 3);
    double g[NG], pd[K2R_QMAX][P];
#pragma unroll
    for (int e = 0; e < NG; ++e) g[e] = 0.0;
#pragma unroll
    for (int q = 0; q < K2R_QMAX; ++q)
#pragma unroll
        for (int m = 0; m < P; ++m) pd[q][m] = 0.0;
    for (long long it = 0; it < my_tiles; ++it) {
        const int s = (int)(it % RNS);
        const long long row0 = (blockIdx.x + it * gridDim.x) * RT;
        const long long rows = a.n - row0 < RT ? a.n - row0 : RT;
        double* sl = stage0 + s * S::STAGE;
        if (tid == 0) issue(it + RNS - 1);   // its stage was released by the barrier ending it-1
        mbar_wait(&bar[s], (unsigned)((it / RNS) & 1));
        if (tid < rows) {
            double w[P], v[P];
            row_ld<P>(sl + tid * P, w);
            row_ld<P>(sl + S::TILE + tid * P, v);
            double r[K2R_QMAX];
#pragma unroll
            for (int q = 0; q < K2R_QMAX; ++q) {
                r[q] = 0.0;
                if (q < Q) {
                    r[q] = sl[2 * S::TILE + tid * qc + qf + q];
#pragma unroll
                    for (int b = 0; b < P; ++b) r[q] = fma(v[b], sF[b * MAXQ + q], r[q]);
                    a.pool[(row0 + tid) * qc + qf + q] = r[q];
                }
            }
#pragma unroll
            for (int b = 0; b < P; ++b) {
                const double x = v[b];
#pragma unroll
                for (int m = 0; m < P; ++m) w[m] = fma(x, sE[b * P + m], w[m]);
            }
            row_st<P>(sl + tid * P, w);
            int e = 0;
#pragma unroll
            for (int i = 0; i < P; ++i)
#pragma unroll
                for (int j = 0; j <= i; ++j, ++e) g[e] = fma(w[i], w[j], g[e]);
#pragma unroll
            for (int q = 0; q < K2R_QMAX; ++q)
                if (q < Q) {
#pragma unroll
                    for (int m = 0; m < P; ++m) pd[q][m] = fma(r[q], w[m], pd[q][m]);
                }
        }
        __syncwarp();
        // W' rows of this warp -> HBM, coalesced (lane-contiguous 16-byte chunks)
        {
            const long long wrow = 32ll * warp;
            const long long nrow = rows - wrow < 32 ? rows - wrow : 32;
            if (nrow > 0) {
                const double* src = sl + wrow * P;
                double* dst = a.W + (row0 + wrow) * P;
                if constexpr (P % 2 == 0) {
                    const int nch = (int)(nrow * P / 2);
                    for (int c = lane; c < nch; c += 32)
                        reinterpret_cast<double2*>(dst)[c] = reinterpret_cast<const double2*>(src)[c];
                } else {
                    const int nd = (int)(nrow * P);
                    for (int c = lane; c < nd; c += 32) dst[c] = src[c];
                }
            }
        }
        __syncthreads();   // stage s is free for the TMA load of tile it+RNS
    }
    trace_pt(tr, 4);
    pdl_trigger();   // the dependent (reduce2) launches while this grid reduces its partials
    // partials: butterfly reduce-scatter per warp -> per-warp slot -> fixed-order sum over warps
    constexpr int NE = 64;
    static_assert(NG + K2R_QMAX * P <= NE, "partials exceed the reduce-scatter width");
    double* red = sTail;
    __syncthreads();   // the prologue scratch in sTail is dead
    {
        double v[NE];
#pragma unroll
        for (int e = 0; e < NE; ++e) v[e] = 0.0;
#pragma unroll
        for (int e = 0; e < NG; ++e) v[e] = g[e];
#pragma unroll
        for (int q = 0; q < K2R_QMAX; ++q)
#pragma unroll
            for (int m = 0; m < P; ++m) v[NG + q * P + m] = pd[q][m];
        warp_reduce_scatter64(v);
        red[warp * NE + 2 * lane] = v[0];
        red[warp * NE + 2 * lane + 1] = v[1];
    }
    __syncthreads();
    for (int t = tid; t < E; t += RT) {
        int src;
        if (t < P * P) {
            const int i = t / P, j = t % P;
            const int hi = i > j ? i : j, lo = i > j ? j : i;
            src = hi * (hi + 1) / 2 + lo;
        } else {
            src = NG + (t - P * P);
        }
        double s = red[src];
        for (int w = 1; w < RT / 32; ++w) s += red[w * NE + src];
        sAcc[t] = s;
    }
    cluster_partials(sAcc, E, st->part2[a.par]);   // reduce2, then K1(k+1) and K3b(k) factor W'
    trace_pt(tr, 5);
}

}  // namespace bmr
