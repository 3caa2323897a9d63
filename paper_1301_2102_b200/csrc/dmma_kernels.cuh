// dmma_kernels.cuh -- panel kernels whose row-local dense products run on the fp64 tensor
// cores (mma.sync m8n8k4 f64, "DMMA"), for block sizes p that are multiples of 8.
//
// A warp owns a tile of TR panel rows.  Tiles are staged in shared memory by cp.async
// (NSTAGE-deep, one commit group per tile) with row stride RS = p + 4 doubles, which makes
// every fragment load bank-conflict free.  Fragment layouts (PTX mma.m8n8k4 .f64, as in
// CuTe's SM80_8x8x4_F64F64F64F64_TN): A(8x4) lane l holds A[l/4][l%4]; B(4x8) B[l%4][l/4];
// C(8x8) C[l/4][2(l%4)+v], v = 0,1.  Constant p x p factors are kept in shared memory in
// fragment order (32 consecutive doubles per 4x8 block) so B-fragment loads are conflict free.
#pragma once
#include "common.cuh"
#include "step_kernels.cuh"

namespace bmr {

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

template <int P>
struct DM {
    static constexpr int RS = P + 4;                 // smem row stride (doubles)
    static constexpr int TR = P <= 8 ? 16 : 8;       // rows per warp tile
    static constexpr int KC = P / 4, NC = P / 8;     // k- and n-chunks of a p x p factor
    static constexpr int FR = KC * NC * 32;          // doubles of one factor in fragment order
    static constexpr int TILE = TR * RS;             // doubles of one staged panel tile
    static constexpr int CPR = P / 2;                // 16-byte chunks per row
};

// store p x p factor M (leading dimension ld, optional sign) into fragment order
template <int P>
__device__ __forceinline__ void to_frag(const double* M, int ld, double sign, double* F) {
    using D = DM<P>;
    for (int t = threadIdx.x; t < D::FR; t += blockDim.x) {
        const int blk = t / 32, l = t % 32, kc = blk / D::NC, nc = blk % D::NC;
        F[t] = sign * M[(kc * 4 + l % 4) * ld + nc * 8 + l / 4];
    }
}

// cp.async one TR x P tile of a row-major panel (rows base.., zero-fill past n) into smem
template <int P>
__device__ __forceinline__ void stage_tile(double* dst, const double* src, long long base, long long n, int lane) {
    using D = DM<P>;
    for (int c = lane; c < D::TR * D::CPR; c += 32) {
        const int r = c / D::CPR, q = c % D::CPR;
        const long long i = base + r;
        const bool ok = i < n;
        cp_async16(dst + r * D::RS + 2 * q, src + (ok ? i : 0) * P + 2 * q, ok);
    }
}

// cp.async one TRU x P tile (rows base.., zero-fill past n) into smem rows of stride P + 4
template <int P, int TRU = 16>
__device__ __forceinline__ void stage_rows(double* dst, const double* src, long long base, long long n, int lane) {
    constexpr int RS = P + 4, CPR = P / 2;
    for (int c = lane; c < TRU * CPR; c += 32) {
        const int r = c / CPR, q = c % CPR;
        const long long i = base + r;
        const bool ok = i < n;
        cp_async16(dst + r * RS + 2 * q, src + (ok ? i : 0) * P + 2 * q, ok);
    }
}

// ------------------------------------------------------------------ M/X update on DMMA (row a5)
//
// M_k = V_k (Tr_k R_kk^{-1}) - M_{k-2} R_{k-2,k}R_kk^{-1} - M_{k-1} R_{k-1,k}R_kk^{-1}
// (eqn.search-dir-comp); X += M_k Z_k (eqn.approx-update).
// Warp w of the CTA streams tiles t0 + w + i*ts (< tend) through an NS-deep cp.async ring.
// Used by the standalone K4b (grid-strided) and, fused, by K1 two blocks later (CTA slab).
template <int P, int WARPS, int NS>
struct UpdSmem {
    static constexpr int doubles = 4 * DM<P>::FR + WARPS * NS * 4 * DM<P>::TILE + 3 * P * P;
};

// The update in three pieces (shared by the pipelined dmma_update below and the interleaved K1):
// upd_setup loads the factors (all threads of the calling group, then a barrier by the caller),
// upd_issue stages one tile's rows of V_k, M_{k-2}, M_{k-1}, X into a 4-tile slot (cp.async, one
// commit group), upd_compute runs the tile's DMMAs from the slot and stores M_k and X.
template <int P>
struct UpdF {   // factor pointers in shared memory (FR doubles each)
    double *fA, *fB2, *fB1, *fZ, *fZp;
};
template <int P>
__device__ __forceinline__ void upd_setup(const K4bArgs& a, const UpdF<P>& f, int tid, int nth) {
    using D = DM<P>;
    constexpr int FR = D::FR;
    static_assert(FR == P * P, "fragment order of a p x p factor");
    DevState* st = a.st;
    const int xmode = a.xmode;
    // K3b(k) left the factors in fragment order (one load instead of a p x p product and four
    // reorderings on the critical path)
    const double* zf = st->ufz[a.zb % 3];   // (xmode != 0)
    for (int t = tid; t < FR; t += nth) {
        f.fA[t] = st->uf[a.par][0][t];
        f.fB2[t] = st->uf[a.par][1][t];
        f.fB1[t] = st->uf[a.par][2][t];
        f.fZp[t] = xmode == 2 ? st->ufz[(a.zb + 2) % 3][t] : 0.0;
        if (xmode != 0) f.fZ[t] = zf[t];
    }
    if (xmode == 0)
        for (int t = tid; t < FR; t += nth) {
            const int blk = t / 32, l = t % 32, kc = blk / D::NC, nc = blk % D::NC;
            f.fZ[t] = st->Z[a.par][(kc * 4 + l % 4) * MAXP + nc * 8 + l / 4];
        }
}
template <int P>
__device__ __forceinline__ void upd_issue(const K4bArgs& a, long long t, double* sl, int lane) {
    using D = DM<P>;
    const int xmode = a.xmode;
    const bool xonly = xmode == 3, with_x = xmode != 1;
    const long long base = t * D::TR;
    if (!xonly) stage_tile<P>(sl, a.U, base, a.n, lane);
    stage_tile<P>(sl + D::TILE, a.M2, base, a.n, lane);
    if (!xonly) stage_tile<P>(sl + 2 * D::TILE, a.M1, base, a.n, lane);
    if (with_x) stage_tile<P>(sl + 3 * D::TILE, a.X, base, a.n, lane);
}
template <int P>
__device__ __forceinline__ void upd_compute(const K4bArgs& a, const UpdF<P>& f, long long t, double* sl, int lane) {
    using D = DM<P>;
    constexpr int TR = D::TR, RS = D::RS, KC = D::KC, NC = D::NC;
    const int xmode = a.xmode;
    const bool xonly = xmode == 3, with_x = xmode != 1;
    const int fr = lane >> 2, fc = lane & 3;   // A-fragment row / col within an 8x4 block
    const double* tV = sl;
    double* tM2 = sl + D::TILE;
    const double* tM1 = sl + 2 * D::TILE;
    const double* tX = sl + 3 * D::TILE;
    const long long base = t * TR;
#pragma unroll
    for (int mc = 0; mc < TR / 8; ++mc) {
        const int r0 = mc * 8;
        const long long row = base + r0 + fr;
        if (xonly) {   // host flush of a deferred X update: X += M_k Z_k (M2 holds M_k)
#pragma unroll
            for (int nc = 0; nc < NC; ++nc) {
                const int col = nc * 8 + 2 * fc;
                double x0 = tX[(r0 + fr) * RS + col], x1 = tX[(r0 + fr) * RS + col + 1];
#pragma unroll
                for (int kc = 0; kc < KC; ++kc)
                    dmma(x0, x1, tM2[(r0 + fr) * RS + kc * 4 + fc], f.fZ[(kc * NC + nc) * 32 + lane]);
                if (row < a.n) *reinterpret_cast<double2*>(a.X + row * P + col) = make_double2(x0, x1);
            }
            continue;
        }
        double mk[NC][2];
#pragma unroll
        for (int nc = 0; nc < NC; ++nc) {
            mk[nc][0] = mk[nc][1] = 0.0;
#pragma unroll
            for (int kc = 0; kc < KC; ++kc) {
                const int ai = (r0 + fr) * RS + kc * 4 + fc;
                const int bi = (kc * NC + nc) * 32 + lane;
                // Tr_k R_kk^{-1} is upper triangular (both factors are): its rows 4kc.. are zero
                // in columns 8nc..8nc+7 when 4kc > 8nc+7
                if (kc <= 2 * nc + 1) dmma(mk[nc][0], mk[nc][1], tV[ai], f.fA[bi]);
                dmma(mk[nc][0], mk[nc][1], tM2[ai], f.fB2[bi]);
                dmma(mk[nc][0], mk[nc][1], tM1[ai], f.fB1[bi]);
            }
        }
        __syncwarp();
        // M_k overwrites this chunk's M_{k-2} rows (in smem and in HBM)
#pragma unroll
        for (int nc = 0; nc < NC; ++nc) {
            const int col = nc * 8 + 2 * fc;
            tM2[(r0 + fr) * RS + col] = mk[nc][0];
            tM2[(r0 + fr) * RS + col + 1] = mk[nc][1];
            if (row < a.n) *reinterpret_cast<double2*>(a.M2 + row * P + col) = make_double2(mk[nc][0], mk[nc][1]);
        }
        __syncwarp();
        if (!with_x) continue;   // xmode 1: this block's X update is deferred to the next one
#pragma unroll
        for (int nc = 0; nc < NC; ++nc) {
            const int col = nc * 8 + 2 * fc;
            double x0 = tX[(r0 + fr) * RS + col], x1 = tX[(r0 + fr) * RS + col + 1];
            if (xmode == 2) {   // first the deferred X += M_{k-1} Z_{k-1}
#pragma unroll
                for (int kc = 0; kc < KC; ++kc)
                    dmma(x0, x1, tM1[(r0 + fr) * RS + kc * 4 + fc], f.fZp[(kc * NC + nc) * 32 + lane]);
            }
#pragma unroll
            for (int kc = 0; kc < KC; ++kc)
                dmma(x0, x1, tM2[(r0 + fr) * RS + kc * 4 + fc], f.fZ[(kc * NC + nc) * 32 + lane]);
            if (row < a.n) *reinterpret_cast<double2*>(a.X + row * P + col) = make_double2(x0, x1);
        }
    }
    __syncwarp();
}

template <int P, int WARPS, int NS>
__device__ void dmma_update(const K4bArgs& a, long long t0, long long ts, long long tend, double* smem) {
    using D = DM<P>;
    constexpr int FR = D::FR;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    UpdF<P> f{smem, smem + FR, smem + 2 * FR, smem + 3 * FR, nullptr};
    double* pipe = smem + 4 * FR;
    double* scr = pipe + WARPS * NS * 4 * D::TILE;
    f.fZp = scr;   // Z_{k-1} (xmode 2), in the factor scratch (3 P^2 >= FR doubles)
    double* wb = pipe + warp * NS * 4 * D::TILE;
    const long long tw = t0 + warp;
    auto issue = [&](long long it, int slot) {
        const long long t = tw + it * ts;
        if (t < tend) upd_issue<P>(a, t, wb + slot * 4 * D::TILE, lane);
        cp_commit();
    };
    // the first stages stream in while the p x p factors are loaded
#pragma unroll
    for (int s = 0; s < NS - 1; ++s) issue(s, s);
    upd_setup<P>(a, f, threadIdx.x, blockDim.x);
    __syncthreads();
    for (long long it = 0; tw + it * ts < tend; ++it) {
        issue(it + NS - 1, (int)((it + NS - 1) % NS));
        cp_wait<NS - 1>();
        __syncwarp();
        upd_compute<P>(a, f, tw + it * ts, wb + (int)(it % NS) * 4 * D::TILE, lane);
    }
    cp_wait<0>();
}

// ------------------------------------------------------------------ K4b on DMMA (standalone)

template <int P>
struct K4bDSmem {
    static constexpr int WARPS = 4;
    static constexpr size_t bytes = sizeof(double) * UpdSmem<P, WARPS, NSTAGE>::doubles;
};

template <int P>
__global__ void __launch_bounds__(128) k4b_dmma(K4bArgs a) {
    constexpr int WARPS = K4bDSmem<P>::WARPS;
    DevState* st = a.st;
    if (!a.force && !st->side_go) return;
    unsigned long long* tr = trace_begin(st, TR_K4B);
    if (a.blk > 0 && blockIdx.x == 0 && threadIdx.x == 0) st->upd_last = a.blk;
    extern __shared__ __align__(16) double dynd4[];
    const long long ntiles = (a.n + DM<P>::TR - 1) / DM<P>::TR;
    dmma_update<P, WARPS, NSTAGE>(a, (long long)blockIdx.x * WARPS, (long long)gridDim.x * WARPS, ntiles, dynd4);
    trace_pt(tr, 5);
}


// Sum one warp-fragment accumulator of an 8x8 block (C layout) into sAcc[base + row*ld + col]
// in fixed warp order (called by every warp in turn between __syncthreads).
__device__ __forceinline__ void frag_acc(double* sAcc, int base, int ld, int m0, int n0, const double (&c)[2],
                                         bool first, int lane) {
    const int r = m0 + (lane >> 2), col = n0 + 2 * (lane & 3);
    double* d = sAcc + base + r * ld + col;
    d[0] = (first ? 0.0 : d[0]) + c[0];
    d[1] = (first ? 0.0 : d[1]) + c[1];
}

// The transpose of one accumulator block: C(r, c) of block (m0, n0) goes to sAcc[(n0+c)*ld + m0+r]
// (the mirrored half of a symmetric Gram), same fixed warp order as frag_acc.
__device__ __forceinline__ void frag_acc_t(double* sAcc, int ld, int m0, int n0, const double (&c)[2], bool first,
                                           int lane) {
    const int r = m0 + (lane >> 2), col = n0 + 2 * (lane & 3);
    double* d0 = sAcc + col * ld + r;
    double* d1 = sAcc + (col + 1) * ld + r;
    *d0 = (first ? 0.0 : *d0) + c[0];
    *d1 = (first ? 0.0 : *d1) + c[1];
}

// ------------------------------------------------------------------ K2 on DMMA

template <int P>
struct K2DSmem {
    // rows per warp tile: 16 (two 8-row DMMA chunks share every B fragment; the k-chunks run
    // outermost so every A fragment feeds NC DMMAs -- at p = 32 the 8-row version was bound by
    // shared-memory bandwidth, two LDS.64 per DMMA)
    static constexpr int TR = 16, MC = TR / 8, RS = DM<P>::RS, TILE = TR * RS;
#ifndef K2_NS32
#define K2_NS32 2
#endif
    static constexpr int WARPS = P >= 32 ? 4 : (P >= 16 ? 8 : 4);
    static constexpr int NS = P >= 32 ? K2_NS32 : (P >= 16 ? 2 : NSTAGE);   // cp.async stages (shared-memory budget)
    static constexpr int RSQ = 12;                        // pool tile row stride (8 columns + pad)
    static constexpr int TQ = TR * RSQ;
    static constexpr int STG = 2 * TILE + TQ;         // one stage of one warp
    // slot-major: stage s of warp w at pipe + (s * WARPS + w) * STG
    static constexpr int pipe = WARPS * NS * STG;
    static constexpr int LD = P + 1;
    // prologue scratch: sTk, sX, sG, sCo, k2_prologue's (P*P + P, then sGs).  It overlays the last
    // pipeline slot, which is first issued after the prologue (2 CTAs/SM at p = 16, 32)
    static constexpr int tail = 4 * P * P + P * MAXQ + P;
    static constexpr bool OVERLAY = tail <= WARPS * STG;
    static constexpr size_t bytes =
        sizeof(double) * (DM<P>::FR + DM<P>::KC * 32 + pipe + P * P + MAXQ * P + (OVERLAY ? 0 : tail));
};

template <int P>
__global__ void __launch_bounds__(K2DSmem<P>::WARPS * 32) k2_dmma(K2Args a) {
    using D = DM<P>;
    using S = K2DSmem<P>;
    constexpr int WARPS = S::WARPS, TR = S::TR, MC = S::MC, RS = S::RS, KC = D::KC, NC = D::NC, FR = D::FR;
    constexpr int RSQ = S::RSQ, TILE = S::TILE;
    DevState* st = a.st;
    unsigned long long* tr = trace_begin(st, TR_K2);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int fr = lane >> 2, fc = lane & 3;
    const int Q = st->q_live, qf = st->q_first, qc = st->pool_cap;
    const int E = P * P + Q * P;
    extern __shared__ __align__(16) double dynd2[];
    double* fE = dynd2;              // -(Tr_k G_s) in fragment order
    double* fF = fE + FR;            // -(Tr_k coef_{k-1}) (P x 8) in fragment order (KC blocks)
    double* pipe = fF + KC * 32;
    double* sAcc = pipe + S::pipe;
    double* sTail = S::OVERLAY ? pipe + (S::NS - 1) * WARPS * S::STG : sAcc + P * P + MAXQ * P;
    double* wb = pipe + warp * S::STG;
    const long long ntiles = (a.n + TR - 1) / TR;
    const long long t0 = (long long)blockIdx.x * WARPS + warp, ts = (long long)gridDim.x * WARPS;
    auto issue = [&](long long it, int slot) {
        const long long t = t0 + it * ts;
        if (t < ntiles) {
            double* sl = wb + slot * WARPS * S::STG;
            const long long base = t * TR;
            stage_rows<P, TR>(sl, a.W, base, a.n, lane);
            stage_rows<P, TR>(sl + TILE, a.V, base, a.n, lane);
            for (int c = lane; c < TR * MAXQ; c += 32) {
                const int r = c / MAXQ, q = c % MAXQ;
                const long long i = base + r;
                const bool ok = i < a.n && q < Q;
                cp_async8(sl + 2 * TILE + r * RSQ + q, a.pool + (ok ? i * qc + qf + q : 0), ok);
            }
        }
        cp_commit();
    };
    // the first stages stream in during the wait and the prologue (K1 completed before
    // reduce1 started; only the totals come from reduce1)
#pragma unroll
    for (int s = 0; s < S::NS - 1; ++s) issue(s, s);
    pdl_wait();   // red1 (reduce1) is ready
    if (!st->run_main) {   // (stopped; uniform over the launch: see publish_breakdown)
        cp_wait<0>();
        k2_stopped(st);
        return;
    }
    trace_pt(tr, 1);
    {
        // G = Tr_k^T (V_k^T W) from K1's partials; G_s: lower triangle mirrored (the paper
        // computes h_{i,j} for i >= j)
        double* sTk = sTail;
        double* sX = sTail + P * P;
        double* sG = sTail + 2 * P * P;
        double* sCo = sTail + 3 * P * P;                // P x MAXQ
        double* sScr = sCo + P * MAXQ;                  // k2_prologue's red1 copy, then sGs
        double* sGs = sScr;
        const double* Co = st->coef[a.par ^ 1];
        for (int t = threadIdx.x; t < P * MAXQ; t += blockDim.x) sCo[t] = Co[t];
        k2_prologue<P>(st, a.par, a.sk, sG, sTk, sScr);   // (syncs after its loads)
        for (int t = threadIdx.x; t < P * P; t += blockDim.x) {
            const int r = t / P, c = t % P;
            sGs[t] = r >= c ? sG[r * P + c] : sG[c * P + r];
        }
        __syncthreads();
        cta_matmul_nn<P>(sTk, P, sGs, P, sX, P);
        // F = Tr_k coef_{k-1}: P x 8 (pool columns q < Q, the rest 0), fragment order over KC blocks
        for (int t = threadIdx.x; t < KC * 32; t += blockDim.x) {
            const int kc = t / 32, l = t % 32, r = kc * 4 + l % 4, q = l / 4;
            double s = 0.0;
            if (q < Q)
                for (int i = 0; i < P; ++i) s = fma(sTk[r * P + i], sCo[i * MAXQ + q], s);
            fF[t] = -s;
        }
        __syncthreads();
        to_frag<P>(sX, P, -1.0, fE);
        __syncthreads();
    }
    trace_pt(tr, 3);
    double g[NC][NC][2], pq[NC][2];
#pragma unroll
    for (int i = 0; i < NC; ++i) {
        pq[i][0] = pq[i][1] = 0.0;
#pragma unroll
        for (int j = 0; j < NC; ++j) g[i][j][0] = g[i][j][1] = 0.0;
    }
    for (long long it = 0; t0 + it * ts < ntiles; ++it) {
        issue(it + S::NS - 1, (int)((it + S::NS - 1) % S::NS));
        cp_wait<S::NS - 1>();
        __syncwarp();
        double* sl = wb + (int)(it % S::NS) * WARPS * S::STG;
        double* tW = sl;
        const double* tV = sl + TILE;
        double* tR = sl + 2 * TILE;
        const long long base = (t0 + it * ts) * TR;
        // pool r_q -= U_k coef_{k-1}(:,q) = V_k F(:,q) and W' = W - U_k G_s = W - V_k (Tr_k G_s),
        // k-chunks outermost (each output accumulates over kc in increasing order)
        double c[MC][NC][2], cq[MC][2];
#pragma unroll
        for (int mc = 0; mc < MC; ++mc) {
            cq[mc][0] = tR[(mc * 8 + fr) * RSQ + 2 * fc];
            cq[mc][1] = tR[(mc * 8 + fr) * RSQ + 2 * fc + 1];
#pragma unroll
            for (int nc = 0; nc < NC; ++nc) {
                c[mc][nc][0] = tW[(mc * 8 + fr) * RS + nc * 8 + 2 * fc];
                c[mc][nc][1] = tW[(mc * 8 + fr) * RS + nc * 8 + 2 * fc + 1];
            }
        }
#pragma unroll
        for (int kc = 0; kc < KC; ++kc) {
            double aV[MC];
#pragma unroll
            for (int mc = 0; mc < MC; ++mc) aV[mc] = tV[(mc * 8 + fr) * RS + kc * 4 + fc];
            if (Q > 0) {
                const double bq = fF[kc * 32 + lane];
#pragma unroll
                for (int mc = 0; mc < MC; ++mc) dmma(cq[mc][0], cq[mc][1], aV[mc], bq);
            }
#pragma unroll
            for (int nc = 0; nc < NC; ++nc) {
                const double be = fE[(kc * NC + nc) * 32 + lane];
#pragma unroll
                for (int mc = 0; mc < MC; ++mc) dmma(c[mc][nc][0], c[mc][nc][1], aV[mc], be);
            }
        }
        __syncwarp();
#pragma unroll
        for (int mc = 0; mc < MC; ++mc) {
            const int r0 = mc * 8;
            const long long row = base + r0 + fr;
            const bool rok = row < a.n;
            if (Q > 0) {
                tR[(r0 + fr) * RSQ + 2 * fc] = cq[mc][0];
                tR[(r0 + fr) * RSQ + 2 * fc + 1] = cq[mc][1];
                if (rok) {
                    if (2 * fc < Q) a.pool[row * qc + qf + 2 * fc] = cq[mc][0];
                    if (2 * fc + 1 < Q) a.pool[row * qc + qf + 2 * fc + 1] = cq[mc][1];
                }
            }
#pragma unroll
            for (int nc = 0; nc < NC; ++nc) {
                const int col = nc * 8 + 2 * fc;
                tW[(r0 + fr) * RS + col] = c[mc][nc][0];
                tW[(r0 + fr) * RS + col + 1] = c[mc][nc][1];
                if (rok) *reinterpret_cast<double2*>(a.W + row * P + col) = make_double2(c[mc][nc][0], c[mc][nc][1]);
            }
        }
        __syncwarp();
        // W'^T W' and R^T W' over the tile's rows, 4 rows per MMA
#pragma unroll
        for (int k0 = 0; k0 < TR; k0 += 4) {
            const double* rw = tW + (k0 + fc) * RS;
#pragma unroll
            for (int i = 0; i < NC; ++i) {
                const double av = rw[i * 8 + fr];
                // W'^T W' is symmetric: the blocks j <= i only (mirrored in the CTA sum)
#pragma unroll
                for (int j = 0; j <= i; ++j) dmma(g[i][j][0], g[i][j][1], av, rw[j * 8 + fr]);
            }
            if (Q > 0) {
                const double ar = tR[(k0 + fc) * RSQ + fr];
#pragma unroll
                for (int j = 0; j < NC; ++j) dmma(pq[j][0], pq[j][1], ar, rw[j * 8 + fr]);
            }
        }
        __syncwarp();
    }
    cp_wait<0>();
    trace_pt(tr, 4);
    pdl_trigger();   // the dependent (reduce2) launches while this grid reduces its partials
    // rows past n were zero-filled, so they contribute nothing; reduce across warps (fixed order)
    for (int w = 0; w < WARPS; ++w) {
        if (warp == w) {
#pragma unroll
            for (int i = 0; i < NC; ++i)
#pragma unroll
                for (int j = 0; j <= i; ++j) {
                    frag_acc(sAcc, 0, P, i * 8, j * 8, g[i][j], w == 0, lane);
                    if (j < i) frag_acc_t(sAcc, P, i * 8, j * 8, g[i][j], w == 0, lane);
                }
            if (Q > 0) {
                // pdot(q, m) = (R^T W')(q, m) at P*P + q*P + m, q < Q
                const int q = fr;
#pragma unroll
                for (int j = 0; j < NC; ++j) {
                    const int col = j * 8 + 2 * fc;
                    if (q < Q) {
                        double* d = sAcc + P * P + q * P + col;
                        d[0] = (w == 0 ? 0.0 : d[0]) + pq[j][0];
                        d[1] = (w == 0 ? 0.0 : d[1]) + pq[j][1];
                    }
                }
            }
        }
        __syncthreads();
    }
    cluster_partials(sAcc, E, st->part2[a.par]);   // reduce2, then K1(k+1) and K3b(k) factor W' from these
    trace_pt(tr, 5);
}


// ------------------------------------------------------------------ start block on DMMA
//
// The start block's CholQR2 (eqn.init-QR, reading C13): the Gram F^T F of the n x p
// panel and U = F R^{-1}, with the row-local products on DMMA (once per solve; they replace the
// generic k_gram / k_materialize for p in {8, 16, 32}).

template <int P>
struct GramDSmem {
    static constexpr int WARPS = 8, NS = 2;
    static constexpr size_t bytes = sizeof(double) * (WARPS * NS * DM<P>::TILE + P * P);
};

// out = F^T F: per-CTA partials (part[e*nb + cta]), the last CTA sums them in fixed order
template <int P>
__global__ void __launch_bounds__(256) k_gram_dmma(const double* X, long long n, int, double* part, int nb, double* out,
                                                   unsigned* cnt) {
    using D = DM<P>;
    using S = GramDSmem<P>;
    constexpr int TR = D::TR, RS = D::RS, NC = D::NC, NS = S::NS, WARPS = S::WARPS, E = P * P;
    extern __shared__ __align__(16) double dyng[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int fr = lane >> 2, fc = lane & 3;
    double* wb = dyng + warp * NS * D::TILE;
    double* sAcc = dyng + WARPS * NS * D::TILE;
    const long long ntiles = (n + TR - 1) / TR;
    const long long t0 = (long long)blockIdx.x * WARPS + warp, ts = (long long)gridDim.x * WARPS;
    auto issue = [&](long long it) {
        const long long t = t0 + it * ts;
        if (t < ntiles) stage_tile<P>(wb + (int)(it % NS) * D::TILE, X, t * TR, n, lane);
        cp_commit();
    };
    double g[NC][NC][2];
#pragma unroll
    for (int i = 0; i < NC; ++i)
#pragma unroll
        for (int j = 0; j < NC; ++j) g[i][j][0] = g[i][j][1] = 0.0;
    issue(0);
    for (long long it = 0; t0 + it * ts < ntiles; ++it) {
        issue(it + 1);
        cp_wait<1>();
        __syncwarp();
        const double* tl = wb + (int)(it % NS) * D::TILE;
#pragma unroll
        for (int k0 = 0; k0 < TR; k0 += 4) {
            const double* rw = tl + (k0 + fc) * RS;
#pragma unroll
            for (int i = 0; i < NC; ++i) {
                const double av = rw[i * 8 + fr];
#pragma unroll
                for (int j = 0; j <= i; ++j) dmma(g[i][j][0], g[i][j][1], av, rw[j * 8 + fr]);
            }
        }
        __syncwarp();
    }
    cp_wait<0>();
    for (int w = 0; w < WARPS; ++w) {
        if (warp == w) {
#pragma unroll
            for (int i = 0; i < NC; ++i)
#pragma unroll
                for (int j = 0; j <= i; ++j) {
                    frag_acc(sAcc, 0, P, i * 8, j * 8, g[i][j], w == 0, lane);
                    if (j < i) frag_acc_t(sAcc, P, i * 8, j * 8, g[i][j], w == 0, lane);
                }
        }
        __syncthreads();
    }
    for (int e = threadIdx.x; e < E; e += blockDim.x) part[(size_t)e * nb + blockIdx.x] = sAcc[e];
    __shared__ int s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(cnt, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    for (int e = warp; e < E; e += WARPS) {
        double t = 0.0;
        for (int b = lane; b < nb; b += 32) t += __ldcg(part + (size_t)e * nb + b);
        t = warp_sum(t);
        if (lane == 0) out[e] = t;
    }
    if (threadIdx.x == 0) *cnt = 0u;
}

// out = V Tr (n x P row-major panels; Tr P x P with leading dimension MAXP)
template <int P>
__global__ void __launch_bounds__(256) k_materialize_dmma(const double* V, const double* Tr, double* out, long long n,
                                                          int) {
    using D = DM<P>;
    constexpr int TR = D::TR, RS = D::RS, KC = D::KC, NC = D::NC, NS = 2, WARPS = 8;
    extern __shared__ __align__(16) double dynm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int fr = lane >> 2, fc = lane & 3;
    double* fT = dynm;
    double* wb = fT + D::FR + warp * NS * D::TILE;
    to_frag<P>(Tr, MAXP, 1.0, fT);
    __syncthreads();
    const long long ntiles = (n + TR - 1) / TR;
    const long long t0 = (long long)blockIdx.x * WARPS + warp, ts = (long long)gridDim.x * WARPS;
    auto issue = [&](long long it) {
        const long long t = t0 + it * ts;
        if (t < ntiles) stage_tile<P>(wb + (int)(it % NS) * D::TILE, V, t * TR, n, lane);
        cp_commit();
    };
    issue(0);
    for (long long it = 0; t0 + it * ts < ntiles; ++it) {
        issue(it + 1);
        cp_wait<1>();
        __syncwarp();
        const double* tl = wb + (int)(it % NS) * D::TILE;
        const long long base = (t0 + it * ts) * TR;
#pragma unroll
        for (int mc = 0; mc < TR / 8; ++mc) {
            const long long row = base + mc * 8 + fr;
#pragma unroll
            for (int nc = 0; nc < NC; ++nc) {
                double c0 = 0.0, c1 = 0.0;
#pragma unroll
                for (int kc = 0; kc < KC; ++kc)
                    dmma(c0, c1, tl[(mc * 8 + fr) * RS + kc * 4 + fc], fT[(kc * NC + nc) * 32 + lane]);
                if (row < n) *reinterpret_cast<double2*>(out + row * P + nc * 8 + 2 * fc) = make_double2(c0, c1);
            }
        }
        __syncwarp();
    }
    cp_wait<0>();
}
template <int P>
constexpr size_t mat_dmma_smem() { return sizeof(double) * (DM<P>::FR + 8 * 2 * DM<P>::TILE); }

// ------------------------------------------------------------------ the M/X update as its own kernel
//
// Row a5 (eqn.search-dir-comp, eqn.approx-update) for large panels (split mode,
// p in {16, 32}): the update of block k-2 on the main stream right before K1a(k) (its V_{k-2} rows
// are overwritten by K1(k)'s W).  Same arithmetic as dmma_update -- for every output the DMMAs
// accumulate in the same order ([Tr R^{-1}], -B2, -B1 per k-chunk; then Z_{k-1}, then Z_k) -- so the
// results are bitwise those of the fused update.  The difference is register blocking: a warp
// owns TRU = 16 rows (two 8-row DMMA chunks) and walks the k-chunks outermost, so each A fragment
// feeds NC DMMAs and each B fragment (a p x p factor in fragment order) two, instead of one each
// (at p = 32 the fused update was bound by shared-memory bandwidth: 2 LDS.64 per DMMA).
template <int P>
struct UpdB {
    // p = 32: sixteen warps of 8-row tiles (single-staged: shared-memory budget) -- twice the warps
    // in flight per SM of sixteen-row tiles, at 82 registers (config 4: 4.83 -> 4.56 ms per launch;
    // 8 rows double-staged: 5.13 ms); p = 16: eight warps of 16 rows, double-staged
#ifndef K1U_WARPS32
#define K1U_WARPS32 16
#endif
#ifndef K1U_NS32
#define K1U_NS32 1
#endif
    static constexpr int WARPS = P >= 32 ? K1U_WARPS32 : 8;
    static constexpr int TRU = P >= 32 ? 8 : 16;
    static constexpr int MC = TRU / 8;
    static constexpr int NS = P >= 32 ? K1U_NS32 : 2;     // cp.async stages per warp (shared-memory budget)
    static constexpr int RS = P + 4;
    static constexpr int TILE = TRU * RS;
    static constexpr int SLOT = 4 * TILE;          // V_b, M_{b-2} (-> M_b), M_{b-1}, X
    static constexpr size_t bytes = sizeof(double) * (5 * P * P + WARPS * NS * SLOT);
};


template <int P>
__global__ void __launch_bounds__(UpdB<P>::WARPS * 32, 1) k1u_update(K1Args a) {
    using U = UpdB<P>;
    using D = DM<P>;
    constexpr int WARPS = U::WARPS, TRU = U::TRU, MC = U::MC, NS = U::NS, RS = U::RS, TILE = U::TILE;
    constexpr int KC = D::KC, NC = D::NC, FR = D::FR;
    DevState* st = a.st;
    pdl_wait();   // (reduce2 of block k-1 has completed; K1a(k) and K1(k) wait for this grid)
    const long long k = st->k_main, b = k - 2;
    // the same condition as K1's fused update (uniform over CTAs; see k1_dmma)
    if (!(b >= st->k_upd_min && b < st->k_side && b < st->stop_side_at)) return;
    unsigned long long* tr = trace_begin(st, TR_K4B);
    if (blockIdx.x == 0 && threadIdx.x == 0) st->upd_last = b;
    const int xm = a.xdefer ? (((b - st->k_upd_min) & 1) ? 2 : 1) : 0;
    const bool with_x = xm != 1;
    K4bArgs u{a.Y, a.Mk2, a.Mk1, a.Xs, a.n, st, (a.sk + 1) % 3, 0, a.par, 1, b, xm, b};
    extern __shared__ __align__(16) double dynu[];
    UpdF<P> f{dynu, dynu + FR, dynu + 2 * FR, dynu + 3 * FR, dynu + 4 * FR};
    double* pipe = dynu + 5 * FR;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int fr = lane >> 2, fc = lane & 3;
    double* wb = pipe + warp * NS * U::SLOT;
    const long long ntiles = (a.n + TRU - 1) / TRU;
    const long long tw = (long long)blockIdx.x * WARPS + warp, ts = (long long)gridDim.x * WARPS;
    auto issue = [&](long long it) {
        const long long t = tw + it * ts;
        if (t < ntiles) {
            double* sl = wb + (int)(it % NS) * U::SLOT;
            const long long base = t * TRU;
            stage_rows<P, TRU>(sl, u.U, base, a.n, lane);
            stage_rows<P, TRU>(sl + TILE, u.M2, base, a.n, lane);
            stage_rows<P, TRU>(sl + 2 * TILE, u.M1, base, a.n, lane);
            if (with_x) stage_rows<P, TRU>(sl + 3 * TILE, u.X, base, a.n, lane);
        }
        cp_commit();
    };
#pragma unroll
    for (int s = 0; s < NS - 1; ++s) issue(s);
    upd_setup<P>(u, f, threadIdx.x, blockDim.x);
    __syncthreads();
    for (long long it = 0; tw + it * ts < ntiles; ++it) {
        if (NS > 1) {
            issue(it + NS - 1);
            cp_wait<NS - 1>();
        } else {
            issue(it);
            cp_wait<0>();
        }
        __syncwarp();
        double* sl = wb + (int)(it % NS) * U::SLOT;
        const double* tV = sl;
        double* tM2 = sl + TILE;
        const double* tM1 = sl + 2 * TILE;
        const double* tX = sl + 3 * TILE;
        const long long base = (tw + it * ts) * TRU;
        // M_b = V_b (Tr_b R^{-1}) - M_{b-2} B2 - M_{b-1} B1, k-chunks outermost
        double mk[MC][NC][2];
#pragma unroll
        for (int mc = 0; mc < MC; ++mc)
#pragma unroll
            for (int nc = 0; nc < NC; ++nc) mk[mc][nc][0] = mk[mc][nc][1] = 0.0;
#pragma unroll
        for (int kc = 0; kc < KC; ++kc) {
            double aV[MC], a2[MC], a1[MC];
#pragma unroll
            for (int mc = 0; mc < MC; ++mc) {
                const int ai = (mc * 8 + fr) * RS + kc * 4 + fc;
                aV[mc] = tV[ai];
                a2[mc] = tM2[ai];
                a1[mc] = tM1[ai];
            }
#pragma unroll
            for (int nc = 0; nc < NC; ++nc) {
                const int bi = (kc * NC + nc) * 32 + lane;
                const bool tri = kc <= 2 * nc + 1;   // Tr_b R^{-1} is upper triangular
                const double bA = tri ? f.fA[bi] : 0.0, b2 = f.fB2[bi], b1 = f.fB1[bi];
#pragma unroll
                for (int mc = 0; mc < MC; ++mc) {
                    if (tri) dmma(mk[mc][nc][0], mk[mc][nc][1], aV[mc], bA);
                    dmma(mk[mc][nc][0], mk[mc][nc][1], a2[mc], b2);
                    dmma(mk[mc][nc][0], mk[mc][nc][1], a1[mc], b1);
                }
            }
        }
        __syncwarp();
        // M_b overwrites M_{b-2} (in the tile and in HBM)
#pragma unroll
        for (int mc = 0; mc < MC; ++mc) {
            const long long row = base + mc * 8 + fr;
#pragma unroll
            for (int nc = 0; nc < NC; ++nc) {
                const int col = nc * 8 + 2 * fc;
                tM2[(mc * 8 + fr) * RS + col] = mk[mc][nc][0];
                tM2[(mc * 8 + fr) * RS + col + 1] = mk[mc][nc][1];
                if (row < a.n) *reinterpret_cast<double2*>(u.M2 + row * P + col) = make_double2(mk[mc][nc][0], mk[mc][nc][1]);
            }
        }
        __syncwarp();
        if (with_x) {
            // X += M_{b-1} Z_{b-1} (deferred, xm = 2), then X += M_b Z_b
            double x[MC][NC][2];
#pragma unroll
            for (int mc = 0; mc < MC; ++mc)
#pragma unroll
                for (int nc = 0; nc < NC; ++nc) {
                    const int col = nc * 8 + 2 * fc;
                    x[mc][nc][0] = tX[(mc * 8 + fr) * RS + col];
                    x[mc][nc][1] = tX[(mc * 8 + fr) * RS + col + 1];
                }
            if (xm == 2) {
#pragma unroll
                for (int kc = 0; kc < KC; ++kc) {
                    double a1[MC];
#pragma unroll
                    for (int mc = 0; mc < MC; ++mc) a1[mc] = tM1[(mc * 8 + fr) * RS + kc * 4 + fc];
#pragma unroll
                    for (int nc = 0; nc < NC; ++nc) {
                        const double bz = f.fZp[(kc * NC + nc) * 32 + lane];
#pragma unroll
                        for (int mc = 0; mc < MC; ++mc) dmma(x[mc][nc][0], x[mc][nc][1], a1[mc], bz);
                    }
                }
            }
#pragma unroll
            for (int kc = 0; kc < KC; ++kc) {
                double a2[MC];
#pragma unroll
                for (int mc = 0; mc < MC; ++mc) a2[mc] = tM2[(mc * 8 + fr) * RS + kc * 4 + fc];
#pragma unroll
                for (int nc = 0; nc < NC; ++nc) {
                    const double bz = f.fZ[(kc * NC + nc) * 32 + lane];
#pragma unroll
                    for (int mc = 0; mc < MC; ++mc) dmma(x[mc][nc][0], x[mc][nc][1], a2[mc], bz);
                }
            }
#pragma unroll
            for (int mc = 0; mc < MC; ++mc) {
                const long long row = base + mc * 8 + fr;
                if (row < a.n)
#pragma unroll
                    for (int nc = 0; nc < NC; ++nc)
                        *reinterpret_cast<double2*>(u.X + row * P + nc * 8 + 2 * fc) =
                            make_double2(x[mc][nc][0], x[mc][nc][1]);
            }
        }
        __syncwarp();
    }
    cp_wait<0>();
    trace_pt(tr, 5);
}

// ------------------------------------------------------------------ K1a: the SpMM alone (split mode)
//
// Row a1's operator product AV = A V_k (eqn.block-Lanczos-recurr's A u_j, applied to the
// p vectors of the block at once), for large panels: a register-light kernel at full
// occupancy (no shared memory, no epilogue) keeps ~2.5x more gathers in flight per SM than the
// fused K1 can; K1<P, true> then streams AV like a panel.  Rows are summed
// in CSR order with fma from 0, exactly as K1's own gathers, so AV is bitwise the same.
// Order: CTA chunks of WARPS*KU consecutive row groups, round-robin over the CTAs -- neighbouring
// rows stay in one SM's L1 and all SMs sweep the matrix together, so far (z-plane) neighbours are
// re-read from L2.
#ifndef K1A_STREAM
#define K1A_STREAM 0
#endif
template <int P>
struct K1aCfg {
    // a lane gathers 32 bytes of a row per entry (one 256-bit load, LDG.E.ENL2.256) when 4 | p:
    // half the lanes per row of the 16-byte mapping, so half the redundant column-index / value
    // loads and address arithmetic per gathered byte (ncu: the 16-byte version issued 55-58%)
    static constexpr int VEC = (P % 4 == 0) ? 4 : (P % 2 == 0 ? 2 : 1);
    static constexpr int LANES = P / VEC;
    static constexpr int LP = LANES <= 1 ? 1 : LANES <= 2 ? 2 : LANES <= 4 ? 4 : LANES <= 8 ? 8 : LANES <= 16 ? 16 : 32;
    static constexpr int RPW = 32 / LP;
    static constexpr int CH = VEC == 4 ? 4 : 8;   // CSR entries per gather batch
    static constexpr int KU = 8;                  // row groups per warp per CTA chunk
    static constexpr int MINB = 5;                // CTAs per SM (<= 48 registers)
    static constexpr int MINB_LONG = 4;           // the long-row variant (<= 64 registers)
};

template <int P>
struct K1Gather {
    static constexpr int VEC = (P == 16 || P == 8) ? 4 : PC<P>::VEC;
    static constexpr int LANES = P / VEC;
    static constexpr int LP = LANES <= 1 ? 1 : LANES <= 2 ? 2 : LANES <= 4 ? 4 : LANES <= 8 ? 8 : LANES <= 16 ? 16 : 32;
    static constexpr int RPW = 32 / LP;
};

template <int VEC>
__device__ __forceinline__ void ldg_vec(const double* p, double (&r)[VEC]) {
    if constexpr (VEC == 4) {
        asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                     : "=d"(r[0]), "=d"(r[1]), "=d"(r[2]), "=d"(r[3])
                     : "l"(p));
    } else {
        ldv<VEC>(p, r);
    }
}

// LONG: the variant for matrices with long rows (>= 12 entries per row on average, i.e. three or
// more gather batches per row): the next batch's column indices / values are loaded while this
// batch's gathers are in flight, so a row's dependent chain is index -> gather -> gather -> ...
// instead of index -> gather -> index -> gather -> ...; 12 more registers, 4 CTAs per SM instead of 5.
// Config 5 (~27 entries per row): K1a 1.61 -> 1.47 ms, 5844 -> 6110 it/s; config 4 (7 entries, two
// batches): 2.98 -> 3.22 ms, so short rows keep the plain variant (same sums in the same order).
template <int P, bool LONG = false>
__global__ void __launch_bounds__(NT, LONG ? K1aCfg<P>::MINB_LONG : K1aCfg<P>::MINB) k1a_spmm(K1Args a) {
    using C = K1aCfg<P>;
    constexpr int VEC = C::VEC, LANES = C::LANES, LP = C::LP, RPW = C::RPW;
    constexpr int CH = C::CH, KU = C::KU;
    DevState* st = a.st;   // null: plain SpMM (exit residual, bminres_spmm)
    unsigned long long* tr = st ? trace_begin(st, TR_K1A) : nullptr;
    pdl_wait();   // V_k (K2 of block k-1) is complete and visible
    trace_pt(tr, 1);
    if (st && !st->run_main) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int sub = lane % LP, rsub = lane / LP;
    const bool act = sub < LANES;
    const int c0 = sub * VEC;
    // rows: all n, or (row partition, halo overlap) the interior range / the boundary rows around it
    const long long nr = a.nrows >= 0 ? a.nrows : a.n;
    const long long ngroups = (nr + RPW - 1) / RPW;
    const long long chunk = (long long)nw * (a.ku > 0 ? a.ku : KU);
    // chunk order: static round robin over the CTAs, or (dyn) taken in increasing order from a
    // counter by whichever CTA is resident -- all resident CTAs then sweep the rows together even
    // when some become resident late (K1a running beside the update kernel), so the far stencil
    // neighbours (z planes) stay in L2
    __shared__ long long s_chunk;
    unsigned long long* ctr = (st && a.dyn) ? st->k1a_ctr + (a.dyn - 1) : nullptr;
    auto next_chunk = [&](long long cur) -> long long {
        if (!ctr) return cur < 0 ? (long long)blockIdx.x : cur + gridDim.x;
        __syncthreads();   // every warp is done with the current chunk's s_chunk
        if (threadIdx.x == 0) s_chunk = (long long)atomicAdd(ctr, 1ull);
        __syncthreads();
        return s_chunk;
    };
    long long cidx = next_chunk(-1);
    int cpos = warp;
    auto phys = [&](long long c) -> long long { return c; };
    int pr0 = 0, pr1 = 0;
    bool have = false;
    for (long long g = cidx * chunk + cpos; g < ngroups || (ctr && cidx * chunk < ngroups);) {
        if (g >= ngroups) {   // (dyn: this warp has no group in the chunk's tail; the others may)
            have = false;
            cpos = warp;
            cidx = next_chunk(cidx);
            g = cidx * chunk + cpos;
            continue;
        }
        const long long v = g * RPW + rsub;
        const long long i = a.r0 + v + ((a.gap_at >= 0 && v >= a.gap_at) ? a.gap : 0);
        const bool live = act && v < nr;
        int r0, r1;
        if (have) {
            r0 = pr0;
            r1 = pr1;
        } else {
            r0 = live ? __ldg(a.rowptr + i) : 0;
            r1 = live ? __ldg(a.rowptr + i + 1) : 0;
        }
        if constexpr (LONG) {
            // the next group's row pointers too, where the next group is known (inside the chunk;
            // static order): config 5 K1a 1.46 -> 1.40 ms (the plain variant loses with it: 48
            // registers spill, config 4 2.98 -> 3.18 ms)
            int ncpos = cpos + nw;
            long long ncidx = cidx;
            const bool same = ncpos < chunk;
            if (!same && !ctr) {
                ncpos = warp;
                ncidx = cidx + gridDim.x;
            }
            have = false;
            if (same || !ctr) {
                const long long gn = phys(ncidx) * chunk + ncpos;
                if (gn < ngroups) {
                    const long long vn = gn * RPW + rsub;
                    const long long in = a.r0 + vn + ((a.gap_at >= 0 && vn >= a.gap_at) ? a.gap : 0);
                    const bool ln = act && vn < nr;
                    pr0 = ln ? __ldg(a.rowptr + in) : 0;
                    pr1 = ln ? __ldg(a.rowptr + in + 1) : 0;
                    have = true;
                }
            }
        }
        double acc[VEC];
#pragma unroll
        for (int v = 0; v < VEC; ++v) acc[v] = 0.0;
        if constexpr (LONG) {
        int c[CH];
        double av[CH];
#pragma unroll
        for (int t = 0; t < CH; ++t) {
            const bool pr = r0 + t < r1;
            c[t] = pr ? __ldg(a.col + r0 + t) : -1;
            av[t] = pr ? __ldg(a.val + r0 + t) : 0.0;
        }
        for (int kb = r0; __any_sync(FULL, kb < r1); kb += CH) {
            double xv[CH][VEC];
#pragma unroll
            for (int t = 0; t < CH; ++t) {
                if (c[t] >= 0) {
                    ldg_vec<VEC>(a.X + (long long)c[t] * P + c0, xv[t]);
                } else {
#pragma unroll
                    for (int v = 0; v < VEC; ++v) xv[t][v] = 0.0;
                }
            }
            int cn[CH];
            double an[CH];
#pragma unroll
            for (int t = 0; t < CH; ++t) {
                const bool pr = kb + CH + t < r1;
                cn[t] = pr ? __ldg(a.col + kb + CH + t) : -1;
                an[t] = pr ? __ldg(a.val + kb + CH + t) : 0.0;
            }
#pragma unroll
            for (int t = 0; t < CH; ++t)
                if (c[t] >= 0) {
#pragma unroll
                    for (int v = 0; v < VEC; ++v) acc[v] = fma(av[t], xv[t][v], acc[v]);
                }
#pragma unroll
            for (int t = 0; t < CH; ++t) {
                c[t] = cn[t];
                av[t] = an[t];
            }
        }
        } else {
        for (int kb = r0; __any_sync(FULL, kb < r1); kb += CH) {
            int c[CH];
            double av[CH];
#pragma unroll
            for (int t = 0; t < CH; ++t) {
                const bool pr = kb + t < r1;
#if K1A_STREAM
                // A is read once per block step: evict-first, so it does not push the gathered V_k
                // rows (re-read as stencil neighbours planes later) out of L2
                c[t] = pr ? __ldcs(a.col + kb + t) : -1;
                av[t] = pr ? __ldcs(a.val + kb + t) : 0.0;
#else
                c[t] = pr ? __ldg(a.col + kb + t) : -1;
                av[t] = pr ? __ldg(a.val + kb + t) : 0.0;
#endif
            }
            double xv[CH][VEC];
#pragma unroll
            for (int t = 0; t < CH; ++t) {
                if (c[t] >= 0) {
                    ldg_vec<VEC>(a.X + (long long)c[t] * P + c0, xv[t]);
                } else {
#pragma unroll
                    for (int v = 0; v < VEC; ++v) xv[t][v] = 0.0;
                }
            }
#pragma unroll
            for (int t = 0; t < CH; ++t)
                if (c[t] >= 0) {
#pragma unroll
                    for (int v = 0; v < VEC; ++v) acc[v] = fma(av[t], xv[t][v], acc[v]);
                }
        }
        }
        if (live) {
            double* y = a.Y + i * P + c0;   // Y = the AV panel
            if constexpr (VEC == 4) {
#if K1A_STREAM
                // (the AV panel is read once, by K1's epilogue: streaming stores)
                __stcs(reinterpret_cast<double2*>(y), make_double2(acc[0], acc[1]));
                __stcs(reinterpret_cast<double2*>(y + 2), make_double2(acc[2], acc[3]));
#else
                *reinterpret_cast<double2*>(y) = make_double2(acc[0], acc[1]);
                *reinterpret_cast<double2*>(y + 2) = make_double2(acc[2], acc[3]);
#endif
            } else {
                stv<VEC>(y, acc);
            }
        }
        cpos += nw;
        if (cpos >= chunk) {
            cpos = warp;
            cidx = next_chunk(cidx);
        }
        g = cidx * chunk + cpos;
    }
    trace_pt(tr, 4);
    pdl_trigger();
    trace_pt(tr, 5);
}

// ------------------------------------------------------------------ K1 on DMMA (epilogue)

template <int P, bool PRE = false>
struct K1DSmem {
    // p = 32: one 512-thread CTA per SM (16 warps, <= 128 registers) instead of one 256-thread
    // CTA at 209 registers -- the gathers need the warps; the fused update single-staged
#ifndef K1PRE_WARPS32
#define K1PRE_WARPS32 16
#endif
#ifndef K1PRE_NSP32
#define K1PRE_NSP32 1
#endif
    static constexpr int WARPS = (PRE && P >= 32) ? K1PRE_WARPS32 : (P >= 32 ? 16 : 8);
#ifndef K1_DISJ
#define K1_DISJ 1
#endif
    // DISJ (p <= 16, fused): the update's staging is disjoint from the SpMM's, single-staged, so a
    // warp starts its first SpMM tile as soon as its own update tiles are done (each warp updates
    // exactly the rows whose W it writes later: same tiling, no cross-warp hazard)
    static constexpr bool DISJ = K1_DISJ && !PRE && P <= 16;
    static constexpr int UNS = (P >= 32 || DISJ) ? 1 : 2;    // cp.async stages of the fused update
    // split mode (PRE): the A V_k rows are staged like the panels; two stages where they fit
    static constexpr int NSP = PRE ? (P < 32 ? 2 : K1PRE_NSP32) : 1;
    static constexpr int pipe = WARPS * 3 * DM<P>::TILE * NSP;   // V_k, V_{k-1} tiles + A V tile per warp
    static constexpr int scr = prologue_scratch<P>() + 2 * P * P;
    static constexpr int upd = UpdSmem<P, WARPS, UNS>::doubles;   // the update runs first, then the SpMM
#ifndef K1PRE_OVL
#define K1PRE_OVL 0
#endif
    // (split mode, p = 32, K1PRE_OVL: the prologue scratch overlays the pipeline, whose first tiles
    // are then issued after the prologue -- room for a second stage)
    static constexpr bool OVL = PRE && P >= 32 && K1PRE_OVL;
    static constexpr int region = OVL ? ((pipe > scr ? pipe : scr) > upd ? (pipe > scr ? pipe : scr) : upd)
                                      : DISJ ? pipe + scr + upd : ((pipe + scr > upd) ? pipe + scr : upd);
    static constexpr size_t bytes = sizeof(double) * (2 * DM<P>::FR + region + P * P + P);
};

// W = (A V_k) Tr_k - V_{k-1} (Tr_{k-1} C_{k-1}^T); ||A u_j||^2; V_k^T W.  The gathers of the SpMM
// are per lane (LP lanes x 16 B per row, each row summed in CSR order with fma); the three
// row-local products run as DMMA on the staged tiles.
//
// Latency structure: a warp walks its rows as a stream of row groups (RPW rows per warp
// instruction, TR/RPW groups per tile) with a software pipeline -- while the gathers of group
// q are in flight, the column indices and values of group q+1 and the row pointers of group
// q+2 are loaded.  The SpMM of the warp's first tile runs before the prologue (the Cholesky of
// the previous block's Gram), which only the epilogue needs.
template <int P, bool PRE = false>
__global__ void __launch_bounds__(K1DSmem<P, PRE>::WARPS * 32, P <= 16 ? 2 : 1) k1_dmma(K1Args a) {
    using D = DM<P>;
    // gather mapping: 32 bytes per lane and entry (256-bit loads) at p = 8 and 16 (config 2:
    // 108.8k -> 112.8k it/s; config 3: 86k -> 95k); 16 bytes at p = 32 (spills at 128 registers)
    using C = K1Gather<P>;
    using KS = K1DSmem<P, PRE>;
    constexpr int WARPS = K1DSmem<P, PRE>::WARPS, TR = D::TR, RS = D::RS, KC = D::KC, NC = D::NC, FR = D::FR;
    constexpr int VEC = C::VEC, LANES = C::LANES, LP = C::LP, RPW = C::RPW;
    constexpr int E = P * P + P;
    // CSR entries per gather batch: 7 at p = 8 (a 7-point stencil row in one batch, 28 doubles in
    // flight per lane at 128 registers; 8 spills), 4 at p = 16 / 32
    constexpr int CH = P <= 8 ? 7 : 4;
    constexpr int G = TR / RPW;   // row groups per tile
    DevState* st = a.st;
    unsigned long long* tr = trace_begin(st, TR_K1);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int fr = lane >> 2, fc = lane & 3;
    const int sub = lane % LP, rsub = lane / LP;
    const bool act = sub < LANES;
    const int c0 = sub * VEC;
    extern __shared__ __align__(16) double dynd1[];
    double* fT = dynd1;            // Tr_k
    double* fD = fT + FR;          // -(Tr_{k-1} C_{k-1}^T)
    double* pipe = fD + FR;
    double* scr = KS::OVL ? pipe : pipe + KS::pipe;
    double* sAcc = pipe + KS::region;
    // each CTA owns a contiguous slab of tiles (its warps interleave inside it), so the
    // gathers of neighbouring rows (stencil offsets +-1, +-nx) hit this SM's L1
    const long long ntiles = (a.n + TR - 1) / TR;
    const long long tpc = (ntiles + gridDim.x - 1) / gridDim.x;
    const long long cbeg = (long long)blockIdx.x * tpc, cend = cbeg + tpc < ntiles ? cbeg + tpc : ntiles;
    double* wb = pipe + warp * 3 * D::TILE;
    double* tA = wb + 2 * D::TILE;   // A V_k rows, then W rows
    const long long t0 = cbeg + warp, ts = WARPS;
    const long long my_tiles = t0 < cend ? (cend - 1 - t0) / ts + 1 : 0;
    const long long nq = my_tiles * G;   // row groups of this warp
    auto row_of = [&](long long q) -> long long {
        return (t0 + (q / G) * ts) * TR + (int)(q % G) * RPW + rsub;
    };
    // pipeline registers: row pointers of group q+1 (rn0, rn1); cols / values of group q
    int k0 = 0, k1 = 0, rn0 = 0, rn1 = 0;
    int cc[CH];
    double av[CH];
    auto load_rp = [&](long long q, int& r0, int& r1) {
        r0 = r1 = 0;
        if (q < nq) {
            const long long i = row_of(q);
            if (act && i < a.n) {
                r0 = __ldg(a.rowptr + i);
                r1 = __ldg(a.rowptr + i + 1);
            }
        }
    };
    auto load_cv = [&](int r0, int r1, int (&c)[CH], double (&v)[CH]) {
#pragma unroll
        for (int t = 0; t < CH; ++t) {
            const bool pr = r0 + t < r1;
            c[t] = pr ? __ldg(a.col + r0 + t) : -1;
            v[t] = pr ? __ldg(a.val + r0 + t) : 0.0;
        }
    };
    if constexpr (!PRE) {
        // the first row pointers / column indices of the SpMM (A only: no dependence on the update
        // or the wait) are in flight during the fused update
        load_rp(0, k0, k1);
        load_rp(1, rn0, rn1);
        load_cv(k0, k1, cc, av);
    }
    if (a.fuse) {
        // M/X update of block b = k-2 (row a5), on this CTA's slab before its W rows overwrite
        // V_b (same slot): it needs only K3b(b) and the panels, not the red2 totals, so it runs
        // before pdl_wait.  The condition reads state that K3b(k-1), running beside this
        // kernel, can change only in ways that leave it unchanged (uniform over CTAs).
        const long long k = st->k_main, b = k - 2;
        if (b >= st->k_upd_min && b < st->k_side && b < st->stop_side_at) {
            if (blockIdx.x == 0 && threadIdx.x == 0) st->upd_last = b;
            // X updates in pairs from the first fused block: defer b's, then apply both with b+1's
            const int xm = a.xdefer ? (((b - st->k_upd_min) & 1) ? 2 : 1) : 0;
            K4bArgs u{a.Y, a.Mk2, a.Mk1, a.Xs, a.n, st, (a.sk + 1) % 3, 0, a.par, 1, b, xm, b};
            if constexpr (KS::DISJ) {
                dmma_update<P, WARPS, KS::UNS>(u, cbeg, WARPS, cend, pipe + KS::pipe + KS::scr);
            } else {
                dmma_update<P, WARPS, KS::UNS>(u, cbeg, WARPS, cend, pipe);
                __syncthreads();   // the region is reused by the SpMM
            }
        }
    }
    trace_pt(tr, 1);
    // (the stopped-main-branch exit is taken after griddepcontrol.wait, where every CTA reads the
    // same run_main -- see publish_breakdown; the first SpMM tile below only reads V_k into
    // shared memory)
    const bool has_prev = st->k_main > 1;
    double g[NC][NC][2], om[NC][2];
#pragma unroll
    for (int i = 0; i < NC; ++i) {
        om[i][0] = om[i][1] = 0.0;
#pragma unroll
        for (int j = 0; j < NC; ++j) g[i][j][0] = g[i][j][1] = 0.0;
    }
    // group q: gathers (first CH entries) || loads of group q+1 || row pointers of q+2
    auto process_group = [&](long long q) {
        if (q % G == 0) {   // first group of a tile: stage the tile's V_k, V_{k-1} rows
            const long long base = (t0 + (q / G) * ts) * TR;
            stage_tile<P>(wb, a.X, base, a.n, lane);
            if (has_prev) stage_tile<P>(wb + D::TILE, a.Vprev, base, a.n, lane);
            cp_commit();
        }
        double xv[CH][VEC];
#pragma unroll
        for (int t = 0; t < CH; ++t) {
            if (cc[t] >= 0) {
                ldg_vec<VEC>(a.X + (long long)cc[t] * P + c0, xv[t]);
            } else {
#pragma unroll
                for (int v = 0; v < VEC; ++v) xv[t][v] = 0.0;
            }
        }
        const int gk0 = k0, gk1 = k1;
        k0 = rn0;
        k1 = rn1;
        int cn[CH];
        double an[CH];
        load_cv(k0, k1, cn, an);
        load_rp(q + 2, rn0, rn1);
        double acc[VEC];
#pragma unroll
        for (int v = 0; v < VEC; ++v) acc[v] = 0.0;
#pragma unroll
        for (int t = 0; t < CH; ++t)
            if (cc[t] >= 0) {
#pragma unroll
                for (int v = 0; v < VEC; ++v) acc[v] = fma(av[t], xv[t][v], acc[v]);
            }
        // rows longer than CH entries: the remaining chunks, in CSR order
        for (int kb = gk0 + CH; kb < gk1; kb += CH) {
            int c2[CH];
            double a2[CH];
            load_cv(kb, gk1, c2, a2);
#pragma unroll
            for (int t = 0; t < CH; ++t) {
                if (c2[t] >= 0) {
                    ldg_vec<VEC>(a.X + (long long)c2[t] * P + c0, xv[t]);
#pragma unroll
                    for (int v = 0; v < VEC; ++v) acc[v] = fma(a2[t], xv[t][v], acc[v]);
                }
            }
        }
#pragma unroll
        for (int t = 0; t < CH; ++t) {
            cc[t] = cn[t];
            av[t] = an[t];
        }
        if (act) {
            const int rl = (int)(q % G) * RPW + rsub;
#pragma unroll
            for (int v = 0; v < VEC; ++v) tA[rl * RS + c0 + v] = acc[v];
        }
    };
    // ---- the prologue: C_{k-1} (Cholesky of K2(k-1)'s W'^T W' partials), Tr_k, D
    auto prologue = [&]() -> bool {
        if (st->red2_fac && st->k_main > 1 && st->given_blk != st->k_main - 1) {
            // reduce2 factored the block: load Tr_k and -D in fragment order
            if (st->fac_bad) return false;   // (breakdown published by reduce2)
            for (int t = threadIdx.x; t < FR; t += blockDim.x) {
                fT[t] = st->fT[t];
                fD[t] = st->fD[t];
            }
            __syncthreads();
            return true;
        }
        double* sTk = scr;
        double* sD = scr + P * P;
        if (!k1_prologue<P>(st, a.par, a.sk, sTk, sD, scr + 2 * P * P)) return false;
        to_frag<P>(sTk, P, 1.0, fT);
        to_frag<P>(sD, P, -1.0, fD);
        __syncthreads();
        return true;
    };
    // ---- epilogue of tile `it`: tAV holds its A V_k rows (overwritten by its W rows), tV / tP its
    // V_k / V_{k-1} rows
    auto epilogue = [&](long long it, const double* tV, const double* tP, double* tAV) {
        const long long base = (t0 + it * ts) * TR;
#pragma unroll
        for (int mc = 0; mc < TR / 8; ++mc) {
            const int r0 = mc * 8;
            const long long row = base + r0 + fr;
            const bool rok = row < a.n;
            double w[NC][2];
#pragma unroll
            for (int nc = 0; nc < NC; ++nc) w[nc][0] = w[nc][1] = 0.0;
            // W = (A V_k) Tr_k = A U_k, the raw candidates; ||A u_j||^2 (C14).  Tr_k = C_{k-1}^{-1}
            // (or I) is upper triangular: k-chunks below the column block are zero.  k-chunks
            // outermost: one A-fragment load feeds every column block (per output the DMMAs still
            // accumulate in increasing kc, the Tr_k products before the D products)
#pragma unroll
            for (int kc = 0; kc < KC; ++kc) {
                const double aA = tAV[(r0 + fr) * RS + kc * 4 + fc];
#pragma unroll
                for (int nc = 0; nc < NC; ++nc)
                    if (kc <= 2 * nc + 1) dmma(w[nc][0], w[nc][1], aA, fT[(kc * NC + nc) * 32 + lane]);
            }
#pragma unroll
            for (int nc = 0; nc < NC; ++nc) {
                om[nc][0] = fma(w[nc][0], w[nc][0], om[nc][0]);
                om[nc][1] = fma(w[nc][1], w[nc][1], om[nc][1]);
            }
            // W -= U_{k-1} C_{k-1}^T = V_{k-1} D  (h_{i,j} = h_{j,i})
            if (has_prev) {
#pragma unroll
                for (int kc = 0; kc < KC; ++kc) {
                    const double aP = tP[(r0 + fr) * RS + kc * 4 + fc];
#pragma unroll
                    for (int nc = 0; nc < NC; ++nc) dmma(w[nc][0], w[nc][1], aP, fD[(kc * NC + nc) * 32 + lane]);
                }
            }
            __syncwarp();
#pragma unroll
            for (int nc = 0; nc < NC; ++nc) {
                const int col = nc * 8 + 2 * fc;
                tAV[(r0 + fr) * RS + col] = w[nc][0];
                tAV[(r0 + fr) * RS + col + 1] = w[nc][1];
                if (rok) *reinterpret_cast<double2*>(a.Y + row * P + col) = make_double2(w[nc][0], w[nc][1]);
            }
        }
        __syncwarp();
        // V_k^T W over the tile (rows past n are zero in both tiles)
#pragma unroll
        for (int k0 = 0; k0 < TR; k0 += 4) {
            const double* rv = tV + (k0 + fc) * RS;
            const double* rw = tAV + (k0 + fc) * RS;
#pragma unroll
            for (int i = 0; i < NC; ++i) {
                const double av = rv[i * 8 + fr];
#pragma unroll
                for (int j = 0; j < NC; ++j) dmma(g[i][j][0], g[i][j][1], av, rw[j * 8 + fr]);
            }
        }
        __syncwarp();
    };
    if constexpr (PRE) {
        // split mode: A V_k (k1a_spmm, the predecessor) is streamed like the panels -- NSP-deep
        // cp.async ring of {V_k, V_{k-1}, A V_k} tiles per warp
        constexpr int NSP = KS::NSP;
        double* wpre = pipe + warp * 3 * D::TILE * NSP;
        auto stage3 = [&](long long it) {
            if (it < my_tiles) {
                double* sl = wpre + (int)(it % NSP) * 3 * D::TILE;
                const long long base = (t0 + it * ts) * TR;
                stage_tile<P>(sl, a.X, base, a.n, lane);
                if (has_prev) stage_tile<P>(sl + D::TILE, a.Vprev, base, a.n, lane);
                stage_tile<P>(sl + 2 * D::TILE, a.AV, base, a.n, lane);
            }
            cp_commit();
        };
        pdl_wait();   // A V_k (k1a) and, through it, red2 of block k-1 are complete
        if (!st->run_main) return;
        if (blockIdx.x == 0 && threadIdx.x == 0) st->k1a_ctr[0] = st->k1a_ctr[1] = 0ull;   // for K1a(k+1)
        trace_pt(tr, 2);
        if constexpr (!KS::OVL) {
#pragma unroll
            for (int s = 0; s < NSP; ++s) stage3(s);   // the first tiles stream in during the prologue
        }
        if (!prologue()) {
            cp_wait<0>();
            return;
        }
        if constexpr (KS::OVL) {
#pragma unroll
            for (int s = 0; s < NSP; ++s) stage3(s);
        }
        trace_pt(tr, 3);
        for (long long it = 0; it < my_tiles; ++it) {
            cp_wait<NSP - 1>();
            __syncwarp();
            double* sl = wpre + (int)(it % NSP) * 3 * D::TILE;
            epilogue(it, sl, sl + D::TILE, sl + 2 * D::TILE);
            stage3(it + NSP);
        }
    } else {
        // (pipeline filled before the update) the SpMM of the first tile (no dependence on the
        // prologue)
        long long q = 0;
        for (; q < G && q < nq; ++q) process_group(q);
        pdl_wait();   // red2 (reduce2 of block k-1) is ready
        if (!st->run_main) {
            cp_wait<0>();
            return;
        }
        trace_pt(tr, 2);
        if (!prologue()) {
            cp_wait<0>();
            return;
        }
        trace_pt(tr, 3);
        for (long long it = 0; it < my_tiles; ++it) {
            if (it > 0)
                for (int gq = 0; gq < G; ++gq, ++q) process_group(q);
            cp_wait<0>();
            __syncwarp();
            epilogue(it, wb, wb + D::TILE, tA);
        }
    }
    cp_wait<0>();
    trace_pt(tr, 4);
    pdl_trigger();   // the dependent (reduce1) launches while this grid reduces its partials
    // om: sum over the 8 row-lanes that share a column pair
#pragma unroll
    for (int o = 4; o < 32; o <<= 1)
#pragma unroll
        for (int nc = 0; nc < NC; ++nc) {
            om[nc][0] += __shfl_xor_sync(FULL, om[nc][0], o);
            om[nc][1] += __shfl_xor_sync(FULL, om[nc][1], o);
        }
    if constexpr (WARPS * E <= K1DSmem<P>::pipe) {
        // one slot per warp in the (now idle) pipeline area, then a fixed-order sum over warps
        __syncthreads();
        double* slot = pipe + warp * E;
#pragma unroll
        for (int i = 0; i < NC; ++i)
#pragma unroll
            for (int j = 0; j < NC; ++j) frag_acc(slot, 0, P, i * 8, j * 8, g[i][j], true, lane);
        if (fr == 0) {
#pragma unroll
            for (int nc = 0; nc < NC; ++nc) {
                slot[P * P + nc * 8 + 2 * fc] = om[nc][0];
                slot[P * P + nc * 8 + 2 * fc + 1] = om[nc][1];
            }
        }
        __syncthreads();
        for (int e = threadIdx.x; e < E; e += blockDim.x) {
            double t = pipe[e];
            for (int w = 1; w < WARPS; ++w) t += pipe[w * E + e];
            sAcc[e] = t;
        }
    } else {
        for (int w = 0; w < WARPS; ++w) {
            if (warp == w) {
#pragma unroll
                for (int i = 0; i < NC; ++i)
#pragma unroll
                    for (int j = 0; j < NC; ++j) frag_acc(sAcc, 0, P, i * 8, j * 8, g[i][j], w == 0, lane);
                if (fr == 0) {
#pragma unroll
                    for (int nc = 0; nc < NC; ++nc) {
                        double* d = sAcc + P * P + nc * 8 + 2 * fc;
                        d[0] = (w == 0 ? 0.0 : d[0]) + om[nc][0];
                        d[1] = (w == 0 ? 0.0 : d[1]) + om[nc][1];
                    }
                }
            }
            __syncthreads();
        }
    }
    cluster_partials(sAcc, E, st->part1);   // reduce1, then K2 forms G = Tr_k^T (V_k^T W)
    trace_pt(tr, 5);
}

// ------------------------------------------------------------------ K1, warp-specialised (large panels)
//
// Row a1 for large panels (p in {16, 32}) in ONE kernel instead of K1a + K1<P, true>: per CTA,
// NPW producer warps run the SpMM gathers (A V_k, each row summed in CSR order with fma from 0 --
// bitwise K1a's rows) into a ring of NSLOT shared-memory tiles of T rows, and NCW consumer warps run
// the DMMA epilogue on them (W = (A V_k) Tr_k - V_{k-1} D, ||A u_j||^2, V_k^T W; per output the same
// DMMA order as K1<P, true>, so W is bitwise the split mode's), register-blocked 16 rows per warp.
// The A V_k panel never goes to HBM (split mode wrote it and read it back: 2 panels per block
// step), and the latency-bound gathers overlap the tensor-pipe-bound epilogue.  Producers and
// consumers hand tiles over with named barriers (FULL / EMPTY per slot, bar.arrive + bar.sync).
// Tiles are dealt round-robin over the CTAs, so all SMs sweep the rows together and the far
// stencil neighbours (z planes at config 4) are re-read from L2.
template <int P>
struct K1WS {
#ifndef K1WS_NPW
#define K1WS_NPW 8   // (12 producers: 128 registers per thread, the consumers spill -- config 4 9.2 ms)
#endif
    static constexpr int NPW = K1WS_NPW, NCW = 4;
    static constexpr int THREADS = (NPW + NCW) * 32;
    static constexpr int TRW = 16, MC = TRW / 8;       // rows per consumer warp (two DMMA row chunks)
    static constexpr int T = NCW * TRW;                // rows per CTA tile
    static constexpr int RS = P + 4;
    static constexpr int NSLOT = 3, NSC = 2;           // A V_k ring slots; consumer cp.async stages
    static constexpr int VEC = 4, LANES = P / VEC, RPW = 32 / LANES, CH = 8;
    static constexpr int FR = DM<P>::FR;
    static constexpr int ring = NSLOT * T * RS;
    static constexpr int stage = NCW * NSC * 2 * TRW * RS;   // V_k, V_{k-1} rows of each consumer warp
    static constexpr int scr = prologue_scratch<P>() + 2 * P * P;
    static constexpr int body = ring + stage > scr ? ring + stage : scr;
    static constexpr size_t bytes = sizeof(double) * (2 * FR + body + P * P + P);
};

__device__ __forceinline__ void named_sync(int id, int count) {
    asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int count) {
    asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}

template <int P>
__global__ void __launch_bounds__(K1WS<P>::THREADS, 1) k1_ws(K1Args a) {
    using S = K1WS<P>;
    using D = DM<P>;
    constexpr int NPW = S::NPW, NCW = S::NCW, TH = S::THREADS, TRW = S::TRW, MC = S::MC, T = S::T, RS = S::RS;
    constexpr int NSLOT = S::NSLOT, NSC = S::NSC, VEC = S::VEC, LANES = S::LANES, RPW = S::RPW, CH = S::CH;
    constexpr int KC = D::KC, NC = D::NC, FR = D::FR, E = P * P + P;
    constexpr int BAR_FULL = 1, BAR_EMPTY = 1 + NSLOT;
    DevState* st = a.st;
    unsigned long long* tr = trace_begin(st, TR_K1);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    extern __shared__ __align__(16) double dynws[];
    double* fT = dynws;             // Tr_k in fragment order
    double* fD = fT + FR;           // -(Tr_{k-1} C_{k-1}^T)
    double* ring = fD + FR;         // NSLOT x T x RS: A V_k rows, overwritten by W rows
    double* stg = ring + S::ring;   // consumer staging
    double* sAcc = fD + FR + S::body;
    pdl_wait();   // V_k (K2 of block k-1), the reduce2 totals / fragments, the update kernel are complete
    if (!st->run_main) return;
    trace_pt(tr, 2);
    const bool has_prev = st->k_main > 1;
    // ---- prologue (all threads): C_{k-1}, Tr_k, D (the scratch overlays the ring)
    {
        if (st->red2_fac && st->k_main > 1 && st->given_blk != st->k_main - 1) {
            if (st->fac_bad) return;
            for (int t = threadIdx.x; t < FR; t += blockDim.x) {
                fT[t] = st->fT[t];
                fD[t] = st->fD[t];
            }
        } else {
            double* sTk = ring;
            double* sD = ring + P * P;
            if (!k1_prologue<P>(st, a.par, a.sk, sTk, sD, ring + 2 * P * P)) return;
            to_frag<P>(sTk, P, 1.0, fT);
            to_frag<P>(sD, P, -1.0, fD);
        }
        __syncthreads();
    }
    trace_pt(tr, 3);
    const long long ntiles = (a.n + T - 1) / T;
    double g[NC][NC][2], om[NC][2];
#pragma unroll
    for (int i = 0; i < NC; ++i) {
        om[i][0] = om[i][1] = 0.0;
#pragma unroll
        for (int j = 0; j < NC; ++j) g[i][j][0] = g[i][j][1] = 0.0;
    }
    if (warp < NPW) {
        // ================= producers: A V_k rows of each tile into the ring.  A warp walks its row
        // groups (G per tile, tiles round-robin over the CTAs) as one stream with a software
        // pipeline: while group q's gathers are in flight, the column indices / values of group
        // q+1 and the row pointers of group q+2 are loaded (one dependent round trip per group
        // instead of three).  The slot's EMPTY barrier is taken just before the first store.
        const int sub = lane % LANES, rsub = lane / LANES;
        const int c0 = sub * VEC;
        constexpr int NG = T / RPW;   // row groups per tile
        const int G = warp < NG ? (NG - warp + NPW - 1) / NPW : 0;   // this warp's groups per tile
        const long long my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
        const long long nq = my_tiles * G;
        if (G == 0)   // (no rows in a tile: the barriers only)
            for (long long it = 0; it < my_tiles; ++it) {
                const int s = (int)(it % NSLOT);
                if (it >= NSLOT) named_sync(BAR_EMPTY + s, TH);
                named_arrive(BAR_FULL + s, TH);
            }
        auto row_of = [&](long long q) -> long long {
            const long long it = q / G;
            const int gi = (int)(q % G);
            return (blockIdx.x + it * gridDim.x) * T + (warp + gi * NPW) * RPW + rsub;
        };
        auto load_rp = [&](long long q, int& r0, int& r1) {
            r0 = r1 = 0;
            if (q < nq) {
                const long long i = row_of(q);
                if (i < a.n) {
                    r0 = __ldg(a.rowptr + i);
                    r1 = __ldg(a.rowptr + i + 1);
                }
            }
        };
        auto load_cv = [&](int r0, int r1, int (&c)[CH], double (&v)[CH]) {
#pragma unroll
            for (int t = 0; t < CH; ++t) {
                const bool pr = r0 + t < r1;
                c[t] = pr ? __ldg(a.col + r0 + t) : -1;
                v[t] = pr ? __ldg(a.val + r0 + t) : 0.0;
            }
        };
        int k0 = 0, k1 = 0, rn0 = 0, rn1 = 0;
        int cc[CH];
        double avv[CH];
        load_rp(0, k0, k1);
        load_rp(1, rn0, rn1);
        load_cv(k0, k1, cc, avv);
        for (long long q = 0; q < nq; ++q) {
            const long long it = q / G;
            const int gi = (int)(q % G);
            const int s = (int)(it % NSLOT);
            double xv[CH][VEC];
#pragma unroll
            for (int t = 0; t < CH; ++t) {
                if (cc[t] >= 0) {
                    ldg_vec<VEC>(a.X + (long long)cc[t] * P + c0, xv[t]);
                } else {
#pragma unroll
                    for (int v = 0; v < VEC; ++v) xv[t][v] = 0.0;
                }
            }
            const int gk0 = k0, gk1 = k1;
            k0 = rn0;
            k1 = rn1;
            int cn[CH];
            double an[CH];
            load_cv(k0, k1, cn, an);
            load_rp(q + 2, rn0, rn1);
            double acc[VEC];
#pragma unroll
            for (int v = 0; v < VEC; ++v) acc[v] = 0.0;
#pragma unroll
            for (int t = 0; t < CH; ++t)
                if (cc[t] >= 0) {
#pragma unroll
                    for (int v = 0; v < VEC; ++v) acc[v] = fma(avv[t], xv[t][v], acc[v]);
                }
            // rows longer than CH entries: the remaining chunks, in CSR order
            for (int kb = gk0 + CH; __any_sync(FULL, kb < gk1); kb += CH) {
                int c2[CH];
                double a2[CH];
                load_cv(kb, gk1, c2, a2);
#pragma unroll
                for (int t = 0; t < CH; ++t) {
                    if (c2[t] >= 0) {
                        ldg_vec<VEC>(a.X + (long long)c2[t] * P + c0, xv[t]);
#pragma unroll
                        for (int v = 0; v < VEC; ++v) acc[v] = fma(a2[t], xv[t][v], acc[v]);
                    }
                }
            }
#pragma unroll
            for (int t = 0; t < CH; ++t) {
                cc[t] = cn[t];
                avv[t] = an[t];
            }
            if (gi == 0 && it >= NSLOT) named_sync(BAR_EMPTY + s, TH);
            double* tl = ring + s * T * RS;
            const int rl = (warp + gi * NPW) * RPW + rsub;
#pragma unroll
            for (int v = 0; v < VEC; ++v) tl[rl * RS + c0 + v] = acc[v];   // (rows past n: zeros)
            if (gi == G - 1) named_arrive(BAR_FULL + s, TH);
        }
        // complete the EMPTY barriers of the last slots (every arrival gets its matching sync)
        for (long long q = my_tiles > NSLOT ? my_tiles - NSLOT : 0; q < my_tiles; ++q)
            named_sync(BAR_EMPTY + (int)(q % NSLOT), TH);
    } else {
        // ================= consumers: the DMMA epilogue on their 16 rows of each tile
        const int cw = warp - NPW;
        const int fr = lane >> 2, fc = lane & 3;
        double* wst = stg + cw * NSC * 2 * TRW * RS;
        auto issue = [&](long long itn) {
            const long long t = blockIdx.x + itn * gridDim.x;
            if (t < ntiles) {
                double* sl = wst + (int)(itn % NSC) * 2 * TRW * RS;
                const long long base = t * T + cw * TRW;
                stage_rows<P, TRW>(sl, a.X, base, a.n, lane);
                if (has_prev) stage_rows<P, TRW>(sl + TRW * RS, a.Vprev, base, a.n, lane);
            }
            cp_commit();
        };
#pragma unroll
        for (int q = 0; q < NSC - 1; ++q) issue(q);
        long long it = 0;
        for (long long t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
            issue(it + NSC - 1);
            cp_wait<NSC - 1>();
            __syncwarp();
            const int s = (int)(it % NSLOT);
            named_sync(BAR_FULL + s, TH);
            const double* tV = wst + (int)(it % NSC) * 2 * TRW * RS;
            const double* tP = tV + TRW * RS;
            double* tW = ring + s * T * RS + cw * TRW * RS;   // A V_k rows in, W rows out
            const long long base = t * T + cw * TRW;
            double w[MC][NC][2];
#pragma unroll
            for (int mc = 0; mc < MC; ++mc)
#pragma unroll
                for (int nc = 0; nc < NC; ++nc) w[mc][nc][0] = w[mc][nc][1] = 0.0;
            // W = (A V_k) Tr_k (Tr_k upper triangular: k-chunks below the column block are zero)
#pragma unroll
            for (int kc = 0; kc < KC; ++kc) {
                double av[MC];
#pragma unroll
                for (int mc = 0; mc < MC; ++mc) av[mc] = tW[(mc * 8 + fr) * RS + kc * 4 + fc];
#pragma unroll
                for (int nc = 0; nc < NC; ++nc)
                    if (kc <= 2 * nc + 1) {
                        const double b = fT[(kc * NC + nc) * 32 + lane];
#pragma unroll
                        for (int mc = 0; mc < MC; ++mc) dmma(w[mc][nc][0], w[mc][nc][1], av[mc], b);
                    }
            }
            // ||A u_j||^2 (C14)
#pragma unroll
            for (int mc = 0; mc < MC; ++mc)
#pragma unroll
                for (int nc = 0; nc < NC; ++nc) {
                    om[nc][0] = fma(w[mc][nc][0], w[mc][nc][0], om[nc][0]);
                    om[nc][1] = fma(w[mc][nc][1], w[mc][nc][1], om[nc][1]);
                }
            // W -= U_{k-1} C_{k-1}^T = V_{k-1} D (h_{i,j} = h_{j,i})
            if (has_prev) {
#pragma unroll
                for (int kc = 0; kc < KC; ++kc) {
                    double ap[MC];
#pragma unroll
                    for (int mc = 0; mc < MC; ++mc) ap[mc] = tP[(mc * 8 + fr) * RS + kc * 4 + fc];
#pragma unroll
                    for (int nc = 0; nc < NC; ++nc) {
                        const double b = fD[(kc * NC + nc) * 32 + lane];
#pragma unroll
                        for (int mc = 0; mc < MC; ++mc) dmma(w[mc][nc][0], w[mc][nc][1], ap[mc], b);
                    }
                }
            }
            __syncwarp();
#pragma unroll
            for (int mc = 0; mc < MC; ++mc) {
                const long long row = base + mc * 8 + fr;
#pragma unroll
                for (int nc = 0; nc < NC; ++nc) {
                    const int col = nc * 8 + 2 * fc;
                    tW[(mc * 8 + fr) * RS + col] = w[mc][nc][0];
                    tW[(mc * 8 + fr) * RS + col + 1] = w[mc][nc][1];
                    if (row < a.n) *reinterpret_cast<double2*>(a.Y + row * P + col) = make_double2(w[mc][nc][0], w[mc][nc][1]);
                }
            }
            __syncwarp();
            // V_k^T W over the warp's rows (rows past n are zero in both tiles)
#pragma unroll
            for (int k0 = 0; k0 < TRW; k0 += 4) {
                const double* rv = tV + (k0 + fc) * RS;
                const double* rw = tW + (k0 + fc) * RS;
                double bw[NC];
#pragma unroll
                for (int j = 0; j < NC; ++j) bw[j] = rw[j * 8 + fr];
#pragma unroll
                for (int i = 0; i < NC; ++i) {
                    const double av = rv[i * 8 + fr];
#pragma unroll
                    for (int j = 0; j < NC; ++j) dmma(g[i][j][0], g[i][j][1], av, bw[j]);
                }
            }
            __syncwarp();
            named_arrive(BAR_EMPTY + s, TH);
        }
        cp_wait<0>();
    }
    trace_pt(tr, 4);
    pdl_trigger();   // the dependent (reduce1) launches while this grid reduces its partials
    __syncthreads();
    if (warp >= NPW) {
        // om: sum over the 8 row-lanes that share a column pair
#pragma unroll
        for (int o = 4; o < 32; o <<= 1)
#pragma unroll
            for (int nc = 0; nc < NC; ++nc) {
                om[nc][0] += __shfl_xor_sync(FULL, om[nc][0], o);
                om[nc][1] += __shfl_xor_sync(FULL, om[nc][1], o);
            }
    }
    // consumer warps in fixed order -> sAcc (the ring is idle now)
    for (int w2 = NPW; w2 < NPW + NCW; ++w2) {
        if (warp == w2) {
#pragma unroll
            for (int i = 0; i < NC; ++i)
#pragma unroll
                for (int j = 0; j < NC; ++j) frag_acc(sAcc, 0, P, i * 8, j * 8, g[i][j], w2 == NPW, lane);
            if ((lane >> 2) == 0) {
#pragma unroll
                for (int nc = 0; nc < NC; ++nc) {
                    double* d = sAcc + P * P + nc * 8 + 2 * (lane & 3);
                    d[0] = (w2 == NPW ? 0.0 : d[0]) + om[nc][0];
                    d[1] = (w2 == NPW ? 0.0 : d[1]) + om[nc][1];
                }
            }
        }
        __syncthreads();
    }
    cluster_partials(sAcc, E, st->part1);   // reduce1, then K2 forms G = Tr_k^T (V_k^T W)
    trace_pt(tr, 5);
}

}  // namespace bmr
