// common.cuh -- shared definitions of the B200 block-MINRES hot path.
//
// Paper: Soodhalter, arXiv:1301.2102.  "P:L" = PAPER.md line L.
// Block form of one block step k (iterations j = (k-1)p+1 .. kp; DESIGN.md
// "Block form"):  A U_k = U_{k-1} C_{k-1}^T + U_k G_s + U_{k+1} C_k, i.e. the
// paper's banded recurrence (eqn.block-Lanczos-recurr) with the
// operator applied to p vectors every p iterations and the known
// coefficients reused by symmetry.
//
// Two branches per block:
//   main  K1 (SpMM+epilogue) -> K2 (orthogonalise, Grams, Cholesky = C_k)
//   side  K3b (banded QR, z_j, residuals, stop) -> K4b (M_k, X)
// The side branch of block k runs concurrently with the main branch of block k+1.
// The basis is never normalised in memory: U_k = V_k Tr_k row by row, where V_k is the
// orthogonalised candidate block W'_{k-1} and Tr_k = C_{k-1}^{-1} (SURVEY design D2), or
// V_k = U_k, Tr_k = I after the column path / for the start block.
#pragma once
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace bmr {

namespace cg = cooperative_groups;

constexpr int MAXP = 32;      // largest compiled block size
constexpr int MAXQ = 8;       // largest replacement pool
constexpr int NB_MAX = 1024;  // largest grid of the reducing kernels
constexpr int CL = 8;         // thread-block cluster size of the reducing kernels
constexpr int NT = 256;       // threads of the panel kernels
constexpr long long KINF = 1ll << 62;
constexpr unsigned FULL = 0xffffffffu;

// Panel-row mapping of a warp: a row of p doubles is split over LANES lanes of VEC
// contiguous doubles (16 B when VEC = 2); RPW rows per warp instruction.
template <int P>
struct PC {
    static constexpr int VEC = (P % 2 == 0) ? 2 : 1;
    static constexpr int LANES = P / VEC;
    static constexpr int LP = LANES <= 1 ? 1 : LANES <= 2 ? 2 : LANES <= 4 ? 4 : LANES <= 8 ? 8 : LANES <= 16 ? 16 : 32;
    static constexpr int RPW = 32 / LP;
    // shared-memory row stride: p + 2 doubles (p + 1 for odd p) so that the RPW rows a warp
    // reads in one instruction fall on distinct banks, keeping 16-byte alignment for cp.async
    static constexpr int RS = P + (VEC == 2 ? 2 : 1);
};

// Mapped (pinned, host-visible) flags the kernels publish; the host polls them.
struct HostFlags {
    volatile int side_done;      // the solve ended (converged / maxit / error)
    volatile int status;
    volatile int need_slow;      // the main branch stopped at block bd_at (breakdown / guard)
    volatile int pad;
    volatile long long bd_at;
    volatile long long j_done;
    volatile long long k_side;
    volatile long long k_main;
    volatile long long stop_blk;   // the block whose K3b ended the solve (side_done)
};

// Device-resident solver state.  p x p matrices are row-major [a*MAXP + b].
struct DevState {
    // ---- main branch (K1, K2, K4a)
    int run_main;       // main-branch kernels run
    int need_slow;      // breakdown or Cholesky cancellation at block bd_at (K1 or K3b)
    int ncl1, ncl2;     // cluster partials written by K1 / K2
    long long given_blk;   // block whose C_k, Tr_{k+1}, coef_k the host supplied (column path)
    int q_first;        // first live pool vector
    int q_live;         // number of live pool vectors
    int pool_cap;       // pool panel row stride
    long long k_main;   // block of the next K1/K2
    long long bd_at;    // block with a pending breakdown (KINF: none)
    // ---- side branch (K3b, K4b)
    int side_go;        // K3b -> K4b: apply this block's update
    int status;         // BMINRES_* (1 while running)
    int stop_after;     // >0: K3b stops after block column stop_after-1 (pool exhausted)
    int pad0;
    long long k_side;        // block of the next K3b
    long long stop_side_at;  // side kernels of blocks >= this are no-ops
    long long j_done;        // completed iterations
    long long maxit;
    long long hist_cap;
    double tol, tau;
    unsigned cnt1, cnt2, cnt3, cnt4;   // tickets (cnt2: k_red2f's last CTA)
    // K1a chunk counters (split mode, dynamic chunk order; [1]: the boundary launch of a row
    // partition), reset by K1(k) -- which runs after K1a(k) completes -- for K1a(k+1)
    unsigned long long k1a_ctr[2];
    // k_red2f (single rank): reduce2's last CTA factors the new block once -- C_k, Tr_{k+1},
    // coef_k in the state, and K1(k+1)'s fragments of Tr_{k+1} and -(Tr_k C_k^T) below; fac_bad:
    // breakdown / cancellation of the block (published as by K1's own prologue)
    int red2_fac, fac_bad;
    long long fac_blk;   // the block whose C_k (Ck[k & 1]) / fac_bad reduce2 (or k_fac2) last stored
    // block-size reduction ("shrink", policy 1): lane m of every block
    // >= absent_from[m] holds a removed (zero) basis vector -- A 0 = 0, so a removed lane stays
    // removed; KINF: present.  The block form keeps p columns; removed ones are zero.
    int policy;
    int pad_policy;
    long long absent_from[MAXP];
    double fT[MAXP * MAXP], fD[MAXP * MAXP];
    // ---- written by the main branch, double-buffered by block parity
    double G[2][MAXP * MAXP];      // G(a,m) = u_{(k-1)p+a}^T w_m (K1, after the known subtraction)
    double om2[2][MAXP];           // ||A u_j||^2, raw candidate norms (C14)
    double Ck[2][MAXP * MAXP];     // C_k: W' = U_{k+1} C_k (upper triangular)
    double Tr[3][MAXP * MAXP];     // Tr_k (slot k mod 3): U_k = V_k Tr_k
    double coef[2][MAXP * MAXQ];   // coef(a,q) = u_{kp+a}^T r_q, applied to the pool by K2(k+1)
    double Gram2[MAXP * MAXP];     // W'^T W' (K2 only)
    double pdot[MAXQ * MAXP];      // pdot(q,m) = r_q^T w'_m (K2 only)
    // ---- side-branch state
    double CprevS[MAXP * MAXP];    // C_{k-1} for the Hessenberg assembly
    double T[MAXP * MAXP];         // tail of \bar Z (rows j..j+p-1), T(r,c)
    // K3b(k) outputs for the M/X update of block k, double-buffered by block parity (the update
    // of block k runs in K1(k+2), beside K3b(k+1))
    double Z[2][MAXP * MAXP];      // Z_k: row m = z_{(k-1)p+m+1}^T (rows past the stop are 0)
    double Zh[3][MAXP * MAXP];     // Z_k again, slot k mod 3 (the deferred X update of block k-1
                                   // runs in K1(k+2) beside K3b(k+1))
    // the M/X update's DMMA factors in fragment order (p = 8, 16, 32), written by K3b(k): by block
    // parity Tr_k R_kk^{-1}, -R_{k-2,k}R_kk^{-1}, -R_{k-1,k}R_kk^{-1}; Z_k by k mod 3
    double uf[2][3][MAXP * MAXP];
    double ufz[3][MAXP * MAXP];
    double Ainv[2][MAXP * MAXP];   // R_kk^{-1}
    double B1[2][MAXP * MAXP];     // R_{k-1,k} R_kk^{-1}
    double B2[2][MAXP * MAXP];     // R_{k-2,k} R_kk^{-1}
    long long k_upd_min;           // fused updates (K1(k) applies block k-2's) only for blocks >= this
    long long upd_last;            // last block whose M/X update was applied
    // accumulated Householder: Qacc[b & 1] = H_{bp} ... H_{(b-1)p+1}
    // restricted to the block's 2p rows (b-1)p+1 .. (b+1)p, row-major with ld 2 MAXP
    double Qacc[2][(2 * MAXP) * (2 * MAXP)];
    double beta[MAXP];             // ||b_i||
    double res[MAXP];              // latest computed relative residuals
    double* hist;                  // (hist_cap) x p computed relative residuals, or null
    HostFlags* hflags;             // device alias of the mapped host flags
    double* part1;                 // K1 cluster partials: ncl1 x (p*p + p)
    double* part2[2];              // K2 cluster partials by block parity: ncl2 x (p*p + q*p)
    double red1[MAXP * MAXP + MAXP];            // totals of part1: V_k^T W (p*p), ||A u_j||^2 (p)
    double red2[2][MAXP * MAXP + MAXQ * MAXP];  // totals of part2 by parity: W'^T W' (p*p), r_q^T W'
    // ---- timeline tracing (tooling; null when off): %globaltimer stamps of launch number
    // trace_launch of each kernel type, per CTA, TRACE_PTS points (see trace_begin)
    unsigned long long* trace;
    unsigned* trace_tick;
    long long trace_launch;
};

// lanes whose basis vector of block blk was removed (shrink policy), bit m = lane m
__device__ __forceinline__ unsigned absent_mask(const DevState* st, long long blk, int P) {
    unsigned m = 0u;
    if (st->policy == 1)
        for (int l = 0; l < P; ++l)
            if (st->absent_from[l] <= blk) m |= 1u << l;
    return m;
}

// kernel types of the trace buffer
enum TraceKind { TR_K1 = 0, TR_RED1, TR_K2, TR_RED2, TR_K3B, TR_K4B, TR_K1A, TR_NKIND };
constexpr int TRACE_PTS = 8;
constexpr int TRACE_CTAS = 1024;

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// thread 0 of each CTA: the stamp row of this CTA if this launch is the traced one, else null
__device__ __forceinline__ unsigned long long* trace_begin(const DevState* st, int kind) {
    if (st->trace == nullptr || threadIdx.x != 0) return nullptr;
    const unsigned t = atomicAdd(st->trace_tick + kind, 1u);
    if ((long long)(t / gridDim.x) != st->trace_launch || blockIdx.x >= TRACE_CTAS) return nullptr;
    unsigned long long* r = st->trace + ((size_t)kind * TRACE_CTAS + blockIdx.x) * TRACE_PTS;
    r[0] = gtimer();
    return r;
}
__device__ __forceinline__ void trace_pt(unsigned long long* r, int pt) {
    if (r) r[pt] = gtimer();
}

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
// coherent load (data written by a previous kernel that this kernel also writes)
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

// cp.async (LDGSTS) helpers: src-size 0 zero-fills the destination without reading src
__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc, bool pred) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
    const int nb = pred ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gsrc), "r"(nb) : "memory");
}
__device__ __forceinline__ void cp_async8(void* sdst, const void* gsrc, bool pred) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
    const int nb = pred ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gsrc), "r"(nb) : "memory");
}
template <int VEC>
__device__ __forceinline__ void cp_async_vec(double* sdst, const double* gsrc, bool pred) {
    if constexpr (VEC == 2)
        cp_async16(sdst, gsrc, pred);
    else
        cp_async8(sdst, gsrc, pred);
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// ---- TMA bulk copies (cp.async.bulk, SASS UBLKCP) and mbarriers (1-D: contiguous panel rows)
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// global -> shared, completion counted on bar (bytes: multiple of 16, both addresses 16-aligned)
__device__ __forceinline__ void bulk_g2s(void* sdst, const void* gsrc, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(sdst)),
                 "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
// shared -> global (bulk group)
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, unsigned bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(gdst), "r"(smem_u32(ssrc)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(N) : "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait() { asm volatile("cp.async.bulk.wait_group %0;\n" ::"n"(N) : "memory"); }
// generic-proxy shared-memory writes -> visible to the async proxy (before a bulk store reads them)
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// ---- Programmatic dependent launch (PDL).  A kernel launched with programmatic stream
// serialization may start while its predecessor drains; pdl_wait() blocks until the predecessor
// has completed and its memory is visible.  Work before pdl_wait() may only read data of kernels
// that completed before the predecessor started.  Both are no-ops without the launch attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}
// Deterministic butterfly reduce-scatter of 64 per-lane values over a warp (62 shuffles instead
// of 64 x 5): on return, v[0] and v[1] of lane l hold the warp totals of entries 2l and 2l+1.
__device__ __forceinline__ void warp_reduce_scatter64(double (&v)[64]) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int lvl = 0; lvl < 5; ++lvl) {
        const int o = 16 >> lvl, half = 32 >> lvl;
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < half; ++i) {
            const double keep = up ? v[half + i] : v[i];
            const double send = up ? v[i] : v[half + i];
            v[i] = keep + __shfl_xor_sync(FULL, send, o);
        }
    }
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(FULL, v, o));
    return v;
}

// Cluster partials.  Every CTA of a reducing panel kernel ends with its sums in shared memory
// sAcc[E].  The CTAs of a thread-block cluster are combined through distributed shared memory
// by the cluster's rank-0 CTA (fixed rank order), which writes one partial row
// part[cluster_id*E .. +E).  There is no last-CTA step: every CTA of the consuming kernel
// reduces the rows with k_reduce (many CTAs in parallel; a single last-CTA tail measured slower).
__device__ __forceinline__ void cluster_partials(const double* sAcc, int E, double* part) {
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    const int csz = (int)cl.num_blocks();
    if (cl.block_rank() == 0) {
        const int cid = blockIdx.x / csz;
        for (int e = threadIdx.x; e < E; e += blockDim.x) {
            double s = 0.0;
            for (int r = 0; r < csz; ++r) s += cl.map_shared_rank(sAcc, r)[e];
            part[(size_t)cid * E + e] = s;
        }
    }
    cl.sync();  // remote shared memory must outlive the leader's reads
}

// The totals of one set of cluster partials: one warp per entry, lanes stride over the partial
// rows, a fixed shuffle tree -> deterministic.  which = 1: part1 -> red1; which = 2: part2[par]
// -> red2[par].  Entry counts come from the state (q_live may change between launches).  Launched
// with PDL after K1 / K2.  reduce1 triggers its dependent at exit; reduce2 (early = 1) right after
// its wait -- K1(k+1)'s pre-wait work (the fused update, the first SpMM tile) reads only panels of
// kernels that have completed, K2(k) included, and its griddepcontrol.wait covers the totals.
__global__ void __launch_bounds__(256) k_reduce(DevState* st, int which, int par, int P, int early) {
    unsigned long long* tr = trace_begin(st, which == 1 ? TR_RED1 : TR_RED2);
    pdl_wait();
    // early: the dependent launches now -- its pre-wait work (K1's fused update and first SpMM
    // tile) reads only panels of kernels that have completed (the producer of these partials
    // included), and it waits for the totals at its own griddepcontrol.wait
    if (early) pdl_trigger();
    trace_pt(tr, 1);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int e = blockIdx.x * 8 + warp;
    if (!st->run_main) return;
    const int E = which == 1 ? P * P + P : P * P + st->q_live * P;
    const int ncl = which == 1 ? st->ncl1 : st->ncl2;
    const double* part = which == 1 ? st->part1 : st->part2[par];
    double* out = which == 1 ? st->red1 : st->red2[par];
    if (e >= E) return;
    // all of a lane's rows are loaded before the first add (one L2 round trip, not ncl/32);
    // the sum order is unchanged: b = lane, lane + 32, ... then the fixed shuffle tree
    constexpr int U = 8;   // rows per lane in flight (ncl <= 256 in one round: cluster size >= 2)
    double s = 0.0;
    for (int b0 = 0; b0 < ncl; b0 += 32 * U) {
        double v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int b = b0 + lane + 32 * u;
            v[u] = b < ncl ? __ldcg(part + (size_t)b * E + e) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (b0 + lane + 32 * u < ncl) s += v[u];
    }
    s = warp_sum(s);
    if (lane == 0) out[e] = s;
    trace_pt(tr, 5);
}

// Cholesky W'^T W' = C^T C of the new block (right-looking, warp 0), the breakdown /
// cancellation test (h_{j+p,j}^2 = pivot <= tau^2 ||A u_j||^2; pivot < 1e-4 of
// ||w'_m||^2 -> column path, R2), C^{-1} and the pool coefficients
// coef(:,q) = C^{-T} (W'^T r_q) = U_{k+1}^T r_q.  Inputs in shared memory: sG (Gram, ld P,
// destroyed), sOm (p), sPd (q x p).  Outputs: sC (ld P), sCi (ld P), sCo (P x MAXQ).
// Returns true on breakdown.  Identical in every CTA that calls it.  All threads call it.
//
// Latency: this sits on the critical path of every block step (K1's prologue, K3b), so the
// serial chain has no divisions and no square roots: one rsqrt per pivot (r_m = 1/C(m,m),
// C(m,m) = d r_m), and the inverse is built row by row inside the same loop -- with L = C^T,
// row m of L^{-1} = (e_m - sum_{i<m} L(m,i) L^{-1}(i,:)) r_m needs only rows < m of C.
template <int P>
__device__ bool factor_block(double* sG, const double* sOm, const double* sPd, int Q, double tau, double* sC,
                             double* sCi, double* sCo, unsigned amask = 0u) {
    // amask (shrink policy): lanes whose candidate is a removed (zero) vector.  Their pivot is a
    // placeholder 1 (C' = C + e_m e_m^T, so Tr = C'^{-1} keeps the zero column zero) and no
    // dependence test applies; sC returns the true C (diagonal 0 there: h_{j+p,j} = 0)
    __shared__ int s_bad;
    const int tid = threadIdx.x, lane = tid & 31;
    if constexpr (P <= 16) {
        // register version: lane j < P holds column j of the Gram (fully unrolled, the
        // trailing update takes C(m, i) from lane i by shuffle)
        if (tid < 32) {
            const double tau2 = tau * tau;
            const bool own = lane < P;
            double g[P];
#pragma unroll
            for (int i = 0; i < P; ++i) g[i] = own ? sG[i * P + lane] : 0.0;
            const double d0 = own ? sG[lane * P + lane] : 0.0;
            double cm[P], rr[P];
            bool bad = false;
#pragma unroll
            for (int m = 0; m < P; ++m) {
                const bool gone = (amask >> m) & 1u;
                const double dm = gone ? 1.0 : __shfl_sync(FULL, g[m], m);
                const double d0m = __shfl_sync(FULL, d0, m);
                if (!gone && (!(dm > tau2 * sOm[m]) || !(dm >= 1e-4 * d0m))) {
                    bad = true;
                    break;
                }
                const double r = rsqrt(dm);
                rr[m] = r;
                const double cmj = lane > m ? g[m] * r : (lane == m ? dm * r : 0.0);
                cm[m] = cmj;
#pragma unroll
                for (int i = m + 1; i < P; ++i) g[i] = fma(-__shfl_sync(FULL, cmj, i), cmj, g[i]);
            }
            if (lane == 0) s_bad = bad;
            if (!bad) {
                if (own)
#pragma unroll
                    for (int m = 0; m < P; ++m) sC[m * P + lane] = cm[m];
                __syncwarp();
                // C^{-1}(:, l) by back substitution, lane l (x(c) = 0 for c > l)
                double x[P];
#pragma unroll
                for (int r = P - 1; r >= 0; --r) {
                    double s = (r == lane) ? 1.0 : 0.0;
#pragma unroll
                    for (int c = r + 1; c < P; ++c) s = fma(-sC[r * P + c], x[c], s);
                    x[r] = (r <= lane) ? s * rr[r] : 0.0;
                }
                if (own)
#pragma unroll
                    for (int r = 0; r < P; ++r) sCi[r * P + lane] = x[r];
                for (int t = lane; t < P * MAXQ; t += 32) sCo[t] = 0.0;
                __syncwarp();
                if (own && ((amask >> lane) & 1u)) sC[lane * P + lane] = 0.0;   // the true C
                __syncwarp();
                for (int t = lane; t < P * Q; t += 32) {
                    const int m = t % P, q = t / P;
                    double s = 0.0;
                    for (int c = 0; c <= m; ++c) s = fma(sCi[c * P + m], sPd[q * P + c], s);
                    sCo[m * MAXQ + q] = s;
                }
            }
        }
        __syncthreads();
        return s_bad != 0;
    }
    if (tid < 32) {
        for (int t = lane; t < P * P; t += 32) {
            sC[t] = 0.0;
            sCi[t] = 0.0;
        }
        for (int t = lane; t < P * MAXQ; t += 32) sCo[t] = 0.0;
        const double tau2 = tau * tau;
        double d0[(P + 31) / 32];   // the pivots before elimination (cancellation guard)
#pragma unroll
        for (int u = 0; u < (P + 31) / 32; ++u) d0[u] = (lane + 32 * u < P) ? sG[(lane + 32 * u) * (P + 1)] : 0.0;
        __syncwarp();
        bool bad = false;
        for (int m = 0; m < P; ++m) {
            const bool gone = (amask >> m) & 1u;
            const double d = gone ? 1.0 : sG[m * P + m];
            const double dm0 = __shfl_sync(FULL, d0[m / 32], m % 32);
            if (!gone && (!(d > tau2 * sOm[m]) || !(d >= 1e-4 * dm0))) {
                bad = true;
                break;
            }
            const double r = rsqrt(d);   // 1 / C(m,m)
            for (int c = m + lane; c < P; c += 32) sC[m * P + c] = (c == m) ? d * r : sG[m * P + c] * r;
            // C^{-1}(c, m) = L^{-1}(m, c), c <= m
            for (int c = lane; c <= m; c += 32) {
                double s = (c == m) ? 1.0 : 0.0;
                for (int i = c; i < m; ++i) s = fma(-sC[i * P + m], sCi[c * P + i], s);
                sCi[c * P + m] = s * r;
            }
            __syncwarp();
            for (int t = lane; t < P * P; t += 32) {
                const int i = t / P, j = t % P;
                if (i > m && j >= i) sG[i * P + j] = fma(-sC[m * P + i], sC[m * P + j], sG[i * P + j]);
            }
            __syncwarp();
        }
        if (lane == 0) s_bad = bad;
        // coef(:, q) = C^{-T} pd(q, :): coef(m, q) = sum_{c <= m} C^{-1}(c, m) pd(q, c)
        if (!bad)
            for (int t = lane; t < P * Q; t += 32) {
                const int m = t % P, q = t / P;
                double s = 0.0;
                for (int c = 0; c <= m; ++c) s = fma(sCi[c * P + m], sPd[q * P + c], s);
                sCo[m * MAXQ + q] = s;
            }
        __syncwarp();
        if (!bad)
            for (int m = lane; m < P; m += 32)
                if ((amask >> m) & 1u) sC[m * P + m] = 0.0;   // the true C
    }
    __syncthreads();
    return s_bad != 0;
}

// The main branch has stopped (breakdown of a block, run_main = 0): K2 still advances k_main, so
// the K1 launches still in flight compute later blocks and never re-apply the fused M/X update
// of a block that has been applied (their update condition b < k_side then fails).
__device__ __forceinline__ void k2_stopped(DevState* st) {
    if (blockIdx.x == 0 && threadIdx.x == 0) st->k_main = st->k_main + 1;
}

// Publish a breakdown of block b (main branch stops; the host runs the column path).
//
// run_main is cleared only by main-branch kernels (reduce2's factorisation, K1's prologue), so every
// main-branch kernel reads it after griddepcontrol.wait with its predecessors complete and all CTAs
// of a launch see the same value -- the CTAs of a cluster must take the same early exit, since a
// reducing kernel's leader reads its peers' shared memory in cluster_partials.  K3b (side stream)
// reports its breakdowns to the host only (side_only): had it cleared run_main, the flag could
// change between two CTAs' reads of one launch, and a cluster split that way read an exited CTA's
// shared memory ("unspecified launch failure": p = 8 with K1 / K3b factoring, BMINRES_NO_RED2F, a
// mid-solve dependence; test_reduce2_factorisation_reused_bitwise).
__device__ __forceinline__ void publish_breakdown(DevState* st, long long b, bool side_only = false) {
    st->need_slow = 1;
    if (!side_only) st->run_main = 0;
    st->bd_at = b;
    st->hflags->bd_at = b;
    st->hflags->need_slow = 1;
    __threadfence_system();
}

// C = A B (transB: C = A B^T) for P x P row-major in shared memory, all threads of the CTA.
template <int P>
__device__ __forceinline__ void smm_nn(const double* Am, const double* Bm, double* Cm, bool transB = false) {
    for (int t = threadIdx.x; t < P * P; t += blockDim.x) {
        const int r = t / P, c = t % P;
        double s = 0.0;
        for (int i = 0; i < P; ++i) s = fma(Am[r * P + i], transB ? Bm[c * P + i] : Bm[i * P + c], s);
        Cm[r * P + c] = s;
    }
}
// C = A^T B
template <int P>
__device__ __forceinline__ void smm_tn(const double* Am, const double* Bm, double* Cm) {
    for (int t = threadIdx.x; t < P * P; t += blockDim.x) {
        const int r = t / P, c = t % P;
        double s = 0.0;
        for (int i = 0; i < P; ++i) s = fma(Am[i * P + r], Bm[i * P + c], s);
        Cm[r * P + c] = s;
    }
}
// shared <- global P x P block with leading dimension MAXP
template <int P>
__device__ __forceinline__ void load_pp(double* dst, const double* src) {
    for (int t = threadIdx.x; t < P * P; t += blockDim.x) dst[t] = src[(t / P) * MAXP + t % P];
}
template <int P>
__device__ __forceinline__ void store_pp(double* dst, const double* src) {
    for (int t = threadIdx.x; t < P * P; t += blockDim.x) dst[(t / P) * MAXP + t % P] = src[t];
}

// Scratch (doubles) the K1 / K2 prologues need: K1's is the largest -- totals (P*P + MAXQ*P),
// C, C^{-1}, Tr_{k-1} (3 P*P), pool coefficients (P*MAXQ), ||A u_j||^2 (P).
template <int P>
__host__ __device__ constexpr int prologue_scratch() { return (P * P + MAXQ * P) + 3 * P * P + P * MAXQ + P; }

// K1 prologue, block k: C_{k-1}, Tr_k = C_{k-1}^{-1}, coef_{k-1} from K2(k-1)'s partials (or the
// host's values after the column path), and D = Tr_{k-1} C_{k-1}^T.  Writes sTk and sD (P x P,
// ld P).  Returns false when the CTA must exit (breakdown of block k-1, published by CTA 0).
template <int P>
__device__ bool k1_prologue(DevState* st, int par, int sk, double* sTk, double* sD, double* scr) {
    const long long k = st->k_main;
    if (k <= 1) {
        for (int t = threadIdx.x; t < P * P; t += blockDim.x) {
            sTk[t] = (t / P == t % P) ? 1.0 : 0.0;
            sD[t] = 0.0;
        }
        __syncthreads();
        return true;
    }
    double* sRed = scr;                          // Gram (P*P) + pool dots (MAXQ*P)
    double* sC = sRed + P * P + MAXQ * P;
    double* sCi = sC + P * P;
    double* sTp = sCi + P * P;
    double* sCo = sTp + P * P;
    double* sOm = sCo + P * MAXQ;
    const int pp = par ^ 1;                      // parity of block k-1
    load_pp<P>(sTp, st->Tr[(sk + 2) % 3]);       // Tr_{k-1} (in flight with the totals)
    if (st->given_blk == k - 1) {
        load_pp<P>(sC, st->Ck[pp]);
        load_pp<P>(sTk, st->Tr[sk]);
    } else {
        const int Q = st->q_live;
        for (int t = threadIdx.x; t < P * P + Q * P; t += blockDim.x) sRed[t] = st->red2[pp][t];
        for (int t = threadIdx.x; t < P; t += blockDim.x) sOm[t] = st->om2[pp][t];
        __syncthreads();
        if (factor_block<P>(sRed, sOm, sRed + P * P, Q, st->tau, sC, sCi, sCo, absent_mask(st, k, P))) {
            if (blockIdx.x == 0 && threadIdx.x == 0) publish_breakdown(st, k - 1);
            return false;
        }
        for (int t = threadIdx.x; t < P * P; t += blockDim.x) sTk[t] = sCi[t];
        if (blockIdx.x == 0) {
            store_pp<P>(st->Ck[pp], sC);
            store_pp<P>(st->Tr[sk], sCi);
            for (int t = threadIdx.x; t < P * MAXQ; t += blockDim.x) st->coef[pp][t] = sCo[t];
        }
    }
    __syncthreads();
    smm_nn<P>(sTp, sC, sD, true);                // D = Tr_{k-1} C_{k-1}^T
    __syncthreads();
    return true;
}

// The factorisation of block k's new candidates from reduce2's totals in sm[0 .. P*P + q*P):
// factor_block (Cholesky of W'^T W', the breakdown / cancellation tests), C_k,
// Tr_{k+1} = C_k^{-1}, coef_k, D = Tr_k C_k^T, and K1(k+1)'s fragments of Tr_{k+1} and -D.
// k = k_main - 1 (K2(k) advanced k_main).  All threads of one CTA.
template <int P, int FRN, int NCF>
__device__ void red2_factor(DevState* st, int par, double* sm, unsigned long long* tr) {
    const int Q = st->q_live;
    double* sRed = sm;                           // totals (P*P + MAXQ*P)
    double* sC = sRed + P * P + MAXQ * P;
    double* sCi = sC + P * P;
    double* sTp = sCi + P * P;
    double* sCo = sTp + P * P;
    double* sOm = sCo + P * MAXQ;
    double* sD = sOm + P;
    const long long k = st->k_main - 1;
    const int sk1 = (int)((k + 1) % 3), sk = (int)(k % 3);
    for (int t = threadIdx.x; t < P; t += blockDim.x) sOm[t] = st->om2[par][t];
    load_pp<P>(sTp, st->Tr[sk]);                 // Tr_k
    __syncthreads();
    const bool bad = factor_block<P>(sRed, sOm, sRed + P * P, Q, st->tau, sC, sCi, sCo, absent_mask(st, k + 1, P));
    if (bad) {
        if (threadIdx.x == 0) {
            st->fac_bad = 1;
            st->fac_blk = k;
            publish_breakdown(st, k);
        }
        trace_pt(tr, 5);
        return;
    }
    store_pp<P>(st->Ck[par], sC);
    store_pp<P>(st->Tr[sk1], sCi);
    for (int t = threadIdx.x; t < P * MAXQ; t += blockDim.x) st->coef[par][t] = sCo[t];
    smm_nn<P>(sTp, sC, sD, true);                // D = Tr_k C_k^T
    __syncthreads();
    // fragment order of the DMMA K1 (to_frag: 4 x 8 blocks, KC = P/4 k-chunks, NCF = P/8 n-chunks)
    for (int t = threadIdx.x; t < FRN; t += blockDim.x) {
        const int blk = t / 32, l = t % 32, kc = blk / NCF, nc = blk % NCF;
        const int r = kc * 4 + l % 4, c = nc * 8 + l / 4;
        st->fT[t] = sCi[r * P + c];
        st->fD[t] = -sD[r * P + c];
    }
    if (threadIdx.x == 0) {
        st->fac_bad = 0;
        st->fac_blk = k;   // (K3b(k), launched after this kernel completes, loads C_k instead of refactoring)
    }
    trace_pt(tr, 5);
}

// reduce2 with the factorisation (red2_fac, single rank): the totals of K2(k)'s partials as
// k_reduce computes them (same order), then the last CTA to finish (ticket) factors the new block
// exactly as K1(k+1)'s prologue would -- factor_block on the totals, C_k, Tr_{k+1} = C_k^{-1},
// coef_k, D = Tr_k C_k^T -- and stores Tr_{k+1} and -D in fragment order (to_frag of the DMMA K1),
// so K1(k+1), which launches at this kernel's early trigger and runs its fused update meanwhile,
// only loads them.  k = k_main - 1 (K2(k) advanced k_main).
// Ticketed variant (p = 16: 34 CTAs x 8 warps, one entry per warp; the last CTA to finish factors):
template <int P, int FRN, int NCF>
__global__ void __launch_bounds__(256) k_red2f_t(DevState* st, int par, int early) {
    unsigned long long* tr = trace_begin(st, TR_RED2);
    pdl_wait();
    if (early) pdl_trigger();   // K1(k+1) may launch now (see k_reduce's early trigger)
    trace_pt(tr, 1);
    if (!st->run_main) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int Q = st->q_live;
    const int E = P * P + Q * P;
    const int ncl = st->ncl2;
    const double* part = st->part2[par];
    for (int e = blockIdx.x * 8 + warp; e < E; e += gridDim.x * 8) {
        constexpr int U = 8;
        double s = 0.0;
        for (int b0 = 0; b0 < ncl; b0 += 32 * U) {
            double v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int b = b0 + lane + 32 * u;
                v[u] = b < ncl ? __ldcg(part + (size_t)b * E + e) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (b0 + lane + 32 * u < ncl) s += v[u];
        }
        s = warp_sum(s);
        if (lane == 0) st->red2[par][e] = s;
    }
    // last CTA: factor
    __shared__ int s_last;
    __shared__ double sm[P * P + MAXQ * P + 3 * P * P + P * MAXQ + P + 2 * P * P];
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(&st->cnt2, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (threadIdx.x == 0) st->cnt2 = 0u;
    for (int t = threadIdx.x; t < E; t += blockDim.x) sm[t] = __ldcg(st->red2[par] + t);
    red2_factor<P, FRN, NCF>(st, par, sm, tr);
}

// One thread-block cluster of RF_CL CTAs x RF_W warps: each warp sums its entries (k_reduce's
// order) and stores them into the leader CTA's shared memory (distributed shared memory); after
// the cluster barrier the leader factors.  No global round trips between the totals and the
// factorisation -- the tail runs while K1(k+1)'s fused update saturates HBM, where each L2 round
// trip costs several microseconds (a ticketed last-CTA tail took ~22 us there).
constexpr int RF_CL = 8;   // (measured: 8 x 16 warps 136k it/s at config 2; 4 x 32: 135k; 2 x 32: 134.7k)
template <int P>
__host__ __device__ constexpr int rf_warps() { return P <= 8 ? 16 : 32; }   // p = 16: 256 warps, <= 2 entries each
template <int P, int FRN, int NCF>
__global__ void __launch_bounds__(rf_warps<P>() * 32) k_red2f(DevState* st, int par, int early) {
    constexpr int RF_W = rf_warps<P>();
    unsigned long long* tr = trace_begin(st, TR_RED2);
    pdl_wait();
    if (early) pdl_trigger();   // K1(k+1) may launch now (see k_reduce's early trigger)
    trace_pt(tr, 1);
    if (!st->run_main) return;   // (uniform: every CTA of the cluster returns)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int Q = st->q_live;
    const int E = P * P + Q * P;
    const int ncl = st->ncl2;
    const double* part = st->part2[par];
    __shared__ double sm[P * P + MAXQ * P + 3 * P * P + P * MAXQ + P + 2 * P * P];
    cg::cluster_group cl = cg::this_cluster();
    double* lead = cl.map_shared_rank(sm, 0);    // the leader's totals (sRed)
    for (int e = (int)cl.block_rank() * RF_W + warp; e < E; e += RF_CL * RF_W) {
        constexpr int U = 8;
        double s = 0.0;
        for (int b0 = 0; b0 < ncl; b0 += 32 * U) {
            double v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int b = b0 + lane + 32 * u;
                v[u] = b < ncl ? __ldcg(part + (size_t)b * E + e) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (b0 + lane + 32 * u < ncl) s += v[u];
        }
        s = warp_sum(s);
        if (lane == 0) lead[e] = s;
    }
    cl.sync();
    if (cl.block_rank() != 0) return;   // (the leader reads only its own shared memory)
    for (int t = threadIdx.x; t < E; t += blockDim.x) st->red2[par][t] = sm[t];   // (K3b(k) reads them)
    red2_factor<P, FRN, NCF>(st, par, sm, tr);
}

// Factor-only reduce2 tail for a row partition: the totals were summed by k_reduce and allreduced
// over the ranks (bitwise identical on every rank), so every rank factors them once here -- one
// CTA, the same code as k_red2f's -- and K1(k+1)'s prologue only loads the fragments.
template <int P, int FRN, int NCF>
__global__ void __launch_bounds__(256) k_fac2(DevState* st, int par) {
    unsigned long long* tr = trace_begin(st, TR_RED2);
    pdl_wait();
    if (!st->run_main) return;
    __shared__ double sm[P * P + MAXQ * P + 3 * P * P + P * MAXQ + P + 2 * P * P];
    const int E = P * P + st->q_live * P;
    for (int t = threadIdx.x; t < E; t += blockDim.x) sm[t] = __ldcg(st->red2[par] + t);
    red2_factor<P, FRN, NCF>(st, par, sm, tr);
}

// K2 prologue, block k: G = Tr_k^T (V_k^T W) from K1's partials, om2; CTA 0 publishes G, om2 for
// the side branch and the column path.  Writes sG (P x P, ld P, G itself) and sTk (Tr_k).
template <int P>
__device__ void k2_prologue(DevState* st, int par, int sk, double* sG, double* sTk, double* scr) {
    double* sRed = scr;   // P*P + P
    for (int t = threadIdx.x; t < P * P + P; t += blockDim.x) sRed[t] = st->red1[t];
    load_pp<P>(sTk, st->Tr[sk]);
    __syncthreads();
    smm_tn<P>(sTk, sRed, sG);
    __syncthreads();
    if (blockIdx.x == 0) {
        store_pp<P>(st->G[par], sG);
        for (int t = threadIdx.x; t < P; t += blockDim.x) st->om2[par][t] = sRed[P * P + t];
        if (threadIdx.x == 0) st->k_main = st->k_main + 1;
    }
}


}  // namespace bmr
