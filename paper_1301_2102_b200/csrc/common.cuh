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
};

// Device-resident solver state.  p x p matrices are row-major [a*MAXP + b].
struct DevState {
    // ---- main branch (K1, K2, K4a)
    int run_main;       // main-branch kernels run
    int need_slow;      // K2: breakdown or Cholesky cancellation at block bd_at
    int pad_m;
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
    unsigned cnt1, cnt2, cnt3, cnt4;   // tickets of the cluster reductions
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
    double Z[MAXP * MAXP];         // Z_k: row m = z_{(k-1)p+m+1}^T (rows past the stop are 0)
    double Ainv[MAXP * MAXP];      // R_kk^{-1}
    double B1[MAXP * MAXP];        // R_{k-1,k} R_kk^{-1}
    double B2[MAXP * MAXP];        // R_{k-2,k} R_kk^{-1}
    double rv[(2 * MAXP + 1) * (MAXP + 1)];   // Householder ring, slot = i mod (2p+1)
    double rtau[2 * MAXP + 1];
    double beta[MAXP];             // ||b_i||
    double res[MAXP];              // latest computed relative residuals
    double* hist;                  // (hist_cap) x p computed relative residuals, or null
    HostFlags* hflags;             // device alias of the mapped host flags
};

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

// Cluster reduction.  Every CTA of a reducing panel kernel ends with its sums in shared
// memory sAcc[E].  The CTAs of a thread-block cluster are combined through distributed
// shared memory by the cluster's rank-0 CTA (fixed rank order), which writes one partial
// per cluster; the last cluster leader to arrive sums the per-cluster partials in fixed
// order into outA (entries e < P*P, at [(e/P)*MAXP + e%P]) and outB (the rest, at
// [((e-P*P)/P)*MAXP + (e-P*P)%P]).  Returns true in the CTA that produced the totals.
// Deterministic: no floating-point atomics.
__device__ __forceinline__ bool cluster_reduce(double* sAcc, int E, int P, double* part, double* outA,
                                               double* outB, unsigned* cnt) {
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    const unsigned rank = cl.block_rank();
    const int csz = (int)cl.num_blocks();
    const int ncl = gridDim.x / csz, cid = blockIdx.x / csz;
    if (rank == 0) {
        for (int e = threadIdx.x; e < E; e += blockDim.x) {
            double s = 0.0;
            for (int r = 0; r < csz; ++r) s += cl.map_shared_rank(sAcc, r)[e];
            part[(size_t)cid * E + e] = s;   // partial-major: the final sum reads coalesced rows
        }
    }
    cl.sync();  // remote shared memory must outlive the leader's reads
    if (rank != 0) return false;
    __shared__ int s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(cnt, 1u) == (unsigned)ncl - 1);
    __syncthreads();
    if (!s_last) return false;
    __threadfence();
    // one thread per entry; 8 independent accumulators (fixed order), loads coalesced across threads
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
        double acc[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[u] = 0.0;
        int b = 0;
        for (; b + 8 <= ncl; b += 8) {
#pragma unroll
            for (int u = 0; u < 8; ++u) acc[u] += __ldcg(part + (size_t)(b + u) * E + e);
        }
        for (; b < ncl; ++b) acc[0] += __ldcg(part + (size_t)b * E + e);
        const double s = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
        if (e < P * P)
            outA[(e / P) * MAXP + e % P] = s;
        else
            outB[((e - P * P) / P) * MAXP + (e - P * P) % P] = s;
    }
    if (threadIdx.x == 0) *cnt = 0u;
    __syncthreads();
    return true;
}

}  // namespace bmr
