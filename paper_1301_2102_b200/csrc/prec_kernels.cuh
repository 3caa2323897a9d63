// prec_kernels.cuh -- SURVEY §8(f) row f3: split preconditioning with an IC(0) factor.
//
// the paper preconditions with "the incomplete Cholesky factors of -L constructed
// using Matlab's ichol() function with the default settings" (zero fill).  Reading R8
// (DESIGN.md): the split form -- the block method runs on Ahat = L^-1 A L^-T with
// Rhat_0 = L^-1 (B - A X_0), and X = X_0 + L^-T Yhat.  Per block step the operator application
// (row a1's SpMM) becomes three steps, run here as two kernels:
//   k_trsv<P, UPPER=true,  SPMM=false>   Z  = L^-T V_k          (backward substitution on U = L^T)
//   k_trsv<P, UPPER=false, SPMM=true>    AV = L^-1 (A Z)        (SpMM row, then forward substitution)
// after which K1 streams AV exactly as in split mode.
//
// Scheduling: a triangular solve is a DAG over rows (row i waits for the rows its off-diagonal
// entries reference).  The host sorts rows by level (1 + the deepest dependency) and cuts each
// level into tasks of RPW rows (one warp instruction of the panel-row mapping PC<P>).  Tasks are
// dealt round-robin to the warps of a persistent grid no larger than the resident capacity;
// each warp runs its tasks in increasing order and a row waits on per-row flags (acquire loads)
// of the rows it reads, which publish with a release store after their panel row is written.
// No level barriers, no atomics on the hot path.  Deadlock-free: the smallest unfinished task's
// dependencies are all in earlier tasks (finished), and its warp has finished its own earlier
// tasks, so it runs.  Flags carry an epoch (one per launch; every triangular launch of a handle
// shares one counter and one flag array, launched in stream order), so they are never reset.
//
// Arithmetic order (bitwise the oracle's orc_trsv_lower / orc_trsv_upper / csr_matvec):
//   forward:  s = (A z)_i (CSR order, fma from 0) or b_i;  s = fma(-l_ij, y_j, s) for j < i ascending;
//             y_i = s / l_ii
//   backward: s = v_i;  s = fma(-l_ji, z_j, s) for j > i ascending;  z_i = s / l_ii
//   IC(0):    the up-looking row algorithm of orc_ic0, one thread per row.
#pragma once
#include "common.cuh"

namespace bmr {

// control words of the triangular kernels of a handle (device memory, zero-initialised once)
struct TriCtl {
    unsigned epoch;   // flags written by the last completed launch hold this value
    unsigned done;    // CTAs finished in the current launch
    int bad_row;      // IC(0): smallest row with a pivot <= 0 (INT_MAX: none)
    int pad;
};

struct TriSched {
    const int* order;    // rows sorted by level
    const int* tstart;   // task t covers order[tstart[t] .. tstart[t+1])
    long long ntask;
};

struct TriArgs {
    const int* rowptr;   // A (SPMM only)
    const int* col;
    const double* val;
    const int* Tp;       // triangular rows: L (diagonal last) or U = L^T (diagonal first)
    const int* Ti;
    const double* Tx;
    const double* X;     // input panel: b (forward), v (backward), or the SpMM input z
    double* Y;           // output panel
    unsigned* flags;     // one per row
    TriCtl* ctl;
    TriSched s;
    long long n;
};

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void wait_flag(const unsigned* f, unsigned ep) {
    if (ld_acquire_u32(f) == ep) return;
    int spins = 0;
    while (ld_acquire_u32(f) != ep)
        if (++spins > 64) __nanosleep(32);
}

// The epoch this launch publishes (all CTAs read it before any CTA finishes, see tri_finish).
__device__ __forceinline__ unsigned tri_epoch(const TriCtl* c) {
    return *reinterpret_cast<const volatile unsigned*>(&c->epoch) + 1u;
}
// Last CTA of the launch advances the epoch (every CTA has read it: each reads it first and
// counts itself done last).
__device__ __forceinline__ void tri_finish(TriCtl* c, unsigned ep) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned d = atomicAdd(&c->done, 1u);
        if (d == gridDim.x - 1) {
            c->done = 0;
            __threadfence();
            *reinterpret_cast<volatile unsigned*>(&c->epoch) = ep;
        }
    }
}

template <int P, bool UPPER, bool SPMM>
__global__ void __launch_bounds__(NT) k_trsv(TriArgs a) {
    using C = PC<P>;
    constexpr int VEC = C::VEC, LANES = C::LANES, LP = C::LP, WARPS = NT / 32;
    constexpr int CH = 4;
    const unsigned ep = tri_epoch(a.ctl);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int sub = lane % LP, rsub = lane / LP;
    const bool act = sub < LANES;
    const int c0 = sub * VEC;
    const long long W = (long long)gridDim.x * WARPS;
    for (long long t = (long long)blockIdx.x * WARPS + warp; t < a.s.ntask; t += W) {
        const int r0 = __ldg(a.s.tstart + t), r1 = __ldg(a.s.tstart + t + 1);
        const bool has = r0 + rsub < r1;
        const long long i = has ? __ldg(a.s.order + r0 + rsub) : 0;
        double acc[VEC];
#pragma unroll
        for (int v = 0; v < VEC; ++v) acc[v] = 0.0;
        if (has && act) {
            if constexpr (SPMM) {
                const int k0 = __ldg(a.rowptr + i), k1 = __ldg(a.rowptr + i + 1);
                for (int kb = k0; kb < k1; kb += CH) {
                    int cc[CH];
                    double av[CH], xv[CH][VEC];
#pragma unroll
                    for (int q = 0; q < CH; ++q) {
                        const bool pr = kb + q < k1;
                        cc[q] = pr ? __ldg(a.col + kb + q) : -1;
                        av[q] = pr ? __ldg(a.val + kb + q) : 0.0;
                    }
#pragma unroll
                    for (int q = 0; q < CH; ++q) {
                        if (cc[q] >= 0) {
                            ldv<VEC>(a.X + (long long)cc[q] * P + c0, xv[q]);
                        } else {
#pragma unroll
                            for (int v = 0; v < VEC; ++v) xv[q][v] = 0.0;
                        }
                    }
#pragma unroll
                    for (int q = 0; q < CH; ++q)
                        if (cc[q] >= 0) {
#pragma unroll
                            for (int v = 0; v < VEC; ++v) acc[v] = fma(av[q], xv[q][v], acc[v]);
                        }
                }
            } else {
                ldv<VEC>(a.X + i * P + c0, acc);
            }
        }
        if (has) {
            const int e0 = __ldg(a.Tp + i), e1 = __ldg(a.Tp + i + 1);
            const int ed = UPPER ? e0 : e1 - 1;             // the diagonal
            const int o0 = UPPER ? e0 + 1 : e0, o1 = UPPER ? e1 : e1 - 1;
            const double d = __ldg(a.Tx + ed);
            for (int e = o0; e < o1; ++e) {
                const int j = __ldg(a.Ti + e);
                const double l = __ldg(a.Tx + e);
                wait_flag(a.flags + j, ep);
                if (act) {
                    double y[VEC];
                    ldc<VEC>(a.Y + (long long)j * P + c0, y);
#pragma unroll
                    for (int v = 0; v < VEC; ++v) acc[v] = fma(-l, y[v], acc[v]);
                }
            }
            if (act) {
#pragma unroll
                for (int v = 0; v < VEC; ++v) acc[v] = acc[v] / d;
                stv<VEC>(a.Y + i * P + c0, acc);
                __threadfence();
            }
        }
        __syncwarp();
        if (has && sub == 0) st_release_u32(a.flags + i, ep);
    }
    tri_finish(a.ctl, ep);
}

// IC(0), one thread per row (orc_ic0's order).  Tx holds M's lower entries (diagonal last) on
// entry and L on exit.  A pivot <= 0 records the row in ctl->bad_row (the factor is then invalid;
// the host reports BMINRES_EPIVOT) and still publishes the row, so no thread waits forever.
__global__ void __launch_bounds__(NT) k_ic0(TriArgs a) {
    const unsigned ep = tri_epoch(a.ctl);
    const long long T = (long long)gridDim.x * NT;
    for (long long t = (long long)blockIdx.x * NT + threadIdx.x; t < a.s.ntask; t += T) {
        // (tasks of the factor are single rows)
        const long long i = __ldg(a.s.order + t);
        const int e0 = a.Tp[i], ed = a.Tp[i + 1] - 1;
        double* Lx = const_cast<double*>(a.Tx);
        for (int e = e0; e < ed; ++e) {
            const int k = a.Ti[e];
            wait_flag(a.flags + k, ep);
            double s = Lx[e];
            int x = e0, y = a.Tp[k];
            const int yend = a.Tp[k + 1] - 1;
            while (x < e && y < yend) {
                const int cx = a.Ti[x], cy = a.Ti[y];
                if (cx < cy) {
                    ++x;
                } else if (cx > cy) {
                    ++y;
                } else {
                    s = fma(-Lx[x], Lx[y], s);
                    ++x;
                    ++y;
                }
            }
            Lx[e] = s / Lx[yend];
        }
        double d = Lx[ed];
        for (int e = e0; e < ed; ++e) d = fma(-Lx[e], Lx[e], d);
        if (!(d > 0.0)) atomicMin(&a.ctl->bad_row, (int)i);
        Lx[ed] = sqrt(d);
        __threadfence();
        st_release_u32(a.flags + i, ep);
    }
    tri_finish(a.ctl, ep);
}

// Ux[e] = Lx[perm[e]] (the values of U = L^T in U's CSR order)
__global__ void k_gather_vals(const double* __restrict__ src, const int* __restrict__ perm, double* __restrict__ dst,
                              long long m) {
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += (long long)gridDim.x * blockDim.x)
        dst[e] = src[perm[e]];
}

// X = (add ? X : 0) + Z, elementwise over a panel
__global__ void k_add_panel(double* __restrict__ X, const double* __restrict__ Z, long long m, int add) {
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += (long long)gridDim.x * blockDim.x)
        X[e] = add ? X[e] + Z[e] : Z[e];
}

}  // namespace bmr
