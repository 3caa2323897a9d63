// aux_kernels.cuh -- generic column kernels: start block (eqn.init-QR), the column-by-column
// path of a block with a dependent candidate, norms, replacement RNG.
// Rare or once per solve; deterministic reductions.
#pragma once
#include "common.cuh"

namespace bmr {

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
#pragma unroll 8
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

__device__ __forceinline__ unsigned long long splitmix64(unsigned long long x) {
    unsigned long long z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// The start block's column path in ONE cooperative launch (single rank): for each column the
// same three passes as k_colstep (normalise the previous column + dots, subtract + dots,
// subtract + norm), separated by grid barriers instead of kernel boundaries; the deflation
// test and the replacement (k_rand's generator, C17) are decided on the device.  Every CTA
// reduces the partials itself in one fixed order, so all CTAs hold the same (bitwise) values.
// Outputs: S (p x p, ld MAXP), ev[m] = {ratio, kind} of step-0 events (col m+1, kind -1: none).
struct StartArgs {
    double* F;
    long long n;
    const double* f0n;   // ||F0(:,i)|| (device)
    double tau;
    unsigned long long seed;
    long long row_begin;
    double* part;        // nb x (P + 1) partials
    double* S;           // out
    double* ev;          // out: 2 x P (ratio, kind)
    int shrink;          // policy 1: a dependent start column is removed (zeroed), not replaced
};

template <int P>
__global__ void __launch_bounds__(256, 4) k_start_cgs(StartArgs a) {
    constexpr int LP = P <= 1 ? 1 : P <= 2 ? 2 : P <= 4 ? 4 : P <= 8 ? 8 : P <= 16 ? 16 : 32;
    constexpr int RPW = 32 / LP;
    constexpr int NV = P + 1;
    cg::grid_group grid = cg::this_grid();
    __shared__ double sred[8][LP + 1];
    __shared__ double sv[2][NV];   // reduced values of the last pass (d: dots, then the norm)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int sub = lane % LP, rsub = lane / LP;
    const bool in = sub < P;
    const int nb = gridDim.x;
    const long long nw = (long long)nb * 8;
    const long long stride = nw * RPW * P;
    const long long e0 = ((long long)blockIdx.x * 8 + warp) * RPW * P + rsub * P + sub;
    const long long ne = a.n * P;
    unsigned long long nrep = 0;
    int npass = 0;
    // one pass: [normalise column ncol by inv] [col = rand] [col -= sum_{l<Kc} c_l F(:,l)];
    // dots of F(:,l), l < Kd, with F(:,col) and its norm -> sv[slot] (every CTA)
    auto pass = [&](int col, int ncol, double inv, bool rnd, unsigned long long key, int Kc, const double* cin,
                    int Kd, int slot) {
        const double c = (cin && sub < Kc) ? cin[sub] : 0.0;
        const int src = rsub * LP + col;
        double acc = 0.0, accn = 0.0;
        constexpr int UNR = 8;
        for (long long eb0 = e0; eb0 - sub - rsub * P < ne; eb0 += stride * UNR) {
            double xs[UNR];
#pragma unroll
            for (int u = 0; u < UNR; ++u) {
                const long long eb = eb0 + u * stride;
                xs[u] = (in && eb < ne) ? a.F[eb] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < UNR; ++u) {
                const long long eb = eb0 + u * stride;
                const bool ok = in && eb < ne;
                double x = xs[u];
                if (sub == ncol) {
                    x = x * inv;
                    if (ok) a.F[eb] = x;
                }
                if (rnd && sub == col) {
                    const long long row = (eb - sub) / P;
                    const unsigned long long h = splitmix64(key ^ (unsigned long long)(a.row_begin + row));
                    x = 2.0 * ((double)(h >> 11) * 0x1.0p-53) - 1.0;
                    if (ok) a.F[eb] = x;
                }
                double t = __shfl_sync(0xffffffffu, x, src);
                if (cin) {
                    double sdot = c * x;
#pragma unroll
                    for (int o = LP / 2; o > 0; o >>= 1) sdot += __shfl_xor_sync(0xffffffffu, sdot, o);
                    t = t - sdot;
                    if (sub == col && ok) a.F[eb] = t;
                }
                if (sub < Kd) acc = fma(x, t, acc);
                if (sub == col) accn = fma(t, t, accn);
            }
        }
#pragma unroll
        for (int o = LP; o < 32; o <<= 1) {
            acc += __shfl_xor_sync(0xffffffffu, acc, o);
            accn += __shfl_xor_sync(0xffffffffu, accn, o);
        }
        if (lane < LP) sred[warp][lane] = acc;
        if (lane == col) sred[warp][LP] = accn;
        __syncthreads();
        double* part = a.part + (size_t)(npass & 1) * NV * nb;   // double-buffered: one barrier per pass
        npass++;
        for (int v = threadIdx.x; v <= Kd; v += blockDim.x) {
            const int l = v < Kd ? v : LP;
            double s = 0.0;
            for (int w = 0; w < 8; ++w) s += sred[w][l];
            part[(size_t)v * nb + blockIdx.x] = s;
        }
        grid.sync();
        for (int v = warp; v <= Kd; v += 8) {
            double s = 0.0;
            for (int b = lane; b < nb; b += 32) s += __ldcg(part + (size_t)v * nb + b);
            s = warp_sum(s);
            if (lane == 0) sv[slot][v] = s;
        }
        __syncthreads();
    };
    __shared__ double d1[P], d2[P];
    int pend = -1;
    double pinv = 1.0;
    for (int i = 0; i < P; ++i) {
        pass(i, pend, pinv, false, 0ull, 0, nullptr, i, 0);
        for (int l = threadIdx.x; l < i; l += blockDim.x) d1[l] = sv[0][l];
        __syncthreads();
        pass(i, -1, 1.0, false, 0ull, i, d1, i, 1);
        for (int l = threadIdx.x; l < i; l += blockDim.x) d2[l] = sv[1][l];
        __syncthreads();
        pass(i, -1, 1.0, false, 0ull, i, d2, 0, 0);
        const double hh = sqrt(sv[0][0]);
        const double fn = a.f0n[i];
        if (blockIdx.x == 0)
            for (int l = threadIdx.x; l < i; l += blockDim.x) a.S[l * MAXP + i] = d1[l] + d2[l];
        if (hh <= a.tau * fn) {
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                a.S[i * MAXP + i] = 0.0;
                a.ev[2 * i] = fn > 0.0 ? hh / fn : 0.0;
                a.ev[2 * i + 1] = hh <= 1e-12 * fn ? 0.0 : 1.0;
            }
            if (a.shrink) {   // removed: u_i = 0, no normalisation (each thread zeroes the
                              // elements it reads in the later passes: no grid barrier needed)
                for (long long eb = e0; eb - sub - rsub * P < ne; eb += stride)
                    if (in && eb < ne && sub == i) a.F[eb] = 0.0;
                pend = -1;
                pinv = 1.0;
                __syncthreads();
                continue;
            }
            // replacement (C17, stream 0, event nrep), orthogonalised twice, normalised (deferred)
            const unsigned long long key = splitmix64(a.seed ^ (0ull << 56) ^ (nrep << 32));
            nrep++;
            pass(i, -1, 1.0, true, key, 0, nullptr, i, 0);
            __syncthreads();
            for (int l = threadIdx.x; l < i; l += blockDim.x) d1[l] = sv[0][l];
            __syncthreads();
            pass(i, -1, 1.0, false, 0ull, i, d1, i, 1);
            for (int l = threadIdx.x; l < i; l += blockDim.x) d2[l] = sv[1][l];
            __syncthreads();
            pass(i, -1, 1.0, false, 0ull, i, d2, 0, 0);
        } else if (blockIdx.x == 0 && threadIdx.x == 0) {
            a.S[i * MAXP + i] = hh;
            a.ev[2 * i + 1] = -1.0;
        }
        pend = i;
        pinv = 1.0 / sqrt(sv[0][0]);
        __syncthreads();
    }
    // the last column's normalisation
    for (long long eb = e0; eb - sub - rsub * P < ne; eb += stride)
        if (in && eb < ne && pend >= 0 && sub == pend) a.F[eb] = a.F[eb] * pinv;
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

// One step of the start block's column-by-column thin QR (eqn.init-QR, reading C13)
// on a row-major n x P panel F, one pass over the panel:
//   1. if ncol >= 0: F(:,ncol) *= 1/sqrt(*nsrc)        (the previous column's deferred normalisation)
//   2. if cin:      F(:,col) -= sum_{l<Kc} cin[l] F(:,l)  (one classical Gram-Schmidt pass)
//   3. out[l] = F(:,l)^T F(:,col), l < Kd; if want_norm: out[Kd] = F(:,col)^T F(:,col)
// With text != null the target vector is text[i * ts] (a vector outside the panel, e.g. a
// replacement-pool vector) instead of F(:,col); col must then be 0.
// Each thread owns whole rows (the row's P values in registers), so 1-3 need no ordering beyond
// the row; the reductions are deterministic (per-thread, warp, CTA, then CTAs in order).
struct ColStepArgs {
    double* F;
    long long n;
    int col, Kc, Kd, ncol, want_norm;
    const double* cin;
    const double* nsrc;
    double* part;
    int nb;
    double* out;
    unsigned* cnt;
    double* text;
    long long ts;
};

// Lane layout: LP = next power of two >= P lanes per row (lane sub holds F(i, sub)), 32 / LP rows
// per warp instruction, so each load is a contiguous, coalesced run of rows.
template <int P, bool TEXT>
__global__ void __launch_bounds__(256, 4) k_colstep(ColStepArgs a) {
    constexpr int LP = P <= 1 ? 1 : P <= 2 ? 2 : P <= 4 ? 4 : P <= 8 ? 8 : P <= 16 ? 16 : 32;
    constexpr int RPW = 32 / LP;
    constexpr int UNR = 8;
    __shared__ double sred[8][LP + 1];
    __shared__ int s_last;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int sub = lane % LP, rsub = lane / LP;
    const int Kc = a.Kc, Kd = a.Kd, col = a.col, ncol = a.ncol;
    const bool in = sub < P;
    const double c = (a.cin && sub < Kc) ? a.cin[sub] : 0.0;
    const double inv = ncol >= 0 ? 1.0 / sqrt(*a.nsrc) : 1.0;
    const bool upd = a.cin != nullptr;
    const int src = rsub * LP + col;
    double acc = 0.0, accn = 0.0;
    const long long nw = (long long)gridDim.x * 8;   // warps in the grid
    const long long stride = nw * RPW * P;           // elements between a warp's consecutive row groups
    // element (row, sub) of row group g: (g * RPW + rsub) * P + sub
    const long long e0 = ((long long)blockIdx.x * 8 + warp) * RPW * P + rsub * P + sub;
    const long long ne = a.n * P;
    for (long long eb = e0; eb - sub - rsub * P < ne; eb += stride * UNR) {
        double x[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const long long e = eb + u * stride;
            x[u] = (in && e < ne) ? a.F[e] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const long long e = eb + u * stride;
            const bool ok = in && e < ne;
            if (sub == ncol) {
                x[u] = x[u] * inv;
                if (ok) a.F[e] = x[u];
            }
            double t;
            long long row = 0;
            if constexpr (TEXT) {
                row = (e - sub) / P;
                t = row < a.n ? a.text[row * a.ts] : 0.0;
            } else {
                t = __shfl_sync(0xffffffffu, x[u], src);
            }
            if (upd) {
                double sdot = c * x[u];
#pragma unroll
                for (int o = LP / 2; o > 0; o >>= 1) sdot += __shfl_xor_sync(0xffffffffu, sdot, o);
                t = t - sdot;
                if constexpr (TEXT) {
                    if (sub == 0 && row < a.n) a.text[row * a.ts] = t;
                } else {
                    if (sub == col && ok) a.F[e] = t;
                }
            }
            if (sub < Kd) acc = fma(x[u], t, acc);
            if (sub == col) accn = fma(t, t, accn);
        }
    }
    // lane sub of every row group holds column sub's partial: sum over the RPW groups, then warps
#pragma unroll
    for (int o = LP; o < 32; o <<= 1) {
        acc += __shfl_xor_sync(0xffffffffu, acc, o);
        accn += __shfl_xor_sync(0xffffffffu, accn, o);
    }
    if (lane < LP) sred[warp][lane] = acc;
    if (lane == col) sred[warp][LP] = accn;   // (lane col < LP is in row group 0)
    __syncthreads();
    const int nv = Kd + (a.want_norm ? 1 : 0);
    for (int v = threadIdx.x; v < nv; v += blockDim.x) {
        const int l = v < Kd ? v : LP;
        double s = 0.0;
        for (int w = 0; w < 8; ++w) s += sred[w][l];
        a.part[(size_t)v * a.nb + blockIdx.x] = s;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(a.cnt, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    for (int v = warp; v < nv; v += 8) {
        double s = 0.0;
        for (int b = lane; b < a.nb; b += 32) s += __ldcg(a.part + (size_t)v * a.nb + b);
        s = warp_sum(s);
        if (lane == 0) a.out[v] = s;
    }
    if (threadIdx.x == 0) *a.cnt = 0u;
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

// out[a*P + b] = sum_i X(i,a) X(i,b): the Gram of a row-major n x P panel (start block, CholQR2).
// Thread t owns entries e = t, t+256, ... < P*P and a fixed row order; CTA partials, then the
// last CTA sums them in fixed order (deterministic).
__global__ void __launch_bounds__(256) k_gram(const double* X, long long n, int P, double* part, int nb, double* out,
                                              unsigned* cnt) {
    const int E = P * P;
    const int per = (E + 255) / 256;   // entries per thread (<= 4 for P <= 32)
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    const int rows_par = E >= 256 ? 1 : 256 / E;   // rows processed in parallel by this CTA
    const int e0 = E >= 256 ? threadIdx.x : threadIdx.x % E;
    const int r0 = E >= 256 ? 0 : threadIdx.x / E;
    if (r0 < rows_par) {
        int ia[4], ib[4];
        for (int u = 0; u < 4; ++u) {
            const int e = e0 + u * 256;
            ia[u] = e < E ? e / P : 0;
            ib[u] = e < E ? e % P : 0;
        }
        // rows in groups of 8 so that 16 loads per entry are in flight (the loop is latency-bound)
        const long long stride = (long long)gridDim.x * rows_par;
        long long i = (long long)blockIdx.x * rows_par + r0;
        for (; i + 7 * stride < n; i += 8 * stride) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (u >= per || e0 + u * 256 >= E) break;
                double xa[8], xb[8];
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    xa[r] = X[(i + r * stride) * P + ia[u]];
                    xb[r] = X[(i + r * stride) * P + ib[u]];
                }
#pragma unroll
                for (int r = 0; r < 8; ++r) s[u] = fma(xa[r], xb[r], s[u]);
            }
        }
        for (; i < n; i += stride)
            for (int u = 0; u < per; ++u)
                if (e0 + u * 256 < E) s[u] = fma(X[i * P + ia[u]], X[i * P + ib[u]], s[u]);
    }
    __shared__ double sred[256][4];
    for (int u = 0; u < 4; ++u) sred[threadIdx.x][u] = s[u];
    __syncthreads();
    for (int e = threadIdx.x; e < E; e += 256) {
        double r = 0.0;
        if (E >= 256) {
            r = sred[e % 256][e / 256];
        } else {
            for (int y = 0; y < rows_par; ++y) r += sred[y * E + e][0];
        }
        part[(size_t)e * nb + blockIdx.x] = r;
    }
    __shared__ int s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(cnt, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int e = warp; e < E; e += 8) {
        double t = 0.0;
        for (int b = lane; b < nb; b += 32) t += __ldcg(part + (size_t)e * nb + b);
        t = warp_sum(t);
        if (lane == 0) out[e] = t;
    }
    if (threadIdx.x == 0) *cnt = 0u;
}

// out = V Tr (row-major n x P panels; Tr P x P with leading dimension MAXP): materialises
// U_k = V_k Tr_k for the column-by-column path
__global__ void k_materialize(const double* V, const double* Tr, double* out, long long n, int P) {
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n * P; e += (long long)gridDim.x * blockDim.x) {
        const long long i = e / P;
        const int c = (int)(e % P);
        double s = 0.0;
        for (int b = 0; b < P; ++b) s = fma(V[i * P + b], Tr[b * MAXP + c], s);
        out[e] = s;
    }
}

// Y = B - Y (row-major panels, same shape)
__global__ void k_sub_from(const double* B, double* Y, long long total) {
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x)
        Y[e] = B[e] - Y[e];
}



}  // namespace bmr
