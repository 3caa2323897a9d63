// spmm_lab.cu -- standalone microbenchmark of CSR x tall-skinny SpMM gather strategies on
// the BASELINE configs' matrix structures (not part of the product; design exploration).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/spmm_lab spmm_lab.cu
// Run:   /tmp/spmm_lab CFG   (CFG 2: 64^3 p=8; 3: 512^2 p=16; 4: 256^3 p=32; 5: band13+4 random p=16)
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

#define CK(x)                                                                            \
    do {                                                                                 \
        cudaError_t e_ = (x);                                                            \
        if (e_ != cudaSuccess) {                                                         \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            exit(1);                                                                     \
        }                                                                                \
    } while (0)

struct Csr {
    long long n;
    std::vector<int> rp, ci;
    std::vector<double> v;
};

static Csr stencil(int nx, int ny, int nz, double diag) {
    Csr A;
    A.n = (long long)nx * ny * nz;
    A.rp.resize(A.n + 1);
    A.rp[0] = 0;
    for (int z = 0; z < nz; ++z)
        for (int y = 0; y < ny; ++y)
            for (int x = 0; x < nx; ++x) {
                long long i = ((long long)z * ny + y) * nx + x;
                auto add = [&](long long j, double val) {
                    A.ci.push_back((int)j);
                    A.v.push_back(val);
                };
                if (nz > 1 && z > 0) add(i - (long long)nx * ny, -1);
                if (y > 0) add(i - nx, -1);
                if (x > 0) add(i - 1, -1);
                add(i, diag);
                if (x < nx - 1) add(i + 1, -1);
                if (y < ny - 1) add(i + nx, -1);
                if (nz > 1 && z < nz - 1) add(i + (long long)nx * ny, -1);
                A.rp[i + 1] = (int)A.ci.size();
            }
    return A;
}

static Csr band_random(long long n, int hw, int nlong) {
    std::mt19937_64 g(1);
    std::vector<std::vector<int>> extra(n);
    for (long long t = 0; t < n * nlong / 2; ++t) {
        long long i = g() % n, j = g() % n;
        if (std::llabs(i - j) > hw) {
            extra[i].push_back((int)j);
            extra[j].push_back((int)i);
        }
    }
    Csr A;
    A.n = n;
    A.rp.resize(n + 1);
    A.rp[0] = 0;
    for (long long i = 0; i < n; ++i) {
        std::vector<int> c;
        for (long long j = std::max(0ll, i - hw); j <= std::min(n - 1, i + hw); ++j) c.push_back((int)j);
        for (int j : extra[i]) c.push_back(j);
        std::sort(c.begin(), c.end());
        c.erase(std::unique(c.begin(), c.end()), c.end());
        for (int j : c) {
            A.ci.push_back(j);
            A.v.push_back(j == i ? 1.0 : 0.1);
        }
        A.rp[i + 1] = (int)A.ci.size();
    }
    return A;
}

template <int P>
struct PCx {
    static constexpr int VEC = 2;
    static constexpr int LANES = P / VEC;
    static constexpr int LP = LANES;
    static constexpr int RPW = 32 / LP;
};

// Variant A: lane group (P/2 lanes x 16 B) per row, U row groups per warp step, CH entries
// loaded per batch.  ORDER 0: CTA slabs (contiguous rows per CTA, warps interleaved);
// ORDER 1: grid-stride over warp units.
template <int P, int U, int CH, int ORDER>
__global__ void __launch_bounds__(256) spmm_a(const int* __restrict__ rp, const int* __restrict__ ci,
                                              const double* __restrict__ va, const double* __restrict__ X,
                                              double* __restrict__ Y, long long n) {
    using C = PCx<P>;
    constexpr int RPW = C::RPW;
    constexpr int ROWS = U * RPW;   // rows per warp step
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int sub = lane % C::LP, rsub = lane / C::LP;
    const int c0 = sub * 2;
    const long long nunits = (n + ROWS - 1) / ROWS;
    long long ubeg, uend, ustep;
    if (ORDER == 0) {
        const long long per = (nunits + gridDim.x - 1) / gridDim.x;
        ubeg = blockIdx.x * per + warp;
        uend = min(nunits, (long long)(blockIdx.x + 1) * per);
        ustep = nw;
    } else {
        ubeg = (long long)blockIdx.x * nw + warp;
        uend = nunits;
        ustep = (long long)gridDim.x * nw;
    }
    constexpr int KU = 8;   // ORDER 2: CTA chunks of nw*KU consecutive units, round-robin over CTAs
    const long long chunk = (long long)nw * KU;
    long long cidx = blockIdx.x, cpos = warp;
    if (ORDER == 2) {
        ubeg = blockIdx.x * chunk + warp;
        uend = nunits;
    }
    for (long long u = ubeg; u < uend;) {
        int r0[U], r1[U];
#pragma unroll
        for (int x = 0; x < U; ++x) {
            const long long i = u * ROWS + x * RPW + rsub;
            r0[x] = i < n ? __ldg(rp + i) : 0;
            r1[x] = i < n ? __ldg(rp + i + 1) : 0;
        }
        double acc[U][2];
#pragma unroll
        for (int x = 0; x < U; ++x) acc[x][0] = acc[x][1] = 0.0;
        int kb[U];
#pragma unroll
        for (int x = 0; x < U; ++x) kb[x] = r0[x];
        while (true) {
            bool any = false;
#pragma unroll
            for (int x = 0; x < U; ++x) any |= kb[x] < r1[x];
            if (!__any_sync(0xffffffffu, any)) break;
            int c[U][CH];
            double a[U][CH];
#pragma unroll
            for (int x = 0; x < U; ++x)
#pragma unroll
                for (int t = 0; t < CH; ++t) {
                    const bool pr = kb[x] + t < r1[x];
                    c[x][t] = pr ? __ldg(ci + kb[x] + t) : -1;
                    a[x][t] = pr ? __ldg(va + kb[x] + t) : 0.0;
                }
            double2 g[U][CH];
#pragma unroll
            for (int x = 0; x < U; ++x)
#pragma unroll
                for (int t = 0; t < CH; ++t)
                    g[x][t] = c[x][t] >= 0 ? __ldg(reinterpret_cast<const double2*>(X + (long long)c[x][t] * P + c0))
                                           : make_double2(0.0, 0.0);
#pragma unroll
            for (int x = 0; x < U; ++x)
#pragma unroll
                for (int t = 0; t < CH; ++t) {
                    acc[x][0] = fma(a[x][t], g[x][t].x, acc[x][0]);
                    acc[x][1] = fma(a[x][t], g[x][t].y, acc[x][1]);
                }
#pragma unroll
            for (int x = 0; x < U; ++x) kb[x] += CH;
        }
#pragma unroll
        for (int x = 0; x < U; ++x) {
            const long long i = u * ROWS + x * RPW + rsub;
            if (i < n) *reinterpret_cast<double2*>(Y + i * P + c0) = make_double2(acc[x][0], acc[x][1]);
        }
        if (ORDER == 2) {
            cpos += nw;
            if (cpos >= chunk) {
                cpos = warp;
                cidx += gridDim.x;
            }
            u = cidx * chunk + cpos;
        } else {
            u += ustep;
        }
    }
}


__device__ __forceinline__ void cpa16(void* sdst, const void* gsrc, bool pred) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
    const int nb = pred ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gsrc), "r"(nb) : "memory");
}
__device__ __forceinline__ void cpa8(void* sdst, const void* gsrc, bool pred) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
    const int nb = pred ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gsrc), "r"(nb) : "memory");
}
__device__ __forceinline__ void cpcommit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cpwait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// Variant C: cp.async gather ring.  A unit = one CH-entry chunk of the warp's RPW rows; D units
// in flight per warp (no registers held per in-flight gather).  Column indices of the next unit
// are loaded one step ahead, row pointers two groups ahead.
template <int P, int CH, int D>
struct CSm {
    static constexpr int RPW = PCx<P>::RPW;
    static constexpr int SLOT = CH * RPW * P + CH * RPW;   // doubles: x rows, then vals
    static constexpr int WARP = D * SLOT;
};
template <int P, int CH, int D, int ORDER, int MINB>
__global__ void __launch_bounds__(256, MINB) spmm_c(const int* __restrict__ rp, const int* __restrict__ ci,
                                              const double* __restrict__ va, const double* __restrict__ X,
                                              double* __restrict__ Y, long long n) {
    using C = PCx<P>;
    using S = CSm<P, CH, D>;
    constexpr int RPW = C::RPW;
    extern __shared__ __align__(16) double smc[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int sub = lane % C::LP, rsub = lane / C::LP;
    const int c0 = sub * 2;
    double* ring = smc + warp * S::WARP;
    int* meta = reinterpret_cast<int*>(smc + nw * S::WARP) + warp * D * 2;
    const long long ngroups = (n + RPW - 1) / RPW;
    long long gbeg, gend, gstep;
    if (ORDER == 0) {
        const long long per = (ngroups + gridDim.x - 1) / gridDim.x;
        gbeg = blockIdx.x * per + warp;
        gend = min(ngroups, (long long)(blockIdx.x + 1) * per);
        gstep = nw;
    } else {
        gbeg = (long long)blockIdx.x * nw + warp;
        gend = ngroups;
        gstep = (long long)gridDim.x * nw;
    }
    // issuer state
    long long gi = gbeg;           // group being issued
    int ci_ = 0, mc = 0;           // chunk, chunks of the group
    int k0 = 0, k1 = 0;            // lane's row range (group gi)
    int nk0 = 0, nk1 = 0;          // row pointers of the next group
    int cn[CH];
    auto rowp = [&](long long g, int& a, int& b) {
        a = b = 0;
        if (g < gend) {
            const long long i = g * RPW + rsub;
            if (i < n) {
                a = __ldg(rp + i);
                b = __ldg(rp + i + 1);
            }
        }
    };
    auto chunks = [&](int a, int b) { return __reduce_max_sync(0xffffffffu, (unsigned)((b - a + CH - 1) / CH)); };
    auto loadc = [&]() {
#pragma unroll
        for (int t = 0; t < CH; ++t) {
            const int k = k0 + ci_ * CH + t;
            cn[t] = k < k1 ? __ldg(ci + k) : -1;
        }
    };
    rowp(gi, k0, k1);
    rowp(gi + gstep, nk0, nk1);
    mc = chunks(k0, k1);
    loadc();
    auto advance = [&]() {
        if (++ci_ >= mc) {
            ci_ = 0;
            gi += gstep;
            k0 = nk0;
            k1 = nk1;
            rowp(gi + gstep, nk0, nk1);
            mc = chunks(k0, k1);
            if (gi < gend && mc == 0) mc = 1;   // empty rows: one (empty) unit to write zeros
        }
        loadc();
    };
    if (mc == 0 && gi < gend) mc = 1;
    auto issue = [&](int slot) {
        if (gi < gend) {
            double* sx = ring + slot * S::SLOT;
            double* sv = sx + CH * RPW * P;
#pragma unroll
            for (int t = 0; t < CH; ++t) {
                const bool ok = cn[t] >= 0;
                cpa16(sx + (t * RPW + rsub) * P + c0, X + (long long)(ok ? cn[t] : 0) * P + c0, ok);
                if (sub == 0) {
                    const int k = k0 + ci_ * CH + t;
                    cpa8(sv + t * RPW + rsub, va + (ok ? k : 0), ok);
                }
            }
            if (lane == 0) {
                meta[slot * 2] = (int)((gi - gbeg) / gstep);
                meta[slot * 2 + 1] = (ci_ == mc - 1) ? 1 : 0;
            }
            advance();
        } else if (lane == 0) {
            meta[slot * 2] = -1;
        }
        cpcommit();
    };
#pragma unroll
    for (int s = 0; s < D - 1; ++s) issue(s);
    double acc0 = 0.0, acc1 = 0.0;
    for (int u = 0;; ++u) {
        issue((u + D - 1) % D);
        cpwait<D - 1>();
        __syncwarp();
        const int slot = u % D;
        const int gl = meta[slot * 2];
        if (gl < 0) break;
        const double* sx = ring + slot * S::SLOT;
        const double* sv = sx + CH * RPW * P;
#pragma unroll
        for (int t = 0; t < CH; ++t) {
            const double a = sv[t * RPW + rsub];
            const double2 x = *reinterpret_cast<const double2*>(sx + (t * RPW + rsub) * P + c0);
            acc0 = fma(a, x.x, acc0);
            acc1 = fma(a, x.y, acc1);
        }
        if (meta[slot * 2 + 1]) {
            const long long i = (gbeg + (long long)gl * gstep) * RPW + rsub;
            if (i < n) *reinterpret_cast<double2*>(Y + i * P + c0) = make_double2(acc0, acc1);
            acc0 = acc1 = 0.0;
        }
        __syncwarp();
    }
    cpwait<0>();
}

__global__ void copyk(const double2* __restrict__ a, double2* __restrict__ b, long long m) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x)
        b[i] = a[i];
}

struct Dev {
    int *rp, *ci;
    double *va, *X, *Y, *Yref;
    long long n, nnz;
    double bytes;
};

template <typename K>
static float timeit(K kern, int grid, int nt, const Dev& d, int reps = 7) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(e0);
        kern<<<grid, nt>>>(d.rp, d.ci, d.va, d.X, d.Y, d.n);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = std::min(best, ms);
    }
    CK(cudaGetLastError());
    return best;
}

template <int P, int U, int CH, int ORDER>
static void run_a(const Dev& d, int ctas_per_sm, const char* tag) {
    auto k = spmm_a<P, U, CH, ORDER>;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 256, 0);
    const int per = std::min(occ, ctas_per_sm);
    const int grid = 148 * per;
    float ms = timeit(k, grid, 256, d);
    // check
    std::vector<double> y(d.n * P), yr(d.n * P);
    CK(cudaMemcpy(y.data(), d.Y, y.size() * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(yr.data(), d.Yref, yr.size() * 8, cudaMemcpyDeviceToHost));
    bool ok = memcmp(y.data(), yr.data(), y.size() * 8) == 0;
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k);
    printf("%-28s U=%d CH=%2d order=%d occ=%d/%d regs=%3d  %8.1f us  %7.1f GB/s  %s\n", tag, U, CH, ORDER, per, occ,
           fa.numRegs, ms * 1e3, d.bytes / (ms * 1e-3) / 1e9, ok ? "ok" : "MISMATCH");
    CK(cudaMemset(d.Y, 0, d.n * P * 8));
}


template <int P, int CH, int D, int ORDER, int MINB>
static void run_c(const Dev& d, int ctas_per_sm, const char* tag) {
    auto k = spmm_c<P, CH, D, ORDER, MINB>;
    const size_t smem = sizeof(double) * 8 * CSm<P, CH, D>::WARP + 8 * D * 2 * 4;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 256, smem);
    const int per = std::min(occ, ctas_per_sm);
    if (per < 1) { printf("%s: no occupancy\n", tag); return; }
    const int grid = 148 * per;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 7; ++r) {
        cudaEventRecord(e0);
        k<<<grid, 256, smem>>>(d.rp, d.ci, d.va, d.X, d.Y, d.n);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = std::min(best, ms);
    }
    CK(cudaGetLastError());
    std::vector<double> y(d.n * P), yr(d.n * P);
    CK(cudaMemcpy(y.data(), d.Y, y.size() * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(yr.data(), d.Yref, yr.size() * 8, cudaMemcpyDeviceToHost));
    bool ok = memcmp(y.data(), yr.data(), y.size() * 8) == 0;
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k);
    printf("%-28s CH=%2d D=%d order=%d occ=%d/%d regs=%3d smem=%6zu %8.1f us  %7.1f GB/s  %s\n", tag, CH, D, ORDER, per, occ,
           fa.numRegs, smem, best * 1e3, d.bytes / (best * 1e-3) / 1e9, ok ? "ok" : "MISMATCH");
    CK(cudaMemset(d.Y, 0, d.n * P * 8));
}

template <int P>
static void lab(const Csr& A) {
    Dev d;
    d.n = A.n;
    d.nnz = A.ci.size();
    CK(cudaMalloc(&d.rp, (d.n + 1) * 4));
    CK(cudaMalloc(&d.ci, d.nnz * 4));
    CK(cudaMalloc(&d.va, d.nnz * 8));
    CK(cudaMalloc(&d.X, d.n * P * 8 + 256));
    CK(cudaMalloc(&d.Y, d.n * P * 8 + 256));
    CK(cudaMalloc(&d.Yref, d.n * P * 8 + 256));
    CK(cudaMemcpy(d.rp, A.rp.data(), (d.n + 1) * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d.ci, A.ci.data(), d.nnz * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d.va, A.v.data(), d.nnz * 8, cudaMemcpyHostToDevice));
    {
        std::vector<double> x(d.n * P);
        std::mt19937_64 g(7);
        for (auto& v : x) v = (double)(g() >> 11) * 0x1.0p-53 - 0.5;
        CK(cudaMemcpy(d.X, x.data(), x.size() * 8, cudaMemcpyHostToDevice));
    }
    d.bytes = 12.0 * d.nnz + 4.0 * (d.n + 1) + 16.0 * d.n * P;
    printf("n=%lld nnz=%lld p=%d  algorithmic bytes %.1f MB  (nnz/row %.2f)\n", d.n, d.nnz, P, d.bytes / 1e6,
           (double)d.nnz / d.n);
    // reference = variant U=1 CH=8 order 0
    spmm_a<P, 1, 8, 0><<<148, 256>>>(d.rp, d.ci, d.va, d.X, d.Yref, d.n);
    CK(cudaDeviceSynchronize());
    {
        const long long m = (long long)(d.bytes / 32);
        double2 *a, *b;
        CK(cudaMalloc(&a, m * 16));
        CK(cudaMalloc(&b, m * 16));
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        float best = 1e30f;
        for (int r = 0; r < 7; ++r) {
            cudaEventRecord(e0);
            copyk<<<148 * 8, 256>>>(a, b, m);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = std::min(best, ms);
        }
        printf("%-28s %8.1f us  %7.1f GB/s\n", "copy (same bytes)", best * 1e3, d.bytes / (best * 1e-3) / 1e9);
        cudaFree(a);
        cudaFree(b);
    }
    for (int cps : {4, 8}) {
        printf("-- ctas/SM cap %d\n", cps);
        run_a<P, 1, 8, 0>(d, cps, "A slab");
        run_a<P, 1, 8, 1>(d, cps, "A stride");
        run_a<P, 1, 8, 2>(d, cps, "A chunked");
        run_a<P, 1, 4, 2>(d, cps, "A chunked");
        run_a<P, 1, 16, 2>(d, cps, "A chunked");
        run_a<P, 2, 4, 2>(d, cps, "A chunked");
    }
    cudaFree(d.rp);
    cudaFree(d.ci);
    cudaFree(d.va);
    cudaFree(d.X);
    cudaFree(d.Y);
    cudaFree(d.Yref);
}


__global__ void dmma_peak(double* out, int iters) {
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
    double c[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.0) out[0] = s;
}
__global__ void dfma_peak(double* out, int iters) {
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
    double c[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) c[i] = fma(a, c[i], b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i];
    if (s == 12345.0) out[0] = s;
}
static void peaks() {
    double* o;
    cudaMalloc(&o, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int warps : {4, 8, 16}) {
        const int iters = 4096;
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(e0);
            dmma_peak<<<148 * 4, warps * 32>>>(o, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = std::min(best, ms);
        }
        const double fl = 148.0 * 4 * warps * iters * 8 * 512;
        printf("DMMA m8n8k4: %d warps/CTA x 4 CTA/SM: %.2f TFLOP/s\n", warps, fl / (best * 1e-3) / 1e12);
        best = 1e30f;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(e0);
            dfma_peak<<<148 * 4, warps * 32>>>(o, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = std::min(best, ms);
        }
        const double f2 = 148.0 * 4 * warps * 32 * iters * 8 * 2;
        printf("DFMA:        %d warps/CTA x 4 CTA/SM: %.2f TFLOP/s\n", warps, f2 / (best * 1e-3) / 1e12);
    }
    CK(cudaGetLastError());
}

int main(int argc, char** argv) {
    if (argc > 1 && atoi(argv[1]) == 0) { peaks(); return 0; }
    const int cfg = argc > 1 ? atoi(argv[1]) : 2;
    if (cfg == 2) lab<8>(stencil(64, 64, 64, 3.0));
    if (cfg == 3) lab<16>(stencil(512, 512, 1, 1.5));
    if (cfg == 4) lab<32>(stencil(256, 256, 256, 3.0));
    if (cfg == 5) lab<16>(band_random(4194304, 13, 4));
    if (cfg == 6) lab<8>(stencil(256, 256, 256, 3.0));
    return 0;
}
