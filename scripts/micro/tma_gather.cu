// tma_gather.cu -- standalone microbenchmark (design exploration, not the product): the CSR x
// tall-skinny SpMM A X with every gathered X row fetched by a bulk copy (cp.async.bulk, TMA,
// mbarrier completion) into a shared-memory ring, then summed in CSR order from shared memory --
// gathers that hold no registers, the precondition for fusing K1a into K1's DMMA epilogue at
// p = 32.  Compared with the register-gather SpMM (K1a's scheme).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/tma_gather tma_gather.cu
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA error %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1); } } while (0)

constexpr int P = 32;
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect(unsigned long long* b, unsigned tx) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((unsigned)__cvta_generic_to_shared(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned par) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(b);
    unsigned done = 0;
    while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(a), "r"(par) : "memory");
}
__device__ __forceinline__ void bulk_row(void* dst, const void* src, unsigned bytes, unsigned long long* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(b)) : "memory");
}

// T rows per tile, CAP gathered rows per slot, NS slots, NCW consumer warps (+1 producer warp)
template <int T, int CAP, int NS, int NCW, bool STORE>
__global__ void __launch_bounds__((NCW + 1) * 32, 1) spmm_tma(const int* __restrict__ rp, const int* __restrict__ ci,
                                                        const double* __restrict__ va, const double* __restrict__ X,
                                                        double* __restrict__ Y, long long n) {
    extern __shared__ __align__(128) double sm[];
    __shared__ unsigned long long full[NS], empty[NS];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long ntiles = (n + T - 1) / T;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], NCW); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == NCW) {   // producer
        long long it = 0;
        for (long long t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
            const int s = (int)(it % NS);
            if (it >= NS) mbar_wait(&empty[s], (unsigned)(((it / NS) - 1) & 1));
            const long long r0 = t * T, r1 = r0 + T < n ? r0 + T : n;
            const int e0 = rp[r0], e1 = rp[r1];
            if (lane == 0) mbar_expect(&full[s], (unsigned)(e1 - e0) * P * 8);
            __syncwarp();
            double* slot = sm + (size_t)s * CAP * P;
            for (int e = e0 + lane; e < e1; e += 32)
                bulk_row(slot + (size_t)(e - e0) * P, X + (long long)__ldg(ci + e) * P, P * 8, &full[s]);
        }
    } else {              // consumers: 8 lanes x 4 doubles per row, 4 rows per warp instruction
        const int sub = lane & 7, rsub = lane >> 3, c0 = sub * 4;
        long long it = 0;
        for (long long t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
            const int s = (int)(it % NS);
            mbar_wait(&full[s], (unsigned)((it / NS) & 1));
            const long long r0 = t * T;
            const int e0 = rp[r0];
            const double* slot = sm + (size_t)s * CAP * P;
            for (int g = warp; g < T / 4; g += NCW) {
                const long long r = r0 + g * 4 + rsub;
                if (r < n) {
                    const int k0 = rp[r], k1 = rp[r + 1];
                    double acc[4] = {0.0, 0.0, 0.0, 0.0};
                    for (int k = k0; k < k1; ++k) {
                        const double a = __ldg(va + k);
                        const double4 x = *reinterpret_cast<const double4*>(slot + (size_t)(k - e0) * P + c0);
                        acc[0] = fma(a, x.x, acc[0]); acc[1] = fma(a, x.y, acc[1]);
                        acc[2] = fma(a, x.z, acc[2]); acc[3] = fma(a, x.w, acc[3]);
                    }
                    if (STORE) {
                        double* y = Y + r * P + c0;
                        *reinterpret_cast<double2*>(y) = make_double2(acc[0], acc[1]);
                        *reinterpret_cast<double2*>(y + 2) = make_double2(acc[2], acc[3]);
                    } else if (acc[0] == 12345.678) Y[0] = acc[1];
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
    }
}

// register gathers, K1a's scheme (chunked round robin, 8 lanes x 32 B per row, 4 entries per batch)
__global__ void __launch_bounds__(256, 5) spmm_reg(const int* __restrict__ rp, const int* __restrict__ ci,
                                                   const double* __restrict__ va, const double* __restrict__ X,
                                                   double* __restrict__ Y, long long n) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int sub = lane & 7, rsub = lane >> 3, c0 = sub * 4;
    const long long ng = (n + 3) / 4, chunk = 8 * 8;
    for (long long c = blockIdx.x; c * chunk < ng; c += gridDim.x)
        for (long long g = c * chunk + warp; g < (c + 1) * chunk && g < ng; g += 8) {
            const long long r = g * 4 + rsub;
            if (r >= n) continue;
            const int k0 = rp[r], k1 = rp[r + 1];
            double acc[4] = {0.0, 0.0, 0.0, 0.0};
            for (int kb = k0; kb < k1; kb += 4) {
                double4 x[4]; double a[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const bool pr = kb + q < k1;
                    a[q] = pr ? __ldg(va + kb + q) : 0.0;
                    if (pr) {
                        const double* px = X + (long long)__ldg(ci + kb + q) * P + c0;
                        asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(x[q].x), "=d"(x[q].y), "=d"(x[q].z), "=d"(x[q].w) : "l"(px));
                    } else {
                        x[q] = make_double4(0, 0, 0, 0);
                    }
                }
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (kb + q < k1) {
                        acc[0] = fma(a[q], x[q].x, acc[0]); acc[1] = fma(a[q], x[q].y, acc[1]);
                        acc[2] = fma(a[q], x[q].z, acc[2]); acc[3] = fma(a[q], x[q].w, acc[3]);
                    }
            }
            double* y = Y + r * P + c0;
            *reinterpret_cast<double2*>(y) = make_double2(acc[0], acc[1]);
            *reinterpret_cast<double2*>(y + 2) = make_double2(acc[2], acc[3]);
        }
}

template <typename F>
static float timeit(F launch) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 6; ++r) {
        cudaEventRecord(e0); launch(); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1); best = std::min(best, ms);
    }
    CK(cudaGetLastError());
    return best;
}

template <int T, int NS, int NCW, bool STORE>
static void run_tma(const int* rp, const int* ci, const double* va, const double* X, double* Y, long long n,
                    const std::vector<double>& yref, int ctas_per_sm) {
    constexpr int CAP = 7 * T;
    auto k = spmm_tma<T, CAP, NS, NCW, STORE>;
    const size_t smem = sizeof(double) * (size_t)NS * CAP * P;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int grid = 148 * ctas_per_sm;
    CK(cudaMemset(Y, 0, n * P * 8));
    float ms = timeit([&] { k<<<grid, (NCW + 1) * 32, smem>>>(rp, ci, va, X, Y, n); });
    bool ok = true;
    if (STORE) {
        std::vector<double> y(n * P);
        CK(cudaMemcpy(y.data(), Y, y.size() * 8, cudaMemcpyDeviceToHost));
        ok = memcmp(y.data(), yref.data(), y.size() * 8) == 0;
    }
    printf("tma T=%3d NS=%d NCW=%2d store=%d ctas/SM=%d smem=%6zu  %8.1f us  %s\n", T, NS, NCW, (int)STORE, ctas_per_sm,
           smem, ms * 1e3, STORE ? (ok ? "bitwise ok" : "MISMATCH") : "");
}

int main() {
    const int nx = 256;
    const long long n = (long long)nx * nx * nx;
    std::vector<int> rp(n + 1), ci; std::vector<double> v;
    ci.reserve(7 * n); v.reserve(7 * n);
    for (int z = 0; z < nx; ++z) for (int y = 0; y < nx; ++y) for (int x = 0; x < nx; ++x) {
        long long i = ((long long)z * nx + y) * nx + x;
        auto add = [&](long long j, double a) { ci.push_back((int)j); v.push_back(a); };
        if (z > 0) add(i - nx * nx, -1); if (y > 0) add(i - nx, -1); if (x > 0) add(i - 1, -1);
        add(i, 3.0);
        if (x < nx - 1) add(i + 1, -1); if (y < nx - 1) add(i + nx, -1); if (z < nx - 1) add(i + (long long)nx * nx, -1);
        rp[i + 1] = (int)ci.size();
    }
    const long long nnz = ci.size();
    int *drp, *dci; double *dva, *dX, *dY;
    CK(cudaMalloc(&drp, (n + 1) * 4)); CK(cudaMalloc(&dci, nnz * 4)); CK(cudaMalloc(&dva, nnz * 8));
    CK(cudaMalloc(&dX, n * P * 8)); CK(cudaMalloc(&dY, n * P * 8));
    CK(cudaMemcpy(drp, rp.data(), (n + 1) * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dci, ci.data(), nnz * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dva, v.data(), nnz * 8, cudaMemcpyHostToDevice));
    {
        std::vector<double> x(n * P); std::mt19937_64 g(7);
        for (auto& t : x) t = (double)(g() >> 11) * 0x1.0p-53 - 0.5;
        CK(cudaMemcpy(dX, x.data(), x.size() * 8, cudaMemcpyHostToDevice));
    }
    float ms = timeit([&] { spmm_reg<<<148 * 5 - 1, 256>>>(drp, dci, dva, dX, dY, n); });
    std::vector<double> yref(n * P);
    CK(cudaMemcpy(yref.data(), dY, yref.size() * 8, cudaMemcpyDeviceToHost));
    printf("n=%lld nnz=%lld  register gathers (K1a scheme, 739 CTAs): %8.1f us\n", n, nnz, ms * 1e3);
    run_tma<32, 3, 8, true>(drp, dci, dva, dX, dY, n, yref, 1);
    run_tma<32, 3, 8, false>(drp, dci, dva, dX, dY, n, yref, 1);
    run_tma<32, 2, 8, true>(drp, dci, dva, dX, dY, n, yref, 2);
    run_tma<16, 4, 4, true>(drp, dci, dva, dX, dY, n, yref, 2);
    run_tma<16, 3, 4, true>(drp, dci, dva, dX, dY, n, yref, 3);
    run_tma<64, 2, 16, true>(drp, dci, dva, dX, dY, n, yref, 1);
    run_tma<64, 2, 16, false>(drp, dci, dva, dX, dY, n, yref, 1);
    return 0;
}
