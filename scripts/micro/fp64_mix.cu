// Micro: fp64 tensor-core (DMMA m8n8k4) and fp64 FMA (DFMA) throughput alone and mixed in one
// kernel (half the warps of each CTA on each pipe) -- do the two pipes add up on sm_100a?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_mix fp64_mix.cu && ./fp64_mix
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int MODE>   // 0 dmma, 1 dfma, 2 mixed (even warps dmma, odd dfma)
__global__ void k(double* out, int iters, double a, double b) {
    const int warp = threadIdx.x >> 5;
    const bool use_mma = MODE == 0 || (MODE == 2 && (warp & 1) == 0);
    double acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = i * 1e-3;
    if (use_mma) {
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int i = 0; i < 8; ++i) dmma(acc[2 * i], acc[2 * i + 1], a, b);
        }
    } else {
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int r = 0; r < 16; ++r)   // 16 x 16 = 256 FMA per lane (32 DMMA-equivalents of 512 flops per warp)
#pragma unroll
                for (int i = 0; i < 16; ++i) acc[i] = fma(acc[i], a, b);
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += acc[i];
    if (s == 12345.0) out[threadIdx.x] = s;
}

int main() {
    double* out;
    cudaMalloc(&out, 1024 * sizeof(double));
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000, threads = 256, blocks = nsm * 4;
    const char* names[3] = {"DMMA alone", "DFMA alone", "mixed (half/half)"};
    for (int mode = 0; mode < 3; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            if (mode == 0) k<0><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
            if (mode == 1) k<1><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
            if (mode == 2) k<2><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            // per warp and iteration: 8 DMMA of 512 flops (4096), or 256 FMA per lane (16384 flops);
            // mixed: half the warps each
            const double wi = (double)blocks * (threads / 32) * iters;
            const double flops = mode == 0 ? wi * 4096.0 : mode == 1 ? wi * 16384.0 : wi * 0.5 * (4096.0 + 16384.0);
            if (rep) printf("%-20s %.2f ms  %.1f TFLOP/s\n", names[mode], ms, flops / ms / 1e9);
        }
    }
    return 0;
}
