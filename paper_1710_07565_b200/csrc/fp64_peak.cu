// FP64-pipe peak probe: the roofline denominator for the edge kernels
// (MEASURED_PEAKS.json has no FP64 entry).  Measures the non-FMA DMUL+DADD
// instruction rate the predicate is made of, and the dependent-DMUL latency
// that bounds the serial sorted-uniform chain (sampler.cu S3).
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/rhg_b200.h"

namespace {

constexpr int kChains = 8;

__global__ void fp64_throughput_kernel(double* out, int iters, double m, double c) {
    double x[kChains];
#pragma unroll
    for (int k = 0; k < kChains; ++k) x[k] = 1.0 + 1e-9 * (threadIdx.x + k);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < kChains; ++k) x[k] = __dadd_rn(__dmul_rn(x[k], m), c); // 1 DMUL + 1 DADD
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < kChains; ++k) s += x[k];
    if (s == 12345.678) out[0] = s; // keep the work alive
}

__global__ void fp64_latency_kernel(double* out, long long* cycles, int iters, double m) {
    double          x  = out[1];
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) x = __dmul_rn(x, m);
    const long long t1 = clock64();
    out[0]             = x;
    cycles[0]          = t1 - t0;
}

} // namespace

extern "C" int rhg_fp64_peak(int device, double* ops_per_s, double* dmul_latency_cycles, double* kernel_ms) {
    if (cudaSetDevice(device) != cudaSuccess) return RHG_CUDA;
    cudaDeviceProp prop{};
    cudaGetDeviceProperties(&prop, device);
    double*    d   = nullptr;
    long long* cyc = nullptr;
    if (cudaMalloc(&d, 2 * sizeof(double)) != cudaSuccess) return RHG_CUDA;
    cudaMalloc(&cyc, sizeof(long long));
    const double init[2] = {0.0, 1.0};
    cudaMemcpy(d, init, sizeof init, cudaMemcpyHostToDevice);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int blocks = prop.multiProcessorCount * 8, threads = 256, iters = 4096;
    float     best   = 1e30f;
    for (int rep = 0; rep < 6; ++rep) {
        cudaEventRecord(a);
        fp64_throughput_kernel<<<blocks, threads>>>(d, iters, 0.999999999, 1e-12);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        if (rep > 0 && ms < best) best = ms;
    }
    const double ops = double(blocks) * threads * iters * kChains * 2.0;
    *ops_per_s       = ops / (best * 1e-3);
    *kernel_ms       = best;
    const int liters = 1 << 16;
    fp64_latency_kernel<<<1, 1>>>(d, cyc, liters, 0.999999999);
    long long c = 0;
    cudaMemcpy(&c, cyc, sizeof c, cudaMemcpyDeviceToHost);
    *dmul_latency_cycles = double(c) / liters;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(d);
    cudaFree(cyc);
    return cudaGetLastError() == cudaSuccess ? RHG_OK : RHG_CUDA;
}
