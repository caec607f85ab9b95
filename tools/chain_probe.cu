// Micro-probe of the serial sorted-uniform chain (sampler.cu S3): cycles per
// chain step for several kernel shapes, alone and beside FP64 load.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o chain_probe tools/chain_probe.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

constexpr int kQ = 16, kT = 32 * kQ;

// (a) lane 0 runs the chain from shared memory (current product kernel shape)
__global__ void __launch_bounds__(32) chain_smem(double* x, long n, long long* cyc) {
    __shared__ __align__(16) double tile[kT];
    const int lane = threadIdx.x;
    double* p = x + blockIdx.x * n;
    double cur = 1.0, nxt[kQ];
    long long t0 = clock64();
    for (int q = 0; q < kQ; ++q) { long k = lane + 32 * q; nxt[q] = k < n ? p[k] : 1.0; }
    for (long base = 0; base < n; base += kT) {
        for (int q = 0; q < kQ; ++q) tile[lane + 32 * q] = nxt[q];
#pragma unroll
        for (int q = 0; q < kQ; ++q) { long k = base + kT + lane + 32 * q; nxt[q] = k < n ? p[k] : 1.0; }
        __syncwarp();
        if (lane == 0) {
            const double2* t2 = reinterpret_cast<const double2*>(tile);
            double2* o2 = reinterpret_cast<double2*>(tile);
            constexpr int kB = 8;
            double2 A[kB];
#pragma unroll
            for (int i = 0; i < kB; ++i) A[i] = t2[i];
#pragma unroll 1
            for (int bb = 0; bb < kT / 2; bb += kB) {
                double2 B[kB];
                const int nb2 = bb + kB < kT / 2 ? bb + kB : bb;
#pragma unroll
                for (int i = 0; i < kB; ++i) B[i] = t2[nb2 + i];
#pragma unroll
                for (int i = 0; i < kB; ++i) {
                    double2 o;
                    cur = __dmul_rn(cur, A[i].x), o.x = cur;
                    cur = __dmul_rn(cur, A[i].y), o.y = cur;
                    o2[bb + i] = o;
                }
#pragma unroll
                for (int i = 0; i < kB; ++i) A[i] = B[i];
            }
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < kQ; ++q) {
            long k = base + lane + 32 * q;
            double y = __dadd_rn(0.1, __dmul_rn(0.5, __dsub_rn(1.0, tile[lane + 32 * q])));
            if (k < n) p[k] = y;
        }
        __syncwarp();
    }
    if (lane == 0) cyc[blockIdx.x] = clock64() - t0;
}

// (b) pure register chain: n dependent DMULs (the floor)
__global__ void chain_reg(double* x, long n, long long* cyc) {
    double cur = x[blockIdx.x], m = x[blockIdx.x + 1] * 0.0 + 0.999999;
    long long t0 = clock64();
    for (long i = 0; i < n; ++i) cur = __dmul_rn(cur, m);
    long long t1 = clock64();
    if (threadIdx.x == 0) { x[blockIdx.x] = cur; cyc[blockIdx.x] = t1 - t0; }
}

// (c) lane-0 chain from smem without stores of the products (is STS the cost?)
__global__ void __launch_bounds__(32) chain_lds_only(double* x, long n, long long* cyc) {
    __shared__ __align__(16) double tile[kT];
    const int lane = threadIdx.x;
    for (int q = 0; q < kQ; ++q) tile[lane + 32 * q] = 1.0 - 1e-12 * (lane + q);
    __syncwarp();
    double cur = 1.0;
    long long t0 = clock64();
    if (lane == 0) {
        const double2* t2 = reinterpret_cast<const double2*>(tile);
        for (long base = 0; base < n; base += kT) {
#pragma unroll 4
            for (int i = 0; i < kT / 2; ++i) {
                const double2 a = t2[i];
                cur = __dmul_rn(cur, a.x);
                cur = __dmul_rn(cur, a.y);
            }
        }
        x[blockIdx.x] = cur;
        cyc[blockIdx.x] = clock64() - t0;
    }
}


// (d) lane 0 chain, ping-pong register batches (no moves), products stored per pair
__global__ void __launch_bounds__(32) chain_pp(double* x, long n, long long* cyc) {
    __shared__ __align__(16) double tile[kT];
    const int lane = threadIdx.x;
    double* p = x + blockIdx.x * n;
    double cur = 1.0, nxt[kQ];
    long long t0 = clock64();
    for (int q = 0; q < kQ; ++q) { long k = lane + 32 * q; nxt[q] = k < n ? p[k] : 1.0; }
    for (long base = 0; base < n; base += kT) {
        for (int q = 0; q < kQ; ++q) tile[lane + 32 * q] = nxt[q];
#pragma unroll
        for (int q = 0; q < kQ; ++q) { long k = base + kT + lane + 32 * q; nxt[q] = k < n ? p[k] : 1.0; }
        __syncwarp();
        if (lane == 0) {
            const double2* t2 = reinterpret_cast<const double2*>(tile);
            double2* o2 = reinterpret_cast<double2*>(tile);
            constexpr int kB = 8;
            double2 A[kB], B[kB];
#pragma unroll
            for (int i = 0; i < kB; ++i) A[i] = t2[i];
#pragma unroll 1
            for (int bb = 0; bb < kT / 2; bb += 2 * kB) {
#pragma unroll
                for (int i = 0; i < kB; ++i) B[i] = t2[bb + kB + i];
#pragma unroll
                for (int i = 0; i < kB; ++i) {
                    double2 o;
                    cur = __dmul_rn(cur, A[i].x), o.x = cur;
                    cur = __dmul_rn(cur, A[i].y), o.y = cur;
                    o2[bb + i] = o;
                }
                const int na = bb + 2 * kB < kT / 2 ? bb + 2 * kB : 0;
#pragma unroll
                for (int i = 0; i < kB; ++i) A[i] = t2[na + i];
#pragma unroll
                for (int i = 0; i < kB; ++i) {
                    double2 o;
                    cur = __dmul_rn(cur, B[i].x), o.x = cur;
                    cur = __dmul_rn(cur, B[i].y), o.y = cur;
                    o2[bb + kB + i] = o;
                }
            }
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < kQ; ++q) {
            long k = base + lane + 32 * q;
            double y = __dadd_rn(0.1, __dmul_rn(0.5, __dsub_rn(1.0, tile[lane + 32 * q])));
            if (k < n) p[k] = y;
        }
        __syncwarp();
    }
    if (lane == 0) cyc[blockIdx.x] = clock64() - t0;
}

__global__ void fp64_load(double* out, int iters) {
    double a = threadIdx.x * 1e-9 + 1.0, b = a + 1, c = a + 2, d = a + 3;
    for (int i = 0; i < iters; ++i) {
        a = __dmul_rn(a, 0.9999999); b = __dmul_rn(b, 0.9999999); c = __dmul_rn(c, 0.9999999); d = __dmul_rn(d, 0.9999999);
    }
    if (a + b + c + d == 1.2345) out[0] = a;
}

int main() {
    const long n = 131072;
    const int G = 1024;
    double* x; long long* cyc;
    cudaMalloc(&x, sizeof(double) * n * G);
    cudaMalloc(&cyc, sizeof(long long) * G);
    std::vector<double> h(n * G);
    for (long i = 0; i < n * G; ++i) h[i] = 1.0 - 1e-7 * double(i % 1000);
    std::vector<long long> hc(G);
    cudaStream_t s2; cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto run = [&](const char* name, auto k, int grid, bool load) {
        cudaMemcpy(x, h.data(), sizeof(double) * n * G, cudaMemcpyHostToDevice);
        for (int rep = 0; rep < 2; ++rep) {
            if (load) fp64_load<<<148 * 4, 256, 0, s2>>>(x + n * G - 1, 20000);
            cudaEventRecord(e0);
            k<<<grid, 32>>>(x, n, cyc);
            cudaEventRecord(e1);
            cudaDeviceSynchronize();
        }
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        cudaMemcpy(hc.data(), cyc, sizeof(long long) * grid, cudaMemcpyDeviceToHost);
        long long mx = 0; for (int i = 0; i < grid; ++i) mx = hc[i] > mx ? hc[i] : mx;
        std::printf("%-28s grid %3d load %d: %.3f ms  %.2f cycles/step (max over CTAs)  err=%s\n", name, grid, int(load), ms,
                    double(mx) / double(n), cudaGetErrorString(cudaGetLastError()));
    };
    run("chain_reg", chain_reg, 1, false);
    run("chain_smem", chain_smem, 1, false);
    run("chain_pp", chain_pp, 1, false);
    for (int g : {148, 296, 592, 1024}) {
        run("chain_reg", chain_reg, g, false);
        run("chain_smem", chain_smem, g, false);
        run("chain_pp", chain_pp, g, false);
    }
    run("chain_pp", chain_pp, 64, true);
    return 0;
}
