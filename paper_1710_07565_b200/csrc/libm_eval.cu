// Verification hook for glibc_libm.cuh: the device restatement of the glibc 2.39
// routines the reference's point set passes through, evaluated elementwise.
// tests/test_gpu_libm.py compares every result bit for bit with the host libm
// (the library the reference links) on seeded inputs from the sampler's argument
// ranges; tools/libm/check_host.cpp runs the same source on the CPU.
#include "../../include/rhg_b200.h"
#include "device.cuh"

namespace rhgb {
namespace {

__global__ void libm_eval_kernel(int fn, const double* __restrict__ x, const double* __restrict__ y,
                                 double* __restrict__ out, std::uint64_t n) {
    for (std::uint64_t i = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += std::uint64_t(gridDim.x) * blockDim.x) {
        const double a = x[i];
        double       r = 0.0;
        switch (fn) {
        case 0: r = gl::gl_exp(a); break;
        case 1: r = gl::gl_log(a); break;
        case 2: r = gl::gl_log1p(a); break;
        case 3: r = gl::gl_acosh(a); break;
        case 4: r = gl::gl_acos(a); break;
        case 5: r = gl::gl_pow(a, y[i]); break;
        case 6:
        case 7: {
            double s, c;
            gl::gl_sincos(a, &s, &c);
            r = fn == 6 ? s : c;
            break;
        }
        }
        out[i] = r;
    }
}

} // namespace
} // namespace rhgb

extern "C" int rhg_libm_eval(int device, int fn, const double* x, const double* y, double* out, uint64_t n) {
    if (fn < 0 || fn > 7 || !x || !out || (fn == 5 && !y)) return RHG_INVALID_ARGUMENT;
    if (n == 0) return RHG_OK;
    if (cudaSetDevice(device) != cudaSuccess) return RHG_CUDA;
    double *dx = nullptr, *dy = nullptr, *dout = nullptr;
    const size_t bytes = size_t(n) * sizeof(double);
    bool ok = cudaMalloc(&dx, bytes) == cudaSuccess && cudaMalloc(&dout, bytes) == cudaSuccess &&
              (fn != 5 || cudaMalloc(&dy, bytes) == cudaSuccess);
    ok = ok && cudaMemcpy(dx, x, bytes, cudaMemcpyHostToDevice) == cudaSuccess &&
         (fn != 5 || cudaMemcpy(dy, y, bytes, cudaMemcpyHostToDevice) == cudaSuccess);
    if (ok) {
        rhgb::libm_eval_kernel<<<148 * 8, 256>>>(fn, dx, dy, dout, n);
        ok = cudaGetLastError() == cudaSuccess && cudaMemcpy(out, dout, bytes, cudaMemcpyDeviceToHost) == cudaSuccess;
    }
    cudaFree(dx);
    cudaFree(dy);
    cudaFree(dout);
    return ok ? RHG_OK : RHG_CUDA;
}
