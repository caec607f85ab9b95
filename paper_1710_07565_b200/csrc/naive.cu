// Brute-force edge oracle on the GPU (oracle.hpp:41-54 naive_edges): every
// pair u < v of a given point set with hyperbolic_distance(p_u, p_v) < R by
// the direct formula (geometry.hpp:117-123) — deliberately independent of the
// sweep and of the precomputed adjacency test, like the reference's.  Used by
// verify_against_oracle (oracle.hpp:106-111) as a fast GPU check for
// n <= naive_oracle_guard = 100000.
#include <cstdint>

#include <cuda_runtime.h>

#include "device.cuh"

namespace rhgb {
namespace {

constexpr int kNT = 128; // pair tile edge

__device__ __forceinline__ double acosh_clamped(double x) { return x <= 1.0 ? 0.0 : acosh(x); }

// geometry.hpp:117-123, operands in the reference's canonical order (r1 <= r2)
__device__ __forceinline__ double hyperbolic_distance(double ra, double ta, double sa, double rb, double tb, double sb) {
    const bool   o  = ra <= rb;
    const double r1 = o ? ra : rb, r2 = o ? rb : ra;
    const double s1 = o ? sa : sb, s2 = o ? sb : sa;
    const double arg = fadd(cosh(fsub(r2, r1)), fmul(fmul(fsub(1.0, cos(fabs(fsub(ta, tb)))), s1), s2));
    return acosh_clamped(arg);
}

__global__ void __launch_bounds__(kNT) naive_pairs_kernel(const double* __restrict__ r, const double* __restrict__ th,
                                                           const double* __restrict__ sh, std::uint64_t n, double R,
                                                           std::uint64_t nT, ulonglong2* __restrict__ out,
                                                           unsigned long long cap, unsigned long long* count) {
    __shared__ double sr[kNT], st[kNT], ss[kNT];
    const std::uint64_t t  = blockIdx.x;
    // tile t -> (I, J), I <= J, row-major over the upper triangle
    const double  fn = double(nT) + 0.5;
    std::uint64_t I  = std::uint64_t(fn - sqrt(fn * fn - 2.0 * double(t)));
    auto start = [nT](std::uint64_t q) { return q * nT - q * (q - 1) / 2; };
    while (I > 0 && start(I) > t) --I;
    while (start(I + 1) <= t) ++I;
    const std::uint64_t J   = I + (t - start(I));
    const std::uint64_t col = J * kNT + threadIdx.x;
    if (col < n) sr[threadIdx.x] = r[col], st[threadIdx.x] = th[col], ss[threadIdx.x] = sh[col];
    __syncthreads();
    const std::uint64_t i = I * kNT + threadIdx.x;
    if (i >= n) return;
    const double ri = r[i], ti = th[i], si = sh[i];
    std::uint64_t k0 = J * kNT;
    if (k0 <= i) k0 = i + 1;
    const std::uint64_t k1 = (J + 1) * kNT < n ? (J + 1) * kNT : n;
    for (std::uint64_t k = k0; k < k1; ++k) {
        const std::uint32_t c = std::uint32_t(k - J * kNT);
        if (hyperbolic_distance(ri, ti, si, sr[c], st[c], ss[c]) < R) {
            const unsigned long long slot = atomicAdd(count, 1ull);
            if (slot < cap) out[slot] = make_ulonglong2(i, k);
        }
    }
}

__global__ void sinh_kernel(const double* __restrict__ r, double* __restrict__ sh, std::uint64_t n) {
    const std::uint64_t i = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) sh[i] = sinh(r[i]);
}

} // namespace

// All pairs of n points (device arrays r, theta; scratch sh of n doubles) with
// distance < R into out (cap pairs); *count (device) receives the total.
void launch_naive_pairs(const double* r, const double* theta, double* sh, std::uint64_t n, double R, ulonglong2* out,
                        unsigned long long cap, unsigned long long* count, cudaStream_t st) {
    cudaMemsetAsync(count, 0, sizeof(unsigned long long), st);
    if (n < 2) return;
    sinh_kernel<<<unsigned((n + 255) / 256), 256, 0, st>>>(r, sh, n);
    const std::uint64_t nT = (n + kNT - 1) / kNT, tiles = nT * (nT + 1) / 2;
    naive_pairs_kernel<<<unsigned(tiles), kNT, 0, st>>>(r, theta, sh, n, R, nT, out, cap, count);
}

} // namespace rhgb
