// Shared device definitions for the B200 (sm_100a) threshold-RHG kernels.
//
// Every arithmetic step that the reference performs in FP64 with plain
// IEEE rounding and NO fused multiply-add (proj/CMakeLists.txt: -O3, no
// -march) is written with __dmul_rn / __dadd_rn / __dsub_rn, which nvcc
// never contracts into DFMA; the TUs are also compiled with --fmad=false.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "glibc_libm.cuh"

namespace rhgb {

constexpr double kTwoPiD = 6.283185307179586476925286766559; // geometry.hpp:11
constexpr double kPiD    = 3.14159265358979323846;           // M_PI

// Per-annulus constants (partition.hpp:42-45) plus this shard's extended
// point-array geometry for streaming annuli.
struct AnnulusDev {
    double lower, coth_lower, cris, cal, cau; // cris = cosh(R)/sinh(lower)
    // streaming annuli only:
    std::uint64_t off, halo, end;      // [off, halo) owned chunks, [halo, end) halo chunk
    std::int64_t  dlt0, dlt1;          // id = idx + dlt0 (idx < halo) else idx + dlt1
    double        cell_origin, cell_inv_w;
    std::uint64_t cell_off;            // into the beta- and lambda-cell tables
    std::uint32_t ncells, pad;
    std::uint64_t wrap;                // first sorted owned index with lambda >= 2pi (device-written; halo if none)
};

// One sorted-uniform / radius stream pair = one (annulus, chunk) point
// source (sweep.hpp:102-111), written to [out_off, out_off + count).
struct StreamJob {
    std::uint64_t out_off, count;
    double        a, b;               // chunk angular bounds (sweep.hpp:80-85)
    std::uint32_t annulus, lift;      // lift: halo copy of chunk 0 seen from chunk P-1
    std::uint32_t chunk, pad;
};

// rng.hpp:15-19 + 41-46: derive_seed(root, {phase, annulus, chunk}) of a stream,
// computed where the stream is drawn (the host plan no longer carries seeds).
__device__ __forceinline__ std::uint64_t splitmix_mix_d(std::uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ std::uint64_t stream_seed(std::uint64_t root, std::uint64_t phase, std::uint64_t annulus,
                                                     std::uint64_t chunk) {
    constexpr std::uint64_t kG = 0x9E3779B97F4A7C15ull;
    std::uint64_t           h  = splitmix_mix_d(root + kG);
    h                          = splitmix_mix_d((h + kG) ^ phase);
    h                          = splitmix_mix_d((h + kG) ^ annulus);
    return splitmix_mix_d((h + kG) ^ chunk);
}

struct Counters { // one per edge-producing kernel family
    unsigned long long edges, fp, comps;
};
struct SlotCounter { // one of kSlots partial counters of a family (32 B apart)
    unsigned long long edges, fp, comps, pad;
};
constexpr int kSlots = 4096;

__device__ __forceinline__ double fmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double fadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double fsub(double a, double b) { return __dsub_rn(a, b); }

// sweep.hpp:60-67 request_half_width_raw; acos is glibc's (glibc_libm.cuh), bit for bit.
__device__ __forceinline__ double request_half_width(double coth_r, double inv_r, double coth_b, double cris_b) {
    const double arg = fsub(fmul(coth_r, coth_b), fmul(cris_b, inv_r));
    if (arg <= -1.0) return kPiD;
    if (arg >= 1.0) return 0.0;
    return gl::gl_acos(arg);
}
// sweep.hpp:365-370 half_width_in
__device__ __forceinline__ double half_width_in(const AnnulusDev& A, double coth_r, double inv_r) {
    if (A.lower <= 0.0) return kPiD;
    return request_half_width(coth_r, inv_r, A.coth_lower, A.cris);
}

// Order-preserving key of a non-negative double (window bounds are clamped
// at +0 first; node angles are always >= +0): integer compares replace FP64
// compares in the pair loops, keeping the FP64 pipe for the predicate.
__device__ __forceinline__ unsigned long long nonneg_key(double x) {
    return x > 0.0 ? static_cast<unsigned long long>(__double_as_longlong(x)) : 0ull;
}

} // namespace rhgb
