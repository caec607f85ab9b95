// Device point sampler (sm_100a): the reference's ChunkPointSource
// (sweep.hpp:102-141) for every (annulus, chunk) stream of a shard.
//
//   S1 angle_side_kernel    one CTA per chain bin (the host packs each wave's
//                           streams longest-first into bins of about the longest
//                           chain): per stream, a 3-stage pipeline over 312-value
//                           blocks — std::mt19937_64 seeded by derive_seed(seed,
//                           {3,i,c}) (rng.hpp:41-69, warp-parallel twist), the
//                           factors pow(U_k, 1/remaining) (rng.hpp:221), and the
//                           serial product chain cur *= x_k with beta = a + w (1 -
//                           cur), clamped (rng.hpp:218-229) — the only serial
//                           dependency, run by one lane from shared memory.
//   S2 mt_uniforms_kernel   one CTA per (stream, radii): the radius uniforms
//                           (seed {4,i,c}), a block-wide two-phase twist.
//      point_radial_kernel  per point, on a side stream beside S1: the radius-only
//                           attributes r, coth r, 1/sinh r, half-width
//                           (partition.hpp:64-70, sweep.hpp:121-134).
//   S3 point_angular_kernel per global point: theta = beta + hw (mod 2pi), cos, sin
//                           (sweep.hpp:135-139); streaming points get theirs in the
//                           sort phase (edges.cu rank_kernel, angular_scatter_point).
//
// All exact-rounding steps use __dmul_rn/__dadd_rn (no FMA contraction); pow, acosh,
// exp, acos and sincos are glibc 2.39's, restated bit for bit in glibc_libm.cuh.
#include <cstdlib>

#include "device.cuh"
#include "kernels.hpp"

namespace rhgb {

namespace {

constexpr int kMtN = 312, kMtM = 156;

__device__ __forceinline__ std::uint64_t mt_temper(std::uint64_t y) {
    y ^= (y >> 29) & 0x5555555555555555ull;
    y ^= (y << 17) & 0x71D67FFFEDA60000ull;
    y ^= (y << 37) & 0xFFF7EEE000000000ull;
    return y ^ (y >> 43);
}
__device__ __forceinline__ std::uint64_t mt_mix(std::uint64_t cur, std::uint64_t nxt, std::uint64_t far) {
    const std::uint64_t x = (cur & 0xFFFFFFFF80000000ull) | (nxt & 0x7FFFFFFFull);
    return far ^ (x >> 1) ^ ((x & 1ull) ? 0xB5026F5AA96619E9ull : 0ull);
}

// Out-of-place twist: B = twist(A), equal to the in-place sequential twist of
// [rand.predef] (words 0..155 read old words only, 156..310 read new words
// i-156, word 311 reads new words 0 and 155).
__device__ __forceinline__ void mt_twist_to(const std::uint64_t* __restrict__ A, std::uint64_t* __restrict__ B,
                                            int lane) {
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const int i = lane + 32 * k;
        if (i < kMtN - kMtM) B[i] = mt_mix(A[i], A[i + 1], A[i + kMtM]);
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const int i = kMtN - kMtM + lane + 32 * k;
        if (i < kMtN - 1) B[i] = mt_mix(A[i], A[i + 1], B[i - (kMtN - kMtM)]);
    }
    if (lane == 0) B[kMtN - 1] = mt_mix(A[kMtN - 1], B[0], B[kMtM - 1]);
    __syncwarp();
}

#ifndef RHG_MT_THREADS
#define RHG_MT_THREADS 320 // measured cfg2: 160 -> 4.12 ms/step, 320 -> 4.07
#endif
constexpr int kMtThreads = RHG_MT_THREADS; // >= 156: one state word per thread and twist phase
// radius streams from which mt_radial_kernel runs (measured cfg3 22.13 -> 22.02 ms, cfg4 33.55 ->
// 33.20, cfg5 155.9 -> 154.1; cfg2's 832 long streams: 3.20 -> 3.58 fused)
constexpr int kFusedRadialJobs = 4096;

// One CTA per (stream, {angles, radii}): thread 0 seeds ([rand.predef]
// seeding recurrence, serial by definition); then per 312-word block the
// whole CTA regenerates the state out of place in two phases (words 0..155
// read old words only; 156..311 read new words 0..155), one word per thread
// and phase, while tempering the previous block into (x >> 11) * 2^-53,
// written coalesced — two barriers per block.  A long stream's serial chain of
// twists (the radius side's critical path) is then two shared-memory round
// trips per block instead of a warp walking 5 words per phase.
// which: 0 = both streams of every job, 1 = angle streams only, 2 = radius streams only
__global__ void __launch_bounds__(kMtThreads) mt_uniforms_kernel(const StreamJob* __restrict__ jobs, int njobs,
                                                                 double* __restrict__ u_ang,
                                                                 double* __restrict__ u_rad, int which,
                                                                 std::uint64_t seed) {
    static_assert(kMtThreads >= kMtN - kMtM && kMtThreads % 32 == 0, "one twist word per thread and phase");
    __shared__ std::uint64_t st[2][kMtN]; // st[k & 1]: the state after k twists
    const int t  = threadIdx.x;
    const int gw = blockIdx.x;
    if (gw >= (which ? 1 : 2) * njobs) return;
    const StreamJob&    J   = jobs[which ? gw : gw >> 1];
    const bool          ang = which ? which == 1 : (gw & 1) == 0;
    double*             dst = (ang ? u_ang : u_rad) + J.out_off;
    const std::uint64_t n   = J.count;
    if (n == 0) return;
    if (t == 0) {
        std::uint64_t x = stream_seed(seed, ang ? 3 : 4, J.annulus, J.chunk); // kPhaseAngles / kPhaseRadii
        st[0][0]        = x;
        for (int i = 1; i < kMtN; ++i) {
            x        = 6364136223846793005ull * (x ^ (x >> 62)) + std::uint64_t(i);
            st[0][i] = x;
        }
    }
    __syncthreads();
    const std::uint64_t nblk = (n + kMtN - 1) / kMtN;
    for (std::uint64_t k = 0; k <= nblk; ++k) {
        const std::uint64_t* A = st[k & 1];       // the state after k twists (block k - 1)
        std::uint64_t*       B = st[(k + 1) & 1]; // block k
        if (k > 0) { // temper and store block k - 1
            const std::uint64_t base = (k - 1) * kMtN;
            const int           cnt  = n - base < std::uint64_t(kMtN) ? int(n - base) : kMtN;
            for (int i = t; i < cnt; i += kMtThreads) dst[base + i] = double(mt_temper(A[i]) >> 11) * 0x1.0p-53;
        }
        if (k < nblk) {
            if (t < kMtN - kMtM) B[t] = mt_mix(A[t], A[t + 1], A[t + kMtM]);
            __syncthreads();
            if (t < kMtN - kMtM) {
                const int i = kMtN - kMtM + t;
                B[i] = i < kMtN - 1 ? mt_mix(A[i], A[i + 1], B[t]) : mt_mix(A[kMtN - 1], B[0], B[kMtM - 1]);
            }
        }
        __syncthreads();
    }
}

__device__ __forceinline__ int find_job(const StreamJob* __restrict__ jobs, int njobs, std::uint64_t i) {
    int lo = 0, hi = njobs - 1; // last job with out_off <= i
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (jobs[mid].out_off <= i) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// partition.hpp:64-70 radius_from_uniform, then sweep.hpp:125-134.
// The annulus of point i from the point-segment table (pseg[s] = first point << 8 | annulus,
// ascending, pseg[nseg] = total << 8): one search per block for its first point, and a
// per-thread search only past that segment's end (blocks rarely straddle two annuli).
__device__ __forceinline__ int pseg_find(const std::uint64_t* __restrict__ pseg, int nseg, std::uint64_t i) {
    int lo = 0, hi = nseg - 1; // last segment starting at or before i
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if ((pseg[mid] >> 8) <= i) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}
// The radius-only attributes of one point from its radius uniform u (partition.hpp:64-70,
// sweep.hpp:121-134).
__device__ __forceinline__ void radial_point(const AnnulusDev& A, double alpha, double u, double& hw, double2& rec2,
                                             double& r) {
    const double c = fadd(A.cal, fmul(u, fsub(A.cau, A.cal)));
    r              = __ddiv_rn(gl::gl_acosh(c < 1.0 ? 1.0 : c), alpha);
    r              = r > 1e-12 ? r : 1e-12;
    const double ex   = gl::gl_exp(r);
    const double mex  = __ddiv_rn(1.0, ex);
    const double sh   = fmul(0.5, fsub(ex, mex));
    const double coth = __ddiv_rn(fmul(0.5, fadd(ex, mex)), sh);
    const double inv  = __ddiv_rn(1.0, sh);
    hw                = A.lower > 0.0 ? request_half_width(coth, inv, A.coth_lower, A.cris) : kPiD;
    rec2              = make_double2(coth, inv);
}
__global__ void point_radial_kernel(const std::uint64_t* __restrict__ pseg, int nseg, const AnnulusDev* __restrict__ ann,
                                    double alpha, std::uint64_t first, std::uint64_t total, double* __restrict__ hw_out,
                                    double2* __restrict__ rec2, double* __restrict__ r_out) {
    const std::uint64_t i0 = first + std::uint64_t(blockIdx.x) * blockDim.x; // points [first, total)
    const std::uint64_t i  = i0 + threadIdx.x;
    __shared__ int           s_a;
    __shared__ std::uint64_t s_end;
    if (threadIdx.x == 0) {
        const int sg = pseg_find(pseg, nseg, i0);
        s_a = int(pseg[sg] & 0xffu), s_end = pseg[sg + 1] >> 8;
    }
    __syncthreads();
    if (i >= total) return;
    const int a = i < s_end ? s_a : int(pseg[pseg_find(pseg, nseg, i)] & 0xffu);
    double    hw, r;
    double2   q;
    radial_point(ann[a], alpha, hw_out[i], hw, q, r);
    hw_out[i] = hw;
    rec2[i]   = q;
    if (r_out) r_out[i] = r;
}

// The radius side of one stream in one CTA for many short streams (small average degree, large
// P): mt_uniforms_kernel's radius stream (seed {4, annulus, chunk}) with each tempered block turned
// straight into the radius attributes, so the uniforms never go through HBM and the attributes'
// FP64 work overlaps other streams' twists (few long streams leave it latency-bound: cfg2).
__global__ void __launch_bounds__(kMtThreads) mt_radial_kernel(const StreamJob* __restrict__ jobs, int njobs,
                                                               const AnnulusDev* __restrict__ ann, double alpha,
                                                               double* __restrict__ hw_out, double2* __restrict__ rec2,
                                                               double* __restrict__ r_out, std::uint64_t seed) {
    __shared__ std::uint64_t st[2][kMtN];
    const int t = threadIdx.x;
    if (int(blockIdx.x) >= njobs) return;
    const StreamJob&    J = jobs[blockIdx.x];
    const std::uint64_t n = J.count;
    if (n == 0) return;
    const AnnulusDev& A = ann[J.annulus];
    if (t == 0) {
        std::uint64_t x = stream_seed(seed, 4, J.annulus, J.chunk); // kPhaseRadii
        st[0][0]        = x;
        for (int i = 1; i < kMtN; ++i) {
            x        = 6364136223846793005ull * (x ^ (x >> 62)) + std::uint64_t(i);
            st[0][i] = x;
        }
    }
    __syncthreads();
    const std::uint64_t nblk = (n + kMtN - 1) / kMtN;
    for (std::uint64_t k = 0; k <= nblk; ++k) {
        const std::uint64_t* S = st[k & 1];       // the state after k twists (block k - 1)
        std::uint64_t*       B = st[(k + 1) & 1]; // block k
        std::uint64_t        w = 0, idx = 0;
        bool                 have = false;
        if (k > 0) { // this thread's word of block k - 1 (read before the state is rewritten)
            idx  = (k - 1) * kMtN + std::uint64_t(t);
            have = t < kMtN && idx < n;
            if (have) w = S[t];
        }
        if (k < nblk) {
            if (t < kMtN - kMtM) B[t] = mt_mix(S[t], S[t + 1], S[t + kMtM]);
            __syncthreads();
            if (t < kMtN - kMtM) {
                const int i = kMtN - kMtM + t;
                B[i] = i < kMtN - 1 ? mt_mix(S[i], S[i + 1], B[t]) : mt_mix(S[kMtN - 1], B[0], B[kMtM - 1]);
            }
        }
        __syncthreads();
        if (have) {
            double  hw, r;
            double2 q;
            radial_point(A, alpha, double(mt_temper(w) >> 11) * 0x1.0p-53, hw, q, r);
            const std::uint64_t i = J.out_off + idx;
            hw_out[i] = hw;
            rec2[i]   = q;
            if (r_out) r_out[i] = r;
        }
    }
}

// The whole angle side of one chain bin in one CTA (rng.hpp:58-69 + 209-244):
// warp 1 regenerates the stream's std::mt19937_64 output (seeding, warp-
// parallel twist, tempering -> 53-bit uniforms) one 312-value block at a time,
// warps 2.. turn block b-1 into the factors pow(U_k, 1/remaining_k) (about
// one per thread: pow's latency, not its throughput, bounds the stage), and
// warp 0 runs the serial chain cur = fl(cur * x_k) over block b-2 (lane 0,
// from shared memory), and the pow warps also map block b-3's products to
// beta_k = a + w (1 - cur) (clamped) — a four-stage pipeline with one
// __syncthreads per block in which the chain warp does nothing but the chain
// (the only serial dependency), starting after the first two blocks instead
// of after two full-array kernels.  Same arithmetic, same order as the separate
// mt_uniforms / point_pow / sorted_chain kernels.
#ifndef RHG_ANG_WARPS
#define RHG_ANG_WARPS 8 // measured: 6 -> 4.35 ms, 8 -> 4.31, 10 -> 4.34, 12 -> 4.34 (cfg2 step, round 1); round 2: 6 / 8 / 12 / 16 -> cfg4 32.10 / 31.77 / 33.66 / 36.02 ms
#endif
constexpr int kAngWarps = RHG_ANG_WARPS; // warp 0: chain, warp kMtWarp: MT, the others: pow factors
#ifndef RHG_MT_WARP
#define RHG_MT_WARP 4 // shares the chain warp's SM sub-partition (integer work only), so no pow warp does
#endif
constexpr int kMtWarp = RHG_MT_WARP;
#ifndef RHG_CHAIN_KB
#define RHG_CHAIN_KB 6 // double2 per register batch of the chain lane (must divide 78)
#endif
static_assert(78 % RHG_CHAIN_KB == 0, "the chain's batches must tile a 312-value block");
struct AngSmem {
    std::uint64_t st[2][kMtN];   // MT state, double-buffered (warp 1)
    double        u[2][kMtN];    // uniforms of blocks b, b-1
    double        x[3][kMtN];    // pow factors of block b-1, products of b-2, block b-3 being mapped to beta
};
__global__ void __launch_bounds__(32 * kAngWarps) angle_side_kernel(const StreamJob* __restrict__ jobs,
                                                                    const std::uint32_t* __restrict__ bins,
                                                                    int nbins, const std::uint32_t* __restrict__ order,
                                                                    double* __restrict__ beta_out, std::uint64_t seed) {
    __shared__ __align__(16) AngSmem S;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int bin  = blockIdx.x;
    if (bin >= nbins) return;
    for (std::uint32_t jb = bins[bin]; jb < bins[bin + 1]; ++jb) {
        const StreamJob&    J    = jobs[order[jb]];
        const std::uint64_t n    = J.count;
        const std::uint64_t nblk = (n + kMtN - 1) / kMtN;
        double*             p    = beta_out + J.out_off;
        const double        a = J.a, b = J.b, wd = fsub(b, a);
        const double        bmax = nextafter(b, a);
        double              cur  = 1.0; // lane 0 of warp 0
        if (warp == kMtWarp && lane == 0) { // [rand.predef] seeding recurrence (serial by definition)
            std::uint64_t z = stream_seed(seed, 3, J.annulus, J.chunk); // kPhaseAngles
            S.st[0][0]      = z;
            for (int i = 1; i < kMtN; ++i) {
                z          = 6364136223846793005ull * (z ^ (z >> 62)) + std::uint64_t(i);
                S.st[0][i] = z;
            }
        }
        __syncwarp();
        for (std::uint64_t s = 0; s < nblk + 3; ++s) {
            if (warp == kMtWarp && s < nblk) { // block s: state after s + 1 twists
                const std::uint64_t* A = S.st[s & 1];
                std::uint64_t*       B = S.st[(s + 1) & 1];
                mt_twist_to(A, B, lane);
                double* u = S.u[s & 1];
                for (int i = lane; i < kMtN; i += 32) u[i] = double(mt_temper(B[i]) >> 11) * 0x1.0p-53;
            } else if (warp != 0 && warp != kMtWarp) {
                const int pw = warp - 1 - (warp > kMtWarp); // 0 .. kAngWarps - 3
                if (s >= 1 && s <= nblk) {                  // block s - 1: pow factors
                    const std::uint64_t base = (s - 1) * kMtN;
                    const double*       u    = S.u[(s - 1) & 1];
                    double*             x    = S.x[(s - 1) % 3];
                    for (int i = pw * 32 + lane; i < kMtN; i += 32 * (kAngWarps - 2)) {
                        const std::uint64_t k = base + std::uint64_t(i);
                        x[i] = k < n ? gl::gl_pow(u[i], __ddiv_rn(1.0, double(n - k))) : 1.0; // rng.hpp:221, past the end: 1
                    }
                }
                if (s >= 3) { // block s - 3: the chain's products -> beta (off the chain warp's path)
                    const std::uint64_t base = (s - 3) * kMtN;
                    const double*       x    = S.x[(s - 3) % 3];
                    for (int i = pw * 32 + lane; i < kMtN; i += 32 * (kAngWarps - 2)) {
                        const std::uint64_t k = base + std::uint64_t(i);
                        const double        y = fadd(a, fmul(wd, fsub(1.0, x[i])));
                        if (k < n) p[k] = y >= b ? bmax : y;
                    }
                }
            } else if (warp == 0 && s >= 2 && s <= nblk + 1) { // block s - 2: the chain
                double* x = S.x[(s - 2) % 3];
                if (lane == 0) {
                    double2*      x2 = reinterpret_cast<double2*>(x);
                    constexpr int kB = RHG_CHAIN_KB;   // 156 double2 = (78 / kB) batches of 2 kB values
                    double2       A[kB], B[kB];
#pragma unroll
                    for (int i = 0; i < kB; ++i) A[i] = x2[i];
#pragma unroll 1
                    for (int bb = 0; bb < kMtN / 2; bb += 2 * kB) {
#pragma unroll
                        for (int i = 0; i < kB; ++i) B[i] = bb + kB + i < kMtN / 2 ? x2[bb + kB + i] : make_double2(1.0, 1.0);
#pragma unroll
                        for (int i = 0; i < kB; ++i) {
                            double2 o;
                            cur = fmul(cur, A[i].x), o.x = cur;
                            cur = fmul(cur, A[i].y), o.y = cur;
                            x2[bb + i] = o;
                        }
                        if (bb + kB >= kMtN / 2) break;
#pragma unroll
                        for (int i = 0; i < kB; ++i) A[i] = bb + 2 * kB + i < kMtN / 2 ? x2[bb + 2 * kB + i] : make_double2(1.0, 1.0);
#pragma unroll
                        for (int i = 0; i < kB; ++i) {
                            double2 o;
                            cur = fmul(cur, B[i].x), o.x = cur;
                            cur = fmul(cur, B[i].y), o.y = cur;
                            x2[bb + kB + i] = o;
                        }
                    }
                }
                __syncwarp();
            }
            __syncthreads();
        }
    }
}

// sweep.hpp:135-139 + 478-480: node angle, trig, engine-frame begin/centre.
__global__ void point_angular_kernel(const StreamJob* __restrict__ jobs, int njobs, std::uint64_t first,
                                     std::uint64_t total, double* __restrict__ beta, const double* __restrict__ hw,
                                     double2* __restrict__ rec0, double2* __restrict__ rec1,
                                     double* __restrict__ theta_out) {
    const std::uint64_t i = first + std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= total) return;
    const StreamJob& J  = jobs[find_job(jobs, njobs, i)];
    const double     b0 = beta[i];
    const double     h  = hw[i];
    double           th = fadd(b0, h);
    if (th >= kTwoPiD) th = fsub(th, kTwoPiD);
    double s, c;
    gl::gl_sincos(th, &s, &c);
    const double bf = J.lift ? fadd(b0, kTwoPiD) : b0;
    rec0[i]         = make_double2(fadd(bf, h), th);
    rec1[i]         = make_double2(c, s);
    if (theta_out) theta_out[i] = b0; // unlifted beta for point export
    beta[i] = bf;
}

// "Same points" mode: given uploaded beta(unlifted)/hw/theta/cos/sin, build
// the engine frames exactly as S4 does (no libm involved).
__global__ void frames_from_points_kernel(const StreamJob* __restrict__ jobs, int njobs, std::uint64_t total,
                                          double* __restrict__ beta, const double* __restrict__ hw,
                                          double2* __restrict__ rec0) {
    const std::uint64_t i = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= total) return;
    const StreamJob& J  = jobs[find_job(jobs, njobs, i)];
    const double     b0 = beta[i];
    const double     bf = J.lift ? fadd(b0, kTwoPiD) : b0;
    rec0[i].x           = fadd(bf, hw[i]);
    beta[i]             = bf;
}

} // namespace

// Streams: the angle side of every chain bin is one fused kernel
// (angle_side_kernel: MT -> pow -> serial chain -> beta), wave 1 on st and
// wave 2 (the outermost annulus, the longest chains) on S.late, signalling
// S.ev_late, so the inner annuli's sort and edge work overlaps its tail; the
// radius side (MT -> radial attributes) runs on S.side and joins st.
void launch_sampler(const SamplerArgs& S, cudaStream_t st, std::uint64_t* launches) {
    if (S.total == 0 || S.njobs == 0) return;
    cudaStream_t side = S.side ? S.side : st;
    if (S.side) {
        cudaEventRecord(S.ev_fork, st);
        cudaStreamWaitEvent(side, S.ev_fork, 0);
    }
    const bool split = S.wave2_jobs && S.late;
    const int  nb1   = split ? S.chain_bins1 : S.chain_bins_total;
    // the global annuli (few, short streams) on their own stream: their points are ready long
    // before the streaming chains finish, so the global unit runs during the chain phase
    const bool gsplit = split && S.glob && S.ev_glob && S.side && S.glob_job0 < S.njobs && S.chain_bins_g > 0 &&
                        S.total > S.angular_from;
    const int  njs    = gsplit ? S.glob_job0 : S.njobs; // the side stream's radius streams
    if (split && S.chain_bins_total > nb1) {
        cudaEventRecord(S.ev_pow, st);
        cudaStreamWaitEvent(S.late, S.ev_pow, 0);
        angle_side_kernel<<<S.chain_bins_total - nb1, 32 * kAngWarps, 0, S.late>>>(
            S.jobs, S.chain_bins + nb1, S.chain_bins_total - nb1, S.job_order, S.beta, S.seed);
        cudaEventRecord(S.ev_late, S.late);
        S.mark("chain_wave2(late)", S.late);
        ++*launches;
    }
    if (gsplit) {
        cudaStreamWaitEvent(S.glob, S.ev_fork, 0);
        const int ng = S.njobs - S.glob_job0;
        mt_uniforms_kernel<<<ng, kMtThreads, 0, S.glob>>>(S.jobs + S.glob_job0, ng, S.beta, S.hw, 2, S.seed);
        angle_side_kernel<<<S.chain_bins_g, 32 * kAngWarps, 0, S.glob>>>(S.jobs, S.chain_bins, S.chain_bins_g,
                                                                         S.job_order, S.beta, S.seed);
        const std::uint64_t first = S.angular_from;
        point_radial_kernel<<<unsigned((S.total - first + 255) / 256), 256, 0, S.glob>>>(
            S.pseg, S.npseg, S.ann, S.alpha, first, S.total, S.hw, S.rec2, S.r_out);
        point_angular_kernel<<<unsigned((S.total - first + 255) / 256), 256, 0, S.glob>>>(
            S.jobs, S.njobs, first, S.total, S.beta, S.hw, S.rec0, S.rec1, S.beta_unlifted_out);
        cudaEventRecord(S.ev_glob, S.glob);
        S.mark("global_points", S.glob);
        *launches += 4;
    }
    // the radius attributes run beside the angle side (measured at cfg2: serialising them after
    // the wave-1 chains is slower — the wave-1 sort then waits for the whole radius side — and
    // so is splitting them by wave: the GPU is saturated either way). Many short streams (large P):
    // uniforms and attributes fused per stream (RHG_MT_RADIAL=0 / 1 forces either)
    const char* fr    = std::getenv("RHG_MT_RADIAL");
    const bool  fused = fr ? fr[0] == '1' : njs >= kFusedRadialJobs;
    if (fused) {
        mt_radial_kernel<<<njs, kMtThreads, 0, side>>>(S.jobs, njs, S.ann, S.alpha, S.hw, S.rec2, S.r_out, S.seed);
        *launches += 1;
    } else {
        mt_uniforms_kernel<<<njs, kMtThreads, 0, side>>>(S.jobs, njs, S.beta, S.hw, 2, S.seed);
        S.mark("mt_radii", side);
        const std::uint64_t rad_end = gsplit ? S.angular_from : S.total;
        point_radial_kernel<<<unsigned((rad_end + 255) / 256), 256, 0, side>>>(S.pseg, S.npseg, S.ann, S.alpha, 0,
                                                                              rad_end, S.hw, S.rec2, S.r_out);
        *launches += 2;
    }
    S.mark("radial", side);
    const int nbw = gsplit ? S.chain_bins_g : 0; // the main stream's wave-1 bins
    if (nb1 > nbw) {
        angle_side_kernel<<<nb1 - nbw, 32 * kAngWarps, 0, st>>>(S.jobs, S.chain_bins + nbw, nb1 - nbw, S.job_order,
                                                               S.beta, S.seed);
        ++*launches;
    }
    S.mark("chain_wave1", st);
    if (S.side) {
        cudaEventRecord(S.ev_join, side);
        cudaStreamWaitEvent(st, S.ev_join, 0);
    }
    // generate mode: streaming points get their frames in the sort phase (edges.cu rank_kernel, angular_scatter_point)
    const std::uint64_t first = S.angular_from;
    if (S.total > first && !gsplit) {
        point_angular_kernel<<<unsigned((S.total - first + 255) / 256), 256, 0, st>>>(
            S.jobs, S.njobs, first, S.total, S.beta, S.hw, S.rec0, S.rec1, S.beta_unlifted_out);
        *launches += 1;
    }
}

void launch_mt_uniforms(const SamplerArgs& S, cudaStream_t st, std::uint64_t* launches) {
    if (S.total == 0 || S.njobs == 0) return;
    mt_uniforms_kernel<<<2 * S.njobs, kMtThreads, 0, st>>>(S.jobs, S.njobs, S.beta, S.hw, 0, S.seed);
    *launches += 1;
}

void launch_frames_from_points(const SamplerArgs& S, cudaStream_t st, std::uint64_t* launches) {
    if (S.total == 0 || S.njobs == 0) return;
    const unsigned pblocks = unsigned((S.total + 255) / 256);
    frames_from_points_kernel<<<pblocks, 256, 0, st>>>(S.jobs, S.njobs, S.total, S.beta, S.hw, S.rec0);
    *launches += 1;
}

} // namespace rhgb
