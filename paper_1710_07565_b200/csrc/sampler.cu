// Device point sampler (sm_100a): the reference's ChunkPointSource
// (sweep.hpp:102-141) for every (annulus, chunk) stream of a shard.
//
//   S1 mt_uniforms_kernel   one warp per (stream, {angles, radii}): std::mt19937_64
//                           seeded by derive_seed(seed,{3|4,i,c}) (rng.hpp:41-69),
//                           312-word twist done warp-parallel in shared memory,
//                           output (x >> 11) * 2^-53 written coalesced.
//   S2 point_pow_kernel     per point: x_k = pow(U_k, 1/remaining) for the
//                           sorted stream (rng.hpp:221);
//      point_radial_kernel  per point, on a side stream beside S2/S3: the
//                           radius-only attributes r, coth r, 1/sinh r,
//                           half-width (partition.hpp:64-70, sweep.hpp:121-134).
//   S3 sorted_chain_kernel  one warp per angle stream: the serial product
//                           chain cur *= x_k, beta = a + w (1 - cur), clamp
//                           (rng.hpp:218-229) — the only serial dependency.
//   S4 point_angular_kernel per point: theta = beta + hw (mod 2pi), cos, sin,
//                           engine-frame beta/lambda (sweep.hpp:135-139, 478-480).
//
// All exact-rounding steps use __dmul_rn/__dadd_rn (no FMA contraction).
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

// Warp-parallel regeneration of the 312-word state, equal to the sequential
// in-place twist of [rand.predef] mersenne_twister_engine.
__device__ __forceinline__ void mt_twist_warp(std::uint64_t* mt, int lane) {
    std::uint64_t nv[5];
    // words 0..155 read only old words
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const int i = lane + 32 * k;
        if (i < kMtN - kMtM) nv[k] = mt_mix(mt[i], mt[i + 1], mt[i + kMtM]);
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const int i = lane + 32 * k;
        if (i < kMtN - kMtM) mt[i] = nv[k];
    }
    __syncwarp();
    // words 156..310 read new words i-156 and old words i, i+1
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const int i = kMtN - kMtM + lane + 32 * k;
        if (i < kMtN - 1) nv[k] = mt_mix(mt[i], mt[i + 1], mt[i - (kMtN - kMtM)]);
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const int i = kMtN - kMtM + lane + 32 * k;
        if (i < kMtN - 1) mt[i] = nv[k];
    }
    __syncwarp();
    if (lane == 0) mt[kMtN - 1] = mt_mix(mt[kMtN - 1], mt[0], mt[kMtM - 1]);
    __syncwarp();
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

constexpr int kMtWarps = 4;

// One CTA per (stream, {angles, radii}): warp 0 seeds ([rand.predef]
// seeding recurrence, serial by definition) and regenerates the 312-word state
// block k into buffer k % 2 while warps 1..3 temper block k - 1 and write its
// outputs (x >> 11) * 2^-53 coalesced; one __syncthreads per block.  A long
// stream then costs ~one twist per block instead of twist + tempering.
// which: 0 = both streams of every job, 1 = angle streams only, 2 = radius streams only
__global__ void __launch_bounds__(32 * kMtWarps) mt_uniforms_kernel(const StreamJob* __restrict__ jobs, int njobs,
                                                                     double* __restrict__ u_ang,
                                                                     double* __restrict__ u_rad, int which) {
    __shared__ std::uint64_t st[2][kMtN]; // st[k & 1]: the state after k twists
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gw   = blockIdx.x;
    if (gw >= (which ? 1 : 2) * njobs) return;
    const StreamJob&    J   = jobs[which ? gw : gw >> 1];
    const bool          ang = which ? which == 1 : (gw & 1) == 0;
    double*             dst = (ang ? u_ang : u_rad) + J.out_off;
    const std::uint64_t n   = J.count;
    if (n == 0) return;
    if (warp == 0 && lane == 0) {
        std::uint64_t x = ang ? J.seed_ang : J.seed_rad;
        st[0][0]        = x;
        for (int i = 1; i < kMtN; ++i) {
            x        = 6364136223846793005ull * (x ^ (x >> 62)) + std::uint64_t(i);
            st[0][i] = x;
        }
    }
    __syncthreads();
    const std::uint64_t nblk = (n + kMtN - 1) / kMtN;
    for (std::uint64_t k = 0; k <= nblk; ++k) {
        if (warp == 0) {
            if (k < nblk) mt_twist_to(st[k & 1], st[(k + 1) & 1], lane); // block k
        } else if (k > 0) { // temper and store block k - 1 (the state after k twists)
            const std::uint64_t  base = (k - 1) * kMtN;
            const int            cnt  = n - base < std::uint64_t(kMtN) ? int(n - base) : kMtN;
            const std::uint64_t* o    = st[k & 1];
            for (int i = threadIdx.x - 32; i < cnt; i += 32 * (kMtWarps - 1))
                dst[base + i] = double(mt_temper(o[i]) >> 11) * 0x1.0p-53;
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

// rng.hpp:221: cur_max *= pow(U, 1.0 / remaining), remaining = count - k
__global__ void point_pow_kernel(const StreamJob* __restrict__ jobs, int njobs, std::uint64_t total,
                                 double* __restrict__ u_ang) {
    const std::uint64_t i = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= total) return;
    const StreamJob&    J   = jobs[find_job(jobs, njobs, i)];
    const double        rem = double(J.count - (i - J.out_off));
    u_ang[i]                = pow(u_ang[i], __ddiv_rn(1.0, rem));
}

// partition.hpp:64-70 radius_from_uniform, then sweep.hpp:125-134.
__global__ void point_radial_kernel(const StreamJob* __restrict__ jobs, int njobs, const AnnulusDev* __restrict__ ann,
                                    double alpha, std::uint64_t total, double* __restrict__ hw_out,
                                    double2* __restrict__ rec2, double* __restrict__ r_out) {
    const std::uint64_t i = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= total) return;
    const StreamJob&  J = jobs[find_job(jobs, njobs, i)];
    const AnnulusDev& A = ann[J.annulus];
    const double      u = hw_out[i];
    const double      c = fadd(A.cal, fmul(u, fsub(A.cau, A.cal)));
    double            r = __ddiv_rn(acosh(c < 1.0 ? 1.0 : c), alpha);
    r                   = r > 1e-12 ? r : 1e-12;
    const double ex   = exp(r);
    const double mex  = __ddiv_rn(1.0, ex);
    const double sh   = fmul(0.5, fsub(ex, mex));
    const double coth = __ddiv_rn(fmul(0.5, fadd(ex, mex)), sh);
    const double inv  = __ddiv_rn(1.0, sh);
    hw_out[i]         = A.lower > 0.0 ? request_half_width(coth, inv, A.coth_lower, A.cris) : kPiD;
    rec2[i]           = make_double2(coth, inv);
    if (r_out) r_out[i] = r;
}

// rng.hpp:218-229.  One single-warp CTA per chain bin (the host packs the
// streams into bins whose lengths add up to about the longest chain, so few
// chain warps share an SM): for each stream of its bin the 32 lanes stage a
// tile of pow factors into shared memory (coalesced, the next tile prefetched
// into registers), lane 0 alone runs the serial chain cur = fl(cur * x_k)
// over the tile from shared memory (vector loads two batches ahead in
// ping-pong registers, so the loop-carried dependency is one DMUL per point
// and no shuffles), and the warp maps the tile's products to
// beta = a + w (1 - cur), clamped, with a coalesced store.  Past-the-end
// factors are 1.0: fl(cur * 1.0) == cur.
constexpr int kChainQ = 16;               // tile = 32 * kChainQ points
constexpr int kChainT = 32 * kChainQ;
__global__ void __launch_bounds__(32) sorted_chain_kernel(const StreamJob* __restrict__ jobs,
                                                          const std::uint32_t* __restrict__ bins,
                                                          const std::uint32_t* __restrict__ order,
                                                          double* __restrict__ x) {
    __shared__ __align__(16) double tile[kChainT];
    const int lane = threadIdx.x;
    for (std::uint32_t jb = bins[blockIdx.x]; jb < bins[blockIdx.x + 1]; ++jb) {
        const StreamJob&    J = jobs[order[jb]];
        double*             p = x + J.out_off;
        const std::uint64_t n = J.count;
        const double        a = J.a, b = J.b, wd = fsub(b, a);
        const double        bmax = nextafter(b, a);
        double              cur  = 1.0; // lane 0's chain state
        double              nxt[kChainQ];
#pragma unroll
        for (int q = 0; q < kChainQ; ++q) {
            const std::uint64_t k = std::uint64_t(lane) + 32u * q;
            nxt[q]                = k < n ? p[k] : 1.0;
        }
        for (std::uint64_t base = 0; base < n; base += kChainT) {
#pragma unroll
            for (int q = 0; q < kChainQ; ++q) tile[lane + 32 * q] = nxt[q];
            const std::uint64_t nb = base + kChainT;
#pragma unroll
            for (int q = 0; q < kChainQ; ++q) { // prefetch the next tile while the chain runs
                const std::uint64_t k = nb + std::uint64_t(lane) + 32u * q;
                nxt[q]                = k < n ? p[k] : 1.0;
            }
            __syncwarp();
            if (lane == 0) {
                const double2* t2 = reinterpret_cast<const double2*>(tile);
                double2*       o2 = reinterpret_cast<double2*>(tile);
                constexpr int  kB = 8; // double2 per batch (16 points); batches A, B alternate
                double2        A[kB], B[kB];
#pragma unroll
                for (int i = 0; i < kB; ++i) A[i] = t2[i];
#pragma unroll 1
                for (int bb = 0; bb < kChainT / 2; bb += 2 * kB) {
#pragma unroll
                    for (int i = 0; i < kB; ++i) B[i] = t2[bb + kB + i];
#pragma unroll
                    for (int i = 0; i < kB; ++i) {
                        double2 o;
                        cur = fmul(cur, A[i].x), o.x = cur;
                        cur = fmul(cur, A[i].y), o.y = cur;
                        o2[bb + i] = o;
                    }
                    const int na = bb + 2 * kB < kChainT / 2 ? bb + 2 * kB : 0;
#pragma unroll
                    for (int i = 0; i < kB; ++i) A[i] = t2[na + i];
#pragma unroll
                    for (int i = 0; i < kB; ++i) {
                        double2 o;
                        cur = fmul(cur, B[i].x), o.x = cur;
                        cur = fmul(cur, B[i].y), o.y = cur;
                        o2[bb + kB + i] = o;
                    }
                }
            }
            __syncwarp();
#pragma unroll
            for (int q = 0; q < kChainQ; ++q) {
                const std::uint64_t k = base + std::uint64_t(lane) + 32u * q;
                const double        y = fadd(a, fmul(wd, fsub(1.0, tile[lane + 32 * q])));
                if (k < n) p[k] = y >= b ? bmax : y;
            }
            __syncwarp();
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
    sincos(th, &s, &c);
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

// Two streams: the angle side (MT -> pow -> serial chain) is latency-bound
// and occupies few SMs, so the radius side (MT -> radial attributes) runs
// beside it on a second stream; the angular kernel joins both.
void launch_sampler(const SamplerArgs& S, cudaStream_t st, std::uint64_t* launches) {
    if (S.total == 0 || S.njobs == 0) return;
    const int      mt_blocks = S.njobs; // one CTA per stream
    const unsigned pblocks   = unsigned((S.total + 255) / 256);
    cudaStream_t   side      = S.side ? S.side : st;
    if (S.side) {
        cudaEventRecord(S.ev_fork, st);
        cudaStreamWaitEvent(side, S.ev_fork, 0);
    }
    // the radius attributes are needed only by the sort phase: they run beside the (few-SM)
    // chains, after pow, instead of competing with pow for the FP64 pipes
    mt_uniforms_kernel<<<mt_blocks, 32 * kMtWarps, 0, side>>>(S.jobs, S.njobs, S.beta, S.hw, 2);
    S.mark("mt_radii", side);
    mt_uniforms_kernel<<<mt_blocks, 32 * kMtWarps, 0, st>>>(S.jobs, S.njobs, S.beta, S.hw, 1);
    S.mark("mt_angles", st);
    static const int sched = std::getenv("RHG_SCHED") ? std::atoi(std::getenv("RHG_SCHED")) : 0;
    if (sched == 1) {
        point_radial_kernel<<<pblocks, 256, 0, side>>>(S.jobs, S.njobs, S.ann, S.alpha, S.total, S.hw, S.rec2, S.r_out);
        S.mark("radial", side);
    }
    point_pow_kernel<<<pblocks, 256, 0, st>>>(S.jobs, S.njobs, S.total, S.beta);
    S.mark("pow", st);
    if (sched == 2) {
        point_radial_kernel<<<pblocks, 256, 0, st>>>(S.jobs, S.njobs, S.ann, S.alpha, S.total, S.hw, S.rec2, S.r_out);
        S.mark("radial", st);
    }
    if (S.side) {
        cudaEventRecord(S.ev_fork, st);
        cudaStreamWaitEvent(side, S.ev_fork, 0);
    }
    if (sched == 0) {
        point_radial_kernel<<<pblocks, 256, 0, side>>>(S.jobs, S.njobs, S.ann, S.alpha, S.total, S.hw, S.rec2, S.r_out);
        S.mark("radial", side);
    }
    // chains: wave 1 on st; wave 2 (the outermost annulus, the longest chains) on S.late,
    // signalling S.ev_late, so the inner annuli's edge work overlaps its tail
    const bool split = S.wave2_jobs && S.late;
    const int  nb1   = split ? S.chain_bins1 : S.chain_bins_total;
    if (split && S.chain_bins_total > nb1) {
        cudaEventRecord(S.ev_pow, st);
        cudaStreamWaitEvent(S.late, S.ev_pow, 0);
        sorted_chain_kernel<<<S.chain_bins_total - nb1, 32, 0, S.late>>>(S.jobs, S.chain_bins + nb1, S.job_order,
                                                                         S.beta);
        cudaEventRecord(S.ev_late, S.late);
        S.mark("chain_wave2(late)", S.late);
        ++*launches;
    }
    if (nb1) sorted_chain_kernel<<<nb1, 32, 0, st>>>(S.jobs, S.chain_bins, S.job_order, S.beta);
    S.mark("chain_wave1", st);
    if (S.side) {
        cudaEventRecord(S.ev_join, side);
        cudaStreamWaitEvent(st, S.ev_join, 0);
    }
    // generate mode: streaming points get their frames in the sort phase (edges.cu angular_scatter_kernel)
    const std::uint64_t first = S.angular_from;
    if (S.total > first)
        point_angular_kernel<<<unsigned((S.total - first + 255) / 256), 256, 0, st>>>(
            S.jobs, S.njobs, first, S.total, S.beta, S.hw, S.rec0, S.rec1, S.beta_unlifted_out);
    *launches += 6;
}

void launch_mt_uniforms(const SamplerArgs& S, cudaStream_t st, std::uint64_t* launches) {
    if (S.total == 0 || S.njobs == 0) return;
    mt_uniforms_kernel<<<2 * S.njobs, 32 * kMtWarps, 0, st>>>(S.jobs, S.njobs, S.beta, S.hw, 0);
    *launches += 1;
}

void launch_frames_from_points(const SamplerArgs& S, cudaStream_t st, std::uint64_t* launches) {
    if (S.total == 0 || S.njobs == 0) return;
    const unsigned pblocks = unsigned((S.total + 255) / 256);
    frames_from_points_kernel<<<pblocks, 256, 0, st>>>(S.jobs, S.njobs, S.total, S.beta, S.hw, S.rec0);
    *launches += 1;
}

} // namespace rhgb
