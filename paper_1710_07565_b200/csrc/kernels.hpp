// Host-visible launch interfaces of the device kernels (sampler.cu, edges.cu).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "device.cuh"

namespace rhgb {

struct SamplerArgs {
    const StreamJob*  jobs = nullptr;
    int               njobs = 0;
    const AnnulusDev* ann   = nullptr;
    double            alpha = 1.0;
    std::uint64_t     total = 0; // points (streaming extended arrays + global points)
    double*           beta  = nullptr;
    double*           hw    = nullptr;
    double2*          rec0  = nullptr; // (lambda, theta)
    double2*          rec1  = nullptr; // (cos theta, sin theta)
    double2*          rec2  = nullptr; // (coth r, 1/sinh r)
    double*           r_out = nullptr;             // optional: radius
    double*           beta_unlifted_out = nullptr; // optional: raw beta
    cudaStream_t      side = nullptr;                // optional second stream (fork/join with events)
    cudaEvent_t       ev_fork = nullptr, ev_join = nullptr;
};

void launch_sampler(const SamplerArgs& a, cudaStream_t st, std::uint64_t* launches);
void launch_frames_from_points(const SamplerArgs& a, cudaStream_t st, std::uint64_t* launches);
void launch_mt_uniforms(const SamplerArgs& a, cudaStream_t st, std::uint64_t* launches);

struct EdgeArgs {
    const AnnulusDev* ann = nullptr;
    AnnulusDev*       ann_rw = nullptr; // same table (lambda_cells_kernel writes `wrap`)
    int               count = 0, first_streaming = 0;
    std::uint64_t     n_ext = 0;   // streaming extended points; global points follow
    std::uint64_t     n_glob = 0;  // global points (ids 0..n_glob-1)
    const double*     beta = nullptr;
    const double*     hw   = nullptr;
    const double2*    rec0 = nullptr;
    const double2*    rec1 = nullptr;
    const double2*    rec2 = nullptr;
    std::uint64_t*    cellstart = nullptr;  // beta cells (sampler order)
    std::uint64_t*    lcellstart = nullptr; // lambda cells (sorted owned blocks)
    std::uint64_t*    perm = nullptr;       // sampler index -> sorted index
    // lambda-sorted copies (per annulus: owned block, halo block)
    double*           s_beta = nullptr;
    double*           s_hw   = nullptr;
    double2*          s_rec0 = nullptr;
    double2*          s_rec1 = nullptr;
    double2*          s_rec2 = nullptr;
    unsigned long long* s_id = nullptr;     // [n_ext + 2] vertex ids
    const std::uint32_t* gperm = nullptr;  // global requests in (annulus, theta) order (null: id order)
    const std::uint32_t* ann_blk = nullptr; // [count + 1] prefix of 256-point blocks per streaming annulus
    unsigned long long* dmax_bits = nullptr; // per annulus, max half-width (bits)
    double            cosh_R = 1.0;
    double            chunk0_upper = 0.0; // chunk_upper_bound(0, P)
    int               lift_part = 0;      // shard owns engine P-1 (halo = lifted chunk 0)
    const PairJob*    stream_jobs = nullptr;
    int               n_stream_jobs = 0;
    std::uint64_t     stream_warps = 0;      // work items (batches of 32 requests x target annulus)
    const std::uint64_t* blk_prefix = nullptr; // [nblk + 1] items before angular block b
    const std::uint32_t* blk_job_off = nullptr; // [nblk * n_stream_jobs] item offset of job k inside block b
    int               nblk = 1;
    cudaEvent_t       ev_pairs0 = nullptr, ev_pairs1 = nullptr; // optional: time the streaming pair kernel
    const PairJob*    glob_jobs = nullptr;
    int               n_glob_jobs = 0;
    std::uint64_t     glob_warps = 0;
    std::uint64_t     gg_tile_begin = 0, gg_tile_end = 0; // this shard's global-unit tiles
    TileTask*         tasks = nullptr;
    std::uint64_t     task_cap = 0;
    unsigned long long* task_ctr = nullptr;
    Counters*         ctr = nullptr; // [0] streaming, [1] global requests, [2] global unit
    unsigned long long* dbg = nullptr; // optional path statistics (RHG_DEBUG_STATS=1), kDbgSlots entries
    unsigned int*     degrees = nullptr;
};

void launch_cell_index(const EdgeArgs& a, std::uint64_t nblocks, cudaStream_t st, std::uint64_t* launches);
void launch_edges(const EdgeArgs& a, cudaStream_t st, std::uint64_t* launches);
// Sorts the global points by (annulus, theta) into a.gperm (scratch layout
// internal); with scratch == nullptr only reports the bytes needed in *need.
void launch_sort_globals(EdgeArgs& a, const std::uint64_t* seg_off_dev, int nseg, void* scratch,
                         std::size_t scratch_bytes, std::size_t* need, cudaStream_t st, std::uint64_t* launches);

constexpr int kGGTile = 128;
// dbg layout: [0..5] groups per lgR, [6..11] sum U per lgR, [12..17] slots per lgR, [18] serial warps,
// [19] serial slots (32*maxlen), [20] serial candidates, [21] tasks, [22] warps, [23] candidates total
constexpr int kDbgSlots = 32;

} // namespace rhgb
