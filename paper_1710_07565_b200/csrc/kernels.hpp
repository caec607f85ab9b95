// Host-visible launch interfaces of the device kernels (sampler.cu, edges.cu).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "device.cuh"

namespace rhgb {

// Optional phase timeline (RHG_TIMELINE=1): launch code calls mark(...) at phase
// boundaries; the context records an event on the given stream per mark.
struct Timeline {
    void (*fn)(void* self, const char* name, cudaStream_t st) = nullptr;
    void* self = nullptr;
    void  operator()(const char* name, cudaStream_t st) const {
        if (fn) fn(self, name, st);
    }
};

struct SamplerArgs {
    const StreamJob*  jobs = nullptr;
    int               njobs = 0;
    const std::uint32_t* job_order = nullptr; // jobs grouped by chain bin (chain kernel schedule)
    const std::uint32_t* chain_bins = nullptr; // bin b = job_order[chain_bins[b], chain_bins[b + 1])
    int                  chain_bins1 = 0, chain_bins_total = 0; // wave-1 bins come first
    const AnnulusDev* ann   = nullptr;
    const std::uint64_t* pseg = nullptr; // [npseg + 1] point segments: first point << 8 | annulus, total << 8
    int               npseg = 0;
    std::uint64_t     seed  = 0; // root seed: stream seeds are derive_seed(seed, {3|4, annulus, chunk})
    double            alpha = 1.0;
    std::uint64_t     total = 0; // points (streaming extended arrays + global points)
    double*           beta  = nullptr;
    double*           hw    = nullptr;
    double2*          rec0  = nullptr; // (lambda, theta)
    double2*          rec1  = nullptr; // (cos theta, sin theta)
    double2*          rec2  = nullptr; // (coth r, 1/sinh r)
    double*           r_out = nullptr;             // optional: radius
    double*           beta_unlifted_out = nullptr; // optional: raw beta
    std::uint64_t     angular_from = 0; // point_angular_kernel runs on [angular_from, total) (generate mode: n_ext)
    cudaStream_t      side = nullptr;                // optional second stream (fork/join with events)
    cudaEvent_t       ev_fork = nullptr, ev_join = nullptr;
    Timeline          mark;
    int               wave2_jobs = 0;     // the last wave2_jobs entries of job_order chain on `late`
    cudaStream_t      late = nullptr;
    cudaEvent_t       ev_pow = nullptr, ev_late = nullptr; // pow done (main) / wave-2 chains done (late)
    // the global annuli's points on their own stream (generate mode): their bins come first
    // (chain_bins_g), their jobs last in `jobs` ([glob_job0, njobs)); ev_glob marks them sampled
    cudaStream_t      glob = nullptr;
    cudaEvent_t       ev_glob = nullptr;
    int               chain_bins_g = 0, glob_job0 = 0;
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
    // lambda-sorted copies (per annulus: owned block, halo block)
    double*           s_beta = nullptr;
    double*           s_hw   = nullptr;
    double*           s_lam   = nullptr; // lambda (engine-frame centre)
    double*           s_theta = nullptr; // raw theta (same-annulus dedup)
    double2*          s_rec1 = nullptr;
    double2*          s_rec2 = nullptr;
    unsigned long long* s_id = nullptr;     // [n_ext + 2] vertex ids
    const std::uint32_t* gperm = nullptr;  // global requests in (annulus, theta) order (null: id order)
    std::uint32_t*    cseg = nullptr;      // [kMaxCls + 1] sorted-position starts of the non-empty segments
    int*              n_cls = nullptr;     // number of non-empty (source, class) segments (device-written)
    std::uint32_t*    bk_off = nullptr;    // [kMaxCls + 1] segment c's angle-bucket table at gbk + bk_off[c]
    std::uint32_t*    bk_shift = nullptr;  // [kMaxCls] 32 - log2(buckets of segment c)
    std::uint32_t*    gbk = nullptr;       // bucket starts (sorted positions), <= 2 n_req + 65 kMaxCls entries
    // dense engine: unified requests u (global points, then the streaming requests of annuli with
    // dense targets), sorted by (source, radial class, angle) into positions s
    std::uint64_t     n_req = 0;
    const std::uint64_t* req_off = nullptr;      // [count] first unified index of streaming annulus a
    const unsigned long long* dense_mask = nullptr; // [count] bit j: (a, j) runs on the dense engine
    const uint4*      row_tasks = nullptr;  // dense rows: (j | source << 16, s0, s1, first block) by target
    std::uint32_t     row_t0 = 0, row_t1 = 0, row_b0 = 0; // this wave's tasks / first block
    double2*          g_rec = nullptr;     // [2 n_req] sorted requests: (cos, sin), (coth, coshR/sinh)
    std::uint32_t*    g_id = nullptr;      // [n_req] vertex id
    double*           g_inv = nullptr;     // [n_req] 1 / sinh r
    std::uint32_t*    g_u = nullptr;       // [n_req] unified request index
    double4*          g_aux = nullptr;     // [n_req] (lambda or theta, beta, hw, theta)
    uint4*            deferred = nullptr;  // [defer_cap] (sorted request, k0, k1, dedup) ranges of deferred_kernel
    unsigned long long* defer_ctr = nullptr; // [0] ranges reserved, [1] ranges dropped (must stay 0)
    std::uint64_t     defer_cap = 0;
    std::uint32_t*    seg_first = nullptr; // [(count - first_streaming + 1) << 10] first sorted position per segment id
    std::uint32_t*    g_rows = nullptr;    // [streaming annuli][n_req][8] window pieces (s0, s1) as owned indices
    unsigned long long* hmax_bits = nullptr; // [kMaxCls * count] max half-width per (radial class, target) (bits)
    const std::uint64_t* gt_prefix = nullptr; // [count + 1] dense-engine warps (128-node owned tiles) before annulus j
    std::uint64_t     glob_tile_warps = 0;
    const std::uint32_t* ann_blk = nullptr; // [count + 1] prefix of 256-point blocks per streaming annulus
    unsigned long long* dmax_bits = nullptr; // per annulus, max half-width (bits)
    int               rank_gallop = 0;      // generate mode, small windows: rank by galloping (no beta cells)
    double            cosh_R = 1.0;
    double            chunk0_upper = 0.0; // chunk_upper_bound(0, P)
    int               lift_part = 0;      // shard owns engine P-1 (halo = lifted chunk 0)
    int               gen = 0;            // generate mode (see launch_cell_index)
    Timeline          mark;
    // wave parameters (set by the launch functions): sort-phase block offset, target annuli
    // [j0, j1) (cell tails, rows, node tiles), first slab of the wave
    std::uint32_t     blk0 = 0;
    int               j0 = 0, j1 = 0;
    std::uint64_t     slab0 = 0;
    // slab join (sparse pairs): slabs of 1024 owned nodes of every target annulus with sparse sources
    const unsigned long long* slab_tab = nullptr; // [n_slabs] (j << 32) | slab index in j, angle-interleaved order
    std::uint64_t     n_slabs = 0;
    const unsigned long long* src_mask = nullptr; // [count] bit a: (a, j) is sparse (slab join)
    const double*     hbound = nullptr;           // [count * count] bound on the half-width of a's requests in j
    const std::uint64_t* tail_prefix = nullptr;   // [count + 1] tail requests (owned tail + halo block) before annulus a
    const double*     tail_lam = nullptr;         // [count] owned requests with lambda >= tail_lam[a] are tail requests
    std::uint64_t     n_tail = 0;
    cudaEvent_t       ev_pairs0 = nullptr, ev_pairs1 = nullptr; // optional: time the streaming pair kernel
    std::uint64_t     gg_tile_begin = 0, gg_tile_end = 0; // this shard's global-unit tiles
    Counters*         ctr = nullptr; // [0] streaming kernel, [1] dense engine, [2] global unit
    SlotCounter*      slots = nullptr; // [3 * kSlots] partial counters (folded into ctr at the end)
    int               ablate = 0;       // RHG_ABLATE bit flags: skip kernel phases (timing experiments; results invalid)
    unsigned long long* ann_ctr = nullptr;    // [kAnnSlots][2 * kMaxAnnuli]: per-annulus edges, then comps
    const std::uint64_t* gseg = nullptr;      // [first_streaming + 1] global-id base of each inner annulus
    double*             lam_tmp = nullptr;    // [n_ext] engine-frame lambda in sampler order (sort phase)
    ulonglong2*         edge_out = nullptr;   // optional materialised edges (MODE 2): canonical (u, v)
    unsigned long long  edge_cap = 0;
    unsigned long long* edge_count = nullptr; // device counter of emitted edges (may exceed edge_cap)
    unsigned long long* dbg = nullptr; // optional path statistics (RHG_DEBUG_STATS=1), kDbgSlots entries
    unsigned long long* audit = nullptr; // predicate audit (rhg_audit_predicate): kAuditSlots entries
    unsigned int*     degrees = nullptr;
};

// gen: the beta array holds the sampler's unlifted beta and no frames yet (rank from beta + hw, the
// frames are computed while scattering); otherwise frames_from_points already built beta/rec0/rec1.
void launch_cell_index(const EdgeArgs& a, std::uint32_t blk_begin, std::uint32_t blk_end, int j_begin, int j_end,
                       bool gen, cudaStream_t st, std::uint64_t* launches);
struct EdgeWave {
    int           j0 = 0, j1 = 0;                 // target annuli of the dense rows / node tiles
    std::uint64_t tile_warps = 0;                 // gt_prefix[j1] - gt_prefix[j0]
    std::uint64_t slab_begin = 0, slab_end = 0;   // slab-join CTAs (slab_tab range)
    bool          exact_slabs = false;            // the wave's slabs are mostly exact-predicate pairs
    bool          dense_occ4 = false;             // node tiles at 4 CTAs/SM (wide dense windows)
    bool          first_wave = false;             // wave 1's dense targets (node-tile launch bounds)
    std::uint32_t row_t0 = 0, row_t1 = 0;         // dense-row tasks of the targets [j0, j1)
    std::uint32_t row_b0 = 0, row_nb = 0;         // their first block and block count
    bool          global_unit = false, tail = false, finish = false;
    cudaEvent_t   ev0 = nullptr, ev1 = nullptr;   // optional: time the wave's sparse engine
};
void launch_edges(const EdgeArgs& a, const EdgeWave& w, cudaStream_t st, std::uint64_t* launches);
// naive.cu: brute-force pairs with hyperbolic distance < R (oracle.hpp:41-54), unsorted.
void launch_naive_pairs(const double* r, const double* theta, double* sh, std::uint64_t n, double R, ulonglong2* out,
                        unsigned long long cap, unsigned long long* count, cudaStream_t st);
// Sorts m canonical edges in place into (u, v) order (keys ka/kb: m each; ids < 2^32).
// With tmp == nullptr or *tmp_bytes too small, only reports the scratch bytes needed.
void launch_sort_edges(ulonglong2* edges, std::uint64_t m, unsigned long long* ka, unsigned long long* kb, void* tmp,
                       std::size_t* tmp_bytes, int end_bit, cudaStream_t st);
// Sorts the global points by (annulus, theta) into a.gperm (scratch layout
// internal); with scratch == nullptr only reports the bytes needed in *need.
void launch_sort_globals(EdgeArgs& a, void* scratch, std::size_t scratch_bytes, std::size_t* need, cudaStream_t st,
                         std::uint64_t* launches);

constexpr int kGGTile = 128;
constexpr int kMaxAnnuli = 64;  // annulus masks are 64-bit
constexpr int kAnnSlots  = 64;  // spread per-annulus counter slots (folded by reduce_counters_kernel)
constexpr int kTileNodes = 128; // owned nodes per dense-engine node tile (edges.cu glob_tiles_kernel; 64: 0.64 vs 0.58 ms)
constexpr int kSlabNodes = 512; // owned nodes per slab of the slab join (edges.cu)
constexpr int kMaxCls = 1024; // (source, radial class) segments of the dense-engine requests
// audit layout (slab_kernel MODE 3): [0] pairs the FP32 pre-filter decided, [1] pairs it left to
// the exact recheck, [2] pairs of exact-only groups, [3] pre-filter decisions that differ from the
// reference predicate, [4] max |D32 - D64| / tau over decided pairs (float bits), [5] pairs with
// |D64| below 1e-15 (the rounding-noise band of the reference predicate)
constexpr int kAuditSlots = 8;
// dbg layout (RHG_DEBUG_STATS=1): [0] stream (warp, target) steps, [1] staged unions, [2] per-lane
// searches, [3] long rows, [4] flattened pairs, [5] serial pairs, [8] dense candidates loaded,
// [9] dense (request, tile) pieces evaluated, [10] dense warps
constexpr int kDbgSlots = 32;

} // namespace rhgb
