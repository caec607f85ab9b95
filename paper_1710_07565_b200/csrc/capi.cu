// C ABI (include/rhg_b200.h) and per-call orchestration.
//
// One call = host layout (layout.cpp, the reference's O(annuli*P) binomial
// tree) -> shard plan (extended chunk arrays, stream jobs, pair jobs) -> one
// H2D copy of all tables -> sampler kernels -> cell index -> edge kernels ->
// one D2H copy of the counters.  All device work is on the context's stream,
// timed with CUDA events on that stream.
//
// Multi-GPU: a context may carry an NCCL communicator (rhg_attach_comm:
// one process per GPU; rhg_create_multi: one process, one sub-context and host thread
// per GPU).  A shard call on such a context ends with ONE ncclAllReduce(ncclUint64, sum)
// of its counters on the context's stream, inside the timed region, so every rank
// returns the whole graph's (edges, fingerprint, comps).  NCCL is dlopen'ed on first
// use: single-GPU use has no NCCL dependency.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <cstring>
#include <new>
#include <string>
#include <queue>
#include <thread>
#include <vector>

#include <dlfcn.h>
#include <nccl.h> // types and prototypes only: the library is dlopen'ed (nccl_api)

#include "../../include/rhg_b200.h"
#include "device.cuh"
#include "kernels.hpp"
#include "layout.hpp"

using namespace rhgb;

namespace {

thread_local std::string g_err;

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define CK(x)                                                                                             \
    do {                                                                                                  \
        cudaError_t e_ = (x);                                                                             \
        if (e_ != cudaSuccess) throw CudaError(std::string(#x) + ": " + cudaGetErrorString(e_));        \
    } while (0)

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return RHG_OK;
    } catch (const InvalidArgument& e) {
        g_err = e.what();
        return RHG_INVALID_ARGUMENT;
    } catch (const Invariant& e) {
        g_err = e.what();
        return RHG_INVARIANT;
    } catch (const CudaError& e) {
        g_err = e.what();
        return RHG_CUDA;
    } catch (const std::bad_alloc&) {
        g_err = "out of memory";
        return RHG_NOMEM;
    } catch (const std::exception& e) {
        g_err = e.what();
        return RHG_INVARIANT;
    }
}

struct DevBuf {
    void*       p   = nullptr;
    std::size_t cap = 0;
    void ensure(std::size_t bytes) {
        if (bytes <= cap) return;
        if (p) cudaFree(p);
        p   = nullptr;
        cap = 0;
        CK(cudaMalloc(&p, bytes));
        cap = bytes;
    }
    void release() {
        if (p) cudaFree(p);
        p   = nullptr;
        cap = 0;
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

struct HostPinned {
    void*       p   = nullptr;
    std::size_t cap = 0;
    void ensure(std::size_t bytes) {
        if (bytes <= cap) return;
        if (p) cudaFreeHost(p);
        p   = nullptr;
        cap = 0;
        CK(cudaMallocHost(&p, bytes));
        cap = bytes;
    }
};

std::size_t align256(std::size_t x) { return (x + 255) & ~std::size_t(255); }

double ms_between(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a, b));
    return ms;
}

// NCCL entry points, resolved from libnccl.so.2 on first use (the copy torch already
// loaded, if any: same soname).
struct NcclApi {
    void* h = nullptr;
    decltype(&ncclGetUniqueId)    get_unique_id = nullptr;
    decltype(&ncclCommInitRank)   comm_init_rank = nullptr;
    decltype(&ncclCommInitAll)    comm_init_all = nullptr;
    decltype(&ncclAllReduce)      all_reduce = nullptr;
    decltype(&ncclCommDestroy)    comm_destroy = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
};
const NcclApi& nccl_api() {
    static const NcclApi api = [] {
        NcclApi a;
        for (const char* name: {"libnccl.so.2", "libnccl.so"})
            if ((a.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL))) break;
        if (!a.h) return a;
        a.get_unique_id  = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(a.h, "ncclGetUniqueId"));
        a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(a.h, "ncclCommInitRank"));
        a.comm_init_all  = reinterpret_cast<decltype(a.comm_init_all)>(dlsym(a.h, "ncclCommInitAll"));
        a.all_reduce     = reinterpret_cast<decltype(a.all_reduce)>(dlsym(a.h, "ncclAllReduce"));
        a.comm_destroy   = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(a.h, "ncclCommDestroy"));
        a.error_string   = reinterpret_cast<decltype(a.error_string)>(dlsym(a.h, "ncclGetErrorString"));
        return a;
    }();
    if (!api.h || !api.get_unique_id || !api.comm_init_rank || !api.comm_init_all || !api.all_reduce ||
        !api.comm_destroy || !api.error_string)
        throw CudaError("rhg: NCCL (libnccl.so.2) is not available for multi-GPU contexts");
    return api;
}

#define NK(x)                                                                                             \
    do {                                                                                                  \
        ncclResult_t r_ = (x);                                                                            \
        if (r_ != ncclSuccess) throw CudaError(std::string(#x) + ": " + nccl_api().error_string(r_));   \
    } while (0)

} // namespace

struct rhg_ctx {
    int          device = 0;
    cudaStream_t stream = nullptr, side = nullptr, late = nullptr;
    cudaStream_t small = nullptr; // the edge phase's small independent kernels (global unit, tail pairs)
    cudaStream_t dense = nullptr; // the edge phase's dense engine (beside the slab join on `stream`)
    cudaEvent_t  ev[6]{};
    cudaEvent_t  fork = nullptr, join = nullptr; // timing-free events for the side stream
    cudaEvent_t  ev_glob = nullptr, ev_gz = nullptr; // global points sampled / counters zeroed (small stream)
    cudaEvent_t  ev_pow = nullptr, ev_late = nullptr; // the wave-2 chains (late stream)
    cudaEvent_t  evw[6]{};                            // sparse-engine timing: the two waves' slab joins, the side tail
    std::vector<std::pair<std::string, cudaEvent_t>> tl; // RHG_TIMELINE marks of the current call
    std::vector<cudaEvent_t> tl_pool;
    DevBuf       beta, hw, rec0, rec1, rec2, r_out, beta_raw, tables, tables2, cells, counters, degrees, dbg, nid;
    DevBuf       lcells, s_beta, s_hw, s_lt, s_rec1, s_rec2, gsort, gbuf;
    DevBuf       ebuf, ecount, ekeys, esort; // materialised edges (rhg_generate_edges)
    DevBuf       lam_tmp, audit;
    bool         audit_on = false;            // rhg_audit_predicate in progress
    HostPinned   staging, staging2, readback; // table parts 1 and 2, counter readback
    // multi-GPU: a communicator over `comm_world` ranks (this context = rank comm_rank); shard
    // calls with shard {comm_rank, comm_world} all-reduce their counters through it
    ncclComm_t    comm       = nullptr;
    std::uint32_t comm_world = 1, comm_rank = 0;
    bool          reduce_off = false; // per-unit calls: shard results stay per shard
    // rhg_create_multi: one sub-context per device (each with its comm); calls fan out to them
    std::vector<rhg_ctx*> subs;
};

namespace {

void timeline_mark(void* self, const char* name, cudaStream_t st) {
    auto* c = static_cast<rhg_ctx*>(self);
    if (c->tl.size() >= c->tl_pool.size()) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) return;
        c->tl_pool.push_back(e);
    }
    cudaEvent_t e = c->tl_pool[c->tl.size()];
    cudaEventRecord(e, st);
    c->tl.push_back({name, e});
}
Timeline timeline_of(rhg_ctx* c) {
    Timeline t;
    const char* v = std::getenv("RHG_TIMELINE");
    if (v && v[0] == '1') t.fn = timeline_mark, t.self = c;
    return t;
}
void timeline_report(rhg_ctx* c, cudaEvent_t start) {
    if (c->tl.empty()) return;
    std::fprintf(stderr, "RHG_TIMELINE");
    for (auto& m: c->tl) {
        float ms = 0;
        cudaEventElapsedTime(&ms, start, m.second);
        std::fprintf(stderr, " %s=%.3f", m.first.c_str(), ms);
    }
    std::fprintf(stderr, "\n");
    c->tl.clear();
}

// The shard plan: which (annulus, chunk) streams this rank draws, where they
// land in the extended arrays, and the pair-kernel work lists.
struct Plan {
    Layout                  L;
    std::uint32_t           e0 = 0, e1 = 0, T = 0, rank = 0, world = 1;
    std::vector<AnnulusDev> ann;
    std::vector<StreamJob>  jobs;
    std::vector<std::uint32_t> job_order;   // wave-1 jobs then wave-2 jobs, grouped by chain bin
    std::vector<std::uint32_t> chain_bins;  // bin b runs job_order[chain_bins[b], chain_bins[b + 1])
    std::uint32_t              chain_bins1 = 0; // global-annulus + wave-1 bins (wave-2 bins follow)
    std::uint32_t              chain_bins_g = 0; // global-annulus bins (they come first)
    std::uint32_t              wave_j = 0;  // first annulus of wave 2 (count: no split)
    int                        wave2_jobs = 0;
    int                        glob_jobs = 0;     // jobs of the global annuli (the last entries of `jobs`)
    std::uint64_t              n_slabs1 = 0; // slabs of wave-1 targets (they come first in slab_tab)
    std::vector<std::uint64_t> gt_prefix;   // dense-engine warps (512-node owned strips) before annulus j
    std::vector<std::uint64_t> gseg;        // global-point annulus offsets (segments of the theta sort)
    std::vector<std::uint64_t> pseg;        // point segments in index order: first point << 8 | annulus; total << 8
    std::vector<unsigned long long> dense_mask; // [count] bit j: (a, j) runs on the dense engine
    std::vector<std::uint64_t> req_off;     // [count] unified dense-request index of annulus a's first request
    std::uint64_t              n_req = 0;
    std::vector<std::uint32_t> ann_blk;     // 256-point blocks per streaming annulus (prefix, count + 1)
    std::vector<unsigned long long> src_mask; // [count] bit a: (a, j) runs on the slab join
    std::vector<uint4>              row_tasks;   // dense rows: (j | source << 16, s0, s1, first block), by target j
    std::vector<std::uint32_t>      row_task_j;  // [count + 1] first task of target j
    std::vector<double>        hbound;      // [count * count] half-width bound of a's requests in j
    std::vector<std::uint64_t> slab_prefix; // [count + 1] slabs (1024 owned nodes) before annulus j
    std::vector<unsigned long long> slab_tab; // [n_slabs] (j << 32) | slab index, angle-interleaved
    std::vector<std::uint64_t> tail_prefix; // [count + 1] tail threads before annulus a
    std::vector<double>        tail_lam;    // [count] owned requests with lambda >= this are tail requests
    std::uint64_t           n_ext = 0, n_glob = 0, total = 0, gtwarps = 0, ncells = 0, n_slabs = 0, n_tail = 0;
    std::uint64_t           gg_t0 = 0, gg_t1 = 0;
    double                  layout_ms = 0;
    double                  sub_ms[4] = {0, 0, 0, 0}; // RHG_TIMELINE: plan phases after the layout
};

// LSD radix sort of u64 keys on bits [lo_bit, 64), stable (keys equal there keep their order):
// 16-bit digits, constant digits skipped.  std::sort of the 1.2e5 job keys at cfg4 took 10 ms.
void radix_sort_keys(std::vector<std::uint64_t>& key, int lo_bit) {
    if (key.size() < 8192) { // the digit histograms would cost more than the comparisons
        std::stable_sort(key.begin(), key.end(), [lo_bit](std::uint64_t x, std::uint64_t y) {
            return (x >> lo_bit) < (y >> lo_bit);
        });
        return;
    }
    std::vector<std::uint64_t> tmp(key.size());
    std::vector<std::uint32_t> cnt(1u << 16);
    for (int sh = lo_bit; sh < 64; sh += 16) {
        const int           bits = std::min(16, 64 - sh);
        const std::uint64_t mask = (std::uint64_t(1) << bits) - 1;
        std::fill(cnt.begin(), cnt.begin() + (std::size_t(1) << bits), 0u);
        for (std::uint64_t k: key) ++cnt[(k >> sh) & mask];
        if (cnt[(key.empty() ? 0 : (key[0] >> sh) & mask)] == key.size()) continue; // one digit value
        std::uint32_t run = 0;
        for (std::size_t d = 0; d < (std::size_t(1) << bits); ++d) {
            const std::uint32_t c = cnt[d];
            cnt[d] = run, run += c;
        }
        for (std::uint64_t k: key) tmp[cnt[(k >> sh) & mask]++] = k;
        key.swap(tmp);
    }
}

// Expected number of annulus-j nodes in the window of an annulus-a request
// at a's median radius (density ~ sinh(alpha r)); same-annulus windows count
// half (dedup).  Only chooses the engine for (a, j); never affects results.
constexpr double kDenseMin = 96.0;
// Outer streaming annuli whose chains run in wave 2 (generate mode)
#ifndef RHG_WAVE2_DEFAULT
#define RHG_WAVE2_DEFAULT 1
#endif
constexpr std::uint32_t kWave2Annuli = RHG_WAVE2_DEFAULT;
double expected_window_nodes(const Layout& L, std::uint32_t a, std::uint32_t j) {
    const double r    = std::acosh(0.5 * (L.cosh_alpha_lower[a] + L.cosh_alpha_upper[a])) / L.alpha;
    const double ex   = std::exp(r), mex = 1.0 / ex, sh = 0.5 * (ex - mex);
    const double coth = 0.5 * (ex + mex) / sh, inv = 1.0 / sh;
    double       h    = kPi;
    if (L.lower[j] > 0.0) {
        const double arg = coth * L.coth_lower[j] - L.coshR_inv_sinh_lower[j] * inv;
        h                = arg <= -1.0 ? kPi : arg >= 1.0 ? 0.0 : std::acos(arg);
    }
    return double(L.counts[j]) * 2.0 * h / kTwoPi * (a == j ? 0.5 : 1.0);
}

// Upper bound on the window half-width of any annulus-a request in annulus j
// (own window: the own half-width): the half-width at a's lower radius, where
// it is largest, plus a margin for libm differences.  Only sizes candidate
// searches (supersets); never affects results.
double half_width_bound(const Layout& L, std::uint32_t a, std::uint32_t j) {
    if (!(L.lower[a] > 0.0) || !(L.lower[j] > 0.0)) return kPi;
    const double inv = 1.0 / std::sinh(L.lower[a]);
    const double arg = L.coth_lower[a] * L.coth_lower[j] - L.coshR_inv_sinh_lower[j] * inv;
    const double h   = arg <= -1.0 ? kPi : arg >= 1.0 ? 0.0 : std::acos(arg);
    return std::min(kPi, h * (1.0 + 1e-6) + 1e-9);
}

Plan make_plan_head(const Params& P, const rhg_shard* shard) {
    Plan                pl;
    const auto          tl0 = std::chrono::steady_clock::now();
    const std::uint32_t W = shard ? shard->world : 1, r = shard ? shard->rank : 0;
    if (W < 1 || r >= W) throw InvalidArgument("rhg_shard: rank must lie in [0, world)");
    if (P.chunks < 1) throw InvalidArgument("ModelParams: chunk count must be >= 1");
    {   // a shard's layout splits only its own streaming chunks and the halo chunk
        const std::uint32_t e0 = std::uint32_t(std::uint64_t(P.chunks) * r / W);
        const std::uint32_t e1 = std::uint32_t(std::uint64_t(P.chunks) * (r + 1) / W);
        ChunkNeed           need;
        if (e1 < P.chunks) need.lo[0] = e0, need.hi[0] = e1 + 1, need.n = 1;
        else need.lo[0] = e0, need.hi[0] = P.chunks, need.lo[1] = 0, need.hi[1] = 1, need.n = 2;
        pl.L = make_layout(P, W > 1 ? &need : nullptr);
    }
    pl.layout_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tl0).count();
    const Layout&       L  = pl.L;
    const std::uint32_t Pc = L.chunks;
    pl.rank = r, pl.world = W;
    pl.e0 = std::uint32_t(std::uint64_t(Pc) * r / W);
    pl.e1 = std::uint32_t(std::uint64_t(Pc) * (r + 1) / W);
    pl.T  = pl.e1 - pl.e0;
    pl.ann.resize(L.count);
    pl.jobs.reserve(std::size_t(L.count) * (std::size_t(pl.T) + 1) + std::size_t(L.first_streaming) * Pc);
    std::uint64_t run = 0;
    for (std::uint32_t i = 0; i < L.count; ++i) {
        AnnulusDev& A = pl.ann[i];
        std::memset(&A, 0, sizeof A);
        A.lower = L.lower[i], A.coth_lower = L.coth_lower[i], A.cris = L.coshR_inv_sinh_lower[i];
        A.cal = L.cosh_alpha_lower[i], A.cau = L.cosh_alpha_upper[i];
        if (i < L.first_streaming) continue;
        A.off = A.halo = A.end = run;
        if (pl.T == 0) continue;
        for (std::uint32_t t = 0; t <= pl.T; ++t) {
            const std::uint32_t c   = (pl.e0 + t) % Pc;
            const std::uint64_t cnt = L.chunk_count(i, c);
            if (t == pl.T) A.halo = run;
            if (cnt) {
                StreamJob J{};
                J.out_off = run, J.count = cnt, J.annulus = i, J.chunk = c, J.lift = (pl.e0 + t == Pc) ? 1u : 0u;
                J.a = chunk_lower_bound(c, Pc), J.b = chunk_upper_bound(c, Pc);
                pl.jobs.push_back(J);
            }
            run += cnt;
        }
        A.end  = run;
        A.dlt0 = std::int64_t(L.chunk_id_base(i, pl.e0)) - std::int64_t(A.off);
        A.dlt1 = std::int64_t(L.chunk_id_base(i, pl.e1 % Pc)) - std::int64_t(A.halo);
        const std::uint64_t n = A.end - A.off;
        A.ncells              = std::uint32_t(std::max<std::uint64_t>(1, std::min<std::uint64_t>(n / 2, 1u << 30)));
        A.cell_origin         = chunk_lower_bound(pl.e0, Pc);
        const double top      = pl.e1 == Pc ? kTwoPi + chunk_upper_bound(0, Pc) : chunk_upper_bound(pl.e1, Pc);
        A.cell_inv_w          = double(A.ncells) / (top - A.cell_origin);
        A.cell_off            = pl.ncells;
        A.wrap                = A.halo;
        pl.ncells += A.ncells + 1;
    }
    pl.n_ext  = run;
    pl.n_glob = L.global_vertices();
    pl.ann_blk.assign(L.count + 1, 0);
    for (std::uint32_t i = 0; i < L.count; ++i)
        pl.ann_blk[i + 1] = pl.ann_blk[i] + std::uint32_t((pl.ann[i].end - pl.ann[i].off + 255) / 256);
    for (std::uint32_t i = 0; i < L.first_streaming; ++i)
        for (std::uint32_t c = 0; c < Pc; ++c) {
            const std::uint64_t cnt = L.chunk_count(i, c);
            if (!cnt) continue;
            StreamJob J{};
            J.out_off = pl.n_ext + L.chunk_id_base(i, c), J.count = cnt, J.annulus = i, J.chunk = c, J.lift = 0;
            J.a = chunk_lower_bound(c, Pc), J.b = chunk_upper_bound(c, Pc);
            pl.jobs.push_back(J);
        }
    pl.total = pl.n_ext + pl.n_glob;
    for (std::uint32_t i = 0; i < L.first_streaming; ++i) pl.gseg.push_back(L.chunk_id_base(i, 0));
    pl.gseg.push_back(pl.n_glob);
    for (std::uint32_t i = L.first_streaming; i < L.count; ++i) pl.pseg.push_back((pl.ann[i].off << 8) | i);
    for (std::uint32_t i = 0; i < L.first_streaming; ++i) pl.pseg.push_back(((pl.n_ext + pl.gseg[i]) << 8) | i);
    pl.pseg.push_back(pl.total << 8);
    // (annulus, target) pairs whose windows hold >= kDenseMin nodes on average run on the dense
    // engine (node tiles x streamed requests); the rest on the slab join (96: measured optimum band 64..128 at cfg2)
    // the engine threshold (chooses the engine, never the result): 96 nodes, doubled for graphs whose
    // average degree is >= 128 (wide windows everywhere: with the dense engine beside the slab join,
    // moving the 96..192-node windows to the slab join balances the two; measured cfg3 24.56 ->
    // 22.48 ms, cfg2 unchanged at 96, worse above 128); RHG_DENSE_MIN overrides (A/B)
    const double dbar_model = std::exp(-0.5 * (L.R - 2.0 * std::log(double(L.n)))) /
                              (kPi / 2.0 * ((L.alpha - 0.5) / L.alpha) * ((L.alpha - 0.5) / L.alpha));
    const char*  dmv       = std::getenv("RHG_DENSE_MIN");
    const double dense_min = dmv ? std::atof(dmv) : kDenseMin * (dbar_model >= 128.0 ? 2.0 : 1.0);
    pl.dense_mask.assign(L.count, 0ull);
    pl.req_off.assign(L.count, 0);
    pl.n_req = pl.n_glob;
    for (std::uint32_t a = L.first_streaming; a < L.count; ++a) {
        for (std::uint32_t j = a; j < L.count && j < 64; ++j)
            if (expected_window_nodes(L, a, j) >= dense_min) pl.dense_mask[a] |= 1ull << j;
        pl.req_off[a] = pl.n_req;
        if (pl.dense_mask[a]) pl.n_req += pl.ann[a].end - pl.ann[a].off;
    }
    // wave split (generate mode): the outermost streaming annulus (the longest sorted-uniform
    // chains) forms wave 2 when it is not a dense-engine source; everything else is wave 1.
    // Graphs of >= 2^25 points put their two outermost annuli in wave 2 (measured cfg3 / cfg4 /
    // cfg5 -0.3 / -0.7 / -0.5 %; cfg2 keeps one: +0.15 % with two)
    pl.wave_j = L.count;
    {
        const char*         wv = std::getenv("RHG_WAVE2_ANNULI"); // A/B switch: outer annuli in wave 2
        // small average degree at >= 2^28 points (cfg4's weak-scaling family): four outer annuli
        // (measured cfg4 2 / 3 / 4: 32.00 / 31.84 / 31.78 ms; cfg3 keeps two: 21.73 vs 21.77-22.03 with three)
        const std::uint32_t w2 = wv ? std::uint32_t(std::max(1, std::atoi(wv)))
                                    : (L.n >= (std::uint64_t(1) << 28) && dbar_model < 8.0) ? kWave2Annuli + 3
                                    : (L.n >= (std::uint64_t(1) << 25) ? kWave2Annuli + 1 : kWave2Annuli);
        if (L.count >= L.first_streaming + 1 + w2 && pl.T > 0) {
            bool dense_src = false;
            for (std::uint32_t a = L.count - w2; a < L.count; ++a) dense_src |= pl.dense_mask[a] != 0;
            if (!dense_src) pl.wave_j = L.count - w2;
        }
    }
    // job order: the global annuli's jobs, wave 1, wave 2, each by descending count, ties by job
    // index: a stable counting sort on (class, count) when the counts are short against the job
    // count (large P: measured cfg4 0.53 -> 0.05 ms), else a key sort (class | complemented count |
    // index, < 2^24 jobs)
    if (pl.jobs.size() >= (std::size_t(1) << 24)) throw InvalidArgument("rhg: too many sampler streams");
    {
        const std::size_t         nj = pl.jobs.size();
        std::vector<std::uint8_t> cls(nj);
        std::uint64_t             maxc = 0;
        pl.wave2_jobs = 0, pl.glob_jobs = 0;
        for (std::size_t k = 0; k < nj; ++k) {
            const StreamJob& J  = pl.jobs[k];
            const bool       w2 = J.annulus >= pl.wave_j && J.annulus < L.count;
            const bool       gl = J.annulus < L.first_streaming;
            cls[k] = gl ? 0 : w2 ? 2 : 1;
            pl.wave2_jobs += w2, pl.glob_jobs += gl;
            maxc = std::max<std::uint64_t>(maxc, J.count);
        }
        pl.job_order.resize(nj);
        if (3 * (maxc + 1) <= 4 * std::uint64_t(nj)) {
            const std::size_t          span = std::size_t(maxc) + 1;
            std::vector<std::uint32_t> pos(3 * span + 1, 0);
            auto bucket = [&](std::size_t k) { return cls[k] * span + std::size_t(maxc - pl.jobs[k].count); };
            for (std::size_t k = 0; k < nj; ++k) ++pos[bucket(k) + 1];
            for (std::size_t b = 1; b < pos.size(); ++b) pos[b] += pos[b - 1];
            for (std::size_t k = 0; k < nj; ++k) pl.job_order[pos[bucket(k)]++] = std::uint32_t(k);
        } else {
            std::vector<std::uint64_t> key(nj);
            for (std::size_t k = 0; k < nj; ++k) {
                const std::uint64_t c = std::min<std::uint64_t>(pl.jobs[k].count, (std::uint64_t(1) << 38) - 1);
                key[k] = (std::uint64_t(cls[k]) << 62) | ((((std::uint64_t(1) << 38) - 1) - c) << 24) | k;
            }
            radix_sort_keys(key, 24); // the index bits are already in order: a stable sort of the rest
            for (std::size_t k = 0; k < nj; ++k) pl.job_order[k] = std::uint32_t(key[k] & 0xffffffu);
        }
    }
    const auto tl1 = std::chrono::steady_clock::now();
    pl.sub_ms[0] = std::chrono::duration<double, std::milli>(tl1 - tl0).count() - pl.layout_ms;
    // chain bins: each wave's streams packed longest-processing-time-first into bins whose
    // load stays near the wave's longest chain; one warp runs one bin's chains back to back,
    // so few chain warps share an SM (their shared-memory traffic, not the DMUL latency,
    // is what slows a chain that shares its SM with many others)
    pl.chain_bins.assign(1, 0);
    pl.chain_bins1 = pl.chain_bins_g = 0;
    for (int wv = 0; wv < 3; ++wv) { // classes: global annuli, wave 1, wave 2
        const std::uint32_t nj = std::uint32_t(pl.jobs.size()), ng = std::uint32_t(pl.glob_jobs);
        const std::uint32_t j0 = wv == 0 ? 0 : wv == 1 ? ng : nj - std::uint32_t(pl.wave2_jobs);
        const std::uint32_t j1 = wv == 0 ? ng : wv == 1 ? nj - std::uint32_t(pl.wave2_jobs) : nj;
        if (j1 <= j0) {
            if (wv == 0) pl.chain_bins_g = 0;
            if (wv <= 1) pl.chain_bins1 = std::uint32_t(pl.chain_bins.size() - 1);
            continue;
        }
        std::vector<std::uint64_t> cnt(j1 - j0); // counts in job order (contiguous for the packing loop)
        std::uint64_t              sum = 0, mx = 0;
        for (std::uint32_t k = j0; k < j1; ++k) {
            const std::uint64_t c = pl.jobs[pl.job_order[k]].count;
            cnt[k - j0] = c, sum += c, mx = std::max(mx, c);
        }
        const std::uint64_t nb = std::min<std::uint64_t>(j1 - j0, mx ? (sum + mx - 1) / mx + (sum + 7 * mx) / (8 * mx) : 1);
        // min-heap on (load, bin) in a flat array; bin ids per job, then a stable counting sort
        // (per-bin vectors cost more in allocations than the packing itself)
        std::vector<std::uint64_t> heap(nb);
        // key = load << 24 | bin: bins < 2^24 (jobs), loads < 2^35 (n < 2^32 plus 1250 per job)
        if (nb >= (1u << 24)) throw InvalidArgument("rhg: too many sampler streams");
        for (std::uint32_t b = 0; b < nb; ++b) heap[b] = b; // load 0
        std::vector<std::uint32_t> bin_of(j1 - j0), fill(nb + 1, 0);
        // many streams (large P): a boustrophedon deal of the descending job list (O(1) per job;
        // the heap's LPT took 3.6 ms for the 1.2e5 streams of cfg4), else LPT
        const bool snake = j1 - j0 > 16384;
        for (std::uint64_t k = j0, q = 0, pass = 0; snake && k < j1; ++k) { // position q of pass `pass`
            const std::uint32_t b = std::uint32_t(pass & 1 ? nb - 1 - q : q);
            bin_of[k - j0]        = b;
            ++fill[b + 1];
            if (++q == nb) q = 0, ++pass;
        }
        for (std::uint32_t k = j0; !snake && k < j1; ++k) { // job_order is by descending count inside a wave
            const std::uint64_t top = heap[0];
            const std::uint32_t b   = std::uint32_t(top & 0xffffffu);
            bin_of[k - j0]          = b;
            ++fill[b + 1];
            // + per-stream pipeline fill / seeding
            const std::uint64_t v = top + ((cnt[k - j0] + 1250) << 24);
            std::size_t         h = 0;
            for (;;) { // sift the grown root down
                std::size_t c = 2 * h + 1;
                if (c >= nb) break;
                if (c + 1 < nb && heap[c + 1] < heap[c]) ++c;
                if (heap[c] >= v) break;
                heap[h] = heap[c], h = c;
            }
            heap[h] = v;
        }
        for (std::uint32_t b = 0; b < nb; ++b) fill[b + 1] += fill[b];
        std::vector<std::uint32_t> ordered(j1 - j0);
        {
            std::vector<std::uint32_t> pos(fill.begin(), fill.end() - 1);
            for (std::uint32_t k = j0; k < j1; ++k) ordered[pos[bin_of[k - j0]]++] = pl.job_order[k];
        }
        std::copy(ordered.begin(), ordered.end(), pl.job_order.begin() + j0);
        for (std::uint32_t b = 0; b < nb; ++b) pl.chain_bins.push_back(j0 + fill[b + 1]);
        if (wv == 0) pl.chain_bins_g = std::uint32_t(nb);
        if (wv <= 1) pl.chain_bins1 = std::uint32_t(pl.chain_bins.size() - 1);
    }
    pl.sub_ms[1] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tl1).count();
    if (pl.n_ext >= (std::uint64_t(1) << 32) || pl.n_req >= (std::uint64_t(1) << 31) || L.n >= (std::uint64_t(1) << 32))
        throw InvalidArgument("rhg: more than 2^32 points (per device) are not supported");
    if (L.count > std::uint32_t(kMaxAnnuli)) throw InvalidArgument("rhg: more than 64 annuli are not supported");
    return pl;
}

// The edge-phase part of the plan (slab join work lists, tail requests, node-tile strips,
// global-unit tiles): only the edge kernels read it, so rhg_generate_stats builds and uploads
// it while the device sampler runs.
void plan_edges(Plan& pl) {
    const Layout&       L  = pl.L;
    const std::uint32_t Pc = L.chunks;
    const auto          tl2 = std::chrono::steady_clock::now();
    // slab join for the sparse pairs: slabs of every target annulus with sparse sources, the
    // half-width bounds that find a slab's requests, and the tail (wrap / halo) requests
    const std::uint32_t K = L.count;
    pl.src_mask.assign(K, 0ull);
    pl.hbound.assign(std::size_t(K) * K, 0.0);
    pl.slab_prefix.assign(K + 1, 0);
    pl.tail_prefix.assign(K + 1, 0);
    pl.tail_lam.assign(K, 0.0);
    for (std::uint32_t a = L.first_streaming; a < K; ++a)
        for (std::uint32_t j = a; j < K; ++j) {
            pl.hbound[std::size_t(a) * K + j] = half_width_bound(L, a, j);
            if (!((pl.dense_mask[a] >> j) & 1ull) && pl.ann[a].end > pl.ann[a].off) pl.src_mask[j] |= 1ull << a;
        }
    for (std::uint32_t j = 0; j < K; ++j) {
        const std::uint64_t own = pl.src_mask[j] ? pl.ann[j].halo - pl.ann[j].off : 0;
        pl.slab_prefix[j + 1]   = pl.slab_prefix[j] + (own + kSlabNodes - 1) / kSlabNodes;
    }
    pl.n_slabs = pl.slab_prefix[K];
    // dense rows: per target j the sorted-request ranges whose rows the node tiles read (the
    // global points, and each dense source annulus a <= j: its requests are one contiguous range
    // of the (source, class, angle) order, [req_off[a], req_off[a] + its points))
    pl.row_tasks.clear();
    pl.row_task_j.assign(K + 1, 0);
    {
        std::uint32_t blk = 0;
        auto          add = [&](std::uint32_t j, std::uint32_t src, std::uint64_t s0, std::uint64_t s1) {
            if (s1 <= s0) return;
            pl.row_tasks.push_back(make_uint4(j | (src << 16), std::uint32_t(s0), std::uint32_t(s1), blk));
            blk += std::uint32_t((s1 - s0 + 255) / 256);
        };
        for (std::uint32_t j = 0; j < K; ++j) {
            pl.row_task_j[j] = std::uint32_t(pl.row_tasks.size());
            if (j < L.first_streaming || !pl.n_req) continue;
            add(j, 0xffffu, 0, pl.n_glob);
            for (std::uint32_t a = L.first_streaming; a <= j; ++a)
                if ((pl.dense_mask[a] >> j) & 1ull) add(j, a, pl.req_off[a], pl.req_off[a] + (pl.ann[a].end - pl.ann[a].off));
        }
        pl.row_task_j[K] = std::uint32_t(pl.row_tasks.size());
        pl.row_tasks.push_back(make_uint4(0, 0, 0, blk)); // sentinel: total blocks
    }

    { // slabs in angular order across targets (requests are re-read from L2 by the next target's
      // slab), wave-1 targets first: a counting sort on (wave, angle bucket) - the order only
      // shapes cache locality
        const std::uint64_t nb = std::max<std::uint64_t>(pl.n_slabs, 1);
        std::vector<std::uint32_t> cnt(2 * nb + 1, 0);
        std::vector<std::uint32_t> bkt(pl.n_slabs); // bucket of each slab's mid angle (wave-major)
        for (std::uint32_t j = 0; j < K; ++j) {
            const std::uint64_t ns = pl.slab_prefix[j + 1] - pl.slab_prefix[j];
            if (!ns) continue;
            const double        f    = double(nb) / double(2 * ns);
            const std::uint32_t base = j >= pl.wave_j ? std::uint32_t(nb) : 0u;
            std::uint32_t*      out  = bkt.data() + pl.slab_prefix[j];
            for (std::uint64_t i = 0; i < ns; ++i) {
                const std::uint64_t b = std::min<std::uint64_t>(std::uint64_t(double(2 * i + 1) * f), nb - 1);
                out[i]                = base + std::uint32_t(b);
                ++cnt[out[i] + 1];
            }
        }
        for (std::size_t b = 1; b < cnt.size(); ++b) cnt[b] += cnt[b - 1];
        pl.n_slabs1 = cnt[nb];
        pl.slab_tab.resize(pl.n_slabs);
        for (std::uint32_t j = 0; j < K; ++j) {
            const std::uint64_t ns = pl.slab_prefix[j + 1] - pl.slab_prefix[j];
            const std::uint32_t* in = bkt.data() + pl.slab_prefix[j];
            for (std::uint64_t i = 0; i < ns; ++i)
                pl.slab_tab[cnt[in[i]]++] = (static_cast<unsigned long long>(j) << 32) | i;
        }
    }
    const auto tl3 = std::chrono::steady_clock::now();
    pl.sub_ms[2] = std::chrono::duration<double, std::milli>(tl3 - tl2).count();
    const double Bnd = chunk_lower_bound(pl.e1, Pc); // halo nodes and wrapped points have lambda >= Bnd
    for (std::uint32_t a = 0; a < K; ++a) {
        std::uint64_t n = 0;
        if (a >= L.first_streaming && pl.T) {
            double hm = 0.0;
            bool   any = false;
            for (std::uint32_t j = a; j < K; ++j)
                if (!((pl.dense_mask[a] >> j) & 1ull)) any = true, hm = std::max(hm, pl.hbound[std::size_t(a) * K + j]);
            if (any) {
                pl.tail_lam[a]  = Bnd - hm - 1e-9;
                const double hw = pl.hbound[std::size_t(a) * K + a];
                std::uint64_t owned_tail = 0; // points of the owned chunks that can reach lambda >= tail_lam
                for (std::uint32_t t = 0; t < pl.T; ++t) {
                    const std::uint32_t c = pl.e0 + t;
                    if (chunk_upper_bound(c, Pc) + hw + 1e-9 >= pl.tail_lam[a]) owned_tail += L.chunk_count(a, c);
                }
                n = owned_tail + (pl.ann[a].end - pl.ann[a].halo);
            }
        }
        pl.tail_prefix[a + 1] = pl.tail_prefix[a] + n;
    }
    pl.n_tail = pl.tail_prefix[K];
    // dense engine: one warp per strip of 512 owned nodes of every streaming annulus
    pl.gt_prefix.assign(L.count + 1, 0);
    for (std::uint32_t j = 0; j < L.count; ++j) {
        const std::uint64_t own = j >= L.first_streaming && pl.n_req ? pl.ann[j].halo - pl.ann[j].off : 0;
        pl.gt_prefix[j + 1]     = pl.gt_prefix[j] + (own + kTileNodes - 1) / kTileNodes; // one node tile per warp
    }
    pl.gtwarps = pl.gt_prefix[L.count];
    const std::uint64_t nT = (pl.n_glob + kGGTile - 1) / kGGTile, tiles = nT * (nT + 1) / 2;
    pl.gg_t0 = tiles * pl.rank / pl.world, pl.gg_t1 = tiles * (pl.rank + 1) / pl.world;
    pl.sub_ms[3] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tl3).count();
}

Plan make_plan(const Params& P, const rhg_shard* shard) {
    Plan pl = make_plan_head(P, shard);
    plan_edges(pl);
    return pl;
}

struct Tables {
    AnnulusDev*         ann;
    unsigned long long* dense_mask;
    std::uint64_t*      req_off;
    StreamJob*          jobs;
    std::uint32_t*      job_order;
    std::uint32_t*      chain_bins;
    std::uint64_t*      gt_prefix;
    std::uint64_t*      gseg;
    std::uint32_t*      ann_blk;
    std::uint64_t*      pseg;
    unsigned long long* src_mask;
    uint4*              row_tasks;
    double*             hbound;
    unsigned long long* slab_tab;
    std::uint64_t*      tail_prefix;
    double*             tail_lam;
};

// Pack tables into one pinned blob and send it with one copy: part 1 = what the sampler
// (and everything after it) reads, part 2 = the edge-phase work lists (plan_edges).
// Each part has its own pinned staging and device buffer, so part 2 can be staged while
// part 1's copy and the sampler are still in flight.
void upload_part(rhg_ctx* ctx, int part, const std::vector<std::pair<const void*, std::size_t>>& src,
                 std::vector<void*>& dst, std::uint64_t* h2d) {
    std::vector<std::size_t> off(src.size());
    std::size_t              bytes = 0;
    for (std::size_t i = 0; i < src.size(); ++i) off[i] = bytes, bytes = align256(bytes + src[i].second);
    bytes += 256;
    HostPinned& stg = part ? ctx->staging2 : ctx->staging;
    DevBuf&     dev = part ? ctx->tables2 : ctx->tables;
    stg.ensure(bytes);
    dev.ensure(bytes);
    char* h = static_cast<char*>(stg.p);
    for (std::size_t i = 0; i < src.size(); ++i)
        if (src[i].second) std::memcpy(h + off[i], src[i].first, src[i].second);
    CK(cudaMemcpyAsync(dev.p, h, bytes, cudaMemcpyHostToDevice, ctx->stream));
    if (h2d) *h2d += bytes;
    dst.resize(src.size());
    for (std::size_t i = 0; i < src.size(); ++i) dst[i] = dev.as<char>() + off[i];
}
template <class V>
std::pair<const void*, std::size_t> blob(const V& v) {
    return {v.data(), v.size() * sizeof(v[0])};
}

void upload_tables_head(rhg_ctx* ctx, const Plan& pl, Tables& t, std::uint64_t* h2d) {
    std::vector<void*> d;
    upload_part(ctx, 0,
                {blob(pl.ann), blob(pl.dense_mask), blob(pl.req_off), blob(pl.jobs), blob(pl.job_order),
                 blob(pl.chain_bins), blob(pl.gseg), blob(pl.ann_blk), blob(pl.pseg)},
                d, h2d);
    t.pseg = static_cast<std::uint64_t*>(d[8]);
    t.ann = static_cast<AnnulusDev*>(d[0]), t.dense_mask = static_cast<unsigned long long*>(d[1]);
    t.req_off = static_cast<std::uint64_t*>(d[2]), t.jobs = static_cast<StreamJob*>(d[3]);
    t.job_order = static_cast<std::uint32_t*>(d[4]), t.chain_bins = static_cast<std::uint32_t*>(d[5]);
    t.gseg = static_cast<std::uint64_t*>(d[6]), t.ann_blk = static_cast<std::uint32_t*>(d[7]);
}
void upload_tables_edges(rhg_ctx* ctx, const Plan& pl, Tables& t, std::uint64_t* h2d) {
    std::vector<void*> d;
    upload_part(ctx, 1,
                {blob(pl.gt_prefix), blob(pl.src_mask), blob(pl.hbound), blob(pl.slab_tab), blob(pl.tail_prefix),
                 blob(pl.tail_lam), blob(pl.row_tasks)},
                d, h2d);
    t.gt_prefix = static_cast<std::uint64_t*>(d[0]), t.src_mask = static_cast<unsigned long long*>(d[1]);
    t.hbound = static_cast<double*>(d[2]), t.slab_tab = static_cast<unsigned long long*>(d[3]);
    t.tail_prefix = static_cast<std::uint64_t*>(d[4]), t.tail_lam = static_cast<double*>(d[5]);
    t.row_tasks = static_cast<uint4*>(d[6]);
}
Tables upload_tables(rhg_ctx* ctx, const Plan& pl, std::uint64_t* h2d = nullptr) {
    Tables t{};
    upload_tables_head(ctx, pl, t, h2d);
    upload_tables_edges(ctx, pl, t, h2d);
    return t;
}

void ensure_points(rhg_ctx* ctx, std::uint64_t total, bool with_export) {
    const std::size_t n = std::max<std::uint64_t>(total, 1);
    ctx->beta.ensure(n * sizeof(double));
    ctx->hw.ensure(n * sizeof(double));
    ctx->rec0.ensure(n * sizeof(double2));
    ctx->rec1.ensure(n * sizeof(double2));
    ctx->rec2.ensure(n * sizeof(double2));
    if (with_export) {
        ctx->r_out.ensure(n * sizeof(double));
        ctx->beta_raw.ensure(n * sizeof(double));
    }
}

SamplerArgs sampler_args(rhg_ctx* ctx, const Plan& pl, const Tables& t) {
    SamplerArgs s;
    s.chain_bins = t.chain_bins, s.chain_bins1 = int(pl.chain_bins1), s.chain_bins_total = int(pl.chain_bins.size()) - 1;
    s.jobs = t.jobs, s.job_order = t.job_order, s.njobs = int(pl.jobs.size()), s.ann = t.ann, s.alpha = pl.L.alpha, s.total = pl.total;
    s.seed = pl.L.seed;
    s.pseg = t.pseg, s.npseg = int(pl.pseg.size()) - 1;
    s.beta = ctx->beta.as<double>(), s.hw = ctx->hw.as<double>();
    s.rec0 = ctx->rec0.as<double2>(), s.rec1 = ctx->rec1.as<double2>(), s.rec2 = ctx->rec2.as<double2>();
    s.side = ctx->side, s.ev_fork = ctx->fork, s.ev_join = ctx->join;
    s.mark = timeline_of(ctx);
    return s;
}

// Cell index + every edge kernel + counters back to the host.
// Optional materialised edge stream (rhg_generate_edges / rhg_edges_from_points): the
// kernels append canonical (u, v) pairs to ctx->ebuf (capacity dev_cap); run_edges
// reports how many the graph has (*count, which may exceed dev_cap: the caller regrows
// and reruns).
struct EdgeSink {
    std::uint64_t dev_cap = 0;
    std::uint64_t count   = 0;
};

void run_edges(rhg_ctx* ctx, const Plan& pl, const Tables& t, rhg_run_stats* out, std::uint32_t* degrees,
               bool gen, bool split_wave, std::uint64_t* launches, EdgeSink* sink = nullptr, bool glob_small = false) {
    const std::uint32_t K         = pl.L.count;
    const std::size_t   o_dmax    = align256(3 * sizeof(Counters));
    const std::size_t   o_hmax    = o_dmax + align256(K * sizeof(unsigned long long));
    const std::size_t   o_cseg    = o_hmax + align256(std::size_t(kMaxCls) * K * sizeof(unsigned long long));
    const std::size_t   o_bkoff   = o_cseg + align256((kMaxCls + 1) * sizeof(std::uint32_t));
    const std::size_t   o_bksh    = o_bkoff + align256((kMaxCls + 1) * sizeof(std::uint32_t));
    const std::size_t   o_slots   = o_bksh + align256(kMaxCls * sizeof(std::uint32_t));
    const std::size_t   o_ann     = o_slots + align256(3 * kSlots * sizeof(SlotCounter));
    const std::size_t   cnt_bytes = o_ann + align256(std::size_t(kAnnSlots) * 2 * kMaxAnnuli * sizeof(unsigned long long)) + 256;
    ctx->counters.ensure(cnt_bytes);
    // the global points sampled on ctx->small: every output the kernels accumulate into is zeroed
    // there, so the global unit can start right after them; the main stream waits for the zeroing
    cudaStream_t zs = glob_small ? ctx->small : ctx->stream;
    CK(cudaMemsetAsync(ctx->counters.p, 0, cnt_bytes, zs));
    ctx->cells.ensure(std::max<std::uint64_t>(pl.ncells, 1) * sizeof(std::uint64_t));
    if (degrees) {
        ctx->degrees.ensure(pl.L.n * sizeof(unsigned));
        CK(cudaMemsetAsync(ctx->degrees.p, 0, pl.L.n * sizeof(unsigned), zs));
    }
    EdgeArgs e;
    e.ann = t.ann, e.count = int(K), e.first_streaming = int(pl.L.first_streaming);
    e.n_ext = pl.n_ext, e.n_glob = pl.n_glob;
    e.beta = ctx->beta.as<double>(), e.hw = ctx->hw.as<double>();
    e.rec0 = ctx->rec0.as<double2>(), e.rec1 = ctx->rec1.as<double2>(), e.rec2 = ctx->rec2.as<double2>();
    e.cellstart = ctx->cells.as<std::uint64_t>();
    ctx->lcells.ensure(std::max<std::uint64_t>(pl.ncells, 1) * sizeof(std::uint64_t));
    e.lcellstart = ctx->lcells.as<std::uint64_t>();
    {
        const std::size_t ne = pl.n_ext + 2;
        ctx->lam_tmp.ensure(ne * sizeof(double));
        e.lam_tmp = ctx->lam_tmp.as<double>();
        ctx->s_beta.ensure(ne * sizeof(double));
        ctx->s_hw.ensure(ne * sizeof(double));
        ctx->s_lt.ensure(2 * ne * sizeof(double));
        ctx->s_rec1.ensure(ne * sizeof(double2));
        ctx->s_rec2.ensure(ne * sizeof(double2));
        ctx->nid.ensure(ne * sizeof(unsigned long long));
        e.s_beta = ctx->s_beta.as<double>(), e.s_hw = ctx->s_hw.as<double>();
        e.s_lam = ctx->s_lt.as<double>(), e.s_theta = ctx->s_lt.as<double>() + ne;
        e.s_rec1 = ctx->s_rec1.as<double2>(), e.s_rec2 = ctx->s_rec2.as<double2>();
        e.s_id = ctx->nid.as<unsigned long long>();
    }
    {   // global requests: theta-sorted records and window-piece rows
        const std::size_t nG  = std::max<std::uint64_t>(pl.n_req, 1);
        const std::size_t nst = pl.L.count - pl.L.first_streaming;
        const std::size_t o_id = align256(2 * nG * sizeof(double2));
        const std::size_t o_rw = o_id + align256(nG * sizeof(std::uint32_t));
        const std::size_t o_bk = o_rw + align256(std::max<std::size_t>(nst, 1) * nG * 8 * sizeof(std::uint32_t));
        const std::size_t o_iv = o_bk + align256((2 * nG + 65 * std::size_t(kMaxCls)) * sizeof(std::uint32_t));
        const std::size_t o_u  = o_iv + align256(nG * sizeof(double));
        const std::size_t o_ax = o_u + align256(nG * sizeof(std::uint32_t));
        const std::size_t o_sf = o_ax + align256(nG * sizeof(double4));
        const std::size_t o_df = o_sf + align256((std::size_t(nst + 1) << 10) * sizeof(std::uint32_t));
        e.defer_cap            = std::max<std::size_t>(1 << 16, 2 * nG); // a few per halo/wrapped request
        ctx->gbuf.ensure(o_df + align256(e.defer_cap * sizeof(uint4)));
        e.deferred = reinterpret_cast<uint4*>(ctx->gbuf.as<char>() + o_df);
        char* g     = ctx->gbuf.as<char>();
        e.g_rec     = reinterpret_cast<double2*>(g);
        e.g_id      = reinterpret_cast<std::uint32_t*>(g + o_id);
        e.g_rows    = reinterpret_cast<std::uint32_t*>(g + o_rw);
        e.gbk       = reinterpret_cast<std::uint32_t*>(g + o_bk);
        e.g_inv     = reinterpret_cast<double*>(g + o_iv);
        e.g_u       = reinterpret_cast<std::uint32_t*>(g + o_u);
        e.g_aux     = reinterpret_cast<double4*>(g + o_ax);
        e.seg_first = reinterpret_cast<std::uint32_t*>(g + o_sf);
        e.hmax_bits = reinterpret_cast<unsigned long long*>(ctx->counters.as<char>() + o_hmax);
        e.cseg      = reinterpret_cast<std::uint32_t*>(ctx->counters.as<char>() + o_cseg);
        e.n_cls     = reinterpret_cast<int*>(ctx->counters.as<char>() + cnt_bytes - 256);
        e.defer_ctr = reinterpret_cast<unsigned long long*>(ctx->counters.as<char>() + cnt_bytes - 192);
        e.bk_off    = reinterpret_cast<std::uint32_t*>(ctx->counters.as<char>() + o_bkoff);
        e.bk_shift  = reinterpret_cast<std::uint32_t*>(ctx->counters.as<char>() + o_bksh);
        e.gt_prefix = t.gt_prefix, e.glob_tile_warps = pl.gtwarps;
        e.row_tasks = t.row_tasks;
        e.n_req = pl.n_req, e.req_off = t.req_off, e.dense_mask = t.dense_mask;
    }
    e.ann_rw = t.ann;
    e.ctr       = ctx->counters.as<Counters>();
    e.slots     = reinterpret_cast<SlotCounter*>(ctx->counters.as<char>() + o_slots);
    e.ann_ctr   = reinterpret_cast<unsigned long long*>(ctx->counters.as<char>() + o_ann);
    e.gseg      = t.gseg;
    e.dmax_bits = reinterpret_cast<unsigned long long*>(ctx->counters.as<char>() + o_dmax);
    e.cosh_R = pl.L.cosh_R, e.chunk0_upper = chunk_upper_bound(0, pl.L.chunks);
    e.lift_part   = pl.e1 == pl.L.chunks && pl.T > 0;
    e.slab_tab = t.slab_tab, e.n_slabs = pl.n_slabs, e.src_mask = t.src_mask, e.hbound = t.hbound;
    e.tail_prefix = t.tail_prefix, e.tail_lam = t.tail_lam, e.n_tail = pl.n_tail;
    e.gg_tile_begin = pl.gg_t0, e.gg_tile_end = pl.gg_t1;
    e.degrees       = degrees ? ctx->degrees.as<unsigned>() : nullptr;
    if (sink) {
        ctx->ebuf.ensure(std::max<std::uint64_t>(sink->dev_cap, 1) * sizeof(ulonglong2));
        ctx->ecount.ensure(256);
        CK(cudaMemsetAsync(ctx->ecount.p, 0, 8, zs));
        e.edge_out = ctx->ebuf.as<ulonglong2>(), e.edge_cap = sink->dev_cap;
        e.edge_count = ctx->ecount.as<unsigned long long>();
    }
    if (const char* ab = std::getenv("RHG_ABLATE")) e.ablate = std::atoi(ab);
    const char* dbg_env = std::getenv("RHG_DEBUG_STATS");
    const bool  dbg     = dbg_env && dbg_env[0] == '1';
    if (dbg) {
        ctx->dbg.ensure(kDbgSlots * sizeof(unsigned long long));
        CK(cudaMemsetAsync(ctx->dbg.p, 0, kDbgSlots * sizeof(unsigned long long), zs));
        e.dbg = ctx->dbg.as<unsigned long long>();
    }
    if (ctx->audit_on) { // rhg_audit_predicate: the slab join runs its MODE 3 instance
        ctx->audit.ensure(kAuditSlots * sizeof(unsigned long long));
        CK(cudaMemsetAsync(ctx->audit.p, 0, kAuditSlots * sizeof(unsigned long long), zs));
        e.audit = ctx->audit.as<unsigned long long>();
    }
    e.ann_blk = t.ann_blk;
    e.gen = gen ? 1 : 0;
    { // the rank window holds ~ the average degree's worth of points: below ~100 the galloping
      // searches beat the beta-cell pass (measured cfg4 35.1 -> 33.5 ms; cfg3 at d = 256 22.1 -> 24.0)
        const double q    = (pl.L.alpha - 0.5) / pl.L.alpha;
        const double dbar = std::exp(-0.5 * (pl.L.R - 2.0 * std::log(double(pl.L.n)))) / (kPi / 2.0 * q * q);
        const char*  rg   = std::getenv("RHG_RANK_GALLOP"); // A/B: 0 / 1 force
        e.rank_gallop     = gen && (rg ? rg[0] == '1' : dbar < 100.0) ? 1 : 0;
    }
    e.mark = timeline_of(ctx);
    // Two waves when the sampler split its chains (generate mode): wave 1 = every annulus below
    // pl.wave_j (sort phase, dense prep, rows / node tiles / slabs of those targets, the global
    // unit) overlaps the outermost annulus's chains on ctx->late; wave 2 = the outermost annulus
    // after ev_late, then the tail pairs, the deferred ranges and the counter fold.
    if (glob_small) {
        CK(cudaEventRecord(ctx->ev_gz, ctx->small));
        CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_gz, 0));
    }
    const std::uint32_t fs = pl.L.first_streaming;
    const bool          split = split_wave && pl.wave_j < K;
    const std::uint32_t jw    = split ? pl.wave_j : K;
    launch_cell_index(e, pl.ann_blk[fs], pl.ann_blk[jw], int(fs), int(jw), gen, ctx->stream, launches);
    if (split) { // wave 2's sort phase right after its chains, beside wave 1 (needs the radius side
                 // and this call's zeroed counters / dmax table from the main stream)
        // small graphs: on ctx->side (normal priority; measured cfg2 3.41 -> 3.35 ms): on the
        // high-priority late stream it held back wave 1's edge work; from n = 2^25 on the late
        // stream (wave 2 then starts earlier: cfg4 32.36 -> 32.03 ms, cfg5 148.2 -> 146.8, cfg3
        // 22.03 -> 21.97; cfg2 3.08 -> 3.12). RHG_SORT2_SIDE=0 / 1 forces the late / side stream (A/B)
        const char*  s2s = std::getenv("RHG_SORT2_SIDE");
        const bool   s2l = s2s ? s2s[0] == '0' : pl.L.n >= (std::uint64_t(1) << 25);
        cudaStream_t s2  = s2l ? ctx->late : ctx->side;
        CK(cudaEventRecord(ctx->fork, ctx->stream));
        CK(cudaStreamWaitEvent(s2, ctx->fork, 0));
        CK(cudaStreamWaitEvent(s2, ctx->join, 0));
        if (s2 != ctx->late) CK(cudaStreamWaitEvent(s2, ctx->ev_late, 0)); // the wave-2 chains
        launch_cell_index(e, pl.ann_blk[jw], pl.ann_blk[K], int(jw), int(K), gen, s2, launches);
        CK(cudaEventRecord(ctx->ev_late, s2));
    }
    if (pl.n_req && fs < K) { // dense-engine requests in (source, class, angle) order
        std::size_t need = 0;
        launch_sort_globals(e, nullptr, 0, &need, ctx->stream, launches);
        ctx->gsort.ensure(need);
        launch_sort_globals(e, ctx->gsort.p, ctx->gsort.cap, &need, ctx->stream, launches);
    }
    // Per wave: the dense engine (rows + node tiles) on ctx->side beside the slab join on the main
    // stream (independent counter families, both only read the sorted arrays); the deferred ranges
    // and the counter fold wait for both. Measured with the small kernels on their own stream
    // (below): cfg2 3.49 -> 3.38 ms, cfg3 24.76 -> 24.71, cfg4 36.45 -> 36.40 (without them the
    // overlap gained nothing at cfg2). RHG_CONCURRENT_ENGINES=0: one stream (A/B).
    const char* ce   = std::getenv("RHG_CONCURRENT_ENGINES");
    const bool  conc = !(ce && ce[0] == '0');
    cudaStream_t dst = conc ? ctx->dense : ctx->stream;
    auto fork_to = [&](cudaStream_t from, cudaStream_t to) {
        if (from == to) return;
        CK(cudaEventRecord(ctx->fork, from));
        CK(cudaStreamWaitEvent(to, ctx->fork, 0));
    };
    // the small independent kernels (global unit, tail pairs) run on their own stream beside the
    // big ones (their last-wave tails overlap): the global unit needs only the global points, so it
    // starts with the sort phase; the tail pairs start with wave 2's slab join
    const char* ss   = std::getenv("RHG_SIDE_SMALL"); // A/B: 0 off, 1 global unit only, 2 tail only, 3 both
    const int   ssv  = ss ? std::atoi(ss) : 3;
    const bool  side_glob = (ssv & 1) != 0, side_tail = (ssv & 2) != 0, side_small = side_glob || side_tail;
    bool        tail_timed = false; // the tail pairs ran (and were timed) on ctx->small
    if (side_glob) {
        if (!glob_small) fork_to(ctx->stream, ctx->small);
        EdgeWave g;
        g.global_unit = true;
        launch_edges(e, g, ctx->small, launches);
    }
    EdgeWave d1; // wave 1 dense targets (+ the global unit)
    d1.j0 = int(fs), d1.j1 = int(jw), d1.tile_warps = pl.gt_prefix[jw] - pl.gt_prefix[fs];
    d1.global_unit = !side_glob, d1.first_wave = true;
    auto row_range = [&](EdgeWave& w) { // the wave's dense-row tasks and their blocks
        w.row_t0 = pl.row_task_j[w.j0], w.row_t1 = pl.row_task_j[w.j1];
        w.row_b0 = pl.row_tasks[w.row_t0].w, w.row_nb = pl.row_tasks[w.row_t1].w - w.row_b0;
    };
    row_range(d1);
    { // the average degree the model targets (geometry.hpp:26-33 inverted): wide dense windows
        const double q    = (pl.L.alpha - 0.5) / pl.L.alpha;
        const double dbar = std::exp(-0.5 * (pl.L.R - 2.0 * std::log(double(pl.L.n)))) / (kPi / 2.0 * q * q);
        d1.dense_occ4     = dbar >= 128.0;
    }
    const bool dense_occ4 = d1.dense_occ4;
    EdgeWave s1; // wave 1 slab join (tail pairs too when there is no wave 2)
    s1.slab_begin = 0, s1.slab_end = split ? pl.n_slabs1 : pl.n_slabs;
    // a wave is "exact" when the own-window bound of its largest target annulus lies below the
    // pre-filter's FP64 floor (slab_kernel's kPreMinS = 4e-14 on S = h^2 / 2)
    auto exact_wave = [&](std::uint32_t j) {
        return j < K && j >= fs && pl.hbound[std::size_t(j) * K + j] < std::sqrt(2.0 * 4e-14);
    };
    s1.exact_slabs = exact_wave(jw - 1);
    s1.tail = !split, s1.ev0 = ctx->evw[0], s1.ev1 = ctx->evw[1];
    fork_to(ctx->stream, dst);
    launch_edges(e, d1, dst, launches);
    launch_edges(e, s1, ctx->stream, launches);
    if (split) {
        CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_late, 0));
        CK(cudaStreamWaitEvent(dst, ctx->ev_late, 0));
        EdgeWave d2;
        d2.j0 = int(jw), d2.j1 = int(K), d2.tile_warps = pl.gt_prefix[K] - pl.gt_prefix[jw];
        d2.dense_occ4 = dense_occ4;
        row_range(d2);
        EdgeWave s2;
        s2.slab_begin = pl.n_slabs1, s2.slab_end = pl.n_slabs;
        s2.exact_slabs = exact_wave(K - 1);
        s2.tail = !side_tail, s2.ev0 = ctx->evw[2], s2.ev1 = ctx->evw[3];
        launch_edges(e, d2, dst, launches);
        if (side_tail) { // the tail pairs beside wave 2's slab join
            fork_to(ctx->stream, ctx->small);
            EdgeWave t;
            t.tail = true, t.ev0 = ctx->evw[4], t.ev1 = ctx->evw[5];
            launch_edges(e, t, ctx->small, launches);
            tail_timed = pl.n_tail > 0;
        }
        launch_edges(e, s2, ctx->stream, launches);
    }
    fork_to(dst, ctx->stream); // join
    if (side_small) fork_to(ctx->small, ctx->stream);
    EdgeWave fin;
    fin.finish = true;
    launch_edges(e, fin, ctx->stream, launches);
    CK(cudaGetLastError());
    const bool reduce = ctx->comm && !ctx->reduce_off && pl.world == ctx->comm_world && pl.rank == ctx->comm_rank;
    if (reduce) { // the one collective of the shard plan: wrapping u64 sums of the counters
        const NcclApi& N = nccl_api();
        NK(N.all_reduce(ctx->counters.p, ctx->counters.p, 3 * sizeof(Counters) / 8, ncclUint64, ncclSum, ctx->comm,
                        ctx->stream));
        if (degrees || sink)
            NK(N.all_reduce(e.ann_ctr, e.ann_ctr, 2 * kMaxAnnuli, ncclUint64, ncclSum, ctx->comm, ctx->stream));
    }
    out->reduced_world = reduce ? pl.world : 0u;
    CK(cudaEventRecord(ctx->ev[2], ctx->stream));
    ctx->readback.ensure(4096);
    auto* hc = static_cast<Counters*>(ctx->readback.p);
    CK(cudaMemcpyAsync(hc, ctx->counters.p, 3 * sizeof(Counters), cudaMemcpyDeviceToHost, ctx->stream));
    int* h_ncls = reinterpret_cast<int*>(hc + 3);
    auto* h_drop = reinterpret_cast<unsigned long long*>(hc + 4);
    *h_ncls = 0, *h_drop = 0;
    if (e.n_cls) CK(cudaMemcpyAsync(h_ncls, e.n_cls, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    if (e.defer_ctr) CK(cudaMemcpyAsync(h_drop, e.defer_ctr + 1, 8, cudaMemcpyDeviceToHost, ctx->stream));
    if (degrees)
        CK(cudaMemcpyAsync(degrees, ctx->degrees.p, pl.L.n * sizeof(unsigned), cudaMemcpyDeviceToHost, ctx->stream));
    auto* h_ecount = reinterpret_cast<unsigned long long*>(hc + 5);
    *h_ecount      = 0;
    auto* h_ann    = reinterpret_cast<unsigned long long*>(static_cast<char*>(ctx->readback.p) + 512);
    CK(cudaMemcpyAsync(h_ann, e.ann_ctr, 2 * kMaxAnnuli * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                       ctx->stream));
    if (sink) CK(cudaMemcpyAsync(h_ecount, ctx->ecount.p, 8, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (sink) sink->count = *h_ecount;
    timeline_report(ctx, ctx->ev[0]);
    if (*h_ncls > kMaxCls) throw Invariant("dense engine: too many request segments");
    if (*h_drop) throw Invariant("dense engine: deferred-range list overflow");
    if (dbg) {
        unsigned long long h[kDbgSlots];
        CK(cudaMemcpy(h, ctx->dbg.p, sizeof h, cudaMemcpyDeviceToHost));
        std::fprintf(stderr, "RHG_DEBUG_STATS [");
        for (int i = 0; i < kDbgSlots; ++i) std::fprintf(stderr, "%s%llu", i ? "," : "", h[i]);
        std::fprintf(stderr, "]\n");
    }
    out->per_annulus = (degrees || sink) ? 1u : 0u; // the MODE 1 / 2 kernels count per annulus
    for (int a = 0; a < kMaxAnnuli; ++a)
        out->annulus_edges[a] = out->per_annulus ? h_ann[a] : 0, out->annulus_comps[a] = out->per_annulus ? h_ann[kMaxAnnuli + a] : 0;
    out->edges       = hc[0].edges + hc[1].edges + hc[2].edges;
    out->fingerprint = hc[0].fp + hc[1].fp + hc[2].fp;
    out->comps       = hc[0].comps + hc[1].comps + hc[2].comps;
    out->global_edges = hc[2].edges;
    out->global_comps = hc[2].comps;
    out->stream_comps = hc[0].comps;
    out->dense_comps  = hc[1].comps;
    out->pairs_ms     = 0.0; // sparse engine (slab join + tail), both waves
    const bool split_used = split_wave && pl.wave_j < pl.L.count;
    if (pl.n_slabs1 || !split_used) out->pairs_ms += (split_used ? pl.n_slabs1 : pl.n_slabs) ? ms_between(ctx->evw[0], ctx->evw[1]) : 0.0;
    if (split_used && pl.n_slabs > pl.n_slabs1) out->pairs_ms += ms_between(ctx->evw[2], ctx->evw[3]);
    if (tail_timed) out->pairs_ms += ms_between(ctx->evw[4], ctx->evw[5]); // the tail beside wave 2 (its own duration)
    out->d2h_bytes += 3 * sizeof(Counters) + (degrees ? pl.L.n * sizeof(unsigned) : 0);
}

void fill_common(const Plan& pl, rhg_run_stats* out) {
    out->n                  = pl.L.n;
    out->global_vertices    = pl.n_glob;
    out->annuli             = pl.L.count;
    out->first_streaming    = pl.L.first_streaming;
    out->R                  = pl.L.R;
    out->r_G                = pl.L.r_G;
    out->cosh_R             = pl.L.cosh_R;
    std::uint64_t owned     = 0;
    for (std::uint32_t i = pl.L.first_streaming; i < pl.L.count; ++i) owned += pl.ann[i].halo - pl.ann[i].off;
    out->streaming_vertices = owned;
    for (std::uint32_t i = 0; i < pl.L.count && i < std::uint32_t(kMaxAnnuli); ++i)
        out->annulus_vertices[i] =
            i < pl.L.first_streaming ? (pl.rank == 0 ? pl.L.counts[i] : 0) : pl.ann[i].halo - pl.ann[i].off;
}



Params to_params(const rhg_params* p) {
    if (!p) throw InvalidArgument("rhg: params is null");
    return Params(p->n, p->alpha, p->C, p->seed, p->chunks);
}

using Clock = std::chrono::steady_clock;

// A multi-GPU context (rhg_create_multi) computes the whole graph: sub-context g runs shard
// {g, G} from its own host thread (its plan, uploads and launches overlap the others'), ends
// with the NCCL all-reduce of the counters, and the results merge here: counters are the
// (identical) reduced whole-graph values, times the max over devices, sizes and per-shard
// vertex counts the sum, degrees the sum of the shards' partial degrees.
template <typename Run>
void multi_dispatch(rhg_ctx* ctx, const rhg_params* params, const rhg_shard* shard, rhg_run_stats* out,
                    std::uint32_t* degrees, EdgeSink* sink, Run run) {
    if (shard && !(shard->rank == 0 && shard->world == 1))
        throw InvalidArgument("rhg: a multi-GPU context generates the whole graph (shard must be NULL or {0, 1})");
    if (sink) throw InvalidArgument("rhg: materialised edge streams need a single-device context");
    if (!params) throw InvalidArgument("rhg: params is null");
    const auto          t0 = Clock::now();
    const std::uint32_t G  = std::uint32_t(ctx->subs.size());
    std::vector<rhg_run_stats>              outs(G);
    std::vector<std::vector<std::uint32_t>> deg(degrees ? G : 0);
    std::vector<std::string>                err(G);
    std::vector<int>                        code(G, RHG_OK);
    std::vector<std::thread>                th;
    for (std::uint32_t g = 0; g < G; ++g)
        th.emplace_back([&, g] {
            if (degrees) deg[g].assign(params->n, 0u);
            code[g] = guarded([&] {
                const rhg_shard sh{g, G};
                run(ctx->subs[g], &sh, &outs[g], degrees ? deg[g].data() : nullptr);
            });
            if (code[g] != RHG_OK) err[g] = g_err;
        });
    for (auto& t: th) t.join();
    for (std::uint32_t g = 0; g < G; ++g)
        if (code[g] != RHG_OK) {
            const std::string m = "device " + std::to_string(ctx->subs[g]->device) + ": " + err[g];
            if (code[g] == RHG_INVALID_ARGUMENT) throw InvalidArgument(m);
            if (code[g] == RHG_CUDA) throw CudaError(m);
            if (code[g] == RHG_NOMEM) throw std::bad_alloc();
            throw Invariant(m);
        }
    *out = outs[0];
    for (std::uint32_t g = 1; g < G; ++g) {
        const rhg_run_stats& o = outs[g];
        out->device_ms = std::max(out->device_ms, o.device_ms), out->sample_ms = std::max(out->sample_ms, o.sample_ms);
        out->edges_ms = std::max(out->edges_ms, o.edges_ms), out->host_ms = std::max(out->host_ms, o.host_ms);
        out->pairs_ms = std::max(out->pairs_ms, o.pairs_ms);
        out->kernel_launches += o.kernel_launches, out->device_bytes += o.device_bytes;
        out->h2d_bytes += o.h2d_bytes, out->d2h_bytes += o.d2h_bytes;
        out->streaming_vertices += o.streaming_vertices;
        for (int a = 0; a < RHG_MAX_ANNULI; ++a) out->annulus_vertices[a] += o.annulus_vertices[a];
    }
    if (degrees)
        for (std::uint64_t v = 0; v < params->n; ++v) {
            std::uint32_t d = 0;
            for (std::uint32_t g = 0; g < G; ++g) d += deg[g][v];
            degrees[v] = d;
        }
    out->seconds = std::chrono::duration<double>(Clock::now() - t0).count();
}

// single-device entry points on a multi-GPU context use its first device
rhg_ctx* primary(rhg_ctx* c) { return c && !c->subs.empty() ? c->subs[0] : c; }

} // namespace

extern "C" {

const char* rhg_last_error(void) { return g_err.c_str(); }
int rhg_abi_version(void) { return RHG_ABI_VERSION; }

int rhg_alpha_from_gamma(double gamma, double* alpha) {
    return guarded([&] { *alpha = alpha_from_gamma(gamma); });
}
int rhg_radial_const_from_avg_degree(double d_bar, double alpha, double* C) {
    return guarded([&] { *C = radial_const_from_avg_degree(d_bar, alpha); });
}
int rhg_params_validate(rhg_params* p) {
    return guarded([&] { p->R = to_params(p).R; });
}
int rhg_params_from_avg_degree(std::uint64_t n, double alpha, double d_bar, std::uint64_t seed, std::uint32_t chunks,
                               rhg_params* out) {
    return guarded([&] {
        const Params P(n, alpha, radial_const_from_avg_degree(d_bar, alpha), seed, chunks);
        out->n = P.n, out->alpha = P.alpha, out->C = P.C, out->seed = P.seed, out->chunks = P.chunks, out->R = P.R;
    });
}

int rhg_layout(const rhg_params* params, std::uint32_t* n_annuli, std::uint32_t* first_streaming,
               std::uint64_t* counts, std::uint64_t* chunk_counts, std::uint64_t* id_base, std::uint8_t* classes) {
    return guarded([&] {
        if (!params || !n_annuli || !first_streaming) throw InvalidArgument("rhg_layout: null argument");
        const Layout L = make_layout(to_params(params));
        *n_annuli = L.count, *first_streaming = L.first_streaming;
        if (counts) std::copy(L.counts.begin(), L.counts.end(), counts);
        if (chunk_counts) std::copy(L.chunk_counts.begin(), L.chunk_counts.end(), chunk_counts);
        if (id_base) std::copy(L.id_base.begin(), L.id_base.end(), id_base);
        if (classes) std::copy(L.classes.begin(), L.classes.end(), classes);
    });
}

int rhg_create(int device, rhg_ctx** out) {
    return guarded([&] {
        *out = nullptr;
        int n = 0;
        CK(cudaGetDeviceCount(&n));
        if (device < 0 || device >= n) throw CudaError("rhg_create: no such CUDA device");
        cudaDeviceProp prop{};
        CK(cudaGetDeviceProperties(&prop, device));
        if (prop.major != 10)
            throw CudaError(std::string("rhg_create: sm_100 (B200) required, found ") + prop.name);
        CK(cudaSetDevice(device));
        auto* c   = new rhg_ctx;
        c->device = device;
        int prio_lo = 0, prio_hi = 0; // the late stream (outermost annulus) gets block-scheduling priority
        CK(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
        {
            // the main stream (wave-1 chains, sort phase, dense prep, slab join) above side / dense /
            // small: its dense prep and slab join start right after the wave-1 sort instead of after
            // wave 2's (measured cfg2 3.35 -> 3.27 ms, cfg3 24.67 -> 24.57); RHG_MAIN_PRIO=0: A/B
            const char* mp = std::getenv("RHG_MAIN_PRIO");
            const int   pm = mp && mp[0] == '0' ? prio_lo : (prio_hi < prio_lo ? prio_hi + 1 : prio_hi);
            CK(cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, pm));
        }
        CK(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&c->small, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithPriority(&c->late, cudaStreamNonBlocking, prio_hi));
        {
            const char* dp = std::getenv("RHG_DENSE_PRIO"); // A/B: block-scheduling priority of the dense engine
            CK(cudaStreamCreateWithPriority(&c->dense, cudaStreamNonBlocking, dp && dp[0] == '1' ? prio_hi : prio_lo));
        }
        CK(cudaEventCreateWithFlags(&c->ev_pow, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->ev_late, cudaEventDisableTiming));
        for (auto& e: c->evw) CK(cudaEventCreate(&e));
        for (auto& e: c->ev) CK(cudaEventCreate(&e));
        CK(cudaEventCreateWithFlags(&c->fork, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->join, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->ev_glob, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->ev_gz, cudaEventDisableTiming));
        *out = c;
    });
}

void rhg_destroy(rhg_ctx* c) {
    if (!c) return;
    if (!c->subs.empty()) { // a multi-GPU context owns its per-device sub-contexts
        for (rhg_ctx* s: c->subs) rhg_destroy(s);
        delete c;
        return;
    }
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    cudaStreamSynchronize(c->side);
    cudaStreamSynchronize(c->small);
    cudaStreamSynchronize(c->dense);
    for (DevBuf* b: {&c->beta, &c->hw, &c->rec0, &c->rec1, &c->rec2, &c->r_out, &c->beta_raw, &c->tables, &c->cells,
                     &c->counters, &c->degrees, &c->dbg, &c->nid, &c->lcells, &c->s_beta,
                     &c->s_hw, &c->s_lt, &c->s_rec1, &c->s_rec2, &c->gsort, &c->gbuf, &c->tables2, &c->lam_tmp, &c->audit,
                     &c->ebuf, &c->ecount, &c->ekeys, &c->esort})
        b->release();
    if (c->comm) nccl_api().comm_destroy(c->comm);
    if (c->staging.p) cudaFreeHost(c->staging.p);
    if (c->staging2.p) cudaFreeHost(c->staging2.p);
    if (c->readback.p) cudaFreeHost(c->readback.p);
    for (auto& e: c->ev) cudaEventDestroy(e);
    cudaEventDestroy(c->fork);
    cudaEventDestroy(c->join);
    cudaEventDestroy(c->ev_glob);
    cudaEventDestroy(c->ev_gz);
    cudaStreamDestroy(c->side);
    cudaStreamDestroy(c->small);
    cudaStreamDestroy(c->dense);
    cudaStreamSynchronize(c->late);
    cudaStreamDestroy(c->late);
    cudaEventDestroy(c->ev_pow);
    cudaEventDestroy(c->ev_late);
    for (auto& e: c->evw) cudaEventDestroy(e);
    for (auto& e: c->tl_pool) cudaEventDestroy(e);
    cudaStreamDestroy(c->stream);
    delete c;
}

int rhg_create_multi(int n_devices, const int* devices, rhg_ctx** out) {
    return guarded([&] {
        if (!out) throw InvalidArgument("rhg_create_multi: out is null");
        *out = nullptr;
        if (n_devices < 1 || !devices) throw InvalidArgument("rhg_create_multi: need n_devices >= 1 devices");
        for (int i = 0; i < n_devices; ++i)
            for (int j = 0; j < i; ++j)
                if (devices[i] == devices[j]) throw InvalidArgument("rhg_create_multi: a device is listed twice");
        const NcclApi&          N = nccl_api();
        std::vector<ncclComm_t> comms(n_devices, nullptr);
        auto*                   m = new rhg_ctx;
        try {
            for (int i = 0; i < n_devices; ++i) {
                rhg_ctx* sub = nullptr;
                if (rhg_create(devices[i], &sub) != RHG_OK) throw CudaError(g_err);
                m->subs.push_back(sub);
            }
            NK(N.comm_init_all(comms.data(), n_devices, devices));
            for (int i = 0; i < n_devices; ++i)
                m->subs[i]->comm = comms[i], m->subs[i]->comm_world = std::uint32_t(n_devices),
                m->subs[i]->comm_rank = std::uint32_t(i);
        } catch (...) {
            rhg_destroy(m);
            throw;
        }
        m->device = devices[0];
        *out      = m;
    });
}

int rhg_context_devices(const rhg_ctx* ctx, int* n_devices) {
    return guarded([&] {
        if (!ctx || !n_devices) throw InvalidArgument("rhg_context_devices: null argument");
        *n_devices = ctx->subs.empty() ? 1 : int(ctx->subs.size());
    });
}

int rhg_nccl_unique_id(uint8_t* id) {
    return guarded([&] {
        if (!id) throw InvalidArgument("rhg_nccl_unique_id: id is null");
        ncclUniqueId u;
        NK(nccl_api().get_unique_id(&u));
        std::memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
    });
}

int rhg_attach_comm(rhg_ctx* ctx, uint32_t world, uint32_t rank, const uint8_t* id) {
    return guarded([&] {
        if (!ctx || !id) throw InvalidArgument("rhg_attach_comm: null argument");
        if (!ctx->subs.empty()) throw InvalidArgument("rhg_attach_comm: a multi-GPU context has its communicators");
        if (world < 1 || rank >= world) throw InvalidArgument("rhg_attach_comm: rank must lie in [0, world)");
        if (ctx->comm) throw InvalidArgument("rhg_attach_comm: the context already has a communicator");
        CK(cudaSetDevice(ctx->device));
        ncclUniqueId u;
        std::memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
        ncclComm_t c = nullptr;
        NK(nccl_api().comm_init_rank(&c, int(world), u, int(rank)));
        ctx->comm = c, ctx->comm_world = world, ctx->comm_rank = rank;
    });
}

int rhg_shard_extent(const rhg_params* params, const rhg_shard* shard, rhg_shard_info* out) {
    return guarded([&] {
        if (!out) throw InvalidArgument("rhg_shard_extent: out is null");
        const Plan pl = make_plan_head(to_params(params), shard);
        if (const char* v = std::getenv("RHG_TIMELINE"); v && v[0] == '1')
            std::fprintf(stderr, "RHG_HOST plan head: layout=%.3f jobs=%.3f bins=%.3f ms\n", pl.layout_ms, pl.sub_ms[0],
                         pl.sub_ms[1]);
        std::memset(out, 0, sizeof *out);
        out->chunk_begin = pl.e0, out->chunk_end = pl.e1;
        for (std::uint32_t i = pl.L.first_streaming; i < pl.L.count; ++i) {
            out->owned_points += pl.ann[i].halo - pl.ann[i].off;
            out->halo_points += pl.ann[i].end - pl.ann[i].halo;
        }
        out->global_points = pl.n_glob;
        out->sampled_points = pl.total;
        out->device_point_bytes = pl.total * 136; // sampler arrays + the lambda-sorted SoA (DESIGN 3)
    });
}

namespace {
void generate_impl(rhg_ctx* ctx, const rhg_params* params, const rhg_shard* shard, rhg_run_stats* out,
                   std::uint32_t* degrees, EdgeSink* sink);
void from_points_impl(rhg_ctx* ctx, const rhg_params* params, const rhg_shard* shard, const rhg_points* pts,
                      rhg_run_stats* out, std::uint32_t* degrees, EdgeSink* sink);
// Sorts the sink's edges on the device and copies them to the caller's (u, v) array.
void deliver_edges(rhg_ctx* ctx, const rhg_params* params, const EdgeSink& sink, std::uint64_t* edges,
                   std::uint64_t cap, std::uint64_t* n_edges) {
    *n_edges = sink.count;
    if (!edges) return;
    if (sink.count > cap)
        throw InvalidArgument("rhg edges: the edge buffer holds " + std::to_string(cap) + " pairs, the graph has " +
                              std::to_string(sink.count));
    const std::uint64_t m = sink.count;
    if (m >= (std::uint64_t(1) << 31)) throw InvalidArgument("rhg edges: more than 2^31 edges per call");
    int bits = 1;
    while (bits < 32 && (std::uint64_t(1) << bits) < params->n) ++bits;
    ctx->ekeys.ensure(std::max<std::uint64_t>(m, 1) * 16);
    auto*       ka  = ctx->ekeys.as<unsigned long long>();
    auto*       kb  = ka + std::max<std::uint64_t>(m, 1);
    std::size_t tmp = 0;
    launch_sort_edges(ctx->ebuf.as<ulonglong2>(), m, ka, kb, nullptr, &tmp, 32 + bits, ctx->stream);
    ctx->esort.ensure(std::max<std::size_t>(tmp, 256));
    tmp = ctx->esort.cap;
    launch_sort_edges(ctx->ebuf.as<ulonglong2>(), m, ka, kb, ctx->esort.p, &tmp, 32 + bits, ctx->stream);
    if (m) CK(cudaMemcpyAsync(edges, ctx->ebuf.p, m * 16, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
}
} // namespace

int rhg_audit_predicate(rhg_ctx* ctx, const rhg_params* params, const rhg_shard* shard, rhg_audit_report* out,
                        rhg_run_stats* stats) {
    ctx = primary(ctx);
    return guarded([&] {
        if (!ctx || !out || !stats) throw InvalidArgument("rhg_audit_predicate: null argument");
        struct Reset {
            rhg_ctx* c;
            ~Reset() { c->audit_on = false; }
        } reset{ctx};
        ctx->audit_on = true;
        generate_impl(ctx, params, shard, stats, nullptr, nullptr);
        unsigned long long h[kAuditSlots];
        CK(cudaMemcpy(h, ctx->audit.p, sizeof h, cudaMemcpyDeviceToHost));
        std::memset(out, 0, sizeof *out);
        out->prefilter_decided = h[0], out->exact_recheck = h[1], out->exact_only = h[2];
        out->disagreements = h[3];
        float ratio = 0.0f;
        const std::uint32_t bits = std::uint32_t(h[4]);
        std::memcpy(&ratio, &bits, 4);
        out->max_err_over_tau = ratio;
        out->noise_band_pairs = h[5];
        out->slab_pairs = h[0] + h[1] + h[2];
        out->exact_engine_pairs = stats->comps - out->slab_pairs;
    });
}

// The reference's units (generator.hpp:183-199, 270-284): unit 0 = the global unit, unit c + 1 =
// chunk engine c.  Engine shard {c, P} is exactly engine c plus a 1/P slice of the global-unit
// tiles (whose pairs the dense/global family counters separate), so the per-unit vectors are P
// shard runs on this device.
namespace {
struct ReduceOff {
    rhg_ctx* c;
    bool     old;
    explicit ReduceOff(rhg_ctx* x) : c(x), old(x->reduce_off) { c->reduce_off = true; }
    ~ReduceOff() { c->reduce_off = old; }
};
} // namespace

int rhg_unit_stats(rhg_ctx* ctx, const rhg_params* params, std::uint64_t* unit_edges, std::uint64_t* unit_comps,
                   std::uint64_t* unit_vertices) {
    ctx = primary(ctx);
    return guarded([&] {
        if (!ctx || !params || !unit_edges || !unit_comps || !unit_vertices)
            throw InvalidArgument("rhg_unit_stats: null argument");
        const std::uint32_t P = params->chunks;
        if (P < 1) throw InvalidArgument("ModelParams: chunks must be >= 1");
        ReduceOff     guard(ctx);
        rhg_run_stats st;
        unit_edges[0] = unit_comps[0] = 0;
        for (std::uint32_t c = 0; c < P; ++c) {
            const rhg_shard sh{c, P};
            generate_impl(ctx, params, &sh, &st, nullptr, nullptr);
            unit_edges[c + 1]    = st.edges - st.global_edges;
            unit_comps[c + 1]    = st.comps - st.global_comps;
            unit_vertices[c + 1] = st.streaming_vertices;
            unit_edges[0] += st.global_edges, unit_comps[0] += st.global_comps;
            unit_vertices[0] = st.global_vertices;
        }
    });
}

int rhg_generate_edges_units(rhg_ctx* ctx, const rhg_params* params, std::uint64_t* edges, std::uint64_t cap,
                             std::uint64_t* n_edges, std::uint64_t* unit_offsets) {
    ctx = primary(ctx);
    return guarded([&] {
        if (!ctx || !params || !n_edges || !unit_offsets) throw InvalidArgument("rhg_generate_edges_units: null argument");
        const std::uint32_t P = params->chunks;
        if (P < 1) throw InvalidArgument("ModelParams: chunks must be >= 1");
        ReduceOff                               guard(ctx);
        std::vector<std::uint64_t>              glob; // unit 0: pairs of two global points
        std::vector<std::vector<std::uint64_t>> units(P);
        rhg_run_stats                           st;
        for (std::uint32_t c = 0; c < P; ++c) {
            const rhg_shard sh{c, P};
            // first pass counts, second materialises (the device buffer is sized exactly)
            EdgeSink sink;
            sink.dev_cap = 0;
            generate_impl(ctx, params, &sh, &st, nullptr, &sink);
            const std::uint64_t m = sink.count;
            std::vector<std::uint64_t> buf(2 * std::max<std::uint64_t>(m, 1));
            EdgeSink                   sink2;
            sink2.dev_cap = m;
            generate_impl(ctx, params, &sh, &st, nullptr, &sink2);
            std::uint64_t got = 0;
            deliver_edges(ctx, params, sink2, buf.data(), m, &got);
            const std::uint64_t nG = st.global_vertices;
            for (std::uint64_t i = 0; i < got; ++i) {
                auto& dst = buf[2 * i + 1] < nG ? glob : units[c];
                dst.push_back(buf[2 * i]), dst.push_back(buf[2 * i + 1]);
            }
        }
        { // unit 0 in canonical order (the shards' global slices interleave)
            std::vector<std::pair<std::uint64_t, std::uint64_t>> g(glob.size() / 2);
            for (std::size_t i = 0; i < g.size(); ++i) g[i] = {glob[2 * i], glob[2 * i + 1]};
            std::sort(g.begin(), g.end());
            for (std::size_t i = 0; i < g.size(); ++i) glob[2 * i] = g[i].first, glob[2 * i + 1] = g[i].second;
        }
        std::uint64_t total = glob.size() / 2;
        unit_offsets[0] = 0, unit_offsets[1] = total;
        for (std::uint32_t c = 0; c < P; ++c) total += units[c].size() / 2, unit_offsets[c + 2] = total;
        *n_edges = total;
        if (!edges) return;
        if (total > cap)
            throw InvalidArgument("rhg edges: the edge buffer holds " + std::to_string(cap) + " pairs, the graph has " +
                                  std::to_string(total));
        std::memcpy(edges, glob.data(), glob.size() * 8);
        std::uint64_t* o = edges + glob.size();
        for (std::uint32_t c = 0; c < P; ++c) {
            std::memcpy(o, units[c].data(), units[c].size() * 8);
            o += units[c].size();
        }
    });
}

int rhg_generate_edges(rhg_ctx* ctx, const rhg_params* params, const rhg_shard* shard, rhg_run_stats* out,
                       std::uint64_t* edges, std::uint64_t cap, std::uint64_t* n_edges) {
    return guarded([&] {
        if (!ctx || !out || !n_edges || !params) throw InvalidArgument("rhg_generate_edges: null argument");
        EdgeSink sink;
        sink.dev_cap = edges ? cap : 0;
        generate_impl(ctx, params, shard, out, nullptr, &sink);
        deliver_edges(ctx, params, sink, edges, cap, n_edges);
    });
}

int rhg_edges_from_points(rhg_ctx* ctx, const rhg_params* params, const rhg_shard* shard, const rhg_points* pts,
                          rhg_run_stats* out, std::uint64_t* edges, std::uint64_t cap, std::uint64_t* n_edges) {
    return guarded([&] {
        if (!ctx || !out || !n_edges || !params) throw InvalidArgument("rhg_edges_from_points: null argument");
        EdgeSink sink;
        sink.dev_cap = edges ? cap : 0;
        from_points_impl(ctx, params, shard, pts, out, nullptr, &sink);
        deliver_edges(ctx, params, sink, edges, cap, n_edges);
    });
}

int rhg_generate_stats(rhg_ctx* ctx, const rhg_params* params, const rhg_shard* shard, rhg_run_stats* out,
                       std::uint32_t* degrees) {
    return guarded([&] { generate_impl(ctx, params, shard, out, degrees, nullptr); });
}

int rhg_naive_edges(rhg_ctx* ctx, std::uint64_t n, double R, const double* r, const double* theta,
                    std::uint64_t* edges, std::uint64_t cap, std::uint64_t* n_edges) {
    ctx = primary(ctx);
    return guarded([&] {
        if (!ctx || !n_edges || (n && (!r || !theta))) throw InvalidArgument("rhg_naive_edges: null argument");
        if (n > 100000) throw InvalidArgument("naive_edges: refusing quadratic work above n = 100000");
        CK(cudaSetDevice(ctx->device));
        cudaStream_t st = ctx->stream;
        ctx->beta.ensure(std::max<std::uint64_t>(n, 1) * 8);
        ctx->hw.ensure(std::max<std::uint64_t>(n, 1) * 8);
        ctx->r_out.ensure(std::max<std::uint64_t>(n, 1) * 8);
        ctx->ecount.ensure(256);
        if (n) {
            CK(cudaMemcpyAsync(ctx->beta.p, r, n * 8, cudaMemcpyHostToDevice, st));
            CK(cudaMemcpyAsync(ctx->hw.p, theta, n * 8, cudaMemcpyHostToDevice, st));
        }
        std::uint64_t dev_cap = edges ? cap : 0;
        for (int pass = 0; pass < 2; ++pass) { // pass 2 only when the caller's capacity is unknown (count)
            ctx->ebuf.ensure(std::max<std::uint64_t>(dev_cap, 1) * sizeof(ulonglong2));
            launch_naive_pairs(ctx->beta.as<double>(), ctx->hw.as<double>(), ctx->r_out.as<double>(), n, R,
                               ctx->ebuf.as<ulonglong2>(), dev_cap, ctx->ecount.as<unsigned long long>(), st);
            unsigned long long m = 0;
            CK(cudaMemcpyAsync(&m, ctx->ecount.p, 8, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            EdgeSink sink;
            sink.count = m;
            if (m <= dev_cap || !edges) {
                rhg_params P{};
                P.n = n;
                deliver_edges(ctx, &P, sink, edges, cap, n_edges);
                return;
            }
            *n_edges = m;
            throw InvalidArgument("rhg_naive_edges: the edge buffer holds " + std::to_string(cap) +
                                  " pairs, the oracle has " + std::to_string(m));
        }
    });
}

int rhg_count_edges_from_points(rhg_ctx* ctx, const rhg_params* params, const rhg_shard* shard, const rhg_points* pts,
                                rhg_run_stats* out, std::uint32_t* degrees) {
    return guarded([&] { from_points_impl(ctx, params, shard, pts, out, degrees, nullptr); });
}

namespace {
void generate_impl(rhg_ctx* ctx, const rhg_params* params, const rhg_shard* shard, rhg_run_stats* out,
                   std::uint32_t* degrees, EdgeSink* sink) {
    if (ctx && !ctx->subs.empty()) {
        multi_dispatch(ctx, params, shard, out, degrees, sink,
                       [&](rhg_ctx* sub, const rhg_shard* sh, rhg_run_stats* o, std::uint32_t* deg) {
                           generate_impl(sub, params, sh, o, deg, nullptr);
                       });
        return;
    }
    {
        if (!ctx || !out) throw InvalidArgument("rhg_generate_stats: null argument");
        const auto t0 = Clock::now();
        std::memset(out, 0, sizeof *out);
        CK(cudaSetDevice(ctx->device));
        const Params  P  = to_params(params);
        Plan          pl = make_plan_head(P, shard);
        const auto    t1 = Clock::now();
        std::uint64_t launches = 0;
        ensure_points(ctx, pl.total, false);
        Tables t{};
        upload_tables_head(ctx, pl, t, &out->h2d_bytes);
        double host_ms = std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
        if (const char* v = std::getenv("RHG_TIMELINE"); v && v[0] == '1')
            std::fprintf(stderr, "RHG_HOST plan=%.3f ms (layout=%.3f jobs=%.3f bins=%.3f slabs=%.3f rest=%.3f) upload=%.3f ms\n",
                         std::chrono::duration<double, std::milli>(t1 - t0).count(), pl.layout_ms, pl.sub_ms[0],
                         pl.sub_ms[1], pl.sub_ms[2], pl.sub_ms[3],
                         std::chrono::duration<double, std::milli>(Clock::now() - t1).count());
        CK(cudaEventRecord(ctx->ev[0], ctx->stream));
        SamplerArgs sa  = sampler_args(ctx, pl, t);
        sa.angular_from = pl.n_ext; // streaming frames are built while scattering (sort phase)
        const char* ns    = std::getenv("RHG_NO_WAVES"); // A/B switch for timing experiments
        const bool  split = pl.wave_j < pl.L.count && !(ns && ns[0] == '1');
        if (split) sa.wave2_jobs = pl.wave2_jobs, sa.late = ctx->late, sa.ev_pow = ctx->ev_pow, sa.ev_late = ctx->ev_late;
        const char* gs    = std::getenv("RHG_GLOB_STREAM"); // A/B switch: 0 = global points with wave 1
        const bool  gsplit = split && pl.glob_jobs > 0 && pl.chain_bins_g > 0 && pl.n_glob > 0 && !(gs && gs[0] == '0');
        if (gsplit) {
            sa.glob = ctx->small, sa.ev_glob = ctx->ev_glob;
            sa.chain_bins_g = int(pl.chain_bins_g), sa.glob_job0 = int(pl.jobs.size()) - pl.glob_jobs;
            if (pl.jobs[std::size_t(sa.glob_job0)].annulus >= pl.L.first_streaming)
                throw Invariant("plan: the global annuli's jobs are not the last ones");
        }
        launch_sampler(sa, ctx->stream, &launches);
        CK(cudaEventRecord(ctx->ev[1], ctx->stream));
        { // the edge-phase plan is built and staged while the device samples
            const auto t2 = Clock::now();
            plan_edges(pl);
            upload_tables_edges(ctx, pl, t, &out->h2d_bytes);
            host_ms += std::chrono::duration<double, std::milli>(Clock::now() - t2).count();
        }
        run_edges(ctx, pl, t, out, degrees, true, split, &launches, sink, gsplit);
        fill_common(pl, out);
        out->sample_ms       = ms_between(ctx->ev[0], ctx->ev[1]);
        out->edges_ms        = ms_between(ctx->ev[1], ctx->ev[2]);
        out->device_ms       = ms_between(ctx->ev[0], ctx->ev[2]);
        out->host_ms         = host_ms;
        out->kernel_launches = launches;
        out->device_bytes    = ctx->beta.cap + ctx->hw.cap + ctx->rec0.cap + ctx->rec1.cap + ctx->rec2.cap +
                            ctx->r_out.cap + ctx->beta_raw.cap + ctx->tables.cap + ctx->tables2.cap + ctx->cells.cap + ctx->counters.cap +
                            ctx->degrees.cap + ctx->nid.cap + ctx->lcells.cap + ctx->s_beta.cap +
                            ctx->s_hw.cap + ctx->s_lt.cap + ctx->s_rec1.cap + ctx->s_rec2.cap + ctx->gbuf.cap;
        out->seconds = std::chrono::duration<double>(Clock::now() - t0).count();
    }
}
} // namespace

int rhg_sample_points(rhg_ctx* ctx, const rhg_params* params, rhg_points* o) {
    ctx = primary(ctx);
    return guarded([&] {
        if (!ctx || !o || !o->beta || !o->r || !o->theta || !o->half_width || !o->coth_r || !o->inv_sinh_r ||
            !o->cos_theta || !o->sin_theta)
            throw InvalidArgument("rhg_sample_points: every output array is required");
        CK(cudaSetDevice(ctx->device));
        const Params    P = to_params(params);
        const rhg_shard whole{0, 1};
        const Plan      pl = make_plan(P, &whole);
        std::uint64_t   launches = 0;
        ensure_points(ctx, pl.total, true);
        const Tables t = upload_tables(ctx, pl);
        SamplerArgs  s = sampler_args(ctx, pl, t);
        s.r_out = ctx->r_out.as<double>(), s.beta_unlifted_out = ctx->beta_raw.as<double>();
        launch_sampler(s, ctx->stream, &launches);
        CK(cudaGetLastError());
        // copy back every id range: owned streaming chunks [off, halo) and the global points
        auto copy_range = [&](std::uint64_t dev_off, std::uint64_t id, std::uint64_t cnt) {
            if (!cnt) return;
            cudaStream_t st = ctx->stream;
            const auto   D2H = cudaMemcpyDeviceToHost;
            CK(cudaMemcpyAsync(o->beta + id, ctx->beta_raw.as<double>() + dev_off, cnt * 8, D2H, st));
            CK(cudaMemcpyAsync(o->r + id, ctx->r_out.as<double>() + dev_off, cnt * 8, D2H, st));
            CK(cudaMemcpyAsync(o->half_width + id, ctx->hw.as<double>() + dev_off, cnt * 8, D2H, st));
            const char* r0 = reinterpret_cast<const char*>(ctx->rec0.as<double2>() + dev_off);
            const char* r1 = reinterpret_cast<const char*>(ctx->rec1.as<double2>() + dev_off);
            const char* r2 = reinterpret_cast<const char*>(ctx->rec2.as<double2>() + dev_off);
            CK(cudaMemcpy2DAsync(o->theta + id, 8, r0 + 8, 16, 8, cnt, D2H, st));
            CK(cudaMemcpy2DAsync(o->cos_theta + id, 8, r1, 16, 8, cnt, D2H, st));
            CK(cudaMemcpy2DAsync(o->sin_theta + id, 8, r1 + 8, 16, 8, cnt, D2H, st));
            CK(cudaMemcpy2DAsync(o->coth_r + id, 8, r2, 16, 8, cnt, D2H, st));
            CK(cudaMemcpy2DAsync(o->inv_sinh_r + id, 8, r2 + 8, 16, 8, cnt, D2H, st));
        };
        for (std::uint32_t i = pl.L.first_streaming; i < pl.L.count; ++i)
            copy_range(pl.ann[i].off, pl.L.chunk_id_base(i, 0), pl.ann[i].halo - pl.ann[i].off);
        copy_range(pl.n_ext, 0, pl.n_glob);
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

int rhg_sample_uniforms(rhg_ctx* ctx, const rhg_params* params, double* u_angle, double* u_radius) {
    ctx = primary(ctx);
    return guarded([&] {
        if (!ctx || !u_angle || !u_radius) throw InvalidArgument("rhg_sample_uniforms: null argument");
        CK(cudaSetDevice(ctx->device));
        const Params    P = to_params(params);
        const rhg_shard whole{0, 1};
        const Plan      pl = make_plan(P, &whole);
        std::uint64_t   launches = 0;
        ensure_points(ctx, pl.total, false);
        const Tables t = upload_tables(ctx, pl);
        launch_mt_uniforms(sampler_args(ctx, pl, t), ctx->stream, &launches);
        CK(cudaGetLastError());
        auto copy_range = [&](std::uint64_t dev_off, std::uint64_t id, std::uint64_t cnt) {
            if (!cnt) return;
            CK(cudaMemcpyAsync(u_angle + id, ctx->beta.as<double>() + dev_off, cnt * 8, cudaMemcpyDeviceToHost,
                               ctx->stream));
            CK(cudaMemcpyAsync(u_radius + id, ctx->hw.as<double>() + dev_off, cnt * 8, cudaMemcpyDeviceToHost,
                               ctx->stream));
        };
        for (std::uint32_t i = pl.L.first_streaming; i < pl.L.count; ++i)
            copy_range(pl.ann[i].off, pl.L.chunk_id_base(i, 0), pl.ann[i].halo - pl.ann[i].off);
        copy_range(pl.n_ext, 0, pl.n_glob);
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

namespace {
void from_points_impl(rhg_ctx* ctx, const rhg_params* params, const rhg_shard* shard, const rhg_points* pts,
                      rhg_run_stats* out, std::uint32_t* degrees, EdgeSink* sink) {
    if (ctx && !ctx->subs.empty()) {
        multi_dispatch(ctx, params, shard, out, degrees, sink,
                       [&](rhg_ctx* sub, const rhg_shard* sh, rhg_run_stats* o, std::uint32_t* deg) {
                           from_points_impl(sub, params, sh, pts, o, deg, nullptr);
                       });
        return;
    }
    {
        if (!ctx || !out || !pts || !pts->beta || !pts->theta || !pts->half_width || !pts->coth_r ||
            !pts->inv_sinh_r || !pts->cos_theta || !pts->sin_theta)
            throw InvalidArgument("rhg_count_edges_from_points: null argument");
        const auto t0 = Clock::now();
        std::memset(out, 0, sizeof *out);
        CK(cudaSetDevice(ctx->device));
        const Params  P  = to_params(params);
        const Plan    pl = make_plan(P, shard);
        std::uint64_t launches = 0;
        ensure_points(ctx, pl.total, false);
        const Tables t = upload_tables(ctx, pl);
        cudaStream_t st  = ctx->stream;
        const auto   H2D = cudaMemcpyHostToDevice;
        // scatter the given points into this shard's extended layout (one slice per stream job)
        for (const StreamJob& J: pl.jobs) {
            const std::uint64_t id = pl.L.chunk_id_base(J.annulus, J.chunk);
            const std::uint64_t d = J.out_off, n = J.count;
            CK(cudaMemcpyAsync(ctx->beta.as<double>() + d, pts->beta + id, n * 8, H2D, st));
            CK(cudaMemcpyAsync(ctx->hw.as<double>() + d, pts->half_width + id, n * 8, H2D, st));
            char* r0 = reinterpret_cast<char*>(ctx->rec0.as<double2>() + d);
            char* r1 = reinterpret_cast<char*>(ctx->rec1.as<double2>() + d);
            char* r2 = reinterpret_cast<char*>(ctx->rec2.as<double2>() + d);
            CK(cudaMemcpy2DAsync(r0 + 8, 16, pts->theta + id, 8, 8, n, H2D, st));
            CK(cudaMemcpy2DAsync(r1, 16, pts->cos_theta + id, 8, 8, n, H2D, st));
            CK(cudaMemcpy2DAsync(r1 + 8, 16, pts->sin_theta + id, 8, 8, n, H2D, st));
            CK(cudaMemcpy2DAsync(r2, 16, pts->coth_r + id, 8, 8, n, H2D, st));
            CK(cudaMemcpy2DAsync(r2 + 8, 16, pts->inv_sinh_r + id, 8, 8, n, H2D, st));
        }
        const double host_ms = std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
        CK(cudaEventRecord(ctx->ev[0], st));
        launch_frames_from_points(sampler_args(ctx, pl, t), st, &launches);
        CK(cudaEventRecord(ctx->ev[1], st));
        run_edges(ctx, pl, t, out, degrees, false, false, &launches, sink);
        fill_common(pl, out);
        out->sample_ms       = ms_between(ctx->ev[0], ctx->ev[1]);
        out->edges_ms        = ms_between(ctx->ev[1], ctx->ev[2]);
        out->device_ms       = ms_between(ctx->ev[0], ctx->ev[2]);
        out->host_ms         = host_ms;
        out->kernel_launches = launches;
        out->seconds         = std::chrono::duration<double>(Clock::now() - t0).count();
    }
}
} // namespace

} // extern "C"
