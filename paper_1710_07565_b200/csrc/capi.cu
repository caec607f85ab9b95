// C ABI (include/rhg_b200.h) and per-call orchestration.
//
// One call = host layout (layout.cpp, the reference's O(annuli*P) binomial
// tree) -> shard plan (extended chunk arrays, stream jobs, pair jobs) -> one
// H2D copy of all tables -> sampler kernels -> cell index -> edge kernels ->
// one D2H copy of the counters.  All device work is on the context's stream,
// timed with CUDA events on that stream.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <cstring>
#include <new>
#include <string>
#include <vector>

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
        p = nullptr;
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

} // namespace

struct rhg_ctx {
    int          device = 0;
    cudaStream_t stream = nullptr, side = nullptr;
    cudaEvent_t  ev[6]{};
    cudaEvent_t  fork = nullptr, join = nullptr; // timing-free events for the side stream
    DevBuf       beta, hw, rec0, rec1, rec2, r_out, beta_raw, tables, cells, counters, degrees, tasks, dbg, nid;
    DevBuf       lcells, perm, s_beta, s_hw, s_rec0, s_rec1, s_rec2, gsort;
    HostPinned   staging;
};

namespace {

// The shard plan: which (annulus, chunk) streams this rank draws, where they
// land in the extended arrays, and the pair-kernel work lists.
struct Plan {
    Layout                  L;
    std::uint32_t           e0 = 0, e1 = 0, T = 0;
    std::vector<AnnulusDev> ann;
    std::vector<StreamJob>  jobs;
    std::vector<PairJob>    sjobs, gjobs;
    std::vector<std::uint64_t> gseg;        // global-point annulus offsets (segments of the theta sort)
    std::vector<std::uint32_t> ann_blk;     // 256-point blocks per streaming annulus (prefix, count + 1)
    std::vector<std::uint64_t> blk_prefix;  // angular-block item order (see edges.cu map_item)
    std::vector<std::uint32_t> blk_job_off;
    int                        nblk = 1;
    std::uint64_t           n_ext = 0, n_glob = 0, total = 0, swarps = 0, gwarps = 0, ncells = 0;
    std::uint64_t           gg_t0 = 0, gg_t1 = 0;
};

Plan make_plan(const Params& P, const rhg_shard* shard) {
    Plan pl;
    pl.L                  = make_layout(P);
    const Layout&       L = pl.L;
    const std::uint32_t W = shard ? shard->world : 1, r = shard ? shard->rank : 0;
    if (W < 1 || r >= W) throw InvalidArgument("rhg_shard: rank must lie in [0, world)");
    const std::uint32_t Pc = L.chunks;
    pl.e0 = std::uint32_t(std::uint64_t(Pc) * r / W);
    pl.e1 = std::uint32_t(std::uint64_t(Pc) * (r + 1) / W);
    pl.T  = pl.e1 - pl.e0;
    pl.ann.resize(L.count);
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
                J.seed_ang = derive_seed3(L.seed, kPhaseAngles, i, c);
                J.seed_rad = derive_seed3(L.seed, kPhaseRadii, i, c);
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
            J.seed_ang = derive_seed3(L.seed, kPhaseAngles, i, c);
            J.seed_rad = derive_seed3(L.seed, kPhaseRadii, i, c);
            J.a = chunk_lower_bound(c, Pc), J.b = chunk_upper_bound(c, Pc);
            pl.jobs.push_back(J);
        }
    pl.total = pl.n_ext + pl.n_glob;
    for (std::uint32_t i = 0; i < L.first_streaming; ++i) pl.gseg.push_back(L.chunk_id_base(i, 0));
    pl.gseg.push_back(pl.n_glob);
    // pair work lists
    for (std::uint32_t a = L.first_streaming; a < L.count; ++a) {
        const std::uint64_t na = pl.ann[a].end - pl.ann[a].off;
        if (!na) continue;
        // one item = 32 requests of annulus a against every target annulus j >= a
        PairJob J{};
        J.warp_begin = pl.swarps, J.req_off = pl.ann[a].off, J.req_end = pl.ann[a].end, J.a = int(a), J.j = -1;
        pl.sjobs.push_back(J);
        pl.swarps += (na + 31) / 32;
    }
    if (pl.n_glob)
        for (std::uint32_t s = L.first_streaming; s < L.count; ++s) {
            if (pl.ann[s].halo == pl.ann[s].off) continue;
            PairJob J{};
            J.warp_begin = pl.gwarps, J.req_off = pl.n_ext, J.req_end = pl.n_ext + pl.n_glob, J.a = -1, J.j = int(s);
            pl.gjobs.push_back(J);
            pl.gwarps += (pl.n_glob + 31) / 32;
        }
    // angular blocks: ~32 MB of node data per block so one block of every annulus stays in L2
    {
        const std::uint64_t bytes = pl.n_ext * 72;
        std::uint64_t       M     = bytes / (32ull << 20);
        M                         = std::max<std::uint64_t>(1, std::min<std::uint64_t>(M, 1024));
        pl.nblk                   = int(M);
        const std::size_t nj      = pl.sjobs.size();
        pl.blk_prefix.assign(M + 1, 0);
        pl.blk_job_off.assign(M * std::max<std::size_t>(nj, 1), 0);
        std::uint64_t acc = 0;
        for (std::uint64_t b = 0; b < M; ++b) {
            pl.blk_prefix[b] = acc;
            std::uint32_t in = 0;
            for (std::size_t k = 0; k < nj; ++k) {
                const std::uint64_t nb = (pl.sjobs[k].req_end - pl.sjobs[k].req_off + 31) / 32;
                pl.blk_job_off[b * nj + k] = in;
                in += std::uint32_t((b + 1) * nb / M - b * nb / M);
            }
            acc += in;
        }
        pl.blk_prefix[M] = acc;
        if (acc != pl.swarps) throw Invariant("plan: angular block item count mismatch");
    }
    const std::uint64_t nT = (pl.n_glob + kGGTile - 1) / kGGTile, tiles = nT * (nT + 1) / 2;
    pl.gg_t0 = tiles * r / W, pl.gg_t1 = tiles * (r + 1) / W;
    return pl;
}

struct Tables {
    AnnulusDev*    ann;
    StreamJob*     jobs;
    PairJob *      sjobs, *gjobs;
    std::uint64_t* blk_prefix;
    std::uint32_t* blk_job_off;
    std::uint64_t* gseg;
    std::uint32_t* ann_blk;
};

// Pack all tables into one pinned blob and send it with one copy.
Tables upload_tables(rhg_ctx* ctx, const Plan& pl, std::uint64_t* h2d = nullptr) {
    const std::size_t o_ann = 0, o_jobs = align256(o_ann + pl.ann.size() * sizeof(AnnulusDev));
    const std::size_t o_sj = align256(o_jobs + pl.jobs.size() * sizeof(StreamJob));
    const std::size_t o_gj = align256(o_sj + pl.sjobs.size() * sizeof(PairJob));
    const std::size_t o_bp = align256(o_gj + pl.gjobs.size() * sizeof(PairJob));
    const std::size_t o_bj = align256(o_bp + pl.blk_prefix.size() * sizeof(std::uint64_t));
    const std::size_t o_gs = align256(o_bj + pl.blk_job_off.size() * sizeof(std::uint32_t));
    const std::size_t o_ab = align256(o_gs + pl.gseg.size() * sizeof(std::uint64_t));
    const std::size_t bytes = align256(o_ab + pl.ann_blk.size() * sizeof(std::uint32_t)) + 256;
    ctx->staging.ensure(bytes);
    char* h = static_cast<char*>(ctx->staging.p);
    std::memcpy(h + o_ann, pl.ann.data(), pl.ann.size() * sizeof(AnnulusDev));
    std::memcpy(h + o_jobs, pl.jobs.data(), pl.jobs.size() * sizeof(StreamJob));
    std::memcpy(h + o_sj, pl.sjobs.data(), pl.sjobs.size() * sizeof(PairJob));
    std::memcpy(h + o_gj, pl.gjobs.data(), pl.gjobs.size() * sizeof(PairJob));
    std::memcpy(h + o_bp, pl.blk_prefix.data(), pl.blk_prefix.size() * sizeof(std::uint64_t));
    std::memcpy(h + o_bj, pl.blk_job_off.data(), pl.blk_job_off.size() * sizeof(std::uint32_t));
    std::memcpy(h + o_gs, pl.gseg.data(), pl.gseg.size() * sizeof(std::uint64_t));
    std::memcpy(h + o_ab, pl.ann_blk.data(), pl.ann_blk.size() * sizeof(std::uint32_t));
    ctx->tables.ensure(bytes);
    CK(cudaMemcpyAsync(ctx->tables.p, h, bytes, cudaMemcpyHostToDevice, ctx->stream));
    if (h2d) *h2d += bytes;
    char* d = ctx->tables.as<char>();
    return {reinterpret_cast<AnnulusDev*>(d + o_ann), reinterpret_cast<StreamJob*>(d + o_jobs),
            reinterpret_cast<PairJob*>(d + o_sj), reinterpret_cast<PairJob*>(d + o_gj),
            reinterpret_cast<std::uint64_t*>(d + o_bp), reinterpret_cast<std::uint32_t*>(d + o_bj),
            reinterpret_cast<std::uint64_t*>(d + o_gs), reinterpret_cast<std::uint32_t*>(d + o_ab)};
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
    s.jobs = t.jobs, s.njobs = int(pl.jobs.size()), s.ann = t.ann, s.alpha = pl.L.alpha, s.total = pl.total;
    s.beta = ctx->beta.as<double>(), s.hw = ctx->hw.as<double>();
    s.rec0 = ctx->rec0.as<double2>(), s.rec1 = ctx->rec1.as<double2>(), s.rec2 = ctx->rec2.as<double2>();
    s.side = ctx->side, s.ev_fork = ctx->fork, s.ev_join = ctx->join;
    return s;
}

// Cell index + every edge kernel + counters back to the host.
void run_edges(rhg_ctx* ctx, const Plan& pl, const Tables& t, rhg_run_stats* out, std::uint32_t* degrees,
               std::uint64_t* launches) {
    const std::size_t cnt_bytes = align256(3 * sizeof(Counters)) + align256(pl.L.count * sizeof(unsigned long long)) +
                                  256;
    ctx->counters.ensure(cnt_bytes);
    CK(cudaMemsetAsync(ctx->counters.p, 0, cnt_bytes, ctx->stream));
    ctx->cells.ensure(std::max<std::uint64_t>(pl.ncells, 1) * sizeof(std::uint64_t));
    if (degrees) {
        ctx->degrees.ensure(pl.L.n * sizeof(unsigned));
        CK(cudaMemsetAsync(ctx->degrees.p, 0, pl.L.n * sizeof(unsigned), ctx->stream));
    }
    EdgeArgs e;
    e.ann = t.ann, e.count = int(pl.L.count), e.first_streaming = int(pl.L.first_streaming);
    e.n_ext = pl.n_ext, e.n_glob = pl.n_glob;
    e.beta = ctx->beta.as<double>(), e.hw = ctx->hw.as<double>();
    e.rec0 = ctx->rec0.as<double2>(), e.rec1 = ctx->rec1.as<double2>(), e.rec2 = ctx->rec2.as<double2>();
    e.cellstart = ctx->cells.as<std::uint64_t>();
    ctx->lcells.ensure(std::max<std::uint64_t>(pl.ncells, 1) * sizeof(std::uint64_t));
    e.lcellstart = ctx->lcells.as<std::uint64_t>();
    {
        const std::size_t ne = pl.n_ext + 2;
        ctx->perm.ensure(ne * sizeof(std::uint64_t));
        ctx->s_beta.ensure(ne * sizeof(double));
        ctx->s_hw.ensure(ne * sizeof(double));
        ctx->s_rec0.ensure(ne * sizeof(double2));
        ctx->s_rec1.ensure(ne * sizeof(double2));
        ctx->s_rec2.ensure(ne * sizeof(double2));
        ctx->nid.ensure(ne * sizeof(unsigned long long));
        e.perm = ctx->perm.as<std::uint64_t>(), e.s_beta = ctx->s_beta.as<double>(), e.s_hw = ctx->s_hw.as<double>();
        e.s_rec0 = ctx->s_rec0.as<double2>(), e.s_rec1 = ctx->s_rec1.as<double2>(), e.s_rec2 = ctx->s_rec2.as<double2>();
        e.s_id = ctx->nid.as<unsigned long long>();
    }
    e.ann_rw = t.ann;
    e.ctr       = ctx->counters.as<Counters>();
    e.dmax_bits = reinterpret_cast<unsigned long long*>(ctx->counters.as<char>() + align256(3 * sizeof(Counters)));
    e.task_ctr  = reinterpret_cast<unsigned long long*>(ctx->counters.as<char>() + cnt_bytes - 256);
    e.task_cap  = std::uint64_t(1) << 21; // 64 MiB of deferred dense tiles; overflow runs inline
    ctx->tasks.ensure(e.task_cap * sizeof(TileTask));
    e.tasks = ctx->tasks.as<TileTask>();
    e.cosh_R = pl.L.cosh_R, e.chunk0_upper = chunk_upper_bound(0, pl.L.chunks);
    e.lift_part   = pl.e1 == pl.L.chunks && pl.T > 0;
    e.stream_jobs = t.sjobs, e.n_stream_jobs = int(pl.sjobs.size()), e.stream_warps = pl.swarps;
    e.blk_prefix = t.blk_prefix, e.blk_job_off = t.blk_job_off, e.nblk = pl.nblk;
    e.ev_pairs0 = ctx->ev[4], e.ev_pairs1 = ctx->ev[5];
    e.glob_jobs = t.gjobs, e.n_glob_jobs = int(pl.gjobs.size()), e.glob_warps = pl.gwarps;
    e.gg_tile_begin = pl.gg_t0, e.gg_tile_end = pl.gg_t1;
    e.degrees       = degrees ? ctx->degrees.as<unsigned>() : nullptr;
    const char* dbg_env = std::getenv("RHG_DEBUG_STATS");
    const bool  dbg     = dbg_env && dbg_env[0] == '1';
    if (dbg) {
        ctx->dbg.ensure(kDbgSlots * sizeof(unsigned long long));
        CK(cudaMemsetAsync(ctx->dbg.p, 0, kDbgSlots * sizeof(unsigned long long), ctx->stream));
        e.dbg = ctx->dbg.as<unsigned long long>();
    }
    e.ann_blk = t.ann_blk;
    launch_cell_index(e, pl.ann_blk[pl.L.count], ctx->stream, launches);
    if (pl.n_glob && pl.gwarps) { // global requests in (annulus, theta) order
        std::size_t need = 0;
        launch_sort_globals(e, t.gseg, int(pl.gseg.size() - 1), nullptr, 0, &need, ctx->stream, launches);
        ctx->gsort.ensure(need);
        launch_sort_globals(e, t.gseg, int(pl.gseg.size() - 1), ctx->gsort.p, ctx->gsort.cap, &need, ctx->stream,
                            launches);
    }
    launch_edges(e, ctx->stream, launches);
    CK(cudaGetLastError());
    CK(cudaEventRecord(ctx->ev[2], ctx->stream));
    ctx->staging.ensure(4096);
    auto* hc = static_cast<Counters*>(ctx->staging.p);
    CK(cudaMemcpyAsync(hc, ctx->counters.p, 3 * sizeof(Counters), cudaMemcpyDeviceToHost, ctx->stream));
    if (degrees)
        CK(cudaMemcpyAsync(degrees, ctx->degrees.p, pl.L.n * sizeof(unsigned), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (dbg) {
        unsigned long long h[kDbgSlots];
        CK(cudaMemcpy(h, ctx->dbg.p, sizeof h, cudaMemcpyDeviceToHost));
        std::fprintf(stderr, "RHG_DEBUG_STATS {\"groups\": [%llu,%llu,%llu,%llu,%llu,%llu], \"sumU\": [%llu,%llu,%llu,%llu,%llu,%llu], "
                             "\"slots\": [%llu,%llu,%llu,%llu,%llu,%llu], \"serial_warps\": %llu, \"serial_slots\": %llu, "
                             "\"serial_cands\": %llu, \"tasks\": %llu, \"warps\": %llu, \"cands\": %llu}\n",
                     h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7], h[8], h[9], h[10], h[11], h[12], h[13], h[14], h[15],
                     h[16], h[17], h[18], h[19], h[20], h[21], h[22], h[23]);
    }
    out->edges       = hc[0].edges + hc[1].edges + hc[2].edges;
    out->fingerprint = hc[0].fp + hc[1].fp + hc[2].fp;
    out->comps       = hc[0].comps + hc[1].comps + hc[2].comps;
    out->global_edges = hc[2].edges;
    out->global_comps = hc[2].comps;
    out->pairs_ms     = pl.swarps ? ms_between(ctx->ev[4], ctx->ev[5]) : 0.0;
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
}



Params to_params(const rhg_params* p) {
    if (!p) throw InvalidArgument("rhg: params is null");
    return Params(p->n, p->alpha, p->C, p->seed, p->chunks);
}

using Clock = std::chrono::steady_clock;

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
        CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
        for (auto& e: c->ev) CK(cudaEventCreate(&e));
        CK(cudaEventCreateWithFlags(&c->fork, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->join, cudaEventDisableTiming));
        *out = c;
    });
}

void rhg_destroy(rhg_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    cudaStreamSynchronize(c->side);
    for (DevBuf* b: {&c->beta, &c->hw, &c->rec0, &c->rec1, &c->rec2, &c->r_out, &c->beta_raw, &c->tables, &c->cells,
                     &c->counters, &c->degrees, &c->tasks, &c->dbg, &c->nid, &c->lcells, &c->perm, &c->s_beta,
                     &c->s_hw, &c->s_rec0, &c->s_rec1, &c->s_rec2, &c->gsort})
        b->release();
    if (c->staging.p) cudaFreeHost(c->staging.p);
    for (auto& e: c->ev) cudaEventDestroy(e);
    cudaEventDestroy(c->fork);
    cudaEventDestroy(c->join);
    cudaStreamDestroy(c->side);
    cudaStreamDestroy(c->stream);
    delete c;
}

int rhg_generate_stats(rhg_ctx* ctx, const rhg_params* params, const rhg_shard* shard, rhg_run_stats* out,
                       std::uint32_t* degrees) {
    return guarded([&] {
        if (!ctx || !out) throw InvalidArgument("rhg_generate_stats: null argument");
        const auto t0 = Clock::now();
        std::memset(out, 0, sizeof *out);
        CK(cudaSetDevice(ctx->device));
        const Params  P  = to_params(params);
        const Plan    pl = make_plan(P, shard);
        std::uint64_t launches = 0;
        ensure_points(ctx, pl.total, false);
        const Tables t = upload_tables(ctx, pl, &out->h2d_bytes);
        const double host_ms = std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
        CK(cudaEventRecord(ctx->ev[0], ctx->stream));
        launch_sampler(sampler_args(ctx, pl, t), ctx->stream, &launches);
        CK(cudaEventRecord(ctx->ev[1], ctx->stream));
        run_edges(ctx, pl, t, out, degrees, &launches);
        fill_common(pl, out);
        out->sample_ms       = ms_between(ctx->ev[0], ctx->ev[1]);
        out->edges_ms        = ms_between(ctx->ev[1], ctx->ev[2]);
        out->device_ms       = ms_between(ctx->ev[0], ctx->ev[2]);
        out->host_ms         = host_ms;
        out->kernel_launches = launches;
        out->device_bytes    = ctx->beta.cap + ctx->hw.cap + ctx->rec0.cap + ctx->rec1.cap + ctx->rec2.cap +
                            ctx->r_out.cap + ctx->beta_raw.cap + ctx->tables.cap + ctx->cells.cap + ctx->counters.cap +
                            ctx->degrees.cap + ctx->tasks.cap + ctx->nid.cap + ctx->lcells.cap + ctx->perm.cap +
                            ctx->s_beta.cap + ctx->s_hw.cap + ctx->s_rec0.cap + ctx->s_rec1.cap + ctx->s_rec2.cap;
        out->seconds = std::chrono::duration<double>(Clock::now() - t0).count();
    });
}

int rhg_sample_points(rhg_ctx* ctx, const rhg_params* params, rhg_points* o) {
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

int rhg_count_edges_from_points(rhg_ctx* ctx, const rhg_params* params, const rhg_shard* shard, const rhg_points* pts,
                                rhg_run_stats* out, std::uint32_t* degrees) {
    return guarded([&] {
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
        run_edges(ctx, pl, t, out, degrees, &launches);
        fill_common(pl, out);
        out->sample_ms       = ms_between(ctx->ev[0], ctx->ev[1]);
        out->edges_ms        = ms_between(ctx->ev[1], ctx->ev[2]);
        out->device_ms       = ms_between(ctx->ev[0], ctx->ev[2]);
        out->host_ms         = host_ms;
        out->kernel_launches = launches;
        out->seconds         = std::chrono::duration<double>(Clock::now() - t0).count();
    });
}

} // extern "C"
