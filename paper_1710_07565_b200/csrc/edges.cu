// Edge kernels (sm_100a): every candidate pair the reference's sweep tests
// (sweep.hpp:509-543 match_node, generator.hpp:77-104 run_global_unit),
// evaluated with the reference's exact FP64 predicate and reduced to
// (edges, fingerprint, comps) without materialising a single edge.
//
// The pair set is the pure-function restatement of the sweep documented in
// DESIGN.md §3 (and SURVEY Appendix A): a request p in extended chunk t of
// annulus a tests node q of annulus j >= a iff q's engine-frame angle lambda
// lies in p's window W_j(p) = own [b, b+2hw) (j == a) or [lambda-h_j,
// lambda+h_j) (j > a), q is in chunk t-1, t or t+1 of this shard's extended
// array (halo requests only against the last owned chunk), not q == p, and for
// j == a the request has the smaller (theta, id).  Global points request
// clipped windows (sweep.hpp:404-432) against owned nodes.
//
//   cell_index_kernel    per-annulus cell -> first-index table over beta, the
//                        exact max half-width (candidate superset bound) and the
//                        node-id array (vertex id | halo bit) the tiles stage
//   stream_pairs_kernel  streaming requests: one warp per 32 requests x target
//                        annulus, processed as an adaptive R x C register tile
//                        (see process_warp) or thread-serially when sparse
//   glob_req_kernel      global requests x owned streaming nodes (same engine)
//   tile_tasks_kernel    deferred pieces of very large tiles, load-balanced
//   glob_pairs_kernel    global unit, 128x128 tiles of the upper triangle
#include "device.cuh"
#include "kernels.hpp"

namespace rhgb {

namespace {

constexpr unsigned kFull  = 0xffffffffu;

struct Acc {
    unsigned long long edges = 0, fp = 0, comps = 0;
};

__device__ __forceinline__ void flush(Acc& acc, Counters* c, int lane) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        acc.edges += __shfl_down_sync(kFull, acc.edges, o);
        acc.fp += __shfl_down_sync(kFull, acc.fp, o);
        acc.comps += __shfl_down_sync(kFull, acc.comps, o);
    }
    if (lane == 0 && (acc.comps | acc.edges)) {
        atomicAdd(&c->edges, acc.edges);
        atomicAdd(&c->fp, acc.fp);
        atomicAdd(&c->comps, acc.comps);
    }
}

__device__ __forceinline__ std::uint32_t cellf(const AnnulusDev& A, double x) {
    const double t = fmul(fsub(x, A.cell_origin), A.cell_inv_w);
    if (!(t > 0.0)) return 0;
    if (t >= double(A.ncells)) return A.ncells - 1;
    return std::uint32_t(t);
}

__device__ __forceinline__ int streaming_annulus_of(const AnnulusDev* __restrict__ ann, int fs, int count,
                                                    std::uint64_t i) {
    int lo = fs, hi = count - 1; // last streaming annulus with off <= i
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (ann[mid].off <= i) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

__global__ void cell_index_kernel(EdgeArgs A) {
    const std::uint64_t i = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int           lane = threadIdx.x & 31;
    // empty streaming annuli: their 1-cell table is [off, off]
    if (i < std::uint64_t(A.count) && int(i) >= A.first_streaming) {
        const AnnulusDev& E = A.ann[i];
        if (E.end == E.off)
            for (std::uint32_t k = 0; k <= E.ncells; ++k) A.cellstart[E.cell_off + k] = E.off;
    }
    unsigned long long hwbits = 0;
    int                j      = -1;
    if (i < A.n_ext) {
        j                   = streaming_annulus_of(A.ann, A.first_streaming, A.count, i);
        const AnnulusDev& J = A.ann[j];
        const double      b = A.beta[i];
        const std::uint32_t k  = cellf(J, b);
        const std::int64_t  kp = i > J.off ? std::int64_t(cellf(J, A.beta[i - 1])) : -1;
        for (std::int64_t c = kp + 1; c <= std::int64_t(k); ++c) A.cellstart[J.cell_off + c] = i;
        if (i + 1 == J.end)
            for (std::uint32_t c = k + 1; c <= J.ncells; ++c) A.cellstart[J.cell_off + c] = J.end;
        hwbits = static_cast<unsigned long long>(__double_as_longlong(A.hw[i])); // hw >= +0
        A.nid[i] = i < J.halo ? (i + static_cast<unsigned long long>(J.dlt0))
                              : ((i + static_cast<unsigned long long>(J.dlt1)) | (1ull << 63));
    }
    // warp max per annulus (lanes of one warp almost always share it)
    const int  j0   = __shfl_sync(kFull, j, 0);
    const bool same = __all_sync(kFull, j == j0);
    if (same) {
        unsigned long long m = hwbits;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long t = __shfl_down_sync(kFull, m, o);
            m = t > m ? t : m;
        }
        if (lane == 0 && j0 >= 0) atomicMax(&A.dmax_bits[j0], m);
    } else if (j >= 0) {
        atomicMax(&A.dmax_bits[j], hwbits);
    }
}

struct Req {
    double             cs, sn, coth, rci; // rci = fl(cosh(R) * inv_sinh_r), hoisted (sweep.hpp:532 order)
    unsigned long long tkey, id;
};

// One request against one target annulus: its window as order-preserving
// keys, its candidate superset [c0, c1) over the beta-sorted nodes, and
// hmask = bit 63 for halo requests (they must not test halo nodes).
struct Lane {
    Req                q;
    unsigned long long lo, hi, hmask;
    std::uint64_t      c0, c1;
};

constexpr unsigned long long kHaloBit = 1ull << 63;

// Candidate index range [c0, c1) over the beta-sorted nodes of annulus J that
// can hold lambda in [lo, hi): lambda = fl(beta + hw) in [beta, beta + dmax].
__device__ __forceinline__ void cand_range(const EdgeArgs& A, const AnnulusDev& J, double dmax, double lo, double hi,
                                           std::uint64_t& c0, std::uint64_t& c1) {
    if (!(hi > lo)) {
        c0 = c1 = 0;
        return;
    }
    const double        x0 = fsub(fsub(lo, dmax), 1e-12);
    const std::uint32_t k0 = cellf(J, x0), k1 = cellf(J, hi);
    c0                     = A.cellstart[J.cell_off + k0];
    c1                     = A.cellstart[J.cell_off + k1 + 1];
}

__device__ __forceinline__ double dmax_of(const EdgeArgs& A, int j) {
    return __longlong_as_double(static_cast<long long>(A.dmax_bits[j]));
}

// Streaming request p of annulus Jb.a against annulus Jb.j (sweep.hpp:455-461, 478-479).
__device__ __forceinline__ void setup_stream(const EdgeArgs& A, const PairJob& Jb, std::uint64_t p, Lane& L) {
    L = Lane{};
    if (p >= Jb.req_end) return;
    const AnnulusDev& Aa = A.ann[Jb.a];
    const AnnulusDev& Aj = A.ann[Jb.j];
    const double  b  = A.beta[p];
    const double  hw = A.hw[p];
    const double2 r0 = A.rec0[p], r1 = A.rec1[p], r2 = A.rec2[p];
    L.q.cs = r1.x, L.q.sn = r1.y, L.q.coth = r2.x, L.q.rci = fmul(A.cosh_R, r2.y);
    L.q.tkey        = nonneg_key(r0.y);
    const bool halo = p >= Aa.halo;
    L.q.id          = p + static_cast<unsigned long long>(halo ? Aa.dlt1 : Aa.dlt0);
    L.hmask         = halo ? kHaloBit : 0ull;
    double lo, hi;
    if (Jb.j == Jb.a) { // own window [b, b + 2hw)
        lo = b;
        hi = fadd(b, fmul(2.0, hw));
    } else { // propagated window [lambda - h_j, lambda + h_j)
        const double h = half_width_in(Aj, r2.x, r2.y);
        lo             = fsub(r0.x, h);
        hi             = fadd(r0.x, h);
    }
    L.lo = nonneg_key(lo), L.hi = nonneg_key(hi);
    cand_range(A, Aj, dmax_of(A, Jb.j), lo, hi, L.c0, L.c1);
    if (halo && L.c1 > Aj.halo) L.c1 = Aj.halo; // no Foreign x Foreign
    if (L.c1 < L.c0) L.c1 = L.c0;
}

// Global request g against streaming annulus Jb.j, window number w (0..3):
// split_wraparound pieces (sweep.hpp:41-58) and, when this shard owns engine
// P-1, their chunk-0 parts lifted by 2pi (sweep.hpp:404-432).  Owned nodes only.
__device__ __forceinline__ void setup_global(const EdgeArgs& A, const PairJob& Jb, std::uint64_t g, int w, Lane& L) {
    L = Lane{};
    if (g >= Jb.req_end) return;
    const AnnulusDev& Aj = A.ann[Jb.j];
    const double2     r0 = A.rec0[g], r1 = A.rec1[g], r2 = A.rec2[g];
    const double      th = r0.y;
    const double      h  = half_width_in(Aj, r2.x, r2.y); // generator.hpp:67
    const double      a = fsub(th, h), b = fadd(th, h);
    double            pa[2], pb[2];
    int               np = 1;
    if (fsub(b, a) >= kTwoPiD) {
        pa[0] = 0.0, pb[0] = kTwoPiD;
    } else if (a < 0.0) {
        pa[0] = fadd(a, kTwoPiD), pb[0] = kTwoPiD, pa[1] = 0.0, pb[1] = b, np = 2;
    } else if (b > kTwoPiD) {
        pa[0] = a, pb[0] = kTwoPiD, pa[1] = 0.0, pb[1] = fsub(b, kTwoPiD), np = 2;
    } else {
        pa[0] = a, pb[0] = b;
    }
    double lo = 0.0, hi = 0.0;
    int    nw = 0;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        if (k >= np) break;
        if (nw == w) lo = pa[k], hi = pb[k];
        ++nw;
        if (A.lift_part) {
            const double l2 = pa[k] < 0.0 ? 0.0 : pa[k];                      // max(begin, w0 = 0)
            const double h2 = A.chunk0_upper < pb[k] ? A.chunk0_upper : pb[k]; // min(end, w1)
            if (l2 < h2) {
                if (nw == w) lo = fadd(l2, kTwoPiD), hi = fadd(h2, kTwoPiD);
                ++nw;
            }
        }
    }
    if (w >= nw) return;
    L.q.cs = r1.x, L.q.sn = r1.y, L.q.coth = r2.x, L.q.rci = fmul(A.cosh_R, r2.y);
    L.q.id = g - A.n_ext;
    L.lo = nonneg_key(lo), L.hi = nonneg_key(hi);
    cand_range(A, Aj, dmax_of(A, Jb.j), lo, hi, L.c0, L.c1);
    if (L.c1 > Aj.halo) L.c1 = Aj.halo;
    if (L.c1 < L.c0) L.c1 = L.c0;
}

// The exact test of one (request, node) pair: window membership, the
// Foreign x Foreign / self / same-annulus dedup filters (sweep.hpp:515-527),
// then the predicate in the reference's rounding order:
//   lhs = fl(fl(c_r c_n) + fl(s_r s_n)),  rhs = fl(fl(k_r k_n) - fl(fl(coshR i_r) i_n)),  edge iff lhs > rhs.
template <bool DEG, bool SAME>
__device__ __forceinline__ void test_pair(const EdgeArgs& A, const Lane& L, double2 n0, double2 n1, double2 n2,
                                          unsigned long long nidf, Acc& acc) {
    const unsigned long long lam = static_cast<unsigned long long>(__double_as_longlong(n0.x));
    const unsigned long long nid = nidf & ~kHaloBit;
    bool in = lam >= L.lo && lam < L.hi && !(nidf & L.hmask);
    if (SAME) {
        const unsigned long long tk = nonneg_key(n0.y);
        in = in && nid != L.q.id && !(L.q.tkey > tk || (L.q.tkey == tk && L.q.id > nid));
    }
    const double lhs = fadd(fmul(L.q.cs, n1.x), fmul(L.q.sn, n1.y));
    const double rhs = fsub(fmul(L.q.coth, n2.x), fmul(L.q.rci, n2.y));
    acc.comps += in;
    if (in && lhs > rhs) {
        ++acc.edges;
        acc.fp += L.q.id + nid;
        if (DEG) {
            atomicAdd(&A.degrees[L.q.id], 1u);
            atomicAdd(&A.degrees[nid], 1u);
        }
    }
}

// ---------------------------------------------------------------- tiles ---
// Per-warp shared memory: a kStages-deep ring of kBatch-node batches filled
// by TMA bulk copies (cp.async.bulk, completion on an mbarrier), SoA so that
// lanes reading consecutive nodes are conflict-free and a whole-warp read of
// one node is a broadcast.
constexpr int kBatch  = 64;
constexpr int kStages = 3;

struct Stage {
    double2            r0[kBatch], r1[kBatch], r2[kBatch];
    unsigned long long nid[kBatch + 2]; // copied from an even index: node t is nid[t + (base & 1)]
};
struct WarpSmem {
    Stage              st[kStages];
    unsigned long long bar[kStages];
    int                meta_g[kStages];
    int                meta_cnt[kStages];
    std::uint64_t      meta_base[kStages];
};
constexpr int kWarpsPerBlock = 8;
constexpr int kTileSmem      = kWarpsPerBlock * int(sizeof(WarpSmem));

__device__ __forceinline__ std::uint32_t smem_u32(const void* p) {
    return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, std::uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, std::uint32_t bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, std::uint32_t parity) {
    std::uint32_t done = 0;
    while (!done) {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(done)
                     : "r"(smem_u32(bar)), "r"(parity)
                     : "memory");
    }
}

__device__ __forceinline__ void warp_smem_init(WarpSmem* ws, int lane) {
    if (lane == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&ws->bar[s]);
        fence_mbar_init();
    }
    __syncwarp();
}

// Lane 0 queues one batch [base, base+cnt) of annulus-array nodes into stage
// s.  The 8-byte node ids are copied from the even index below base (bulk
// copies need 16 B alignment and size); the 16-byte records need nothing.
__device__ __forceinline__ void issue_batch(const EdgeArgs& A, WarpSmem* ws, int s, int g, std::uint64_t base,
                                            int cnt) {
    const std::uint32_t b16  = std::uint32_t(cnt) * 16u;
    const std::uint64_t nb   = base & ~1ull;
    const std::uint32_t bid  = std::uint32_t(((base + cnt + 1) & ~1ull) - nb) * 8u;
    ws->meta_g[s] = g, ws->meta_cnt[s] = cnt, ws->meta_base[s] = base;
    mbar_expect_tx(&ws->bar[s], 3 * b16 + bid);
    bulk_g2s(ws->st[s].r0, A.rec0 + base, b16, &ws->bar[s]);
    bulk_g2s(ws->st[s].r1, A.rec1 + base, b16, &ws->bar[s]);
    bulk_g2s(ws->st[s].r2, A.rec2 + base, b16, &ws->bar[s]);
    bulk_g2s(ws->st[s].nid, A.nid + nb, bid, &ws->bar[s]);
}

__device__ __forceinline__ Lane shfl_lane(const Lane& L, int src) {
    Lane o;
    o.q.cs   = __shfl_sync(kFull, L.q.cs, src);
    o.q.sn   = __shfl_sync(kFull, L.q.sn, src);
    o.q.coth = __shfl_sync(kFull, L.q.coth, src);
    o.q.rci  = __shfl_sync(kFull, L.q.rci, src);
    o.q.tkey = __shfl_sync(kFull, L.q.tkey, src);
    o.q.id   = __shfl_sync(kFull, L.q.id, src);
    o.lo     = __shfl_sync(kFull, L.lo, src);
    o.hi     = __shfl_sync(kFull, L.hi, src);
    o.hmask  = __shfl_sync(kFull, L.hmask, src);
    o.c0     = __shfl_sync(kFull, L.c0, src);
    o.c1     = __shfl_sync(kFull, L.c1, src);
    return o;
}

// Batch cursor over the groups' unions: group g spans [ga_g, gb_g);
// unions live in lanes g*R (ga, gb); empty groups (gb <= ga) are skipped.
struct Cursor {
    int           g;
    std::uint64_t base, end;
};
__device__ __forceinline__ bool cursor_group(Cursor& c, int R, int C, std::uint64_t ga, std::uint64_t gb) {
    for (; c.g < C; ++c.g) {
        const std::uint64_t a = __shfl_sync(kFull, ga, c.g * R), b = __shfl_sync(kFull, gb, c.g * R);
        if (b > a) {
            c.base = a, c.end = b;
            return true;
        }
    }
    return false;
}

// R x C register tile, TMA-pipelined: the warp's C groups of R requests (one
// per lane row, replicated over C = 32/R columns) against the unions of their
// candidate ranges; lane (r, c) tests nodes c, c+C, ... of every batch against
// request r of the current group.  Equivalent to testing each request's own
// [c0, c1): nodes outside it cannot lie in its window.
template <bool DEG, bool SAME, int R>
__device__ __forceinline__ void tile_run(const EdgeArgs& A, const Lane& L, std::uint64_t ga, std::uint64_t gb,
                                         Acc& acc, int lane, WarpSmem* ws, std::uint32_t& phase) {
    constexpr int C   = 32 / R;
    const int     col = lane % C, row = lane / C;
    Cursor        prod{0, 0, 0};
    bool          more = cursor_group(prod, R, C, ga, gb);
    int           s_issue = 0, inflight = 0;
    // prologue: fill the ring
    while (more && inflight < kStages) {
        const int cnt = prod.end - prod.base < kBatch ? int(prod.end - prod.base) : kBatch;
        if (lane == 0) issue_batch(A, ws, s_issue, prod.g, prod.base, cnt);
        prod.base += kBatch;
        if (prod.base >= prod.end) {
            ++prod.g;
            more = cursor_group(prod, R, C, ga, gb);
        }
        s_issue = s_issue + 1 == kStages ? 0 : s_issue + 1;
        ++inflight;
    }
    int  s = 0, cur_g = -1;
    Lane Lr;
    while (inflight) {
        mbar_wait(&ws->bar[s], (phase >> s) & 1u);
        phase ^= 1u << s;
        const int g = ws->meta_g[s], cnt = ws->meta_cnt[s], no = int(ws->meta_base[s] & 1);
        if (g != cur_g) {
            cur_g = g;
            Lr    = shfl_lane(L, g * R + row);
        }
        const Stage& S = ws->st[s];
        if (cnt == kBatch) {
#pragma unroll 4
            for (int i = 0; i < kBatch / C; ++i) {
                const int t = col + C * i;
                test_pair<DEG, SAME>(A, Lr, S.r0[t], S.r1[t], S.r2[t], S.nid[t + no], acc);
            }
        } else {
            for (int t = col; t < cnt; t += C)
                test_pair<DEG, SAME>(A, Lr, S.r0[t], S.r1[t], S.r2[t], S.nid[t + no], acc);
        }
        __syncwarp();
        --inflight;
        if (more) { // refill this stage
            const int c2 = prod.end - prod.base < kBatch ? int(prod.end - prod.base) : kBatch;
            if (lane == 0) issue_batch(A, ws, s, prod.g, prod.base, c2);
            prod.base += kBatch;
            if (prod.base >= prod.end) {
                ++prod.g;
                more = cursor_group(prod, R, C, ga, gb);
            }
            ++inflight;
        }
        s = s + 1 == kStages ? 0 : s + 1;
    }
    __syncwarp();
}

template <bool DEG, bool SAME>
__device__ __forceinline__ void tile_dispatch(int lgR, const EdgeArgs& A, const Lane& L, std::uint64_t ga,
                                              std::uint64_t gb, Acc& acc, int lane, WarpSmem* ws,
                                              std::uint32_t& phase) {
    switch (lgR) {
    case 0: tile_run<DEG, SAME, 1>(A, L, ga, gb, acc, lane, ws, phase); break;
    case 1: tile_run<DEG, SAME, 2>(A, L, ga, gb, acc, lane, ws, phase); break;
    case 2: tile_run<DEG, SAME, 4>(A, L, ga, gb, acc, lane, ws, phase); break;
    case 3: tile_run<DEG, SAME, 8>(A, L, ga, gb, acc, lane, ws, phase); break;
    case 4: tile_run<DEG, SAME, 16>(A, L, ga, gb, acc, lane, ws, phase); break;
    default: tile_run<DEG, SAME, 32>(A, L, ga, gb, acc, lane, ws, phase); break;
    }
}

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
}

constexpr std::uint64_t kTilePiece = 4096;   // node range of one deferred tile task
constexpr std::uint64_t kDeferCost = 150000; // defer a warp's big groups above this estimated cost

// One warp = 32 requests (one per lane) x one target annulus.  Picks, from
// the lanes' candidate ranges, the cheapest of: thread-serial (each lane its
// own list; sparse warps) or an R x C tile for R in {1..32} (cost model in
// issue cycles: ~22 per 32 pair slots, ~12 per staged batch, ~40 per group).
// Groups of very expensive warps are cut into tile tasks (balanced later).
template <bool DEG, bool SAME>
__device__ __forceinline__ void process_warp(const EdgeArgs& A, const AnnulusDev& J, const Lane& L, int kind, int job,
                                             std::uint64_t p0, int w, Acc& acc, int lane, WarpSmem* ws,
                                             std::uint32_t& phase) {
    const std::uint64_t len = L.c1 - L.c0;
    std::uint64_t       mx  = len;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const std::uint64_t t = __shfl_xor_sync(kFull, mx, o);
        mx                    = t > mx ? t : mx;
    }
    if (mx == 0) return;
    std::uint64_t gmin = len ? L.c0 : ~0ull, gmax = len ? L.c1 : 0ull;
    std::uint64_t best = mx * 48 + 16; // thread-serial: per-lane loop, latency-exposed loads
    int           lgR  = -1;
    std::uint64_t ga = 0, gb = 0; // this lane's group union for the chosen R (valid in group leaders)
#pragma unroll
    for (int k = 0; k <= 5; ++k) {
        if (k > 0) {
            const std::uint64_t a = __shfl_xor_sync(kFull, gmin, 1 << (k - 1));
            const std::uint64_t b = __shfl_xor_sync(kFull, gmax, 1 << (k - 1));
            gmin                  = a < gmin ? a : gmin;
            gmax                  = b > gmax ? b : gmax;
        }
        const bool          leader = (lane & ((1 << k) - 1)) == 0;
        const std::uint64_t U      = gmax > gmin ? gmax - gmin : 0;
        const std::uint64_t mine   = leader && U ? (U << k) * 22 / 32 + ((U + kBatch - 1) / kBatch) * 12 + 40 : 0;
        const std::uint64_t cost   = warp_sum_u64(mine);
        if (cost < best) best = cost, lgR = k, ga = gmin, gb = gmax;
    }
    if (A.dbg) {
        const unsigned long long tl = warp_sum_u64(len);
        if (lane == 0) atomicAdd(&A.dbg[22], 1ull), atomicAdd(&A.dbg[23], tl);
        if (lgR < 0 && lane == 0) atomicAdd(&A.dbg[18], 1ull), atomicAdd(&A.dbg[19], 32ull * mx), atomicAdd(&A.dbg[20], tl);
    }
    if (lgR < 0) { // sparse: every lane walks its own few candidates
        for (std::uint64_t k = L.c0; k < L.c1; ++k)
            test_pair<DEG, SAME>(A, L, A.rec0[k], A.rec1[k], A.rec2[k], A.nid[k], acc);
        return;
    }
    const int  R      = 1 << lgR;
    const bool leader = (lane & (R - 1)) == 0;
    if (!leader) ga = gb = 0;
    if (A.dbg && leader && gb > ga) {
        atomicAdd(&A.dbg[lgR], 1ull);
        atomicAdd(&A.dbg[6 + lgR], static_cast<unsigned long long>(gb - ga));
        atomicAdd(&A.dbg[12 + lgR], static_cast<unsigned long long>((gb - ga) << lgR));
    }
    if (best > kDeferCost && A.task_cap) { // cut big groups into balanced tile tasks
        const std::uint64_t npc = leader && gb - ga > kTilePiece ? (gb - (ga & ~1ull) + kTilePiece - 1) / kTilePiece : 0;
        // warp-wide reservation
        std::uint64_t incl = npc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const std::uint64_t t = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += t;
        }
        const std::uint64_t total = __shfl_sync(kFull, incl, 31);
        if (total) {
            unsigned long long t0 = 0;
            if (lane == 0) t0 = atomicAdd(A.task_ctr, static_cast<unsigned long long>(total));
            t0 = __shfl_sync(kFull, t0, 0);
            if (t0 + total <= A.task_cap) {
                if (lane == 0) {
                    atomicMax(A.task_ctr + 1, static_cast<unsigned long long>(t0 + total)); // valid prefix
                    if (A.dbg) atomicAdd(&A.dbg[21], static_cast<unsigned long long>(total));
                }
                const std::uint64_t first = t0 + incl - npc;
                const std::uint64_t a0    = ga & ~1ull; // even piece starts: the TMA base rounding stays inside a piece
                for (std::uint64_t i = 0; i < npc; ++i) {
                    TileTask& T = A.tasks[first + i];
                    T.p0 = p0 + std::uint64_t(lane), T.u0 = i ? a0 + i * kTilePiece : ga;
                    T.u1 = a0 + (i + 1) * kTilePiece < gb ? a0 + (i + 1) * kTilePiece : gb;
                    T.job = job, T.kind = std::int16_t(kind), T.lgR = std::int16_t(lgR), T.w = w;
                }
                if (npc) gb = ga; // handed off
            }
        }
    }
    tile_dispatch<DEG, SAME>(lgR, A, L, ga, gb, acc, lane, ws, phase);
}

__device__ __forceinline__ int find_pair_job(const PairJob* __restrict__ jobs, int n, std::uint64_t gw) {
    int lo = 0, hi = n - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (jobs[mid].warp_begin <= gw) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

__device__ __forceinline__ WarpSmem* my_warp_smem() {
    extern __shared__ __align__(128) unsigned char dyn_smem[];
    return reinterpret_cast<WarpSmem*>(dyn_smem) + (threadIdx.x >> 5);
}

template <bool DEG>
__global__ void __launch_bounds__(256, 2) stream_pairs_kernel(EdgeArgs A) {
    const int           lane = threadIdx.x & 31;
    const std::uint64_t gw   = (std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (gw >= A.stream_warps) return;
    WarpSmem* ws = my_warp_smem();
    warp_smem_init(ws, lane);
    std::uint32_t       phase = 0;
    const int           job = find_pair_job(A.stream_jobs, A.n_stream_jobs, gw);
    const PairJob       Jb  = A.stream_jobs[job];
    const std::uint64_t p0  = Jb.req_off + (gw - Jb.warp_begin) * 32;
    Lane                L;
    setup_stream(A, Jb, p0 + lane, L);
    Acc acc;
    const AnnulusDev& J = A.ann[Jb.j];
    if (Jb.j == Jb.a) process_warp<DEG, true>(A, J, L, 0, job, p0, 0, acc, lane, ws, phase);
    else process_warp<DEG, false>(A, J, L, 0, job, p0, 0, acc, lane, ws, phase);
    flush(acc, &A.ctr[0], lane);
}

template <bool DEG>
__global__ void __launch_bounds__(256, 2) glob_req_kernel(EdgeArgs A) {
    const int           lane = threadIdx.x & 31;
    const std::uint64_t gw   = (std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (gw >= A.glob_warps) return;
    WarpSmem* ws = my_warp_smem();
    warp_smem_init(ws, lane);
    std::uint32_t       phase = 0;
    const int           job = find_pair_job(A.glob_jobs, A.n_glob_jobs, gw);
    const PairJob       Jb  = A.glob_jobs[job];
    const std::uint64_t g0  = Jb.req_off + (gw - Jb.warp_begin) * 32;
    const AnnulusDev&   J   = A.ann[Jb.j];
    Acc                 acc;
#pragma unroll 1
    for (int w = 0; w < 4; ++w) {
        Lane L;
        setup_global(A, Jb, g0 + lane, w, L);
        process_warp<DEG, false>(A, J, L, 1, job, g0, w, acc, lane, ws, phase);
    }
    flush(acc, &A.ctr[1], lane);
}

// Deferred tile pieces: the R requests of one group x kTilePiece nodes
// (KIND 0 streaming requests, 1 global requests).
template <bool DEG, int KIND>
__global__ void __launch_bounds__(256, 2) tile_tasks_kernel(EdgeArgs A) {
    const int           lane  = threadIdx.x & 31;
    const std::uint64_t ntask = A.task_ctr[1]; // reservations that fit (later ones ran inline)
    const std::uint64_t nw    = (std::uint64_t(gridDim.x) * blockDim.x) >> 5;
    WarpSmem*           ws    = my_warp_smem();
    warp_smem_init(ws, lane);
    std::uint32_t phase = 0;
    Acc           acc;
    for (std::uint64_t t = (std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; t < ntask; t += nw) {
        const TileTask T = A.tasks[t];
        if (T.kind != KIND) continue;
        // lanes 0..R-1 hold the group's requests; lane 0 leads the single group
        const std::uint64_t p  = lane < (1 << T.lgR) ? T.p0 + std::uint64_t(lane) : ~0ull;
        const std::uint64_t ga = lane == 0 ? T.u0 : 0, gb = lane == 0 ? T.u1 : 0;
        Lane                L;
        if (KIND == 0) {
            const PairJob Jb = A.stream_jobs[T.job];
            setup_stream(A, Jb, p, L);
            if (Jb.j == Jb.a) tile_dispatch<DEG, true>(T.lgR, A, L, ga, gb, acc, lane, ws, phase);
            else tile_dispatch<DEG, false>(T.lgR, A, L, ga, gb, acc, lane, ws, phase);
        } else {
            const PairJob Jb = A.glob_jobs[T.job];
            setup_global(A, Jb, p, T.w, L);
            tile_dispatch<DEG, false>(T.lgR, A, L, ga, gb, acc, lane, ws, phase);
        }
    }
    flush(acc, &A.ctr[KIND], lane);
}

// generator.hpp:84-102: all pairs i < k of the global points, request = i.
template <bool DEG>
__global__ void __launch_bounds__(kGGTile) glob_pairs_kernel(EdgeArgs A, std::uint64_t nT) {
    __shared__ double2 s1[kGGTile], s2[kGGTile];
    const std::uint64_t t = A.gg_tile_begin + blockIdx.x;
    // tile t -> (I, J), I <= J, row-major over the upper triangle
    const double  fn = double(nT) + 0.5;
    std::uint64_t I  = std::uint64_t(fn - sqrt(fn * fn - 2.0 * double(t)));
    auto start = [nT](std::uint64_t r) { return r * nT - r * (r - 1) / 2; };
    while (I > 0 && start(I) > t) --I;
    while (start(I + 1) <= t) ++I;
    const std::uint64_t J = I + (t - start(I));
    const std::uint64_t nG = A.n_glob;
    const std::uint64_t col = J * kGGTile + threadIdx.x;
    if (col < nG) {
        s1[threadIdx.x] = A.rec1[A.n_ext + col];
        s2[threadIdx.x] = A.rec2[A.n_ext + col];
    }
    __syncthreads();
    const std::uint64_t i = I * kGGTile + threadIdx.x;
    Acc                 acc;
    if (i < nG) {
        const double2 r1 = A.rec1[A.n_ext + i], r2 = A.rec2[A.n_ext + i];
        const double  rci = fmul(A.cosh_R, r2.y);
        std::uint64_t k0  = J * kGGTile;
        if (k0 <= i) k0 = i + 1;
        const std::uint64_t k1 = (J + 1) * kGGTile < nG ? (J + 1) * kGGTile : nG;
        for (std::uint64_t k = k0; k < k1; ++k) {
            const double2 n1  = s1[k - J * kGGTile], n2 = s2[k - J * kGGTile];
            const double  lhs = fadd(fmul(r1.x, n1.x), fmul(r1.y, n1.y));
            const double  rhs = fsub(fmul(r2.x, n2.x), fmul(rci, n2.y));
            ++acc.comps;
            if (lhs > rhs) {
                ++acc.edges;
                acc.fp += i + k;
                if (DEG) {
                    atomicAdd(&A.degrees[i], 1u);
                    atomicAdd(&A.degrees[k], 1u);
                }
            }
        }
    }
    flush(acc, &A.ctr[2], threadIdx.x & 31);
}

} // namespace

void launch_cell_index(const EdgeArgs& a, std::uint64_t, cudaStream_t st, std::uint64_t* launches) {
    const std::uint64_t n = a.n_ext > std::uint64_t(a.count) ? a.n_ext : std::uint64_t(a.count);
    if (a.first_streaming >= a.count) return;
    cell_index_kernel<<<unsigned((n + 255) / 256), 256, 0, st>>>(a);
    ++*launches;
}

void launch_edges(const EdgeArgs& a, cudaStream_t st, std::uint64_t* launches) {
    const bool deg = a.degrees != nullptr;
    static bool attrs = false;
    if (!attrs) { // > 48 KiB of dynamic shared memory per block
        cudaFuncSetAttribute(stream_pairs_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTileSmem);
        cudaFuncSetAttribute(stream_pairs_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTileSmem);
        cudaFuncSetAttribute(glob_req_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTileSmem);
        cudaFuncSetAttribute(glob_req_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTileSmem);
        cudaFuncSetAttribute(tile_tasks_kernel<true, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTileSmem);
        cudaFuncSetAttribute(tile_tasks_kernel<false, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTileSmem);
        cudaFuncSetAttribute(tile_tasks_kernel<true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTileSmem);
        cudaFuncSetAttribute(tile_tasks_kernel<false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTileSmem);
        attrs = true;
    }
    if (a.stream_warps) {
        const unsigned blocks = unsigned((a.stream_warps + kWarpsPerBlock - 1) / kWarpsPerBlock);
        if (deg) stream_pairs_kernel<true><<<blocks, 32 * kWarpsPerBlock, kTileSmem, st>>>(a);
        else stream_pairs_kernel<false><<<blocks, 32 * kWarpsPerBlock, kTileSmem, st>>>(a);
        ++*launches;
    }
    if (a.glob_warps) {
        const unsigned blocks = unsigned((a.glob_warps + kWarpsPerBlock - 1) / kWarpsPerBlock);
        if (deg) glob_req_kernel<true><<<blocks, 32 * kWarpsPerBlock, kTileSmem, st>>>(a);
        else glob_req_kernel<false><<<blocks, 32 * kWarpsPerBlock, kTileSmem, st>>>(a);
        ++*launches;
    }
    if (a.stream_warps && a.task_cap) {
        if (deg) tile_tasks_kernel<true, 0><<<148 * 2, 32 * kWarpsPerBlock, kTileSmem, st>>>(a);
        else tile_tasks_kernel<false, 0><<<148 * 2, 32 * kWarpsPerBlock, kTileSmem, st>>>(a);
        ++*launches;
    }
    if (a.glob_warps && a.task_cap) {
        if (deg) tile_tasks_kernel<true, 1><<<148 * 2, 32 * kWarpsPerBlock, kTileSmem, st>>>(a);
        else tile_tasks_kernel<false, 1><<<148 * 2, 32 * kWarpsPerBlock, kTileSmem, st>>>(a);
        ++*launches;
    }
    if (a.gg_tile_end > a.gg_tile_begin) {
        const std::uint64_t nT     = (a.n_glob + kGGTile - 1) / kGGTile;
        const unsigned      blocks = unsigned(a.gg_tile_end - a.gg_tile_begin);
        if (deg) glob_pairs_kernel<true><<<blocks, kGGTile, 0, st>>>(a, nT);
        else glob_pairs_kernel<false><<<blocks, kGGTile, 0, st>>>(a, nT);
        ++*launches;
    }
}

} // namespace rhgb
