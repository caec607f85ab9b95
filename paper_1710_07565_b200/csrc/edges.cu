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
//   cell_index_kernel    per-annulus cell -> first-index table over beta, and
//                        the exact max half-width (candidate superset bound)
//   stream_pairs_kernel  streaming requests, one warp per 32 requests x target
//                        annulus; short candidate lists run thread-serial, long
//                        ones warp-cooperative (coalesced 16 B node loads)
//   glob_req_kernel      global requests x owned streaming nodes
//   glob_pairs_kernel    global unit, 128x128 tiles of the upper triangle
#include "device.cuh"
#include "kernels.hpp"

namespace rhgb {

namespace {

constexpr unsigned kFull  = 0xffffffffu;
constexpr int      kShort = 12; // candidate lists up to this length run thread-serial

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

__device__ __forceinline__ Req shfl_req(const Req& q, int src) {
    Req r;
    r.cs   = __shfl_sync(kFull, q.cs, src);
    r.sn   = __shfl_sync(kFull, q.sn, src);
    r.coth = __shfl_sync(kFull, q.coth, src);
    r.rci  = __shfl_sync(kFull, q.rci, src);
    r.tkey = __shfl_sync(kFull, q.tkey, src);
    r.id   = __shfl_sync(kFull, q.id, src);
    return r;
}

// One candidate: exact window membership, self / same-annulus dedup filters
// (sweep.hpp:515-526), then the predicate in the reference's rounding order:
//   lhs = fl(fl(c_r c_n) + fl(s_r s_n)),  rhs = fl(fl(k_r k_n) - fl(fl(coshR i_r) i_n)),  edge iff lhs > rhs.
template <bool DEG, bool SAME>
__device__ __forceinline__ void test_node(const EdgeArgs& A, const AnnulusDev& J, const Req& q,
                                          unsigned long long lo, unsigned long long hi, std::uint64_t k, Acc& acc) {
    const double2            n0  = A.rec0[k];
    const unsigned long long lam = static_cast<unsigned long long>(__double_as_longlong(n0.x));
    if (lam < lo || lam >= hi) return;
    const unsigned long long nid = k + static_cast<unsigned long long>(k < J.halo ? J.dlt0 : J.dlt1);
    if (SAME) {
        if (nid == q.id) return;
        const unsigned long long tk = nonneg_key(n0.y);
        if (q.tkey > tk || (q.tkey == tk && q.id > nid)) return;
    }
    const double2 n1  = A.rec1[k];
    const double2 n2  = A.rec2[k];
    const double  lhs = fadd(fmul(q.cs, n1.x), fmul(q.sn, n1.y));
    const double  rhs = fsub(fmul(q.coth, n2.x), fmul(q.rci, n2.y));
    ++acc.comps;
    if (lhs > rhs) {
        ++acc.edges;
        acc.fp += q.id + nid;
        if (DEG) {
            atomicAdd(&A.degrees[q.id], 1u);
            atomicAdd(&A.degrees[nid], 1u);
        }
    }
}

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

// Hand a very long candidate list to long_pairs_kernel; false if the list
// is full (the caller then processes it inline — capacity never changes results).
__device__ __forceinline__ bool defer_long(const EdgeArgs& A, int j, bool same, const Req& q, unsigned long long lo,
                                           unsigned long long hi, std::uint64_t c0, std::uint64_t c1) {
    const std::uint64_t      nch = (c1 - c0 + kLongChunk - 1) / kLongChunk;
    const unsigned long long old = atomicAdd(A.long_ctr, (1ull << kCtrShift) | nch);
    const std::uint64_t      seg = old >> kCtrShift;
    if (seg >= A.long_cap) return false;
    LongSeg& L = A.long_segs[seg];
    L.cs = q.cs, L.sn = q.sn, L.coth = q.coth, L.rci = q.rci, L.tkey = q.tkey, L.id = q.id, L.lo = lo, L.hi = hi;
    L.c0 = c0, L.c1 = c1, L.chunk_base = old & ((1ull << kCtrShift) - 1), L.j = j, L.same = same;
    return true;
}

template <bool DEG, bool SAME>
__device__ __forceinline__ void run_segment(const EdgeArgs& A, int jidx, const AnnulusDev& J, const Req& q,
                                            unsigned long long lo, unsigned long long hi, std::uint64_t c0,
                                            std::uint64_t c1, Acc& acc, int lane) {
    std::uint64_t len = c1 > c0 ? c1 - c0 : 0;
    if (len > kLongSeg && defer_long(A, jidx, SAME, q, lo, hi, c0, c1)) len = 0;
    const bool lng = len > std::uint64_t(kShort);
    if (!lng)
        for (std::uint64_t k = c0; k < c0 + len; ++k) test_node<DEG, SAME>(A, J, q, lo, hi, k, acc);
    unsigned mask = __ballot_sync(kFull, lng);
    while (mask) {
        const int src = __ffs(mask) - 1;
        mask &= mask - 1;
        const Req                b   = shfl_req(q, src);
        const unsigned long long blo = __shfl_sync(kFull, lo, src), bhi = __shfl_sync(kFull, hi, src);
        const std::uint64_t      b0 = __shfl_sync(kFull, c0, src), b1 = b0 + __shfl_sync(kFull, len, src);
        for (std::uint64_t k = b0 + lane; k < b1; k += 32) test_node<DEG, SAME>(A, J, b, blo, bhi, k, acc);
    }
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

// A streaming request's lane state for one target annulus (sweep.hpp:455-461, 478-479).
struct Lane {
    Req                q;
    unsigned long long lo, hi; // window keys
    std::uint64_t      c0, c1; // candidate superset [c0, c1)
    bool               ok, halo;
};

__device__ __forceinline__ void lane_setup(const EdgeArgs& A, const PairJob& Jb, const AnnulusDev& Aa,
                                           const AnnulusDev& Aj, double dmax, std::uint64_t p, Lane& L) {
    L.ok = p < Jb.req_end;
    L.lo = L.hi = 0;
    L.c0 = L.c1 = 0;
    L.q        = Req{};
    L.halo     = false;
    if (!L.ok) return;
    const double  b  = A.beta[p];
    const double  hw = A.hw[p];
    const double2 r0 = A.rec0[p], r1 = A.rec1[p], r2 = A.rec2[p];
    L.q.cs = r1.x, L.q.sn = r1.y, L.q.coth = r2.x, L.q.rci = fmul(A.cosh_R, r2.y);
    L.q.tkey = nonneg_key(r0.y);
    L.halo   = p >= Aa.halo;
    L.q.id   = p + static_cast<unsigned long long>(L.halo ? Aa.dlt1 : Aa.dlt0);
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
    cand_range(A, Aj, dmax, lo, hi, L.c0, L.c1);
    if (L.halo && L.c1 > Aj.halo) L.c1 = Aj.halo; // halo requests: owned nodes only (no Foreign x Foreign)
    if (L.c1 < L.c0) L.c1 = L.c0;
}

// Warp tile: the 32 lanes' requests stay in registers; the union [u0, u1) of
// their candidate nodes streams through shared memory 32 nodes at a time
// (coalesced 16 B loads, next batch prefetched into registers) and every
// node is broadcast to all lanes.  Equivalent to testing each lane's own
// [c0, c1): nodes outside it cannot lie in its window.
struct NodeSm {
    double2 r0, r1, r2;
};

template <bool DEG, bool SAME>
__device__ __forceinline__ void tile_path(const EdgeArgs& A, const AnnulusDev& J, const Lane& L, std::uint64_t u0,
                                          std::uint64_t u1, Acc& acc, int lane, NodeSm* sm) {
    double2 p0{}, p1{}, p2{};
    if (u0 + lane < u1) p0 = A.rec0[u0 + lane], p1 = A.rec1[u0 + lane], p2 = A.rec2[u0 + lane];
    const unsigned long long dl0 = static_cast<unsigned long long>(J.dlt0), dl1 = static_cast<unsigned long long>(J.dlt1);
    for (std::uint64_t base = u0; base < u1; base += 32) {
        sm[lane].r0 = p0, sm[lane].r1 = p1, sm[lane].r2 = p2;
        __syncwarp();
        const std::uint64_t nk = base + 32 + lane;
        if (nk < u1) p0 = A.rec0[nk], p1 = A.rec1[nk], p2 = A.rec2[nk];
        const int cnt = u1 - base < 32 ? int(u1 - base) : 32;
#pragma unroll 4
        for (int t = 0; t < cnt; ++t) {
            const std::uint64_t      k   = base + t;
            const double2            n0  = sm[t].r0;
            const unsigned long long lam = static_cast<unsigned long long>(__double_as_longlong(n0.x));
            const unsigned long long nid = k + (k < J.halo ? dl0 : dl1);
            bool in = L.ok && lam >= L.lo && lam < L.hi && !(L.halo && k >= J.halo);
            if (SAME) {
                const unsigned long long tk = nonneg_key(n0.y);
                in = in && nid != L.q.id && !(L.q.tkey > tk || (L.q.tkey == tk && L.q.id > nid));
            }
            const double2 n1  = sm[t].r1;
            const double2 n2  = sm[t].r2;
            const double  lhs = fadd(fmul(L.q.cs, n1.x), fmul(L.q.sn, n1.y));
            const double  rhs = fsub(fmul(L.q.coth, n2.x), fmul(L.q.rci, n2.y));
            const bool    e   = in && lhs > rhs;
            acc.comps += in;
            if (e) {
                ++acc.edges;
                acc.fp += L.q.id + nid;
                if (DEG) {
                    atomicAdd(&A.degrees[L.q.id], 1u);
                    atomicAdd(&A.degrees[nid], 1u);
                }
            }
        }
        __syncwarp();
    }
}

__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long t = __shfl_xor_sync(kFull, v, o);
        v                          = t < v ? t : v;
    }
    return v;
}
__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long t = __shfl_xor_sync(kFull, v, o);
        v                          = t > v ? t : v;
    }
    return v;
}
__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
}

constexpr std::uint64_t kTileInline = 4096; // dense unions up to this many nodes run inline
constexpr std::uint64_t kTilePiece  = 2048; // larger unions become kTilePiece-node tile tasks

template <bool DEG, bool SAME>
__device__ __forceinline__ void stream_warp(const EdgeArgs& A, int job, const PairJob& Jb, std::uint64_t p0,
                                            Acc& acc, int lane, NodeSm* sm) {
    const AnnulusDev& Aa   = A.ann[Jb.a];
    const AnnulusDev& Aj   = A.ann[Jb.j];
    const double      dmax = __longlong_as_double(static_cast<long long>(A.dmax_bits[Jb.j]));
    Lane              L;
    lane_setup(A, Jb, Aa, Aj, dmax, p0 + lane, L);
    const std::uint64_t len = L.c1 - L.c0;
    const std::uint64_t u0  = warp_min_u64(len ? L.c0 : ~0ull);
    const std::uint64_t u1  = warp_max_u64(len ? L.c1 : 0ull);
    const std::uint64_t sum = warp_sum_u64(len);
    if (sum == 0) return;
    const std::uint64_t U = u1 - u0;
    // density f = sum / (32 U): the tile pays ~1 broadcast iteration per union
    // node, the per-request path ~1 load-bound iteration per 32 candidates.
    if (sum * 100 >= std::uint64_t(32) * 35 * U) {
        if (U <= kTileInline) {
            tile_path<DEG, SAME>(A, Aj, L, u0, u1, acc, lane, sm);
            return;
        }
        const std::uint64_t npc = (U + kTilePiece - 1) / kTilePiece;
        std::uint64_t       t0  = 0;
        if (lane == 0) t0 = atomicAdd(A.task_ctr, static_cast<unsigned long long>(npc));
        t0 = __shfl_sync(kFull, t0, 0);
        if (t0 + npc <= A.task_cap) {
            if (lane == 0) atomicMax(A.task_ctr + 1, static_cast<unsigned long long>(t0 + npc)); // valid prefix
            for (std::uint64_t i = lane; i < npc; i += 32) {
                TileTask& T = A.tasks[t0 + i];
                T.p0 = p0, T.u0 = u0 + i * kTilePiece, T.u1 = u0 + (i + 1) * kTilePiece < u1 ? u0 + (i + 1) * kTilePiece : u1;
                T.job = job;
            }
            return;
        }
        tile_path<DEG, SAME>(A, Aj, L, u0, u1, acc, lane, sm); // task list full: inline
        return;
    }
    run_segment<DEG, SAME>(A, Jb.j, Aj, L.q, L.lo, L.hi, L.c0, L.c1, acc, lane);
}

template <bool DEG>
__global__ void __launch_bounds__(256) stream_pairs_kernel(EdgeArgs A) {
    __shared__ NodeSm   smem[8][32];
    const int           lane = threadIdx.x & 31;
    const std::uint64_t gw   = (std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (gw >= A.stream_warps) return;
    const int     job = find_pair_job(A.stream_jobs, A.n_stream_jobs, gw);
    const PairJob Jb  = A.stream_jobs[job];
    const std::uint64_t p0 = Jb.req_off + (gw - Jb.warp_begin) * 32;
    Acc acc;
    if (Jb.j == Jb.a) stream_warp<DEG, true>(A, job, Jb, p0, acc, lane, smem[threadIdx.x >> 5]);
    else stream_warp<DEG, false>(A, job, Jb, p0, acc, lane, smem[threadIdx.x >> 5]);
    flush(acc, &A.ctr[0], lane);
}

// Deferred dense tiles: (32 requests, target annulus, kTilePiece nodes).
template <bool DEG>
__global__ void __launch_bounds__(256) tile_tasks_kernel(EdgeArgs A) {
    __shared__ NodeSm   smem[8][32];
    const int           lane = threadIdx.x & 31;
    const std::uint64_t ntask = A.task_ctr[1]; // reservations that fit (later ones ran inline)
    const std::uint64_t nw    = (std::uint64_t(gridDim.x) * blockDim.x) >> 5;
    Acc                 acc;
    for (std::uint64_t t = (std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; t < ntask; t += nw) {
        const TileTask    T  = A.tasks[t];
        const PairJob     Jb = A.stream_jobs[T.job];
        const AnnulusDev& Aa = A.ann[Jb.a];
        const AnnulusDev& Aj = A.ann[Jb.j];
        const double      dmax = __longlong_as_double(static_cast<long long>(A.dmax_bits[Jb.j]));
        Lane              L;
        lane_setup(A, Jb, Aa, Aj, dmax, T.p0 + lane, L);
        if (Jb.j == Jb.a) tile_path<DEG, true>(A, Aj, L, T.u0, T.u1, acc, lane, smem[threadIdx.x >> 5]);
        else tile_path<DEG, false>(A, Aj, L, T.u0, T.u1, acc, lane, smem[threadIdx.x >> 5]);
    }
    flush(acc, &A.ctr[0], lane);
}

template <bool DEG>
__global__ void __launch_bounds__(256) glob_req_kernel(EdgeArgs A) {
    const int           lane = threadIdx.x & 31;
    const std::uint64_t gw   = (std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (gw >= A.glob_warps) return;
    const PairJob     Jb   = A.glob_jobs[find_pair_job(A.glob_jobs, A.n_glob_jobs, gw)];
    const AnnulusDev& Aj   = A.ann[Jb.j];
    const double      dmax = __longlong_as_double(static_cast<long long>(A.dmax_bits[Jb.j]));
    const std::uint64_t g  = Jb.req_off + (gw - Jb.warp_begin) * 32 + lane;
    const bool          ok = g < Jb.req_end;
    Req                 q{};
    double              win[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}}; // 2 pieces x (plain, lifted)
    if (ok) {
        const double2 r0 = A.rec0[g], r1 = A.rec1[g], r2 = A.rec2[g];
        q.cs = r1.x, q.sn = r1.y, q.coth = r2.x, q.rci = fmul(A.cosh_R, r2.y);
        q.id = g - A.n_ext;
        const double th = r0.y;
        const double h  = half_width_in(Aj, r2.x, r2.y); // generator.hpp:67
        // sweep.hpp:41-58 split_wraparound of [theta - h, theta + h)
        const double a = fsub(th, h), b = fadd(th, h);
        double       pc[2][2];
        int          np = 1;
        if (fsub(b, a) >= kTwoPiD) {
            pc[0][0] = 0.0, pc[0][1] = kTwoPiD;
        } else if (a < 0.0) {
            pc[0][0] = fadd(a, kTwoPiD), pc[0][1] = kTwoPiD, pc[1][0] = 0.0, pc[1][1] = b, np = 2;
        } else if (b > kTwoPiD) {
            pc[0][0] = a, pc[0][1] = kTwoPiD, pc[1][0] = 0.0, pc[1][1] = fsub(b, kTwoPiD), np = 2;
        } else {
            pc[0][0] = a, pc[0][1] = b;
        }
        int nw = 0;
        for (int k = 0; k < np; ++k) {
            win[nw][0] = pc[k][0], win[nw][1] = pc[k][1], ++nw;
            if (A.lift_part) { // the part clipped to chunk 0 seen from engine P-1 (sweep.hpp:405-420)
                const double lo = pc[k][0] < 0.0 ? 0.0 : pc[k][0];
                const double hi = A.chunk0_upper < pc[k][1] ? A.chunk0_upper : pc[k][1];
                if (lo < hi) win[nw][0] = fadd(lo, kTwoPiD), win[nw][1] = fadd(hi, kTwoPiD), ++nw;
            }
        }
    }
    Acc acc;
#pragma unroll 1
    for (int w = 0; w < 4; ++w) {
        std::uint64_t c0 = 0, c1 = 0;
        if (ok) {
            cand_range(A, Aj, dmax, win[w][0], win[w][1], c0, c1);
            if (c1 > Aj.halo) c1 = Aj.halo;
        }
        run_segment<DEG, false>(A, Jb.j, Aj, q, nonneg_key(win[w][0]), nonneg_key(win[w][1]), c0, c1, acc, lane);
    }
    flush(acc, &A.ctr[1], lane);
}

// Deferred long candidate lists, kLongChunk nodes per warp task: every warp
// of the grid strides over the chunk space, so one request with 10^6
// candidates is spread over the whole GPU.
template <bool DEG>
__global__ void __launch_bounds__(256) long_pairs_kernel(EdgeArgs A) {
    const int                lane = threadIdx.x & 31;
    const unsigned long long ctr  = *A.long_ctr;
    const std::uint64_t      nseg = (ctr >> kCtrShift) < A.long_cap ? (ctr >> kCtrShift) : A.long_cap;
    Acc                      acc;
    if (nseg) {
        const LongSeg&      last  = A.long_segs[nseg - 1];
        const std::uint64_t total = last.chunk_base + (last.c1 - last.c0 + kLongChunk - 1) / kLongChunk;
        const std::uint64_t nw    = (std::uint64_t(gridDim.x) * blockDim.x) >> 5;
        for (std::uint64_t c = (std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; c < total; c += nw) {
            std::uint64_t lo = 0, hi = nseg - 1; // last segment with chunk_base <= c
            while (lo < hi) {
                const std::uint64_t mid = (lo + hi + 1) >> 1;
                if (A.long_segs[mid].chunk_base <= c) lo = mid;
                else hi = mid - 1;
            }
            const LongSeg&      L  = A.long_segs[lo];
            const AnnulusDev&   J  = A.ann[L.j];
            const std::uint64_t k0 = L.c0 + (c - L.chunk_base) * kLongChunk;
            const std::uint64_t k1 = k0 + kLongChunk < L.c1 ? k0 + kLongChunk : L.c1;
            const Req           q{L.cs, L.sn, L.coth, L.rci, L.tkey, L.id};
            if (L.same)
                for (std::uint64_t k = k0 + lane; k < k1; k += 32) test_node<DEG, true>(A, J, q, L.lo, L.hi, k, acc);
            else
                for (std::uint64_t k = k0 + lane; k < k1; k += 32) test_node<DEG, false>(A, J, q, L.lo, L.hi, k, acc);
        }
    }
    flush(acc, &A.ctr[0], lane);
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
    if (a.stream_warps) {
        const unsigned blocks = unsigned((a.stream_warps + 7) / 8);
        if (deg) stream_pairs_kernel<true><<<blocks, 256, 0, st>>>(a);
        else stream_pairs_kernel<false><<<blocks, 256, 0, st>>>(a);
        ++*launches;
    }
    if (a.glob_warps) {
        const unsigned blocks = unsigned((a.glob_warps + 7) / 8);
        if (deg) glob_req_kernel<true><<<blocks, 256, 0, st>>>(a);
        else glob_req_kernel<false><<<blocks, 256, 0, st>>>(a);
        ++*launches;
    }
    if (a.stream_warps && a.task_cap) {
        if (deg) tile_tasks_kernel<true><<<148 * 8, 256, 0, st>>>(a);
        else tile_tasks_kernel<false><<<148 * 8, 256, 0, st>>>(a);
        ++*launches;
    }
    if ((a.stream_warps || a.glob_warps) && a.long_cap) {
        if (deg) long_pairs_kernel<true><<<148 * 8, 256, 0, st>>>(a);
        else long_pairs_kernel<false><<<148 * 8, 256, 0, st>>>(a);
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
