// Edge kernels (sm_100a): every candidate pair the reference's sweep tests
// (sweep.hpp:509-543 match_node, generator.hpp:77-104 run_global_unit),
// evaluated with the reference's exact FP64 predicate and reduced to
// (edges, fingerprint, comps) without materialising a single edge.
//
// The pair set is the pure-function restatement of the sweep documented in
// a request p of annulus a tests node q of annulus j >= a iff
// q's engine-frame angle lambda lies in p's window W_j(p) (own [b, b+2hw) for
// j == a, [lambda-h_j, lambda+h_j) for j > a), q is reachable from p's chunk
// (halo requests: owned nodes only), q != p, and for j == a (theta_p, id_p) <
// (theta_q, id_q).  Global points request clipped windows (sweep.hpp:404-432)
// against owned nodes.
//
// Layout: each streaming annulus keeps two lambda-sorted blocks, the owned
// chunks [off, halo) and the halo chunk [halo, end).  A window is then an
// EXACT index range, and for ordinary same-annulus pairs (both owned, lambda <
// 2pi, where lambda == theta) the (theta, id) dedup is just "node index >
// request index" — the hot loop has no window or dedup compares at all.
//
//   beta_cells_kernel   beta-cell starts of the beta-ordered sampler output and
//                       the exact per-annulus max half-width
//   rank_kernel         exact rank of every point by (lambda, id) inside its block
//   scatter_kernel      the lambda-sorted arrays (+ node ids)
//   lambda_cells_kernel lambda-cell starts of the owned blocks, first wrapped index
//   stream_pairs_kernel streaming requests: one warp per 32 requests x target
//                       annulus; adaptive R x C register tile over TMA-staged
//                       node batches, a flattened pair list when sparse
//   glob_req_kernel     global requests x owned streaming nodes (same engine)
//   tile_tasks_kernel   deferred pieces of very large tiles, load-balanced
//   glob_pairs_kernel   global unit, 128x128 tiles of the upper triangle
#include <cub/cub.cuh>

#include "device.cuh"
#include "kernels.hpp"

namespace rhgb {

namespace {

constexpr unsigned kFull = 0xffffffffu;

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

// Monotone cell index of an angle (same origin/width for the beta and the
// lambda tables of an annulus).
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

// Sort-phase kernels run ceil(n_j / 256) blocks per streaming annulus j
// (prefix table A.ann_blk), so every block knows its annulus without a search
// per thread.  Returns the annulus of this block and sets i (maybe >= end).
__device__ __forceinline__ int block_annulus(const EdgeArgs& A, std::uint64_t& i) {
    const std::uint32_t b  = blockIdx.x;
    int                 lo = A.first_streaming, hi = A.count - 1; // last annulus with ann_blk <= b
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (A.ann_blk[mid] <= b) lo = mid;
        else hi = mid - 1;
    }
    i = A.ann[lo].off + std::uint64_t(b - A.ann_blk[lo]) * 256u + threadIdx.x;
    return lo;
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

// Fill a cell-start table: entries (kp, k] = i.  The tail after the last
// point, (k_last, ncells] = end, is filled in parallel by cell_tail_kernel.
__device__ __forceinline__ void cell_fill(std::uint64_t* tab, std::int64_t kp, std::uint32_t k, std::uint64_t i) {
    for (std::int64_t c = kp + 1; c <= std::int64_t(k); ++c) tab[c] = i;
}

// ---------------------------------------------------------------- sort ---
__global__ void __launch_bounds__(256) beta_cells_kernel(EdgeArgs A) {
    const int lane = threadIdx.x & 31;
    if (blockIdx.x == 0 && int(threadIdx.x) < A.count && int(threadIdx.x) >= A.first_streaming) {
        const AnnulusDev& E = A.ann[threadIdx.x]; // empty blocks: [off, off]
        if (E.end == E.off)
            for (std::uint32_t k = 0; k <= E.ncells; ++k) A.cellstart[E.cell_off + k] = E.off;
        if (E.halo == E.off)
            for (std::uint32_t k = 0; k <= E.ncells; ++k) A.lcellstart[E.cell_off + k] = E.off;
    }
    std::uint64_t       i;
    const int           j = block_annulus(A, i);
    const AnnulusDev&   J = A.ann[j];
    unsigned long long  hwbits = 0;
    if (i < J.end) {
        const std::uint32_t k  = cellf(J, A.beta[i]);
        const std::int64_t  kp = i > J.off ? std::int64_t(cellf(J, A.beta[i - 1])) : -1;
        cell_fill(A.cellstart + J.cell_off, kp, k, i);
        hwbits = static_cast<unsigned long long>(__double_as_longlong(A.hw[i])); // hw >= +0
    }
    __shared__ unsigned long long wmax[8]; // one atomic per block (all its points share the annulus)
    const unsigned long long m = warp_max_u64(hwbits);
    if (lane == 0) wmax[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long b = 0;
        for (int w = 0; w < int(blockDim.x >> 5); ++w) b = wmax[w] > b ? wmax[w] : b;
        if (b) atomicMax(&A.dmax_bits[j], b);
    }
}

// Exact rank of point i by (lambda, beta-order index) inside its block; in the
// owned block beta-order index order is id order, so the sorted order is
// (lambda, id).  Only points whose beta lies in [lambda_i - dmax, lambda_i]
// can compare either way: everything before that window is smaller
// (lambda <= beta + dmax), everything after is larger (lambda >= beta).
__global__ void __launch_bounds__(256) rank_kernel(EdgeArgs A) {
    std::uint64_t       i;
    const int           j = block_annulus(A, i);
    const AnnulusDev&   J = A.ann[j];
    if (i >= J.end) return;
    const bool          hb = i >= J.halo;
    const std::uint64_t bs = hb ? J.halo : J.off, be = hb ? J.end : J.halo;
    const double        li = A.rec0[i].x;
    const double        dm = __longlong_as_double(static_cast<long long>(A.dmax_bits[j]));
    std::uint64_t       k0 = A.cellstart[J.cell_off + cellf(J, fsub(fsub(li, dm), 1e-12))];
    std::uint64_t       k1 = A.cellstart[J.cell_off + cellf(J, li) + 1];
    k0 = k0 < bs ? bs : k0;
    k1 = k1 > be ? be : k1;
    std::uint64_t rank = k0 - bs;
    for (std::uint64_t k = k0; k < k1; ++k) {
        const double lk = A.rec0[k].x;
        rank += (lk < li) || (lk == li && k < i);
    }
    A.perm[i] = bs + rank;
}

__global__ void __launch_bounds__(256) scatter_kernel(EdgeArgs A) {
    std::uint64_t       i;
    const int           j = block_annulus(A, i);
    const AnnulusDev&   J = A.ann[j];
    if (i >= J.end) return;
    const std::uint64_t d = A.perm[i];
    A.s_beta[d]           = A.beta[i];
    A.s_hw[d]             = A.hw[i];
    A.s_rec0[d]           = A.rec0[i];
    A.s_rec1[d]           = A.rec1[i];
    A.s_rec2[d]           = A.rec2[i];
    A.s_id[d]             = i + static_cast<unsigned long long>(i < J.halo ? J.dlt0 : J.dlt1);
}

// Lambda-cell starts of every owned block, and the first owned index with
// lambda >= 2pi (wrapped points: theta = lambda - 2pi there).
__global__ void __launch_bounds__(256) lambda_cells_kernel(EdgeArgs A) {
    std::uint64_t i;
    const int     j = block_annulus(A, i);
    AnnulusDev&   J = A.ann_rw[j];
    if (i >= J.halo) return;
    const double        l  = A.s_rec0[i].x;
    const std::uint32_t k  = cellf(J, l);
    const std::int64_t  kp = i > J.off ? std::int64_t(cellf(J, A.s_rec0[i - 1].x)) : -1;
    cell_fill(A.lcellstart + J.cell_off, kp, k, i);
    if (l >= kTwoPiD && (i == J.off || A.s_rec0[i - 1].x < kTwoPiD)) J.wrap = i;
}

// Tails of both cell tables: cells after the last point of a block hold the
// block end (beta table: whole annulus array; lambda table: owned block).
__global__ void cell_tail_kernel(EdgeArgs A, int lambda) {
    const int         j  = A.first_streaming + int(blockIdx.y);
    const AnnulusDev& J  = A.ann[j];
    const std::uint64_t e = lambda ? J.halo : J.end;
    if (e == J.off) return; // empty: initialised by beta_cells_kernel
    const double        last = lambda ? A.s_rec0[e - 1].x : A.beta[e - 1];
    const std::uint32_t k0   = cellf(J, last) + 1;
    std::uint64_t*      tab  = (lambda ? A.lcellstart : A.cellstart) + J.cell_off;
    for (std::uint32_t c = k0 + blockIdx.x * blockDim.x + threadIdx.x; c <= J.ncells; c += gridDim.x * blockDim.x)
        tab[c] = e;
}

// ------------------------------------------------------------ requests ---
// First index k in the sorted owned block with lambda[k] >= x (exact).
__device__ __forceinline__ std::uint64_t lower_bound_owned(const EdgeArgs& A, const AnnulusDev& J, double x) {
    const std::uint32_t c = cellf(J, x);
    std::uint64_t       k = A.lcellstart[J.cell_off + c];
    const std::uint64_t e = A.lcellstart[J.cell_off + c + 1];
    while (k < e && A.s_rec0[k].x < x) ++k;
    return k;
}
__device__ __forceinline__ std::uint64_t lower_bound_halo(const EdgeArgs& A, const AnnulusDev& J, double x) {
    std::uint64_t lo = J.halo, hi = J.end; // binary search (one chunk, rarely searched)
    while (lo < hi) {
        const std::uint64_t mid = (lo + hi) >> 1;
        if (A.s_rec0[mid].x < x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

struct Req {
    double             cs, sn, coth, rci; // rci = fl(cosh(R) * inv_sinh_r), hoisted (sweep.hpp:532 order)
    unsigned long long id;
    double             theta;
};

// One request against one target annulus: the simple index range handled by
// the tile engine, the halo-block range and the "general" range of pairs that
// need the full (theta, id) dedup (same-annulus pairs with wrapped or halo points).
struct Lane {
    Req           q;
    std::uint64_t s0, s1; // simple owned range
    std::uint64_t h0, h1; // halo-block range (simple when j != a, general when j == a)
    std::uint64_t g0, g1; // general owned range (j == a only)
};

__device__ __forceinline__ void window_ranges(const EdgeArgs& A, const AnnulusDev& J, double lo, double hi,
                                              bool want_halo, Lane& L) {
    if (!(hi > lo)) return;
    { // both lower bounds interleaved: independent loads in flight together
        const std::uint32_t ca = cellf(J, lo), cb = cellf(J, hi);
        std::uint64_t       ka = A.lcellstart[J.cell_off + ca], kb = A.lcellstart[J.cell_off + cb];
        const std::uint64_t ea = A.lcellstart[J.cell_off + ca + 1], eb = A.lcellstart[J.cell_off + cb + 1];
        bool                ma = ka < ea, mb = kb < eb;
        while (ma || mb) {
            const double xa = ma ? A.s_rec0[ka].x : 0.0, xb = mb ? A.s_rec0[kb].x : 0.0;
            if (ma) {
                if (xa < lo) ma = ++ka < ea;
                else ma = false;
            }
            if (mb) {
                if (xb < hi) mb = ++kb < eb;
                else mb = false;
            }
        }
        L.s0 = ka, L.s1 = kb;
    }
    if (want_halo && J.end > J.halo && hi > A.s_rec0[J.halo].x && lo <= A.s_rec0[J.end - 1].x) {
        L.h0 = lower_bound_halo(A, J, lo);
        L.h1 = lower_bound_halo(A, J, hi);
    }
}

// Streaming request at sorted index p of annulus a against annulus j
// (sweep.hpp:455-461, 478-479).
__device__ __forceinline__ void setup_stream(const EdgeArgs& A, const PairJob& Jb, int j, std::uint64_t p, Lane& L) {
    L = Lane{};
    if (p >= Jb.req_end) return;
    const AnnulusDev& Aa = A.ann[Jb.a];
    const AnnulusDev& Aj = A.ann[j];
    const double      b  = A.s_beta[p];
    const double      hw = A.s_hw[p];
    const double2     r0 = A.s_rec0[p], r1 = A.s_rec1[p], r2 = A.s_rec2[p];
    L.q.cs = r1.x, L.q.sn = r1.y, L.q.coth = r2.x, L.q.rci = fmul(A.cosh_R, r2.y);
    L.q.id          = A.s_id[p];
    L.q.theta       = r0.y;
    const bool halo = p >= Aa.halo;
    double     lo, hi;
    if (j == Jb.a) { // own window [b, b + 2hw)
        lo = b;
        hi = fadd(b, fmul(2.0, hw));
    } else { // propagated window [lambda - h_j, lambda + h_j)
        const double h = half_width_in(Aj, r2.x, r2.y);
        lo             = fsub(r0.x, h);
        hi             = fadd(r0.x, h);
    }
    window_ranges(A, Aj, lo, hi, !halo, L); // halo requests: owned nodes only (no Foreign x Foreign)
    if (j == Jb.a) {
        if (!halo && p < Aa.wrap) { // theta == lambda and index order == (lambda, id) order
            const std::uint64_t w = Aj.wrap;
            L.g0 = L.s0 > w ? L.s0 : w, L.g1 = L.s1; // wrapped nodes: general
            L.s1 = L.s1 < w ? L.s1 : w;
            L.s0 = L.s0 > p + 1 ? L.s0 : p + 1;      // dedup == index order, self excluded
        } else {
            L.g0 = L.s0, L.g1 = L.s1, L.s0 = L.s1 = 0; // all general
        }
    }
    if (L.s1 < L.s0) L.s1 = L.s0;
    if (L.g1 < L.g0) L.g1 = L.g0;
    if (L.h1 < L.h0) L.h1 = L.h0;
}

// Global request g against streaming annulus Jb.j, window number w (0..3):
// split_wraparound pieces (sweep.hpp:41-58) and, when this shard owns engine
// P-1, their chunk-0 parts lifted by 2pi (sweep.hpp:404-432).  Owned nodes only.
__device__ __forceinline__ void setup_global(const EdgeArgs& A, const PairJob& Jb, std::uint64_t gs, int w, Lane& L) {
    L = Lane{};
    if (gs >= Jb.req_end) return;
    // requests run in (annulus, theta) order so that neighbouring lanes share nodes
    const std::uint64_t g  = A.gperm ? A.n_ext + A.gperm[gs - A.n_ext] : gs;
    const AnnulusDev&   Aj = A.ann[Jb.j];
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
    window_ranges(A, Aj, lo, hi, false, L);
    if (L.s1 < L.s0) L.s1 = L.s0;
}

// The reference predicate (sweep.hpp:531-533), in its rounding order:
//   lhs = fl(fl(c_r c_n) + fl(s_r s_n)),  rhs = fl(fl(k_r k_n) - fl(fl(coshR i_r) i_n)),  edge iff lhs > rhs.
template <bool DEG>
__device__ __forceinline__ void predicate(const EdgeArgs& A, const Req& q, bool in, double2 n1, double2 n2,
                                          unsigned long long nid, Acc& acc) {
    const double lhs = fadd(fmul(q.cs, n1.x), fmul(q.sn, n1.y));
    const double rhs = fsub(fmul(q.coth, n2.x), fmul(q.rci, n2.y));
    const bool   e   = in & (lhs > rhs);
    acc.comps += in;
    acc.edges += e;
    acc.fp += e ? q.id + nid : 0ull;
    if (DEG && e) {
        atomicAdd(&A.degrees[q.id], 1u);
        atomicAdd(&A.degrees[nid], 1u);
    }
}

// Tile-loop variant: per-row 32-bit counters; the fingerprint is folded as
// E * id_p + sum(node ids) when the row changes (RowAcc::fold).
struct RowAcc {
    std::uint32_t      comps = 0, edges = 0;
    unsigned long long nsum  = 0;
    __device__ __forceinline__ void fold(Acc& acc, unsigned long long id) {
        acc.comps += comps, acc.edges += edges, acc.fp += edges * id + nsum;
        comps = edges = 0, nsum = 0;
    }
};
template <bool DEG>
__device__ __forceinline__ void predicate_row(const EdgeArgs& A, const Req& q, bool in, double2 n1, double2 n2,
                                              unsigned long long nid, RowAcc& ra) {
    const double lhs = fadd(fmul(q.cs, n1.x), fmul(q.sn, n1.y));
    const double rhs = fsub(fmul(q.coth, n2.x), fmul(q.rci, n2.y));
    const bool   e   = in & (lhs > rhs);
    ra.comps += in;
    ra.edges += e;
    ra.nsum += e ? nid : 0ull;
    if (DEG && e) {
        atomicAdd(&A.degrees[q.id], 1u);
        atomicAdd(&A.degrees[nid], 1u);
    }
}

// Same-annulus pairs that need the full dedup (sweep.hpp:517-526): not self,
// and (theta_p, id_p) < (theta_q, id_q).  Rare; thread-serial.
template <bool DEG>
__device__ __forceinline__ void general_range(const EdgeArgs& A, const Req& q, std::uint64_t k0, std::uint64_t k1,
                                              Acc& acc) {
    for (std::uint64_t k = k0; k < k1; ++k) {
        const unsigned long long nid = A.s_id[k];
        const double             tq  = A.s_rec0[k].y;
        const bool in = nid != q.id && (q.theta < tq || (q.theta == tq && q.id < nid));
        predicate<DEG>(A, q, in, A.s_rec1[k], A.s_rec2[k], nid, acc);
    }
}

// ---------------------------------------------------------------- tiles ---
// Per-warp shared memory: a kStages-deep ring of kBatch-node batches filled
// by TMA bulk copies (cp.async.bulk, completion on an mbarrier), SoA so that
// lanes reading consecutive nodes are conflict-free and a whole-warp read of
// one node is a broadcast.
constexpr int kBatch  = 128;
constexpr int kStages = 2;

struct Stage {
    double2            r1[kBatch], r2[kBatch];
    unsigned long long id[kBatch + 2]; // copied from an even index: node t is id[t + (base & 1)]
};
// A tile row as the tile loop needs it (staged once per warp in shared memory).
struct RowSm {
    double             cs, sn, coth, rci;
    unsigned long long id, r0, r1, pad; // simple range [r0, r1)
};
struct WarpSmem {
    Stage              st[kStages];
    RowSm              rows[32];
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

// Lane 0 queues one batch [base, base+cnt) of sorted nodes into stage s.  The
// 8-byte ids are copied from the even index below base (bulk copies need 16 B
// alignment and size); the 16-byte records need nothing.
__device__ __forceinline__ void issue_batch(const EdgeArgs& A, WarpSmem* ws, int s, int g, std::uint64_t base,
                                            int cnt) {
    const std::uint32_t b16 = std::uint32_t(cnt) * 16u;
    const std::uint64_t nb  = base & ~1ull;
    const std::uint32_t bid = std::uint32_t(((base + cnt + 1) & ~1ull) - nb) * 8u;
    ws->meta_g[s] = g, ws->meta_cnt[s] = cnt, ws->meta_base[s] = base;
    mbar_expect_tx(&ws->bar[s], 2 * b16 + bid);
    bulk_g2s(ws->st[s].r1, A.s_rec1 + base, b16, &ws->bar[s]);
    bulk_g2s(ws->st[s].r2, A.s_rec2 + base, b16, &ws->bar[s]);
    bulk_g2s(ws->st[s].id, A.s_id + nb, bid, &ws->bar[s]);
}

// Batch cursor over the groups' unions: group g spans [ga_g, gb_g); unions
// live in lanes g*R; empty groups (gb <= ga) are skipped.
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
// simple ranges; lane (r, c) tests nodes c, c+C, ... of every batch against
// request r of the current group.  Exact: a node is tested iff its index lies
// in the row's range.
template <bool DEG, int R>
__device__ __forceinline__ void tile_run(const EdgeArgs& A, std::uint64_t ga, std::uint64_t gb, Acc& acc, int lane,
                                         WarpSmem* ws, std::uint32_t& phase) {
    constexpr int C   = 32 / R;
    const int     col = lane % C, row = lane / C;
    Cursor        prod{0, 0, 0};
    bool          more    = cursor_group(prod, R, C, ga, gb);
    int           s_issue = 0, inflight = 0;
    while (more && inflight < kStages) { // prologue: fill the ring
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
    int           s = 0, cur_g = -1;
    Req           q{};
    std::uint64_t r0 = 0, r1 = 0;
    RowAcc        ra;
    while (inflight) {
        mbar_wait(&ws->bar[s], (phase >> s) & 1u);
        phase ^= 1u << s;
        const int           g = ws->meta_g[s], cnt = ws->meta_cnt[s];
        const std::uint64_t base = ws->meta_base[s];
        const int           no   = int(base & 1);
        if (g != cur_g) {
            ra.fold(acc, q.id);
            cur_g            = g;
            const RowSm& src = ws->rows[g * R + row];
            q.cs = src.cs, q.sn = src.sn, q.coth = src.coth, q.rci = src.rci, q.id = src.id;
            r0 = src.r0, r1 = src.r1;
        }
        // the row's range relative to this batch, clamped to [0, kBatch]: int compares
        const int    lo = r0 > base ? int(r0 - base < kBatch ? r0 - base : kBatch) : 0;
        const int    hi = r1 > base ? int(r1 - base < kBatch ? r1 - base : kBatch) : 0;
        const Stage& S  = ws->st[s];
        if (cnt == kBatch) {
#pragma unroll 4
            for (int i = 0; i < kBatch / C; ++i) {
                const int t = col + C * i;
                predicate_row<DEG>(A, q, (t >= lo) & (t < hi), S.r1[t], S.r2[t], S.id[t + no], ra);
            }
        } else {
            for (int t = col; t < cnt; t += C)
                predicate_row<DEG>(A, q, (t >= lo) & (t < hi), S.r1[t], S.r2[t], S.id[t + no], ra);
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
    ra.fold(acc, q.id);
    __syncwarp();
}

template <bool DEG>
__device__ __forceinline__ void tile_dispatch(int lgR, const EdgeArgs& A, const Req& q, std::uint64_t c0,
                                              std::uint64_t c1, std::uint64_t ga, std::uint64_t gb, Acc& acc,
                                              int lane, WarpSmem* ws, std::uint32_t& phase) {
    __syncwarp();
    RowSm& me = ws->rows[lane];
    me.cs = q.cs, me.sn = q.sn, me.coth = q.coth, me.rci = q.rci, me.id = q.id, me.r0 = c0, me.r1 = c1;
    __syncwarp();
    switch (lgR) {
    case 0: tile_run<DEG, 1>(A, ga, gb, acc, lane, ws, phase); break;
    case 1: tile_run<DEG, 2>(A, ga, gb, acc, lane, ws, phase); break;
    case 2: tile_run<DEG, 4>(A, ga, gb, acc, lane, ws, phase); break;
    case 3: tile_run<DEG, 8>(A, ga, gb, acc, lane, ws, phase); break;
    case 4: tile_run<DEG, 16>(A, ga, gb, acc, lane, ws, phase); break;
    default: tile_run<DEG, 32>(A, ga, gb, acc, lane, ws, phase); break;
    }
}

// Flattened pairs: the warp's (request, candidate) pairs numbered 0..T-1 in
// lane order and processed 32 per round, one pair per lane — no divergence,
// independent loads.  The owner of pair t is the last lane whose exclusive
// prefix is <= t (5-step shuffle search).  For sparse and medium warps.
template <bool DEG>
__device__ __forceinline__ void flat_run(const EdgeArgs& A, const Req& q, std::uint64_t c0, std::uint32_t len,
                                         std::uint32_t excl, std::uint32_t total, Acc& acc, int lane,
                                         WarpSmem* ws) {
    __syncwarp();
    RowSm& me = ws->rows[lane];
    me.cs = q.cs, me.sn = q.sn, me.coth = q.coth, me.rci = q.rci, me.id = q.id, me.r0 = c0 - excl;
    __syncwarp();
    constexpr int kU = 4; // rounds per iteration: 3*kU independent loads in flight per lane
    for (std::uint32_t B = 0; B < total; B += 32 * kU) {
        std::uint64_t k[kU];
        int           own[kU];
        bool          ok[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const std::uint32_t t = B + 32u * u + std::uint32_t(lane);
            int                 o = 0;
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                const std::uint32_t v = __shfl_sync(kFull, excl, o + step);
                if (v <= t) o += step;
            }
            own[u] = o;
            ok[u]  = t < total;
            k[u]   = ok[u] ? ws->rows[o].r0 + t : 0; // = c0_o + (t - excl_o)
        }
        double2            n1[kU], n2[kU];
        unsigned long long nid[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            n1[u]  = A.s_rec1[k[u]];
            n2[u]  = A.s_rec2[k[u]];
            nid[u] = A.s_id[k[u]];
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const RowSm& r = ws->rows[own[u]];
            Req          rq;
            rq.cs = r.cs, rq.sn = r.sn, rq.coth = r.coth, rq.rci = r.rci, rq.id = r.id;
            predicate<DEG>(A, rq, ok[u], n1[u], n2[u], nid[u], acc);
        }
    }
    __syncwarp();
}

constexpr std::uint64_t kTilePiece = 4096;   // node range of one deferred tile task
constexpr std::uint64_t kDeferCost = 150000; // defer a warp's big groups above this estimated cost

constexpr std::uint32_t kFlatMax = 1u << 16; // flattened path only below this many pairs per warp

// One warp = 32 requests (one per lane) with one simple index range each.
// Picks, from the ranges, the cheapest of: the flattened pair list (sparse and
// medium warps) or an R x C tile for R in {1..32} (cost model in issue
// cycles: ~20 per 32 pair slots, ~10 per staged batch, ~40 per group; ~40
// per flattened round).  Groups of very expensive warps are cut into tile
// tasks (balanced later).
template <bool DEG>
__device__ __forceinline__ void process_range(const EdgeArgs& A, const Req& q, std::uint64_t c0, std::uint64_t c1,
                                              int kind, int job, int j, std::uint64_t p0, int pass, Acc& acc,
                                              int lane, WarpSmem* ws, std::uint32_t& phase) {
    const std::uint64_t len  = c1 > c0 ? c1 - c0 : 0;
    const std::uint32_t lenS = len < (1u << 26) ? std::uint32_t(len) : (1u << 26); // saturated: sums fit 32 bits
    const std::uint32_t tot  = __reduce_add_sync(kFull, lenS);
    if (tot == 0) return;
    const std::uint64_t total = tot;
    std::uint64_t       gmin = len ? c0 : ~0ull, gmax = len ? c1 : 0ull;
    std::uint32_t       best = tot < kFlatMax ? (tot + 31) / 32 * 40 + 60 : 0xffffffffu;
    int                 lgR  = -1;
    std::uint64_t       ga = 0, gb = 0; // this lane's group union for the chosen R (valid in group leaders)
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
        const std::uint64_t U1     = U < (1ull << 20) ? U : (1ull << 20); // saturate (cost only ranks options)
        const std::uint32_t mine   = leader && U ? std::uint32_t((U1 << k) * 20 / 32 + ((U1 + kBatch - 1) / kBatch) * 10 + 40) : 0;
        const std::uint32_t cost   = __reduce_add_sync(kFull, mine);
        if (cost < best) best = cost, lgR = k, ga = gmin, gb = gmax;
    }
    if (A.dbg && lane == 0) {
        atomicAdd(&A.dbg[22], 1ull), atomicAdd(&A.dbg[23], total);
        if (lgR < 0) atomicAdd(&A.dbg[18], 1ull), atomicAdd(&A.dbg[19], (total + 31) / 32 * 32), atomicAdd(&A.dbg[20], total);
    }
    if (lgR < 0) {
        std::uint32_t incl = std::uint32_t(len);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const std::uint32_t t = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += t;
        }
        flat_run<DEG>(A, q, c0, std::uint32_t(len), incl - std::uint32_t(len), tot, acc, lane, ws);
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
        const std::uint64_t a0   = ga & ~1ull;
        const std::uint64_t npc  = leader && gb - ga > kTilePiece ? (gb - a0 + kTilePiece - 1) / kTilePiece : 0;
        std::uint64_t       incl = npc;
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
                for (std::uint64_t i = 0; i < npc; ++i) { // even piece starts (TMA id copies)
                    TileTask& T = A.tasks[first + i];
                    T.p0 = p0 + std::uint64_t(lane), T.u0 = i ? a0 + i * kTilePiece : ga;
                    T.u1 = a0 + (i + 1) * kTilePiece < gb ? a0 + (i + 1) * kTilePiece : gb;
                    T.job = job, T.kind = std::int16_t(kind), T.lgR = std::int16_t(lgR), T.w = pass, T.j = j;
                }
                if (npc) gb = ga; // handed off
            }
        }
    }
    tile_dispatch<DEG>(lgR, A, q, c0, c1, ga, gb, acc, lane, ws, phase);
}

__device__ __forceinline__ WarpSmem* my_warp_smem() {
    extern __shared__ __align__(128) unsigned char dyn_smem[];
    return reinterpret_cast<WarpSmem*>(dyn_smem) + (threadIdx.x >> 5);
}

// Work item t -> (pair job, batch of 32 requests).  Items are ordered by
// angular block first (block b holds batches [floor(b nb/M), floor((b+1) nb/M))
// of every job), so the warps in flight all work on one narrow angular band.
__device__ __forceinline__ void map_item(const EdgeArgs& A, std::uint64_t t, int& job, std::uint64_t& batch) {
    int lo = 0, hi = A.nblk - 1; // last block with prefix <= t
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (A.blk_prefix[mid] <= t) lo = mid;
        else hi = mid - 1;
    }
    const int            b     = lo;
    const std::uint32_t  local = std::uint32_t(t - A.blk_prefix[b]);
    const std::uint32_t* off   = A.blk_job_off + std::size_t(b) * A.n_stream_jobs;
    int                  k0 = 0, k1 = A.n_stream_jobs - 1; // last job with off <= local
    while (k0 < k1) {
        const int mid = (k0 + k1 + 1) >> 1;
        if (off[mid] <= local) k0 = mid;
        else k1 = mid - 1;
    }
    job                    = k0;
    const PairJob&      J  = A.stream_jobs[job];
    const std::uint64_t nb = (J.req_end - J.req_off + 31) / 32;
    batch                  = std::uint64_t(b) * nb / std::uint64_t(A.nblk) + (local - off[k0]);
}

template <bool DEG>
__global__ void __launch_bounds__(256, 2) stream_pairs_kernel(EdgeArgs A) {
    const int           lane = threadIdx.x & 31;
    const std::uint64_t t    = (std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (t >= A.stream_warps) return;
    WarpSmem* ws = my_warp_smem();
    warp_smem_init(ws, lane);
    std::uint32_t phase = 0;
    Acc           acc;
    int           job;
    std::uint64_t batch;
    map_item(A, t, job, batch);
    const PairJob       Jb = A.stream_jobs[job];
    const std::uint64_t p0 = Jb.req_off + batch * 32;
#pragma unroll 1
    for (int j = Jb.a; j < A.count; ++j) { // every target annulus of these 32 requests
        if (A.ann[j].end == A.ann[j].off) continue;
        Lane L;
        setup_stream(A, Jb, j, p0 + lane, L);
        process_range<DEG>(A, L.q, L.s0, L.s1, 0, job, j, p0, 0, acc, lane, ws, phase);
        if (j != Jb.a) {
            process_range<DEG>(A, L.q, L.h0, L.h1, 0, job, j, p0, 1, acc, lane, ws, phase);
        } else { // same-annulus pairs with wrapped or halo points: full dedup
            general_range<DEG>(A, L.q, L.g0, L.g1, acc);
            general_range<DEG>(A, L.q, L.h0, L.h1, acc);
        }
    }
    flush(acc, &A.ctr[0], lane);
}

template <bool DEG>
__global__ void __launch_bounds__(256, 2) glob_req_kernel(EdgeArgs A) {
    const int           lane = threadIdx.x & 31;
    const std::uint64_t gw   = (std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (gw >= A.glob_warps) return;
    WarpSmem* ws = my_warp_smem();
    warp_smem_init(ws, lane);
    std::uint32_t phase = 0;
    int           lo = 0, hi = A.n_glob_jobs - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (A.glob_jobs[mid].warp_begin <= gw) lo = mid;
        else hi = mid - 1;
    }
    const int           job = lo;
    const PairJob       Jb  = A.glob_jobs[job];
    const std::uint64_t g0  = Jb.req_off + (gw - Jb.warp_begin) * 32;
    Acc                 acc;
#pragma unroll 1
    for (int w = 0; w < 4; ++w) {
        Lane L;
        setup_global(A, Jb, g0 + lane, w, L);
        process_range<DEG>(A, L.q, L.s0, L.s1, 1, job, Jb.j, g0, w, acc, lane, ws, phase);
    }
    flush(acc, &A.ctr[1], lane);
}

// Deferred tile pieces: the R requests of one group x kTilePiece nodes
// (KIND 0 streaming requests with T.w = pass 0 owned / 1 halo block, KIND 1
// global requests with T.w = window).
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
            setup_stream(A, A.stream_jobs[T.job], T.j, p, L);
            if (T.w == 0) tile_dispatch<DEG>(T.lgR, A, L.q, L.s0, L.s1, ga, gb, acc, lane, ws, phase);
            else tile_dispatch<DEG>(T.lgR, A, L.q, L.h0, L.h1, ga, gb, acc, lane, ws, phase);
        } else {
            setup_global(A, A.glob_jobs[T.job], p, T.w, L);
            tile_dispatch<DEG>(T.lgR, A, L.q, L.s0, L.s1, ga, gb, acc, lane, ws, phase);
        }
    }
    flush(acc, &A.ctr[KIND], lane);
}

// Sort keys of the global points: theta quantised to 32 bits (any order is
// exact; this one makes neighbouring requests' windows overlap).
__global__ void glob_keys_kernel(EdgeArgs A, std::uint32_t* keys, std::uint32_t* vals) {
    const std::uint64_t i = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= A.n_glob) return;
    const double th = A.rec0[A.n_ext + i].y; // [0, 2pi)
    const double q  = th * (4294967296.0 / kTwoPiD);
    keys[i]         = q >= 4294967295.0 ? 0xffffffffu : std::uint32_t(q);
    vals[i]         = std::uint32_t(i);
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
    const std::uint64_t J   = I + (t - start(I));
    const std::uint64_t nG  = A.n_glob;
    const std::uint64_t col = J * kGGTile + threadIdx.x;
    if (col < nG) {
        s1[threadIdx.x] = A.rec1[A.n_ext + col];
        s2[threadIdx.x] = A.rec2[A.n_ext + col];
    }
    __syncthreads();
    const std::uint64_t i = I * kGGTile + threadIdx.x;
    Acc                 acc;
    if (i < nG) {
        Req           q{};
        const double2 r1 = A.rec1[A.n_ext + i], r2 = A.rec2[A.n_ext + i];
        q.cs = r1.x, q.sn = r1.y, q.coth = r2.x, q.rci = fmul(A.cosh_R, r2.y), q.id = i;
        std::uint64_t k0 = J * kGGTile;
        if (k0 <= i) k0 = i + 1;
        const std::uint64_t k1 = (J + 1) * kGGTile < nG ? (J + 1) * kGGTile : nG;
        for (std::uint64_t k = k0; k < k1; ++k)
            predicate<DEG>(A, q, true, s1[k - J * kGGTile], s2[k - J * kGGTile], k, acc);
    }
    flush(acc, &A.ctr[2], threadIdx.x & 31);
}

} // namespace

void launch_cell_index(const EdgeArgs& a, std::uint64_t nblocks, cudaStream_t st, std::uint64_t* launches) {
    if (a.first_streaming >= a.count) return;
    const unsigned g = unsigned(nblocks ? nblocks : 1); // >= 1: block 0 also initialises empty annuli
    const dim3     tails(64, unsigned(a.count - a.first_streaming));
    beta_cells_kernel<<<g, 256, 0, st>>>(a);
    cell_tail_kernel<<<tails, 256, 0, st>>>(a, 0);
    *launches += 2;
    if (nblocks) {
        rank_kernel<<<g, 256, 0, st>>>(a);
        scatter_kernel<<<g, 256, 0, st>>>(a);
        lambda_cells_kernel<<<g, 256, 0, st>>>(a);
        cell_tail_kernel<<<tails, 256, 0, st>>>(a, 1);
        *launches += 4;
    }
}

void launch_sort_globals(EdgeArgs& a, const std::uint64_t* seg_off_dev, int nseg, void* scratch,
                         std::size_t scratch_bytes, std::size_t* need, cudaStream_t st, std::uint64_t* launches) {
    // scratch: keys_in | keys_out | vals_in | perm(out) | cub temp
    const std::size_t n   = a.n_glob;
    const std::size_t al  = (n * 4 + 255) & ~std::size_t(255);
    std::size_t       tmp = 0;
    cub::DeviceSegmentedRadixSort::SortPairs(nullptr, tmp, static_cast<const std::uint32_t*>(nullptr),
                                             static_cast<std::uint32_t*>(nullptr),
                                             static_cast<const std::uint32_t*>(nullptr),
                                             static_cast<std::uint32_t*>(nullptr), int(n), nseg, seg_off_dev,
                                             seg_off_dev + 1, 0, 32, st);
    *need = 4 * al + tmp + 256;
    if (!scratch || scratch_bytes < *need || n == 0) return;
    char*          p    = static_cast<char*>(scratch);
    std::uint32_t* kin  = reinterpret_cast<std::uint32_t*>(p);
    std::uint32_t* kout = reinterpret_cast<std::uint32_t*>(p + al);
    std::uint32_t* vin  = reinterpret_cast<std::uint32_t*>(p + 2 * al);
    std::uint32_t* perm = reinterpret_cast<std::uint32_t*>(p + 3 * al);
    glob_keys_kernel<<<unsigned((n + 255) / 256), 256, 0, st>>>(a, kin, vin);
    cub::DeviceSegmentedRadixSort::SortPairs(p + 4 * al, tmp, kin, kout, vin, perm, int(n), nseg, seg_off_dev,
                                             seg_off_dev + 1, 0, 32, st);
    a.gperm = perm;
    *launches += 2;
}

void launch_edges(const EdgeArgs& a, cudaStream_t st, std::uint64_t* launches) {
    const bool  deg   = a.degrees != nullptr;
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
    if (a.stream_warps) { // one warp per item, items in angular-block order
        const unsigned blocks = unsigned((a.stream_warps + kWarpsPerBlock - 1) / kWarpsPerBlock);
        if (a.ev_pairs0) cudaEventRecord(a.ev_pairs0, st);
        if (deg) stream_pairs_kernel<true><<<blocks, 32 * kWarpsPerBlock, kTileSmem, st>>>(a);
        else stream_pairs_kernel<false><<<blocks, 32 * kWarpsPerBlock, kTileSmem, st>>>(a);
        if (a.ev_pairs1) cudaEventRecord(a.ev_pairs1, st);
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
