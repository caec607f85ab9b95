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
// request index" — the hot loops have no window or dedup compares at all.
//
//   beta_cells_kernel   beta-cell starts of the beta-ordered sampler output and
//                       the exact per-annulus max half-width
//   rank_kernel         exact rank of every point by (lambda, id) inside its block,
//                       and the point written straight to its slot of the
//                       lambda-sorted arrays (generate mode: with its angular step)
//   lambda_cells_kernel lambda-cell starts of the owned blocks, first wrapped index
//   cell_tail_kernel    the cell tables' tails
//   req_*_kernel        dense-engine prep: requests sorted by (source, class, angle),
//                       segment tables, window-piece rows per target (req_rows)
//   glob_tiles_kernel   dense engine: one warp = 128 owned nodes held in registers x
//                       every dense request whose window can reach them
//   glob_pairs_kernel   global unit, 128x128 tiles of the upper triangle
//   slab_kernel         sparse engine: one CTA = a 512-node slab of a target annulus
//                       x the requests whose windows reach it (FP32 pre-filter,
//                       exact FP64 recheck), pairs flattened over the warp
//   tail_kernel         halo / wrapped pairs the slab join leaves out
//   deferred_kernel     dense-engine ranges deferred from the tiles
//   reduce_counters_kernel  folds the spread counter slots
//   edge_keys / edge_unpack  materialised edges: canonical sort (MODE 2)
#include <cstdlib>

#include <cub/cub.cuh>

#include "device.cuh"
#include "kernels.hpp"

namespace rhgb {

namespace {

constexpr unsigned kFull = 0xffffffffu;

struct Acc {
    unsigned long long edges = 0, fp = 0, comps = 0;
};

// Warp-reduce the lane accumulators and add them to one of kSlots spread
// counter slots of family f (same-address atomics from every warp would
// serialise in L2); reduce_counters_kernel folds the slots at the end.
// With j >= 0 the warp's totals also go to the per-annulus counters of annulus j
// (ChunkStats::edges_by_annulus / comps_by_annulus, sweep.hpp:530-539: the node's annulus).
template <bool ANN = false>
__device__ __forceinline__ void flush(Acc& acc, const EdgeArgs& A, int f, int lane, int j = -1) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        acc.edges += __shfl_down_sync(kFull, acc.edges, o);
        acc.fp += __shfl_down_sync(kFull, acc.fp, o);
        acc.comps += __shfl_down_sync(kFull, acc.comps, o);
    }
    if (lane == 0 && (acc.comps | acc.edges)) {
        const unsigned w    = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
        SlotCounter&   slot = A.slots[f * kSlots + (w & (kSlots - 1))];
        atomicAdd(&slot.edges, acc.edges);
        atomicAdd(&slot.fp, acc.fp);
        atomicAdd(&slot.comps, acc.comps);
        if (ANN && j >= 0) {
            unsigned long long* c = A.ann_ctr + std::size_t(w & (kAnnSlots - 1)) * 2 * kMaxAnnuli;
            atomicAdd(&c[j], acc.edges), atomicAdd(&c[kMaxAnnuli + j], acc.comps);
        }
    }
}

// Per-annulus counters accumulated in shared memory by a CTA whose threads see several
// annuli (tail, rows, deferred, global unit), then added to A.ann_ctr once per CTA.
struct AnnAcc {
    unsigned long long e[kMaxAnnuli], c[kMaxAnnuli];
};
template <bool ANN>
__device__ __forceinline__ void ann_zero(AnnAcc& S) {
    if (!ANN) return;
    for (int i = threadIdx.x; i < kMaxAnnuli; i += blockDim.x) S.e[i] = 0, S.c[i] = 0;
}
template <bool ANN>
__device__ __forceinline__ void ann_add(AnnAcc& S, int j, unsigned long long e, unsigned long long c) {
    if (!ANN) return;
    if (e) atomicAdd(&S.e[j], e);
    if (c) atomicAdd(&S.c[j], c);
}
template <bool ANN>
__device__ __forceinline__ void ann_flush(const AnnAcc& S, const EdgeArgs& A) {
    if (!ANN) return;
    unsigned long long* c = A.ann_ctr + std::size_t(blockIdx.x & (kAnnSlots - 1)) * 2 * kMaxAnnuli;
    for (int i = threadIdx.x; i < kMaxAnnuli; i += blockDim.x) {
        if (S.e[i]) atomicAdd(&c[i], S.e[i]);
        if (S.c[i]) atomicAdd(&c[kMaxAnnuli + i], S.c[i]);
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

// Sort-phase kernels run ceil(n_j / 256) blocks per streaming annulus j
// (prefix table A.ann_blk), so every block knows its annulus without a search
// per thread.  Returns the annulus of this block and sets i (maybe >= end).
__device__ __forceinline__ int block_annulus(const EdgeArgs& A, std::uint64_t& i) {
    const std::uint32_t b    = A.blk0 + blockIdx.x; // waves launch a sub-range of the blocks
    const int           lane = threadIdx.x & 31;
    int                 j    = A.first_streaming; // last annulus with ann_blk <= b (one ballot per 32 annuli)
    for (int base = 0; base < A.count; base += 32) {
        const int      a = base + lane;
        const unsigned m = __ballot_sync(0xffffffffu, a < A.count && a >= A.first_streaming && A.ann_blk[a] <= b);
        if (m) j = base + 31 - __clz(m);
    }
    i = A.ann[j].off + std::uint64_t(b - A.ann_blk[j]) * 256u + threadIdx.x;
    return j;
}

__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long t = __shfl_xor_sync(kFull, v, o);
        v                          = t > v ? t : v;
    }
    return v;
}

// Fill a cell-start table: entries (kp, k] = i.  The tail after the last
// point, (k_last, ncells] = end, is filled in parallel by cell_tail_kernel.
__device__ __forceinline__ void cell_fill(std::uint64_t* tab, std::int64_t kp, std::uint32_t k, std::uint64_t i) {
    for (std::uint32_t c = std::uint32_t(kp + 1); c <= k; ++c) tab[c] = i; // kp >= -1: kp + 1 >= 0
}

// ---------------------------------------------------------------- sort ---
// Engine-frame begin of point i of annulus block J (generate mode: the beta
// array holds the unlifted beta; the halo block of the shard owning engine
// P-1 is chunk 0 lifted by 2pi, sweep.hpp:252, 466-467).
template <bool GEN>
__device__ __forceinline__ double frame_beta(const EdgeArgs& A, const AnnulusDev& J, std::uint64_t i) {
    const double b = A.beta[i];
    return GEN && A.lift_part && i >= J.halo ? fadd(b, kTwoPiD) : b;
}

#ifndef RHG_RANK_MINB
#define RHG_RANK_MINB 8 // sort-phase rank/scatter at full occupancy (32 registers: rank 0.23 -> 0.20 ms, cfg2 3.82 -> 3.77)
#endif
template <bool GEN>
__global__ void __launch_bounds__(256, RHG_RANK_MINB) beta_cells_kernel(EdgeArgs A) {
    const int lane = threadIdx.x & 31;
    if (blockIdx.x == 0 && A.blk0 == 0 && int(threadIdx.x) < A.count && int(threadIdx.x) >= A.first_streaming) {
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
        const double        bi = frame_beta<GEN>(A, J, i), hi = A.hw[i];
        const std::uint32_t k  = cellf(J, bi);
        const std::int64_t  kp = i > J.off ? std::int64_t(cellf(J, frame_beta<GEN>(A, J, i - 1))) : -1;
        cell_fill(A.cellstart + J.cell_off, kp, k, i);
        hwbits     = static_cast<unsigned long long>(__double_as_longlong(hi)); // hw >= +0
        A.lam_tmp[i] = GEN ? fadd(bi, hi) : A.rec0[i].x; // engine-frame lambda, read by rank_kernel
    }
    if constexpr (!GEN) { // same-points runs: the annulus's largest uploaded half-width, measured
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
}

// Point i of annulus block J to its sorted position d.  Same-points mode: copy the given frames.
__device__ __forceinline__ void scatter_point(const EdgeArgs& A, const AnnulusDev& J, std::uint64_t i,
                                              std::uint64_t d) {
    const double2       r0 = A.rec0[i];
    A.s_beta[d]            = A.beta[i];
    A.s_hw[d]              = A.hw[i];
    A.s_lam[d]             = r0.x;
    A.s_theta[d]           = r0.y;
    A.s_rec1[d]            = A.rec1[i];
    A.s_rec2[d]            = A.rec2[i];
    A.s_id[d]              = i + static_cast<unsigned long long>(i < J.halo ? J.dlt0 : J.dlt1);
}
// Generate mode: the sampler's angular step (sweep.hpp:135-139, 478-480: theta = beta + hw
// mod 2pi, cos, sin, engine-frame begin/centre) fused with the scatter, so the frames go
// straight to their sorted positions.
__device__ __forceinline__ void angular_scatter_point(const EdgeArgs& A, const AnnulusDev& J, std::uint64_t i,
                                                      std::uint64_t d) {
    const double b0 = A.beta[i], h = A.hw[i];
    double       th = fadd(b0, h);
    if (th >= kTwoPiD) th = fsub(th, kTwoPiD);
    double sn, cs;
    gl::gl_sincos(th, &sn, &cs);
    const double bf = A.lift_part && i >= J.halo ? fadd(b0, kTwoPiD) : b0;
    A.s_beta[d]     = bf;
    A.s_hw[d]       = h;
    A.s_lam[d]      = fadd(bf, h);
    if (A.lift_part && i >= J.halo) A.s_theta[d] = th; // elsewhere theta follows from lambda (theta_of)
    A.s_rec1[d]     = make_double2(cs, sn);
    A.s_rec2[d]     = A.rec2[i];
    A.s_id[d]       = i + static_cast<unsigned long long>(i < J.halo ? J.dlt0 : J.dlt1);
}

// theta of sorted point k (sweep.hpp:135-139): in generate mode an unlifted point's lambda is
// fl(beta + hw) itself, so theta = lambda, or fl(lambda - 2pi) from 2pi on, exactly as the angular
// step computes it; only the lifted halo block (k >= lift_from) and same-points runs store it.
__device__ __forceinline__ double theta_of(const EdgeArgs& A, std::uint64_t k, std::uint64_t lift_from) {
    if (!A.gen || k >= lift_from) return A.s_theta[k];
    const double l = A.s_lam[k];
    return l >= kTwoPiD ? fsub(l, kTwoPiD) : l;
}
__device__ __forceinline__ std::uint64_t lift_from(const EdgeArgs& A, const AnnulusDev& J) {
    return A.lift_part ? J.halo : ~std::uint64_t(0);
}

// Exact rank of point i by (lambda, beta-order index) inside its block; in the
// owned block beta-order index order is id order, so the sorted order is
// (lambda, id).  Only points whose beta lies in [lambda_i - dmax, lambda_i]
// can compare either way: everything before that window is smaller
// (lambda <= beta + dmax), everything after is larger (lambda >= beta).
template <bool GEN, bool GALLOP = false>
__global__ void __launch_bounds__(256, RHG_RANK_MINB) rank_kernel(EdgeArgs A) {
    std::uint64_t       i;
    const int           j = block_annulus(A, i);
    const AnnulusDev&   J = A.ann[j];
    if (i >= J.end) return;
    const bool          hb = i >= J.halo;
    const std::uint64_t bs = hb ? J.halo : J.off, be = hb ? J.end : J.halo;
    // the annulus's largest half-width: in generate mode the host bound at its lower radius
    // (half-widths fall with the radius; hbound carries a 1e-6 relative margin over the device's
    // rounding), in same-points runs the measured maximum
    const double        dm = GEN ? A.hbound[std::size_t(j) * A.count + j]
                                 : __longlong_as_double(static_cast<long long>(A.dmax_bits[j]));
    std::uint64_t       rank;
    double              li;
    if constexpr (GALLOP) {
        // no beta-cell table: walk the window outwards from i itself (it holds ~d points, and
        // every one of them is compared anyway), lambdas computed in place; the block's points
        // are all lifted or none (the lifted halo block), so the frame shift is one flag
        const bool lift = A.lift_part && hb;
        auto       fb   = [&](std::uint64_t k) {
            const double b = A.beta[k];
            return lift ? fadd(b, kTwoPiD) : b;
        };
        li              = fadd(fb(i), A.hw[i]);
        const double lo = fsub(fsub(li, dm), 1e-12);
        rank            = 0;
        for (std::uint64_t k = i; k > bs;) { // beta(k) < lo: k and everything before it is smaller
            --k;
            const double b = fb(k);
            if (b < lo) { rank += k - bs + 1; break; }
            rank += fadd(b, A.hw[k]) <= li; // k < i: ties count
        }
        for (std::uint64_t k = i + 1; k < be; ++k) { // beta(k) > li: k and everything after is larger
            const double b = fb(k);
            if (b > li) break;
            rank += fadd(b, A.hw[k]) < li;
        }
    } else { // the beta-cell table and lambdas of beta_cells_kernel
        li               = A.lam_tmp[i];
        std::uint64_t k0 = A.cellstart[J.cell_off + cellf(J, fsub(fsub(li, dm), 1e-12))];
        std::uint64_t k1 = A.cellstart[J.cell_off + cellf(J, li) + 1];
        k0               = k0 < bs ? bs : k0;
        k1               = k1 > be ? be : k1;
        rank             = k0 - bs;
        for (std::uint64_t k = k0; k < k1; ++k) {
            const double lk = A.lam_tmp[k];
            rank += (lk < li) || (lk == li && k < i);
        }
    }
    // the point goes straight to its sorted slot (measured cfg2: rank 0.20 + scatter 0.31 ms
    // as two kernels through a permutation array -> 0.41 ms fused)
    if (GEN) angular_scatter_point(A, J, i, bs + rank);
    else scatter_point(A, J, i, bs + rank);
}

// Lambda-cell starts of every owned block, and the first owned index with
// lambda >= 2pi (wrapped points: theta = lambda - 2pi there).
__global__ void __launch_bounds__(256) lambda_cells_kernel(EdgeArgs A) {
    if (blockIdx.x == 0 && A.blk0 == 0 && A.gen && A.rank_gallop && int(threadIdx.x) < A.count &&
        int(threadIdx.x) >= A.first_streaming) {
        const AnnulusDev& E = A.ann[threadIdx.x]; // empty owned blocks: [off, off] (beta_cells does it otherwise)
        if (E.halo == E.off)
            for (std::uint32_t k = 0; k <= E.ncells; ++k) A.lcellstart[E.cell_off + k] = E.off;
    }
    std::uint64_t i;
    const int     j = block_annulus(A, i);
    AnnulusDev&   J = A.ann_rw[j];
    if (i >= J.halo) return;
    const double        l  = A.s_lam[i];
    const std::uint32_t k  = cellf(J, l);
    const std::int64_t  kp = i > J.off ? std::int64_t(cellf(J, A.s_lam[i - 1])) : -1;
    cell_fill(A.lcellstart + J.cell_off, kp, k, i);
    if (l >= kTwoPiD && (i == J.off || A.s_lam[i - 1] < kTwoPiD)) J.wrap = i;
}

// Tails of both cell tables: cells after the last point of a block hold the
// block end (beta table: whole annulus array; lambda table: owned block).
__global__ void cell_tail_kernel(EdgeArgs A, int lambda) {
    const int           j = A.j0 + int(blockIdx.y);
    const AnnulusDev&   J = A.ann[j];
    const std::uint64_t e = lambda ? J.halo : J.end;
    if (e == J.off) return; // empty: initialised by beta_cells_kernel
    const double        last = lambda ? A.s_lam[e - 1] : (A.gen ? frame_beta<true>(A, J, e - 1) : A.beta[e - 1]);
    const std::uint32_t k0   = cellf(J, last) + 1;
    std::uint64_t*      tab  = (lambda ? A.lcellstart : A.cellstart) + J.cell_off;
    for (std::uint32_t c = k0 + blockIdx.x * blockDim.x + threadIdx.x; c <= J.ncells; c += gridDim.x * blockDim.x)
        tab[c] = e;
}

// ------------------------------------------------------- window search ---
// Advance k over the nodes of [k, e) with lambda < x, four independent loads
// at a time (cells hold ~2 nodes, so one step almost always suffices).
__device__ __forceinline__ std::uint64_t scan_lt(const double* __restrict__ lam, std::uint64_t k, std::uint64_t e,
                                                 double x) {
    while (k < e) {
        const std::uint64_t n = e - k;
        const double        x0 = lam[k];
        const double        x1 = n > 1 ? lam[k + 1] : x;
        const double        x2 = n > 2 ? lam[k + 2] : x;
        const double        x3 = n > 3 ? lam[k + 3] : x;
        const unsigned      c  = unsigned(x0 < x) + unsigned(x1 < x) + unsigned(x2 < x) + unsigned(x3 < x);
        k += c;
        if (c < 4) break;
    }
    return k;
}
// First index k in the sorted owned block with lambda[k] >= x (exact): the
// lambda cell of x bounds it from both sides (cellf is monotone).
__device__ __forceinline__ std::uint64_t lower_bound_owned(const EdgeArgs& A, const AnnulusDev& J, double x) {
    const std::uint32_t c = cellf(J, x);
    return scan_lt(A.s_lam, A.lcellstart[J.cell_off + c], A.lcellstart[J.cell_off + c + 1], x);
}
// Both bounds of [lo, hi): the four cell-table loads are issued together.
__device__ __forceinline__ void owned_range(const EdgeArgs& A, const AnnulusDev& J, double lo, double hi,
                                            std::uint64_t& s0, std::uint64_t& s1) {
    const std::uint32_t ca = cellf(J, lo), cb = cellf(J, hi);
    const std::uint64_t ka = A.lcellstart[J.cell_off + ca], kb = A.lcellstart[J.cell_off + cb];
    const std::uint64_t ea = A.lcellstart[J.cell_off + ca + 1], eb = A.lcellstart[J.cell_off + cb + 1];
    s0 = scan_lt(A.s_lam, ka, ea, lo);
    s1 = scan_lt(A.s_lam, kb, eb, hi);
}
__device__ __forceinline__ std::uint64_t lower_bound_halo(const EdgeArgs& A, const AnnulusDev& J, double x) {
    std::uint64_t lo = J.halo, hi = J.end; // binary search (one chunk, rarely searched)
    while (lo < hi) {
        const std::uint64_t mid = (lo + hi) >> 1;
        if (A.s_lam[mid] < x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// The reference predicate (sweep.hpp:531-533), in its rounding order:
//   lhs = fl(fl(c_r c_n) + fl(s_r s_n)),  rhs = fl(fl(k_r k_n) - fl(fl(coshR i_r) i_n)),  edge iff lhs > rhs.
// rci = fl(coshR * i_r) is hoisted per request.
__device__ __forceinline__ bool edge_test(double cs, double sn, double coth, double rci, double2 n1, double2 n2) {
    const double lhs = fadd(fmul(cs, n1.x), fmul(sn, n1.y));
    const double rhs = fsub(fmul(coth, n2.x), fmul(rci, n2.y));
    return lhs > rhs;
}

// Materialised edge stream (MODE 2): canonical (min id, max id) pairs appended
// to A.edge_out with one warp-aggregated atomic per call site; the host sorts
// them (rhg_generate_edges).  Pairs past edge_cap are counted, not written.
__device__ __forceinline__ void emit_edge(const EdgeArgs& A, unsigned long long a, unsigned long long b) {
    const unsigned           m      = __activemask();
    const int                lane   = threadIdx.x & 31;
    const int                leader = __ffs(m) - 1;
    unsigned long long       base   = 0;
    if (lane == leader) base = atomicAdd(A.edge_count, static_cast<unsigned long long>(__popc(m)));
    base                          = __shfl_sync(m, base, leader);
    const unsigned long long slot = base + __popc(m & ((1u << lane) - 1u));
    if (slot < A.edge_cap) A.edge_out[slot] = make_ulonglong2(a < b ? a : b, a < b ? b : a);
}

// MODE: 0 = counters only, 1 = + per-vertex degrees, 2 = + materialised edges
template <int MODE>
__device__ __forceinline__ void count_edge(const EdgeArgs& A, bool e, unsigned long long id_r,
                                           unsigned long long id_n, Acc& acc) {
    acc.edges += e;
    acc.fp += e ? id_r + id_n : 0ull;
    if (MODE == 1 && e) {
        atomicAdd(&A.degrees[id_r], 1u);
        atomicAdd(&A.degrees[id_n], 1u);
    }
    if (MODE == 2 && e) emit_edge(A, id_r, id_n);
}

// ------------------------------------------------ streaming (sparse) ---

struct SRow { // one request as the cooperative loop reads it (broadcast from shared memory)
    double             cs, sn, coth, rci;
    unsigned long long id, pad;
};

// Thread-serial pairs (rare): halo-block ranges and same-annulus pairs that
// need the full (theta, id) dedup (sweep.hpp:517-526).
template <int MODE>
__device__ __forceinline__ void serial_range(const EdgeArgs& A, const SRow& q, double theta, bool dedup,
                                             std::uint64_t k0, std::uint64_t k1, std::uint64_t lift, Acc& acc) {
    for (std::uint64_t k = k0; k < k1; k += 4) { // four independent nodes in flight
        double2            n1[4], n2[4];
        unsigned long long nid[4];
        double             tq[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const std::uint64_t kk = k + u < k1 ? k + u : k;
            n1[u] = A.s_rec1[kk], n2[u] = A.s_rec2[kk], nid[u] = A.s_id[kk];
            tq[u] = dedup ? theta_of(A, kk, lift) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            bool in = k + u < k1;
            if (dedup) in = in && nid[u] != q.id && (theta < tq[u] || (theta == tq[u] && q.id < nid[u]));
            if (!in) continue;
            if (A.dbg) atomicAdd(&A.dbg[5], 1ull);
            acc.comps += 1;
            count_edge<MODE>(A, edge_test(q.cs, q.sn, q.coth, q.rci, n1[u], n2[u]), q.id, nid[u], acc);
        }
    }
}

// ---------------------------------------------------------- slab join ---
// Sparse (annulus a, target j) pairs.  CTA = one slab of kSlab consecutive
// nodes of j's owned block, staged in shared memory once (coalesced).  For
// every sparse source annulus a <= j the requests whose window can reach the
// slab (lambda within hbound(a, j) of it: a contiguous run of a's sorted
// owned block, from a's lambda-cell table) are streamed through the warps,
// 32 at a time; each lane finds its exact node range in the slab by binary
// search over the staged lambdas and tests it lane-serially from shared
// memory.  Every pair belongs to exactly one slab (its node's), so comps add.
// Own annulus (j == a): requests and nodes below the wrap index only, nodes
// after the request (index order == (theta, id) dedup order); everything
// else - halo requests, halo nodes, wrapped points - runs in tail_kernel.
constexpr int kSlab        = kSlabNodes;


// Bucket of an angle inside the slab: monotone in x (fsub, fmul, clamp), so
// lower_bound(x) lies in [bstart[b], bstart[b + 1]] for b = bucket(x).
__device__ __forceinline__ std::uint32_t slab_bucket(double x, double org, double inv_w) {
    const double t = fmul(fsub(x, org), inv_w);
    if (!(t > 0.0)) return 0;
    if (t >= double(kSlab - 1)) return kSlab - 1;
    return std::uint32_t(t);
}
template <class SM>
__device__ __forceinline__ std::uint32_t slab_lb(const SM& S, const double* lam, double x, double org, double inv_w) {
    const std::uint32_t b = slab_bucket(x, org, inv_w);
    std::uint32_t       k = S.bstart[b];
    const std::uint32_t e = S.bstart[b + 1];
    while (k < e && lam[k] < x) ++k;
    return k;
}

// ---- TMA bulk copies (cp.async.bulk global -> shared, completion on an mbarrier) ----
__device__ __forceinline__ unsigned smem_addr(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
// 16-byte shared-memory load by 32-bit shared address (keeps the loop from re-deriving the
// generic shared window base, S2R SR_CgaCtaId, on every pair under register pressure)
__device__ __forceinline__ float4 lds128(unsigned addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint4 lds128u(unsigned addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}
__device__ __forceinline__ void mbar_init(std::uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(std::uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
// bytes: a multiple of 16; src and dst 16-byte aligned
__device__ __forceinline__ void bulk_copy_g2s(void* dst, const void* src, unsigned bytes, std::uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(std::uint64_t* bar, unsigned phase) {
    asm volatile("{\n\t.reg .pred p;\n"
                 "WAIT_%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                 "@!p bra WAIT_%=;\n}"
                 ::"r"(smem_addr(bar)), "r"(phase)
                 : "memory");
}

// FP32 pre-filter of the reference predicate (sweep.hpp:531-533), exact by
// construction: with the stored doubles of request r and node n,
//   D = lhs - rhs = (c_r c_n + s_r s_n) - coth_r coth_n + rci_r inv_n
// is rewritten with three non-negative, well-conditioned terms
//   P = rci_r inv_n,  Q = coth_r coth_n - 1 = m_r + m_n + m_r m_n  (m = coth - 1, exact in FP64),
//   S = 1 - cos(theta_r - theta_n) = Delta^2 / 2 - Delta^4 / 24 + ...  (Delta = lambda_n - lambda_r),
// D ~= P - (Q + S), evaluated in FP32 from float copies (lambda as offsets from
// the slab's first node).  |D32 - D_ref| is bounded by
//   * FP32 rounding of P, Q, S and their inputs        <= 1.1e-6 (P + Q + S)
//   * the float offsets of lambda                      <= |Delta| ed + ed^2,   ed = 2^-24 (|off_r| + span) + 1.5e-15
//   * the reference's own FP64 rounding (6 roundings)  <= 2.3e-16 (2 + P + Q)
//   * the stored cos/sin vs cos(theta) (CUDA sincos, <= 2 ulp) and the 2pi wrap
//     of theta (theta = lambda - 2pi_d)                <= 6.5e-16 + 1.4e-15 |Delta|
// (Appendix of DESIGN.md); tau below covers the sum with a 25% margin.  Only when
// |D32| > tau does the FP32 sign decide; otherwise (and for |Delta| > 2^-6, where
// the truncated series is not used) the pair takes the exact FP64 predicate.
constexpr float  kPreMaxDelta = 0.015625f;
#ifndef RHG_SLAB_MINB
#define RHG_SLAB_MINB 6 // CTAs per SM of the pre-filter slab join (40 registers)
#endif
#ifndef RHG_SLAB_DIRECT
#define RHG_SLAB_DIRECT 8 // groups whose lanes have <= this many pairs each skip the flattening (measured 0 / 2 / 4 / 8 / 16 / 32: cfg4 slab 19.2 / 18.8 / 18.4 / 18.2 / 18.5 / 18.8 ms, cfg2 1.58 / 1.57 / 1.55 / 1.55 / 1.56 / 1.58)
#endif
constexpr int kSlabDirect = RHG_SLAB_DIRECT;
#ifndef RHG_SLAB_DIRECT_LEAN
#define RHG_SLAB_DIRECT_LEAN 20 // the 40-register instance's cheaper direct loop (measured 8 / 12 / 16 / 20 / 28 / 40: cfg2 3.052 / 3.047 / 3.040 / 3.031 / 3.030 / 3.036 ms; cfg3 flat to 20, +0.1 % at 28)
#endif
constexpr int kSlabDirectLean = RHG_SLAB_DIRECT_LEAN;
constexpr double kPreMinS     = 4e-14;
constexpr unsigned long long kCntOne = 1ull << 42; // packed edge count unit (flattened pair loop) // groups whose windows give S below this skip the pre-filter

struct __align__(16) SlabRow32 { // one request with pairs in the slab (rows of a group are compacted)
    float         lamf;  // lambda_r - lam_first (float)
    float         m;     // coth_r - 1
    float         rcif;  // coshR / sinh r_r (the reference's rounded rci), float
    float         e1;    // tau coefficient of |Delta|
    float         c0;    // tau constant
    std::uint32_t qoff;  // request id - id base of its source annulus's owned block
    std::uint32_t pad;   // local node of pair t: pad + t (mod 2^32)
    std::uint32_t incl;  // inclusive prefix of the rows' pair counts
};
struct __align__(16) SlabRow64 { // the same request for the exact predicate
    double cs, sn, coth, rci;
};
// The exact-path node doubles (cos, sin), (coth, 1/sinh): staged in shared memory (R12), or
// read from the sorted arrays in global memory by the rare exact rechecks, which frees 16 KB
// per CTA for a fifth CTA per SM.
template <bool R12>
struct SlabNodes64 {
    double2 r1[kSlabNodes], r2[kSlabNodes];
};
template <>
struct SlabNodes64<false> {};
template <int NT, bool R12 = true>
struct SlabSmem : SlabNodes64<R12> {
    float4             nd[kSlab];         // (lambda - lam_first, coth - 1, 1 / sinh, id offset bits)
    double             lam[kSlab + 2];    // node lambdas from index `sh` (TMA needs 16-byte alignment)
    std::uint64_t      bar;               // completion of the slab's bulk copies
    std::uint16_t      bstart[kSlab + 1]; // bucket b: first local node with bucket(lambda) >= b
    SlabRow32          rows[NT / 32][32];
    SlabRow64          rows64[NT / 32][32];
    std::uint64_t      run_r0[64];        // compacted non-empty sources of the slab
    std::uint32_t      run_g[65];         // group prefix over the compacted sources
    std::uint8_t       run_a[64];
    std::uint32_t      n_run;
};

template <int MODE, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) slab_kernel(EdgeArgs A) {
    constexpr int kSlabThreads = NT;
    extern __shared__ __align__(16) unsigned char slab_raw[];
    constexpr bool           kR12 = MINB < 5; // exact-path node doubles in shared memory
    constexpr bool           kLean = !kR12;   // the 40-register instance (register-saving code forms)
    SlabSmem<NT, kR12>&      S    = *reinterpret_cast<SlabSmem<NT, kR12>*>(slab_raw);
    const int                lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned long long sl   = A.slab_tab[A.slab0 + blockIdx.x]; // (j << 32) | slab index in j, angle order per wave
    const int                j    = int(sl >> 32);
    const AnnulusDev&        Aj   = A.ann[j];
    const std::uint64_t      N0   = Aj.off + (sl & 0xffffffffull) * kSlab;
    const std::uint32_t      m    = std::uint32_t(Aj.halo - N0 < std::uint64_t(kSlab) ? Aj.halo - N0 : kSlab);
    const std::uint64_t      base_j = Aj.off + std::uint64_t(Aj.dlt0); // owned ids of j: [base_j, base_j + n)
    auto node_r1 = [&](std::uint32_t k) {
        if constexpr (kR12) return S.r1[k];
        else return A.s_rec1[N0 + k];
    };
    auto node_r2 = [&](std::uint32_t k) {
        if constexpr (kR12) return S.r2[k];
        else return A.s_rec2[N0 + k];
    };
    // The slab's node data arrive by TMA bulk copies (one elected thread, completion on an
    // mbarrier) into shared memory: lambda into its final place, (coth, 1/sinh) and ids into the
    // group-row buffers (free until the groups start), the exact-path doubles (R12) into place.
    // 8-byte arrays start at the even index N0 & ~1 (16-byte alignment): element i at [sh + i].
    const std::uint32_t sh   = std::uint32_t(N0 & 1u);
    const std::uint32_t n8   = (m + sh + 1u) & ~1u; // 8-byte elements copied (reads < s_lam + n_ext + 2)
    double2* const      st_r2 = [&]() -> double2* {
        if constexpr (kR12) return S.r2;
        else return reinterpret_cast<double2*>(&S.rows[0][0]);
    }();
    unsigned long long* const st_id = reinterpret_cast<unsigned long long*>(&S.rows64[0][0]);
    static_assert(sizeof(S.rows) >= kSlab * sizeof(double2) && sizeof(S.rows64) >= (kSlab + 2) * 8,
                  "the row buffers hold the staged node records");
    if (threadIdx.x == 0) {
        mbar_init(&S.bar, 1);
        const unsigned bytes = n8 * 8 * 2 + m * 16 * (kR12 ? 2 : 1);
        mbar_expect_tx(&S.bar, bytes);
        bulk_copy_g2s(S.lam, A.s_lam + (N0 - sh), n8 * 8, &S.bar);
        bulk_copy_g2s(st_id, A.s_id + (N0 - sh), n8 * 8, &S.bar);
        bulk_copy_g2s(st_r2, A.s_rec2 + N0, m * 16, &S.bar);
        if constexpr (kR12) bulk_copy_g2s(&S.r1[0], A.s_rec1 + N0, m * 16, &S.bar);
    }
    const double* const slam      = S.lam + sh;
    const double        lam_first = A.s_lam[N0];
    const double        lam_last  = A.s_lam[N0 + m - 1];
    // warp 0 finds the slab's request runs (cell-table lookups) while warps 1.. build the node
    // records and bucket starts from the staged data
    const double inv_w = lam_last > lam_first ? double(kSlab - 1) / (lam_last - lam_first) : 0.0;
    const float  span  = float(fsub(lam_last, lam_first)) * 1.0001f;
    __syncthreads(); // the mbarrier is initialised before anyone waits on it
    if (warp != 0) { // node records + bucket starts (cell_fill pattern)
        mbar_wait(&S.bar, 0);
        for (std::uint32_t i = threadIdx.x - 32; i < m; i += kSlabThreads - 32) {
            const double  l  = slam[i];
            const double  lp = i ? slam[i - 1] : 0.0;
            const double2 r2 = st_r2[i];
            S.nd[i]  = make_float4(float(fsub(l, lam_first)), float(fsub(r2.x, 1.0)), float(r2.y),
                                   __uint_as_float(std::uint32_t(st_id[sh + i] - base_j)));
            const std::uint32_t b  = slab_bucket(l, lam_first, inv_w);
            const std::int32_t  bp = i ? std::int32_t(slab_bucket(lp, lam_first, inv_w)) : -1;
            for (std::int32_t c = bp + 1; c <= std::int32_t(b); ++c) S.bstart[c] = std::uint16_t(i);
            if (i == m - 1)
                for (std::uint32_t c = b + 1; c <= kSlab; ++c) S.bstart[c] = std::uint16_t(m);
        }
    }
    // request runs of every sparse source annulus a <= j (lambda within hbound(a, j) of the
    // slab: a superset from a's cell table), compacted to the non-empty ones and numbered as
    // one CTA-wide list of 32-request groups shared by all warps
    else {
        const unsigned long long srcs = (A.ablate & 1) ? 0ull : A.src_mask[j]; // ablate: timing experiments only
        std::uint32_t            nrun = 0, gsum = 0;
        for (int a0 = 0; a0 <= j; a0 += 32) {
            const int     a  = a0 + lane;
            std::uint64_t r0 = 0, r1 = 0;
            if (a <= j && ((srcs >> a) & 1ull)) {
                const AnnulusDev& Aa = A.ann[a];
                const double      hb = A.hbound[a * A.count + j];
                r0 = A.lcellstart[Aa.cell_off + cellf(Aa, lam_first - hb)];
                r1 = A.lcellstart[Aa.cell_off + cellf(Aa, lam_last + hb) + 1];
                if (a == j && r1 > Aa.wrap) r1 = Aa.wrap; // own annulus: unwrapped requests only
                if (a == j && r1 > N0) r1 = N0; // own requests inside the slab: the own pass below
                if (r1 < r0) r1 = r0;
            }
            const std::uint32_t ng = std::uint32_t((r1 - r0 + 31) / 32);
            const unsigned      nz = __ballot_sync(kFull, ng > 0);
            std::uint32_t       incl = ng;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const std::uint32_t x = __shfl_up_sync(kFull, incl, o);
                if (lane >= o) incl += x;
            }
            if (ng) {
                const std::uint32_t r = nrun + __popc(nz & ((1u << lane) - 1u));
                S.run_r0[r] = r0, S.run_a[r] = std::uint8_t(a), S.run_g[r + 1] = gsum + incl;
            }
            nrun += __popc(nz);
            gsum += __shfl_sync(kFull, incl, 31);
        }
        if (lane == 0) S.run_g[0] = 0, S.n_run = nrun;
    }
    __syncthreads();
    const std::uint32_t ngroups = S.run_g[S.n_run];
    // at the 40-register budget the compiler re-derives the shared window base (S2R SR_CgaCtaId)
    // inside the pair loop: an opaque copy keeps it in a register (measured cfg3 slab 8.22 ->
    // 8.01 ms; the 64-register exact-wave variant is faster without it: cfg4 16.6 vs 17.1)
    unsigned nd_base = smem_addr(&S.nd[0]);
    if constexpr (!kR12) asm volatile("mov.u32 %0, %0;" : "+r"(nd_base));
    auto node_rec = [&](std::uint32_t k) {
        if constexpr (kR12) return S.nd[k];
        else return lds128(nd_base + 16u * k);
    };
    SlabRow32* const    rows    = S.rows[warp];
    SlabRow64* const    rows64  = S.rows64[warp];
    std::uint32_t       acc_e = 0, acc_c = 0; // per-thread totals of one slab fit 32 bits
    unsigned long long  acc_fp = 0;
    unsigned long long  au_decided = 0, au_recheck = 0, au_exact = 0, au_disagree = 0, au_noise = 0; // MODE 3
    float               au_ratio = 0.0f;
    int ri = 0; // run of group gi: last ri with run_g[ri] <= gi (gi only grows)
    // ---- own pass: requests of the target annulus inside the slab (p = N0 + i, unwrapped). Their
    // pairs are the slab nodes after them up to lower_bound(beta + 2 hw) (the requests before the
    // slab run through the groups below). Everything but (beta, hw) is staged, so a request costs
    // two coalesced loads and a short scan; the pairs of all requests are then flattened over the
    // whole CTA (one packed prefix sum also compacts the requests with pairs), so every thread
    // gets the same share.
    {
        const std::uint32_t wl  = std::uint32_t(Aj.wrap > N0 ? (Aj.wrap - N0 < m ? Aj.wrap - N0 : m) : 0);
        const bool          on  = ((A.src_mask[j] >> j) & 1ull) && !(A.ablate & 5);
        const std::uint32_t nrq = on ? wl : 0u; // requests p < min(wrap, halo)
        static_assert(2 * kSlabThreads >= kSlab, "two requests per thread cover the slab");
        std::uint32_t len[2] = {0u, 0u};
        bool          fpw[2] = {false, false};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const std::uint32_t i = 2 * threadIdx.x + h;
            if (i < nrq) {
                const double  b  = A.s_beta[N0 + i], hw = A.s_hw[N0 + i];
                const double  hi = fadd(b, fmul(2.0, hw));
                std::uint32_t k  = i + 1;
#pragma unroll 1
                for (int it = 0; it < 4 && k < m && slam[k] < hi; ++it) ++k;
                if (k < m && slam[k] < hi) k = slab_lb(S, slam, hi, lam_first, inv_w);
                const std::uint32_t l1 = k < wl ? k : wl;
                len[h] = l1 > i + 1 ? l1 - (i + 1) : 0u;
                fpw[h] = 0.5 * hw * hw < kPreMinS;
            }
        }
        // packed inclusive scan: pairs << 10 | requests with pairs (<= 130816 pairs, <= 512 requests)
        __shared__ std::uint32_t wsum[kSlabThreads / 32];
        const std::uint32_t      x0 = (len[0] << 10) + (len[0] > 0) + (len[1] << 10) + (len[1] > 0);
        std::uint32_t            x  = x0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const std::uint32_t y = __shfl_up_sync(kFull, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[warp] = x;
        __syncthreads();
        std::uint32_t wb = 0, X = 0;
#pragma unroll
        for (int w = 0; w < kSlabThreads / 32; ++w) wb += w < warp ? wsum[w] : 0u, X += wsum[w];
        // compacted request table in the staged-id buffer (free once the node records exist):
        // (inclusive pair prefix, node of pair t = pad + t, float rci, request | fp64 flag << 31)
        uint4* const  crow = reinterpret_cast<uint4*>(st_id);
        static_assert(sizeof(S.rows64) >= kSlab * sizeof(uint4), "the compacted requests fit the row buffer");
        std::uint32_t pe = (wb + x - x0) >> 10, ce = (wb + x - x0) & 1023u;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const std::uint32_t i = 2 * threadIdx.x + h;
            if (len[h]) {
                const float rcif = float(fmul(A.cosh_R, st_r2[i].y));
                crow[ce] = make_uint4(pe + len[h], i + 1 - pe, __float_as_uint(rcif), i | (fpw[h] ? 0x80000000u : 0u));
                pe += len[h], ++ce;
            }
        }
        __syncthreads();
        const std::uint32_t T = X >> 10, nne = X & 1023u;
        acc_c += threadIdx.x == 0 ? T : 0u;
        const std::uint32_t c  = ((T + kSlabThreads - 1) / kSlabThreads) | 1u;
        std::uint32_t       t  = threadIdx.x * c;
        const std::uint32_t te = t + c < T ? t + c : T;
        if (t < te && !(A.ablate & 2)) {
            std::uint32_t o = 0, ho = nne - 1; // first request whose inclusive prefix exceeds t
            while (o < ho) {
                const std::uint32_t mid = (o + ho) >> 1;
                if (crow[mid].x > t) ho = mid;
                else o = mid + 1;
            }
            // 40-register instance (kLean): the request table's address in a register, and tau
            // coefficients for the whole pass -- the requests lie inside the slab, |lamf| <= span, so the
            // per-request bound ed(|lamf| + span) is at most ed(2 span) (a larger tau only sends more pairs
            // to the exact predicate); recomputing them per request cost 14 divergent instructions on
            // every request change there. The 64-register instance keeps per-request coefficients
            // (measured: the lean form costs it 0.8 ms at cfg4).
            unsigned cb = smem_addr(crow);
            if constexpr (kLean) asm volatile("mov.u32 %0, %0;" : "+r"(cb));
            auto   crow_at = [&](std::uint32_t r) {
                if constexpr (kLean) return lds128u(cb + 16u * r);
                else return crow[r];
            };
            uint4  cr = crow_at(o);
            float4 qr = node_rec(cr.w & 0x7fffffffu); // (lamf, m, 1 / sinh, id offset) of the request
            float  e1f, c0f;
            auto   tau_coef = [&]() {
                const float ed = 5.9604645e-8f * ((kLean ? 2.0f * span : fabsf(qr.x) + span)) + 1.5e-15f;
                e1f = 1.3f * ed + 3e-15f, c0f = 1.3f * ed * ed + 2e-15f;
            };
            tau_coef();
            // the reference predicate for request i, node k (request doubles: staged or global)
            auto d64 = [&](std::uint32_t i, std::uint32_t k, double& lhs, double& rhs) {
                const double2 q1 = [&]() {
                    if constexpr (kR12) return S.r1[i];
                    else return A.s_rec1[N0 + i];
                }();
                const double2 q2 = st_r2[i], n1 = node_r1(k), n2 = st_r2[k];
                lhs = fadd(fmul(q1.x, n1.x), fmul(q1.y, n1.y));
                rhs = fsub(fmul(q2.x, n2.x), fmul(fmul(A.cosh_R, q2.y), n2.y));
            };
            std::uint32_t      cnt = 0;
            unsigned long long sum = 0;
            for (; t < te; ++t) {
                if (t >= cr.x) { // next request (compacted: every entry has pairs)
                    cr = crow_at(++o);
                    qr = node_rec(cr.w & 0x7fffffffu);
                    if constexpr (!kLean) tau_coef();
                }
                const std::uint32_t i  = cr.w & 0x7fffffffu;
                const std::uint32_t k  = cr.y + t;
                const float4        nd = node_rec(k);
                bool                e;
                if (cr.w >> 31) { // window below the pre-filter's floor: exact predicate only
                    double lhs, rhs;
                    d64(i, k, lhs, rhs);
                    e = lhs > rhs;
                    if constexpr (MODE == 3) ++au_exact, au_noise += fabs(fsub(lhs, rhs)) < 1e-15;
                } else {
                    const float df  = nd.x - qr.x;
                    const float y2  = df * df;
                    const float Sv  = y2 * fmaf(y2, -1.0f / 24.0f, 0.5f);
                    const float P   = __uint_as_float(cr.z) * nd.z;
                    const float M   = fmaf(qr.y, nd.y, qr.y + nd.y) + Sv;
                    const float D   = P - M;
                    const float tau = fmaf(fabsf(df), e1f, fmaf(P + M, 1.4e-6f, c0f));
                    e                    = D > 0.0f;
                    const bool undecided = !(fabsf(D) > tau) || fabsf(df) > kPreMaxDelta;
                    if (undecided || MODE == 3) {
                        double lhs, rhs;
                        d64(i, k, lhs, rhs);
                        if constexpr (MODE == 3) { // audit: every pre-filter decision against the reference predicate
                            if (undecided) ++au_recheck;
                            else {
                                ++au_decided;
                                au_disagree += e != (lhs > rhs);
                                au_ratio = fmaxf(au_ratio, float(fabs(double(D) - fsub(lhs, rhs))) / tau);
                            }
                            au_noise += fabs(fsub(lhs, rhs)) < 1e-15;
                        }
                        if (undecided) e = lhs > rhs;
                    }
                }
                if constexpr (MODE == 0 && kLean) { // counters-only kernel: the edge count rides in bits 42..
                    // of the id sum (a thread runs <= 512 pairs here: id sums < 2^41), one predicated add
                    const std::uint32_t nid = __float_as_uint(nd.w), qid = __float_as_uint(qr.w);
                    if (e) sum += static_cast<unsigned long long>(nid + qid) + kCntOne;
                } else if constexpr (MODE == 0) { // branch-free accumulation
                    const std::uint32_t nid = __float_as_uint(nd.w), qid = __float_as_uint(qr.w);
                    sum += e ? static_cast<unsigned long long>(nid + qid) : 0ull;
                    cnt += e;
                } else if (e) {
                    const std::uint32_t nid = __float_as_uint(nd.w), qid = __float_as_uint(qr.w);
                    sum += nid + qid, ++cnt;
                    if (MODE == 1) atomicAdd(&A.degrees[base_j + qid], 1u), atomicAdd(&A.degrees[base_j + nid], 1u);
                    if (MODE == 2) emit_edge(A, base_j + qid, base_j + nid);
                }
            }
            if constexpr (MODE == 0 && kLean) cnt = std::uint32_t(sum >> 42), sum &= kCntOne - 1;
            acc_e += cnt;
            acc_fp += sum + static_cast<unsigned long long>(cnt) * (2 * base_j);
        }
        __syncthreads(); // the group rows below overwrite the staged (coth, 1/sinh) buffer
    }
    for (std::uint32_t gi = warp; gi < ngroups; gi += kSlabThreads / 32) {
        while (S.run_g[ri + 1] <= gi) ++ri;
        const int           a   = S.run_a[ri];
        const AnnulusDev&   Aa  = A.ann[a];
        const bool          own = a == j;
        if ((A.ablate & 4) && own) continue; // timing experiments only
        if ((A.ablate & 8) && !own) continue;
        const std::uint64_t g    = S.run_r0[ri] + std::uint64_t(gi - S.run_g[ri]) * 32;
        const std::uint64_t R1   = S.run_r0[ri] + std::uint64_t(S.run_g[ri + 1] - S.run_g[ri]) * 32; // group end bound
        const std::uint64_t Rend = own ? (Aa.wrap < N0 ? Aa.wrap : N0) : Aa.halo; // own: requests before the slab
        const std::uint64_t p     = g + std::uint64_t(lane);
        const bool          valid = p < R1 && p < Rend;
        const std::uint64_t pc    = valid ? p : g;
        const double2       r2  = A.s_rec2[pc];
        const double        lam = A.s_lam[pc];
        double        lo = 0.0, hi = 0.0, hw_own = 0.0, h_oth = 0.0;
        std::uint32_t l0 = 0, l1 = 0;
        if (own) {
            const double b = A.s_beta[pc], hw = A.s_hw[pc];
            lo = b, hi = fadd(b, fmul(2.0, hw)), hw_own = hw;
            if (valid && hi > lo && hi > lam_first && lo <= lam_last) {
                // own window (requests before the slab): the slab's nodes up to lower_bound(beta + 2 hw):
                // a short linear scan covers the narrow windows of the outer annuli, the bucket search
                // the rest (measured slab ms: cfg2 1.49 -> 1.47, cfg4 16.6 -> 16.0, cfg5 78.3 -> 76.9)
                const std::uint32_t wl = std::uint32_t(Aa.wrap > N0 ? (Aa.wrap - N0 < m ? Aa.wrap - N0 : m) : 0);
                std::uint32_t       k  = 0;
#pragma unroll 1
                for (int it = 0; it < 4 && k < m && slam[k] < hi; ++it) ++k;
                if (k < m && slam[k] < hi) k = slab_lb(S, slam, hi, lam_first, inv_w);
                l1 = k < wl ? k : wl;
            }
        } else if (valid) {
            // window half-width in j (sweep.hpp:60-67, 365-370): h = acos(arg), arg rounded as the
            // reference does. For arg in [1/2, 1) a float estimate hf = 2 asin(sqrt((1 - arg) / 2))
            // (1 - arg exact) is within 1e-6 of glibc's acos relatively; the window ends are
            // bracketed with a 1e-5 margin and glibc's acos runs only when a slab node falls inside
            // a bracket (the exact ends could then differ from the estimate's).
            double arg = 0.0, h = kPiD;
            bool   fast = false;
            if (Aj.lower > 0.0) {
                arg = fsub(fmul(r2.x, Aj.coth_lower), fmul(Aj.cris, r2.y));
                if (arg >= 1.0) h = 0.0;
                else if (arg > -1.0) {
                    fast = arg >= 0.5 && fsub(1.0, arg) >= 1e-30;
                    if (!fast) h = gl::gl_acos(arg);
                }
            }
            if (fast) {
                const float  hf = 2.0f * asinf(sqrtf(float(fsub(1.0, arg)) * 0.5f));
                const double hl = fmul(double(hf), 1.0 - 1e-5), hh = fmul(double(hf), 1.0 + 1e-5);
                const double lo_a = fsub(lam, hh), lo_b = fsub(lam, hl), hi_a = fadd(lam, hl), hi_b = fadd(lam, hh);
                h_oth = hf;
                if (hi_b > lam_first && lo_a <= lam_last) {
                    l0 = slab_lb(S, slam, lo_a, lam_first, inv_w), l1 = slab_lb(S, slam, hi_a, lam_first, inv_w);
                    if ((l0 < m && slam[l0] < lo_b) || (l1 < m && slam[l1] < hi_b)) fast = false, h = gl::gl_acos(arg);
                }
            }
            if (!fast) {
                lo = fsub(lam, h), hi = fadd(lam, h), h_oth = h;
                l0 = l1 = 0;
                if (hi > lo && hi > lam_first && lo <= lam_last)
                    l0 = slab_lb(S, slam, lo, lam_first, inv_w), l1 = slab_lb(S, slam, hi, lam_first, inv_w);
            }
        }
        const std::uint32_t len = l1 > l0 ? l1 - l0 : 0u;
        const unsigned      nz  = __ballot_sync(kFull, len > 0);
        // the pre-filter decides a pair only when its distance term S = 1 - cos(dtheta) is
        // well above the FP64 rounding floor (~2e-15); groups with windows narrower than
        // that (outer annuli at R >~ 33) run the exact FP64 predicate directly
        const double        hwin = own ? hw_own : h_oth;
        const bool          fp64 = __any_sync(kFull, len > 0 && 0.5 * hwin * hwin < kPreMinS);
        if (A.dbg) { // slab-join path statistics (RHG_DEBUG_STATS=1)
            const unsigned nv = __popc(__ballot_sync(kFull, valid));
            const unsigned sl = __reduce_add_sync(kFull, len);
            if (lane == 0)
                atomicAdd(&A.dbg[10], 1ull), atomicAdd(&A.dbg[11], (unsigned long long)nv),
                    atomicAdd(&A.dbg[12], (unsigned long long)__popc(nz)), atomicAdd(&A.dbg[own ? 15 : 16], 1ull),
                    atomicAdd(&A.dbg[own ? 18 : 21], (unsigned long long)nv),
                    atomicAdd(&A.dbg[own ? 19 : 22], (unsigned long long)__popc(nz)),
                    atomicAdd(&A.dbg[own ? 20 : 23], (unsigned long long)sl);
        }
        if (nz == 0) continue;
        // narrow windows (every lane <= kSlabDirect pairs): each lane tests its own pairs with
        // its request in registers -- no prefix sum, row table or row search
        if (MODE != 3 && !(A.ablate & 2) && __reduce_max_sync(kFull, len) <= std::uint32_t(kLean ? kSlabDirectLean : kSlabDirect)) {
            acc_c += len;
            if (kLean && len) {
                const unsigned long long idp = A.s_id[pc];
                std::uint32_t            cnt = 0;
                unsigned long long       sum = 0; // node-id offsets from base_j
                // the exact predicate of request pc and node k; the request's doubles are re-read
                // (L1/L2) rather than held across the loop: at the 40-register budget holding them
                // made the compiler re-derive the float request terms on every pair
                auto exact = [&](std::uint32_t k) {
                    const double2 q1 = A.s_rec1[pc], q2 = A.s_rec2[pc];
                    return edge_test(q1.x, q1.y, q2.x, fmul(A.cosh_R, q2.y), node_r1(k), node_r2(k));
                };
                auto count = [&](bool e, float ndw) {
                    if constexpr (MODE == 0) { // the edge count rides in bits 42.. of the sum (<= 8 pairs)
                        if (e) sum += static_cast<unsigned long long>(__float_as_uint(ndw)) + kCntOne;
                    } else if (e) {
                        const unsigned long long nid = base_j + __float_as_uint(ndw);
                        sum += __float_as_uint(ndw), ++cnt;
                        if (MODE == 1) atomicAdd(&A.degrees[idp], 1u), atomicAdd(&A.degrees[nid], 1u);
                        if (MODE == 2) emit_edge(A, idp, nid);
                    }
                };
                if (fp64) { // every pair exact (request doubles re-read: measured faster here, cfg2 3.10 -> 3.07 ms)
                    for (std::uint32_t k = l0; k < l1; ++k) count(exact(k), node_rec(k).w);
                } else {
                    const float lamf = float(fsub(lam, lam_first));
                    const float ed   = 5.9604645e-8f * (fabsf(lamf) + span) + 1.5e-15f;
                    const float qm = float(fsub(r2.x, 1.0)), qr = float(fmul(A.cosh_R, r2.y));
                    const float e1 = 1.3f * ed + 3e-15f, c0 = 1.3f * ed * ed + 2e-15f;
                    for (std::uint32_t k = l0; k < l1; ++k) {
                        const float4 nd  = node_rec(k);
                        const float  df  = nd.x - lamf;
                        const float  y2  = df * df;
                        const float  Sv  = y2 * fmaf(y2, -1.0f / 24.0f, 0.5f);
                        const float  P   = qr * nd.z;
                        const float  M   = fmaf(qm, nd.y, qm + nd.y) + Sv;
                        const float  D   = P - M;
                        const float  tau = fmaf(fabsf(df), e1, fmaf(P + M, 1.4e-6f, c0));
                        bool         e   = D > 0.0f;
                        if (!(fabsf(D) > tau) || fabsf(df) > kPreMaxDelta) e = exact(k);
                        count(e, nd.w);
                    }
                }
                if constexpr (MODE == 0) cnt = std::uint32_t(sum >> 42), sum &= kCntOne - 1;
                acc_e += cnt, acc_fp += sum + static_cast<unsigned long long>(cnt) * (base_j + idp);
            }
            // the 64-register instance: the request in registers (its base form measured faster there)
            if (!kLean && len) {
                const double2            r1  = A.s_rec1[pc];
                const double             rci = fmul(A.cosh_R, r2.y);
                const unsigned long long idp = A.s_id[pc];
                const std::uint64_t      base_j_ = base_j;
                std::uint32_t            cnt = 0;
                unsigned long long       sum = 0;
                const float              lamf = float(fsub(lam, lam_first));
                const float              ed   = 5.9604645e-8f * (fabsf(lamf) + span) + 1.5e-15f;
                const float              qm = float(fsub(r2.x, 1.0)), qr = float(rci);
                for (std::uint32_t k = l0; k < l1; ++k) {
                    const float4 nd = node_rec(k);
                    bool         e;
                    if (fp64) e = edge_test(r1.x, r1.y, r2.x, rci, node_r1(k), node_r2(k));
                    else {
                        const float df  = nd.x - lamf;
                        const float y2  = df * df;
                        const float Sv  = y2 * fmaf(y2, -1.0f / 24.0f, 0.5f);
                        const float P   = qr * nd.z;
                        const float M   = fmaf(qm, nd.y, qm + nd.y) + Sv;
                        const float D   = P - M;
                        const float tau = fmaf(fabsf(df), 1.3f * ed + 3e-15f, fmaf(P + M, 1.4e-6f, 1.3f * ed * ed + 2e-15f));
                        e = D > 0.0f;
                        if (!(fabsf(D) > tau) || fabsf(df) > kPreMaxDelta)
                            e = edge_test(r1.x, r1.y, r2.x, rci, node_r1(k), node_r2(k));
                    }
                    if constexpr (MODE == 0) { // branch-free accumulation (the counters-only kernel)
                        sum += e ? base_j_ + __float_as_uint(nd.w) + idp : 0ull;
                        cnt += e;
                    } else if (e) {
                        const unsigned long long nid = base_j_ + __float_as_uint(nd.w);
                        sum += nid + idp, ++cnt;
                        if (MODE == 1) atomicAdd(&A.degrees[idp], 1u), atomicAdd(&A.degrees[nid], 1u);
                        if (MODE == 2) emit_edge(A, idp, nid);
                    }
                }
                acc_e += cnt, acc_fp += sum;
            }
            continue;
        }
        // flattened pair list over the warp: pair t belongs to the row whose prefix covers it
        std::uint32_t incl = len;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const std::uint32_t x = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += x;
        }
        const std::uint32_t T  = __shfl_sync(kFull, incl, 31);
        const std::uint32_t nr = __popc(nz);
        acc_c += len;
        if (A.dbg && lane == 0) atomicAdd(&A.dbg[13], (unsigned long long)T), atomicAdd(&A.dbg[14], 32ull * (((T + 31) >> 5) | 1u));
        if (A.ablate & 2) continue;
        const std::uint64_t base_a = Aa.off + std::uint64_t(Aa.dlt0);
        __syncwarp();
        if (len) {
            const double2 r1  = A.s_rec1[pc];
            const double  rci = fmul(A.cosh_R, r2.y);
            const int     w   = __popc(nz & ((1u << lane) - 1u));
            rows64[w]         = SlabRow64{r1.x, r1.y, r2.x, rci};
            const float lamf  = float(fsub(lam, lam_first));
            const float ed    = 5.9604645e-8f * (fabsf(lamf) + span) + 1.5e-15f;
            SlabRow32 R;
            R.lamf = lamf, R.m = float(fsub(r2.x, 1.0)), R.rcif = float(rci);
            R.e1 = 1.3f * ed + 3e-15f, R.c0 = 1.3f * ed * ed + 2e-15f;
            R.qoff = std::uint32_t(A.s_id[pc] - base_a), R.pad = l0 - (incl - len), R.incl = incl;
            rows[w] = R;
        }
        __syncwarp();
        // lane L runs the contiguous pairs [L c, (L + 1) c) of the warp's sequence: its request
        // stays in registers until the owner changes (one step: rows are non-empty), node
        // records (16 B) come from shared memory.  Edge ids are summed as 32-bit offsets from
        // the two annuli's id bases, rebased once per group.
        const std::uint32_t c  = ((T + 31) >> 5) | 1u; // odd: lane starts fall in distinct smem banks
        std::uint32_t       t  = std::uint32_t(lane) * c;
        const std::uint32_t te = t + c < T ? t + c : T;
        if (t < te) {
            std::uint32_t o = 0, ho = nr - 1; // first row whose inclusive prefix exceeds t
            while (o < ho) {
                const std::uint32_t mid = (o + ho) >> 1;
                if (rows[mid].incl > t) ho = mid;
                else o = mid + 1;
            }
            // row o: floats at rb + 32 o, words at rb + 32 o + 16. In the 40-register instance the warp's
            // row-table address is kept in a register (opaque copy): re-deriving it on every row change
            // (S2R SR_CgaCtaId + 8 instructions, divergent) cost 6 % of its instructions at cfg2
            unsigned rb = smem_addr(rows);
            if constexpr (kLean) asm volatile("mov.u32 %0, %0;" : "+r"(rb));
            const float4* rf = reinterpret_cast<const float4*>(rows);
            const uint4*  ru = reinterpret_cast<const uint4*>(rows);
            auto row_f = [&](std::uint32_t r) {
                if constexpr (kLean) return lds128(rb + 32u * r);
                else return rf[2 * r];
            };
            auto row_u = [&](std::uint32_t r) {
                if constexpr (kLean) return lds128u(rb + 32u * r + 16u);
                else return ru[2 * r + 1];
            };
            float4        q  = row_f(o); // (lamf, m, rcif, e1)
            uint4         u  = row_u(o); // (c0 bits, qoff, pad, incl)
            std::uint32_t cnt = 0;
            unsigned long long sum = 0;
            if (!fp64) {
                for (; t < te; ++t) {
                    if (t >= u.w) { // next row
                        ++o;
                        q = row_f(o), u = row_u(o);
                    }
                    const std::uint32_t k  = u.z + t;
                    const float4        nd = node_rec(k);
                    const float         df = nd.x - q.x;
                    const float         y2 = df * df;
                    const float         Sv = y2 * fmaf(y2, -1.0f / 24.0f, 0.5f);
                    const float         P  = q.z * nd.z;
                    const float         M  = fmaf(q.y, nd.y, q.y + nd.y) + Sv;
                    const float         D  = P - M;
                    const float         tau = fmaf(fabsf(df), q.w, fmaf(P + M, 1.4e-6f, __uint_as_float(u.x)));
                    bool                e  = D > 0.0f;
                    const bool          undecided = !(fabsf(D) > tau) || fabsf(df) > kPreMaxDelta;
                    if constexpr (MODE == 3) { // audit: every pre-filter decision against the reference predicate
                        const SlabRow64& R   = rows64[o];
                        const double2    n1  = node_r1(k), n2 = node_r2(k);
                        const double     lhs = fadd(fmul(R.cs, n1.x), fmul(R.sn, n1.y));
                        const double     rhs = fsub(fmul(R.coth, n2.x), fmul(R.rci, n2.y));
                        const double     d64 = fsub(lhs, rhs);
                        if (undecided) ++au_recheck;
                        else {
                            ++au_decided;
                            au_disagree += e != (lhs > rhs);
                            au_ratio = fmaxf(au_ratio, float(fabs(double(D) - d64)) / tau);
                        }
                        au_noise += fabs(d64) < 1e-15;
                    }
                    if (undecided) { // near the threshold: exact FP64
                        const SlabRow64& R = rows64[o];
                        e = edge_test(R.cs, R.sn, R.coth, R.rci, node_r1(k), node_r2(k));
                        if (A.dbg) atomicAdd(&A.dbg[17], 1ull);
                    }
                    if constexpr (MODE == 0 && kLean) { // counters-only kernel: the edge count rides in bits 42..
                        // of the id sum (a lane runs <= 513 pairs of a group: id sums < 2^41), one predicated add
                        const std::uint32_t nid = __float_as_uint(nd.w);
                        if (e) sum += static_cast<unsigned long long>(nid + u.y) + kCntOne; // < 2^32: a shard holds < 2^31 points
                    } else if constexpr (MODE == 0) { // branch-free accumulation
                        const std::uint32_t nid = __float_as_uint(nd.w);
                        sum += e ? static_cast<unsigned long long>(nid + u.y) : 0ull;
                        cnt += e;
                    } else if (e) {
                        const std::uint32_t nid = __float_as_uint(nd.w);
                        sum += nid + u.y, ++cnt;
                        if (MODE == 1) {
                            atomicAdd(&A.degrees[base_a + u.y], 1u);
                            atomicAdd(&A.degrees[base_j + nid], 1u);
                        }
                        if (MODE == 2) emit_edge(A, base_a + u.y, base_j + nid);
                    }
                }
                if constexpr (MODE == 0 && kLean) cnt = std::uint32_t(sum >> 42), sum &= kCntOne - 1;
            } else { // windows so narrow that the FP64 rounding noise dominates: exact predicate only
                const double2* r64 = reinterpret_cast<const double2*>(rows64);
                double2        q0 = r64[2 * o], q1 = r64[2 * o + 1]; // (cs, sn), (coth, rci)
                for (; t < te; ++t) {
                    if (t >= u.w) { // next row
                        ++o;
                        q0 = r64[2 * o], q1 = r64[2 * o + 1], u = ru[2 * o + 1];
                    }
                    const std::uint32_t k = u.z + t;
                    if constexpr (MODE == 3) {
                        const double2 n1 = node_r1(k), n2 = node_r2(k);
                        ++au_exact;
                        au_noise += fabs(fsub(fadd(fmul(q0.x, n1.x), fmul(q0.y, n1.y)),
                                              fsub(fmul(q1.x, n2.x), fmul(q1.y, n2.y)))) < 1e-15;
                    }
                    if (edge_test(q0.x, q0.y, q1.x, q1.y, node_r1(k), node_r2(k))) {
                        const std::uint32_t nid = __float_as_uint(S.nd[k].w);
                        sum += nid + u.y, ++cnt;
                        if (MODE == 1) {
                            atomicAdd(&A.degrees[base_a + u.y], 1u);
                            atomicAdd(&A.degrees[base_j + nid], 1u);
                        }
                        if (MODE == 2) emit_edge(A, base_a + u.y, base_j + nid);
                    }
                }
            }
            acc_e += cnt;
            acc_fp += sum + static_cast<unsigned long long>(cnt) * (base_a + base_j);
        }
        __syncwarp();
    }
    Acc acc;
    acc.edges = acc_e, acc.comps = acc_c, acc.fp = acc_fp;
    flush<MODE == 1 || MODE == 2>(acc, A, 0, lane, j);
    if constexpr (MODE == 3) {
        if (au_decided) atomicAdd(&A.audit[0], au_decided);
        if (au_recheck) atomicAdd(&A.audit[1], au_recheck);
        if (au_exact) atomicAdd(&A.audit[2], au_exact);
        if (au_disagree) atomicAdd(&A.audit[3], au_disagree);
        if (au_ratio > 0.0f) atomicMax(&A.audit[4], static_cast<unsigned long long>(__float_as_uint(au_ratio)));
        if (au_noise) atomicAdd(&A.audit[5], au_noise);
    }
}

// Pairs the slab join leaves out: halo requests (Foreign replica) x owned
// nodes, owned requests x halo nodes, and own-annulus pairs with a wrapped
// request or node (full (theta, id) dedup, sweep.hpp:517-526).  Only the
// requests near the end of the owned block (lambda >= tail_lam(a)) and the
// halo requests can have such pairs; thread = one of them, all its sparse targets.
template <int MODE>
__global__ void __launch_bounds__(256) tail_kernel(EdgeArgs A) {
    const std::uint64_t t  = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    Acc                 acc;
    __shared__ AnnAcc   SA;
    ann_zero<MODE != 0>(SA);
    __syncthreads();
    if (t < A.tail_prefix[A.count]) {
        int a = A.first_streaming, ha = A.count - 1; // last annulus with tail_prefix <= t
        while (a < ha) {
            const int mid = (a + ha + 1) >> 1;
            if (A.tail_prefix[mid] <= t) a = mid;
            else ha = mid - 1;
        }
        const AnnulusDev&   Aa = A.ann[a];
        const std::uint64_t n  = A.tail_prefix[a + 1] - A.tail_prefix[a];
        const std::uint64_t p  = Aa.end - n + (t - A.tail_prefix[a]); // [halo - owned tail, end)
        const bool          halo_req = p >= Aa.halo;
        const double        lam = A.s_lam[p];
        if (halo_req || lam >= A.tail_lam[a]) {
            const double2 r1 = A.s_rec1[p], r2 = A.s_rec2[p];
            SRow          q;
            q.cs = r1.x, q.sn = r1.y, q.coth = r2.x, q.rci = fmul(A.cosh_R, r2.y), q.id = A.s_id[p], q.pad = 0;
            const double             theta = theta_of(A, p, lift_from(A, Aa));
            const unsigned long long srcm  = ~A.dense_mask[a];
            for (int j = a; j < A.count; ++j) {
                const AnnulusDev& Aj = A.ann[j];
                if (Aj.end == Aj.off || !((srcm >> j) & 1ull)) continue;
                // a halo request tests owned nodes only: skip targets whose owned block ends before
                // the request's window can begin (host bound on the half-width; no acos needed)
                if (halo_req && (Aj.halo == Aj.off || fsub(lam, A.hbound[a * A.count + j]) > A.s_lam[Aj.halo - 1]))
                    continue;
                const bool own = j == a;
                double     lo, hi;
                if (own) {
                    const double b = A.s_beta[p], hw = A.s_hw[p];
                    lo = b, hi = fadd(b, fmul(2.0, hw));
                } else {
                    const double h = half_width_in(Aj, r2.x, r2.y);
                    lo = fsub(lam, h), hi = fadd(lam, h);
                }
                if (!(hi > lo)) continue;
                const unsigned long long e0 = acc.edges, c0 = acc.comps;
                if (Aj.halo > Aj.off) {
                    std::uint64_t g0 = 0, g1 = 0;
                    if (halo_req) {
                        owned_range(A, Aj, lo, hi, g0, g1);
                    } else if (own) {
                        if (p >= Aa.wrap) owned_range(A, Aj, lo, hi, g0, g1);
                        else g0 = Aj.wrap, g1 = lower_bound_owned(A, Aj, hi); // wrapped nodes
                    }
                    if (g1 > g0) serial_range<MODE>(A, q, theta, own, g0, g1, lift_from(A, Aj), acc);
                }
                if (!halo_req && Aj.end > Aj.halo && hi > A.s_lam[Aj.halo] && lo <= A.s_lam[Aj.end - 1]) {
                    const std::uint64_t h0 = lower_bound_halo(A, Aj, lo), h1 = lower_bound_halo(A, Aj, hi);
                    if (h1 > h0) serial_range<MODE>(A, q, theta, own, h0, h1, lift_from(A, Aj), acc);
                }
                ann_add<MODE != 0>(SA, j, acc.edges - e0, acc.comps - c0);
            }
        }
    }
    flush(acc, A, 0, threadIdx.x & 31);
    __syncthreads();
    ann_flush<MODE != 0>(SA, A);
}

// --------------------------------------------------------- dense engine ---
// Requests with wide windows: every global point and the streaming requests
// of the (annulus, target) pairs whose windows hold >= ~32 nodes on average
// (host-chosen, A.dense_mask).  Unified request u: u < n_glob is global point
// u; otherwise annulus a's sorted request p = ann[a].off + (u - req_off[a]).

__device__ __forceinline__ int req_annulus(const EdgeArgs& A, std::uint64_t u) {
    int lo = A.first_streaming, hi = A.count - 1; // last annulus with req_off <= u
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (A.req_off[mid] <= u) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// Dense-engine request order: a counting sort by (segment, angle bucket), no general sort.
// Key of a request: (source, radial class, theta or lambda quantised to 32 bits); source 0 =
// global points, a - first_streaming + 1 = streaming annulus a; the class is the binary exponent
// of 1/sinh r halved, so the half-widths of one segment = (source, class) differ by at most ~2x.
// Segment c gets 2^lg >= max(64, size) angle buckets over [0, 2pi).  The node tiles only use
// bucket ranges (supersets; any order inside a bucket is exact: the rows carry exact index
// ranges), so the exclusive scan of the bucket counts IS the bucket table, and a per-bucket
// atomic cursor places every request (replaces a 48-bit radix sort, 6 passes).
__global__ void req_keys_kernel(EdgeArgs A, unsigned long long* keys) {
    const std::uint64_t u = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (u >= A.n_req) return;
    double   th, inv;
    unsigned src = 0;
    if (u < A.n_glob) {
        th = A.rec0[A.n_ext + u].y, inv = A.rec2[A.n_ext + u].y;
    } else {
        const int           a = req_annulus(A, u);
        const std::uint64_t p = A.ann[a].off + (u - A.req_off[a]);
        th = A.s_lam[p], inv = A.s_rec2[p].y;
        while (th >= kTwoPiD) th -= kTwoPiD;
        src = unsigned(a - A.first_streaming + 1);
    }
    const unsigned      cls = unsigned(static_cast<unsigned long long>(__double_as_longlong(inv)) >> 53) & 0x3ffu;
    const double        q   = th * (4294967296.0 / kTwoPiD);
    const std::uint32_t tq  = q >= 4294967295.0 ? 0xffffffffu : std::uint32_t(q);
    const unsigned      seg = (src << 10) | cls;
    keys[u]                 = (static_cast<unsigned long long>(seg) << 32) | tq;
    // segment sizes: consecutive requests share their segment, so one atomic per distinct
    // segment of the warp (per-request atomics on a few hot counters cost 9 ms at cfg3)
    const unsigned same = __match_any_sync(__activemask(), seg);
    if (int(threadIdx.x & 31) == __ffs(same) - 1) atomicAdd(&A.seg_first[seg], unsigned(__popc(same)));
}

// One block: the non-empty segments in id order -> dense index c, start position cseg[c]
// (exclusive prefix of the sizes), n_cls, and the bucket layout (bk_off, bk_shift).
__global__ void __launch_bounds__(1024) req_segments_kernel(EdgeArgs A, std::uint32_t* seg_index) {
    __shared__ int      wn[32];
    __shared__ unsigned ws[32];
    const int      lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const unsigned nseg = unsigned(A.count - A.first_streaming + 1) << 10;
    const unsigned per  = (nseg + 1023) / 1024; // thread t handles ids [t per, (t + 1) per)
    const unsigned i0   = threadIdx.x * per, i1 = i0 + per < nseg ? i0 + per : nseg;
    int            mine_n = 0;
    unsigned       mine_s = 0;
    for (unsigned i = i0; i < i1; ++i) {
        const unsigned c = A.seg_first[i];
        mine_n += c != 0u, mine_s += c;
    }
    int      in_n = mine_n;
    unsigned in_s = mine_s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int      x = __shfl_up_sync(kFull, in_n, o);
        const unsigned y = __shfl_up_sync(kFull, in_s, o);
        if (lane >= o) in_n += x, in_s += y;
    }
    if (lane == 31) wn[w] = in_n, ws[w] = in_s;
    __syncthreads();
    int      bn = 0, total = 0;
    unsigned bs = 0;
    for (int k = 0; k < 32; ++k) {
        bn += k < w ? wn[k] : 0, bs += k < w ? ws[k] : 0u;
        total += wn[k];
    }
    int      idx = bn + in_n - mine_n;
    unsigned pos = bs + in_s - mine_s;
    for (unsigned i = i0; i < i1; ++i) {
        const unsigned c = A.seg_first[i];
        if (!c) continue;
        seg_index[i] = unsigned(idx);
        if (idx < kMaxCls) A.cseg[idx] = pos;
        ++idx, pos += c;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const int n = total < kMaxCls ? total : kMaxCls; // overflow is checked on the host via n_cls
        A.cseg[n]   = std::uint32_t(A.n_req);
        *A.n_cls    = total;
        std::uint32_t off = 0;
        for (int c = 0; c < n; ++c) {
            const std::uint32_t sz = A.cseg[c + 1] - A.cseg[c];
            int                 lg = 6;
            while ((1u << lg) < sz && lg < 24) ++lg;
            A.bk_off[c]   = off;
            A.bk_shift[c] = std::uint32_t(32 - lg);
            off += (1u << lg) + 1; // the extra entry holds the segment end
        }
        A.bk_off[n] = off;
    }
}

__device__ __forceinline__ long long req_bucket(const EdgeArgs& A, unsigned long long key, const std::uint32_t* seg_index) {
    const unsigned c = seg_index[unsigned(key >> 32)];
    if (c >= unsigned(kMaxCls)) return -1;
    return (long long)(A.bk_off[c] + (std::uint32_t(key) >> A.bk_shift[c]));
}
__global__ void req_bucket_count_kernel(EdgeArgs A, const unsigned long long* keys, const std::uint32_t* seg_index,
                                        std::uint32_t* bcount) {
    const std::uint64_t u = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (u >= A.n_req) return;
    const long long g = req_bucket(A, keys[u], seg_index);
    if (g >= 0) atomicAdd(&bcount[g], 1u);
}
__global__ void req_scatter_kernel(EdgeArgs A, const unsigned long long* keys, const std::uint32_t* seg_index,
                                   std::uint32_t* cursor, std::uint32_t* perm) {
    const std::uint64_t u = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (u >= A.n_req) return;
    const long long g = req_bucket(A, keys[u], seg_index);
    if (g >= 0) perm[atomicAdd(&cursor[g], 1u)] = std::uint32_t(u);
}

// Exclusive scan of n u32 (three passes): 2048-entry blocks, their sums (one block), the add.
constexpr int kScanItems = 8;
__global__ void __launch_bounds__(256) scan_blocks_kernel(const std::uint32_t* in, std::uint32_t* out,
                                                          std::uint32_t* bsum, std::size_t n) {
    __shared__ std::uint32_t wsum[8];
    const int         lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const std::size_t i0   = (std::size_t(blockIdx.x) * 256 + threadIdx.x) * kScanItems;
    std::uint32_t     v[kScanItems], t = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) v[k] = i0 + k < n ? in[i0 + k] : 0u, t += v[k];
    std::uint32_t incl = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const std::uint32_t x = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += x;
    }
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    std::uint32_t before = 0, tot = 0;
    for (int k = 0; k < 8; ++k) before += k < w ? wsum[k] : 0u, tot += wsum[k];
    std::uint32_t run = before + incl - t;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k)
        if (i0 + k < n) out[i0 + k] = run, run += v[k];
    if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}
__global__ void __launch_bounds__(1024) scan_sums_kernel(std::uint32_t* bsum, unsigned nb) {
    __shared__ std::uint32_t wsum[32];
    const int      lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const unsigned per  = (nb + 1023) / 1024, i0 = threadIdx.x * per, i1 = i0 + per < nb ? i0 + per : nb;
    std::uint32_t  t = 0;
    for (unsigned i = i0; i < i1; ++i) t += bsum[i];
    std::uint32_t incl = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const std::uint32_t x = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += x;
    }
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    std::uint32_t before = 0;
    for (int k = 0; k < 32; ++k) before += k < w ? wsum[k] : 0u;
    std::uint32_t run = before + incl - t;
    for (unsigned i = i0; i < i1; ++i) {
        const std::uint32_t x = bsum[i];
        bsum[i]               = run, run += x;
    }
}
__global__ void scan_add_kernel(std::uint32_t* out, std::uint32_t* cursor, const std::uint32_t* bsum, std::size_t n) {
    const std::size_t i = std::size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const std::uint32_t v = out[i] + bsum[i / (256 * kScanItems)];
    out[i] = v, cursor[i] = v;
}

// Sorted copies of the dense-engine requests (one gather pass, so the rows
// and tile kernels read them coalesced): (cos, sin), (coth, coshR / sinh),
// 1 / sinh, id, unified index, and (lambda or theta, beta, hw, theta).
__global__ void req_gather_kernel(EdgeArgs A) {
    const std::uint64_t s = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (s >= A.n_req) return;
    const std::uint32_t u = A.gperm[s];
    double2             r1, r2;
    double4             ax;
    unsigned long long  id;
    if (u < A.n_glob) {
        const std::uint64_t g = A.n_ext + u;
        r1 = A.rec1[g], r2 = A.rec2[g];
        const double th = A.rec0[g].y;
        ax = make_double4(th, 0.0, 0.0, th), id = u;
    } else {
        const int           a = req_annulus(A, u);
        const std::uint64_t p = A.ann[a].off + (u - A.req_off[a]);
        r1 = A.s_rec1[p], r2 = A.s_rec2[p];
        const double lam = A.s_lam[p];
        ax = make_double4(lam, A.s_beta[p], A.s_hw[p], theta_of(A, p, lift_from(A, A.ann[a])));
        id = A.s_id[p];
    }
    A.g_rec[2 * s]     = r1;
    A.g_rec[2 * s + 1] = make_double2(r2.x, fmul(A.cosh_R, r2.y));
    A.g_inv[s]         = r2.y;
    A.g_id[s]          = std::uint32_t(id);
    A.g_u[s]           = u;
    A.g_aux[s]         = ax;
}

// Deferred node ranges of a sorted dense request s (dedup: same-annulus pair
// rule of sweep.hpp:517-526).  Full list: the range is dropped and counted in
// defer_ctr[1] (the host rejects the run; cap is sized to make that unreachable).
__device__ __forceinline__ void defer_range(const EdgeArgs& A, std::uint32_t s, std::uint64_t k0, std::uint64_t k1,
                                            bool dedup) {
    const unsigned long long i = atomicAdd(&A.defer_ctr[0], 1ull);
    if (i < A.defer_cap) A.deferred[i] = make_uint4(s, std::uint32_t(k0), std::uint32_t(k1), dedup ? 1u : 0u);
    else atomicAdd(&A.defer_ctr[1], 1ull);
}

// One warp per deferred range: lanes stride its nodes.
template <int MODE>
__global__ void __launch_bounds__(256) deferred_kernel(EdgeArgs A) {
    const int                lane = threadIdx.x & 31;
    const unsigned long long n    = A.defer_ctr[0] < A.defer_cap ? A.defer_ctr[0] : A.defer_cap;
    const unsigned long long nw   = (unsigned long long)(gridDim.x) * (blockDim.x >> 5);
    Acc                      acc;
    __shared__ AnnAcc        SA;
    ann_zero<MODE != 0>(SA);
    __syncthreads();
    for (unsigned long long i = (unsigned long long)(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n;
         i += nw) {
        const uint4   E  = A.deferred[i];
        const unsigned long long e0 = acc.edges, c0 = acc.comps;
        const double2 q1 = A.g_rec[2 * E.x], q2 = A.g_rec[2 * E.x + 1];
        SRow          q;
        q.cs = q1.x, q.sn = q1.y, q.coth = q2.x, q.rci = q2.y, q.id = A.g_id[E.x], q.pad = 0;
        const double theta = A.g_aux[E.x].w;
        int          j     = A.first_streaming; // the range's annulus: the one whose extended block holds node E.y
        for (int base = 0; base < A.count; base += 32) {
            const int      a = base + lane;
            const unsigned m = __ballot_sync(kFull, a < A.count && a >= A.first_streaming && A.ann[a].off <= E.y);
            if (m) j = base + 31 - __clz(m);
        }
        const std::uint64_t lift = lift_from(A, A.ann[j]);
        for (std::uint64_t k = E.y + std::uint64_t(lane); k < E.z; k += 32) {
            const unsigned long long nid = A.s_id[k];
            bool                     in  = true;
            if (E.w) {
                const double tq = theta_of(A, k, lift);
                in              = nid != q.id && (theta < tq || (theta == tq && q.id < nid));
            }
            if (!in) continue;
            acc.comps += 1;
            count_edge<MODE>(A, edge_test(q.cs, q.sn, q.coth, q.rci, A.s_rec1[k], A.s_rec2[k]), q.id, nid, acc);
        }
        ann_add<MODE != 0>(SA, j, acc.edges - e0, acc.comps - c0);
    }
    flush(acc, A, 1, lane);
    __syncthreads();
    ann_flush<MODE != 0>(SA, A);
}

// Row (sorted request s, target annulus j): the exact index ranges ("pieces")
// of j's owned block the request tests there.  Global requests: the
// split_wraparound pieces of [theta - h, theta + h) (sweep.hpp:41-58) and,
// when this shard owns engine P-1, their chunk-0 parts lifted by 2pi
// (sweep.hpp:404-432).  Streaming requests (dense targets only): [s0, s1) of
// the window (own window: (p, lower_bound(hi)) in index order); the rare
// pairs that need the full (theta, id) dedup or live in the halo block run
// right here, thread-serially.  Also writes the sorted request records and
// the per-(segment, target) max half-width.
template <int MODE>
__global__ void __launch_bounds__(256) req_rows_kernel(EdgeArgs A) {
    const std::uint64_t nR  = A.n_req;
    // task of this block (uniform search over the wave's tasks): target j, source, request range
    const std::uint32_t b = A.row_b0 + blockIdx.x;
    std::uint32_t       t0 = A.row_t0, t1 = A.row_t1 - 1; // last task with first block <= b
    while (t0 < t1) {
        const std::uint32_t mid = (t0 + t1 + 1) >> 1;
        if (A.row_tasks[mid].w <= b) t0 = mid;
        else t1 = mid - 1;
    }
    const uint4         task = A.row_tasks[t0];
    const std::uint64_t s    = task.y + std::uint64_t(b - task.w) * blockDim.x + threadIdx.x;
    const bool          ok   = s < task.z;
    const int           j    = int(task.x & 0xffffu);
    Acc                 acc;
    int                 hkey  = -1;
    unsigned long long  hbits = 0;
    if (ok) {
        const int           jt = j - A.first_streaming;
        const std::uint32_t u  = A.g_u[s];
        const AnnulusDev&   Aj = A.ann[j];
        std::uint32_t       pc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        double              h     = -1.0; // half-width that bounds the pieces around the key angle
        // every task row is read by the node tiles: the global points, and the dense (source, j) pairs
        const bool          used  = true;
        const int           a_req = (task.x >> 16) == 0xffffu ? -1 : int(task.x >> 16);
        const double2 q2  = A.g_rec[2 * s + 1]; // (coth, coshR / sinh)
        const double  inv = A.g_inv[s];
        const double4 ax  = A.g_aux[s]; // global: (theta, 0, 0, theta); streaming: (lambda, beta, hw, theta)
        if (u < A.n_glob) {
            const double th = ax.x;
            if (Aj.halo > Aj.off) {
                h              = half_width_in(Aj, q2.x, inv); // generator.hpp:67
                const double a = fsub(th, h), b = fadd(th, h);
                double       pa[2], pb[2];
                int          np = 1;
                if (fsub(b, a) >= kTwoPiD) {
                    pa[0] = 0.0, pb[0] = kTwoPiD;
                } else if (a < 0.0) {
                    pa[0] = fadd(a, kTwoPiD), pb[0] = kTwoPiD, pa[1] = 0.0, pb[1] = b, np = 2;
                } else if (b > kTwoPiD) {
                    pa[0] = a, pb[0] = kTwoPiD, pa[1] = 0.0, pb[1] = fsub(b, kTwoPiD), np = 2;
                } else {
                    pa[0] = a, pb[0] = b;
                }
                int nw = 0;
                for (int k = 0; k < np; ++k) {
                    double lo[2] = {pa[k], 0.0}, hi[2] = {pb[k], 0.0};
                    int    nl    = 1;
                    if (A.lift_part) {
                        const double l2 = pa[k] < 0.0 ? 0.0 : pa[k];                      // max(begin, w0 = 0)
                        const double h2 = A.chunk0_upper < pb[k] ? A.chunk0_upper : pb[k]; // min(end, w1)
                        if (l2 < h2) lo[1] = fadd(l2, kTwoPiD), hi[1] = fadd(h2, kTwoPiD), nl = 2;
                    }
                    for (int v = 0; v < nl; ++v) {
                        if (hi[v] > lo[v]) {
                            std::uint64_t s0, s1;
                            owned_range(A, Aj, lo[v], hi[v], s0, s1);
                            if (s1 > s0) {
                                pc[2 * nw] = std::uint32_t(s0), pc[2 * nw + 1] = std::uint32_t(s1);
                                acc.comps += s1 - s0;
                                ++nw;
                            }
                        }
                    }
                }
            }
        } else {
            const int a = a_req;
            if (used) {
                const AnnulusDev&   Aa = A.ann[a];
                const std::uint64_t p  = Aa.off + (u - A.req_off[a]);
                const bool          halo_req  = p >= Aa.halo;
                const bool          same_simp = !halo_req && p < Aa.wrap;
                double              lo, hi;
                if (j == a) {
                    lo = ax.y, hi = fadd(ax.y, fmul(2.0, ax.z)), h = ax.z;
                } else {
                    h  = half_width_in(Aj, q2.x, inv);
                    lo = fsub(ax.x, h), hi = fadd(ax.x, h);
                }
                if (hi > lo) {
                    std::uint64_t g0 = 0, g1 = 0;
                    if (Aj.halo > Aj.off) {
                        std::uint64_t s0, s1;
                        if (j == a && same_simp) {
                            const std::uint64_t w = Aj.wrap, ub = lower_bound_owned(A, Aj, hi);
                            s0 = p + 1, s1 = ub < w ? ub : w;
                            g0 = w, g1 = ub;
                        } else {
                            owned_range(A, Aj, lo, hi, s0, s1);
                            if (j == a) g0 = s0, g1 = s1, s1 = s0;
                        }
                        if (s1 > s0) {
                            pc[0] = std::uint32_t(s0), pc[1] = std::uint32_t(s1);
                            acc.comps += s1 - s0;
                        }
                    }
                    const bool halo_nodes =
                        !halo_req && Aj.end > Aj.halo && hi > A.s_lam[Aj.halo] && lo <= A.s_lam[Aj.end - 1];
                    // rare pairs needing the full dedup or in the halo block: deferred to
                    // deferred_kernel (one warp per range) so no thread runs them serially
                    if (g1 > g0) defer_range(A, std::uint32_t(s), g0, g1, true);
                    if (halo_nodes) {
                        const std::uint64_t h0 = lower_bound_halo(A, Aj, lo), h1 = lower_bound_halo(A, Aj, hi);
                        if (h1 > h0) defer_range(A, std::uint32_t(s), h0, h1, j == a);
                    }
                }
            }
        }
        if (h >= 0.0 && pc[1] > pc[0]) {
            int c0 = 0, c1 = (*A.n_cls < kMaxCls ? *A.n_cls : kMaxCls) - 1; // segment of s
            while (c0 < c1) {
                const int mid = (c0 + c1 + 1) >> 1;
                if (A.cseg[mid] <= s) c0 = mid;
                else c1 = mid - 1;
            }
            hkey  = c0 * A.count + j;
            hbits = static_cast<unsigned long long>(__double_as_longlong(h));
        }
        if (used) { // rows of non-dense (source, target) pairs are never read: their segments' hmax stays 0
            uint4* row = reinterpret_cast<uint4*>(A.g_rows + (std::uint64_t(jt) * nR + s) * 8);
            row[0]     = make_uint4(pc[0], pc[1], pc[2], pc[3]);
            row[1]     = make_uint4(pc[4], pc[5], pc[6], pc[7]);
        }
    }
    // per-(segment, target) max half-width: one atomic per group of lanes sharing the key
    {   // the high word bounds the value from above (non-negative doubles order like their bits)
        const unsigned grp = __match_any_sync(kFull, hkey);
        const unsigned mx  = __reduce_max_sync(grp, unsigned(hbits >> 32));
        if (hkey >= 0 && int(threadIdx.x & 31) == __ffs(grp) - 1 && hbits)
            atomicMax(&A.hmax_bits[hkey], (static_cast<unsigned long long>(mx) << 32) | 0xffffffffull);
    }
    if constexpr (MODE != 0) { // the rows' comps per target annulus (lanes of one target reduce together;
                               // compiled out of the counters-only kernel, where it also miscompiled)
        const int      jj  = ok ? j : -1;
        const unsigned grp = __match_any_sync(kFull, jj);
        const unsigned cs  = __reduce_add_sync(grp, unsigned(acc.comps));
        if (jj >= 0 && cs && int(threadIdx.x & 31) == __ffs(grp) - 1) {
            const unsigned w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
            atomicAdd(&A.ann_ctr[std::size_t(w & (kAnnSlots - 1)) * 2 * kMaxAnnuli + kMaxAnnuli + jj],
                      static_cast<unsigned long long>(cs));
        }
    }
    flush(acc, A, 1, threadIdx.x & 31);
}

constexpr int kTN    = kTileNodes; // owned nodes per dense-engine tile (kTN / 32 per lane, in registers)
constexpr int kQ     = kTN / 32;
constexpr int kStrip = 1;   // tiles per warp sharing one candidate search

struct GEnt { // one (request, piece) intersecting the current tile, compacted
    double        cs, sn, coth, rci;
    std::uint32_t id, lohi; // piece clipped to the tile: local [lo, hi) packed lo | hi << 16
};
struct GWarp {
    GEnt          e[128];   // up to 4 pieces per candidate, 32 candidates per chunk
    std::uint32_t rng[64];  // candidate range starts (sorted positions), two per segment of a pass
    std::uint32_t pre[65];  // exclusive prefix of the range lengths (pre[64] = total)
};

// angle of the sorted requests of one segment: first position in [lo, hi)
// with angle >= x.
__device__ __forceinline__ std::uint32_t gtheta_lb(const double* th, std::uint32_t lo, std::uint32_t hi, double x) {
    while (lo < hi) {
        const std::uint32_t mid = (lo + hi) >> 1;
        if (th[mid] < x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// One warp = a strip of kStrip consecutive 128-node tiles of annulus j's
// owned block.  The candidate requests of the strip (per segment: angle
// within hmax(segment, j) of the strip, circularly) are found once; per tile
// the nodes sit in registers, each chunk of 32 candidates is clipped to the
// tile and compacted into (request, piece) entries in shared memory, and the
// warp sweeps the entries (32-node slices outside an entry are skipped).
// MINB: CTAs per SM the register budget targets (measured cfg2: wave 1's targets 0.40 ms at 2,
// 0.43 at 3 with small spills; wave 2's outermost target 0.18 at 2, 0.15 at 3)
#ifndef RHG_TILES_MINB_WIDE
#define RHG_TILES_MINB_WIDE 4 // node tiles for wide dense windows (average degree >= 128; measured 3 / 4 / 5: cfg3 22.08 / 21.73 / 25.53 ms)
#endif
#ifndef RHG_TILES_MINB2
#define RHG_TILES_MINB2 3 // node tiles of wave 2 (narrow windows; measured 2 / 3: cfg2 3.045 / 3.030 ms, cfg4 32.37 / 31.99)
#endif
#ifndef RHG_TILES_MINB1
#define RHG_TILES_MINB1 3 // node tiles of wave 1 (measured cfg2, dense engine alone: 2 -> 0.40 ms, 3 -> 0.43; beside
                          // the slab join on its own stream 3 is better: step 3.35 -> 3.28 ms at cfg2, cfg4 36.7 ->
                          // 36.4, cfg5 165.6 -> 163.5; EdgeWave::dense_occ4 picks 4 for average degrees >= 128)
#endif
template <int MODE, int MINB = 2>
__global__ void __launch_bounds__(256, MINB) glob_tiles_kernel(EdgeArgs A) {
    __shared__ GWarp    smem[8];
    const int           lane = threadIdx.x & 31;
    const std::uint64_t w    = A.gt_prefix[A.j0] + ((std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5);
    if (w >= A.gt_prefix[A.j1]) return;
    GWarp* ws = &smem[threadIdx.x >> 5];
    int    j  = A.first_streaming, hj = A.count - 1; // last annulus with gt_prefix <= w
    while (j < hj) {
        const int mid = (j + hj + 1) >> 1;
        if (A.gt_prefix[mid] <= w) j = mid;
        else hj = mid - 1;
    }
    const AnnulusDev&   Aj   = A.ann[j];
    const std::uint32_t sb0  = std::uint32_t(Aj.off + (w - A.gt_prefix[j]) * (kTN * kStrip));
    const std::uint32_t sb1  = std::uint32_t(sb0 + kTN * kStrip < Aj.halo ? sb0 + kTN * kStrip : Aj.halo);
    const std::uint64_t gjb  = std::uint64_t(j - A.first_streaming) * A.n_req;
    const int           ncls = *A.n_cls < kMaxCls ? *A.n_cls : kMaxCls;
    const double        lam_lo = A.s_lam[sb0], lam_hi = A.s_lam[sb1 - 1];
    Acc                 acc;
    unsigned long long  rsum = 0; // this lane's sum of request ids over its edges
    for (int a0 = 0; a0 < ncls; a0 += 32) {
        // candidate ranges of sorted positions: lane = segment a0 + lane
        {
            const int     a  = a0 + lane;
            std::uint32_t r0 = 0, r1 = 0, r2 = 0, r3 = 0;
            if (a < ncls) {
                const std::uint32_t      sa = A.cseg[a], sb = A.cseg[a + 1];
                const unsigned long long hb = A.hmax_bits[a * A.count + j];
                if (sb > sa && hb) {
                    const double hmax = __longlong_as_double(static_cast<long long>(hb));
                    // margin: the angles are sorted by a 32-bit quantised key (2pi/2^32 = 1.5e-9)
                    const double L = (lam_hi - lam_lo) + 2.0 * hmax + 2e-7;
                    if (L >= kTwoPiD) {
                        r0 = sa, r1 = sb;
                    } else {
                        double st = lam_lo - hmax - 1e-7;
                        while (st < 0.0) st += kTwoPiD;
                        while (st >= kTwoPiD) st -= kTwoPiD;
                        const double         en  = st + L;
                        const std::uint32_t  sh  = A.bk_shift[a];
                        const std::uint32_t* tab = A.gbk + A.bk_off[a];
                        // bucket of an angle in [0, 2pi]: quantised like the sort key (superset ranges)
                        auto bkt = [sh](double x) {
                            const double q = x * (4294967296.0 / kTwoPiD);
                            return (q >= 4294967295.0 ? 0xffffffffu : std::uint32_t(q > 0.0 ? q : 0.0)) >> sh;
                        };
                        r0 = tab[bkt(st)];
                        if (en <= kTwoPiD) {
                            r1 = tab[bkt(en) + 1];
                        } else {
                            r1 = sb;
                            r2 = sa, r3 = tab[bkt(en - kTwoPiD) + 1];
                        }
                    }
                }
            }
            // the ranges of this pass as one list: candidate t lies in range r with pre[r] <= t < pre[r + 1]
            const std::uint32_t la = r1 - r0, lb = r3 - r2;
            std::uint32_t       incl = la + lb;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const std::uint32_t x = __shfl_up_sync(kFull, incl, o);
                if (lane >= o) incl += x;
            }
            __syncwarp();
            ws->rng[2 * lane] = r0, ws->rng[2 * lane + 1] = r2;
            ws->pre[2 * lane] = incl - la - lb, ws->pre[2 * lane + 1] = incl - lb;
            if (lane == 31) ws->pre[64] = incl;
            __syncwarp();
        }
        const std::uint32_t C = ws->pre[64];
        for (std::uint32_t t0 = sb0; t0 < sb1; t0 += kTN) {
            const std::uint32_t t1 = t0 + kTN < sb1 ? t0 + kTN : sb1;
            double2             n1[kQ], n2[kQ];
            std::uint32_t       ecnt[kQ];
#pragma unroll
            for (int q = 0; q < kQ; ++q) {
                const std::uint32_t k = t0 + std::uint32_t(lane + 32 * q);
                const std::uint32_t kc = k < t1 ? k : t0;
                n1[q] = A.s_rec1[kc], n2[q] = A.s_rec2[kc];
                ecnt[q] = 0;
            }
            {
                for (std::uint32_t c0 = 0; c0 < C; c0 += 32) {
                    // stage: lane = candidate c0 + lane of the list; its pieces clipped to [t0, t1)
                    std::uint32_t       pc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                    const std::uint32_t tc    = c0 + std::uint32_t(lane);
                    std::uint32_t       s     = 0;
                    if (tc < C) {
                        int r = 0;
#pragma unroll
                        for (int step = 32; step > 0; step >>= 1)
                            if (ws->pre[r + step] <= tc) r += step;
                        s = ws->rng[r] + (tc - ws->pre[r]);
                    }
                    if (tc < C) {
                        const uint4* row = reinterpret_cast<const uint4*>(A.g_rows + (gjb + s) * 8);
                        const uint4  pa = row[0], pb = row[1];
                        pc[0] = pa.x, pc[1] = pa.y, pc[2] = pa.z, pc[3] = pa.w;
                        pc[4] = pb.x, pc[5] = pb.y, pc[6] = pb.z, pc[7] = pb.w;
                    }
                    std::uint32_t ne = 0, lh[4];
#pragma unroll
                    for (int v = 0; v < 4; ++v) { // pieces are disjoint and packed
                        const std::uint32_t ps = pc[2 * v], pe = pc[2 * v + 1];
                        lh[v] = 0;
                        if (pe > ps && pe > t0 && ps < t1) {
                            const std::uint32_t l = ps > t0 ? ps - t0 : 0u, h = (pe < t1 ? pe : t1) - t0;
                            lh[v] = l | (h << 16);
                            ++ne;
                        }
                    }
                    std::uint32_t incl = ne;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const std::uint32_t x = __shfl_up_sync(kFull, incl, o);
                        if (lane >= o) incl += x;
                    }
                    const std::uint32_t tot = __shfl_sync(kFull, incl, 31);
                    if (tot == 0) continue;
                    __syncwarp();
                    if (ne) {
                        const double2 a1 = A.g_rec[2 * s], a2 = A.g_rec[2 * s + 1];
                        const std::uint32_t id = A.g_id[s];
                        std::uint32_t pos = incl - ne;
#pragma unroll
                        for (int v = 0; v < 4; ++v)
                            if (lh[v]) {
                                GEnt& E = ws->e[pos++];
                                E.cs = a1.x, E.sn = a1.y, E.coth = a2.x, E.rci = a2.y, E.id = id, E.lohi = lh[v];
                            }
                    }
                    __syncwarp();
                    if (A.dbg && lane == 0) atomicAdd(&A.dbg[8], 32ull), atomicAdd(&A.dbg[9], static_cast<unsigned long long>(tot));
                    for (std::uint32_t c = 0; c < tot; ++c) {
                        const GEnt&         E  = ws->e[c];
                        const double        cs = E.cs, sn = E.sn, coth = E.coth, rci = E.rci;
                        const std::uint32_t el = E.lohi & 0xffffu, eh = E.lohi >> 16;
                        std::uint32_t       ce = 0; // this lane's edges with request E
                        if (el == 0 && eh == kTN) { // the piece covers the whole tile
#pragma unroll
                            for (int q = 0; q < kQ; ++q) {
                                const bool e = edge_test(cs, sn, coth, rci, n1[q], n2[q]);
                                ecnt[q] += e, ce += e;
                                if (MODE == 1 && e) {
                                    atomicAdd(&A.degrees[E.id], 1u);
                                    atomicAdd(&A.degrees[A.s_id[t0 + std::uint32_t(lane + 32 * q)]], 1u);
                                }
                                if (MODE == 2 && e) emit_edge(A, E.id, A.s_id[t0 + std::uint32_t(lane + 32 * q)]);
                            }
                        } else {
#pragma unroll
                            for (int q = 0; q < kQ; ++q) {
                                if (eh <= std::uint32_t(32 * q) || el >= std::uint32_t(32 * q + 32)) continue; // slice untouched
                                const std::uint32_t kl = std::uint32_t(lane + 32 * q);
                                const bool e = kl >= el && kl < eh && edge_test(cs, sn, coth, rci, n1[q], n2[q]);
                                ecnt[q] += e, ce += e;
                                if (MODE == 1 && e) {
                                    atomicAdd(&A.degrees[E.id], 1u);
                                    atomicAdd(&A.degrees[A.s_id[t0 + kl]], 1u);
                                }
                                if (MODE == 2 && e) emit_edge(A, E.id, A.s_id[t0 + kl]);
                            }
                        }
                        rsum += static_cast<unsigned long long>(ce) * E.id;
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < kQ; ++q) {
                const std::uint32_t k = t0 + std::uint32_t(lane + 32 * q);
                if (ecnt[q]) {
                    acc.edges += ecnt[q];
                    acc.fp += static_cast<unsigned long long>(ecnt[q]) * A.s_id[k];
                }
            }
        }
    }
    acc.fp += rsum; // flush() reduces over the warp
    flush<MODE != 0>(acc, A, 1, lane, j);
}

// generator.hpp:84-102: all pairs i < k of the global points, request = i.
template <int MODE>
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
    __shared__ AnnAcc        SA;
    __shared__ std::uint64_t sg[kMaxAnnuli + 1];
    ann_zero<MODE != 0>(SA);
    for (int a = threadIdx.x; a <= A.first_streaming; a += blockDim.x) sg[a] = A.gseg[a];
    if (col < nG) {
        s1[threadIdx.x] = A.rec1[A.n_ext + col];
        s2[threadIdx.x] = A.rec2[A.n_ext + col];
    }
    __syncthreads();
    const std::uint64_t i = I * kGGTile + threadIdx.x;
    Acc                 acc;
    int                 ai = 0, key = -1; // key: the annulus of all this row's pairs (single-annulus rows)
    // annulus of a global point index: the last inner annulus whose id base is <= it (ids are
    // annulus-major); a pair counts for max(annulus_i, annulus_k) (generator.hpp:89)
    auto ann_of = [&](std::uint64_t g) {
        int a = 0;
        while (a + 1 < A.first_streaming && sg[a + 1] <= g) ++a;
        return a;
    };
    if (i < nG) {
        const double2 r1 = A.rec1[A.n_ext + i], r2 = A.rec2[A.n_ext + i];
        const double  cs = r1.x, sn = r1.y, coth = r2.x, rci = fmul(A.cosh_R, r2.y);
        std::uint64_t k0 = J * kGGTile;
        if (k0 <= i) k0 = i + 1;
        const std::uint64_t k1 = (J + 1) * kGGTile < nG ? (J + 1) * kGGTile : nG;
        acc.comps              = k1 > k0 ? k1 - k0 : 0;
        if constexpr (MODE == 0) { // counters only (the bench path): no per-annulus bookkeeping
            for (std::uint64_t k = k0; k < k1; ++k)
                count_edge<MODE>(A, edge_test(cs, sn, coth, rci, s1[k - J * kGGTile], s2[k - J * kGGTile]), i, k, acc);
        } else {
        ai = ann_of(i);
        const int a0 = k1 > k0 ? ann_of(k0) : ai, a1 = k1 > k0 ? ann_of(k1 - 1) : ai;
        if (a0 == a1) { // the usual case: the row's columns lie in one annulus (booked below, per warp)
            for (std::uint64_t k = k0; k < k1; ++k)
                count_edge<MODE>(A, edge_test(cs, sn, coth, rci, s1[k - J * kGGTile], s2[k - J * kGGTile]), i, k, acc);
            key = ai > a0 ? ai : a0;
        } else { // one run per annulus of k (global ids are annulus-major)
            for (std::uint64_t k = k0; k < k1;) {
                const int           ak = ann_of(k);
                const std::uint64_t kn = sg[ak + 1]; // a0 != a1: ak is not the last annulus
                const std::uint64_t ks = k, ke = kn < k1 ? kn : k1;
                const unsigned long long e0 = acc.edges;
                for (; k < ke; ++k)
                    count_edge<MODE>(A, edge_test(cs, sn, coth, rci, s1[k - J * kGGTile], s2[k - J * kGGTile]), i, k,
                                     acc);
                ann_add<MODE != 0>(SA, ai > ak ? ai : ak, acc.edges - e0, ke - ks);
            }
        }
        }
    }
    if constexpr (MODE != 0) { // single-annulus rows: one shared-memory atomic per annulus per warp
        const unsigned grp = __match_any_sync(kFull, key);
        const unsigned ce  = __reduce_add_sync(grp, key >= 0 ? unsigned(acc.edges) : 0u);
        const unsigned cc  = __reduce_add_sync(grp, key >= 0 ? unsigned(acc.comps) : 0u);
        if (key >= 0 && int(threadIdx.x & 31) == __ffs(grp) - 1) ann_add<MODE != 0>(SA, key, ce, cc);
    }
    flush(acc, A, 2, threadIdx.x & 31);
    __syncthreads();
    ann_flush<MODE != 0>(SA, A);
}

// Fold the counter slots of the three families into A.ctr (blocks 0..2) and the
// per-annulus slots into slot 0 (block 3).
__global__ void __launch_bounds__(1024) reduce_counters_kernel(EdgeArgs A) {
    const int          f = blockIdx.x;
    if (f == 3) {
        for (int i = threadIdx.x; i < 2 * kMaxAnnuli; i += blockDim.x) {
            unsigned long long v = 0;
            for (int s = 0; s < kAnnSlots; ++s) v += A.ann_ctr[std::size_t(s) * 2 * kMaxAnnuli + i];
            A.ann_ctr[i] = v; // slot 0 holds the totals (slots 1.. are left as they are)
        }
        return;
    }
    unsigned long long e = 0, fp = 0, c = 0;
    for (int i = threadIdx.x; i < kSlots; i += blockDim.x) {
        const SlotCounter& s = A.slots[f * kSlots + i];
        e += s.edges, fp += s.fp, c += s.comps;
    }
    __shared__ unsigned long long red[3][32];
    const int                     lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        e += __shfl_down_sync(kFull, e, o);
        fp += __shfl_down_sync(kFull, fp, o);
        c += __shfl_down_sync(kFull, c, o);
    }
    if (lane == 0) red[0][w] = e, red[1][w] = fp, red[2][w] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        Counters out{0, 0, 0};
        for (int k = 0; k < int(blockDim.x >> 5); ++k) out.edges += red[0][k], out.fp += red[1][k], out.comps += red[2][k];
        A.ctr[f] = out;
    }
}


// ------------------------------------------------- materialised edges ---
// Canonical order of an edge list (u < v, ascending by u then v): key = u << 32 | v.
__global__ void edge_keys_kernel(const ulonglong2* __restrict__ e, std::uint64_t m, unsigned long long* __restrict__ k) {
    const std::uint64_t i = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < m) k[i] = (e[i].x << 32) | e[i].y;
}
__global__ void edge_unpack_kernel(const unsigned long long* __restrict__ k, std::uint64_t m, ulonglong2* __restrict__ e) {
    const std::uint64_t i = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < m) e[i] = make_ulonglong2(k[i] >> 32, k[i] & 0xffffffffull);
}
} // namespace

void launch_cell_index(const EdgeArgs& a0, std::uint32_t blk_begin, std::uint32_t blk_end, int j_begin, int j_end,
                       bool gen, cudaStream_t st, std::uint64_t* launches) {
    if (a0.first_streaming >= a0.count || j_end <= j_begin) return;
    EdgeArgs a = a0;
    a.blk0 = blk_begin, a.j0 = j_begin, a.j1 = j_end;
    const std::uint32_t nblocks = blk_end - blk_begin;
    const unsigned      g = unsigned(nblocks ? nblocks : 1); // >= 1: block 0 of wave 1 initialises empty annuli
    const dim3          tails(64, unsigned(j_end - j_begin));
    const bool gallop = gen && a.rank_gallop;
    if (!gallop) { // walking ranks scan the sorted betas around each point themselves (rank_kernel)
        if (gen) beta_cells_kernel<true><<<g, 256, 0, st>>>(a);
        else beta_cells_kernel<false><<<g, 256, 0, st>>>(a);
        cell_tail_kernel<<<tails, 256, 0, st>>>(a, 0);
        *launches += 2;
    }
    if (nblocks) {
        if (gallop) rank_kernel<true, true><<<g, 256, 0, st>>>(a);
        else if (gen) rank_kernel<true><<<g, 256, 0, st>>>(a);
        else rank_kernel<false><<<g, 256, 0, st>>>(a);
        ++*launches;
    }
    if (nblocks || gallop) { // galloping: block 0 of wave 1 also initialises the empty annuli's tables
        lambda_cells_kernel<<<g, 256, 0, st>>>(a);
        cell_tail_kernel<<<tails, 256, 0, st>>>(a, 1);
        *launches += 2;
    }
    a0.mark("sort_phase", st);
}

void launch_sort_globals(EdgeArgs& a, void* scratch, std::size_t scratch_bytes, std::size_t* need, cudaStream_t st,
                         std::uint64_t* launches) {
    // scratch: keys | perm (the sorted order) | bucket counts, then cursors | block sums | segment index
    const std::size_t n    = a.n_req;
    const std::size_t nbk  = 2 * n + 65 * std::size_t(kMaxCls); // bound on the bucket entries
    const std::size_t nsum = (nbk + 256 * kScanItems - 1) / (256 * kScanItems);
    const std::size_t nseg = std::size_t(a.count - a.first_streaming + 1) << 10;
    auto              al   = [](std::size_t x) { return (x + 255) & ~std::size_t(255); };
    const std::size_t o_pm = al(n * 8), o_bc = o_pm + al(n * 4), o_bs = o_bc + al(nbk * 4), o_si = o_bs + al(nsum * 4);
    *need = o_si + al(nseg * 4) + 256;
    if (!scratch || scratch_bytes < *need || n == 0) return;
    char*               p      = static_cast<char*>(scratch);
    unsigned long long* keys   = reinterpret_cast<unsigned long long*>(p);
    std::uint32_t*      perm   = reinterpret_cast<std::uint32_t*>(p + o_pm);
    std::uint32_t*      bcount = reinterpret_cast<std::uint32_t*>(p + o_bc);
    std::uint32_t*      bsum   = reinterpret_cast<std::uint32_t*>(p + o_bs);
    std::uint32_t*      segix  = reinterpret_cast<std::uint32_t*>(p + o_si);
    const unsigned      g      = unsigned((n + 255) / 256);
    cudaMemsetAsync(a.seg_first, 0, nseg * sizeof(std::uint32_t), st);
    cudaMemsetAsync(bcount, 0, nbk * sizeof(std::uint32_t), st);
    req_keys_kernel<<<g, 256, 0, st>>>(a, keys);
    req_segments_kernel<<<1, 1024, 0, st>>>(a, segix);
    req_bucket_count_kernel<<<g, 256, 0, st>>>(a, keys, segix, bcount);
    scan_blocks_kernel<<<unsigned(nsum), 256, 0, st>>>(bcount, a.gbk, bsum, nbk);
    scan_sums_kernel<<<1, 1024, 0, st>>>(bsum, unsigned(nsum));
    scan_add_kernel<<<unsigned((nbk + 255) / 256), 256, 0, st>>>(a.gbk, bcount, bsum, nbk);
    req_scatter_kernel<<<g, 256, 0, st>>>(a, keys, segix, bcount, perm);
    a.gperm = perm;
    req_gather_kernel<<<g, 256, 0, st>>>(a);
    *launches += 8;
    a.mark("dense_prep", st);
}

// Launch kernel K<MODE> for the run-time mode (0 counters, 1 degrees, 2 edges).
#define RHG_LAUNCH_MODE(K, mode, cfg, ...)                          \
    do {                                                            \
        if ((mode) == 2) K<2><<<cfg>>>(__VA_ARGS__);                \
        else if ((mode) == 1) K<1><<<cfg>>>(__VA_ARGS__);           \
        else K<0><<<cfg>>>(__VA_ARGS__);                            \
    } while (0)
#define RHG_CFG(...) __VA_ARGS__

template <int NT, int MINB>
void launch_slab(const EdgeArgs& a, unsigned n, int mode, cudaStream_t st) {
    const int   smem = int(sizeof(SlabSmem<NT, (MINB < 5)>));
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(slab_kernel<0, NT, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(slab_kernel<1, NT, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(slab_kernel<2, NT, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(slab_kernel<3, NT, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr = true;
    }
    if (mode == 3) slab_kernel<3, NT, MINB><<<n, NT, smem, st>>>(a);
    else if (mode == 2) slab_kernel<2, NT, MINB><<<n, NT, smem, st>>>(a);
    else if (mode == 1) slab_kernel<1, NT, MINB><<<n, NT, smem, st>>>(a);
    else slab_kernel<0, NT, MINB><<<n, NT, smem, st>>>(a);
}

// One wave of edge work on st: dense rows and node tiles of the targets
// [W.j0, W.j1), the slab join over slabs [W.slab_begin, W.slab_end), and
// optionally the global unit, the tail pairs, the deferred ranges and the
// final counter fold.  The dense requests must already be sorted
// (launch_sort_globals) and the targets' annuli indexed (launch_cell_index).
void launch_edges(const EdgeArgs& a0, const EdgeWave& W, cudaStream_t st, std::uint64_t* launches) {
    const int  mode = a0.edge_out ? 2 : a0.degrees ? 1 : 0;
    EdgeArgs   a   = a0;
    a.j0 = W.j0, a.j1 = W.j1, a.slab0 = W.slab_begin;
    if (W.j1 > W.j0 && a.n_req && a.first_streaming < a.count) {
        a.row_t0 = W.row_t0, a.row_t1 = W.row_t1, a.row_b0 = W.row_b0;
        if (W.row_nb) {
            RHG_LAUNCH_MODE(req_rows_kernel, mode, RHG_CFG(W.row_nb, 256, 0, st), a);
            ++*launches;
        }
        a.mark("rows", st);
        const std::uint64_t tw = W.tile_warps;
        if (tw) {
            const unsigned g = unsigned((tw + 7) / 8);
            if (W.first_wave && W.dense_occ4) { // wave 1, wide windows: 4 CTAs/SM (64 registers)
                if (mode == 2) glob_tiles_kernel<2, RHG_TILES_MINB_WIDE><<<g, 256, 0, st>>>(a);
                else if (mode == 1) glob_tiles_kernel<1, RHG_TILES_MINB_WIDE><<<g, 256, 0, st>>>(a);
                else glob_tiles_kernel<0, RHG_TILES_MINB_WIDE><<<g, 256, 0, st>>>(a);
            } else if (W.first_wave) { // wave 1
                if (mode == 2) glob_tiles_kernel<2, RHG_TILES_MINB1><<<g, 256, 0, st>>>(a);
                else if (mode == 1) glob_tiles_kernel<1, RHG_TILES_MINB1><<<g, 256, 0, st>>>(a);
                else glob_tiles_kernel<0, RHG_TILES_MINB1><<<g, 256, 0, st>>>(a);
            }
            else if (W.dense_occ4) { // wave 2, wide windows
                if (mode == 2) glob_tiles_kernel<2, RHG_TILES_MINB_WIDE><<<g, 256, 0, st>>>(a);
                else if (mode == 1) glob_tiles_kernel<1, RHG_TILES_MINB_WIDE><<<g, 256, 0, st>>>(a);
                else glob_tiles_kernel<0, RHG_TILES_MINB_WIDE><<<g, 256, 0, st>>>(a);
            }
            else if (mode == 2) glob_tiles_kernel<2, RHG_TILES_MINB2><<<g, 256, 0, st>>>(a);
            else if (mode == 1) glob_tiles_kernel<1, RHG_TILES_MINB2><<<g, 256, 0, st>>>(a);
            else glob_tiles_kernel<0, RHG_TILES_MINB2><<<g, 256, 0, st>>>(a);
            ++*launches;
            a.mark("tiles", st);
        }
    }
    if (W.slab_end > W.slab_begin) {
        if (W.ev0) cudaEventRecord(W.ev0, st);
        const unsigned n   = unsigned(W.slab_end - W.slab_begin);
        static const int scfg = std::getenv("RHG_SLAB_CFG") ? std::atoi(std::getenv("RHG_SLAB_CFG")) : 0;
        // 256 threads x 6 CTAs/SM (40 registers; the exact path's node doubles read from global
        // memory, so 31.5 KB of shared memory per CTA): measured best at cfg2 (x4 with the node
        // doubles staged, 64 registers: 3.96 -> 3.80 ms/step; x5 3.87; x7 4.13, spills), also
        // cfg3 / cfg4 (-1.6% / -3.4%); RHG_SLAB_CFG selects the others for A/B runs
        const int smode = a.audit ? 3 : mode; // the predicate audit instruments the sparse engine's pre-filter
        // waves whose windows lie below the FP64 rounding floor of the pre-filter (outer annuli at
        // R >~ 35: cfg4, cfg5) run the exact predicate on most pairs: 4 CTAs/SM with the node
        // doubles staged by TMA (measured cfg4 slab 17.5 -> 16.6 ms, cfg5 86 -> 78; cfg2 / cfg3
        // keep 6 CTAs/SM without them: 1.52 vs 1.55 ms, 8.22 vs 8.42 ms)
        if (scfg == 4 || (scfg == 0 && W.exact_slabs)) launch_slab<256, 4>(a, n, smode, st);
        else launch_slab<256, RHG_SLAB_MINB>(a, n, smode, st);
        ++*launches;
        if (W.tail && a.n_tail) {
            RHG_LAUNCH_MODE(tail_kernel, mode, RHG_CFG(unsigned((a.n_tail + 255) / 256), 256, 0, st), a);
            ++*launches;
        }
        if (W.ev1) cudaEventRecord(W.ev1, st); // sparse engine of this wave (slab join [+ tail])
        a.mark("slab(+tail)", st);
    } else if (W.tail && a.n_tail) {
        if (W.ev0) cudaEventRecord(W.ev0, st);
        RHG_LAUNCH_MODE(tail_kernel, mode, RHG_CFG(unsigned((a.n_tail + 255) / 256), 256, 0, st), a);
        ++*launches;
        if (W.ev1) cudaEventRecord(W.ev1, st);
    }
    if (W.global_unit && a.gg_tile_end > a.gg_tile_begin) {
        const std::uint64_t nT     = (a.n_glob + kGGTile - 1) / kGGTile;
        const unsigned      blocks = unsigned(a.gg_tile_end - a.gg_tile_begin);
        RHG_LAUNCH_MODE(glob_pairs_kernel, mode, RHG_CFG(blocks, kGGTile, 0, st), a, nT);
        ++*launches;
        a.mark("global_unit", st);
    }
    if (W.finish) {
        if (a.n_req) {
            RHG_LAUNCH_MODE(deferred_kernel, mode, RHG_CFG(148 * 4, 256, 0, st), a);
            ++*launches;
        }
        reduce_counters_kernel<<<4, 1024, 0, st>>>(a);
        ++*launches;
    }
}

void launch_sort_edges(ulonglong2* edges, std::uint64_t m, unsigned long long* ka, unsigned long long* kb, void* tmp,
                       std::size_t* tmp_bytes, int end_bit, cudaStream_t st) {
    std::size_t need = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, need, ka, kb, int(m), 0, end_bit, st);
    if (!tmp || *tmp_bytes < need) {
        *tmp_bytes = need;
        return;
    }
    if (m == 0) return;
    const unsigned g = unsigned((m + 255) / 256);
    edge_keys_kernel<<<g, 256, 0, st>>>(edges, m, ka);
    cub::DeviceRadixSort::SortKeys(tmp, need, ka, kb, int(m), 0, end_bit, st);
    edge_unpack_kernel<<<g, 256, 0, st>>>(kb, m, edges);
}

} // namespace rhgb
