/*
 * rhg_b200.h — C ABI of the B200-native threshold-RHG generator.
 *
 * Drop-in boundary for the reference's stats-only generator path
 * (/root/reference/proj/include/rhg/):
 *
 *   reference                                            this ABI
 *   ---------------------------------------------------  ----------------------------------
 *   alpha_from_gamma              geometry.hpp:35-39      rhg_alpha_from_gamma
 *   radial_const_from_avg_degree  geometry.hpp:26-33      rhg_radial_const_from_avg_degree
 *   ModelParams(n,alpha,C,seed,P) geometry.hpp:49-67      rhg_params + rhg_params_validate
 *   ModelParams::from_avg_degree  geometry.hpp:69-72      rhg_params_from_avg_degree
 *   make_layout                   partition.hpp:233-240   rhg_layout (host only)
 *   GenOptions                    generator.hpp:27-32     rhg_create(device) / rhg_shard
 *   GenOptions.workers -> GPUs    generator.hpp:245-268   rhg_create_multi (one process, N GPUs, NCCL)
 *     (one process per GPU)                               rhg_nccl_unique_id + rhg_attach_comm
 *   RunStats                      generator.hpp:34-46     rhg_run_stats
 *   generate_stats(params, opts,  generator.hpp:219-291   rhg_generate_stats
 *                  degrees*)
 *   materialize_points / the      oracle.hpp:26-39,       rhg_sample_points (device sampler,
 *     ChunkPointSource stream     sweep.hpp:102-151         points copied back in id order)
 *   (parity hook, no ref. twin)                           rhg_count_edges_from_points
 *   generate(params, opts, edge)  generator.hpp:135-215   rhg_generate_edges (canonical order)
 *   TextEdgeWriter/BinaryEdgeWriter io.hpp:20-68           rhg_write_edges_text / _binary
 *   read_binary_edges             io.hpp:70-96            rhg_read_edges_binary
 *   naive_edges                   oracle.hpp:41-54        rhg_naive_edges (GPU brute force)
 *   powerlaw_mle                  stats.hpp:58-75         rhg_powerlaw_mle (host)
 *
 * Conventions: plain pointers and sizes, no exceptions across the ABI.
 * Every call returns RHG_OK (0) or an error code; rhg_last_error() gives the
 * thread-local message.  The reference's std::invalid_argument maps to
 * RHG_INVALID_ARGUMENT, std::logic_error (sweep invariants) to RHG_INVARIANT.
 * A context owns one CUDA device, its streams (five, ordered by events: DESIGN.md
 * section 2) and its device buffers; it is not re-entrant (one call at a time per
 * context).  There is no CPU fallback: without a usable sm_100 device
 * rhg_create fails with RHG_CUDA.
 */
#ifndef RHG_B200_H
#define RHG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RHG_ABI_VERSION 6
#define RHG_MAX_ANNULI 64 /* layouts with more annuli are rejected (RHG_INVALID_ARGUMENT) */

enum {
    RHG_OK = 0,
    RHG_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
    RHG_INVARIANT = 2,        /* std::logic_error in the reference      */
    RHG_CUDA = 3,
    RHG_NOMEM = 4
};

/* Graph identity: (n, alpha, C, seed, chunks) — geometry.hpp:47-56.
 * R is derived (R = 2 ln n + C) and filled by rhg_params_validate. */
typedef struct {
    uint64_t n;
    double alpha;
    double C;
    uint64_t seed;
    uint32_t chunks;
    double R; /* output of rhg_params_validate / from_avg_degree */
} rhg_params;

/* Which engines (angular chunks) this caller owns: rank r of `world` owns
 * chunks [r*P/world, (r+1)*P/world) and the global-unit rows of slice r.
 * {0, 1} = the whole graph (GenOptions default).  Partial results of all
 * ranks sum (wrapping) to the whole-graph result. */
typedef struct {
    uint32_t rank;
    uint32_t world;
} rhg_shard;

/* RunStats (generator.hpp:34-46) plus device timing. */
typedef struct {
    uint64_t n;
    uint64_t edges;           /* total.edges                          */
    uint64_t fingerprint;     /* total.fingerprint, wrapping Σ(u+v)   */
    uint64_t comps;           /* total.comps (distance computations)  */
    uint64_t global_vertices; /* n_G                                  */
    uint64_t streaming_vertices; /* owned streaming points            */
    uint64_t global_edges, global_comps; /* unit 0 share of this shard */
    uint32_t annuli, first_streaming;
    double R, r_G, cosh_R;
    double device_ms;  /* CUDA-event time, first kernel -> counters ready   */
    double sample_ms;  /* sampler kernels                                   */
    double edges_ms;   /* cell index + edge kernels                         */
    double host_ms;    /* host layout (binomial tree), uploads, launches     */
    double seconds;    /* wall time of the whole call (RunStats.seconds)    */
    uint64_t kernel_launches; /* kernels this call launched                 */
    uint64_t device_bytes;    /* device memory held by the context          */
    uint64_t h2d_bytes;       /* host->device bytes this call copied        */
    uint64_t d2h_bytes;       /* device->host bytes this call copied        */
    double pairs_ms;          /* the sparse engine (slab join + tail kernels, dominant) */
    uint64_t stream_comps;    /* predicate tests of the sparse engine (slab join + tail) */
    uint64_t dense_comps;     /* predicate tests of the dense engine (global + wide-window requests) */
    /* ChunkStats::*_by_annulus (sweep.hpp:160, 472, 530-539; generator.hpp:82-98) of this shard:
     * tests and edges counted for the node's annulus (global unit: the larger annulus of the
     * pair), vertices for their home annulus (global points on rank 0).  Entries [0, annuli).
     * annulus_edges / annulus_comps are filled (per_annulus = 1) by the calls that also track
     * degrees or materialise edges — the `stats` path; the counters-only path skips them. */
    uint32_t per_annulus, pad_;
    uint64_t annulus_edges[RHG_MAX_ANNULI];
    uint64_t annulus_comps[RHG_MAX_ANNULI];
    uint64_t annulus_vertices[RHG_MAX_ANNULI];
    /* >= 1: edges / fingerprint / comps (and the per-family and per-annulus counters) are the
     * WHOLE graph's: this call ended with the NCCL all-reduce over `reduced_world` shards
     * (device_ms includes it).  0: no collective ran; the counters are this shard's. */
    uint32_t reduced_world, pad2_;
} rhg_run_stats;

/* Host-side shard plan (no device needed): rank r of `world` owns engines (angular chunks)
 * [chunk_begin, chunk_end), draws its owned streaming points, the halo chunk's points
 * (regenerated from the hash seeds, no communication) and every global point. */
typedef struct {
    uint32_t chunk_begin, chunk_end;
    uint64_t owned_points;   /* streaming points of the owned chunks                */
    uint64_t halo_points;    /* streaming points of chunk chunk_end mod P (the halo)  */
    uint64_t global_points;  /* clique + global annuli (every rank draws them)       */
    uint64_t sampled_points; /* owned + halo + global                                */
    uint64_t device_point_bytes; /* approximate device bytes of the point arrays      */
} rhg_shard_info;

/* Host point arrays in vertex-id order (n entries each; any may be NULL
 * where a call documents it as optional). */
typedef struct {
    double* beta;       /* sorted begin angle (PointDraw.beta)         */
    double* r;          /* radius                                       */
    double* theta;      /* node angle in [0, 2pi)                       */
    double* half_width; /* request half-width in the home annulus       */
    double* coth_r;
    double* inv_sinh_r;
    double* cos_theta;
    double* sin_theta;
} rhg_points;

const char* rhg_last_error(void);
int rhg_abi_version(void);

/* geometry.hpp:35-39 */
int rhg_alpha_from_gamma(double gamma, double* alpha);
/* geometry.hpp:26-33 */
int rhg_radial_const_from_avg_degree(double d_bar, double alpha, double* C);
/* geometry.hpp:57-67: validates and fills p->R */
int rhg_params_validate(rhg_params* p);
/* geometry.hpp:69-72 */
int rhg_params_from_avg_degree(uint64_t n, double alpha, double d_bar, uint64_t seed, uint32_t chunks,
                               rhg_params* out);
/* partition.hpp:233-240 make_layout, on the host (no device needed): *n_annuli and
 * *first_streaming always; when the arrays are non-NULL (room for n_annuli, resp.
 * n_annuli * chunks entries) the per-annulus vertex counts, the per-(annulus, chunk) counts
 * and first vertex ids (row-major by annulus) and the classes (0 clique, 1 global, 2
 * streaming).  Call once with NULL arrays to size them. */
int rhg_layout(const rhg_params* params, uint32_t* n_annuli, uint32_t* first_streaming, uint64_t* counts,
               uint64_t* chunk_counts, uint64_t* id_base, uint8_t* classes);

typedef struct rhg_ctx rhg_ctx;
int rhg_create(int device, rhg_ctx** out);
void rhg_destroy(rhg_ctx* ctx);

/* Multi-GPU, one process (GenOptions.workers mapped to GPUs, generator.hpp:27-32,
 * 245-268): one sub-context, stream and host thread per device and an NCCL communicator over
 * them (ncclCommInitAll).  rhg_generate_stats / rhg_count_edges_from_points on such a context
 * (shard NULL or {0, 1}) run shard {g, n_devices} on device g, end with one
 * ncclAllReduce(ncclUint64, sum) of the counters and return the whole graph
 * (reduced_world = n_devices; device_ms = the slowest device; degrees = summed).  Other calls
 * use devices[0].  Materialised edge streams need a single-device context. */
int rhg_create_multi(int n_devices, const int* devices, rhg_ctx** out);
/* Number of devices a context drives (1 for rhg_create). */
int rhg_context_devices(const rhg_ctx* ctx, int* n_devices);
/* Multi-GPU, one process per GPU: rank 0 creates an id (128 bytes), the caller distributes
 * it (e.g. a torch.distributed broadcast), every rank attaches it to its context.  Shard calls
 * with shard {rank, world} then end with the counter all-reduce and return the whole graph. */
int rhg_nccl_unique_id(uint8_t* id);
int rhg_attach_comm(rhg_ctx* ctx, uint32_t world, uint32_t rank, const uint8_t* id);
/* The shard plan of `shard` (host only): owned chunks and point counts. */
int rhg_shard_extent(const rhg_params* params, const rhg_shard* shard, rhg_shard_info* out);

/* generator.hpp:219-291 generate_stats.  `degrees` (optional, u32[n],
 * host) receives exact per-vertex degrees of the edges this shard emits. */
int rhg_generate_stats(rhg_ctx* ctx, const rhg_params* params, const rhg_shard* shard, rhg_run_stats* out,
                       uint32_t* degrees);

/* The device sampler alone: all n points, id order, copied to host arrays
 * (every field of `out` must be non-NULL).  Same streams as
 * ChunkPointSource (sweep.hpp:102-151). */
int rhg_sample_points(rhg_ctx* ctx, const rhg_params* params, rhg_points* out);

/* Diagnostic: the raw std::mt19937_64 uniforms (x >> 11) * 2^-53 of every
 * point's angle stream and radius stream (rng.hpp:58-69, seeds
 * derive_seed(seed, {3|4, annulus, chunk})), in id order, n entries each.
 * Integer-only, so bit-exact against the reference by construction. */
int rhg_sample_uniforms(rhg_ctx* ctx, const rhg_params* params, double* u_angle, double* u_radius);

/* Parity hook ("same points" mode): run the device edge kernels on a GIVEN
 * point set (host arrays, id order; r may be NULL) instead of the device
 * sampler.  With the reference's own points this must reproduce the
 * reference's edges / fingerprint / comps bit for bit. */
int rhg_count_edges_from_points(rhg_ctx* ctx, const rhg_params* params, const rhg_shard* shard,
                                const rhg_points* pts, rhg_run_stats* out, uint32_t* degrees);

/* Materialised edge stream (generator.hpp:135-215
 * generate(params, opts, edge_sink)).  Every edge this shard owns as a
 * canonical pair (u < v), `edges` = 2 * cap uint64 (u0, v0, u1, v1, ...),
 * sorted ascending by (u, v).  The reference emits the same multiset in its
 * unit / sweep order (its own tests compare sorted multisets, oracle.hpp:
 * 70-104).  *n_edges always receives the edge count; edges == NULL only
 * counts; cap < count fails with RHG_INVALID_ARGUMENT (retry with
 * cap >= *n_edges).  Requires n < 2^32 and < 2^31 edges per call. */
int rhg_generate_edges(rhg_ctx* ctx, const rhg_params* params, const rhg_shard* shard, rhg_run_stats* out,
                       uint64_t* edges, uint64_t cap, uint64_t* n_edges);
/* The same for a GIVEN point set ("same points" mode, as rhg_count_edges_from_points). */
int rhg_edges_from_points(rhg_ctx* ctx, const rhg_params* params, const rhg_shard* shard, const rhg_points* pts,
                          rhg_run_stats* out, uint64_t* edges, uint64_t cap, uint64_t* n_edges);

/* Per-unit counters of generate_stats (RunStats::unit_edges / unit_comps / unit_vertices,
 * generator.hpp:270-284; printed by RunReport::write_text, stats.hpp:189-195): unit 0 = the
 * global unit, unit c + 1 = chunk engine c.  Arrays of chunks + 1 entries.  Runs the P engine
 * shards {c, P} on the context's (first) device. */
int rhg_unit_stats(rhg_ctx* ctx, const rhg_params* params, uint64_t* unit_edges, uint64_t* unit_comps,
                   uint64_t* unit_vertices);
/* The edge stream in the reference's unit order (generator.hpp:183-199: the global unit first,
 * then chunk engines ascending), canonical pairs (u < v), each unit in (u, v) order (the
 * reference's order inside a unit follows its sweep's active-list slots).  unit_offsets
 * (chunks + 2 entries): unit u's pairs are [unit_offsets[u], unit_offsets[u + 1]).  Same
 * buffer protocol as rhg_generate_edges (edges == NULL only counts). */
int rhg_generate_edges_units(rhg_ctx* ctx, const rhg_params* params, uint64_t* edges, uint64_t cap, uint64_t* n_edges,
                             uint64_t* unit_offsets);

/* Brute-force oracle on the GPU (oracle.hpp:41-54 naive_edges): every pair
 * u < v of the n given points (host arrays, id order) with
 * hyperbolic_distance (geometry.hpp:117-123, direct formula) < R, as sorted
 * canonical pairs.  n > 100000 fails like the reference's guard.  Same buffer
 * protocol as rhg_generate_edges.  verify_against_oracle (oracle.hpp:70-111)
 * is built on it in the Python mirror. */
int rhg_naive_edges(rhg_ctx* ctx, uint64_t n, double R, const double* r, const double* theta, uint64_t* edges,
                    uint64_t cap, uint64_t* n_edges);

/* Edge stream file formats, byte-compatible with io.hpp:20-96:
 * text = one "u v\n" per edge (decimal); binary = 8-byte magic "RHGE0001"
 * then little-endian uint64 pairs, no length prefix.  Host-only. */
int rhg_write_edges_text(const char* path, const uint64_t* edges, uint64_t m);
int rhg_write_edges_binary(const char* path, const uint64_t* edges, uint64_t m);
/* io.hpp:70-96 read_binary_edges: bad magic / truncated pair -> RHG_INVALID_ARGUMENT
 * (std::runtime_error in the reference).  edges == NULL only counts. */
int rhg_read_edges_binary(const char* path, uint64_t* edges, uint64_t cap, uint64_t* m);
/* stats.hpp:58-75 powerlaw_mle over a degree array (host; same order and libm as the
 * reference).  Fewer than 100 degrees >= d_min -> RHG_INVALID_ARGUMENT. */
int rhg_powerlaw_mle(const uint32_t* degrees, uint64_t n, uint32_t d_min, double* gamma_hat);
/* message of the last failed edge-file / analytics call (this thread) */
const char* rhg_io_last_error(void);

/* Predicate audit (north_star / SURVEY 8(c) "borderline pairs"): one generate_stats of `shard` in
 * which the slab join (the only engine that does not evaluate the reference predicate
 * sweep.hpp:531-533 directly) also evaluates it, in FP64 and the reference's order, for every
 * pair its FP32 pre-filter decided.  disagreements must be 0 (a decided pair whose FP32 sign
 * differs from the reference's); max_err_over_tau is the largest |D32 - D64| / tau seen (< 1:
 * the pre-filter's error bound held, DESIGN 4.1).  The other engines evaluate the reference
 * predicate itself, so their device decisions equal the reference's by construction.
 * stats receives the call's RunStats (counters unchanged by the audit). */
typedef struct {
    uint64_t slab_pairs;          /* pairs tested by the slab join                             */
    uint64_t prefilter_decided;   /* ... decided by the FP32 pre-filter                        */
    uint64_t exact_recheck;       /* ... left to the exact FP64 predicate near the threshold    */
    uint64_t exact_only;          /* ... in groups whose windows run the exact predicate only  */
    uint64_t disagreements;       /* pre-filter decisions != reference predicate (must be 0)   */
    uint64_t noise_band_pairs;    /* slab pairs with |lhs - rhs| < 1e-15 (rounding-noise band) */
    uint64_t exact_engine_pairs;  /* pairs of the engines that evaluate the predicate directly */
    double max_err_over_tau;      /* max |D32 - D64| / tau over pre-filter decisions           */
} rhg_audit_report;
int rhg_audit_predicate(rhg_ctx* ctx, const rhg_params* params, const rhg_shard* shard, rhg_audit_report* out,
                        rhg_run_stats* stats);

/* Diagnostic (not part of the reference interface): measured non-FMA FP64
 * DMUL+DADD instruction rate of `device` (the edge kernels' roofline
 * denominator) and the dependent-DMUL latency in SM cycles. */
int rhg_fp64_peak(int device, double* ops_per_s, double* dmul_latency_cycles, double* kernel_ms);

/* Diagnostic (not part of the reference interface): the device restatement of the glibc 2.39
 * routines the reference's point set passes through (csrc/glibc_libm.cuh: std::exp, log, log1p,
 * acosh, acos, pow and the gcc-merged sincos of sweep.hpp:125-139, partition.hpp:66,
 * rng.hpp:221), evaluated elementwise on host arrays of n doubles on `device`:
 * fn 0 exp(x), 1 log(x), 2 log1p(x), 3 acosh(x), 4 acos(x), 5 pow(x, y), 6 sin(x), 7 cos(x)
 * (6/7: the two outputs of one sincos call; y is read only for fn 5).  The results must equal
 * the host glibc's bit for bit (tests/test_gpu_libm.py). */
int rhg_libm_eval(int device, int fn, const double* x, const double* y, double* out, uint64_t n);

#ifdef __cplusplus
}
#endif
#endif /* RHG_B200_H */
