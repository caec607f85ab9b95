/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference's
 * threshold-RHG generator (/root/reference/proj/include/rhg/*.hpp), used as
 * the CPU checker for the B200 path.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load it; the product never does.
 *
 * Pinned against the reference itself (oracle/_ref, built in place from the
 * reference headers) and against the committed golden vectors in
 * tests/golden/ — see tests/test_oracle.py.
 */
#ifndef RHG_ORACLE_H
#define RHG_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_OK 0
#define ORC_INVALID_ARGUMENT 1
#define ORC_INVARIANT 2
#define ORC_NOMEM 3

const char* orc_last_error(void);

/* geometry.hpp:26-39 */
int orc_radial_const_from_avg_degree(double d_bar, double alpha, double* C);
int orc_alpha_from_gamma(double gamma, double* alpha);

/* rng.hpp:15-69 known-answer hooks */
uint64_t orc_derive_seed(uint64_t root, const uint64_t* comps, uint32_t k);
void orc_mt_outputs(uint64_t seed, uint64_t count, uint64_t* out);
void orc_sorted_uniforms(uint64_t count, double a, double b, uint64_t root, const uint64_t* comps, uint32_t k,
                         double* out);
uint64_t orc_binomial(uint64_t trials, double p, uint64_t seed);

/* partition.hpp:233-240 make_layout — same buffer convention as
 * ref_layout in oracle/ref_harness.cpp. */
int orc_layout(uint64_t n, double alpha, double C, uint64_t seed, uint32_t chunks, uint32_t* count, double* dbl,
               uint64_t* counts, uint64_t* chunk_counts, uint64_t* id_base, uint64_t* cells, uint8_t* classes,
               double* scal);

/* sweep.hpp:102-151 ChunkPointSource, all n points in id order. */
int orc_points(uint64_t n, double alpha, double C, uint64_t seed, uint32_t chunks, uint32_t threads, double* beta,
               double* r, double* theta, double* half_width, double* coth_r, double* inv_sinh_r,
               double* cos_theta, double* sin_theta, uint32_t* annulus);

/* Result block of a run (generator.hpp:34-46 RunStats subset). */
typedef struct {
    uint64_t edges, fingerprint, comps;
    uint64_t global_vertices, streaming_vertices;
    uint64_t global_edges, global_comps; /* unit 0 */
    uint32_t annuli, first_streaming;
    double R, r_G, cosh_R, seconds;
} orc_stats;

/* generator.hpp:219-291 generate_stats with the oracle's own sampler.
 * degrees: optional u32[n] (exact per-vertex degree). */
int orc_generate_stats(uint64_t n, double alpha, double C, uint64_t seed, uint32_t chunks, uint32_t threads,
                       orc_stats* out, uint32_t* degrees);

/* The same edge rule (global unit + every chunk sweep) applied to a GIVEN
 * point set in id order (e.g. the points a device sampler produced).  Layout
 * tables (counts, ids, classes, annulus constants) are recomputed from the
 * parameters; only the per-point attributes come from the arrays.  r is not
 * needed (the reference never uses r after drawing). */
int orc_count_edges_from_points(uint64_t n, double alpha, double C, uint64_t seed, uint32_t chunks,
                                uint32_t threads, const double* beta, const double* theta,
                                const double* half_width, const double* coth_r, const double* inv_sinh_r,
                                const double* cos_theta, const double* sin_theta, orc_stats* out,
                                uint32_t* degrees);

/* One engine shard: engines [rank*P/world, (rank+1)*P/world) and the
 * global-unit rows i % world == rank (partial results sum to the whole). */
int orc_generate_stats_shard(uint64_t n, double alpha, double C, uint64_t seed, uint32_t chunks, uint32_t rank,
                             uint32_t world, uint32_t threads, orc_stats* out);

/* Diagnostics: chunk-sweep tests per (request home annulus, node annulus). */
int orc_comps_matrix(uint64_t n, double alpha, double C, uint64_t seed, uint32_t chunks, uint32_t threads,
                     uint64_t* mat);

/* Threshold-borderline audit of one engine shard (north_star): every pair the
 * reference tests whose predicate value |lhs - rhs| lies within band x (its terms' magnitude)
 * -- the only pairs whose decision FP64 rounding can flip -- is re-decided with the exact
 * distance test d < R of geometry.hpp:117-123 evaluated in binary128 from (r, theta).
 * flips_* count decisions that differ (informational: the reference's own rounding);
 * border_pairs those with |d - R| < 1e-12, listed (u, v, d - R, reference decision) up to cap. */
typedef struct {
    uint64_t comps, edges;
    uint64_t band_pairs;       /* pairs re-decided in binary128                          */
    uint64_t flips_to_edge;    /* binary128: edge, reference predicate: no edge          */
    uint64_t flips_to_nonedge; /* binary128: no edge, reference predicate: edge          */
    uint64_t border_pairs;     /* |d - R| < 1e-12 (binary128)                            */
    uint64_t listed;
    double max_flip_dmr;       /* largest |d - R| among the flipped pairs                */
    double seconds;
} orc_border;
int orc_borderline(uint64_t n, double alpha, double C, uint64_t seed, uint32_t chunks, uint32_t rank, uint32_t world,
                   uint32_t threads, double band, uint64_t cap, orc_border* out, uint64_t* u, uint64_t* v,
                   double* d_minus_R, uint8_t* ref_edge);

/* The HOST glibc routines the reference calls, elementwise (the checker of
 * rhg_libm_eval): fn 0 exp, 1 log, 2 log1p, 3 acosh, 4 acos, 5 pow(x, y),
 * 6 / 7 sin / cos from one sincos call (what gcc -O3 makes of sweep.hpp:138-139). */
void orc_libm_eval(int fn, const double* x, const double* y, double* out, uint64_t n, uint32_t threads);

#ifdef __cplusplus
}
#endif
#endif
