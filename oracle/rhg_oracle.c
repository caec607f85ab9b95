/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference generator.
 *
 * Follows /root/reference/proj/include/rhg/ function by function (file:line
 * cited at each).  Compiled with -ffp-contract=off against the system glibc
 * libm, exactly like the reference (no -march => no FMA), so its arithmetic
 * is bit-identical to the reference's.  It is the checker for the B200 path
 * (tests/, smoke(), bench.py cpu_baseline) and is never linked into, called
 * by, or shipped with the product library.
 *
 * The sweep below is a faithful restatement of ChunkEngine (sweep.hpp:239-599)
 * — cells, begin/node tokens, propagation, Local/Foreign replica, early stop —
 * driven from point arrays instead of drawing, so that it can judge ANY point
 * set (the reference's own, or the one a device sampler produced).
 */
#define _GNU_SOURCE
#include "rhg_oracle.h"

#include <math.h>
#include <pthread.h>
#include <quadmath.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#include <unistd.h>

static const double TWO_PI = 6.283185307179586476925286766559; /* geometry.hpp:11 */
#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

static __thread char g_err[256];
const char* orc_last_error(void) { return g_err; }
static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

/* ------------------------------------------------------------------ rng --- */
/* rng.hpp:15-19 */
static uint64_t splitmix_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static const uint64_t GOLDEN_GAMMA = 0x9E3779B97F4A7C15ull; /* rng.hpp:20 */

/* rng.hpp:41-46 */
uint64_t orc_derive_seed(uint64_t root, const uint64_t* comps, uint32_t k) {
    uint64_t h = splitmix_mix(root + GOLDEN_GAMMA);
    for (uint32_t i = 0; i < k; ++i) h = splitmix_mix((h + GOLDEN_GAMMA) ^ comps[i]);
    return h;
}
static uint64_t seed3(uint64_t root, uint64_t a, uint64_t b, uint64_t c) {
    uint64_t p[3] = {a, b, c};
    return orc_derive_seed(root, p, 3);
}

/* std::mt19937_64 as specified by [rand.predef] (rng.hpp:58-69 uses it). */
#define MT_N 312
#define MT_M 156
typedef struct {
    uint64_t mt[MT_N];
    int idx;
} mt64;
static void mt_seed(mt64* g, uint64_t s) {
    g->mt[0] = s;
    for (int i = 1; i < MT_N; ++i) g->mt[i] = 6364136223846793005ull * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = MT_N;
}
static void mt_twist(mt64* g) {
    static const uint64_t mag[2] = {0ull, 0xB5026F5AA96619E9ull};
    const uint64_t UM = 0xFFFFFFFF80000000ull, LM = 0x7FFFFFFFull;
    int i;
    uint64_t x;
    for (i = 0; i < MT_N - MT_M; ++i) {
        x = (g->mt[i] & UM) | (g->mt[i + 1] & LM);
        g->mt[i] = g->mt[i + MT_M] ^ (x >> 1) ^ mag[x & 1];
    }
    for (; i < MT_N - 1; ++i) {
        x = (g->mt[i] & UM) | (g->mt[i + 1] & LM);
        g->mt[i] = g->mt[i + MT_M - MT_N] ^ (x >> 1) ^ mag[x & 1];
    }
    x = (g->mt[MT_N - 1] & UM) | (g->mt[0] & LM);
    g->mt[MT_N - 1] = g->mt[MT_M - 1] ^ (x >> 1) ^ mag[x & 1];
    g->idx = 0;
}
static uint64_t mt_next(mt64* g) {
    if (g->idx >= MT_N) mt_twist(g);
    uint64_t y = g->mt[g->idx++];
    y ^= (y >> 29) & 0x5555555555555555ull;
    y ^= (y << 17) & 0x71D67FFFEDA60000ull;
    y ^= (y << 37) & 0xFFF7EEE000000000ull;
    y ^= (y >> 43);
    return y;
}
void orc_mt_outputs(uint64_t seed, uint64_t count, uint64_t* out) {
    mt64 g;
    mt_seed(&g, seed);
    for (uint64_t i = 0; i < count; ++i) out[i] = mt_next(&g);
}
/* rng.hpp:63 */
static double uni(mt64* g) { return (double)(mt_next(g) >> 11) * 0x1.0p-53; }

/* rng.hpp:75-79 */
static double standard_normal(mt64* s) {
    const double u1 = 1.0 - uni(s);
    const double u2 = uni(s);
    return sqrt(-2.0 * log(u1)) * cos(TWO_PI * u2);
}
/* rng.hpp:82-96 */
static double gamma_variate(double a, mt64* s) {
    const double d = a - 1.0 / 3.0;
    const double c = 1.0 / sqrt(9.0 * d);
    for (;;) {
        const double x = standard_normal(s);
        const double t = 1.0 + c * x;
        if (t <= 0.0) continue;
        const double v = t * t * t;
        const double u = 1.0 - uni(s);
        if (log(u) < 0.5 * x * x + d - d * v + d * log(v)) return d * v;
    }
}
/* rng.hpp:98-103 */
static double beta_variate(double a, double b, mt64* s) {
    const double x = gamma_variate(a, s);
    const double y = gamma_variate(b, s);
    const double sum = x + y;
    return sum > 0.0 ? x / sum : 0.5;
}
/* rng.hpp:107-126 */
static uint64_t binomial_inversion(uint64_t n, double p, mt64* s) {
    const double u = uni(s);
    const double ratio_base = p / (1.0 - p);
    const double lpmf0 = (double)n * log1p(-p);
    uint64_t k = 0;
    double lpmf = lpmf0;
    while (lpmf <= -700.0 && k < n) {
        lpmf += log((double)(n - k) / (double)(k + 1) * ratio_base);
        ++k;
    }
    double pmf = exp(lpmf);
    double cum = 0.0;
    for (;; ++k) {
        cum += pmf;
        if (u < cum || k >= n) return k;
        pmf *= (double)(n - k) / (double)(k + 1) * ratio_base;
    }
}
/* rng.hpp:133-164 (caller validated p) */
static uint64_t binomial(uint64_t trials, double p, mt64* s) {
    int64_t base = 0, sign = 1;
    for (;;) {
        if (trials == 0 || p <= 0.0) return (uint64_t)base;
        if (p >= 1.0) return (uint64_t)(base + sign * (int64_t)trials);
        if (p > 0.5) {
            base += sign * (int64_t)trials;
            sign = -sign;
            p = 1.0 - p;
            continue;
        }
        if ((double)trials * p <= 1000.0) return (uint64_t)(base + sign * (int64_t)binomial_inversion(trials, p, s));
        const uint64_t m = (trials + 1) / 2;
        const double v = beta_variate((double)m, (double)(trials + 1 - m), s);
        if (v <= p) {
            base += sign * (int64_t)m;
            trials -= m;
            p = (p - v) / (1.0 - v);
        } else {
            trials = m - 1;
            p = p / v;
        }
    }
}
uint64_t orc_binomial(uint64_t trials, double p, uint64_t seed) {
    mt64 g;
    mt_seed(&g, seed);
    return binomial(trials, p, &g);
}

/* rng.hpp:209-244 SortedUniformStream */
typedef struct {
    mt64 g;
    uint64_t remaining;
    double a, b, width, cur_max;
} sorted_stream;
static void ss_init(sorted_stream* s, uint64_t count, double a, double b, uint64_t seed) {
    mt_seed(&s->g, seed);
    s->remaining = count;
    s->a = a;
    s->b = b;
    s->width = b - a;
    s->cur_max = 1.0;
}
static double ss_next(sorted_stream* s) {
    s->cur_max *= pow(uni(&s->g), 1.0 / (double)s->remaining);
    --s->remaining;
    double v = s->a + s->width * (1.0 - s->cur_max);
    if (v >= s->b) v = nextafter(s->b, s->a);
    return v;
}
void orc_sorted_uniforms(uint64_t count, double a, double b, uint64_t root, const uint64_t* comps, uint32_t k,
                         double* out) {
    sorted_stream s;
    ss_init(&s, count, a, b, orc_derive_seed(root, comps, k));
    for (uint64_t i = 0; i < count; ++i) out[i] = ss_next(&s);
}

/* ------------------------------------------------------------- geometry --- */
/* geometry.hpp:26-33 */
int orc_radial_const_from_avg_degree(double d_bar, double alpha, double* C) {
    if (!(alpha > 0.5)) return fail(ORC_INVALID_ARGUMENT, "radial_const_from_avg_degree: alpha must be > 1/2");
    if (!(d_bar > 0.0))
        return fail(ORC_INVALID_ARGUMENT, "radial_const_from_avg_degree: average degree must be positive");
    const double q = (alpha - 0.5) / alpha;
    *C = -2.0 * log(d_bar * M_PI / 2.0 * q * q);
    return ORC_OK;
}
/* geometry.hpp:35-39 */
int orc_alpha_from_gamma(double gamma, double* alpha) {
    if (!(gamma > 2.0)) return fail(ORC_INVALID_ARGUMENT, "alpha_from_gamma: gamma must be > 2");
    *alpha = (gamma - 1.0) / 2.0;
    return ORC_OK;
}
/* geometry.hpp:95-104 (NDEBUG: no assert) */
static double acos_clamped(double x) {
    if (x >= 1.0) return 0.0;
    if (x <= -1.0) return M_PI;
    return acos(x);
}
/* geometry.hpp:128-134 */
static double angular_deviation(double r, double b, double R) {
    if (r + b <= R) return M_PI;
    const double arg = (cosh(r) * cosh(b) - cosh(R)) / (sinh(r) * sinh(b));
    return acos_clamped(arg);
}
/* sweep.hpp:60-67 */
static double request_half_width_raw(double coth_r, double inv_sinh_r, double coth_b, double cRis_b) {
    const double arg = coth_r * coth_b - cRis_b * inv_sinh_r;
    if (arg <= -1.0) return M_PI;
    if (arg >= 1.0) return 0.0;
    return acos(arg);
}
/* sweep.hpp:80-85 */
static double chunk_lower_bound(uint32_t c, uint32_t P) { return (double)c * (TWO_PI / (double)P); }
static double chunk_upper_bound(uint32_t c, uint32_t P) {
    return c + 1 == P ? TWO_PI : (double)(c + 1) * (TWO_PI / (double)P);
}

/* ------------------------------------------------------------- layout ----- */
typedef struct {
    uint64_t n, seed;
    uint32_t chunks, count, first_streaming;
    double alpha, R, cosh_R, r_G;
    int has_clique;
    double *lower, *upper, *probs, *cal, *cau, *coth_lower, *cris, *cell_width;
    uint64_t *counts, *chunk_counts, *id_base, *cells;
    uint8_t* classes; /* 0 Clique, 1 Global, 2 Streaming */
} layout_t;

static void layout_free(layout_t* L) {
    free(L->lower), free(L->upper), free(L->probs), free(L->cal), free(L->cau), free(L->coth_lower), free(L->cris),
        free(L->cell_width), free(L->counts), free(L->chunk_counts), free(L->id_base), free(L->cells),
        free(L->classes);
    memset(L, 0, sizeof *L);
}

/* partition.hpp:142-156 */
static void split_chunk_range(layout_t* L, uint64_t seed, uint32_t annulus, uint64_t total, uint32_t lo, uint32_t hi,
                              uint64_t node, uint64_t* out) {
    if (hi - lo == 1) {
        out[lo] = total;
        return;
    }
    const uint32_t mid = lo + (hi - lo + 1) / 2;
    /* rng.hpp:197-204 split_count */
    const double ml = (double)(mid - lo), mr = (double)(hi - mid);
    mt64 g;
    mt_seed(&g, seed3(seed, 2, annulus, node));
    const uint64_t left = binomial(total, ml / (ml + mr), &g);
    split_chunk_range(L, seed, annulus, left, lo, mid, 2 * node, out);
    split_chunk_range(L, seed, annulus, total - left, mid, hi, 2 * node + 1, out);
}

/* geometry.hpp:57-67 + partition.hpp:88-240 */
static int make_layout(layout_t* L, uint64_t n, double alpha, double C, uint64_t seed, uint32_t chunks) {
    memset(L, 0, sizeof *L);
    const double R = 2.0 * log((double)n) + C; /* geometry.hpp:14-17 */
    if (n < 1) return fail(ORC_INVALID_ARGUMENT, "ModelParams: n must be >= 1");
    if (!(alpha > 0.5)) return fail(ORC_INVALID_ARGUMENT, "ModelParams: alpha must be > 1/2");
    if (!(R > 0.0)) return fail(ORC_INVALID_ARGUMENT, "ModelParams: R = 2 ln n + C must be positive");
    if (chunks < 1) return fail(ORC_INVALID_ARGUMENT, "ModelParams: chunk count must be >= 1");
    L->n = n, L->seed = seed, L->chunks = chunks, L->alpha = alpha, L->R = R;
    L->cosh_R = cosh(R);

    /* build_annuli, partition.hpp:97-119 */
    double kd = ceil(alpha * R / log(2.0));
    uint64_t k_equal = (uint64_t)kd;
    if (k_equal < 1) k_equal = 1;
    const double height = R / (double)k_equal;
    double* bounds = malloc((k_equal + 1) * sizeof(double));
    for (uint64_t j = 0; j <= k_equal; ++j) bounds[j] = (double)j * height;
    bounds[k_equal] = R;
    uint64_t merged = 0;
    while (merged + 1 < k_equal && bounds[merged + 1] <= R / 2.0) ++merged;
    L->has_clique = merged >= 1;
    const uint64_t first_upper = merged > 1 ? merged : 1;
    const uint32_t count = (uint32_t)(k_equal - first_upper + 1);
    L->count = count;
    L->lower = malloc(count * sizeof(double));
    L->upper = malloc(count * sizeof(double));
    L->lower[0] = 0.0;
    {
        uint32_t ui = 0, li = 1;
        for (uint64_t j = first_upper; j <= k_equal; ++j) {
            L->upper[ui++] = bounds[j];
            if (j < k_equal) L->lower[li++] = bounds[j];
        }
    }
    free(bounds);
    /* partition.hpp:121-137 */
    L->probs = malloc(count * sizeof(double));
    L->cal = malloc(count * sizeof(double));
    L->cau = malloc(count * sizeof(double));
    L->coth_lower = malloc(count * sizeof(double));
    L->cris = malloc(count * sizeof(double));
    const double denom = cosh(alpha * R) - 1.0;
    for (uint32_t i = 0; i < count; ++i) {
        const double cl = cosh(alpha * L->lower[i]);
        const double cu = cosh(alpha * L->upper[i]);
        L->cal[i] = cl;
        L->cau[i] = cu;
        L->probs[i] = (cu - cl) / denom;
        if (L->lower[i] > 0.0) {
            const double ex = exp(L->lower[i]);
            const double sh = 0.5 * (ex - 1.0 / ex);
            L->coth_lower[i] = 0.5 * (ex + 1.0 / ex) / sh;
            L->cris[i] = L->cosh_R / sh;
        } else {
            L->coth_lower[i] = INFINITY;
            L->cris[i] = INFINITY;
        }
    }
    /* assign_counts, partition.hpp:161-169 ; multinomial_counts rng.hpp:168-192 */
    L->counts = calloc(count, sizeof(uint64_t));
    {
        double sum = 0.0;
        for (uint32_t i = 0; i < count; ++i) {
            if (L->probs[i] < 0.0) return fail(ORC_INVALID_ARGUMENT, "multinomial_counts: negative probability");
            sum += L->probs[i];
        }
        if (fabs(sum - 1.0) > 1e-9)
            return fail(ORC_INVALID_ARGUMENT, "multinomial_counts: probabilities must sum to 1");
        mt64 g;
        uint64_t one = 1;
        mt_seed(&g, orc_derive_seed(seed, &one, 1));
        uint64_t remaining = n;
        double mass = 1.0;
        for (uint32_t i = 0; i + 1 < count; ++i) {
            double q;
            if (mass > 0.0) {
                const double x = L->probs[i] / mass;
                const double mx = (0.0 < x) ? x : 0.0; /* std::max(0.0, x) */
                q = (mx < 1.0) ? mx : 1.0;             /* std::min(1.0, .) */
            } else
                q = 1.0;
            if (!(q >= 0.0 && q <= 1.0)) return fail(ORC_INVALID_ARGUMENT, "binomial: p must lie in [0, 1]");
            L->counts[i] = binomial(remaining, q, &g);
            remaining -= L->counts[i];
            mass -= L->probs[i];
        }
        L->counts[count - 1] = remaining;
    }
    L->chunk_counts = calloc((size_t)count * chunks, sizeof(uint64_t));
    for (uint32_t i = 0; i < count; ++i)
        split_chunk_range(L, seed, i, L->counts[i], 0, chunks, 1, L->chunk_counts + (size_t)i * chunks);
    /* build_cell_grid, partition.hpp:173-189 (cell_target 8) */
    L->cells = malloc(count * sizeof(uint64_t));
    L->cell_width = malloc(count * sizeof(double));
    for (uint32_t i = 0; i < count; ++i) {
        uint64_t c = 1;
        if (L->counts[i] >= 8) {
            uint64_t q = L->counts[i] / 8;
            c = 1;
            while (c <= q / 2) c <<= 1; /* bit_floor */
        }
        L->cells[i] = c;
        L->cell_width[i] = TWO_PI / (double)c;
    }
    /* classify, partition.hpp:195-217 */
    L->classes = malloc(count);
    L->first_streaming = count;
    const double chunk_width = TWO_PI / (double)chunks;
    for (uint32_t i = 0; i < count; ++i) {
        L->classes[i] = 1;
        if (i == 0 && L->has_clique) {
            L->classes[i] = 0;
            continue;
        }
        const double l = L->lower[i];
        const double width = l > 0.0 ? 2.0 * angular_deviation(l, l, R) : TWO_PI;
        if (width <= chunk_width) {
            L->classes[i] = 2;
            if (L->first_streaming == count) L->first_streaming = i;
        }
    }
    L->r_G = L->first_streaming < count ? L->lower[L->first_streaming] : R;
    /* assign_vertex_ids, partition.hpp:220-231 */
    L->id_base = malloc((size_t)count * chunks * sizeof(uint64_t));
    uint64_t next = 0;
    for (uint32_t i = 0; i < count; ++i)
        for (uint32_t c = 0; c < chunks; ++c) {
            L->id_base[(size_t)i * chunks + c] = next;
            next += L->chunk_counts[(size_t)i * chunks + c];
        }
    return ORC_OK;
}

int orc_layout(uint64_t n, double alpha, double C, uint64_t seed, uint32_t chunks, uint32_t* count, double* dbl,
               uint64_t* counts, uint64_t* chunk_counts, uint64_t* id_base, uint64_t* cells, uint8_t* classes,
               double* scal) {
    layout_t L;
    int rc = make_layout(&L, n, alpha, C, seed, chunks);
    if (rc) {
        layout_free(&L);
        return rc;
    }
    *count = L.count;
    if (dbl) {
        const double* cols[8] = {L.lower, L.upper, L.probs, L.cal, L.cau, L.coth_lower, L.cris, L.cell_width};
        for (int k = 0; k < 8; ++k) memcpy(dbl + (size_t)k * L.count, cols[k], L.count * sizeof(double));
        memcpy(counts, L.counts, L.count * sizeof(uint64_t));
        memcpy(chunk_counts, L.chunk_counts, (size_t)L.count * chunks * sizeof(uint64_t));
        memcpy(id_base, L.id_base, (size_t)L.count * chunks * sizeof(uint64_t));
        memcpy(cells, L.cells, L.count * sizeof(uint64_t));
        memcpy(classes, L.classes, L.count);
        scal[0] = L.R, scal[1] = L.cosh_R, scal[2] = L.r_G, scal[3] = L.first_streaming;
    }
    layout_free(&L);
    return ORC_OK;
}

/* ------------------------------------------------------------- points ----- */
typedef struct {
    double *beta, *r, *theta, *hw, *coth, *inv, *cs, *sn;
} pts_t;

/* sweep.hpp:102-141 ChunkPointSource::next, one stream */
static void draw_stream(const layout_t* L, uint32_t i, uint32_t c, pts_t* P) {
    const uint64_t cnt = L->chunk_counts[(size_t)i * L->chunks + c];
    uint64_t id = L->id_base[(size_t)i * L->chunks + c];
    sorted_stream ang;
    ss_init(&ang, cnt, chunk_lower_bound(c, L->chunks), chunk_upper_bound(c, L->chunks), seed3(L->seed, 3, i, c));
    mt64 rad;
    mt_seed(&rad, seed3(L->seed, 4, i, c));
    for (uint64_t k = 0; k < cnt; ++k, ++id) {
        const double beta = ss_next(&ang);
        /* partition.hpp:64-70 radius_from_uniform */
        const double u = uni(&rad);
        const double cc = L->cal[i] + u * (L->cau[i] - L->cal[i]);
        double r = acosh(cc < 1.0 ? 1.0 : cc) / L->alpha;
        r = r > 1e-12 ? r : 1e-12;
        const double ex = exp(r);
        const double mex = 1.0 / ex;
        const double sh = 0.5 * (ex - mex);
        const double coth = 0.5 * (ex + mex) / sh;
        const double inv = 1.0 / sh;
        const double hw = L->lower[i] > 0.0 ? request_half_width_raw(coth, inv, L->coth_lower[i], L->cris[i]) : M_PI;
        double theta = beta + hw;
        if (theta >= TWO_PI) theta -= TWO_PI;
        P->beta[id] = beta;
        if (P->r) P->r[id] = r;
        P->theta[id] = theta;
        P->hw[id] = hw;
        P->coth[id] = coth;
        P->inv[id] = inv;
        P->cs[id] = cos(theta);
        P->sn[id] = sin(theta);
    }
}

typedef struct {
    const layout_t* L;
    pts_t* P;
    uint32_t w, W;
} draw_job;
static void* draw_worker(void* arg) {
    draw_job* j = arg;
    const uint64_t streams = (uint64_t)j->L->count * j->L->chunks;
    for (uint64_t s = j->w; s < streams; s += j->W) draw_stream(j->L, (uint32_t)(s / j->L->chunks), (uint32_t)(s % j->L->chunks), j->P);
    return NULL;
}
static uint32_t hw_threads(uint32_t t) {
    if (t) return t;
    long n = sysconf(_SC_NPROCESSORS_ONLN);
    return n > 0 ? (uint32_t)n : 1;
}
static void draw_all(const layout_t* L, pts_t* P, uint32_t threads) {
    threads = hw_threads(threads);
    pthread_t* th = malloc(threads * sizeof(pthread_t));
    draw_job* jobs = malloc(threads * sizeof(draw_job));
    for (uint32_t w = 0; w < threads; ++w) {
        jobs[w] = (draw_job){L, P, w, threads};
        pthread_create(&th[w], NULL, draw_worker, &jobs[w]);
    }
    for (uint32_t w = 0; w < threads; ++w) pthread_join(th[w], NULL);
    free(th), free(jobs);
}

int orc_points(uint64_t n, double alpha, double C, uint64_t seed, uint32_t chunks, uint32_t threads, double* beta,
               double* r, double* theta, double* half_width, double* coth_r, double* inv_sinh_r, double* cos_theta,
               double* sin_theta, uint32_t* annulus) {
    layout_t L;
    int rc = make_layout(&L, n, alpha, C, seed, chunks);
    if (rc) {
        layout_free(&L);
        return rc;
    }
    pts_t P = {beta, r, theta, half_width, coth_r, inv_sinh_r, cos_theta, sin_theta};
    draw_all(&L, &P, threads);
    if (annulus)
        for (uint32_t i = 0; i < L.count; ++i)
            for (uint64_t k = 0; k < L.counts[i]; ++k) annulus[L.id_base[(size_t)i * chunks] + k] = i;
    layout_free(&L);
    return ORC_OK;
}

/* -------------------------------------------------------------- sweep ----- */
/* sweep.hpp:181-199 tokens */
typedef struct {
    double begin, end, lambda, theta, coth, inv, cs, sn;
    uint64_t id;
    uint32_t home;
    uint8_t local, gclip;
} btok;
typedef struct {
    double lambda, theta, coth, inv, cs, sn;
    uint64_t id;
    uint32_t annulus;
    uint8_t local;
} ntok;
typedef struct {
    btok* v;
    size_t n, cap;
} bvec;
typedef struct {
    ntok* v;
    size_t n, cap;
} nvec;
static void bpush(bvec* b, const btok* t) {
    if (b->n == b->cap) {
        b->cap = b->cap ? 2 * b->cap : 8;
        b->v = realloc(b->v, b->cap * sizeof(btok));
    }
    b->v[b->n++] = *t;
}
static void npush(nvec* b, const ntok* t) {
    if (b->n == b->cap) {
        b->cap = b->cap ? 2 * b->cap : 8;
        b->v = realloc(b->v, b->cap * sizeof(ntok));
    }
    b->v[b->n++] = *t;
}

/* sweep.hpp:203-232 ActiveRequests */
typedef struct {
    double *begin, *end, *theta, *coth, *inv, *cs, *sn;
    uint64_t* id;
    int64_t* end_cell;
    uint32_t* home;
    uint8_t* local;
    size_t n, cap;
    uint32_t* freev;
    size_t nfree, capfree;
} active_t;
static uint32_t act_alloc(active_t* a) {
    if (a->nfree) return a->freev[--a->nfree];
    if (a->n == a->cap) {
        a->cap = a->cap ? 2 * a->cap : 16;
        a->begin = realloc(a->begin, a->cap * sizeof(double));
        a->end = realloc(a->end, a->cap * sizeof(double));
        a->theta = realloc(a->theta, a->cap * sizeof(double));
        a->coth = realloc(a->coth, a->cap * sizeof(double));
        a->inv = realloc(a->inv, a->cap * sizeof(double));
        a->cs = realloc(a->cs, a->cap * sizeof(double));
        a->sn = realloc(a->sn, a->cap * sizeof(double));
        a->id = realloc(a->id, a->cap * sizeof(uint64_t));
        a->end_cell = realloc(a->end_cell, a->cap * sizeof(int64_t));
        a->home = realloc(a->home, a->cap * sizeof(uint32_t));
        a->local = realloc(a->local, a->cap);
    }
    a->end_cell[a->n] = -1;
    return (uint32_t)a->n++;
}
static void act_free_slot(active_t* a, uint32_t s) {
    if (a->nfree == a->capfree) {
        a->capfree = a->capfree ? 2 * a->capfree : 16;
        a->freev = realloc(a->freev, a->capfree * sizeof(uint32_t));
    }
    a->freev[a->nfree++] = s;
}
static void act_destroy(active_t* a) {
    free(a->begin), free(a->end), free(a->theta), free(a->coth), free(a->inv), free(a->cs), free(a->sn), free(a->id),
        free(a->end_cell), free(a->home), free(a->local), free(a->freev);
}

/* A point stream read back from arrays: the (annulus, chunk) slice of ids. */
typedef struct {
    uint64_t next, end;
} src_t;

typedef struct {
    uint32_t annulus;
    double cw;
    int64_t first_cell, last_cell, cur_cell;
    src_t main_src, replica_src;
    bvec* bb;
    nvec* nb;
    active_t act;
} asweep;

typedef struct {
    uint64_t edges, comps, fp, streaming_vertices;
} cstats;

typedef struct {
    const layout_t* L;
    const pts_t* P;
    uint32_t chunk, next_chunk;
    double begin_a, lift, end_linear;
    asweep* a;
    uint32_t na;
    uint64_t pend_begins, pend_nodes, active_local, draws_left;
    int stop, err;
    cstats st;
    uint32_t* degrees;
    uint64_t* mat; /* optional [home annulus][node annulus] test counts */
} engine;

static void deg_add(uint32_t* d, uint64_t u, uint64_t v) {
    if (!d) return;
    __atomic_fetch_add(&d[u], 1u, __ATOMIC_RELAXED);
    __atomic_fetch_add(&d[v], 1u, __ATOMIC_RELAXED);
}

static void engine_init(engine* e, const layout_t* L, const pts_t* P, uint32_t chunk, uint32_t* degrees) {
    memset(e, 0, sizeof *e);
    e->L = L, e->P = P, e->chunk = chunk, e->next_chunk = (chunk + 1) % L->chunks, e->degrees = degrees;
    /* sweep.hpp:252-259 */
    e->lift = chunk + 1 == L->chunks ? TWO_PI : 0.0;
    e->begin_a = chunk_lower_bound(chunk, L->chunks);
    e->end_linear = e->lift + chunk_upper_bound(e->next_chunk, L->chunks);
    e->na = L->count - L->first_streaming;
    e->a = calloc(e->na ? e->na : 1, sizeof(asweep));
    for (uint32_t pos = 0; pos < e->na; ++pos) {
        const uint32_t i = L->first_streaming + pos;
        asweep* a = &e->a[pos];
        a->annulus = i;
        a->cw = L->cell_width[i];
        /* sweep.hpp:316-326 */
        const uint64_t b0 = L->id_base[(size_t)i * L->chunks + chunk];
        a->main_src = (src_t){b0, b0 + L->chunk_counts[(size_t)i * L->chunks + chunk]};
        const uint64_t b1 = L->id_base[(size_t)i * L->chunks + e->next_chunk];
        a->replica_src = (src_t){b1, b1 + L->chunk_counts[(size_t)i * L->chunks + e->next_chunk]};
        a->first_cell = (int64_t)(e->begin_a / a->cw);
        a->last_cell = (int64_t)(e->end_linear / a->cw) + 1;
        a->cur_cell = a->first_cell;
        const size_t nb = (size_t)(a->last_cell - a->first_cell + 1);
        a->bb = calloc(nb, sizeof(bvec));
        a->nb = calloc(nb, sizeof(nvec));
        e->draws_left += L->chunk_counts[(size_t)i * L->chunks + chunk];
    }
}
static void engine_destroy(engine* e) {
    for (uint32_t pos = 0; pos < e->na; ++pos) {
        asweep* a = &e->a[pos];
        const size_t nb = (size_t)(a->last_cell - a->first_cell + 1);
        for (size_t k = 0; k < nb; ++k) free(a->bb[k].v), free(a->nb[k].v);
        free(a->bb), free(a->nb);
        act_destroy(&a->act);
    }
    free(e->a);
}

static double half_width_in(const layout_t* L, double coth, double inv, uint32_t annulus) {
    if (L->lower[annulus] <= 0.0) return M_PI; /* sweep.hpp:365-370 */
    return request_half_width_raw(coth, inv, L->coth_lower[annulus], L->cris[annulus]);
}

/* sweep.hpp:372-386 */
static void enqueue_begin(engine* e, asweep* a, const btok* t) {
    int64_t cell = (int64_t)(t->begin / a->cw);
    if (cell > a->last_cell) {
        if (t->local) {
            e->err = fail(ORC_INVARIANT, "sweep: local request begins past the replicated chunk");
        }
        return;
    }
    if (cell < a->cur_cell) cell = a->cur_cell;
    bpush(&a->bb[cell - a->first_cell], t);
    if (t->local) ++e->pend_begins;
}
/* sweep.hpp:388-399 */
static void enqueue_node(engine* e, asweep* a, const ntok* t) {
    int64_t cell = (int64_t)(t->lambda / a->cw);
    if (cell > a->last_cell) {
        if (t->local) e->err = fail(ORC_INVARIANT, "sweep: local node lies past the replicated chunk");
        return;
    }
    if (cell < a->cur_cell) cell = a->cur_cell;
    npush(&a->nb[cell - a->first_cell], t);
    if (t->local) ++e->pend_nodes;
}
/* sweep.hpp:41-58 */
static int split_wraparound(double a, double b, double out[4]) {
    if (b - a >= TWO_PI) {
        out[0] = 0.0, out[1] = TWO_PI;
        return 1;
    }
    if (a < 0.0) {
        out[0] = a + TWO_PI, out[1] = TWO_PI, out[2] = 0.0, out[3] = b;
        return 2;
    }
    if (b > TWO_PI) {
        out[0] = a, out[1] = TWO_PI, out[2] = 0.0, out[3] = b - TWO_PI;
        return 2;
    }
    out[0] = a, out[1] = b;
    return 1;
}
/* sweep.hpp:404-432 */
static void enqueue_clipped(engine* e, asweep* a, double theta_raw, double hw, uint64_t gid, uint32_t ghome,
                            double coth, double inv, double cs, double sn, int local) {
    const uint32_t wc = local ? e->chunk : e->next_chunk;
    const double w0 = chunk_lower_bound(wc, e->L->chunks);
    const double w1 = chunk_upper_bound(wc, e->L->chunks);
    const double lift = local ? 0.0 : e->lift;
    double r[4];
    const int nr = split_wraparound(theta_raw - hw, theta_raw + hw, r);
    for (int k = 0; k < nr; ++k) {
        const double lo = r[2 * k] > w0 ? r[2 * k] : w0;         /* std::max(begin, w0) */
        const double hi = w1 < r[2 * k + 1] ? w1 : r[2 * k + 1]; /* std::min(end, w1)  */
        if (lo >= hi) continue;
        btok t = {lo + lift, hi + lift, theta_raw + lift, theta_raw, coth, inv, cs, sn, gid, ghome, (uint8_t)local, 1};
        enqueue_begin(e, a, &t);
    }
}
/* sweep.hpp:435-463 */
static void activate(engine* e, asweep* a, const btok* t) {
    active_t* act = &a->act;
    const uint32_t s = act_alloc(act);
    act->begin[s] = t->begin, act->end[s] = t->end, act->theta[s] = t->theta, act->coth[s] = t->coth,
    act->inv[s] = t->inv, act->cs[s] = t->cs, act->sn[s] = t->sn, act->id[s] = t->id, act->home[s] = t->home,
    act->local[s] = t->local;
    act->end_cell[s] = (int64_t)(t->end / a->cw);
    if (t->local) ++e->active_local;
    const uint32_t pos = a->annulus - e->L->first_streaming;
    if (!t->gclip && pos + 1 < e->na) {
        asweep* up = &e->a[pos + 1];
        const double hw = half_width_in(e->L, t->coth, t->inv, up->annulus);
        btok t2 = *t;
        t2.begin = t->lambda - hw;
        t2.end = t->lambda + hw;
        enqueue_begin(e, up, &t2);
    }
}
/* sweep.hpp:465-507 */
static void draw_point(engine* e, asweep* a, src_t* src, int local) {
    const pts_t* P = e->P;
    const uint64_t id = src->next++;
    const double lift = local ? 0.0 : e->lift;
    if (local) {
        ++e->st.streaming_vertices;
        --e->draws_left;
    }
    btok t;
    t.begin = P->beta[id] + lift;
    t.end = t.begin + 2.0 * P->hw[id];
    t.lambda = t.begin + P->hw[id];
    t.theta = P->theta[id];
    t.coth = P->coth[id], t.inv = P->inv[id], t.cs = P->cs[id], t.sn = P->sn[id];
    t.id = id, t.home = a->annulus, t.local = (uint8_t)local, t.gclip = 0;
    if (local && t.end > e->end_linear + 1e-9)
        e->err = fail(ORC_INVARIANT, "sweep: local request wider than the replication window");
    ntok nd = {t.lambda, t.theta, t.coth, t.inv, t.cs, t.sn, id, a->annulus, (uint8_t)local};
    activate(e, a, &t);
    enqueue_node(e, a, &nd);
}
/* threshold-borderline audit (orc_borderline; NULL/0 when off) */
static struct {
    int on;
    double band;
    const double *r, *theta;
    __float128 R, coshR;
    uint64_t band_pairs, to_edge, to_nonedge, border, cap, listed;
    double max_flip_dmr; /* largest |d - R| of a pair whose decision flips */
    uint64_t *u, *v;
    double* dmr;
    uint8_t* dec;
    pthread_mutex_t mu;
} g_bd;

/* geometry.hpp:117-123 in binary128 for a pair whose FP64 predicate value is within the band */
static void border_check(uint64_t a, uint64_t b, double lhs, double rhs, double cab, double iab, int ref_edge) {
    const double scale = fabs(lhs) + fabs(cab) + fabs(iab) + 1.0;
    if (!(fabs(lhs - rhs) <= g_bd.band * scale)) return;
    __atomic_fetch_add(&g_bd.band_pairs, 1, __ATOMIC_RELAXED);
    const double ra = g_bd.r[a], rb = g_bd.r[b];
    const __float128 r1 = ra < rb ? ra : rb, r2 = ra < rb ? rb : ra;
    const __float128 dth = fabsq((__float128)g_bd.theta[a] - (__float128)g_bd.theta[b]);
    const __float128 arg = coshq(r2 - r1) + (1 - cosq(dth)) * sinhq(r1) * sinhq(r2);
    const int exact_edge = arg < g_bd.coshR;
    if (exact_edge != ref_edge) {
        __atomic_fetch_add(exact_edge ? &g_bd.to_edge : &g_bd.to_nonedge, 1, __ATOMIC_RELAXED);
        const double dmr = fabs((double)(acoshq(arg < 1 ? 1 : arg) - g_bd.R));
        pthread_mutex_lock(&g_bd.mu);
        if (dmr > g_bd.max_flip_dmr) g_bd.max_flip_dmr = dmr;
        pthread_mutex_unlock(&g_bd.mu);
    }
    if (fabsq(arg / g_bd.coshR - 1) < 1e-9Q) {
        const double dmr = (double)(acoshq(arg < 1 ? 1 : arg) - g_bd.R);
        if (fabs(dmr) < 1e-12) {
            __atomic_fetch_add(&g_bd.border, 1, __ATOMIC_RELAXED);
            pthread_mutex_lock(&g_bd.mu);
            if (g_bd.listed < g_bd.cap) {
                const uint64_t k = g_bd.listed++;
                g_bd.u[k] = a < b ? a : b, g_bd.v[k] = a < b ? b : a, g_bd.dmr[k] = dmr, g_bd.dec[k] = (uint8_t)ref_edge;
            }
            pthread_mutex_unlock(&g_bd.mu);
        }
    }
}

/* sweep.hpp:509-543 — the predicate, evaluated in the reference's order */
static void match_node(engine* e, asweep* a, const ntok* nd) {
    active_t* act = &a->act;
    const double cosh_R = e->L->cosh_R;
    for (size_t i = 0; i < act->n; ++i) {
        if (act->end_cell[i] < 0) continue;
        if (nd->lambda < act->begin[i] || nd->lambda >= act->end[i]) continue;
        if (act->id[i] == nd->id) continue;
        if (act->home[i] == nd->annulus) {
            if (act->theta[i] > nd->theta) continue;
            if (act->theta[i] == nd->theta && act->id[i] > nd->id) continue;
        }
        if (!act->local[i] && !nd->local) continue;
        ++e->st.comps;
        if (e->mat) __atomic_fetch_add(&e->mat[(size_t)act->home[i] * e->L->count + nd->annulus], 1, __ATOMIC_RELAXED);
        const double lhs = act->cs[i] * nd->cs + act->sn[i] * nd->sn;
        const double rhs = act->coth[i] * nd->coth - cosh_R * act->inv[i] * nd->inv;
        if (g_bd.on)
            border_check(act->id[i], nd->id, lhs, rhs, act->coth[i] * nd->coth, cosh_R * act->inv[i] * nd->inv,
                         lhs > rhs);
        if (lhs > rhs) {
            const uint64_t u = act->id[i] < nd->id ? act->id[i] : nd->id;
            const uint64_t v = act->id[i] < nd->id ? nd->id : act->id[i];
            ++e->st.edges;
            e->st.fp += u + v;
            deg_add(e->degrees, u, v);
        }
    }
}
/* sweep.hpp:545-557 */
static void reclaim(engine* e, asweep* a) {
    active_t* act = &a->act;
    for (size_t i = 0; i < act->n; ++i)
        if (act->end_cell[i] >= 0 && act->end_cell[i] < a->cur_cell) {
            act->end_cell[i] = -1;
            act_free_slot(act, (uint32_t)i);
            if (act->local[i]) --e->active_local;
        }
}
/* sweep.hpp:559-598 */
static void process_cell(engine* e, asweep* a) {
    const double cell_end = (double)(a->cur_cell + 1) * a->cw;
    reclaim(e, a);
    while (a->main_src.next < a->main_src.end && e->P->beta[a->main_src.next] < cell_end)
        draw_point(e, a, &a->main_src, 1);
    while (a->replica_src.next < a->replica_src.end && e->P->beta[a->replica_src.next] + e->lift < cell_end)
        draw_point(e, a, &a->replica_src, 0);
    bvec* bb = &a->bb[a->cur_cell - a->first_cell];
    for (size_t k = 0; k < bb->n; ++k) {
        if (bb->v[k].local) --e->pend_begins;
        activate(e, a, &bb->v[k]);
    }
    free(bb->v);
    memset(bb, 0, sizeof *bb);
    nvec* nb = &a->nb[a->cur_cell - a->first_cell];
    for (size_t k = 0; k < nb->n; ++k) {
        if (nb->v[k].local) --e->pend_nodes;
        match_node(e, a, &nb->v[k]);
    }
    free(nb->v);
    memset(nb, 0, sizeof *nb);
    ++a->cur_cell;
    if (e->draws_left == 0 && e->pend_begins == 0 && e->pend_nodes == 0 && e->active_local == 0) e->stop = 1;
}
static int done(const asweep* a) { return a->cur_cell > a->last_cell; }
/* sweep.hpp:354-363 */
static int allowed(const engine* e, uint32_t pos) {
    const asweep* a = &e->a[pos];
    const asweep* below = &e->a[pos - 1];
    if (done(below)) return 1;
    const uint64_t ca = e->L->cells[a->annulus], cb = e->L->cells[below->annulus];
    if (ca >= cb) return below->cur_cell * (int64_t)(ca / cb) >= a->cur_cell + 1;
    return below->cur_cell >= (a->cur_cell + 1) * (int64_t)(cb / ca);
}
/* sweep.hpp:272-302, Schedule::RoundRobin (the GenOptions default) */
static void engine_run(engine* e) {
    if (e->na == 0) return;
    while (!e->stop) {
        int progress = 0;
        for (uint32_t pos = 0; pos < e->na && !e->stop; ++pos) {
            asweep* a = &e->a[pos];
            if (done(a)) continue;
            if (pos == 0) {
                process_cell(e, a);
                progress = 1;
                continue;
            }
            while (!done(a) && !e->stop && allowed(e, pos)) {
                process_cell(e, a);
                progress = 1;
            }
        }
        if (!progress) break;
    }
    if (!e->stop && e->active_local > 0)
        e->err = fail(ORC_INVARIANT, "sweep: a local request survived past the replicated chunk");
}

/* ---------------------------------------------------------- generator ----- */
typedef struct {
    const layout_t* L;
    const pts_t* P;
    uint64_t g_begin, g_end; /* global points = ids [0, nG) */
    double* ghw;             /* [g * ns + pos] */
    uint32_t ns;
    uint32_t w, W;
    cstats st, gst;
    uint32_t* degrees;
    uint64_t* mat;
    uint32_t e0, e1;         /* engines [e0, e1) */
    uint32_t grank, gworld;  /* global-unit rows i with i % gworld == grank */
    int err;
    char errmsg[256];
} unit_job;

/* generator.hpp:77-104 (unit 0) — pairs split over workers by row */
static void global_unit_rows(unit_job* j) {
    const pts_t* P = j->P;
    const double cosh_R = j->L->cosh_R;
    for (uint64_t i = j->w; i < j->g_end; i += j->W) {
        if (i % j->gworld != j->grank) continue;
        for (uint64_t k = i + 1; k < j->g_end; ++k) {
            ++j->gst.comps;
            const double lhs = P->cs[i] * P->cs[k] + P->sn[i] * P->sn[k];
            const double rhs = P->coth[i] * P->coth[k] - cosh_R * P->inv[i] * P->inv[k];
            if (g_bd.on)
                border_check(i, k, lhs, rhs, P->coth[i] * P->coth[k], cosh_R * P->inv[i] * P->inv[k], lhs > rhs);
            if (lhs > rhs) {
                ++j->gst.edges;
                j->gst.fp += i + k;
                deg_add(j->degrees, i, k);
            }
        }
    }
}
/* generator.hpp:106-114 + sweep.hpp:265-270 */
static void* unit_worker(void* arg) {
    unit_job* j = arg;
    const layout_t* L = j->L;
    global_unit_rows(j);
    for (uint32_t c = j->e0 + j->w; c < j->e1; c += j->W) {
        engine e;
        engine_init(&e, L, j->P, c, j->degrees);
        e.mat = j->mat;
        for (uint64_t g = 0; g < j->g_end; ++g) {
            /* global point g's home annulus */
            uint32_t home = 0;
            while (home + 1 < L->count && L->id_base[(size_t)(home + 1) * L->chunks] <= g) ++home;
            for (uint32_t pos = 0; pos < e.na; ++pos) {
                const double hw = j->ghw[g * j->ns + pos];
                enqueue_clipped(&e, &e.a[pos], j->P->theta[g], hw, g, home, j->P->coth[g], j->P->inv[g],
                                j->P->cs[g], j->P->sn[g], 1);
                enqueue_clipped(&e, &e.a[pos], j->P->theta[g], hw, g, home, j->P->coth[g], j->P->inv[g],
                                j->P->cs[g], j->P->sn[g], 0);
            }
        }
        if (!e.err) engine_run(&e);
        j->st.edges += e.st.edges, j->st.comps += e.st.comps, j->st.fp += e.st.fp,
            j->st.streaming_vertices += e.st.streaming_vertices;
        if (e.err && !j->err) {
            j->err = e.err;
            snprintf(j->errmsg, sizeof j->errmsg, "%s", g_err);
        }
        engine_destroy(&e);
    }
    return NULL;
}

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

static uint64_t* g_mat = NULL; /* diagnostics only (orc_comps_matrix) */
static int run_units_shard(const layout_t* L, const pts_t* P, uint32_t threads, orc_stats* out, uint32_t* degrees,
                           uint32_t rank, uint32_t world);
static int run_units(const layout_t* L, const pts_t* P, uint32_t threads, orc_stats* out, uint32_t* degrees) {
    return run_units_shard(L, P, threads, out, degrees, 0, 1);
}
static int run_units_shard(const layout_t* L, const pts_t* P, uint32_t threads, orc_stats* out, uint32_t* degrees,
                           uint32_t rank, uint32_t world) {
    const uint64_t nG = L->first_streaming < L->count ? L->id_base[(size_t)L->first_streaming * L->chunks] : L->n;
    const uint32_t ns = L->count - L->first_streaming;
    /* generator.hpp:58-72: per-global half-widths in every streaming annulus */
    double* ghw = malloc((nG * ns + 1) * sizeof(double));
    for (uint64_t g = 0; g < nG; ++g)
        for (uint32_t pos = 0; pos < ns; ++pos)
            ghw[g * ns + pos] = half_width_in(L, P->coth[g], P->inv[g], L->first_streaming + pos);
    threads = hw_threads(threads);
    pthread_t* th = malloc(threads * sizeof(pthread_t));
    unit_job* jobs = calloc(threads, sizeof(unit_job));
    for (uint32_t w = 0; w < threads; ++w) {
        jobs[w].L = L, jobs[w].P = P, jobs[w].g_end = nG, jobs[w].ghw = ghw, jobs[w].ns = ns, jobs[w].w = w,
        jobs[w].W = threads, jobs[w].degrees = degrees, jobs[w].mat = g_mat;
        jobs[w].e0 = (uint32_t)((uint64_t)L->chunks * rank / world);
        jobs[w].e1 = (uint32_t)((uint64_t)L->chunks * (rank + 1) / world);
        jobs[w].grank = rank, jobs[w].gworld = world;
        pthread_create(&th[w], NULL, unit_worker, &jobs[w]);
    }
    memset(out, 0, sizeof *out);
    int err = 0;
    char msg[256] = {0};
    for (uint32_t w = 0; w < threads; ++w) {
        pthread_join(th[w], NULL);
        out->edges += jobs[w].st.edges + jobs[w].gst.edges;
        out->comps += jobs[w].st.comps + jobs[w].gst.comps;
        out->fingerprint += jobs[w].st.fp + jobs[w].gst.fp;
        out->streaming_vertices += jobs[w].st.streaming_vertices;
        out->global_edges += jobs[w].gst.edges;
        out->global_comps += jobs[w].gst.comps;
        if (jobs[w].err && !err) err = jobs[w].err, memcpy(msg, jobs[w].errmsg, sizeof msg);
    }
    free(th), free(jobs), free(ghw);
    out->global_vertices = nG;
    out->annuli = L->count;
    out->first_streaming = L->first_streaming;
    out->R = L->R, out->r_G = L->r_G, out->cosh_R = L->cosh_R;
    if (err) return fail(err, msg);
    return ORC_OK;
}

int orc_generate_stats(uint64_t n, double alpha, double C, uint64_t seed, uint32_t chunks, uint32_t threads,
                       orc_stats* out, uint32_t* degrees) {
    const double t0 = now_s();
    layout_t L;
    int rc = make_layout(&L, n, alpha, C, seed, chunks);
    if (rc) {
        layout_free(&L);
        return rc;
    }
    pts_t P;
    double* buf = malloc(8 * n * sizeof(double));
    if (!buf) {
        layout_free(&L);
        return fail(ORC_NOMEM, "oracle: out of memory");
    }
    P.beta = buf, P.r = NULL, P.theta = buf + n, P.hw = buf + 2 * n, P.coth = buf + 3 * n, P.inv = buf + 4 * n,
    P.cs = buf + 5 * n, P.sn = buf + 6 * n;
    draw_all(&L, &P, threads);
    if (degrees) memset(degrees, 0, n * sizeof(uint32_t));
    rc = run_units(&L, &P, threads, out, degrees);
    free(buf);
    layout_free(&L);
    out->seconds = now_s() - t0;
    return rc;
}

int orc_count_edges_from_points(uint64_t n, double alpha, double C, uint64_t seed, uint32_t chunks,
                                uint32_t threads, const double* beta, const double* theta, const double* half_width,
                                const double* coth_r, const double* inv_sinh_r, const double* cos_theta,
                                const double* sin_theta, orc_stats* out, uint32_t* degrees) {
    const double t0 = now_s();
    layout_t L;
    int rc = make_layout(&L, n, alpha, C, seed, chunks);
    if (rc) {
        layout_free(&L);
        return rc;
    }
    pts_t P = {(double*)beta, NULL, (double*)theta, (double*)half_width, (double*)coth_r, (double*)inv_sinh_r,
               (double*)cos_theta, (double*)sin_theta};
    if (degrees) memset(degrees, 0, n * sizeof(uint32_t));
    rc = run_units(&L, &P, threads, out, degrees);
    layout_free(&L);
    out->seconds = now_s() - t0;
    return rc;
}

/* Diagnostics: distance computations per (request home annulus, node
 * annulus) of the chunk sweeps; mat must hold annuli*annuli u64 (query the
 * annulus count with orc_layout first).  Not thread-safe across calls. */
int orc_comps_matrix(uint64_t n, double alpha, double C, uint64_t seed, uint32_t chunks, uint32_t threads,
                     uint64_t* mat) {
    orc_stats st;
    g_mat = mat;
    int rc = orc_generate_stats(n, alpha, C, seed, chunks, threads, &st, NULL);
    g_mat = NULL;
    return rc;
}

/* One engine shard (rank of world): engines [rank*P/world, (rank+1)*P/world)
 * and the global-unit rows i % world == rank.  Shards sum to the whole graph. */
int orc_generate_stats_shard(uint64_t n, double alpha, double C, uint64_t seed, uint32_t chunks, uint32_t rank,
                             uint32_t world, uint32_t threads, orc_stats* out) {
    if (world < 1 || rank >= world) return fail(ORC_INVALID_ARGUMENT, "shard: rank must lie in [0, world)");
    const double t0 = now_s();
    layout_t L;
    int rc = make_layout(&L, n, alpha, C, seed, chunks);
    if (rc) {
        layout_free(&L);
        return rc;
    }
    double* buf = malloc(8 * n * sizeof(double));
    pts_t P = {buf, NULL, buf + n, buf + 2 * n, buf + 3 * n, buf + 4 * n, buf + 5 * n, buf + 6 * n};
    draw_all(&L, &P, threads);
    rc = run_units_shard(&L, &P, threads, out, NULL, rank, world);
    free(buf);
    layout_free(&L);
    out->seconds = now_s() - t0;
    return rc;
}

/* Threshold-borderline audit of shard (rank, world): see rhg_oracle.h.  Not re-entrant. */
int orc_borderline(uint64_t n, double alpha, double C, uint64_t seed, uint32_t chunks, uint32_t rank, uint32_t world,
                   uint32_t threads, double band, uint64_t cap, orc_border* out, uint64_t* u, uint64_t* v,
                   double* d_minus_R, uint8_t* ref_edge) {
    if (world < 1 || rank >= world) return fail(ORC_INVALID_ARGUMENT, "shard: rank must lie in [0, world)");
    const double t0 = now_s();
    layout_t L;
    int rc = make_layout(&L, n, alpha, C, seed, chunks);
    if (rc) {
        layout_free(&L);
        return rc;
    }
    double* buf = malloc(8 * n * sizeof(double));
    if (!buf) {
        layout_free(&L);
        return fail(ORC_NOMEM, "oracle: out of memory");
    }
    pts_t P = {buf, buf + 7 * n, buf + n, buf + 2 * n, buf + 3 * n, buf + 4 * n, buf + 5 * n, buf + 6 * n};
    draw_all(&L, &P, threads);
    memset(&g_bd, 0, sizeof g_bd);
    pthread_mutex_init(&g_bd.mu, NULL);
    g_bd.band = band, g_bd.r = P.r, g_bd.theta = P.theta, g_bd.R = L.R, g_bd.coshR = coshq((__float128)L.R);
    g_bd.cap = cap, g_bd.u = u, g_bd.v = v, g_bd.dmr = d_minus_R, g_bd.dec = ref_edge;
    g_bd.on = 1;
    orc_stats st;
    rc = run_units_shard(&L, &P, threads, &st, NULL, rank, world);
    g_bd.on = 0;
    memset(out, 0, sizeof *out);
    out->comps = st.comps, out->edges = st.edges;
    out->band_pairs = g_bd.band_pairs, out->flips_to_edge = g_bd.to_edge, out->flips_to_nonedge = g_bd.to_nonedge;
    out->border_pairs = g_bd.border, out->listed = g_bd.listed, out->max_flip_dmr = g_bd.max_flip_dmr;
    pthread_mutex_destroy(&g_bd.mu);
    free(buf);
    layout_free(&L);
    out->seconds = now_s() - t0;
    return rc;
}

/* ---- host libm evaluator (checker for the device glibc restatement) ---- */
typedef struct {
    int fn;
    const double *x, *y;
    double* out;
    uint64_t lo, hi;
} libm_job;

/* volatile pointers: the calls must reach libm.so.6's ifunc-selected entry
 * points, exactly as the reference's do (no builtin folding or inlining). */
static double (*volatile lm_exp)(double) = exp;
static double (*volatile lm_log)(double) = log;
static double (*volatile lm_log1p)(double) = log1p;
static double (*volatile lm_acosh)(double) = acosh;
static double (*volatile lm_acos)(double) = acos;
static double (*volatile lm_pow)(double, double) = pow;
static void (*volatile lm_sincos)(double, double*, double*) = sincos;

static void* libm_worker(void* arg) {
    libm_job* j = (libm_job*)arg;
    for (uint64_t i = j->lo; i < j->hi; ++i) {
        const double a = j->x[i];
        double r = 0.0, s, c;
        switch (j->fn) {
        case 0: r = lm_exp(a); break;
        case 1: r = lm_log(a); break;
        case 2: r = lm_log1p(a); break;
        case 3: r = lm_acosh(a); break;
        case 4: r = lm_acos(a); break;
        case 5: r = lm_pow(a, j->y[i]); break;
        default: lm_sincos(a, &s, &c); r = j->fn == 6 ? s : c; break;
        }
        j->out[i] = r;
    }
    return NULL;
}

void orc_libm_eval(int fn, const double* x, const double* y, double* out, uint64_t n, uint32_t threads) {
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t th[256];
    libm_job jobs[256];
    for (uint32_t t = 0; t < threads; ++t) {
        jobs[t] = (libm_job){fn, x, y, out, n * t / threads, n * (t + 1) / threads};
        pthread_create(&th[t], NULL, libm_worker, &jobs[t]);
    }
    for (uint32_t t = 0; t < threads; ++t) pthread_join(th[t], NULL);
}
