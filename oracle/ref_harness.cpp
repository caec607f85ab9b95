// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// Thin extern "C" harness over the UNMODIFIED reference headers
// (/root/reference/proj/include/rhg/*.hpp, compiled in place with the
// reference's own flags: -std=c++20 -O3 -DNDEBUG, no -march, hence no FMA
// contraction — proj/CMakeLists.txt:1-20).  Built by oracle/Makefile into
// oracle/_ref/librhg_ref.so.  Used by tests/, tests/golden/make_golden.py and
// bench.py's reference arm / cpu_baseline leg, nothing else.
//
// Nothing here re-implements the reference: every entry point calls the
// reference's own functions.

#include <rhg/generator.hpp>
#include <rhg/io.hpp>
#include <rhg/stats.hpp>
#include <rhg/geometry.hpp>
#include <rhg/oracle.hpp>
#include <rhg/partition.hpp>
#include <rhg/sweep.hpp>

#include <cstdint>
#include <cstring>
#include <fstream>
#include <exception>
#include <string>
#include <thread>
#include <vector>

namespace {
thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}
} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// geometry.hpp:26-39
int ref_radial_const_from_avg_degree(double d_bar, double alpha, double* C) {
    return guarded([&] { *C = rhg::radial_const_from_avg_degree(d_bar, alpha); });
}
int ref_alpha_from_gamma(double gamma, double* alpha) {
    return guarded([&] { *alpha = rhg::alpha_from_gamma(gamma); });
}

// out[0..]: edges, fingerprint, comps, global_vertices, streaming_vertices,
// annuli, first_streaming ; outd[0..]: R, r_G, seconds, cosh_R
int ref_generate_stats(std::uint64_t n, double alpha, double C, std::uint64_t seed, std::uint32_t chunks,
                       std::uint32_t workers, std::uint64_t* out, double* outd, std::uint32_t* degrees) {
    return guarded([&] {
        const rhg::ModelParams params(n, alpha, C, seed, chunks);
        rhg::GenOptions        opts;
        opts.workers = workers;
        std::vector<std::uint32_t> deg;
        const auto st = rhg::generate_stats(params, opts, degrees ? &deg : nullptr);
        const auto layout = rhg::make_layout(params);
        out[0] = st.total.edges;
        out[1] = st.total.fingerprint;
        out[2] = st.total.comps;
        out[3] = st.global_vertices;
        out[4] = st.total.streaming_vertices;
        out[5] = layout.count;
        out[6] = layout.first_streaming;
        outd[0] = params.R;
        outd[1] = st.r_G;
        outd[2] = st.seconds;
        outd[3] = layout.cosh_R;
        if (degrees)
            std::memcpy(degrees, deg.data(), deg.size() * sizeof(std::uint32_t));
    });
}

// ChunkStats::*_by_annulus of generate_stats (arrays sized layout.count).
int ref_generate_annuli(std::uint64_t n, double alpha, double C, std::uint64_t seed, std::uint32_t chunks,
                        std::uint32_t workers, std::uint64_t* edges, std::uint64_t* comps, std::uint64_t* vertices) {
    return guarded([&] {
        const rhg::ModelParams params(n, alpha, C, seed, chunks);
        rhg::GenOptions        opts;
        opts.workers  = workers;
        const auto st = rhg::generate_stats(params, opts);
        for (std::size_t i = 0; i < st.total.edges_by_annulus.size(); ++i) {
            edges[i]    = st.total.edges_by_annulus[i];
            comps[i]    = st.total.comps_by_annulus[i];
            vertices[i] = st.total.vertices_by_annulus[i];
        }
    });
}

// stats.hpp:58-75 powerlaw_mle (std::invalid_argument -> error code).
int ref_powerlaw_mle(const std::uint32_t* degrees, std::uint64_t n, std::uint32_t d_min, double* gamma) {
    return guarded([&] { *gamma = rhg::powerlaw_mle(std::vector<std::uint32_t>(degrees, degrees + n), d_min); });
}

// Per-unit counters of generate_stats (unit 0 = global unit).  edges/comps
// arrays sized chunks+1.
int ref_generate_units(std::uint64_t n, double alpha, double C, std::uint64_t seed, std::uint32_t chunks,
                       std::uint32_t workers, std::uint64_t* unit_edges, std::uint64_t* unit_comps) {
    return guarded([&] {
        const rhg::ModelParams params(n, alpha, C, seed, chunks);
        rhg::GenOptions        opts;
        opts.workers  = workers;
        const auto st = rhg::generate_stats(params, opts);
        for (std::size_t u = 0; u < st.unit_edges.size(); ++u) {
            unit_edges[u] = st.unit_edges[u];
            unit_comps[u] = st.unit_comps[u];
        }
    });
}

// Layout query.  Pass null buffers to learn `count` first (annulus count
// written to *count).  Buffers: dbl[count*8] = lower, upper, probs, cosh_alpha_lower, cosh_alpha_upper,
// coth_lower, coshR_inv_sinh_lower, cell_width (each `count` long, in that
// order); u64 counts[count], chunk_counts[count*chunks], id_base[count*chunks],
// cells[count]; u8 classes[count]; scal[0..3] = R, cosh_R, r_G, first_streaming
int ref_layout(std::uint64_t n, double alpha, double C, std::uint64_t seed, std::uint32_t chunks,
               std::uint32_t* count, double* dbl, std::uint64_t* counts, std::uint64_t* chunk_counts,
               std::uint64_t* id_base, std::uint64_t* cells, std::uint8_t* classes, double* scal) {
    return guarded([&] {
        const rhg::ModelParams params(n, alpha, C, seed, chunks);
        const auto             L = rhg::make_layout(params);
        *count                   = L.count;
        if (!dbl)
            return;
        const std::vector<double>* cols[8] = {&L.lower,      &L.upper,      &L.probs,
                                               &L.cosh_alpha_lower, &L.cosh_alpha_upper, &L.coth_lower,
                                               &L.coshR_inv_sinh_lower, &L.cell_width};
        for (int k = 0; k < 8; ++k)
            for (std::uint32_t i = 0; i < L.count; ++i)
                dbl[k * L.count + i] = (*cols[k])[i];
        for (std::uint32_t i = 0; i < L.count; ++i) {
            counts[i]  = L.counts[i];
            cells[i]   = L.cells[i];
            classes[i] = static_cast<std::uint8_t>(L.classes[i]);
            for (std::uint32_t c = 0; c < chunks; ++c) {
                chunk_counts[i * chunks + c] = L.chunk_counts[i][c];
                id_base[i * chunks + c]      = L.id_base[i][c];
            }
        }
        scal[0] = params.R;
        scal[1] = L.cosh_R;
        scal[2] = L.r_G;
        scal[3] = L.first_streaming;
    });
}

// Full point dump in id order via the reference's own ChunkPointSource
// (sweep.hpp:102-151), one thread per stream group.  Each output array has n
// entries; annulus[] is the generating annulus.
int ref_points(std::uint64_t n, double alpha, double C, std::uint64_t seed, std::uint32_t chunks,
               std::uint32_t threads, double* beta, double* r, double* theta, double* half_width, double* coth_r,
               double* inv_sinh_r, double* cos_theta, double* sin_theta, std::uint32_t* annulus) {
    return guarded([&] {
        const rhg::ModelParams params(n, alpha, C, seed, chunks);
        const auto             L       = rhg::make_layout(params);
        const std::uint64_t    streams = static_cast<std::uint64_t>(L.count) * chunks;
        if (threads == 0)
            threads = std::max(1u, std::thread::hardware_concurrency());
        auto work = [&](std::uint32_t w) {
            for (std::uint64_t s = w; s < streams; s += threads) {
                const std::uint32_t i = static_cast<std::uint32_t>(s / chunks);
                const std::uint32_t c = static_cast<std::uint32_t>(s % chunks);
                rhg::ChunkPointSource src(L, i, c, params.seed);
                while (!src.exhausted()) {
                    const rhg::PointDraw p = src.next();
                    beta[p.id]             = p.beta;
                    r[p.id]                = p.r;
                    theta[p.id]            = p.theta;
                    half_width[p.id]       = p.half_width;
                    coth_r[p.id]           = p.coth_r;
                    inv_sinh_r[p.id]       = p.inv_sinh_r;
                    cos_theta[p.id]        = p.cos_theta;
                    sin_theta[p.id]        = p.sin_theta;
                    annulus[p.id]          = p.annulus;
                }
            }
        };
        std::vector<std::thread> pool;
        for (std::uint32_t w = 0; w < threads; ++w)
            pool.emplace_back(work, w);
        for (auto& t: pool)
            t.join();
    });
}

// Edge list of generate() (unit order, canonical u < v).  Call with
// edges == null to get the count in *m; then again with a buffer of 2*m.
int ref_generate_edges(std::uint64_t n, double alpha, double C, std::uint64_t seed, std::uint32_t chunks,
                       std::uint32_t workers, std::uint64_t* m, std::uint64_t* edges) {
    return guarded([&] {
        const rhg::ModelParams params(n, alpha, C, seed, chunks);
        rhg::GenOptions        opts;
        opts.workers = workers;
        std::vector<std::uint64_t> buf;
        rhg::generate(params, opts, [&](std::uint64_t u, std::uint64_t v) {
            buf.push_back(u);
            buf.push_back(v);
        });
        *m = buf.size() / 2;
        if (edges)
            std::memcpy(edges, buf.data(), buf.size() * sizeof(std::uint64_t));
    });
}

// oracle.hpp:44-54 — brute-force edges by the direct acosh distance.
int ref_naive_edges(std::uint64_t n, double alpha, double C, std::uint64_t seed, std::uint32_t chunks,
                    std::uint64_t* m, std::uint64_t* edges) {
    return guarded([&] {
        const rhg::ModelParams params(n, alpha, C, seed, chunks);
        const auto             trace = rhg::materialize_points(params);
        const auto             e     = rhg::naive_edges(trace, params.R);
        *m                           = e.size();
        if (edges)
            for (std::size_t k = 0; k < e.size(); ++k) {
                edges[2 * k]     = e[k].first;
                edges[2 * k + 1] = e[k].second;
            }
    });
}

// io.hpp:20-68 TextEdgeWriter / BinaryEdgeWriter over an edge list (byte-level
// parity of the B200 library's writers) and io.hpp:70-96 read_binary_edges.
int ref_write_edges(const char* path, const std::uint64_t* edges, std::uint64_t m, int binary) {
    return guarded([&] {
        std::ofstream os(path, std::ios::binary);
        if (binary) {
            rhg::BinaryEdgeWriter w(os);
            for (std::uint64_t k = 0; k < m; ++k) w.edge(edges[2 * k], edges[2 * k + 1]);
        } else {
            rhg::TextEdgeWriter w(os);
            for (std::uint64_t k = 0; k < m; ++k) w.edge(edges[2 * k], edges[2 * k + 1]);
        }
    });
}
int ref_read_edges_binary(const char* path, std::uint64_t* m, std::uint64_t* edges) {
    return guarded([&] {
        std::ifstream is(path, std::ios::binary);
        const auto    e = rhg::read_binary_edges(is);
        *m              = e.size();
        if (edges)
            for (std::size_t k = 0; k < e.size(); ++k) edges[2 * k] = e[k].first, edges[2 * k + 1] = e[k].second;
    });
}

// rng.hpp:41-69 known-answer helpers
std::uint64_t ref_derive_seed(std::uint64_t root, const std::uint64_t* comps, std::uint32_t k) {
    return rhg::derive_seed(root, std::span<const std::uint64_t>(comps, k));
}
void ref_mt_outputs(std::uint64_t seed, std::uint64_t count, std::uint64_t* out) {
    std::mt19937_64 g(seed);
    for (std::uint64_t i = 0; i < count; ++i)
        out[i] = g();
}
void ref_sorted_uniforms(std::uint64_t count, double a, double b, std::uint64_t root, const std::uint64_t* comps,
                         std::uint32_t k, double* out) {
    rhg::SeedPath path(root);
    path.components.assign(comps, comps + k);
    rhg::SortedUniformStream s(count, a, b, path);
    for (std::uint64_t i = 0; i < count; ++i)
        out[i] = s.next();
}
std::uint64_t ref_binomial(std::uint64_t trials, double p, std::uint64_t seed) {
    rhg::UniformStream s(seed);
    return rhg::binomial(trials, p, s);
}

} // extern "C"
