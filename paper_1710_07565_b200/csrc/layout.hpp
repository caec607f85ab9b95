// Host-side model parameters and annulus layout (the O(annuli * P) metadata).
//
// Restates /root/reference/proj/include/rhg/geometry.hpp:14-73 and
// partition.hpp:88-240 (with the binomial / multinomial samplers of
// rng.hpp:75-204 they need).  These draws are a few thousand scalar calls per
// run, so — as in the reference — they run on the host with the system libm;
// this translation unit is compiled with -ffp-contract=off so every value is
// bit-identical to the reference's tables.  Everything per-point runs on the
// device (sampler.cu, edges.cu).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace rhgb {

inline constexpr double kTwoPi = 6.283185307179586476925286766559; // geometry.hpp:11
inline constexpr double kPi    = 3.14159265358979323846;

struct InvalidArgument : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct Invariant : std::logic_error {
    using std::logic_error::logic_error;
};

double alpha_from_gamma(double gamma);                        // geometry.hpp:35-39
double radial_const_from_avg_degree(double d_bar, double a);  // geometry.hpp:26-33

struct Params { // geometry.hpp:49-67
    std::uint64_t n      = 0;
    double        alpha  = 0;
    double        C      = 0;
    double        R      = 0;
    std::uint64_t seed   = 0;
    std::uint32_t chunks = 1;
    Params() = default;
    Params(std::uint64_t n_, double alpha_, double C_, std::uint64_t seed_, std::uint32_t chunks_);
};

// SplitMix seed path (rng.hpp:15-54) and the MT19937-64 seeding constants the
// device sampler uses.
std::uint64_t derive_seed(std::uint64_t root, const std::uint64_t* comps, std::uint32_t k);
inline std::uint64_t derive_seed3(std::uint64_t root, std::uint64_t a, std::uint64_t b, std::uint64_t c) {
    const std::uint64_t p[3] = {a, b, c};
    return derive_seed(root, p, 3);
}
inline constexpr std::uint64_t kPhaseAnnuli = 1, kPhaseChunks = 2, kPhaseAngles = 3, kPhaseRadii = 4;

struct Layout { // partition.hpp:22-82
    std::uint64_t n = 0, seed = 0;
    std::uint32_t chunks = 1, count = 0, first_streaming = 0;
    double        alpha = 1, R = 0, cosh_R = 1, r_G = 0;
    bool          has_clique = false;
    std::vector<double> lower, upper, probs, cosh_alpha_lower, cosh_alpha_upper, coth_lower, coshR_inv_sinh_lower;
    std::vector<std::uint64_t> counts;       // n_i
    std::vector<std::uint64_t> chunk_counts; // [i * chunks + c]
    std::vector<std::uint64_t> id_base;      // [i * chunks + c]
    std::vector<std::uint8_t>  classes;      // 0 clique, 1 global, 2 streaming

    std::uint64_t chunk_count(std::uint32_t i, std::uint32_t c) const { return chunk_counts[std::size_t(i) * chunks + c]; }
    std::uint64_t chunk_id_base(std::uint32_t i, std::uint32_t c) const { return id_base[std::size_t(i) * chunks + c]; }
    std::uint64_t global_vertices() const {
        return first_streaming < count ? chunk_id_base(first_streaming, 0) : n;
    }
};

// Streaming-annulus chunks a shard needs (its owned chunks and the halo chunk): at most two
// ranges [lo, hi).  Counts and id bases of the other streaming chunks are left 0 (the
// reference computes every count with independent per-node seeds, so the needed ones are
// the same either way); global annuli always get every chunk.
struct ChunkNeed {
    std::uint32_t lo[2] = {0, 0}, hi[2] = {0, 0};
    int           n = 0;
    bool          has(std::uint32_t c) const {
        for (int k = 0; k < n; ++k)
            if (c >= lo[k] && c < hi[k]) return true;
        return false;
    }
    bool meets(std::uint32_t a, std::uint32_t b) const { // [a, b) intersects a needed range
        for (int k = 0; k < n; ++k)
            if (a < hi[k] && lo[k] < b) return true;
        return false;
    }
};

// partition.hpp:233-240 make_layout (cell grids are graph-neutral and the
// device builds its own candidate index, so they are not reproduced).  With `need`, only
// those streaming chunks are split (O(owned chunks + log P) binomial draws per annulus).
Layout make_layout(const Params& p, const ChunkNeed* need = nullptr);

// sweep.hpp:80-85
inline double chunk_lower_bound(std::uint32_t c, std::uint32_t P) { return double(c) * (kTwoPi / double(P)); }
inline double chunk_upper_bound(std::uint32_t c, std::uint32_t P) {
    return c + 1 == P ? kTwoPi : double(c + 1) * (kTwoPi / double(P));
}

} // namespace rhgb
