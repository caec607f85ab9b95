// Host layout restatement — see layout.hpp.  Compiled with -ffp-contract=off.
#include "layout.hpp"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <exception>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>

#include <unistd.h>

namespace rhgb {

namespace {

std::uint64_t splitmix_mix(std::uint64_t z) { // rng.hpp:15-19
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
constexpr std::uint64_t kGolden = 0x9E3779B97F4A7C15ull;

// std::mt19937_64 state machine ([rand.predef]); host copy used by the
// binomial draws only.  Most split draws consume a handful of outputs, so the
// seeding recurrence and the first twist run lazily: output k of the first
// block needs seed words up to k + 156 (k < 156: new[k] = f(old[k], old[k+1],
// old[k+156]); k >= 156: f(old[k], old[k+1], new[k-156]); k = 311: f(old[311],
// new[0], new[155])), later blocks twist in place as usual — the same stream.
class Mt64 {
public:
    explicit Mt64(std::uint64_t s) { old_[0] = s; }
    std::uint64_t bits() {
        std::uint64_t y;
        if (first_) {
            const int k = idx_++;
            if (k < 156) {
                seed_to(k + 156);
                y = mix(old_[k], old_[k + 1], old_[k + 156]);
            } else if (k < 311) {
                seed_to(k + 1);
                y = mix(old_[k], old_[k + 1], mt_[k - 156]);
            } else {
                y = mix(old_[311], mt_[0], mt_[155]);
            }
            mt_[k] = y;
            if (idx_ == 312) first_ = false;
        } else {
            if (idx_ >= 312) twist();
            y = mt_[idx_++];
        }
        y ^= (y >> 29) & 0x5555555555555555ull;
        y ^= (y << 17) & 0x71D67FFFEDA60000ull;
        y ^= (y << 37) & 0xFFF7EEE000000000ull;
        return y ^ (y >> 43);
    }
    double uniform() { return double(bits() >> 11) * 0x1.0p-53; } // rng.hpp:63

private:
    static std::uint64_t mix(std::uint64_t cur, std::uint64_t nxt, std::uint64_t far) {
        const std::uint64_t x = (cur & 0xFFFFFFFF80000000ull) | (nxt & 0x7FFFFFFFull);
        return far ^ (x >> 1) ^ ((x & 1) ? 0xB5026F5AA96619E9ull : 0ull);
    }
    void seed_to(int k) { // old_[0..k] hold the seeding recurrence
        for (; seeded_ < k; ++seeded_)
            old_[seeded_ + 1] = 6364136223846793005ull * (old_[seeded_] ^ (old_[seeded_] >> 62)) + std::uint64_t(seeded_ + 1);
    }
    void twist() {
        for (int i = 0; i < 312; ++i) mt_[i] = mix(mt_[i], mt_[(i + 1) % 312], mt_[(i + 156) % 312]);
        idx_ = 0;
    }
    std::uint64_t old_[312];
    std::uint64_t mt_[312];
    int           seeded_ = 0; // old_[0..seeded_] are valid
    int           idx_    = 0;
    bool          first_  = true;
};

// A persistent host worker pool for the layout's independent binomial trees
// (spawning threads per call would cost more than the work at P ~ 64).
class Pool {
public:
    // One pool per process: a forked child (whose copy of the parent's pool has no threads)
    // starts its own.  Pools are never destroyed — their workers block until process exit.
    static Pool& get() {
        static std::mutex m;
        static Pool*      p     = nullptr;
        static pid_t      owner = 0;
        std::lock_guard<std::mutex> g(m);
        if (!p || owner != getpid()) p = new Pool(), owner = getpid();
        return *p;
    }
    unsigned size() const { return unsigned(workers_.size()) + 1; }
    // body(k) for k < n on the pool and the calling thread; rethrows the first exception.
    template <class F>
    void run(std::uint32_t n, F&& body) {
        std::lock_guard<std::mutex> serial(call_mu_); // one parallel region at a time
        std::atomic<std::uint32_t>  next{0};
        std::exception_ptr          err;
        std::atomic<bool>           failed{false};
        std::function<void()>       work = [&] {
            try {
                for (std::uint32_t k = next++; k < n && !failed; k = next++) body(k);
            } catch (...) {
                if (!failed.exchange(true)) err = std::current_exception();
            }
        };
        {
            std::lock_guard<std::mutex> g(mu_);
            job_ = &work, pending_ = unsigned(workers_.size()), ++gen_;
        }
        cv_.notify_all();
        work();
        spin([&] { return pending_.load(std::memory_order_acquire) == 0; });
        std::unique_lock<std::mutex> g(mu_);
        done_.wait(g, [&] { return pending_.load() == 0; });
        job_ = nullptr;
        if (err) std::rethrow_exception(err);
    }

private:
    Pool() {
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        for (unsigned t = 1; t < std::min(hw, 16u); ++t) workers_.emplace_back([this] { loop(); });
    }
    // Busy-wait up to ~50 us before blocking: the layout runs two parallel regions back to
    // back, and a futex wake-up per worker and region costs more than the regions' work.
    template <class P>
    static void spin(P&& ready) {
        const auto t0 = std::chrono::steady_clock::now();
        for (unsigned k = 1; !ready(); ++k)
            if ((k & 255) == 0 && std::chrono::steady_clock::now() - t0 > std::chrono::microseconds(50)) return;
    }
    void loop() {
        std::uint64_t seen = 0;
        for (;;) {
            spin([&] { return gen_.load(std::memory_order_acquire) != seen; });
            std::function<void()>* job;
            {
                std::unique_lock<std::mutex> g(mu_);
                cv_.wait(g, [&] { return gen_.load() != seen; });
                seen = gen_.load(), job = job_;
            }
            (*job)();
            if (pending_.fetch_sub(1, std::memory_order_acq_rel) == 1) {
                std::lock_guard<std::mutex> g(mu_);
                done_.notify_one();
            }
        }
    }
    std::vector<std::thread>  workers_;
    std::mutex                mu_, call_mu_;
    std::condition_variable   cv_, done_;
    std::function<void()>*    job_     = nullptr;
    std::atomic<unsigned>      pending_{0};
    std::atomic<std::uint64_t> gen_{0};
};

double normal(Mt64& s) { // rng.hpp:75-79
    const double u1 = 1.0 - s.uniform();
    const double u2 = s.uniform();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(kTwoPi * u2);
}
double gamma_variate(double a, Mt64& s) { // rng.hpp:82-96, Marsaglia-Tsang
    const double d = a - 1.0 / 3.0;
    const double c = 1.0 / std::sqrt(9.0 * d);
    for (;;) {
        const double x = normal(s);
        const double t = 1.0 + c * x;
        if (t <= 0.0) continue;
        const double v = t * t * t;
        const double u = 1.0 - s.uniform();
        if (std::log(u) < 0.5 * x * x + d - d * v + d * std::log(v)) return d * v;
    }
}
double beta_variate(double a, double b, Mt64& s) { // rng.hpp:98-103
    const double x = gamma_variate(a, s);
    const double y = gamma_variate(b, s);
    const double t = x + y;
    return t > 0.0 ? x / t : 0.5;
}
std::uint64_t binomial_inversion(std::uint64_t n, double p, Mt64& s) { // rng.hpp:107-126
    const double  u     = s.uniform();
    const double  ratio = p / (1.0 - p);
    double        lpmf  = double(n) * std::log1p(-p);
    std::uint64_t k     = 0;
    while (lpmf <= -700.0 && k < n) {
        lpmf += std::log(double(n - k) / double(k + 1) * ratio);
        ++k;
    }
    double pmf = std::exp(lpmf), cum = 0.0;
    for (;; ++k) {
        cum += pmf;
        if (u < cum || k >= n) return k;
        pmf *= double(n - k) / double(k + 1) * ratio;
    }
}
std::uint64_t binomial(std::uint64_t trials, double p, Mt64& s) { // rng.hpp:133-164
    if (!(p >= 0.0 && p <= 1.0)) throw InvalidArgument("binomial: p must lie in [0, 1]");
    std::int64_t base = 0, sign = 1;
    for (;;) {
        if (trials == 0 || p <= 0.0) return std::uint64_t(base);
        if (p >= 1.0) return std::uint64_t(base + sign * std::int64_t(trials));
        if (p > 0.5) {
            base += sign * std::int64_t(trials);
            sign = -sign;
            p    = 1.0 - p;
            continue;
        }
        if (double(trials) * p <= 1000.0)
            return std::uint64_t(base + sign * std::int64_t(binomial_inversion(trials, p, s)));
        const std::uint64_t m = (trials + 1) / 2;
        const double        v = beta_variate(double(m), double(trials + 1 - m), s);
        if (v <= p) {
            base += sign * std::int64_t(m);
            trials -= m;
            p = (p - v) / (1.0 - v);
        } else {
            trials = m - 1;
            p      = p / v;
        }
    }
}

double angular_deviation(double r, double b, double R) { // geometry.hpp:128-134
    if (r + b <= R) return kPi;
    const double arg = (std::cosh(r) * std::cosh(b) - std::cosh(R)) / (std::sinh(r) * std::sinh(b));
    if (arg >= 1.0) return 0.0;
    if (arg <= -1.0) return kPi;
    return std::acos(arg);
}

// partition.hpp:142-156: divide-and-conquer binomial split keyed on the
// recursion node, so every caller recomputes identical per-chunk counts.
void split_chunk_range(std::uint64_t seed, std::uint32_t annulus, std::uint64_t total, std::uint32_t lo,
                       std::uint32_t hi, std::uint64_t node, std::uint64_t* out) {
    if (hi - lo == 1) {
        out[lo] = total;
        return;
    }
    if (total == 0) { // binomial(0, p) = 0 for every node below: nothing to draw
        for (std::uint32_t c = lo; c < hi; ++c) out[c] = 0;
        return;
    }
    const std::uint32_t mid = lo + (hi - lo + 1) / 2;
    const double        ml = double(mid - lo), mr = double(hi - mid);
    Mt64                s(derive_seed3(seed, kPhaseChunks, annulus, node));
    const std::uint64_t left = binomial(total, ml / (ml + mr), s); // rng.hpp:197-204
    split_chunk_range(seed, annulus, left, lo, mid, 2 * node, out);
    split_chunk_range(seed, annulus, total - left, mid, hi, 2 * node + 1, out);
}

// The same tree, descending only into subtrees that hold needed chunks; `before` is the number
// of the annulus's points in chunks below lo, so base[c] is chunk c's offset in the annulus.
void split_chunk_partial(std::uint64_t seed, std::uint32_t annulus, std::uint64_t total, std::uint32_t lo,
                         std::uint32_t hi, std::uint64_t node, const ChunkNeed& need, std::uint64_t before,
                         std::uint64_t* out, std::uint64_t* base) {
    if (!need.meets(lo, hi)) return;
    if (hi - lo == 1 || total == 0) {
        for (std::uint32_t c = lo; c < hi; ++c)
            if (need.has(c)) out[c] = c == lo ? total : 0, base[c] = before + (c == lo ? 0 : total);
        return;
    }
    const std::uint32_t mid = lo + (hi - lo + 1) / 2;
    const double        ml = double(mid - lo), mr = double(hi - mid);
    Mt64                s(derive_seed3(seed, kPhaseChunks, annulus, node));
    const std::uint64_t left = binomial(total, ml / (ml + mr), s); // rng.hpp:197-204
    split_chunk_partial(seed, annulus, left, lo, mid, 2 * node, need, before, out, base);
    split_chunk_partial(seed, annulus, total - left, mid, hi, 2 * node + 1, need, before + left, out, base);
}

} // namespace

std::uint64_t derive_seed(std::uint64_t root, const std::uint64_t* comps, std::uint32_t k) { // rng.hpp:41-46
    std::uint64_t h = splitmix_mix(root + kGolden);
    for (std::uint32_t i = 0; i < k; ++i) h = splitmix_mix((h + kGolden) ^ comps[i]);
    return h;
}

double alpha_from_gamma(double gamma) {
    if (!(gamma > 2.0)) throw InvalidArgument("alpha_from_gamma: gamma must be > 2");
    return (gamma - 1.0) / 2.0;
}

double radial_const_from_avg_degree(double d_bar, double alpha) {
    if (!(alpha > 0.5)) throw InvalidArgument("radial_const_from_avg_degree: alpha must be > 1/2");
    if (!(d_bar > 0.0)) throw InvalidArgument("radial_const_from_avg_degree: average degree must be positive");
    const double q = (alpha - 0.5) / alpha;
    return -2.0 * std::log(d_bar * kPi / 2.0 * q * q);
}

Params::Params(std::uint64_t n_, double alpha_, double C_, std::uint64_t seed_, std::uint32_t chunks_)
    : n(n_), alpha(alpha_), C(C_), R(2.0 * std::log(double(n_)) + C_), seed(seed_), chunks(chunks_) {
    if (n < 1) throw InvalidArgument("ModelParams: n must be >= 1");
    if (!(alpha > 0.5)) throw InvalidArgument("ModelParams: alpha must be > 1/2");
    if (!(R > 0.0)) throw InvalidArgument("ModelParams: R = 2 ln n + C must be positive");
    if (chunks < 1) throw InvalidArgument("ModelParams: chunk count must be >= 1");
}

Layout make_layout(const Params& p, const ChunkNeed* need) {
    Layout L;
    L.n = p.n, L.seed = p.seed, L.chunks = p.chunks, L.alpha = p.alpha, L.R = p.R;
    L.cosh_R = std::cosh(p.R);

    // build_annuli, partition.hpp:97-138
    const std::uint64_t k_equal =
        std::max<std::uint64_t>(1, std::uint64_t(std::ceil(p.alpha * p.R / std::log(2.0))));
    const double        height = p.R / double(k_equal);
    std::vector<double> bounds(k_equal + 1);
    for (std::uint64_t j = 0; j <= k_equal; ++j) bounds[j] = double(j) * height;
    bounds[k_equal] = p.R;
    std::uint64_t merged = 0;
    while (merged + 1 < k_equal && bounds[merged + 1] <= p.R / 2.0) ++merged;
    L.has_clique = merged >= 1;
    L.lower.push_back(0.0);
    for (std::uint64_t j = std::max<std::uint64_t>(merged, 1); j <= k_equal; ++j) {
        L.upper.push_back(bounds[j]);
        if (j < k_equal) L.lower.push_back(bounds[j]);
    }
    L.count = std::uint32_t(L.upper.size());
    const double denom = std::cosh(p.alpha * p.R) - 1.0;
    for (std::uint32_t i = 0; i < L.count; ++i) {
        const double cl = std::cosh(p.alpha * L.lower[i]);
        const double cu = std::cosh(p.alpha * L.upper[i]);
        L.cosh_alpha_lower.push_back(cl);
        L.cosh_alpha_upper.push_back(cu);
        L.probs.push_back((cu - cl) / denom);
        if (L.lower[i] > 0.0) {
            const double ex = std::exp(L.lower[i]);
            const double sh = 0.5 * (ex - 1.0 / ex);
            L.coth_lower.push_back(0.5 * (ex + 1.0 / ex) / sh);
            L.coshR_inv_sinh_lower.push_back(L.cosh_R / sh);
        } else {
            L.coth_lower.push_back(HUGE_VAL);
            L.coshR_inv_sinh_lower.push_back(HUGE_VAL);
        }
    }

    // assign_counts, partition.hpp:161-169 (multinomial chain rng.hpp:168-192)
    double sum = 0.0;
    for (double q: L.probs) {
        if (q < 0.0) throw InvalidArgument("multinomial_counts: negative probability");
        sum += q;
    }
    if (std::abs(sum - 1.0) > 1e-9) throw InvalidArgument("multinomial_counts: probabilities must sum to 1");
    {
        const std::uint64_t one = kPhaseAnnuli;
        Mt64                s(derive_seed(p.seed, &one, 1));
        L.counts.assign(L.count, 0);
        std::uint64_t remaining = p.n;
        double        mass      = 1.0;
        for (std::uint32_t i = 0; i + 1 < L.count; ++i) {
            const double q = mass > 0.0 ? std::min(1.0, std::max(0.0, L.probs[i] / mass)) : 1.0;
            L.counts[i]    = binomial(remaining, q, s);
            remaining -= L.counts[i];
            mass -= L.probs[i];
        }
        L.counts[L.count - 1] = remaining;
    }
    // classify, partition.hpp:195-217
    L.classes.assign(L.count, 1);
    L.first_streaming       = L.count;
    const double chunk_width = kTwoPi / double(p.chunks);
    for (std::uint32_t i = 0; i < L.count; ++i) {
        if (i == 0 && L.has_clique) {
            L.classes[i] = 0;
            continue;
        }
        const double l     = L.lower[i];
        const double width = l > 0.0 ? 2.0 * angular_deviation(l, l, p.R) : kTwoPi;
        if (width <= chunk_width) {
            L.classes[i] = 2;
            if (L.first_streaming == L.count) L.first_streaming = i;
        }
    }
    for (std::uint32_t i = L.first_streaming; i < L.count; ++i)
        if (L.classes[i] != 2) throw Invariant("classify: streaming annuli are not contiguous");
    L.r_G = L.first_streaming < L.count ? L.lower[L.first_streaming] : p.R;

    L.chunk_counts.assign(std::size_t(L.count) * p.chunks, 0);
    // The per-annulus binomial trees are independent (every split node has its own seed path),
    // and so are the subtrees below any node: the first levels are split here, and the
    // subtrees run on host threads (the splits dominate the host time: ~1 us per MT seeding
    // plus up to ~1000 inversion steps each).
    {
        struct Task {
            std::uint32_t annulus, lo, hi;
            std::uint64_t total, node;
        };
        const unsigned threads = p.chunks >= 16 ? Pool::get().size() : 1;
        auto run = [&](std::uint32_t ntasks, auto&& body) { // body(k) for k < ntasks
            if (threads <= 1 || ntasks <= 1) {
                for (std::uint32_t k = 0; k < ntasks; ++k) body(k);
            } else {
                Pool::get().run(ntasks, body);
            }
        };
        // phase 1, one task per annulus: the top levels of its tree (up to 8 subtrees)
        const int         levels = threads > 1 ? 3 : 0;
        std::vector<Task> per(std::size_t(L.count) << levels);
        std::vector<int>  nper(L.count, 0);
        // with `need`, streaming annuli take the partial traversal below instead
        const std::uint32_t nfull = need ? L.first_streaming : L.count;
        run(nfull, [&](std::uint32_t i) {
            std::vector<Task> cur{{i, 0, p.chunks, L.counts[i], 1}};
            for (int level = 0; level < levels; ++level) {
                std::vector<Task> next;
                for (const Task& t: cur) {
                    if (t.hi - t.lo < 4) {
                        next.push_back(t);
                        continue;
                    }
                    const std::uint32_t mid = t.lo + (t.hi - t.lo + 1) / 2;
                    const double        ml = double(mid - t.lo), mr = double(t.hi - mid);
                    Mt64                s(derive_seed3(p.seed, kPhaseChunks, t.annulus, t.node));
                    const std::uint64_t left = binomial(t.total, ml / (ml + mr), s); // rng.hpp:197-204
                    next.push_back({t.annulus, t.lo, mid, left, 2 * t.node});
                    next.push_back({t.annulus, mid, t.hi, t.total - left, 2 * t.node + 1});
                }
                cur.swap(next);
            }
            for (std::size_t k = 0; k < cur.size(); ++k) per[(std::size_t(i) << levels) + k] = cur[k];
            nper[i] = int(cur.size());
        });
        std::vector<Task> tasks;
        for (std::uint32_t i = 0; i < nfull; ++i)
            for (int k = 0; k < nper[i]; ++k) tasks.push_back(per[(std::size_t(i) << levels) + k]);
        std::sort(tasks.begin(), tasks.end(), [](const Task& x, const Task& y) { return x.total > y.total; });
        // phase 2: the subtrees
        run(std::uint32_t(tasks.size()), [&](std::uint32_t k) {
            const Task& t = tasks[k];
            split_chunk_range(p.seed, t.annulus, t.total, t.lo, t.hi, t.node,
                              L.chunk_counts.data() + std::size_t(t.annulus) * p.chunks);
        });
        if (need) { // streaming annuli: only the shard's chunks (relative id bases into id_base)
            L.id_base.assign(std::size_t(L.count) * p.chunks, 0);
            run(L.count - nfull, [&](std::uint32_t k) {
                const std::uint32_t i = nfull + k;
                split_chunk_partial(p.seed, i, L.counts[i], 0, p.chunks, 1, *need, 0,
                                    L.chunk_counts.data() + std::size_t(i) * p.chunks,
                                    L.id_base.data() + std::size_t(i) * p.chunks);
            });
        }
    }

    // assign_vertex_ids, partition.hpp:220-231 (annulus-major, chunk-minor)
    if (!need) L.id_base.assign(std::size_t(L.count) * p.chunks, 0);
    std::uint64_t next = 0;
    for (std::uint32_t i = 0; i < L.count; ++i) {
        if (need && i >= L.first_streaming) { // partial: bases relative to the annulus start
            for (std::uint32_t c = 0; c < p.chunks; ++c)
                if (need->has(c) || c == 0) L.id_base[std::size_t(i) * p.chunks + c] += next;
            next += L.counts[i];
            continue;
        }
        for (std::uint32_t c = 0; c < p.chunks; ++c) {
            L.id_base[std::size_t(i) * p.chunks + c] = next;
            next += L.chunk_counts[std::size_t(i) * p.chunks + c];
        }
    }
    if (next != p.n) throw Invariant("assign_vertex_ids: counts do not sum to n");
    return L;
}

} // namespace rhgb
