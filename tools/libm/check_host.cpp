// Host proof that csrc/glibc_libm.cuh (compiled for the CPU from the SAME source the
// device uses) returns glibc's results bit for bit.  TEST INFRASTRUCTURE ONLY.
//
//   g++ -O2 -mfma -ffp-contract=off -fno-builtin -std=c++17 -pthread \
//       tools/libm/check_host.cpp -o /tmp/check_host -lm
//   /tmp/check_host [samples_per_domain (default 1e7)] [threads]
//
// Each domain draws seeded inputs from the argument ranges the reference's sampler
// produces (sweep.hpp:117-141, partition.hpp:64-70, rng.hpp:221), plus wide random
// ranges, and counts bitwise mismatches against the libm the program links.
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "../../paper_1710_07565_b200/csrc/glibc_libm.cuh"

static uint64_t bits(double x) { uint64_t u; std::memcpy(&u, &x, 8); return u; }
static double frombits(uint64_t u) { double x; std::memcpy(&x, &u, 8); return x; }
static bool same(double a, double b) { return bits(a) == bits(b) || (std::isnan(a) && std::isnan(b)); }

// volatile function pointers: keep gcc from constant-folding or merging calls
static double (*volatile c_exp)(double) = exp;
static double (*volatile c_log)(double) = log;
static double (*volatile c_log1p)(double) = log1p;
static double (*volatile c_acosh)(double) = acosh;
static double (*volatile c_acos)(double) = acos;
static double (*volatile c_pow)(double, double) = pow;
static void (*volatile c_sincos)(double, double*, double*) = sincos;

struct Domain {
    std::string name;
    std::function<void(std::mt19937_64&, double&, double&)> gen;  // fills (x, y)
    int fn;  // 0 exp 1 log 2 log1p 3 acosh 4 acos 5 pow 6 sin(sincos) 7 cos(sincos)
};

static double u01(std::mt19937_64& g) { return (double)(g() >> 11) * 0x1p-53; }
static double logu(std::mt19937_64& g, double lo, double hi) {
    return std::exp2(std::log2(lo) + u01(g) * (std::log2(hi) - std::log2(lo)));
}

int main(int argc, char** argv) {
    const long long N = argc > 1 ? (long long)atof(argv[1]) : 10000000LL;
    const int T = argc > 2 ? atoi(argv[2]) : (int)std::thread::hardware_concurrency();
    const double PI2 = 6.283185307179586;
    std::vector<Domain> D = {
        {"exp r in [1e-12,45]", [](auto& g, double& x, double&) { x = 1e-12 + u01(g) * 45; }, 0},
        {"exp r log-uniform", [](auto& g, double& x, double&) { x = logu(g, 1e-13, 50); }, 0},
        {"exp wide", [](auto& g, double& x, double&) { x = (u01(g) - 0.5) * 1500; }, 0},
        {"exp random bits", [](auto& g, double& x, double&) { x = frombits(g()); }, 0},
        {"log wide", [](auto& g, double& x, double&) { x = logu(g, 1e-300, 1e300); }, 1},
        {"log near 1", [](auto& g, double& x, double&) { x = 0.9 + 0.2 * u01(g); }, 1},
        {"log random bits", [](auto& g, double& x, double&) { x = frombits(g()); }, 1},
        {"log1p (0,3]", [](auto& g, double& x, double&) { x = 3 * u01(g); }, 2},
        {"log1p log-uniform", [](auto& g, double& x, double&) { x = logu(g, 1e-20, 1e20); }, 2},
        {"log1p (-1,0)", [](auto& g, double& x, double&) { x = -u01(g); }, 2},
        {"log1p random bits", [](auto& g, double& x, double&) { x = frombits(g()); }, 2},
        {"acosh (1,2]", [](auto& g, double& x, double&) { x = 1 + u01(g); }, 3},
        {"acosh 1+tiny", [](auto& g, double& x, double&) { x = 1 + logu(g, 1e-16, 1); }, 3},
        {"acosh (2,1e19)", [](auto& g, double& x, double&) { x = logu(g, 2, 1e19); }, 3},
        {"acosh wide", [](auto& g, double& x, double&) { x = logu(g, 1, 1e300); }, 3},
        {"acos (-1,1)", [](auto& g, double& x, double&) { x = 2 * u01(g) - 1; }, 4},
        {"acos near +-1", [](auto& g, double& x, double&) {
             x = 1 - logu(g, 1e-17, 0.05); if (g() & 1) x = -x; }, 4},
        {"acos small", [](auto& g, double& x, double&) {
             x = logu(g, 1e-20, 0.2); if (g() & 1) x = -x; }, 4},
        {"acos random bits", [](auto& g, double& x, double&) { x = frombits(g()); }, 4},
        {"pow(U, 1/k)", [](auto& g, double& x, double& y) {
             x = u01(g); y = 1.0 / (double)(1 + (g() >> (g() % 64 | 33))); }, 5},
        {"pow(U, 1/k) small k", [](auto& g, double& x, double& y) {
             x = u01(g); y = 1.0 / (double)(1 + g() % 4096); }, 5},
        {"pow(U~1, 1/k)", [](auto& g, double& x, double& y) {
             x = 1 - logu(g, 0x1p-53, 1e-3); y = 1.0 / (double)(1 + (g() >> 34)); }, 5},
        {"pow wide", [](auto& g, double& x, double& y) {
             x = logu(g, 1e-300, 1e300); y = (u01(g) - 0.5) * 40; }, 5},
        {"pow random bits", [](auto& g, double& x, double& y) { x = frombits(g()); y = frombits(g()); }, 5},
        {"sin theta in [0,2pi)", [PI2](auto& g, double& x, double&) { x = u01(g) * PI2; }, 6},
        {"cos theta in [0,2pi)", [PI2](auto& g, double& x, double&) { x = u01(g) * PI2; }, 7},
        {"sin small", [](auto& g, double& x, double&) { x = logu(g, 1e-20, 1); if (g() & 1) x = -x; }, 6},
        {"cos small", [](auto& g, double& x, double&) { x = logu(g, 1e-20, 1); if (g() & 1) x = -x; }, 7},
        {"sin wide", [](auto& g, double& x, double&) { x = (u01(g) - 0.5) * 2e8; }, 6},
        {"cos wide", [](auto& g, double& x, double&) { x = (u01(g) - 0.5) * 2e8; }, 7},
    };
    int bad_domains = 0;
    {   // special values, every (x, y) pair for pow
        const double S[] = {0.0, -0.0, 1.0, -1.0, 2.0, 0.5, INFINITY, -INFINITY, NAN, 1e-320, -1e-320,
                            nextafter(1.0, 0), nextafter(1.0, 2), 0x1p-1022, 709.78, -745.1, 268435456.0,
                            268435458.0, 0.96875, -0.96875, 0.125, 0.855468, 2.426265, 1.05e8, -3.0, 3.0,
                            -0.5, 1e300, -1e300, 1e-300};
        const int ns = sizeof S / sizeof S[0];
        long long bad = 0;
        for (int i = 0; i < ns; ++i) {
            const double x = S[i];
            bad += !same(c_exp(x), gl::gl_exp(x)) + !same(c_log(x), gl::gl_log(x)) +
                   !same(c_log1p(x), gl::gl_log1p(x)) + !same(c_acosh(x), gl::gl_acosh(x)) +
                   !same(c_acos(x), gl::gl_acos(x));
            if (!(fabs(x) > 1.05e8)) {  // |x| >= 105414350 (__branred) is outside the path
                double s, c, s2, c2;
                c_sincos(x, &s, &c);
                gl::gl_sincos(x, &s2, &c2);
                bad += !same(s, s2) + !same(c, c2);
            }
            for (int j = 0; j < ns; ++j) bad += !same(c_pow(x, S[j]), gl::gl_pow(x, S[j]));
        }
        printf("%-24s %d values  mismatches %lld\n", "special values", ns, bad);
        if (bad) ++bad_domains;
    }
    for (size_t d = 0; d < D.size(); ++d) {
        std::atomic<long long> bad{0};
        std::mutex mu;
        std::vector<std::string> ex;
        std::vector<std::thread> th;
        for (int t = 0; t < T; ++t)
            th.emplace_back([&, t]() {
                std::mt19937_64 g(0x9e3779b97f4a7c15ull * (d + 1) + t);
                long long lb = 0;
                for (long long i = t; i < N; i += T) {
                    double x = 0, y = 0, want = 0, got = 0;
                    D[d].gen(g, x, y);
                    switch (D[d].fn) {
                    case 0: want = c_exp(x); got = gl::gl_exp(x); break;
                    case 1: want = c_log(x); got = gl::gl_log(x); break;
                    case 2: want = c_log1p(x); got = gl::gl_log1p(x); break;
                    case 3: want = c_acosh(x); got = gl::gl_acosh(x); break;
                    case 4: want = c_acos(x); got = gl::gl_acos(x); break;
                    case 5: want = c_pow(x, y); got = gl::gl_pow(x, y); break;
                    case 6: case 7: {
                        double s, c, s2, c2;
                        c_sincos(x, &s, &c);
                        gl::gl_sincos(x, &s2, &c2);
                        want = D[d].fn == 6 ? s : c; got = D[d].fn == 6 ? s2 : c2; break; }
                    }
                    if (!same(want, got)) {
                        ++lb;
                        std::lock_guard<std::mutex> l(mu);
                        if (ex.size() < 4) {
                            char buf[256];
                            snprintf(buf, sizeof buf, "    x=%a y=%a want=%a got=%a", x, y, want, got);
                            ex.push_back(buf);
                        }
                    }
                }
                bad += lb;
            });
        for (auto& t : th) t.join();
        printf("%-24s %lld samples  mismatches %lld\n", D[d].name.c_str(), N, bad.load());
        for (auto& s : ex) printf("%s\n", s.c_str());
        if (bad.load()) ++bad_domains;
        fflush(stdout);
    }
    printf(bad_domains ? "FAIL: %d domains mismatch\n" : "OK: all domains bit-exact\n", bad_domains);
    return bad_domains ? 1 : 0;
}
