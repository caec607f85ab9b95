// Host-side edge-stream files and degree analytics.
//   * edge stream files, byte-compatible with the reference's io.hpp:20-96:
//     text "u v\n" (decimal), binary magic "RHGE0001" + LE u64 pairs;
//   * the power-law exponent MLE of stats.hpp:58-75 (same summation order and
//     libm as the reference, so the estimate is bit-identical).
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/rhg_b200.h"

namespace {

thread_local std::string g_io_err;

struct File {
    std::FILE* f = nullptr;
    explicit File(const char* path, const char* mode) : f(path ? std::fopen(path, mode) : nullptr) {}
    ~File() {
        if (f) std::fclose(f);
    }
};

int fail(const std::string& msg) {
    g_io_err = msg;
    return RHG_INVALID_ARGUMENT;
}

char* put_dec(char* p, std::uint64_t x) { // io.hpp TextEdgeWriter::append
    char  tmp[20];
    char* t = tmp;
    do {
        *t++ = static_cast<char>('0' + x % 10);
        x /= 10;
    } while (x);
    while (t != tmp) *p++ = *--t;
    return p;
}

} // namespace

extern "C" {

const char* rhg_io_last_error(void) { return g_io_err.c_str(); }

int rhg_write_edges_text(const char* path, const std::uint64_t* edges, std::uint64_t m) {
    File out(path, "wb");
    if (!out.f) return fail(std::string("rhg_write_edges_text: cannot open ") + (path ? path : "(null)"));
    std::vector<char> buf(1 << 20);
    std::size_t       used = 0;
    for (std::uint64_t i = 0; i < m; ++i) {
        if (used + 44 > buf.size()) {
            if (std::fwrite(buf.data(), 1, used, out.f) != used) return fail("rhg_write_edges_text: write failed");
            used = 0;
        }
        char* p = buf.data() + used;
        p       = put_dec(p, edges[2 * i]);
        *p++    = ' ';
        p       = put_dec(p, edges[2 * i + 1]);
        *p++    = '\n';
        used    = std::size_t(p - buf.data());
    }
    if (used && std::fwrite(buf.data(), 1, used, out.f) != used) return fail("rhg_write_edges_text: write failed");
    return RHG_OK;
}

int rhg_write_edges_binary(const char* path, const std::uint64_t* edges, std::uint64_t m) {
    File out(path, "wb");
    if (!out.f) return fail(std::string("rhg_write_edges_binary: cannot open ") + (path ? path : "(null)"));
    static const char magic[8] = {'R', 'H', 'G', 'E', '0', '0', '0', '1'};
    if (std::fwrite(magic, 1, 8, out.f) != 8) return fail("rhg_write_edges_binary: write failed");
    std::vector<unsigned char> buf(1 << 20);
    std::size_t                used = 0;
    for (std::uint64_t i = 0; i < 2 * m; ++i) {
        if (used + 8 > buf.size()) {
            if (std::fwrite(buf.data(), 1, used, out.f) != used) return fail("rhg_write_edges_binary: write failed");
            used = 0;
        }
        const std::uint64_t x = edges[i];
        for (int b = 0; b < 8; ++b) buf[used++] = static_cast<unsigned char>((x >> (8 * b)) & 0xff);
    }
    if (used && std::fwrite(buf.data(), 1, used, out.f) != used) return fail("rhg_write_edges_binary: write failed");
    return RHG_OK;
}

int rhg_read_edges_binary(const char* path, std::uint64_t* edges, std::uint64_t cap, std::uint64_t* m) {
    if (!m) return fail("rhg_read_edges_binary: null argument");
    File in(path, "rb");
    if (!in.f) return fail(std::string("rhg_read_edges_binary: cannot open ") + (path ? path : "(null)"));
    char magic[8];
    if (std::fread(magic, 1, 8, in.f) != 8 || std::memcmp(magic, "RHGE0001", 8) != 0)
        return fail("read_binary_edges: bad magic");
    std::uint64_t      n = 0;
    unsigned char      rec[16];
    for (;;) {
        const std::size_t got = std::fread(rec, 1, 16, in.f);
        if (got == 0) break;
        if (got != 16) return fail("read_binary_edges: truncated pair");
        if (edges && n < cap)
            for (int h = 0; h < 2; ++h) {
                std::uint64_t x = 0;
                for (int b = 7; b >= 0; --b) x = (x << 8) | rec[8 * h + b];
                edges[2 * n + h] = x;
            }
        ++n;
    }
    *m = n;
    if (edges && n > cap) return fail("rhg_read_edges_binary: buffer too small");
    return RHG_OK;
}

// stats.hpp:58-75 powerlaw_mle: continuous MLE with the -0.5 discreteness correction over
// the degrees >= d_min, in id order; fewer than 100 tail samples -> RHG_INVALID_ARGUMENT.
int rhg_powerlaw_mle(const std::uint32_t* degrees, std::uint64_t n, std::uint32_t d_min, double* gamma_hat) {
    if (!gamma_hat || (n && !degrees)) return fail("rhg_powerlaw_mle: null argument");
    double        log_sum = 0.0;
    std::uint64_t k       = 0;
    const double  x_min   = static_cast<double>(d_min) - 0.5;
    for (std::uint64_t i = 0; i < n; ++i)
        if (degrees[i] >= d_min) {
            log_sum += std::log(static_cast<double>(degrees[i]) / x_min);
            ++k;
        }
    if (k < 100) return fail("powerlaw_mle: fewer than 100 degrees above d_min");
    *gamma_hat = 1.0 + static_cast<double>(k) / log_sum;
    return RHG_OK;
}

} // extern "C"
