// bsq_io.cpp -- host-side artifact formatting.
//
// The reference writes ESRI-ASCII snapshots with one Python `f"{v:.17g}"`
// per cell (grid.py:250-268), about 8 s per 4096^2 field.  This formats the
// same text with the C library's correctly rounded %.17g on all host cores.
// Python's float formatting and glibc's agree digit for digit (both round
// correctly, both print at least two exponent digits); the one difference is
// NaN, which Python prints as "nan" whatever its sign bit, so it is written
// explicitly.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/bsq.h"

namespace {

void format_rows(const double *v, long r0, long r1, long nrows, long ncols, long stride,
                 int north_first, std::string *out) {
    char buf[40];
    for (long r = r0; r < r1; r++) {
        const long j = north_first ? nrows - 1 - r : r;
        const double *row = v + j * stride;
        for (long i = 0; i < ncols; i++) {
            const double x = row[i];
            int n;
            if (std::isnan(x)) {
                std::memcpy(buf, "nan", 3);
                n = 3;
            } else {
                n = std::snprintf(buf, sizeof buf, "%.17g", x);
            }
            if (i) out->push_back(' ');
            out->append(buf, (size_t)n);
        }
        out->push_back('\n');
    }
}

}  // namespace

extern "C" long long bsq_append_rows(const char *path, const double *values, long nrows,
                                     long ncols, long stride, int north_first) {
    if (!path || !values || nrows < 0 || ncols < 0 || stride < ncols) return -1;
    unsigned nt = std::thread::hardware_concurrency();
    if (nt == 0) nt = 1;
    if ((long)nt > nrows) nt = nrows > 0 ? (unsigned)nrows : 1;
    std::vector<std::string> parts(nt);
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < nt; t++) {
        const long r0 = nrows * t / nt, r1 = nrows * (t + 1) / nt;
        pool.emplace_back(format_rows, values, r0, r1, nrows, ncols, stride, north_first,
                          &parts[t]);
    }
    for (auto &th : pool) th.join();
    FILE *f = std::fopen(path, "ab");
    if (!f) return -1;
    long long total = 0;
    for (auto &p : parts) {
        if (std::fwrite(p.data(), 1, p.size(), f) != p.size()) {
            std::fclose(f);
            return -1;
        }
        total += (long long)p.size();
    }
    if (std::fclose(f) != 0) return -1;
    return total;
}

// boundary.maker_surface_flux (reference boundary.py:190-199) for the
// per-step host parameters: the same libm sin Python's math.sin calls, the
// same operations in component order, so the sums are bitwise the
// reference's (built with -ffp-contract=off).  comps is n x 4 rows of
// (amplitude, omega, k, phase); out = (eta, flux).
extern "C" int bsq_maker_sums(const double *comps, int n, double t, double *out) {
    if ((!comps && n > 0) || n < 0 || !out) return BSQ_ERR_BAD_ARG;
    double eta = 0.0, flux = 0.0;
    for (int c = 0; c < n; c++) {
        const double *r = comps + 4 * c;
        const double s = r[0] * std::sin(r[1] * t + r[3]);
        eta += s;
        flux += s * (r[1] / r[2]);
    }
    out[0] = eta;
    out[1] = flux;
    return BSQ_OK;
}
