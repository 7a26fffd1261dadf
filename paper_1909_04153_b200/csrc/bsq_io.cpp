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
