// Host test of paper_2401_03365_b200/csrc/dconv.h (the formatter / parser the
// cloud IO kernels run on the device) against libstdc++'s std::to_chars /
// std::from_chars, which the reference's writer and reader call
// (proj/src/io.cpp:36-48, :240-245).  Built and run by tests/test_dconv.py.
#define __device__
#define __constant__
#include "dconv.h"

#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>

using namespace pcsb::dconv;

static long nfail = 0, nparsed = 0, nfallback = 0;

static void check_fmt(double v) {
    char a[64], b[64];
    const auto r = std::to_chars(a, a + 64, v);
    const int na = (int)(r.ptr - a);
    const int nb = format(v, b);
    if (na != nb || std::memcmp(a, b, na)) {
        if (nfail++ < 20) std::printf("FORMAT %.17g: to_chars '%.*s' got '%.*s'\n", v, na, a, nb, b);
    }
}

static void check_parse(const char* s) {
    const size_t n = std::strlen(s);
    double want = 0.0, got = 0.0;
    const auto r = std::from_chars(s, s + n, want);
    if (!parse(s, s + n, &got)) {
        ++nfallback;
        return;
    }
    ++nparsed;
    if (r.ec != std::errc() || r.ptr != s + n || std::memcmp(&want, &got, 8)) {
        if (nfail++ < 20) std::printf("PARSE '%s': from_chars %.17g got %.17g\n", s, want, got);
    }
}

int main(int argc, char** argv) {
    const long N = argc > 1 ? std::atol(argv[1]) : 1000000;
    std::mt19937_64 g(argc > 2 ? std::atol(argv[2]) : 1);
    const double specials[] = {0.0, -0.0, 1.0, -1.0, 0.1, 0.3, 1e22, 1e23, 5e-324,
                               2.2250738585072014e-308, 1.7976931348623157e308,
                               9007199254740992.0, 9007199254740993.0, 1.2345678901234568e20,
                               123456789012345678.0, 1e-5, 1.5e-5, 0.001, 100, 1e15, 1e16, 123.456,
                               1e21, 1e20, 12345678901234567890.0, 1e-7, 1.25e-6, 1e100, 4.35e17,
                               2.0, 0.5, 1.0 / 3, 2.0 / 3, 1e-300, 1e300, 1.5e-323};
    for (double v : specials) check_fmt(v);
    for (long i = 0; i < N; ++i) {
        uint64_t bits = g();
        double v;
        std::memcpy(&v, &bits, 8);
        if (std::isfinite(v)) check_fmt(v);  // every exponent, subnormals included
        double c = std::ldexp((double)(g() >> 11), -53) * 4 - 2;  // coordinates
        c *= std::pow(10.0, (int)(g() % 9) - 4);
        check_fmt(c);
        check_fmt((double)(g() >> (g() % 64)));  // integers, around 2^53 and beyond
    }
    std::printf("format: %ld mismatches\n", nfail);
    const long f0 = nfail;
    char buf[64];
    for (long i = 0; i < N; ++i) {
        double c = std::ldexp((double)(g() >> 11), -53) * 4 - 2;
        c *= std::pow(10.0, (int)(g() % 9) - 4);
        buf[format(c, buf)] = 0;
        check_parse(buf);
        char s[80];
        int k = 0;
        const int nd = 1 + (int)(g() % 22);
        if (g() & 1) s[k++] = '-';
        const int dot = (int)(g() % (nd + 1));
        for (int j = 0; j < nd; ++j) {
            if (j == dot && j) s[k++] = '.';
            s[k++] = (char)('0' + g() % 10);
        }
        if (g() % 3 == 0) {
            s[k++] = (g() & 1) ? 'e' : 'E';
            k += std::snprintf(s + k, 16, "%d", (int)(g() % 70) - 35);
        }
        s[k] = 0;
        check_parse(s);
        uint64_t bits = g();
        double v;
        std::memcpy(&v, &bits, 8);
        if (std::isfinite(v)) {
            buf[format(v, buf)] = 0;
            check_parse(buf);
        }
    }
    const char* edge[] = {"0", "-0", "0.0", "00012.5000", ".5", "5.", "1e5", "1E-5", "1e+5",
                          "-.5e-3", "1.7976931348623157e308", "4.9e-324", "9007199254740993",
                          "9007199254740992.5", "0.30000000000000004", "123456789012345678",
                          "1234567890123456789", "12345678901234567890", "1e27", "1e-27",
                          "2.5e-27", "9.999999999999999e26", "1e", "-", ".", "e5", "1.2.3",
                          "+1", "--1", "1e+", "0x10", "inf", "nan", "1e999", "1e-999"};
    for (const char* s : edge) check_parse(s);
    std::printf("parse: %ld mismatches, %ld handled on the fast path, %ld left to the host\n",
                nfail - f0, nparsed, nfallback);
    return nfail != 0;
}
