// generators.cpp — seeded host generation of the benchmark inputs.
//
// The draw primitives follow the reference's pinned transforms
// (proj/include/pcs/rng.hpp:16-46: std::mt19937_64, uniform01 from the top 53
// bits, Box-Muller with a cached spare), the surface generators follow
// proj/src/bench.cpp:40-87 and the noise model proj/src/noise.cpp:9-27.  Inputs
// stay on the host on purpose: device RNG would break draw-order parity.
//
// Configurations (BASELINE.json "configs", pinned readings in BASELINE.md §4):
//   1  sphere 20k + sigma 0.01, X0 = 2k subset
//   2  torus R=1 r=0.3, 950k surface + sigma 0.005, + 50k outliers in the AABB, X0 = 100k
//   3  z = 0.1 sin(8x) cos(8y) on [-1,1]^2, 10M, sigma 0.003 on z, X0 = 1M
//   4  sphere with density ~ e^{3.9 z}, 4M, sigma 0.005, X0 = 400k
//   5  8 random ellipsoids, 50M, sigma 0.002, X0 = 5M
// Seeds: surface stream 0, noise stream 1, outliers + X0 subset stream 2.
// X0 is a partial Fisher-Yates draw without replacement (j = i + gen() % (N-i)).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <random>
#include <vector>

#include "../../include/pcs_lop.h"

namespace {

constexpr double kPi = 3.141592653589793238462643383279502884;

inline double uniform01(std::mt19937_64& g) { return static_cast<double>(g() >> 11) * 0x1.0p-53; }
inline double uniform01_open_low(std::mt19937_64& g) {
    return static_cast<double>((g() >> 11) + 1) * 0x1.0p-53;
}

struct Normal {
    double spare = 0.0;
    bool has = false;
    double operator()(std::mt19937_64& g) {
        if (has) {
            has = false;
            return spare;
        }
        const double u1 = uniform01_open_low(g);
        const double u2 = uniform01(g);
        const double radius = std::sqrt(-2.0 * std::log(u1));
        const double angle = 2.0 * kPi * u2;
        spare = radius * std::sin(angle);
        has = true;
        return radius * std::cos(angle);
    }
};

void add_noise(double* xyz, uint64_t n, double sigma, uint64_t seed) {
    std::mt19937_64 g(seed);
    Normal nm;
    for (uint64_t i = 0; i < n; ++i) {
        const double dx = sigma * nm(g);
        const double dy = sigma * nm(g);
        const double dz = sigma * nm(g);
        xyz[3 * i] = xyz[3 * i] + dx;
        xyz[3 * i + 1] = xyz[3 * i + 1] + dy;
        xyz[3 * i + 2] = xyz[3 * i + 2] + dz;
    }
}

void plane(double* xyz, uint64_t n, std::mt19937_64& g) {
    for (uint64_t i = 0; i < n; ++i) {
        const double x = uniform01(g);
        const double y = uniform01(g);
        xyz[3 * i] = x;
        xyz[3 * i + 1] = y;
        xyz[3 * i + 2] = 0.0;
    }
}

void sphere(double* xyz, uint64_t n, std::mt19937_64& g) {
    for (uint64_t i = 0; i < n; ++i) {
        const double z = 1.0 - 2.0 * uniform01(g);
        const double phi = 2.0 * kPi * uniform01(g);
        const double rxy = std::sqrt(std::max(0.0, 1.0 - z * z));
        xyz[3 * i] = rxy * std::cos(phi);
        xyz[3 * i + 1] = rxy * std::sin(phi);
        xyz[3 * i + 2] = z;
    }
}

void torus(double* xyz, uint64_t n, double major, double minor, std::mt19937_64& g) {
    uint64_t k = 0;
    while (k < n) {
        const double u = 2.0 * kPi * uniform01(g);  // tube angle
        const double v = 2.0 * kPi * uniform01(g);  // around the axis
        const double accept = (major + minor * std::cos(u)) / (major + minor);
        if (uniform01(g) > accept) continue;
        const double ring = major + minor * std::cos(u);
        xyz[3 * k] = ring * std::cos(v);
        xyz[3 * k + 1] = ring * std::sin(v);
        xyz[3 * k + 2] = minor * std::sin(u);
        ++k;
    }
}

void bump(double* xyz, uint64_t n, std::mt19937_64& g) {
    for (uint64_t i = 0; i < n; ++i) {
        const double x = 2.0 * uniform01(g) - 1.0;
        const double y = 2.0 * uniform01(g) - 1.0;
        const double z = 0.5 * std::exp(-(x * x + y * y) / 0.25);
        xyz[3 * i] = x;
        xyz[3 * i + 1] = y;
        xyz[3 * i + 2] = z;
    }
}

uint64_t scaled(uint64_t full, double scale) {
    const double v = std::floor((double)full * scale + 0.5);
    return v < 1.0 ? 1 : (uint64_t)v;
}

struct Sizes {
    uint64_t surface, outliers, nx;
};

bool sizes_of(int cfg, double scale, Sizes* s) {
    switch (cfg) {
        case 1: *s = {scaled(20000, scale), 0, scaled(2000, scale)}; return true;
        case 2: *s = {scaled(950000, scale), scaled(50000, scale), scaled(100000, scale)}; return true;
        case 3: *s = {scaled(10000000, scale), 0, scaled(1000000, scale)}; return true;
        case 4: *s = {scaled(4000000, scale), 0, scaled(400000, scale)}; return true;
        case 5: *s = {scaled(50000000, scale), 0, scaled(5000000, scale)}; return true;
        default: return false;
    }
}

void subset(const double* P, uint64_t n, uint64_t m, std::mt19937_64& g, double* X0) {
    std::vector<uint32_t> idx(n);
    for (uint64_t i = 0; i < n; ++i) idx[i] = (uint32_t)i;
    for (uint64_t i = 0; i < m; ++i) {
        const uint64_t j = i + g() % (n - i);
        std::swap(idx[i], idx[j]);
        std::memcpy(X0 + 3 * i, P + 3 * (uint64_t)idx[i], 3 * sizeof(double));
    }
}

double ellipsoid_area(double a, double b, double c) {
    // Knud Thomsen's approximation (max rel. error ~1%)
    const double p = 1.6075;
    const double ap = std::pow(a, p), bp = std::pow(b, p), cp = std::pow(c, p);
    return 4.0 * kPi * std::pow((ap * bp + ap * cp + bp * cp) / 3.0, 1.0 / p);
}

void generate(int cfg, const Sizes& sz, double* P, double* X0) {
    std::mt19937_64 gs(0), gx(2);
    const uint64_t n = sz.surface + sz.outliers;
    switch (cfg) {
        case 1:
            sphere(P, sz.surface, gs);
            add_noise(P, sz.surface, 0.01, 1);
            break;
        case 2: {
            torus(P, sz.surface, 1.0, 0.3, gs);
            add_noise(P, sz.surface, 0.005, 1);
            double lo[3] = {P[0], P[1], P[2]}, hi[3] = {P[0], P[1], P[2]};
            for (uint64_t i = 1; i < sz.surface; ++i)
                for (int a = 0; a < 3; ++a) {
                    lo[a] = std::min(lo[a], P[3 * i + a]);
                    hi[a] = std::max(hi[a], P[3 * i + a]);
                }
            for (uint64_t i = sz.surface; i < n; ++i)
                for (int a = 0; a < 3; ++a) P[3 * i + a] = lo[a] + (hi[a] - lo[a]) * uniform01(gx);
            break;
        }
        case 3: {
            for (uint64_t i = 0; i < n; ++i) {
                const double x = 2.0 * uniform01(gs) - 1.0;
                const double y = 2.0 * uniform01(gs) - 1.0;
                P[3 * i] = x;
                P[3 * i + 1] = y;
                P[3 * i + 2] = 0.1 * std::sin(8.0 * x) * std::cos(8.0 * y);
            }
            std::mt19937_64 gn(1);
            Normal nm;
            for (uint64_t i = 0; i < n; ++i) P[3 * i + 2] = P[3 * i + 2] + 0.003 * nm(gn);
            break;
        }
        case 4: {
            const double k = 3.9, ea = std::exp(-k), eb = std::exp(k);
            for (uint64_t i = 0; i < n; ++i) {
                const double u = uniform01(gs);
                double z = std::log(ea + u * (eb - ea)) / k;  // inverse CDF of ~e^{kz} on [-1,1]
                z = std::min(1.0, std::max(-1.0, z));
                const double phi = 2.0 * kPi * uniform01(gs);
                const double rxy = std::sqrt(std::max(0.0, 1.0 - z * z));
                P[3 * i] = rxy * std::cos(phi);
                P[3 * i + 1] = rxy * std::sin(phi);
                P[3 * i + 2] = z;
            }
            add_noise(P, n, 0.005, 1);
            break;
        }
        case 5: {
            double ax[8][3], ce[8][3], area[8], tot = 0.0;
            for (int e = 0; e < 8; ++e) {
                for (int a = 0; a < 3; ++a) ax[e][a] = 0.2 + 0.4 * uniform01(gs);
                for (int a = 0; a < 3; ++a) ce[e][a] = -1.0 + 2.0 * uniform01(gs);
                area[e] = ellipsoid_area(ax[e][0], ax[e][1], ax[e][2]);
                tot += area[e];
            }
            uint64_t cnt[8], used = 0;
            for (int e = 0; e < 8; ++e) {
                cnt[e] = (uint64_t)std::floor((double)n * area[e] / tot);
                used += cnt[e];
            }
            for (int e = 0; used < n; e = (e + 1) % 8, ++used) cnt[e]++;
            uint64_t k = 0;
            for (int e = 0; e < 8; ++e) {
                const double a = ax[e][0], b = ax[e][1], c = ax[e][2];
                const double gmax = std::max(b * c, std::max(a * c, a * b));
                uint64_t got = 0;
                while (got < cnt[e]) {
                    const double z = 1.0 - 2.0 * uniform01(gs);
                    const double phi = 2.0 * kPi * uniform01(gs);
                    const double r = std::sqrt(std::max(0.0, 1.0 - z * z));
                    const double x = r * std::cos(phi), y = r * std::sin(phi);
                    // area element of the map sphere -> ellipsoid
                    const double gl = std::sqrt((b * c * x) * (b * c * x) + (a * c * y) * (a * c * y) +
                                                (a * b * z) * (a * b * z));
                    if (uniform01(gs) > gl / gmax) continue;
                    P[3 * k] = ce[e][0] + a * x;
                    P[3 * k + 1] = ce[e][1] + b * y;
                    P[3 * k + 2] = ce[e][2] + c * z;
                    ++k;
                    ++got;
                }
            }
            add_noise(P, n, 0.002, 1);
            break;
        }
    }
    if (X0) subset(P, n, sz.nx, gx, X0);
}

}  // namespace

extern "C" {

pcs_status pcs_generate_surface(int32_t kind, uint64_t n, uint64_t seed, double* xyz) {
    if (n < 1 || !xyz) return PCS_ERR_INVALID_PARAM;
    std::mt19937_64 g(seed);
    switch (kind) {
        case 0: plane(xyz, n, g); break;
        case 1: sphere(xyz, n, g); break;
        case 2: torus(xyz, n, 1.0, 0.35, g); break;
        case 3: bump(xyz, n, g); break;
        default: return PCS_ERR_INVALID_PARAM;
    }
    return PCS_OK;
}

pcs_status pcs_add_noise(double* xyz, uint64_t n, double sigma, uint64_t seed) {
    if (!(sigma >= 0.0) || !std::isfinite(sigma)) return PCS_ERR_INVALID_PARAM;
    if (n && !xyz) return PCS_ERR_INVALID_PARAM;
    add_noise(xyz, n, sigma, seed);
    return PCS_OK;
}

pcs_status pcs_config_sizes(int32_t config, double scale, uint64_t* n_p, uint64_t* n_x) {
    Sizes s;
    if (!(scale > 0.0) || !sizes_of(config, scale, &s)) return PCS_ERR_INVALID_PARAM;
    if (s.nx > s.surface + s.outliers) s.nx = s.surface + s.outliers;
    if (n_p) *n_p = s.surface + s.outliers;
    if (n_x) *n_x = s.nx;
    return PCS_OK;
}

pcs_status pcs_generate_config(int32_t config, double scale, double* P_xyz, double* X0_xyz) {
    Sizes s;
    if (!(scale > 0.0) || !sizes_of(config, scale, &s) || !P_xyz) return PCS_ERR_INVALID_PARAM;
    if (s.nx > s.surface + s.outliers) s.nx = s.surface + s.outliers;
    generate(config, s, P_xyz, X0_xyz);
    return PCS_OK;
}

}  // extern "C"
