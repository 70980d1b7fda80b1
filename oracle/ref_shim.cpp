// ref_shim.cpp — extern "C" entry points over the UNMODIFIED reference
// library, compiled together with the reference's own sources where they lie
// (/root/reference/proj/src/{core,kernels,spatial,lop,noise,bench,io}.cpp) by
// oracle/Makefile into oracle/_ref/libpcs_ref.so.
//
// TEST INFRASTRUCTURE ONLY: loaded by tests/ (to pin oracle/lop_oracle.c) and
// by bench.py's --impl reference / cpu_baseline legs (the reference's own CPU
// path, timed on the host cores).  No reference source is copied here; this
// file only calls the reference's public API:
//   pcs::lop_project            proj/include/pcs/lop.hpp:51-53
//   pcs::SpatialIndex           proj/include/pcs/spatial.hpp:19-56
//   pcs::add_noise              proj/include/pcs/noise.hpp
//   pcs::generate_surface       proj/include/pcs/bench.hpp
//   pcs::write_cloud_stream, read_cloud_stream  proj/include/pcs/io.hpp
//   pcs::deviation, deviation_to_mesh, point_triangle_distance
//                               proj/include/pcs/metrics.hpp
#include <chrono>
#include <sstream>
#include <omp.h>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "pcs/bench.hpp"
#include "pcs/errors.hpp"
#include "pcs/io.hpp"
#include "pcs/lop.hpp"
#include "pcs/metrics.hpp"
#include "pcs/mls.hpp"
#include "pcs/noise.hpp"
#include "pcs/parallel.hpp"
#include "pcs/spatial.hpp"

// bench.cpp references the MLS operators (run_benchmark); they need Eigen
// (proj/src/wls.cpp), which this image lacks, and they are off the LOP path.
namespace pcs {
std::pair<PointCloud, SmoothingSummary> smooth_cloud(const PointCloud&, const MlsParams&) {
    throw Error("ref_shim: MLS is not built (Eigen absent); off the LOP path");
}
std::pair<PointCloud, SmoothingSummary> parallel_smooth(const PointCloud&, const MlsParams&,
                                                        std::size_t) {
    throw Error("ref_shim: MLS is not built (Eigen absent); off the LOP path");
}
}  // namespace pcs

namespace {
thread_local std::string g_err;

pcs::PointCloud to_cloud(const double* xyz, std::uint64_t n) {
    pcs::PointCloud c;
    c.points.resize(n);
    for (std::uint64_t i = 0; i < n; ++i) c.points[i] = {xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]};
    return c;
}

void from_cloud(const pcs::PointCloud& c, double* xyz) {
    for (std::size_t i = 0; i < c.size(); ++i) {
        xyz[3 * i] = c[i].x;
        xyz[3 * i + 1] = c[i].y;
        xyz[3 * i + 2] = c[i].z;
    }
}

int code_of(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const pcs::InvalidParam*>(&e)) return 1;
    if (dynamic_cast<const pcs::EmptyCloud*>(&e)) return 2;
    if (dynamic_cast<const pcs::EmptyMesh*>(&e)) return 8;
    return 9;
}
}  // namespace

extern "C" {

struct ref_summary {
    std::int32_t iterations_run;
    std::int32_t converged;
    std::uint64_t isolated_events;
    std::uint64_t coincident_pairs;
    std::uint64_t n_isolated;
};

const char* ref_last_error() { return g_err.c_str(); }

int ref_lop_project(const double* P, std::uint64_t n, const double* X0, std::uint64_t m, double h,
                    double cutoff, double mu, int iterations, double tol, double* out,
                    ref_summary* sum, std::uint32_t* isolated_out) {
    try {
        pcs::LopParams prm;
        prm.kernel.h = h;
        prm.kernel.cutoff_multiple = cutoff;
        prm.mu = mu;
        prm.iterations = iterations;
        prm.convergence_tol = tol;
        const auto data = to_cloud(P, n);
        const auto init = to_cloud(X0, m);
        const auto [q, s] = pcs::lop_project(data, init, prm);
        from_cloud(q, out);
        if (sum) {
            sum->iterations_run = s.iterations_run;
            sum->converged = s.converged ? 1 : 0;
            sum->isolated_events = s.isolated_events;
            sum->coincident_pairs = s.coincident_pairs;
            sum->n_isolated = s.isolated_indices.size();
        }
        if (isolated_out)
            for (std::size_t k = 0; k < s.isolated_indices.size(); ++k)
                isolated_out[k] = s.isolated_indices[k];
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// CSR radius queries through the reference kd-tree.  offsets: m+1 entries.
// Pass idx == nullptr to size the output first.
int ref_radius_query_all(const double* C, std::uint64_t n, const double* Q, std::uint64_t m,
                         double r, std::uint64_t* offsets, std::uint32_t* idx, double* dist) {
    try {
        const auto cloud = to_cloud(C, n);
        const pcs::SpatialIndex index(cloud);
        std::vector<pcs::SpatialIndex::Hit> hits;
        offsets[0] = 0;
        for (std::uint64_t i = 0; i < m; ++i) {
            index.radius_query({Q[3 * i], Q[3 * i + 1], Q[3 * i + 2]}, r, hits);
            if (idx) {
                const std::uint64_t o = offsets[i];
                for (std::size_t k = 0; k < hits.size(); ++k) {
                    idx[o + k] = static_cast<std::uint32_t>(hits[k].index);
                    if (dist) dist[o + k] = hits[k].distance;
                }
            } else {
                offsets[i + 1] = offsets[i] + hits.size();
            }
        }
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

int ref_add_noise(double* xyz, std::uint64_t n, double sigma, std::uint64_t seed) {
    try {
        const auto c = pcs::add_noise(to_cloud(xyz, n), {sigma, seed});
        from_cloud(c, xyz);
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// kind: 0 plane, 1 sphere, 2 torus, 3 gaussian bump (pcs::SurfaceKind order)
int ref_generate_surface(int kind, std::uint64_t n, std::uint64_t seed, double* xyz) {
    try {
        const auto c = pcs::generate_surface(
            {static_cast<pcs::SurfaceKind>(kind), static_cast<std::size_t>(n), seed});
        from_cloud(c, xyz);
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// Wall time (ms) of the reference's one-time data index build
// (SpatialIndex(data), proj/src/lop.cpp:24), so a timed lop_project sample can
// report the sweep alone.
double ref_index_build_ms(const double* P, std::uint64_t n) {
    const auto cloud = to_cloud(P, n);
    const auto t0 = std::chrono::steady_clock::now();
    const pcs::SpatialIndex index(cloud);
    const auto t1 = std::chrono::steady_clock::now();
    return std::chrono::duration<double, std::milli>(t1 - t0).count() + 0.0 * index.size();
}

// SpatialIndex::nearest for every query (reference kd-tree).
int ref_nearest_all(const double* C, std::uint64_t n, const double* Q, std::uint64_t m,
                    std::uint32_t* idx, double* dist, int threads) {
    try {
        const auto cloud = to_cloud(C, n);
        const pcs::SpatialIndex index(cloud);
        int err = 0;
#pragma omp parallel for schedule(dynamic, 256) num_threads(threads > 0 ? threads : omp_get_max_threads())
        for (std::int64_t i = 0; i < (std::int64_t)m; ++i) {
            try {
                const auto h = index.nearest({Q[3 * i], Q[3 * i + 1], Q[3 * i + 2]});
                idx[i] = static_cast<std::uint32_t>(h.index);
                dist[i] = h.distance;
            } catch (...) {
#pragma omp atomic write
                err = 1;
            }
        }
        if (err) throw pcs::EmptyCloud("nearest: index built over an empty cloud");
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// pcs::deviation; out = {n, mean, std (RMS), max}; dist may be null.
int ref_deviation(const double* cloud, std::uint64_t m, const double* ref, std::uint64_t n,
                  double* out, double* dist) {
    try {
        const auto r = pcs::deviation(to_cloud(cloud, m), to_cloud(ref, n), dist != nullptr);
        out[0] = (double)r.n;
        out[1] = r.mean_distance;
        out[2] = r.std_deviation;
        out[3] = r.max_distance;
        if (dist) std::memcpy(dist, r.distances.data(), m * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

int ref_deviation_to_mesh(const double* cloud, std::uint64_t m, const double* tri,
                          std::uint64_t ntri, double* out, double* dist) {
    try {
        pcs::TriangleMesh mesh;
        for (std::uint64_t t = 0; t < ntri; ++t) {
            const double* v = tri + 9 * t;
            mesh.triangles.push_back({{v[0], v[1], v[2]}, {v[3], v[4], v[5]}, {v[6], v[7], v[8]}});
        }
        const auto r = pcs::deviation_to_mesh(to_cloud(cloud, m), mesh, dist != nullptr);
        out[0] = (double)r.n;
        out[1] = r.mean_distance;
        out[2] = r.std_deviation;
        out[3] = r.max_distance;
        if (dist) std::memcpy(dist, r.distances.data(), m * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

double ref_point_triangle_distance(const double* p, const double* t) {
    return pcs::point_triangle_distance({p[0], p[1], p[2]},
                                        {{t[0], t[1], t[2]}, {t[3], t[4], t[5]}, {t[6], t[7], t[8]}});
}

// write_cloud_stream into out (cap bytes); *len = bytes (returns 7 when cap is short)
int ref_format_cloud(const double* xyz, std::uint64_t n, int fmt, char* out, std::uint64_t cap,
                     std::uint64_t* len) {
    try {
        std::ostringstream os;
        pcs::write_cloud_stream(to_cloud(xyz, n), os,
                                fmt == 0 ? pcs::CloudFormat::Xyz : pcs::CloudFormat::PlyAscii);
        const std::string t = os.str();
        *len = t.size();
        if (!out || cap < t.size()) return 7;
        std::memcpy(out, t.data(), t.size());
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// read_cloud_stream; *n = points (returns 7 when cap is short); a ParseError
// returns 10 with its line number and message
int ref_parse_cloud(const char* text, std::uint64_t len, int fmt, double* out, std::uint64_t cap,
                    std::uint64_t* n, std::int64_t* line) {
    try {
        std::istringstream is(std::string(text, len));
        const auto c = pcs::read_cloud_stream(
            is, fmt == 0 ? pcs::CloudFormat::Xyz : pcs::CloudFormat::PlyAscii, "<memory>");
        *n = c.size();
        if (cap < c.size()) return 7;
        from_cloud(c, out);
        return 0;
    } catch (const pcs::ParseError& e) {
        g_err = e.what();
        *line = e.line_number;
        return 10;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

double ref_theta(double d, double h, double cutoff) {
    return pcs::theta(d, pcs::KernelParams{h, cutoff});
}

}  // extern "C"
