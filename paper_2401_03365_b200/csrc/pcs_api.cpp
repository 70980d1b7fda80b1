// pcs_api.cpp — the reference's C++ API (include/pcs/*.hpp) over the C ABI.
//
// pcs::lop_project keeps the declaration, structs, validation order and
// exception types of proj/include/pcs/lop.hpp:51-53 / proj/src/lop.cpp:13-20,
// so the reference's own proj/tests/test_lop.cpp compiles and runs against
// this library unchanged (tests/test_dropin.py).
#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstring>
#include <fstream>
#include <iterator>
#include <sstream>
#include <memory>
#include <string>
#include <vector>

#include "../../include/pcs/bench.hpp"
#include "../../include/pcs/kernels.hpp"
#include "../../include/pcs/lop.hpp"
#include "../../include/pcs/lop_ex.hpp"
#include "../../include/pcs/io.hpp"
#include "../../include/pcs/metrics.hpp"
#include "../../include/pcs/noise.hpp"
#include "../../include/pcs_lop.h"
#include "ptri.h"

namespace pcs {

namespace {

[[noreturn]] void raise(pcs_status st) {
    const std::string msg = pcs_last_error();
    switch (st) {
        case PCS_ERR_INVALID_PARAM: throw InvalidParam(msg);
        case PCS_ERR_EMPTY_CLOUD: throw EmptyCloud(msg);
        case PCS_ERR_EMPTY_MESH: throw EmptyMesh(msg);
        default: throw NumericalFailure(msg);
    }
}

const double* xyz(const PointCloud& c) { return c.empty() ? nullptr : &c.points[0].x; }

}  // namespace

bool PointCloud::all_finite() const {
    for (const Point3& p : points)
        if (!is_finite(p)) return false;
    return true;
}

Aabb bounding_box(const PointCloud& cloud) {
    if (cloud.empty()) throw EmptyCloud("bounding_box: empty cloud");
    Aabb b{cloud[0], cloud[0]};
    for (const Point3& p : cloud) {
        b.min.x = std::fmin(b.min.x, p.x);
        b.min.y = std::fmin(b.min.y, p.y);
        b.min.z = std::fmin(b.min.z, p.z);
        b.max.x = std::fmax(b.max.x, p.x);
        b.max.y = std::fmax(b.max.y, p.y);
        b.max.z = std::fmax(b.max.z, p.z);
    }
    return b;
}

double theta(double d, const KernelParams& params) {
    params.validate();
    if (d > params.support()) return 0.0;
    const double s = d / params.h;
    return std::exp(-s * s);
}

double eta(double d) {
    if (!(d > 0.0)) throw InvalidParam("eta requires d > 0");
    return 1.0 / (3.0 * d * d * d);
}

double eta_derivative_magnitude(double d) {
    if (!(d > 0.0)) throw InvalidParam("eta_derivative_magnitude requires d > 0");
    const double d2 = d * d;
    return 1.0 / (d2 * d2);
}

std::pair<PointCloud, LopSummary> lop_project_ex(const PointCloud& data, const PointCloud& initial,
                                                 const LopParams& params, const LopOptions& options,
                                                 LopStats* stats) {
    params.validate();  // InvalidParam first (lop.cpp:13)
    if (data.empty()) throw EmptyCloud("lop_project: data cloud is empty");
    LopSummary summary;
    PointCloud out = initial;
    if (initial.empty()) return {out, summary};

    pcs_lop_desc d;
    pcs_lop_desc_default(&d);
    d.h = params.kernel.h;
    d.cutoff_multiple = params.kernel.cutoff_multiple;
    d.mu = params.mu;
    d.iterations = params.iterations;
    d.convergence_tol = params.convergence_tol;
    d.eta_kind = options.eta == EtaKind::NegLinear ? PCS_ETA_NEG_LINEAR : PCS_ETA_INV_CUBE;
    d.density_weights = options.density_weights ? 1 : 0;
    d.precision = options.precision == Precision::Fp32 ? PCS_PREC_FP32 : PCS_PREC_FP64;
    d.device = options.device;

    pcs_lop_summary s;
    std::vector<std::uint32_t> iso(initial.size());
    const pcs_status st = pcs_lop_run(&d, xyz(data), data.size(), xyz(initial), initial.size(),
                                      &out.points[0].x, &s, iso.data(), iso.size());
    if (st != PCS_OK) raise(st);
    summary.iterations_run = s.iterations_run;
    summary.converged = s.converged != 0;
    summary.isolated_events = s.isolated_events;
    summary.coincident_pairs = s.coincident_pairs;
    iso.resize(s.n_isolated);
    summary.isolated_indices = std::move(iso);
    if (stats) {
        stats->interactions_attr = s.interactions_attr;
        stats->interactions_rep = s.interactions_rep;
        stats->density_pairs = s.density_pairs;
        stats->careful_points = s.careful_points;
        stats->setup_ms = s.setup_ms;
        stats->sweeps_ms = s.sweeps_ms;
        stats->kernel_ms = s.kernel_ms;
        stats->sort_ms = s.sort_ms;
        stats->last_max_disp = s.last_max_disp;
    }
    return {out, summary};
}

std::pair<PointCloud, LopSummary> lop_project(const PointCloud& data, const PointCloud& initial,
                                              const LopParams& params) {
    return lop_project_ex(data, initial, params, LopOptions{});
}

PointCloud add_noise(const PointCloud& cloud, const NoiseParams& params) {
    if (!(params.sigma >= 0.0) || !std::isfinite(params.sigma))
        throw InvalidParam("add_noise: sigma must be finite and >= 0");
    PointCloud out = cloud;
    if (!out.empty()) {
        const pcs_status st = pcs_add_noise(&out.points[0].x, out.size(), params.sigma, params.seed);
        if (st != PCS_OK) raise(st);
    }
    return out;
}

PointCloud generate_surface(const SyntheticSurface& surface) {
    if (surface.n < 1) throw InvalidParam("generate_surface: n must be >= 1");
    PointCloud c;
    c.points.resize(surface.n);
    const pcs_status st =
        pcs_generate_surface(static_cast<int32_t>(surface.kind), surface.n, surface.seed, &c.points[0].x);
    if (st != PCS_OK) throw InvalidParam("generate_surface: invalid surface kind");
    return c;
}

// ---- deviation metrics (proj/include/pcs/metrics.hpp, proj/src/metrics.cpp) ----

namespace {

DeviationReport to_report(const pcs_deviation_report& r, std::vector<double>&& d, bool keep) {
    DeviationReport out;
    out.n = (std::size_t)r.n;
    out.mean_distance = r.mean_distance;
    out.std_deviation = r.std_deviation;
    out.max_distance = r.max_distance;
    if (keep) out.distances = std::move(d);
    return out;
}

pcs_lop_desc metrics_desc() {
    pcs_lop_desc d;
    pcs_lop_desc_default(&d);
    return d;
}

}  // namespace

DeviationReport deviation(const PointCloud& cloud, const PointCloud& reference,
                          bool keep_distances) {
    const pcs_lop_desc d = metrics_desc();
    pcs_deviation_report r{};
    std::vector<double> dist(keep_distances ? cloud.size() : 0);
    const pcs_status st = pcs_deviation(&d, xyz(cloud), cloud.size(), xyz(reference),
                                        reference.size(), &r, keep_distances ? dist.data() : nullptr);
    if (st != PCS_OK) raise(st);
    return to_report(r, std::move(dist), keep_distances);
}

double point_triangle_distance(Point3 p, const Triangle& tri) {
    using pcsb::ptri::V3;
    return pcsb::ptri::distance(V3{p.x, p.y, p.z}, V3{tri.a.x, tri.a.y, tri.a.z},
                                V3{tri.b.x, tri.b.y, tri.b.z}, V3{tri.c.x, tri.c.y, tri.c.z});
}

DeviationReport deviation_to_mesh(const PointCloud& cloud, const TriangleMesh& mesh,
                                  bool keep_distances) {
    const pcs_lop_desc d = metrics_desc();
    pcs_deviation_report r{};
    std::vector<double> dist(keep_distances ? cloud.size() : 0);
    const double* tri = mesh.empty() ? nullptr : &mesh.triangles[0].a.x;
    const pcs_status st = pcs_deviation_to_mesh(&d, xyz(cloud), cloud.size(), tri, mesh.size(), &r,
                                                keep_distances ? dist.data() : nullptr);
    if (st != PCS_OK) raise(st);
    return to_report(r, std::move(dist), keep_distances);
}

// ---- cloud files (proj/include/pcs/io.hpp, proj/src/io.cpp) ----------------------

namespace {

int32_t fmt_code(CloudFormat f) { return f == CloudFormat::Xyz ? PCS_FMT_XYZ : PCS_FMT_PLY_ASCII; }

std::string slurp(std::istream& in) {
    return std::string(std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>());
}

[[noreturn]] void raise_parse(pcs_status st, const pcs_parse_error& e, const std::string& name) {
    if (st == PCS_ERR_PARSE) throw ParseError(name, (long)e.line, e.reason);
    raise(st);
}

}  // namespace

std::string format_double(double value) {
    char buf[40];
    const int32_t n = pcs_format_double(value, buf);
    return std::string(buf, (size_t)n);
}

CloudFormat format_from_path(const std::string& path) {
    const auto dot = path.find_last_of('.');
    std::string ext = dot == std::string::npos ? std::string() : path.substr(dot);
    for (char& c : ext) c = (char)std::tolower((unsigned char)c);
    if (ext == ".xyz") return CloudFormat::Xyz;
    if (ext == ".ply") return CloudFormat::PlyAscii;
    throw InvalidParam("cannot infer cloud format from '" + path +
                       "' (expected .xyz or .ply); pass the format explicitly");
}

PointCloud read_cloud_stream(std::istream& in, CloudFormat format, const std::string& name) {
    const std::string text = slurp(in);
    pcs_lop_desc d;
    pcs_lop_desc_default(&d);
    // every point needs at least 6 bytes ("0 0 0\n"): an upper bound, no second pass.
    // The landing buffer is left uninitialised (only the pages the n parsed points
    // reach are ever touched; a value-initialised vector of the bound would zero
    // 24 bytes per 6 bytes of text)
    const size_t cap = text.size() / 6 + 1;
    std::unique_ptr<double[]> xyz(new double[3 * cap]);
    uint64_t n = 0;
    pcs_parse_error err{};
    const pcs_status st = pcs_parse_cloud(&d, text.data(), text.size(), fmt_code(format), xyz.get(),
                                          cap, &n, &err);
    if (st != PCS_OK) raise_parse(st, err, name);
    PointCloud cloud;
    cloud.points.resize((size_t)n);
    if (n) std::memcpy(&cloud.points[0].x, xyz.get(), (size_t)n * 3 * sizeof(double));
    return cloud;
}

PointCloud read_cloud(const std::string& path, CloudFormat format) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoError("cannot open '" + path + "' for reading");
    return read_cloud_stream(in, format, path);
}

PointCloud read_cloud(const std::string& path) { return read_cloud(path, format_from_path(path)); }

void write_cloud_stream(const PointCloud& cloud, std::ostream& out, CloudFormat format) {
    pcs_lop_desc d;
    pcs_lop_desc_default(&d);
    char* text = nullptr;
    uint64_t len = 0;
    const pcs_status st = pcs_format_cloud_alloc(&d, xyz(cloud), cloud.size(), fmt_code(format), &text, &len);
    if (st != PCS_OK) raise(st);
    out.write(text, (std::streamsize)len);
    pcs_free_buffer(text);
}

void write_cloud(const PointCloud& cloud, const std::string& path, CloudFormat format) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw IoError("cannot open '" + path + "' for writing");
    write_cloud_stream(cloud, out, format);
    out.flush();
    if (!out) throw IoError("write to '" + path + "' failed");
}

void write_cloud(const PointCloud& cloud, const std::string& path) {
    write_cloud(cloud, path, format_from_path(path));
}

TriangleMesh read_mesh_stream(std::istream& in, const std::string& name) {
    const std::string text = slurp(in);
    uint64_t nt = 0;
    pcs_parse_error err{};
    pcs_status st = pcs_parse_mesh(text.data(), text.size(), nullptr, 0, &nt, &err);
    std::vector<double> tri;
    if (st == PCS_ERR_CAPACITY) {
        tri.resize((size_t)nt * 9);
        st = pcs_parse_mesh(text.data(), text.size(), tri.data(), nt, &nt, &err);
    }
    if (st != PCS_OK) raise_parse(st, err, name);
    TriangleMesh mesh;
    mesh.triangles.resize((size_t)nt);
    if (nt) std::memcpy(&mesh.triangles[0].a.x, tri.data(), tri.size() * sizeof(double));
    return mesh;
}

TriangleMesh read_mesh(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoError("cannot open '" + path + "' for reading");
    return read_mesh_stream(in, path);
}

}  // namespace pcs
