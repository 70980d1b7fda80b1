// mls_api.cpp — the reference's MLS / WLS / spatial / parallel C++ API
// (include/pcs/{spatial,wls,mls,parallel}.hpp) over the C ABI, and the host
// part of the slab decomposition.
//
// Per-point numerics run on the device (mls.cu through pcs_mls_project /
// pcs_mls_smooth).  Host-side work is what the reference's contracts need
// exactly: validation order and messages, radius-query hits re-sorted by index
// with the reference's distance expression, replay of a coverage guard over
// the device's list of query centres, and the halo exchange of
// proj/src/parallel.cpp:129-203 (partition itself is pcs_mls_partition, mls.cu).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <numeric>
#include <vector>

#include "../../include/pcs/mls.hpp"
#include "../../include/pcs/parallel.hpp"
#include "../../include/pcs/spatial.hpp"
#include "../../include/pcs/wls.hpp"
#include "../../include/pcs_lop.h"


namespace pcs {

namespace {

[[noreturn]] void raise_status(pcs_status st) {
    const std::string msg = pcs_last_error();
    switch (st) {
        case PCS_ERR_INVALID_PARAM: throw InvalidParam(msg);
        case PCS_ERR_EMPTY_CLOUD: throw EmptyCloud(msg);
        default: throw NumericalFailure(msg);
    }
}

inline void check(pcs_status st) {
    if (st != PCS_OK) raise_status(st);
}

const double* xyz_of(const PointCloud& c) { return c.empty() ? nullptr : &c.points[0].x; }

pcs_mls_desc mls_desc(const KernelParams& k, int degree, double tol, int max_iter) {
    pcs_mls_desc d;
    pcs_mls_desc_default(&d);
    d.h = k.h;
    d.cutoff_multiple = k.cutoff_multiple;
    d.degree = degree;
    d.plane_tol = tol;
    d.plane_max_iter = max_iter;
    return d;
}

Point3 p3(const double* v) { return Point3{v[0], v[1], v[2]}; }

PlaneFitStatus plane_status_of(int32_t s) {
    switch (s) {
        case 0: return PlaneFitStatus::Ok;
        case 1: return PlaneFitStatus::TooFewNeighbors;
        case 2: return PlaneFitStatus::DegenerateNeighborhood;
        default: return PlaneFitStatus::NoConvergence;
    }
}

ProjectionStatus projection_status_of(int32_t s) {
    switch (s) {
        case 0: return ProjectionStatus::Full;
        case 1: return ProjectionStatus::DegradedDegree;
        case 2: return ProjectionStatus::PlaneOnly;
        default: return ProjectionStatus::Skipped;
    }
}

ProjectionOutcome outcome_of(const pcs_mls_result& R) {
    ProjectionOutcome o;
    o.projected = p3(R.projected);
    o.status = projection_status_of(R.status);
    o.degree_used = R.degree_used;
    o.iterations_used = R.iterations;
    o.plane_status = plane_status_of(R.plane_status);
    return o;
}

double axis_coord(Point3 p, int axis) { return axis == 0 ? p.x : (axis == 1 ? p.y : p.z); }

}  // namespace

// ---- SpatialIndex ---------------------------------------------------------------

struct SpatialIndex::Device {
    pcs_mls_index* h = nullptr;
    std::mutex mu;
    ~Device() { pcs_mls_index_destroy(h); }
};

SpatialIndex::SpatialIndex(const PointCloud& cloud, int leaf_size)
    : cloud_(&cloud), leaf_size_(leaf_size), dev_(std::make_shared<Device>()) {
    if (leaf_size_ < 1) throw InvalidParam("SpatialIndex leaf_size must be >= 1");
}

pcs_mls_index* SpatialIndex::device_index() const {
    std::lock_guard<std::mutex> lk(dev_->mu);
    if (!dev_->h) check(pcs_mls_index_create(xyz_of(*cloud_), cloud_->size(), -1, &dev_->h));
    return dev_->h;
}

void SpatialIndex::radius_query(Point3 center, double r, std::vector<Hit>& out) const {
    if (!(r > 0.0) || !std::isfinite(r)) throw InvalidParam("radius_query requires finite r > 0");
    out.clear();
    if (cloud_->empty()) return;
    uint64_t off[2] = {0, 0};
    pcs_mls_index* ix = device_index();
    check(pcs_mls_index_radius(ix, &center.x, 1, r, off, nullptr, nullptr, 0));
    std::vector<std::uint32_t> idx(off[1]);
    if (!idx.empty())
        check(pcs_mls_index_radius(ix, &center.x, 1, r, off, idx.data(), nullptr, idx.size()));
    std::sort(idx.begin(), idx.end());
    out.reserve(idx.size());
    for (std::uint32_t i : idx) out.push_back(Hit{i, std::sqrt(norm2((*cloud_)[i] - center))});
}

std::vector<SpatialIndex::Hit> SpatialIndex::radius_query(Point3 center, double r) const {
    std::vector<Hit> out;
    radius_query(center, r, out);
    return out;
}

SpatialIndex::Hit SpatialIndex::nearest(Point3 query) const {
    if (cloud_->empty()) throw EmptyCloud("nearest: index built over an empty cloud");
    pcs_lop_desc d;
    pcs_lop_desc_default(&d);
    std::uint32_t idx = 0;
    double dist = 0.0;
    check(pcs_nearest_all(&d, xyz_of(*cloud_), cloud_->size(), &query.x, 1, &idx, &dist));
    return Hit{idx, dist};
}

// ---- WLS fits -------------------------------------------------------------------

double evaluate_polynomial(const BivariatePolynomial& poly, double u, double v) {
    const int m = poly.degree;
    double upow[5] = {1.0, 0.0, 0.0, 0.0, 0.0};
    double vpow[5] = {1.0, 0.0, 0.0, 0.0, 0.0};
    for (int i = 1; i <= m; ++i) {
        upow[i] = upow[i - 1] * u;
        vpow[i] = vpow[i - 1] * v;
    }
    double sum = 0.0;
    std::size_t k = 0;
    for (int s = 0; s <= m; ++s)
        for (int a = s; a >= 0; --a) sum += poly.coefficients[k++] * upow[a] * vpow[s - a];
    return sum;
}

PlaneFitResult fit_reference_plane(const SpatialIndex& index, Point3 r, const KernelParams& kernel,
                                   double tol, int max_iter, const QueryCoverage* guard) {
    kernel.validate();
    if (!(tol > 0.0)) throw InvalidParam("fit_reference_plane: tol must be positive");
    if (max_iter < 1) throw InvalidParam("fit_reference_plane: max_iter must be >= 1");
    const pcs_mls_desc d = mls_desc(kernel, 2, tol, max_iter);
    pcs_mls_result R;
    std::vector<double> centers;
    if (guard) centers.resize((std::size_t)(max_iter + 1) * 3);
    check(pcs_mls_project(index.device_index(), &d, &r.x, 1, PCS_MLS_PLANE, nullptr, &R,
                          guard ? centers.data() : nullptr));
    PlaneFitResult res;
    if (guard) {  // covers(q) is asked at the top of every iteration (wls.cpp:76-80)
        for (int k = 0; k < R.iterations; ++k) {
            if (!guard->covers(p3(&centers[3 * (std::size_t)k]))) {
                res.status = PlaneFitStatus::OutOfCoverage;
                res.iterations = k + 1;
                return res;
            }
        }
    }
    res.iterations = R.iterations;
    res.status = plane_status_of(R.plane_status);
    if (res.status == PlaneFitStatus::Ok || res.status == PlaneFitStatus::NoConvergence) {
        res.frame.origin = p3(R.origin);
        res.frame.normal = p3(R.normal);
        res.frame.u = p3(R.u);
        res.frame.v = p3(R.v);
    }
    return res;
}

PolyFitResult fit_local_polynomial(const SpatialIndex& index, const LocalFrame& frame,
                                   const KernelParams& kernel, int degree,
                                   const QueryCoverage* guard) {
    kernel.validate();
    if (degree < 1 || degree > 4)
        throw InvalidParam("fit_local_polynomial: degree must be in [1,4]");
    PolyFitResult result;
    if (guard && !guard->covers(frame.origin)) {
        result.status = PolyFitStatus::OutOfCoverage;
        return result;
    }
    const pcs_mls_desc d = mls_desc(kernel, degree, 1e-10, 50);
    const double fr[12] = {frame.origin.x, frame.origin.y, frame.origin.z, frame.normal.x,
                           frame.normal.y, frame.normal.z, frame.u.x,      frame.u.y,
                           frame.u.z,      frame.v.x,      frame.v.y,      frame.v.z};
    pcs_mls_result R;
    check(pcs_mls_project(index.device_index(), &d, &frame.origin.x, 1, PCS_MLS_POLY, fr, &R, nullptr));
    if (R.poly_status == 1) {
        result.status = PolyFitStatus::TooFewNeighbors;
    } else if (R.poly_status == 2) {
        result.status = PolyFitStatus::SingularSystem;
    } else {
        result.poly.degree = degree;
        result.poly.coefficients.assign(R.coeffs, R.coeffs + BivariatePolynomial::coefficient_count(degree));
    }
    return result;
}

// ---- MLS projection -------------------------------------------------------------

void SmoothingSummary::add(const ProjectionOutcome& outcome) {
    switch (outcome.status) {
        case ProjectionStatus::Full: ++full; break;
        case ProjectionStatus::DegradedDegree: ++degraded_degree; break;
        case ProjectionStatus::PlaneOnly: ++plane_only; break;
        case ProjectionStatus::Skipped: ++skipped; break;
    }
    if (outcome.plane_status == PlaneFitStatus::NoConvergence) ++plane_no_convergence;
    if (outcome.plane_status == PlaneFitStatus::DegenerateNeighborhood) ++degenerate_neighborhoods;
}

void SmoothingSummary::merge(const SmoothingSummary& other) {
    full += other.full;
    degraded_degree += other.degraded_degree;
    plane_only += other.plane_only;
    skipped += other.skipped;
    plane_no_convergence += other.plane_no_convergence;
    degenerate_neighborhoods += other.degenerate_neighborhoods;
    coverage_fallbacks += other.coverage_fallbacks;
}

std::optional<ProjectionOutcome> project_point_guarded(const SpatialIndex& index, Point3 r,
                                                       const MlsParams& params,
                                                       const QueryCoverage* guard) {
    params.validate();
    const pcs_mls_desc d = mls_desc(params.kernel, params.degree, params.plane_tol, params.plane_max_iter);
    pcs_mls_result R;
    std::vector<double> centers;
    if (guard) centers.resize((std::size_t)(params.plane_max_iter + 1) * 3);
    check(pcs_mls_project(index.device_index(), &d, &r.x, 1, PCS_MLS_PROJECT, nullptr, &R,
                          guard ? centers.data() : nullptr));
    if (guard) {
        // the plane iterates, then (plane usable) the frame origin of the first
        // polynomial fit (mls.cpp:37-58, wls.cpp:76-80, 156-160)
        for (int k = 0; k < R.iterations; ++k)
            if (!guard->covers(p3(&centers[3 * (std::size_t)k]))) return std::nullopt;
        if ((R.plane_status == 0 || R.plane_status == 3) &&
            !guard->covers(p3(&centers[3 * (std::size_t)R.iterations])))
            return std::nullopt;
    }
    return outcome_of(R);
}

ProjectionOutcome project_point(const SpatialIndex& index, Point3 r, const MlsParams& params) {
    return *project_point_guarded(index, r, params, nullptr);
}

std::pair<PointCloud, SmoothingSummary> smooth_cloud(const PointCloud& cloud,
                                                     const MlsParams& params) {
    params.validate();
    PointCloud out;
    SmoothingSummary summary;
    if (cloud.empty()) return {out, summary};
    // the summary needs only each point's outcome (SmoothingSummary::add)
    const pcs_mls_desc d = mls_desc(params.kernel, params.degree, params.plane_tol, params.plane_max_iter);
    std::vector<pcs_mls_outcome> oc(cloud.size());
    out.points.resize(cloud.size());
    check(pcs_mls_smooth_outcomes(&d, xyz_of(cloud), cloud.size(), &out.points[0].x, oc.data()));
    for (std::size_t i = 0; i < oc.size(); ++i) {
        ProjectionOutcome o;
        o.projected = out.points[i];
        o.status = projection_status_of(oc[i].status);
        o.degree_used = oc[i].degree_used;
        o.iterations_used = oc[i].iterations;
        o.plane_status = plane_status_of(oc[i].plane_status);
        summary.add(o);
    }
    return {out, summary};
}

// ---- slab decomposition (proj/src/parallel.cpp) -----------------------------------

std::pair<PartitionLayout, std::vector<WorkerCloud>> partition(const PointCloud& cloud,
                                                               std::size_t workers, double support) {
    std::vector<double> cuts(workers > 1 ? workers - 1 : 1);
    std::vector<std::uint32_t> worker_of(cloud.size());
    int32_t axis = 0;
    check(pcs_mls_partition(xyz_of(cloud), cloud.size(), workers, support, &axis, cuts.data(),
                            worker_of.data()));
    PartitionLayout layout;
    layout.axis = axis;
    layout.workers = workers;
    layout.border_width = support;
    layout.cuts.assign(cuts.begin(), cuts.begin() + (workers - 1));
    std::vector<WorkerCloud> parts(workers);
    for (std::size_t i = 0; i < cloud.size(); ++i) {  // ascending original index
        WorkerCloud& p = parts[worker_of[i]];
        p.original.push_back(static_cast<std::uint32_t>(i));
        p.points.push_back(cloud[i]);
    }
    return {layout, parts};
}

std::vector<WorkerCloud> exchange_borders(const PartitionLayout& layout,
                                          const std::vector<WorkerCloud>& parts) {
    const std::size_t w = layout.workers;
    if (parts.size() != w)
        throw InvalidParam("exchange_borders: parts/layout worker count mismatch");
    std::vector<WorkerCloud> halos(w);
    for (std::size_t u = 0; u < w; ++u) {
        const double band_lo = layout.lo(u) - layout.border_width;
        const double band_hi = layout.hi(u) + layout.border_width;
        std::vector<std::pair<std::uint32_t, Point3>> merged;
        for (std::size_t v = 0; v < w; ++v) {
            if (v == u) continue;
            const WorkerCloud& own = parts[v];
            for (std::size_t i = 0; i < own.points.size(); ++i) {
                const double c = axis_coord(own.points[i], layout.axis);
                if (c >= band_lo && c <= band_hi) merged.emplace_back(own.original[i], own.points[i]);
            }
        }
        std::sort(merged.begin(), merged.end(),
                  [](const auto& a, const auto& b) { return a.first < b.first; });
        halos[u].original.reserve(merged.size());
        halos[u].points.reserve(merged.size());
        for (const auto& [idx, p] : merged) {
            halos[u].original.push_back(idx);
            halos[u].points.push_back(p);
        }
    }
    return halos;
}

// One device launch projects every point against the full cloud.  A worker of
// the reference computes the same point against its own + halo points and gives
// the identical result while every query centre stays inside its slab (the
// reference's own bit-identity contract, parallel.hpp); a point whose centres
// leave the slab is what the reference recomputes on the full cloud — counted
// here from the device's bounds of the centres used (SlabCoverage::covers:
// lo <= c <= hi along the layout axis).
std::pair<PointCloud, SmoothingSummary> parallel_smooth(const PointCloud& cloud,
                                                        const MlsParams& params,
                                                        std::size_t workers) {
    params.validate();
    if (workers < 1) throw InvalidParam("parallel_smooth: workers must be >= 1");
    PointCloud out;
    SmoothingSummary summary;
    if (cloud.empty()) return {out, summary};
    const auto [layout, parts] = partition(cloud, workers, params.kernel.support());
    // the projections, each point's outcome and the bounds of the centres it used
    const pcs_mls_desc d = mls_desc(params.kernel, params.degree, params.plane_tol, params.plane_max_iter);
    std::vector<pcs_mls_outcome> oc(cloud.size());
    std::vector<double> bounds(cloud.size() * 6);
    out.points.resize(cloud.size());
    check(pcs_mls_smooth_bounds(&d, xyz_of(cloud), cloud.size(), &out.points[0].x, oc.data(),
                                bounds.data()));
    std::size_t escaped = 0;
    for (std::size_t u = 0; u < workers; ++u) {
        const double lo = layout.lo(u), hi = layout.hi(u);
        for (std::uint32_t i : parts[u].original) {
            const double cmin = bounds[6 * (std::size_t)i + layout.axis];
            const double cmax = bounds[6 * (std::size_t)i + 3 + layout.axis];
            if (!(cmin >= lo && cmax <= hi)) ++escaped;
            ProjectionOutcome o;
            o.projected = out.points[i];
            o.status = projection_status_of(oc[i].status);
            o.degree_used = oc[i].degree_used;
            o.iterations_used = oc[i].iterations;
            o.plane_status = plane_status_of(oc[i].plane_status);
            summary.add(o);
        }
    }
    summary.coverage_fallbacks = escaped;
    return {out, summary};
}

}  // namespace pcs
