// c_api.cpp — the extern "C" boundary (include/pcs_lop.h).
//
// Every entry point converts pcsb::Failure / std::exception into a pcs_status
// and a thread-local message (pcs_last_error), the C rendering of the
// reference's exception hierarchy (proj/include/pcs/errors.hpp:9-53).
#include <cstdlib>
#include <cstring>
#include <exception>
#include <new>
#include <string>

#include "../../include/pcs_lop.h"
#include "plan.cuh"
#include "io.h"
#include "dconv.h"
#include <functional>
#include <cstdio>

namespace {
thread_local std::string g_last_error;

template <typename F>
pcs_status guarded(F&& f) {
    try {
        g_last_error.clear();
        f();
        return PCS_OK;
    } catch (const pcsb::Failure& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "host allocation failed";
        return PCS_ERR_NUMERICAL;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return PCS_ERR_NUMERICAL;
    }
}

const pcs_lop_desc& checked(const pcs_lop_desc* d) {
    if (!d) throw pcsb::Failure(PCS_ERR_INVALID_PARAM, "null descriptor");
    if (d->struct_size != sizeof(pcs_lop_desc))
        throw pcsb::Failure(PCS_ERR_INVALID_PARAM,
                            "pcs_lop_desc.struct_size mismatch (initialise with pcs_lop_desc_default)");
    return *d;
}
}  // namespace

namespace {
pcs_status parse_guarded(pcs_parse_error* err, const std::function<void()>& f) {
    try {
        f();
        return PCS_OK;
    } catch (const pcsb::ParseFailure& e) {
        if (err) {
            err->line = e.line;
            std::snprintf(err->reason, sizeof(err->reason), "%s", e.reason.c_str());
        }
        return guarded([&] { throw pcsb::Failure(PCS_ERR_PARSE, e.reason); });
    } catch (...) {
        return guarded([&] { throw; });
    }
}
}  // namespace

extern "C" {

void pcs_lop_desc_default(pcs_lop_desc* d) {
    if (!d) return;
    std::memset(d, 0, sizeof(*d));
    d->struct_size = sizeof(pcs_lop_desc);
    // defaults of KernelParams / LopParams (kernels.hpp:13-14, lop.hpp:14-17)
    d->h = 1.0;
    d->cutoff_multiple = 3.0;
    d->mu = 0.4;
    d->iterations = 30;
    d->convergence_tol = 1e-7;
    d->eta_kind = PCS_ETA_INV_CUBE;
    d->density_weights = 0;
    d->precision = PCS_PREC_FP64;
    d->device = -1;
    d->lanes_per_point = 0;
}

const char* pcs_last_error(void) { return g_last_error.c_str(); }

int32_t pcs_lop_abi_version(void) { return PCS_LOP_ABI_VERSION; }

pcs_status pcs_lop_validate(const pcs_lop_desc* d) {
    return guarded([&] { pcsb::validate_desc(checked(d)); });
}

pcs_status pcs_lop_run(const pcs_lop_desc* d, const double* P_xyz, uint64_t n,
                       const double* X0_xyz, uint64_t m, double* X_out_xyz,
                       pcs_lop_summary* summary, uint32_t* isolated_out, uint64_t isolated_cap) {
    return guarded([&] {
        const pcs_lop_desc& desc = checked(d);
        // semantics order of proj/src/lop.cpp:13-20
        pcsb::validate_desc(desc);
        if (n == 0) throw pcsb::Failure(PCS_ERR_EMPTY_CLOUD, "lop_project: data cloud is empty");
        if (summary) std::memset(summary, 0, sizeof(*summary));
        if (m == 0) return;
        if (!P_xyz || !X0_xyz || !X_out_xyz)
            throw pcsb::Failure(PCS_ERR_INVALID_PARAM, "null point buffer");
        pcsb::Plan plan(desc);
        // one run: a captured CUDA graph would never be replayed
        plan.set_graphs(false);
        plan.upload(P_xyz, n, X0_xyz, m);
        plan.run(desc.iterations, true);
        plan.download(X_out_xyz, summary, isolated_out, isolated_cap);
    });
}

pcs_status pcs_lop_plan_create(const pcs_lop_desc* d, pcs_lop_plan** out) {
    return guarded([&] {
        if (!out) throw pcsb::Failure(PCS_ERR_INVALID_PARAM, "null plan pointer");
        *out = nullptr;
        auto* p = new pcsb::Plan(checked(d));
        *out = reinterpret_cast<pcs_lop_plan*>(p);
    });
}

void pcs_lop_plan_destroy(pcs_lop_plan* p) { delete reinterpret_cast<pcsb::Plan*>(p); }

#define PLAN(p)                                                                    \
    if (!(p)) throw pcsb::Failure(PCS_ERR_INVALID_PARAM, "null plan");             \
    auto& plan = *reinterpret_cast<pcsb::Plan*>(p)

pcs_status pcs_lop_plan_upload(pcs_lop_plan* p, const double* P_xyz, uint64_t n,
                               const double* X0_xyz, uint64_t m) {
    return guarded([&] {
        PLAN(p);
        plan.upload(P_xyz, n, X0_xyz, m);
    });
}

pcs_status pcs_nccl_unique_id(uint8_t id_out[128]);

pcs_status pcs_lop_plan_record_counts(pcs_lop_plan* p, int32_t enable) {
    return guarded([&] {
        PLAN(p);
        plan.record_counts(enable != 0);
    });
}

pcs_status pcs_lop_plan_query_counts(pcs_lop_plan* p, int32_t* counts4, uint8_t* ever_flags,
                                     uint64_t m) {
    return guarded([&] {
        PLAN(p);
        plan.query_counts(counts4, ever_flags, m);
    });
}

pcs_status pcs_trim_device_pool(int32_t device) {
    return guarded([&] { pcsb::trim_device_pool(pcsb::select_device(device)); });
}

pcs_status pcs_lop_plan_set_comm(pcs_lop_plan* p, const uint8_t id[128], int32_t nranks,
                                 int32_t rank) {
    return guarded([&] {
        PLAN(p);
        plan.set_comm(id, nranks, rank);
    });
}

pcs_status pcs_loopback_group_create(int32_t nranks, pcs_loopback_group** out) {
    return guarded([&] {
        if (!out) throw pcsb::Failure(PCS_ERR_INVALID_PARAM, "null output pointer");
        *out = reinterpret_cast<pcs_loopback_group*>(new pcsb::LoopbackGroup(nranks));
    });
}

void pcs_loopback_group_destroy(pcs_loopback_group* g) {
    delete reinterpret_cast<pcsb::LoopbackGroup*>(g);
}

pcs_status pcs_lop_plan_set_loopback(pcs_lop_plan* p, pcs_loopback_group* g, int32_t rank) {
    return guarded([&] {
        PLAN(p);
        plan.set_loopback(reinterpret_cast<pcsb::LoopbackGroup*>(g), rank);
    });
}

pcs_status pcs_lop_plan_reset(pcs_lop_plan* p) {
    return guarded([&] {
        PLAN(p);
        plan.reset();
    });
}

pcs_status pcs_lop_plan_run(pcs_lop_plan* p, int32_t sweeps, int32_t sync) {
    return guarded([&] {
        PLAN(p);
        plan.run(sweeps, sync != 0);
    });
}

pcs_status pcs_lop_plan_synchronize(pcs_lop_plan* p) {
    return guarded([&] {
        PLAN(p);
        plan.synchronize();
    });
}

pcs_status pcs_lop_plan_last_run_ms(pcs_lop_plan* p, double* ms) {
    return guarded([&] {
        PLAN(p);
        plan.synchronize();
        if (ms) *ms = plan.last_run_ms();
    });
}

pcs_status pcs_lop_plan_download(pcs_lop_plan* p, double* X_out_xyz, pcs_lop_summary* summary,
                                 uint32_t* isolated_out, uint64_t isolated_cap) {
    return guarded([&] {
        PLAN(p);
        plan.download(X_out_xyz, summary, isolated_out, isolated_cap);
    });
}

uint64_t pcs_lop_plan_launches(const pcs_lop_plan* p) {
    return p ? reinterpret_cast<const pcsb::Plan*>(p)->launches() : 0;
}

pcs_status pcs_lop_plan_set_positions(pcs_lop_plan* p, const double* X_xyz, uint64_t m) {
    return guarded([&] {
        if (!p) throw pcsb::Failure(PCS_ERR_INVALID_PARAM, "null plan");
        reinterpret_cast<pcsb::Plan*>(p)->set_positions(X_xyz, m);
    });
}

pcs_status pcs_lop_plan_set_graphs(pcs_lop_plan* p, int32_t enable) {
    return guarded([&] {
        if (!p) throw pcsb::Failure(PCS_ERR_INVALID_PARAM, "null plan");
        reinterpret_cast<pcsb::Plan*>(p)->set_graphs(enable != 0);
    });
}

uint64_t pcs_lop_plan_graph_launches(const pcs_lop_plan* p) {
    return p ? reinterpret_cast<const pcsb::Plan*>(p)->graph_launches() : 0;
}

pcs_status pcs_radius_query_all(const pcs_lop_desc* d, const double* C_xyz, uint64_t n,
                                const double* Q_xyz, uint64_t m, double r, uint64_t* offsets,
                                uint32_t* idx, uint64_t idx_cap) {
    return guarded([&] {
        if (!offsets) throw pcsb::Failure(PCS_ERR_INVALID_PARAM, "null offsets");
        pcsb::radius_query_all(checked(d), C_xyz, n, Q_xyz, m, r, offsets, idx, idx_cap);
    });
}

pcs_status pcs_density_weights(const pcs_lop_desc* d, const double* C_xyz, uint64_t n,
                               double* v_out) {
    return guarded([&] { pcsb::density_weights(checked(d), C_xyz, n, v_out); });
}

pcs_status pcs_grid_sort(const pcs_lop_desc* d, const double* C_xyz, uint64_t n, double support,
                         uint32_t* keys_out, uint32_t* order_out) {
    return guarded([&] {
        pcsb::grid_sort(checked(d), C_xyz, n, support, keys_out, order_out);
    });
}

pcs_status pcs_nearest_all(const pcs_lop_desc* d, const double* C_xyz, uint64_t n,
                           const double* Q_xyz, uint64_t m, uint32_t* idx_out, double* dist_out) {
    return guarded([&] { pcsb::nearest_all(checked(d), C_xyz, n, Q_xyz, m, idx_out, dist_out); });
}

pcs_status pcs_deviation(const pcs_lop_desc* d, const double* cloud_xyz, uint64_t m,
                         const double* ref_xyz, uint64_t n, pcs_deviation_report* report,
                         double* distances_out) {
    return guarded([&] {
        pcsb::deviation(checked(d), cloud_xyz, m, ref_xyz, n, report, distances_out);
    });
}

pcs_status pcs_deviation_to_mesh(const pcs_lop_desc* d, const double* cloud_xyz, uint64_t m,
                                 const double* tri_xyz, uint64_t ntri,
                                 pcs_deviation_report* report, double* distances_out) {
    return guarded([&] {
        pcsb::deviation_to_mesh(checked(d), cloud_xyz, m, tri_xyz, ntri, report, distances_out);
    });
}

// ---- MLS projection -----------------------------------------------------------
struct pcs_mls_index {
    pcsb::MlsIndex* ix;
};

namespace {
const pcs_mls_desc& checked_mls(const pcs_mls_desc* d) {
    if (!d) throw pcsb::Failure(PCS_ERR_INVALID_PARAM, "null descriptor");
    if (d->struct_size != sizeof(pcs_mls_desc))
        throw pcsb::Failure(PCS_ERR_INVALID_PARAM,
                            "pcs_mls_desc.struct_size mismatch (initialise with pcs_mls_desc_default)");
    return *d;
}
}  // namespace

void pcs_mls_desc_default(pcs_mls_desc* d) {
    if (!d) return;
    std::memset(d, 0, sizeof(*d));
    d->struct_size = sizeof(pcs_mls_desc);
    d->h = 1.0;
    d->cutoff_multiple = 3.0;
    d->degree = 2;
    d->plane_tol = 1e-10;
    d->plane_max_iter = 50;
    d->device = -1;
}

pcs_status pcs_mls_index_create(const double* xyz, uint64_t n, int32_t device, pcs_mls_index** out) {
    return guarded([&] {
        if (!out) throw pcsb::Failure(PCS_ERR_INVALID_PARAM, "null handle");
        *out = nullptr;
        pcsb::MlsIndex* ix = pcsb::mls_index_create(xyz, n, device);
        *out = new pcs_mls_index{ix};
    });
}

void pcs_mls_index_destroy(pcs_mls_index* index) {
    if (!index) return;
    pcsb::mls_index_destroy(index->ix);
    delete index;
}

pcs_status pcs_mls_index_radius(pcs_mls_index* index, const double* centers_xyz, uint64_t m,
                                double r, uint64_t* offsets, uint32_t* idx, double* dist,
                                uint64_t cap) {
    return guarded([&] {
        if (!index) throw pcsb::Failure(PCS_ERR_INVALID_PARAM, "null index");
        pcsb::mls_index_radius(index->ix, centers_xyz, m, r, offsets, idx, dist, cap);
    });
}

pcs_status pcs_mls_project(pcs_mls_index* index, const pcs_mls_desc* d, const double* q_xyz,
                           uint64_t m, int32_t mode, const double* frames, pcs_mls_result* out,
                           double* centers_out) {
    return guarded([&] {
        if (!index) throw pcsb::Failure(PCS_ERR_INVALID_PARAM, "null index");
        pcsb::mls_project(index->ix, checked_mls(d), q_xyz, m, mode, frames, out, centers_out);
    });
}

pcs_status pcs_mls_smooth(const pcs_mls_desc* d, const double* xyz, uint64_t n, double* out_xyz,
                          pcs_mls_result* results) {
    return guarded([&] { pcsb::mls_smooth(checked_mls(d), xyz, n, out_xyz, results); });
}

pcs_status pcs_mls_smooth_outcomes(const pcs_mls_desc* d, const double* xyz, uint64_t n,
                                   double* out_xyz, pcs_mls_outcome* outcomes) {
    return guarded([&] { pcsb::mls_smooth_outcomes(checked_mls(d), xyz, n, out_xyz, outcomes, nullptr); });
}

pcs_status pcs_mls_smooth_bounds(const pcs_mls_desc* d, const double* xyz, uint64_t n, double* out_xyz,
                                 pcs_mls_outcome* outcomes, double* center_bounds) {
    return guarded([&] {
        pcsb::mls_smooth_outcomes(checked_mls(d), xyz, n, out_xyz, outcomes, center_bounds);
    });
}

pcs_status pcs_mls_last_device_ms(double* plane_ms, double* poly_ms) {
    return guarded([&] {
        double v[2];
        pcsb::mls_last_device_ms(v);
        if (plane_ms) *plane_ms = v[0];
        if (poly_ms) *poly_ms = v[1];
    });
}

pcs_status pcs_mls_partition(const double* xyz, uint64_t n, uint64_t workers, double support,
                             int32_t* axis, double* cuts, uint32_t* worker_of) {
    return guarded([&] { pcsb::mls_partition(xyz, n, workers, support, axis, cuts, worker_of); });
}

pcs_status pcs_format_cloud(const pcs_lop_desc* d, const double* xyz, uint64_t n, int32_t format,
                            char* out, uint64_t cap, uint64_t* len) {
    return guarded([&] {
        const pcs_lop_desc& desc = checked(d);
        if (format != PCS_FMT_XYZ && format != PCS_FMT_PLY_ASCII)
            throw pcsb::Failure(PCS_ERR_INVALID_PARAM, "unknown cloud format");
        if (n && !xyz) throw pcsb::Failure(PCS_ERR_INVALID_PARAM, "null points");
        if (!len) throw pcsb::Failure(PCS_ERR_INVALID_PARAM, "null length");
        if (n) pcsb::select_device(desc.device);
        *len = pcsb::format_cloud(xyz, n, format, out, cap);
        if (!out || cap < *len) throw pcsb::Failure(PCS_ERR_CAPACITY, "output buffer too small");
    });
}


pcs_status pcs_parse_cloud(const pcs_lop_desc* d, const char* text, uint64_t len, int32_t format,
                           double* xyz_out, uint64_t cap, uint64_t* n_out, pcs_parse_error* err) {
    return parse_guarded(err, [&] {
        const pcs_lop_desc& desc = checked(d);
        if (format != PCS_FMT_XYZ && format != PCS_FMT_PLY_ASCII)
            throw pcsb::Failure(PCS_ERR_INVALID_PARAM, "unknown cloud format");
        if (len && !text) throw pcsb::Failure(PCS_ERR_INVALID_PARAM, "null text");
        if (!n_out) throw pcsb::Failure(PCS_ERR_INVALID_PARAM, "null count");
        if (len) pcsb::select_device(desc.device);
        pcsb::ParseDst dst;  // points go straight to the caller's buffer when they fit
        dst.ext = xyz_out;
        dst.cap = xyz_out ? cap : 0;
        const std::vector<double> xyz = pcsb::parse_cloud(text, len, format, &dst);
        if (dst.used) {
            *n_out = dst.n;
            return;
        }
        *n_out = xyz.size() / 3;
        if (!xyz_out || cap < *n_out) throw pcsb::Failure(PCS_ERR_CAPACITY, "output buffer too small");
        if (!xyz.empty()) std::memcpy(xyz_out, xyz.data(), xyz.size() * sizeof(double));
    });
}

pcs_status pcs_parse_mesh(const char* text, uint64_t len, double* tri_out, uint64_t cap,
                          uint64_t* ntri_out, pcs_parse_error* err) {
    return parse_guarded(err, [&] {
        if (len && !text) throw pcsb::Failure(PCS_ERR_INVALID_PARAM, "null text");
        if (!ntri_out) throw pcsb::Failure(PCS_ERR_INVALID_PARAM, "null count");
        const std::vector<double> tri = pcsb::parse_mesh(text, len);
        *ntri_out = tri.size() / 9;
        if (!tri_out || cap < *ntri_out) throw pcsb::Failure(PCS_ERR_CAPACITY, "output buffer too small");
        std::memcpy(tri_out, tri.data(), tri.size() * sizeof(double));
    });
}

pcs_status pcs_format_cloud_alloc(const pcs_lop_desc* d, const double* xyz, uint64_t n,
                                  int32_t format, char** out, uint64_t* len) {
    return guarded([&] {
        const pcs_lop_desc& desc = checked(d);
        if (format != PCS_FMT_XYZ && format != PCS_FMT_PLY_ASCII)
            throw pcsb::Failure(PCS_ERR_INVALID_PARAM, "unknown cloud format");
        if (n && !xyz) throw pcsb::Failure(PCS_ERR_INVALID_PARAM, "null points");
        if (!out || !len) throw pcsb::Failure(PCS_ERR_INVALID_PARAM, "null output");
        if (n) pcsb::select_device(desc.device);
        *len = pcsb::format_cloud_alloc(xyz, n, format, out);
    });
}

void pcs_free_buffer(void* p) { std::free(p); }

int32_t pcs_format_double(double v, char* out32) {
    char buf[40];
    const int n = pcsb::dconv::format(v, buf);
    if (out32) std::memcpy(out32, buf, (size_t)n);
    return n;
}

}  // extern "C"

#include "nccl_dl.h"

extern "C" pcs_status pcs_nccl_unique_id(uint8_t id_out[128]) {
    return guarded([&] {
        if (!id_out) throw pcsb::Failure(PCS_ERR_INVALID_PARAM, "null id buffer");
        std::string err;
        const pcsb::NcclApi* api = pcsb::nccl_api(&err);
        if (!api) throw pcsb::Failure(PCS_ERR_NCCL, err);
        ncclUniqueId uid;
        const ncclResult_t r = api->GetUniqueId(&uid);
        if (r != ncclSuccess) throw pcsb::Failure(PCS_ERR_NCCL, api->GetErrorString(r));
        std::memcpy(id_out, &uid, 128);
    });
}
