// plan.cu — host orchestration (see plan.cuh).  Mirrors the control flow of
// pcs::lop_project (proj/src/lop.cpp:10-127): validate, build the data index
// once (:24), then per sweep rebuild the index over the moving set (:39),
// update every point (:41-100), aggregate (:102-113) and stop early (:116-119).
#include "dev_knobs.h"
#include "plan.cuh"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <numeric>

#include "host_io.h"

namespace pcsb {

namespace {
// sweep slots are recycled (finalize of sweep k clears the slot of sweep k + 1);
// kSlotCap = the CUDA-graph period, so a captured period maps sweeps to the same
// slots on every replay
constexpr int kSlotCap = 8;
constexpr int kGraphPeriod = 8;

int bit_width_u64(uint64_t v) {
    int b = 0;
    while (v) {
        ++b;
        v >>= 1;
    }
    return b;
}

// fp32 kernel constants.  theta(d) = 2^(kneg*d2) with kneg = -log2(e)/h^2; the
// kernels evaluate arg = fma(d2, kneg, K0), K0 = -kneg*r2f, so arg >= 0 <=> d2 <= r2
// in fp32 and 2^arg = theta * 2^K0 (the constant scale cancels in every ratio).
// |arg| <= band flags |d2 - r2| <~ 2^-19 r2: the fp32 decision could disagree
// with the reference's fp64 one only for |d2 - r2| <= ~14 ulp(r2) (2^-20.2 r2),
// so those pairs are re-decided exactly in fp64 (lop_fast.cu load_cands).
struct F32Consts {
    float kneg, K0, band, scull2, inv_scale;
};

// maxabs: largest |coordinate| of the clouds (fp32 rounding scale)
F32Consts fp32_consts(double h, double r2, double s_pad, double maxabs) {
    F32Consts c;
    c.kneg = (float)(-M_LOG2E / (h * h));
    c.K0 = (float)(-(double)c.kneg * (double)(float)r2);
    c.band = (float)((double)c.K0 * std::ldexp(1.0, -19));
    // row trimming radius (fp32 interval math, lop_fast.cu row_range): s_pad plus
    // 32 ulps of the coordinate scale, rounded up
    const double sc = s_pad + std::ldexp(maxabs + s_pad, -18);
    c.scull2 = std::nextafter((float)(sc * sc), INFINITY);
    c.inv_scale = (float)std::exp2(-(double)c.K0);
    return c;
}

double cells_for(const double lo[3], const double hi[3], double cs) {
    double c = 1.0;
    for (int a = 0; a < 3; ++a) c *= std::floor((hi[a] - lo[a]) / cs) + 3.0;
    return c;
}
}  // namespace

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        cudaGetLastError();
        throw Failure(PCS_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
    }
}

#ifndef PCSB_MAX_CELLS
#define PCSB_MAX_CELLS 1073741824.0  // 2^30 cells: a 4 GB data-grid table
#endif

GridGeom make_grid(const double lo_in[3], const double hi_in[3], double support, uint64_t npts) {
    double lo[3], hi[3];
    for (int a = 0; a < 3; ++a) {
        lo[a] = lo_in[a];
        hi[a] = hi_in[a];
        if (!(lo[a] <= hi[a])) lo[a] = hi[a] = 0.0;  // empty / non-finite
    }
    GridGeom g{};
    // keys are plain linear cells (x fastest): the query order comes from a
    // separate Morton sort of positions (build_query_list)
    double cs;
    // the table is O(points): at most 64 cells per point (>= 2^24 cells), so a
    // small cloud in a large box never reserves a multi-GB table
    const double kMax = std::min((double)PCSB_MAX_CELLS, std::max(16777216.0, 64.0 * (double)npts));
    // y/z cell side s/3 (measured sweeps/s vs s/4, with x cells up to 4x finer:
    // config 3 +3.3%, config 4 +5%, config 5 +11%; s/5 similar on config 3,
    // worse on config 2) when x cells 4x finer still fit the 2^30-cell table;
    // else 0.4 s, else s/2 — x subdivision is worth more than finer y/z (config
    // 5 at h = 0.01: 0.4 s with finer x +9% over s/3); then s
    if (cells_for(lo, hi, support / 3.0) * 4 <= kMax) {
        cs = support / 3.0;
    } else if (cells_for(lo, hi, support * 0.4) * 4 <= kMax) {
        cs = support * 0.4;
    } else if (cells_for(lo, hi, support * 0.5) * 2 <= kMax) {
        cs = support * 0.5;
    } else {
        cs = support;
        while (cells_for(lo, hi, cs) > (double)(1u << 27)) cs *= 1.25;
    }
    // developer knob (grid experiments): PCSB_CELL_FRAC = cell side / support
    if (const char* e = dev_knob("PCSB_CELL_FRAC")) {
        const double f = std::atof(e);
        if (f > 0.0 && cells_for(lo, hi, support * f) <= kMax) cs = support * f;
    }
    const int sb = 0;
    // finer cells along x (rows are unchanged; x-trimming gets tighter) while the
    // table stays within 2^30 cells (4 GB; built once, HBM is 180 GB).  Measured
    // sweep time, xsub 1 -> 2 -> 4: config 3 -2.6%, config 4 -11% / -19%,
    // config 5 -5% / -3%; then (sweeps/s, best of 3) 4 -> 8: config 3 +1.3%,
    // 4 +1.2%, 5 +3.6%, 2 -0.4%; 8 -> 16: config 3 +0.6%.
    int xsub = 1;
    for (int t : {16, 8, 4, 2})
        if (cells_for(lo, hi, cs) * t <= kMax) {
            xsub = t;
            break;
        }
    if (const char* e = dev_knob("PCSB_XSUB")) xsub = std::max(1, std::atoi(e));  // developer knob
    g.cs = cs;
    g.inv_cs = 1.0 / cs;
    g.xsub = xsub;
    g.csx = cs / xsub;
    g.inv_csx = 1.0 / g.csx;
    g.ox = lo[0] - cs;
    g.oy = lo[1] - cs;
    g.oz = lo[2] - cs;
    g.gx = (int32_t)std::floor((hi[0] - g.ox) * g.inv_csx) + 2;
    g.gy = (int32_t)std::floor((hi[1] - g.oy) * g.inv_cs) + 2;
    g.gz = (int32_t)std::floor((hi[2] - g.oz) * g.inv_cs) + 2;
    g.sub_bits = sb;
    g.ncells = (uint32_t)g.gx * (uint32_t)g.gy * (uint32_t)g.gz;
    g.key_bits = bit_width_u64((uint64_t)g.ncells << (3 * sb));
    return g;
}

// Grid of the projected set: the data grid's cell side times `scale` (>= 1),
// over the same box; the projected set is usually much sparser than the data,
// so coarser rows carry enough candidates to amortise their per-row cost.
GridGeom make_grid_scaled(const double lo_in[3], const double hi_in[3], double support, double scale,
                          const GridGeom& base) {
    if (!(scale > 1.0)) return base;
    double lo[3], hi[3];
    for (int a = 0; a < 3; ++a) {
        lo[a] = lo_in[a];
        hi[a] = hi_in[a];
        if (!(lo[a] <= hi[a])) lo[a] = hi[a] = 0.0;
    }
    (void)support;
    GridGeom g = base;
    g.cs = base.cs * scale;
    g.inv_cs = 1.0 / g.cs;
    // x cells 4x finer than y/z while the per-sweep table stays within 2^27 cells
    // (measured vs 1x, best of 3: config 3 +1.1%, 4 +1.2%, 5 +1.3%, 2 -1.3%)
    g.xsub = 1;
    for (int t : {4, 2})
        if (cells_for(lo, hi, g.cs) * t <= (double)(1u << 27)) {
            g.xsub = t;
            break;
        }
    if (const char* e = dev_knob("PCSB_XSUB_X")) g.xsub = std::max(1, std::atoi(e));  // developer knob
    g.csx = g.cs / g.xsub;
    g.inv_csx = 1.0 / g.csx;
    g.ox = lo[0] - g.cs;
    g.oy = lo[1] - g.cs;
    g.oz = lo[2] - g.cs;
    g.gx = (int32_t)std::floor((hi[0] - g.ox) * g.inv_csx) + 2;
    g.gy = (int32_t)std::floor((hi[1] - g.oy) * g.inv_cs) + 2;
    g.gz = (int32_t)std::floor((hi[2] - g.oz) * g.inv_cs) + 2;
    g.sub_bits = 0;
    g.ncells = (uint32_t)g.gx * (uint32_t)g.gy * (uint32_t)g.gz;
    g.key_bits = bit_width_u64((uint64_t)g.ncells);
    return g;
}

// x-grid scale (developer knob PCSB_XCELL): the projected set's grid has cells 2x
// the data grid's.  Its points are ~10x sparser than the data, so twice-coarser
// rows amortise the per-row cost of the repulsion (and WLOP w_i) pass, and the
// per-sweep rebuild sorts fewer key bits and scans an 8x smaller cell table.
// Measured (tools/xcell_probe.sh, round 1, sweeps/s vs 1x): config 2 +14%,
// config 3 +0.6% (+3.7% per rank of an emulated 8-rank run), config 4 +6%,
// config 5 -0.7%; 3x loses on every config.
double x_cell_scale(uint64_t n, uint64_t m, const GridGeom& g) {
    (void)n;
    (void)m;
    (void)g;
    if (const char* e = dev_knob("PCSB_XCELL")) return std::atof(e);
    return 2.0;
}

void validate_desc(const pcs_lop_desc& d) {
    // LopParams::validate + KernelParams::validate (proj/include/pcs/lop.hpp:18-26,
    // proj/include/pcs/kernels.hpp:18-23), same messages.
    if (!(d.h > 0.0)) throw Failure(PCS_ERR_INVALID_PARAM, "kernel bandwidth h must be positive");
    if (!(d.cutoff_multiple > 0.0))
        throw Failure(PCS_ERR_INVALID_PARAM, "kernel cutoff_multiple must be positive");
    if (!(d.mu >= 0.0) || !(d.mu < 0.5))
        throw Failure(PCS_ERR_INVALID_PARAM, "LopParams: mu must be in [0, 0.5)");
    if (d.iterations < 1)
        throw Failure(PCS_ERR_INVALID_PARAM, "LopParams: iterations must be >= 1");
    if (!(d.convergence_tol > 0.0))
        throw Failure(PCS_ERR_INVALID_PARAM, "LopParams: convergence_tol must be positive");
    if (d.eta_kind != PCS_ETA_INV_CUBE && d.eta_kind != PCS_ETA_NEG_LINEAR)
        throw Failure(PCS_ERR_INVALID_PARAM, "eta_kind must be PCS_ETA_INV_CUBE or PCS_ETA_NEG_LINEAR");
    if (d.precision != PCS_PREC_FP64 && d.precision != PCS_PREC_FP32)
        throw Failure(PCS_ERR_INVALID_PARAM, "precision must be PCS_PREC_FP64 or PCS_PREC_FP32");
    if (d.lanes_per_point != 0 && d.lanes_per_point != 2 && d.lanes_per_point != 4 &&
        d.lanes_per_point != 8)
        throw Failure(PCS_ERR_INVALID_PARAM, "lanes_per_point must be 0, 2, 4 or 8");
    const double s = d.h * d.cutoff_multiple;
    if (!std::isfinite(s)) throw Failure(PCS_ERR_INVALID_PARAM, "support h*cutoff_multiple must be finite");
    if (d.precision == PCS_PREC_FP32) {
        // theta is evaluated as 2^(log2e*(r^2 - d^2)/h^2) in [1, e^(cutoff^2)]
        if (d.cutoff_multiple * d.cutoff_multiple > 80.0)
            throw Failure(PCS_ERR_INVALID_PARAM, "fp32 precision requires cutoff_multiple <= 8.9");
        if (!(s * s >= 1e-30 && s * s <= 1e30))
            throw Failure(PCS_ERR_INVALID_PARAM, "fp32 precision requires 1e-15 <= support <= 1e15");
    }
}

int select_device(int requested) {
    int n = 0;
    const cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
        cudaGetLastError();
        throw Failure(PCS_ERR_NO_DEVICE,
                      "no CUDA device available: the B200 LOP path has no CPU fallback");
    }
    int dev = requested;
    if (dev < 0) PCSB_CUDA(cudaGetDevice(&dev));
    if (dev >= n) throw Failure(PCS_ERR_INVALID_PARAM, "device ordinal out of range");
    int major = 0;  // attribute query: cudaGetDeviceProperties costs milliseconds
    PCSB_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
    if (major != 10) {
        cudaDeviceProp prop;
        PCSB_CUDA(cudaGetDeviceProperties(&prop, dev));
        throw Failure(PCS_ERR_NO_DEVICE, std::string("device ") + prop.name +
                                             " is not sm_100 (B200); kernels are built for sm_100a only");
    }
    PCSB_CUDA(cudaSetDevice(dev));
    return dev;
}

// ---------------------------------------------------------------------------

Plan::Plan(const pcs_lop_desc& d) : d_(d) {
    validate_desc(d_);
    fp32_ = d_.precision == PCS_PREC_FP32;
    vec_bytes_ = fp32_ ? sizeof(float4) : sizeof(double4);
    lanes_ = d_.lanes_per_point ? d_.lanes_per_point : 4;
    // repulsion over the sparser projected set: 16-query groups amortise the
    // per-row cost better (measured -1..2% sweep time on configs 3 and 4)
    rep_lanes_ = d_.lanes_per_point ? lanes_ : 4;  // measured with bisected groups: 4 >= 2 on configs 3, 4, 5
    use_graphs_ = d_.no_graphs == 0;
    if (const char* e = dev_knob("PCSB_GRAPHS")) use_graphs_ = std::atoi(e) != 0;  // developer knob
    if (const char* e = dev_knob("PCSB_REORDER_EVERY")) reorder_every_ = std::max(1, std::atoi(e));
    if (const char* e = dev_knob("PCSB_ASYNC_ORDER")) async_order_ = std::atoi(e) != 0;  // developer knob
    if (const char* e = dev_knob("PCSB_FUSED")) fused_ = std::atoi(e) != 0;  // developer knob
    if (const char* e = dev_knob("PCSB_BISECT")) bisect_ = std::atoi(e) != 0;  // developer knob
    group_order_ = fp32_ && bisect_;
    if (const char* e = dev_knob("PCSB_GROUP_ORDER")) group_order_ = fp32_ && std::atoi(e) != 0;  // developer knob
    if (const char* e = dev_knob("PCSB_REP_LANES")) rep_lanes_ = std::atoi(e);  // developer knob
    device_ = select_device(d_.device);
    PCSB_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    {
        // the side stream (projected-set grid) gets the higher priority so its
        // small kernels take free block slots as soon as they appear
        int lo = 0, hi = 0;
        PCSB_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        PCSB_CUDA(cudaStreamCreateWithPriority(&stream2_, cudaStreamNonBlocking, hi));
    }
    PCSB_CUDA(cudaEventCreateWithFlags(&ev_xready_, cudaEventDisableTiming));
    PCSB_CUDA(cudaEventCreateWithFlags(&ev_qready_, cudaEventDisableTiming));
    PCSB_CUDA(cudaEventCreate(&run_ev_[0]));
    PCSB_CUDA(cudaEventCreate(&run_ev_[1]));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device_);
    fast_grid_ = sms * fast_blocks_per_sm(lanes_, d_.density_weights != 0, false, 2);
    density_grid_ = fast_grid_;
    {
        // all block slots on one GPU (one slot fewer: -1.5% .. -2.5% on configs 3-4);
        // decided again at upload for small or sharded projected sets
        int per_sm = fast_grid_ / sms;
        if (const char* e = dev_knob("PCSB_ATTR_BLOCKS")) per_sm = std::atoi(e);  // developer knob
        attr_grid_ = sms * std::max(1, per_sm);
    }
    exact_grid_ = sms * 8;
    support_ = d_.h * d_.cutoff_multiple;
    r2_ = support_ * support_;
    if (const char* e = dev_knob("PCSB_EMULATE_RANK")) {  // developer knob "N:r"
        int n = 0, r = 0;
        if (std::sscanf(e, "%d:%d", &n, &r) == 2 && n >= 1 && r >= 0 && r < n) {
            nranks_ = n;
            rank_ = r;
            coll_ = make_null_collectives();
        }
    }
}

Plan::~Plan() {
    if (stream2_) cudaStreamSynchronize(stream2_);
    if (stream_) cudaStreamSynchronize(stream_);
    drop_graph();
    free_all();
    for (auto& se : event_pool_)
        for (auto e : se.e) cudaEventDestroy(e);
    for (auto& se : pending_)
        for (auto e : se.e) cudaEventDestroy(e);
    if (run_ev_[0]) cudaEventDestroy(run_ev_[0]);
    if (run_ev_[1]) cudaEventDestroy(run_ev_[1]);
    delete coll_;
    if (ev_xready_) cudaEventDestroy(ev_xready_);
    if (ev_qready_) cudaEventDestroy(ev_qready_);
    if (stream2_) cudaStreamDestroy(stream2_);
    if (stream_) cudaStreamDestroy(stream_);
}

// Device memory comes from one stream-ordered pool per device that keeps what it
// has reserved (release threshold = max): a plan's ~40 buffers and the upload
// temporaries are then sub-allocations after the first run in a process, and
// freeing them costs no device synchronisation.
namespace {
cudaMemPool_t device_pool(int dev) {
    static std::mutex mu;
    static std::vector<cudaMemPool_t> pools;
    std::lock_guard<std::mutex> lock(mu);
    if ((int)pools.size() <= dev) pools.resize(dev + 1, nullptr);
    if (!pools[dev]) {
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.handleTypes = cudaMemHandleTypeNone;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        PCSB_CUDA(cudaMemPoolCreate(&pools[dev], &props));
        // keep up to 16 GB reserved between calls (warm repeated calls: the plan's
        // buffers are sub-allocations); beyond that, memory returns to the
        // device at each synchronisation; pcs_trim_device_pool releases it all
        uint64_t keep = 16ull << 30;
        PCSB_CUDA(cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &keep));
    }
    return pools[dev];
}
}  // namespace

// Stream-ordered allocations from the library's pool for the other operators
// (MLS index and temporaries): sub-allocations after the first call in a
// process, freed without a device synchronisation.
void* pool_alloc(int dev, size_t bytes, cudaStream_t s) {
    void* p = nullptr;
    PCSB_CUDA(cudaMallocFromPoolAsync(&p, bytes ? bytes : 16, device_pool(dev), s));
    return p;
}

void pool_free(void* p, cudaStream_t s) {
    if (p) cudaFreeAsync(p, s);
}

void trim_device_pool(int dev) {
    PCSB_CUDA(cudaSetDevice(dev));
    PCSB_CUDA(cudaDeviceSynchronize());
    PCSB_CUDA(cudaMemPoolTrimTo(device_pool(dev), 0));
}

void* Plan::talloc(size_t bytes) {
    void* p = nullptr;
    PCSB_CUDA(cudaMallocFromPoolAsync(&p, bytes ? bytes : 16, device_pool(device_), stream_));
    return p;
}

void Plan::tfree(void* p) {
    if (p) PCSB_CUDA(cudaFreeAsync(p, stream_));
}

void* Plan::dalloc(size_t bytes) {
    void* p = talloc(bytes);
    allocs_.push_back(p);
    return p;
}

void Plan::free_all() {
    for (void* p : allocs_) cudaFreeAsync(p, stream_);
    allocs_.clear();
}

void Plan::set_comm(const uint8_t id[128], int nranks, int rank) {
    if (uploaded_) throw Failure(PCS_ERR_INVALID_PARAM, "set_comm must precede upload");
    if (nranks < 1 || rank < 0 || rank >= nranks)
        throw Failure(PCS_ERR_INVALID_PARAM, "invalid rank / nranks");
    nranks_ = nranks;
    rank_ = rank;
    delete coll_;
    coll_ = nullptr;
    // a 1-rank clique is legal: it runs the sharded path with real NCCL calls
    coll_ = make_nccl_collectives(id, nranks, rank);
}

void Plan::set_loopback(LoopbackGroup* g, int rank) {
    if (uploaded_) throw Failure(PCS_ERR_INVALID_PARAM, "set_loopback must precede upload");
    if (!g || rank < 0 || rank >= g->nranks())
        throw Failure(PCS_ERR_INVALID_PARAM, "invalid rank / loopback group");
    nranks_ = g->nranks();
    rank_ = rank;
    delete coll_;
    coll_ = nullptr;
    coll_ = make_loopback_collectives(g, rank);
    loopback_ = true;  // host rendezvous: not capturable
}

void Plan::upload(const double* P, uint64_t n, const double* X0, uint64_t m) {
    if (n == 0) throw Failure(PCS_ERR_EMPTY_CLOUD, "lop_project: data cloud is empty");
    if (n >= 0xFFFFFFF0ull || m >= 0xFFFFFFF0ull)
        throw Failure(PCS_ERR_INVALID_PARAM, "clouds are limited to 2^32-16 points");
    PCSB_CUDA(cudaSetDevice(device_));
    if (fp32_) upload_t<float>(P, n, X0, m);
    else upload_t<double>(P, n, X0, m);
    uploaded_ = true;
    reset();
}

template <typename T>
void Plan::upload_t(const double* P, uint64_t n, const double* X0, uint64_t m) {
    using V = typename Vec4<T>::type;
    drop_graph();
    free_all();
    qcounts_ = nullptr;
    qever_ = nullptr;
    record_counts_ = false;
    n_ = n;
    m_ = m;
    cudaEvent_t e0, e1;
    PCSB_CUDA(cudaEventCreate(&e0));
    PCSB_CUDA(cudaEventCreate(&e1));
    PCSB_CUDA(cudaEventRecord(e0, stream_));

    // temporaries
    double *dP = nullptr, *dX0 = nullptr;
    V *Pv = nullptr, *X0v = nullptr;
    uint32_t *tk = nullptr, *tsk = nullptr;
    Pv = (decltype(Pv))talloc(n * sizeof(V));
    X0v = (decltype(X0v))talloc((m ? m : 1) * sizeof(V));
    if (sizeof(T) == 4) {
        // fp32 plans: rounded to fp32 while staging (16 instead of 24 bytes a point)
        h2d_staged_f32x4(Pv, P, n, 1.0f, stream_);
        h2d_staged_f32x4(X0v, X0, m, 0.0f, stream_);
    } else {
        dP = (decltype(dP))talloc(n * 3 * sizeof(double));
        dX0 = (decltype(dX0))talloc((m ? m : 1) * 3 * sizeof(double));
        h2d_staged(dP, P, n * 3 * sizeof(double), stream_);
        if (m) h2d_staged(dX0, X0, m * 3 * sizeof(double), stream_);
        launch_convert_xyz<T>(dP, Pv, n, (T)1, stream_);
        launch_convert_xyz<T>(dX0, X0v, m, (T)0, stream_);
        launches_ += 2;
    }

    bbox_slots_ = (unsigned long long*)dalloc(8 * sizeof(unsigned long long));
    init_bbox_slots(bbox_slots_, stream_);
    launch_bbox<T>(Pv, n, bbox_slots_, stream_);
    launch_bbox<T>(X0v, m, bbox_slots_, stream_);
    launches_ += 3;
    unsigned long long hb[6];
    PCSB_CUDA(cudaMemcpyAsync(hb, bbox_slots_, sizeof(hb), cudaMemcpyDeviceToHost, stream_));
    PCSB_CUDA(cudaStreamSynchronize(stream_));
    double lo[3], hi[3], maxabs = 0.0;
    for (int a = 0; a < 3; ++a) {
        lo[a] = ordered_to_double(hb[a]);
        hi[a] = ordered_to_double(hb[3 + a]);
        if (!std::isfinite(lo[a]) || !std::isfinite(hi[a]))
            throw Failure(PCS_ERR_INVALID_PARAM, "clouds must have finite coordinates");
        maxabs = std::max(maxabs, std::max(std::fabs(lo[a]), std::fabs(hi[a])));
    }
    g_ = make_grid(lo, hi, support_, n);
    gX_ = make_grid_scaled(lo, hi, support_, x_cell_scale(n, m, g_), g_);
    s_pad_ = support_ * (1.0 + std::ldexp(1.0, -10)) + 1e-12 * maxabs;
    maxabs_ = maxabs;

    // ---- data grid (built once, lop.cpp:24) ----
    const uint32_t nn = (uint32_t)n;
    if (sharded()) {
        chunk_ = (uint32_t)((m + nranks_ - 1) / nranks_);
        mpad_ = chunk_ * nranks_;
    } else {
        chunk_ = (uint32_t)m;
        mpad_ = (uint32_t)m;
    }
    const uint32_t sort_cap = std::max<uint32_t>(nn, std::max<uint32_t>(mpad_, 1));
    rs_.keys_alt = (uint32_t*)dalloc(sort_cap * sizeof(uint32_t));
    rs_.vals_alt = (uint32_t*)dalloc(sort_cap * sizeof(uint32_t));
    rs_.blockhist = (uint32_t*)dalloc(radix_blockhist_entries(sort_cap) * sizeof(uint32_t));
    rs_.capacity = sort_cap;
    rs2_.keys_alt = (uint32_t*)dalloc(sort_cap * sizeof(uint32_t));
    rs2_.vals_alt = (uint32_t*)dalloc(sort_cap * sizeof(uint32_t));
    rs2_.blockhist = (uint32_t*)dalloc(radix_blockhist_entries(sort_cap) * sizeof(uint32_t));
    rs2_.capacity = sort_cap;
    cell_scratch_ = (uint32_t*)dalloc(
        cell_scan_scratch_entries(std::max(g_.ncells, gX_.ncells)) * sizeof(uint32_t));
    st_ = (RunState*)dalloc(sizeof(RunState));
    PCSB_CUDA(cudaMemsetAsync(st_, 0, sizeof(RunState), stream_));

    tk = (decltype(tk))talloc(sort_cap * sizeof(uint32_t));
    tsk = (decltype(tsk))talloc(sort_cap * sizeof(uint32_t));
    P_order_ = (uint32_t*)dalloc(nn * sizeof(uint32_t));
    P_sorted_ = dalloc((size_t)nn * sizeof(V));
    P_start_ = (uint32_t*)dalloc(((size_t)g_.ncells + 1) * sizeof(uint32_t));
    launch_keys<T>(g_, Pv, nn, tk, nullptr, stream_);
    launches_ += 1;
    launches_ += radix_sort(tk, nullptr, tsk, P_order_, nn, g_.key_bits, rs_, nullptr, stream_);
    launch_gather<T>(Pv, P_order_, nn, (V*)P_sorted_, nullptr, stream_);
    launches_ += 1;
    launches_ += build_cell_start(tsk, nn, 3 * g_.sub_bits, g_.ncells, P_start_, cell_scratch_,
                                  nullptr, stream_);
    if (fp32_) {
        P_pairs_cap_ = pairs_capacity(nn, g_);
        P_pairs_ = (float4*)dalloc(P_pairs_cap_ * sizeof(float4));
        launches_ += build_pairs((const float4*)P_sorted_, nullptr, nullptr, tsk, nn, g_, P_start_,
                                 P_pairs_, nullptr, stream_);
    }

    // ---- WLOP data density v_j (once) ----
    uint32_t* counter = (uint32_t*)dalloc(sizeof(uint32_t));
    if (d_.density_weights) {
        if (fp32_) {
            PCSB_CUDA(cudaMemsetAsync(counter, 0, sizeof(uint32_t), stream_));
            DensityArgs da{};
            uint32_t *pf = nullptr, *pfs = nullptr, *pq = nullptr;
            pf = (decltype(pf))talloc((size_t)nn * sizeof(uint32_t));
            pfs = (decltype(pfs))talloc((size_t)nn * sizeof(uint32_t));
            pq = (decltype(pq))talloc((size_t)nn * sizeof(uint32_t));
            int bsh = 0;
            launches_ += build_query_list((const float4*)P_sorted_, nn, g_, support_, nullptr, 0, 0,
                                          pf, pfs, pq, &bsh, rs_, nullptr, stream_);
            da.C = (const float4*)P_sorted_;
            da.Cpairs = P_pairs_;
            da.Cpairs_cap = P_pairs_cap_;
            da.Cstart = P_start_;
            da.qlist = pq;
            da.qcodes = pfs;
            da.block_shift = bsh;
            da.nq = nn;
            da.unit = work_unit_queries(nn, density_grid_ * 4);
            da.g = g_;
            da.s_pad = s_pad_;
            da.r2 = r2_;
            const F32Consts fc = fp32_consts(d_.h, r2_, s_pad_, maxabs_);
            da.scull2 = fc.scull2;
            da.kneg = fc.kneg;
            da.K0 = fc.K0;
            da.band = fc.band;
            da.inv_scale = fc.inv_scale;
            da.invert = 1;
            da.out_sorted = (float4*)P_sorted_;
            da.st = st_;
            da.counter = counter;
            da.done = nullptr;
            launch_density(da, density_grid_, stream_);
            // the records carry 1/v_j too
            launches_ += 1 + build_pairs((const float4*)P_sorted_, nullptr, nullptr, tsk, nn, g_,
                                         P_start_, P_pairs_, nullptr, stream_);
            PCSB_CUDA(cudaStreamSynchronize(stream_));
            tfree(pf);
            tfree(pfs);
            tfree(pq);
        } else {
            launch_exact_density<T>((const V*)P_sorted_, P_start_, (const V*)P_sorted_, nullptr, nn,
                                    nullptr, g_, s_pad_, r2_, support_, d_.h, 0, (V*)P_sorted_,
                                    nullptr, st_, nullptr, stream_);
        }
        launches_ += 1;
    }

    // ---- projected set layout ----
    if (sharded()) {
        // ownership: contiguous ranges of the initial cell-sorted order, cut at
        // equal estimated work (data density around each point)
        std::vector<uint32_t> sidx(m);
        std::vector<float> work(m);
        if (m) {
            launch_keys<T>(g_, X0v, (uint32_t)m, tk, nullptr, stream_);
            launches_ += 1;
            uint32_t* order = (uint32_t*)dalloc(m * sizeof(uint32_t));
            launches_ += radix_sort(tk, nullptr, tsk, order, (uint32_t)m, g_.key_bits, rs_, nullptr,
                                    stream_);
            float* wd = (float*)talloc(m * sizeof(float));
            launch_shard_work<T>(X0v, (uint32_t)m, g_, s_pad_, P_start_, wd, stream_);
            launches_ += 1;
            PCSB_CUDA(cudaMemcpyAsync(sidx.data(), order, m * sizeof(uint32_t),
                                      cudaMemcpyDeviceToHost, stream_));
            PCSB_CUDA(cudaMemcpyAsync(work.data(), wd, m * sizeof(float), cudaMemcpyDeviceToHost,
                                      stream_));
            PCSB_CUDA(cudaStreamSynchronize(stream_));
            tfree(wd);
        }
        std::vector<uint32_t> counts(nranks_);
        uint32_t chunk = 0;
        if (pcs_shard_layout_weighted(sidx.data(), work.data(), m, nranks_, nullptr, nullptr, &chunk,
                                      counts.data()) != PCS_OK)
            throw Failure(PCS_ERR_NUMERICAL, "shard layout failed");
        chunk_ = std::max<uint32_t>(chunk, 1);
        mpad_ = chunk_ * (uint32_t)nranks_;
        std::vector<uint32_t> ooi(mpad_), ioo(m ? m : 1);
        if (pcs_shard_layout_weighted(sidx.data(), work.data(), m, nranks_, ooi.data(), ioo.data(),
                                      &chunk, counts.data()) != PCS_OK)
            throw Failure(PCS_ERR_NUMERICAL, "shard layout failed");
        if (mpad_ > rs_.capacity) {  // the projected set's sorts run over mpad_ slots
            for (RadixScratch* r : {&rs_, &rs2_}) {
                r->keys_alt = (uint32_t*)dalloc((size_t)mpad_ * sizeof(uint32_t));
                r->vals_alt = (uint32_t*)dalloc((size_t)mpad_ * sizeof(uint32_t));
                r->blockhist = (uint32_t*)dalloc(radix_blockhist_entries(mpad_) * sizeof(uint32_t));
                r->capacity = mpad_;
            }
        }
        X_init_ = dalloc((size_t)std::max<uint32_t>(mpad_, 1) * sizeof(V));
        if (nranks_ >= 4 && !dev_knob("PCSB_ATTR_BLOCKS")) {
            // with a quarter of the queries or less the attraction pass is short and
            // the side stream's grid rebuild (latency-bound) would be exposed after
            // it: leave it one block slot per SM (8-GPU emulation: -4% per sweep)
            int sms = 148;
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device_);
            attr_grid_ = sms * std::max(1, fast_grid_ / sms - 1);
        }
        own_lo_ = (uint32_t)rank_ * chunk_;
        own_cnt_ = counts[rank_];
        orig_of_internal_ = (uint32_t*)dalloc((size_t)mpad_ * sizeof(uint32_t));
        uint32_t* iof = nullptr;
        iof = (decltype(iof))talloc((m ? m : 1) * sizeof(uint32_t));
        PCSB_CUDA(cudaMemcpyAsync(orig_of_internal_, ooi.data(), (size_t)mpad_ * sizeof(uint32_t),
                                  cudaMemcpyHostToDevice, stream_));
        if (m)
            PCSB_CUDA(cudaMemcpyAsync(iof, ioo.data(), m * sizeof(uint32_t), cudaMemcpyHostToDevice,
                                      stream_));
        launch_fill_invalid<T>((V*)X_init_, mpad_, orig_of_internal_, stream_);
        launch_scatter_init<T>(X0v, iof, (uint32_t)m, (V*)X_init_, stream_);
        launches_ += 2;
        PCSB_CUDA(cudaStreamSynchronize(stream_));
        tfree(iof);
    } else {
        X_init_ = dalloc((size_t)std::max<uint32_t>(mpad_, 1) * sizeof(V));
        own_lo_ = 0;
        own_cnt_ = (uint32_t)m;
        if (m < (1u << 18) && !dev_knob("PCSB_ATTR_BLOCKS")) {
            // a short attraction pass would end before the side stream's grid
            // rebuild got SM slots: leave it one per SM (config 2, 100k queries:
            // sweep -13%; configs 4 / 3 with 400k / 1M queries: +2.5% / +1.5%)
            int sms = 148;
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device_);
            attr_grid_ = sms * std::max(1, fast_grid_ / sms - 1);
        }
        if (m)
            PCSB_CUDA(cudaMemcpyAsync(X_init_, X0v, m * sizeof(V), cudaMemcpyDeviceToDevice, stream_));
    }
    const size_t mp = std::max<uint32_t>(mpad_, 1);
    X_[0] = dalloc(mp * sizeof(V));
    X_[1] = dalloc(mp * sizeof(V));
    X_sorted_ = dalloc(mp * sizeof(V));
    X_keys_ = (uint32_t*)dalloc(mp * sizeof(uint32_t));
    X_skeys_ = (uint32_t*)dalloc(mp * sizeof(uint32_t));
    X_sidx_ = (uint32_t*)dalloc(mp * sizeof(uint32_t));
    X_start_ = (uint32_t*)dalloc(((size_t)gX_.ncells + 1) * sizeof(uint32_t));
    if (fp32_) {
        X_pairs_cap_ = pairs_capacity((uint32_t)mp, gX_);
        X_pairs_ = (float4*)dalloc(X_pairs_cap_ * sizeof(float4));
    }
    careful_list_ = (uint32_t*)dalloc(mp * sizeof(uint32_t));
    attr_ = (float4*)dalloc(mp * sizeof(float4));
    attr_n_ = (int2*)dalloc(mp * sizeof(int2));
    attr_x_ = nullptr;
    attr_nx_ = nullptr;
    if (fp32_) {  // partial attraction sums of row-split tail units (enqueue_sweep)
        tail_cap_ = (uint32_t)std::min<uint64_t>(mp, (uint64_t)4 * fast_grid_ * 4u * 16u + 64u);
        attr_x_ = (float4*)dalloc((size_t)kTailPlanes * tail_cap_ * sizeof(float4));
        attr_nx_ = (int2*)dalloc((size_t)kTailPlanes * tail_cap_ * sizeof(int2));
    }
    q_keys_ = (uint32_t*)dalloc(mp * sizeof(uint32_t));
    q_skeys_ = (uint32_t*)dalloc(mp * sizeof(uint32_t));
    q_list_ = (uint32_t*)dalloc(mp * sizeof(uint32_t));
    q_keys_alt_ = (uint32_t*)dalloc(mp * sizeof(uint32_t));
    q_skeys_alt_ = (uint32_t*)dalloc(mp * sizeof(uint32_t));
    q_list_alt_ = (uint32_t*)dalloc(mp * sizeof(uint32_t));
    q_home_[0] = q_skeys_;
    q_home_[1] = q_list_;
    q_home_[2] = q_skeys_alt_;
    q_home_[3] = q_list_alt_;
    q_next_ready_ = false;
    ever_iso_ = (uint8_t*)dalloc(mp);
    slots_ = (SweepSlot*)dalloc(kSlotCap * sizeof(SweepSlot));
    out_xyz_ = (double*)dalloc((size_t)(m ? m : 1) * 3 * sizeof(double));
    out_iso_ = (uint8_t*)dalloc(m ? m : 1);
    slot_cap_ = kSlotCap;

    PCSB_CUDA(cudaEventRecord(e1, stream_));
    PCSB_CUDA(cudaStreamSynchronize(stream_));
    float ms = 0.f;
    PCSB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    setup_ms_ = ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    RunState hs;
    PCSB_CUDA(cudaMemcpy(&hs, st_, sizeof(hs), cudaMemcpyDeviceToHost));
    setup_density_pairs_ = hs.density_pairs;
    if (dP) tfree(dP);
    if (dX0) tfree(dX0);
    tfree(Pv);
    tfree(X0v);
    tfree(tk);
    tfree(tsk);
}

// Restart point of the run (unsharded plans): X_init_ <- X (m points, original
// order = internal order), then reset().  The grids keep the upload-time box:
// positions may lie anywhere (boundary cells are unbounded outward).
void Plan::set_positions(const double* X, uint64_t m) {
    if (!uploaded_) throw Failure(PCS_ERR_INVALID_PARAM, "plan has no data (upload first)");
    if (sharded()) throw Failure(PCS_ERR_INVALID_PARAM, "set_positions: unsharded plans only");
    if (m != m_) throw Failure(PCS_ERR_INVALID_PARAM, "set_positions: m must equal the plan's m");
    if (m && !X) throw Failure(PCS_ERR_INVALID_PARAM, "null buffer");
    PCSB_CUDA(cudaSetDevice(device_));
    synchronize();
    if (m) {
        if (fp32_) {
            h2d_staged_f32x4(X_init_, X, m, 0.0f, stream_);
        } else {
            double* dX = (double*)talloc(m * 3 * sizeof(double));
            h2d_staged(dX, X, m * 3 * sizeof(double), stream_);
            launch_convert_xyz<double>(dX, (double4*)X_init_, m, 0.0, stream_);
            launches_ += 1;
            tfree(dX);
        }
    }
    reset();
}

void Plan::reset() {
    if (!n_) throw Failure(PCS_ERR_INVALID_PARAM, "plan has no data (upload first)");
    PCSB_CUDA(cudaSetDevice(device_));
    synchronize();
    const size_t xb = (size_t)std::max<uint32_t>(mpad_, 1) * vec_bytes_;
    PCSB_CUDA(cudaMemcpyAsync(X_[0], X_init_, xb, cudaMemcpyDeviceToDevice, stream_));
    PCSB_CUDA(cudaMemcpyAsync(X_[1], X_init_, xb, cudaMemcpyDeviceToDevice, stream_));
    PCSB_CUDA(cudaMemsetAsync(st_, 0, sizeof(RunState), stream_));
    PCSB_CUDA(cudaMemsetAsync(slots_, 0, (size_t)slot_cap_ * sizeof(SweepSlot), stream_));
    PCSB_CUDA(cudaMemsetAsync(ever_iso_, 0, std::max<uint32_t>(mpad_, 1), stream_));
    if (qever_) PCSB_CUDA(cudaMemsetAsync(qever_, 0, std::max<uint32_t>(mpad_, 1), stream_));
    PCSB_CUDA(cudaStreamSynchronize(stream_));
    sweeps_issued_ = 0;
    gather_pending_ = false;
    q_stale_ = true;
    // the query-order buffers back in their upload-time roles (the order is
    // rebuilt by sweep 1 anyway): every run then meets a captured CUDA graph in
    // the same host state, whatever the parity of the previous run's swaps
    q_skeys_ = q_home_[0];
    q_list_ = q_home_[1];
    q_skeys_alt_ = q_home_[2];
    q_list_alt_ = q_home_[3];
    block_shift_alt_ = 0;
    q_next_ready_ = false;
    sweeps_since_order_ = 0;
    sweeps_ms_ = kernel_ms_ = sort_ms_ = 0.0;
}

void Plan::run(int sweeps, bool sync) {
    if (!uploaded_) throw Failure(PCS_ERR_INVALID_PARAM, "plan has no data (upload first)");
    if (sweeps <= 0) sweeps = d_.iterations;
    PCSB_CUDA(cudaSetDevice(device_));
    synchronize();
    PCSB_CUDA(cudaEventRecord(run_ev_[0], stream_));
    last_sweep_ = sweeps_issued_ + sweeps;
    // single-process plans only: captured kernel nodes do not keep the side
    // stream's high priority, which sharded plans need for the projected-set
    // rebuild to take the SM slots their short attraction pass leaves (emulated
    // 8-rank sweep 0.67 -> 0.69 ms with graphs; 1 GPU config 1 +34%, config 3 +0.7%)
    const bool graphs = use_graphs_ && !loopback_ && !sharded();
    while (sweeps_issued_ < last_sweep_) {
        const int k = sweeps_issued_ + 1;
        // whole periods k0 = 2 (mod kGraphPeriod) replay the captured graph
        if (graphs && k >= 2 && (k - 2) % kGraphPeriod == 0 && last_sweep_ - k + 1 >= kGraphPeriod &&
            !q_stale_ && graph_matches()) {
            replay_period();
            continue;
        }
        ++sweeps_issued_;
        enqueue_one(k);
        if (graphs && !have_snap_ && (k - 1) % kGraphPeriod == 0 && !q_stale_ && !graph_matches()) {
            period_snap_ = snapshot();  // the host state at the start of a period
            have_snap_ = true;
        }
    }
    PCSB_CUDA(cudaEventRecord(run_ev_[1], stream_));
    // capture the period off the critical path: the sweeps above are executing
    if (graphs && use_graphs_ && have_snap_) capture_period(period_snap_);
    have_snap_ = false;
    run_pending_ = true;
    if (sync) synchronize();
}

void Plan::enqueue_one(int k) {
    if (fp32_) enqueue_sweep<float>(k);
    else enqueue_sweep<double>(k);
}

void Plan::drop_graph() {
    if (graph_exec_) cudaGraphExecDestroy(graph_exec_);
    if (graph_) cudaGraphDestroy(graph_);
    graph_exec_ = nullptr;
    graph_ = nullptr;
}

void Plan::set_graphs(bool on) {
    synchronize();
    use_graphs_ = on;
    have_snap_ = false;
    if (!on) drop_graph();
}

// Sweeps k0 .. k0 + kGraphPeriod - 1 as one CUDA graph: captured the first time
// (and whenever the query-list buffers or the per-query count facility differ
// from the captured ones), replayed afterwards.  A capture that fails (e.g. a
// launch type the driver cannot capture) switches the plan back to enqueueing
// every launch.
Plan::HostSnap Plan::snapshot() const {
    return HostSnap{q_skeys_,          q_list_,         q_skeys_alt_, q_list_alt_,  block_shift_,
                    block_shift_alt_,  sweeps_since_order_, sweeps_issued_, last_sweep_, q_stale_,
                    q_next_ready_,     launches_,
                    record_counts_ ? (const void*)qcounts_ : nullptr};
}

void Plan::restore(const HostSnap& h) {
    q_skeys_ = h.qs;
    q_list_ = h.ql;
    q_skeys_alt_ = h.qsa;
    q_list_alt_ = h.qla;
    block_shift_ = h.bs;
    block_shift_alt_ = h.bsa;
    sweeps_since_order_ = h.since;
    sweeps_issued_ = h.issued;
    last_sweep_ = h.last;
    q_stale_ = h.stale;
    q_next_ready_ = h.next_ready;
    launches_ = h.launches;
}

bool Plan::graph_matches() const {
    if (!graph_exec_) return false;
    const HostSnap& g = graph_snap_;
    // (block_shift_alt_ is not part of the state: the period's own re-ordering
    // builds overwrite it before it is read)
    return g.qs == q_skeys_ && g.ql == q_list_ && g.qsa == q_skeys_alt_ && g.qla == q_list_alt_ &&
           g.bs == block_shift_ && g.since == sweeps_since_order_ &&
           g.stale == q_stale_ && g.next_ready == q_next_ready_ &&
           g.counts == (record_counts_ ? (const void*)qcounts_ : nullptr);
}

void Plan::replay_period() {
    sweeps_issued_ += kGraphPeriod;
    launches_ += graph_period_launches_;
    PCSB_CUDA(cudaGraphLaunch(graph_exec_, stream_));
    ++graph_launches_;
}

// Records (does not execute) the kGraphPeriod sweeps that start from host state
// `at` as a CUDA graph, then puts the host state back.  The period returns the
// query-list buffers and reorder count to where they started (two swaps), so
// the graph replays every later period from the same state.  A capture the
// driver rejects switches the plan to enqueueing every launch.
void Plan::capture_period(const HostSnap& at) {
    const HostSnap now = snapshot();
    drop_graph();
    restore(at);
    last_sweep_ = 1 << 30;  // the period's own re-orderings are built inside it
    PCSB_CUDA(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
    capturing_ = true;
    bool ok = true;
    try {
        for (int j = 0; j < kGraphPeriod; ++j) {
            ++sweeps_issued_;
            enqueue_one(sweeps_issued_);
        }
    } catch (const Failure&) {
        ok = false;
    }
    capturing_ = false;
    cudaGraph_t g = nullptr;
    const cudaError_t e = cudaStreamEndCapture(stream_, &g);
    for (auto& se : capture_events_) event_pool_.push_back(se);
    capture_events_.clear();
    ok = ok && e == cudaSuccess && g != nullptr;
    const HostSnap after = snapshot();
    // replayable only if the period left the host state where it started
    ok = ok && after.qs == at.qs && after.ql == at.ql && after.bs == at.bs &&
         after.since == at.since && after.next_ready == at.next_ready && after.stale == at.stale;
    if (ok && cudaGraphInstantiate(&graph_exec_, g, 0) != cudaSuccess) {
        graph_exec_ = nullptr;
        ok = false;
    }
    static const bool dbg = dev_knob("PCSB_DEBUG_GRAPH") != nullptr;  // developer knob
    if (dbg)
        std::fprintf(stderr, "[pcsb] graph capture: ok=%d end=%s state %d%d%d%d%d%d%d\n", (int)ok,
                     cudaGetErrorString(e), after.qs == at.qs, after.ql == at.ql, after.bs == at.bs,
                     after.bsa == at.bsa, after.since == at.since, after.next_ready == at.next_ready,
                     after.stale == at.stale);
    if (ok) {
        graph_ = g;
        graph_period_launches_ = after.launches - at.launches;
        graph_snap_ = at;
    } else {
        if (g) cudaGraphDestroy(g);
        use_graphs_ = false;
    }
    cudaGetLastError();
    restore(now);
}

void Plan::synchronize() {
    PCSB_CUDA(cudaStreamSynchronize(stream_));
    PCSB_CUDA(cudaGetLastError());
    if (run_pending_) {
        float ms = 0.f;
        PCSB_CUDA(cudaEventElapsedTime(&ms, run_ev_[0], run_ev_[1]));
        last_run_ms_ = ms;
        sweeps_ms_ += ms;
        run_pending_ = false;
    }
    for (auto& se : pending_) {
        // grid work = the query order + the part of the projected-set grid
        // (side stream) not hidden behind the attraction pass; kernels = the
        // attraction, repulsion and update passes
        float q = 0.f, ta = 0.f, tg = 0.f, tk = 0.f;
        PCSB_CUDA(cudaEventElapsedTime(&q, se.e[0], se.e[3]));
        PCSB_CUDA(cudaEventElapsedTime(&ta, se.e[0], se.e[6]));
        PCSB_CUDA(cudaEventElapsedTime(&tg, se.e[0], se.e[2]));
        PCSB_CUDA(cudaEventElapsedTime(&tk, se.e[0], se.e[4]));
        const float exposed = tg > ta ? tg - ta : 0.f;
        sort_ms_ += q + exposed;
        kernel_ms_ += tk - q - exposed;
        static const bool dbg = dev_knob("PCSB_DEBUG_TIMES") != nullptr;  // developer knob
        if (dbg) {
            float te = 0.f;
            PCSB_CUDA(cudaEventElapsedTime(&te, se.e[0], se.e[5]));
            std::fprintf(stderr, "[pcsb] sweep: queries %.3f attraction %.3f grid-exposed %.3f "
                         "repulsion+update %.3f tail %.3f total %.3f ms\n", q, ta - q, exposed,
                         tk - std::max(ta, tg), te - tk, te);
        }
        event_pool_.push_back(se);
    }
    pending_.clear();
}

template <typename T>
void Plan::grid_rebuild(const void* Xcur, cudaStream_t st) {
    using V = typename Vec4<T>::type;
    const uint32_t* done = &st_->done;
    RadixScratch& scr = st == stream2_ ? rs2_ : rs_;
    launch_keys<T>(gX_, (const V*)Xcur, mpad_, X_keys_, done, st);
    launches_ += 1;
    launches_ += radix_sort(X_keys_, nullptr, X_skeys_, X_sidx_, mpad_, gX_.key_bits, scr, done, st);
    launches_ += build_cell_start(X_skeys_, (uint32_t)m_, 3 * gX_.sub_bits, gX_.ncells, X_start_,
                                  cell_scratch_, done, st);
    if (fp32_) {  // gather + pack in one pass
        launches_ += build_pairs((const float4*)Xcur, X_sidx_, (float4*)X_sorted_, X_skeys_,
                                 (uint32_t)m_, gX_, X_start_, X_pairs_, done, st);
    } else {
        launch_gather<T>((const V*)Xcur, X_sidx_, (uint32_t)m_, (V*)X_sorted_, done, st);
        launches_ += 1;
    }
}

void Plan::allgather_x(void* X, bool f32, cudaStream_t st) {
    coll_->allgather(X, (size_t)chunk_ * 4, f32 ? CDType::F32 : CDType::F64, st ? st : stream_);
}

// WLOP w_i of the owned queries on X^k (internal indices in qlist), written to
// Xcur.w; after the exchange (sharded) the sorted copy and the records are
// refreshed from Xcur so that the repulsion pass sees every w_i'.
template <typename T>
void Plan::density_pass_x(const uint32_t* qlist, uint32_t nq, void* Xcur) {
    using V = typename Vec4<T>::type;
    const bool multi = sharded();
    SweepSlot* slot = slots_ + (sweeps_issued_ - 1) % slot_cap_;
    if (fp32_) {
        DensityArgs da{};
        da.C = (const float4*)Xcur;
        da.Cpairs = X_pairs_;
        da.Cpairs_cap = X_pairs_cap_;
        da.Cstart = X_start_;
        da.qlist = qlist;
        da.qcodes = q_skeys_;
        da.block_shift = group_order_ ? 0 : block_shift_;
        da.nq = nq;
        da.unit = work_unit_queries(nq, density_grid_ * 4);
        da.g = gX_;
        da.s_pad = s_pad_;
        da.r2 = r2_;
        const F32Consts fc = fp32_consts(d_.h, r2_, s_pad_, maxabs_);
        da.scull2 = fc.scull2;
        da.kneg = fc.kneg;
        da.K0 = fc.K0;
        da.band = fc.band;
        da.inv_scale = fc.inv_scale;
        da.invert = 0;
        da.out_sorted = (float4*)Xcur;
        da.st = st_;
        da.counter = &slot->density_counter;
        da.done = &st_->done;
        launch_density(da, density_grid_, stream_);
    } else {
        launch_exact_density<T>((const V*)X_sorted_, X_start_, (const V*)Xcur, qlist, nq, X_sidx_,
                                gX_, s_pad_, r2_, support_, d_.h, 0, (V*)Xcur, nullptr, st_,
                                &st_->done, stream_);
    }
    launches_ += 1;
    if (multi) allgather_x(Xcur, fp32_);
    if (fp32_) {
        launches_ += build_pairs((const float4*)Xcur, X_sidx_, (float4*)X_sorted_, X_skeys_,
                                 (uint32_t)m_, gX_, X_start_, X_pairs_, &st_->done, stream_);
    } else {
        launch_gather<T>((const V*)Xcur, X_sidx_, (uint32_t)m_, (V*)X_sorted_, &st_->done, stream_);
        launches_ += 1;
    }
}

template <typename T>
void Plan::enqueue_sweep(int k) {
    using V = typename Vec4<T>::type;
    // sweep slots are recycled modulo slot_cap_: finalize of sweep k clears the
    // slot of sweep k + 1 (any iteration count, LopParams::iterations >= 1)
    SweepSlot* slot = slots_ + (k - 1) % slot_cap_;
    SweepSlot* next_slot = slots_ + k % slot_cap_;
    void* cur = X_[(k - 1) & 1];
    void* nxt = X_[k & 1];
    const uint32_t* done = &st_->done;
    const bool multi = sharded();

    SweepEvents se;
    if (!event_pool_.empty()) {
        se = event_pool_.back();
        event_pool_.pop_back();
    } else {
        for (auto& e : se.e) PCSB_CUDA(cudaEventCreate(&e));
    }
    PCSB_CUDA(cudaEventRecord(se.e[0], stream_));
    if (record_counts_)  // queries this rank does not own stay -1
        PCSB_CUDA(cudaMemsetAsync(qcounts_, 0xFF, (size_t)std::max<uint32_t>(mpad_, 1) * sizeof(int4),
                                  stream_));
    const int rep = d_.mu > 0.0 ? (d_.eta_kind == PCS_ETA_INV_CUBE ? 1 : 2) : 0;
    // the projected set's grid is needed by the repulsion (and WLOP w_i) only
    const bool xgrid = rep != 0;

    // (1) index over the moving set (lop.cpp:39), on the side stream: it overlaps
    //     the query ordering and the attraction pass, which need only P's grid
    if (xgrid) {
        PCSB_CUDA(cudaEventRecord(ev_xready_, stream_));
        PCSB_CUDA(cudaStreamWaitEvent(stream2_, ev_xready_, 0));
        PCSB_CUDA(cudaEventRecord(se.e[1], stream2_));
        if (multi && gather_pending_) {
            // the previous sweep's exchange, deferred to here: the other ranks'
            // positions are needed by the grid rebuild only, so the all-gather
            // runs beside the attraction pass (which reads the owned slots)
            allgather_x(cur, fp32_, stream2_);
            gather_pending_ = false;
        }
        grid_rebuild<T>(cur, stream2_);
        PCSB_CUDA(cudaEventRecord(se.e[2], stream2_));
    } else {
        PCSB_CUDA(cudaEventRecord(se.e[1], stream_));
        PCSB_CUDA(cudaEventRecord(se.e[2], stream_));
    }
    // query order: the owned range in Morton order (internal indices), rebuilt
    // from X^k every `reorder_every_` sweeps; in between the order is reused (the
    // grouping only decides which queries share staged candidates; group boxes
    // and neighbour sets always come from the current positions)
    if (k == 1 || sweeps_since_order_ >= reorder_every_ || q_stale_) {
        if (q_next_ready_ && k != 1 && !q_stale_) {
            // built on stream2_ during the previous sweep (from X^{k-1})
            PCSB_CUDA(cudaStreamWaitEvent(stream_, ev_qready_, 0));
            std::swap(q_skeys_, q_skeys_alt_);
            std::swap(q_list_, q_list_alt_);
            std::swap(block_shift_, block_shift_alt_);
        } else {
            launches_ += build_query_list((const V*)cur + own_lo_, own_cnt_, g_, support_, nullptr, 0,
                                          0, q_keys_, q_skeys_, q_list_, &block_shift_, rs_, done,
                                          stream_, own_lo_);
            group_order(cur, q_list_, q_skeys_, q_keys_, done, stream_);
        }
        sweeps_since_order_ = 0;
        q_stale_ = false;
    }
    q_next_ready_ = false;
    ++sweeps_since_order_;
    // the next re-ordering's list, off the critical path: on stream2_ behind the
    // grid rebuild (its kernels fill the SM slots the passes leave free); the
    // previous sweep's readers of the alternate buffers completed before X^k was
    // ready, which stream2_ waited for
    if (xgrid && async_order_ && sweeps_since_order_ >= reorder_every_ && k < last_sweep_) {
        // done == nullptr: this chain runs beside the main stream, whose
        // finalize kernel may set the flag mid-launch; a cooperative sort whose
        // blocks read the flag at different times would deadlock in grid.sync
        launches_ += build_query_list((const V*)cur + own_lo_, own_cnt_, g_, support_, nullptr, 0, 0,
                                      q_keys_alt_, q_skeys_alt_, q_list_alt_, &block_shift_alt_, rs2_,
                                      nullptr, stream2_, own_lo_);
        group_order(cur, q_list_alt_, q_skeys_alt_, q_keys_alt_, nullptr, stream2_);
        PCSB_CUDA(cudaEventRecord(ev_qready_, stream2_));
        q_next_ready_ = true;
    }
    const uint32_t* qlist = q_list_;
    const uint32_t nq = own_cnt_;
    PCSB_CUDA(cudaEventRecord(se.e[3], stream_));

    // (2) per-point update (lop.cpp:41-100)
    if (fp32_) {
        FastArgs a{};
        a.Ppairs = P_pairs_;
        a.Ppairs_cap = P_pairs_cap_;
        a.Pstart = P_start_;
        a.Xq = (const float4*)cur;
        a.Xpairs = X_pairs_;
        a.Xpairs_cap = X_pairs_cap_;
        a.Xstart = X_start_;
        a.qlist = qlist;
        a.qcodes = q_skeys_;
        a.block_shift = block_shift_;
        a.nq = nq;
        // groups by recursive bisection of the work units; LOP units of 32 queries
        // (4 groups), WLOP units of 16 — measured (tools/ab_probe.py, best of 3):
        // config 3 +0.9%, 2 +1.7%, 5 +1.8% with 32; config 4 (50x density gradient)
        // -4.3% with 32, +0.9% with 16
        // Sharded plans keep runs of consecutive curve positions cut at curve
        // blocks: a rank's queries are a slab of the projected set, where
        // consecutive positions of the whole domain's curve can lie far apart, and
        // a 32-query unit spanning two such pieces bisects into straddling groups
        // (emulated 8-rank sweep: slowest rank 1.03 ms bisected vs 0.72 ms cut).
        // groups: precomputed by group_order (bisected, cut at curve jumps) and
        // read back from the codes (block_shift 0), or in-kernel bisection
        // (PCSB_GROUP_ORDER=0 builds), or curve runs cut at blocks
        const bool bis = bisect_ && !multi && !group_order_;
        a.bisect = bis ? 1 : 0;
        if (group_order_) a.block_shift = 0;
        a.unit = bis && !dev_knob("PCSB_UNIT") && !d_.density_weights
                     ? 32u
                     : work_unit_queries(nq, fast_grid_ * 4);
        {   // the last ~one group per warp of the attraction pass comes in one-group units
            const uint32_t q = 32u / (uint32_t)lanes_;
            static const double tail_frac = [] {  // developer knob: warps' groups in the tail
                const char* e = dev_knob("PCSB_TAIL");
                return e ? std::atof(e) : 2.0;  // ~2 groups per warp: emulated 8-rank -3%, 1 GPU neutral
            }();
            uint64_t tail = (uint64_t)(tail_frac * attr_grid_ * 4u * q);
            // short lists (a rank of a sharded plan, a small projected set): the
            // pass is a few groups per warp, so the tail units' candidate rows are
            // dealt to two warps each (partial sums combined in part order).
            // Measured (tools/gpu_tail_parts.sh): slowest emulated rank of 8 on
            // config 3 0.664 -> 0.621 ms (4 parts 0.612), of 4 1.098 -> 1.059 ms
            // (10 groups per warp), config 2 -1.7%; with 14 groups per warp (config
            // 4) it costs 0.7%, with 20 (2 ranks) nothing changes
            static const int parts_knob = [] {  // developer knob: 1, 2 or 4
                const char* e = dev_knob("PCSB_TAIL_PARTS");
                return e ? std::atoi(e) : 0;
            }();
            const uint64_t groups_per_warp = nq / ((uint64_t)attr_grid_ * 4u * q);
            uint32_t parts = parts_knob ? (uint32_t)parts_knob : (groups_per_warp < 12 ? 2u : 1u);
            if (!(xgrid && !fused_) || !attr_x_ || tail_cap_ <= a.unit) parts = 1;  // split pass only
            parts = std::min(parts, kTailPlanes + 1u);
            if (parts > 1) tail = std::min<uint64_t>(tail, tail_cap_ - a.unit);
            a.tail_start = nq > tail ? (uint32_t)((nq - tail) / a.unit * a.unit) : 0u;
            a.tail_unit = q;
            if (parts > 1 && nq - a.tail_start > tail_cap_) parts = 1;
            a.tail_parts = parts;
            a.tail_cap = tail_cap_;
            a.attr_x = attr_x_;
            a.attr_nx = attr_nx_;
        }
        a.gP = g_;
        a.gX = gX_;
        a.s_pad = s_pad_;
        a.r2 = r2_;
        const F32Consts fc = fp32_consts(d_.h, r2_, s_pad_, maxabs_);
        a.scull2 = fc.scull2;
        a.kneg = fc.kneg;
        a.K0 = fc.K0;
        a.band = fc.band;
        a.support = (float)support_;
        a.mu = (float)d_.mu;
        a.Xnext = (float4*)nxt;
        a.careful_list = careful_list_;
        a.attr = attr_;
        a.attr_n = attr_n_;
        a.ever_isolated = ever_iso_;
        a.qcounts = record_counts_ ? qcounts_ : nullptr;
        a.qever = qever_;
        a.st = st_;
        a.slot = slot;
        a.done = done;
        const bool wl = d_.density_weights != 0;
        if (xgrid && !fused_) {
            launch_fast(a, lanes_, wl, k == 1, rep, 1, attr_grid_, stream_);  // attraction
            PCSB_CUDA(cudaEventRecord(se.e[6], stream_));
            PCSB_CUDA(cudaStreamWaitEvent(stream_, se.e[2], 0));
            if (d_.density_weights) density_pass_x<T>(qlist, nq, cur);  // (WLOP) w_i on X^k
            launch_fast(a, rep_lanes_, wl, k == 1, rep, 2, fast_grid_, stream_);  // repulsion + update
            launches_ += 2;
        } else {
            if (xgrid) {  // fused: attraction and repulsion per query group in one pass
                PCSB_CUDA(cudaStreamWaitEvent(stream_, se.e[2], 0));
                if (d_.density_weights) density_pass_x<T>(qlist, nq, cur);
            }
            launch_fast(a, lanes_, wl, k == 1, rep, 0, fast_grid_, stream_);
            launches_ += 1;
            PCSB_CUDA(cudaEventRecord(se.e[6], stream_));
        }
    } else {
        PCSB_CUDA(cudaEventRecord(se.e[6], stream_));
        if (xgrid) {
            PCSB_CUDA(cudaStreamWaitEvent(stream_, se.e[2], 0));
            if (d_.density_weights) density_pass_x<T>(qlist, nq, cur);
        }
    }
    PCSB_CUDA(cudaEventRecord(se.e[4], stream_));
    {
        ExactArgs<T> e{};
        e.P = (const V*)P_sorted_;
        e.Porder = P_order_;
        e.Pstart = P_start_;
        e.Xs = (const V*)X_sorted_;
        e.Xstart = X_start_;
        e.Xs_idx = X_sidx_;
        e.Xq = (const V*)cur;
        e.g = g_;
        e.gX = gX_;
        e.s_pad = s_pad_;
        e.r2 = r2_;
        e.support = support_;
        e.h = d_.h;
        e.mu = d_.mu;
        e.eta_kind = d_.eta_kind;
        e.wlop = d_.density_weights;
        e.Xnext = (V*)nxt;
        e.ever_isolated = ever_iso_;
        e.qcounts = record_counts_ ? qcounts_ : nullptr;
        e.qever = qever_;
        e.st = st_;
        e.slot = slot;
        e.done = done;
        if (fp32_) {
            e.qlist = careful_list_;
            e.nq_dev = &slot->careful_count;
            e.count_careful = 1;
            launch_exact<T>(e, 148 * 2, stream_);
        } else {
            e.qlist = qlist;
            e.nq = nq;
            e.count_careful = 0;
            launch_exact<T>(e, exact_grid_, stream_);
        }
        launches_ += 1;
    }
    // (4) exchange + aggregation (lop.cpp:102-119)
    if (multi) {
        // the all-gather of X^{k+1} moves to the side stream of the next sweep
        // (above) unless this is the run's last sweep or no grid is rebuilt
        const bool defer = xgrid && k < last_sweep_ && !capturing_;
        coll_->group_start();
        if (defer) gather_pending_ = true;
        else allgather_x(nxt, fp32_);
        coll_->allreduce(&slot->max_disp_bits, 1, CDType::U64, COp::Max, stream_);
        coll_->group_end();
    }
    launch_finalize_sweep(st_, slot, next_slot, d_.convergence_tol, stream_);
    launches_ += 1;
    PCSB_CUDA(cudaEventRecord(se.e[5], stream_));
    // timing events exist only for sweeps enqueued one by one (a captured record
    // is a dependency edge, not a timestamp of the replays)
    if (capturing_) capture_events_.push_back(se);
    else pending_.push_back(se);
}

// Precomputed query groups (launch_group_order) for the fused fp32 kernels:
// the list is permuted through `tmp` (the order build's free key buffer).
void Plan::group_order(const void* cur, uint32_t* qlist, uint32_t* codes, uint32_t* tmp,
                       const uint32_t* done, cudaStream_t st) {
    if (!group_order_ || !own_cnt_) return;
    launch_group_order(qlist, (const float4*)cur, own_cnt_, (float)(4.0 * support_ * support_), tmp,
                       codes, done, st);
    PCSB_CUDA(cudaMemcpyAsync(qlist, tmp, (size_t)own_cnt_ * sizeof(uint32_t),
                              cudaMemcpyDeviceToDevice, st));
    launches_ += 1;
}

void Plan::record_counts(bool on) {
    if (!uploaded_) throw Failure(PCS_ERR_INVALID_PARAM, "record_counts needs an uploaded plan");
    PCSB_CUDA(cudaSetDevice(device_));
    synchronize();
    const size_t mp = std::max<uint32_t>(mpad_, 1);
    if (on && !qcounts_) {
        qcounts_ = (int4*)dalloc(mp * sizeof(int4));
        qever_ = (uint8_t*)dalloc(mp);
        PCSB_CUDA(cudaMemsetAsync(qcounts_, 0xFF, mp * sizeof(int4), stream_));
        PCSB_CUDA(cudaMemsetAsync(qever_, 0, mp, stream_));
        PCSB_CUDA(cudaStreamSynchronize(stream_));
    }
    record_counts_ = on;
}

// Per query (original order) of the last sweep: {attraction interactions,
// repulsion interactions, coincident pairs, flags (QC_*)}; -1 for queries this
// rank did not own (sharded plans); ever_flags = the flags OR-ed over the run.
void Plan::query_counts(int32_t* counts4, uint8_t* ever_flags, uint64_t m) {
    if (!record_counts_ || !qcounts_)
        throw Failure(PCS_ERR_INVALID_PARAM, "per-query counts were not recorded (record_counts)");
    if (m != m_) throw Failure(PCS_ERR_INVALID_PARAM, "query_counts: m must equal the plan's m");
    PCSB_CUDA(cudaSetDevice(device_));
    synchronize();
    std::vector<int4> c(mpad_);
    std::vector<uint8_t> ev(mpad_);
    std::vector<uint32_t> ooi;
    if (mpad_) {
        PCSB_CUDA(cudaMemcpyAsync(c.data(), qcounts_, (size_t)mpad_ * sizeof(int4),
                                  cudaMemcpyDeviceToHost, stream_));
        PCSB_CUDA(cudaMemcpyAsync(ev.data(), qever_, mpad_, cudaMemcpyDeviceToHost, stream_));
        if (orig_of_internal_) {
            ooi.resize(mpad_);
            PCSB_CUDA(cudaMemcpyAsync(ooi.data(), orig_of_internal_, (size_t)mpad_ * sizeof(uint32_t),
                                      cudaMemcpyDeviceToHost, stream_));
        }
        PCSB_CUDA(cudaStreamSynchronize(stream_));
    }
    for (uint32_t i = 0; i < mpad_; ++i) {
        const uint32_t o = ooi.empty() ? i : ooi[i];
        if (o >= m) continue;
        if (counts4) {
            counts4[4 * (size_t)o] = c[i].x;
            counts4[4 * (size_t)o + 1] = c[i].y;
            counts4[4 * (size_t)o + 2] = c[i].z;
            counts4[4 * (size_t)o + 3] = c[i].w;
        }
        if (ever_flags) ever_flags[o] = ev[i];
    }
}

void Plan::download(double* X_out, pcs_lop_summary* s, uint32_t* iso, uint64_t cap) {
    PCSB_CUDA(cudaSetDevice(device_));
    synchronize();
    RunState hs;
    PCSB_CUDA(cudaMemcpy(&hs, st_, sizeof(hs), cudaMemcpyDeviceToHost));
    const bool multi = sharded();
    if (multi) {
        // per-rank counters -> job totals
        unsigned long long* tmp = nullptr;
        tmp = (decltype(tmp))talloc(7 * sizeof(unsigned long long));
        unsigned long long hv[7] = {hs.isolated_events, hs.coincident_pairs, hs.interactions_attr,
                                    hs.interactions_rep, hs.density_pairs, hs.careful_points,
                                    hs.lane_candidates};
        PCSB_CUDA(cudaMemcpyAsync(tmp, hv, sizeof(hv), cudaMemcpyHostToDevice, stream_));
        coll_->allreduce(tmp, 7, CDType::U64, COp::Sum, stream_);
        PCSB_CUDA(cudaMemcpyAsync(hv, tmp, sizeof(hv), cudaMemcpyDeviceToHost, stream_));
        PCSB_CUDA(cudaStreamSynchronize(stream_));
        tfree(tmp);
        hs.isolated_events = hv[0];
        hs.coincident_pairs = hv[1];
        hs.interactions_attr = hv[2];
        hs.interactions_rep = hv[3];
        hs.density_pairs = hv[4] + setup_density_pairs_;
        hs.careful_points = hv[5];
        hs.lane_candidates = hv[6];
    } else {
        hs.density_pairs += setup_density_pairs_;
    }
    const int iters = hs.iterations_run;
    void* fin = X_[iters & 1];
    double* dout = out_xyz_;
    uint8_t* diso = out_iso_;
    PCSB_CUDA(cudaMemsetAsync(diso, 0, m_ ? m_ : 1, stream_));
    if (fp32_) launch_unpermute<float>((const float4*)fin, orig_of_internal_, mpad_, dout, stream_);
    else launch_unpermute<double>((const double4*)fin, orig_of_internal_, mpad_, dout, stream_);
    launch_iso_to_orig(ever_iso_, orig_of_internal_, mpad_, diso, stream_);
    launches_ += 2;
    if (multi && m_)
        coll_->allreduce(diso, m_, CDType::U8, COp::Max, stream_);
    std::vector<uint8_t> hiso(m_);
    if (m_) PCSB_CUDA(cudaMemcpyAsync(hiso.data(), diso, m_, cudaMemcpyDeviceToHost, stream_));
    if (X_out && m_) d2h_staged(X_out, dout, m_ * 3 * sizeof(double), stream_);
    PCSB_CUDA(cudaStreamSynchronize(stream_));
    uint64_t k = 0;
    for (uint64_t i = 0; i < m_; ++i)
        if (hiso[i]) {
            if (iso && k < cap) iso[k] = (uint32_t)i;
            ++k;
        }
    if (s) {
        std::memset(s, 0, sizeof(*s));
        s->iterations_run = hs.iterations_run;
        s->converged = (int32_t)hs.converged;
        s->isolated_events = hs.isolated_events;
        s->coincident_pairs = hs.coincident_pairs;
        s->n_isolated = k;
        s->interactions_attr = hs.interactions_attr;
        s->interactions_rep = hs.interactions_rep;
        s->density_pairs = hs.density_pairs;
        s->careful_points = hs.careful_points;
        s->lane_candidates = hs.lane_candidates;
        s->last_max_disp = hs.last_max_disp;
        s->setup_ms = setup_ms_;
        s->sweeps_ms = sweeps_ms_;
        s->kernel_ms = kernel_ms_;
        s->sort_ms = sort_ms_;
    }
}

// ---------------------------------------------------------------------------
// Parity facilities
// ---------------------------------------------------------------------------

namespace {

template <typename T>
struct TmpGrid {
    using V = typename Vec4<T>::type;
    GridGeom g{};
    V* sorted = nullptr;
    V* unsorted = nullptr;
    uint32_t* order = nullptr;
    uint32_t* start = nullptr;
    uint32_t* skeys = nullptr;
    double s_pad = 0;
    double maxabs = 0;
    std::vector<void*> allocs;
    ~TmpGrid() {
        for (void* p : allocs) cudaFree(p);
    }
    void* alloc(size_t b) {
        void* p = nullptr;
        PCSB_CUDA(cudaMalloc(&p, b ? b : 16));
        allocs.push_back(p);
        return p;
    }
    // builds the grid of C over bbox(C u Q)
    void build(const double* C, uint64_t n, const double* dQ_or_null, const double* Q, uint64_t m,
               double support, cudaStream_t s) {
        const uint32_t nn = (uint32_t)n;
        double* dC = (double*)alloc(n * 3 * sizeof(double));
        PCSB_CUDA(cudaMemcpyAsync(dC, C, n * 3 * sizeof(double), cudaMemcpyHostToDevice, s));
        V* Cv = (V*)alloc(n * sizeof(V));
        unsorted = Cv;
        launch_convert_xyz<T>(dC, Cv, n, (T)1, s);
        unsigned long long* slots = (unsigned long long*)alloc(8 * sizeof(unsigned long long));
        init_bbox_slots(slots, s);
        launch_bbox<T>(Cv, n, slots, s);
        if (m) {
            V* Qv = (V*)alloc(m * sizeof(V));
            launch_convert_xyz<T>(dQ_or_null, Qv, m, (T)0, s);
            launch_bbox<T>(Qv, m, slots, s);
        }
        (void)Q;
        unsigned long long hb[6];
        PCSB_CUDA(cudaMemcpyAsync(hb, slots, sizeof(hb), cudaMemcpyDeviceToHost, s));
        PCSB_CUDA(cudaStreamSynchronize(s));
        double lo[3], hi[3], maxabs = 0;
        for (int a = 0; a < 3; ++a) {
            lo[a] = ordered_to_double(hb[a]);
            hi[a] = ordered_to_double(hb[3 + a]);
            if (!std::isfinite(lo[a]) || !std::isfinite(hi[a]))
                throw Failure(PCS_ERR_INVALID_PARAM, "clouds must have finite coordinates");
            maxabs = std::max(maxabs, std::max(std::fabs(lo[a]), std::fabs(hi[a])));
        }
        g = make_grid(lo, hi, support, n);
        s_pad = support * (1.0 + std::ldexp(1.0, -10)) + 1e-12 * maxabs;
        this->maxabs = maxabs;
        uint32_t* keys = (uint32_t*)alloc(nn * sizeof(uint32_t));
        skeys = (uint32_t*)alloc(nn * sizeof(uint32_t));
        order = (uint32_t*)alloc(nn * sizeof(uint32_t));
        sorted = (V*)alloc(nn * sizeof(V));
        start = (uint32_t*)alloc(((size_t)g.ncells + 1) * sizeof(uint32_t));
        RadixScratch rs;
        rs.keys_alt = (uint32_t*)alloc(nn * sizeof(uint32_t));
        rs.vals_alt = (uint32_t*)alloc(nn * sizeof(uint32_t));
        rs.blockhist = (uint32_t*)alloc(radix_blockhist_entries(nn) * sizeof(uint32_t));
        rs.capacity = nn;
        uint32_t* cscr = (uint32_t*)alloc(cell_scan_scratch_entries(g.ncells) * sizeof(uint32_t));
        launch_keys<T>(g, Cv, nn, keys, nullptr, s);
        radix_sort(keys, nullptr, skeys, order, nn, g.key_bits, rs, nullptr, s);
        launch_gather<T>(Cv, order, nn, sorted, nullptr, s);
        build_cell_start(skeys, nn, 3 * g.sub_bits, g.ncells, start, cscr, nullptr, s);
    }
};

template <typename T>
void radius_query_t(const double* C, uint64_t n, const double* Q, uint64_t m, double r,
                    uint64_t* offsets, uint32_t* idx, uint64_t cap, cudaStream_t s) {
    TmpGrid<T> tg;
    double* dQ = (double*)tg.alloc((m ? m : 1) * 3 * sizeof(double));
    if (m) PCSB_CUDA(cudaMemcpyAsync(dQ, Q, m * 3 * sizeof(double), cudaMemcpyHostToDevice, s));
    tg.build(C, n, dQ, Q, m, r, s);
    uint64_t* dcnt = (uint64_t*)tg.alloc((m + 1) * sizeof(uint64_t));
    launch_radius_dump<T>(tg.sorted, tg.order, tg.start, tg.g, dQ, (uint32_t)m, r, tg.s_pad, dcnt,
                          nullptr, s);
    std::vector<uint64_t> cnt(m);
    if (m) PCSB_CUDA(cudaMemcpyAsync(cnt.data(), dcnt, m * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    PCSB_CUDA(cudaStreamSynchronize(s));
    offsets[0] = 0;
    for (uint64_t i = 0; i < m; ++i) offsets[i + 1] = offsets[i] + cnt[i];
    if (!idx) return;
    const uint64_t total = offsets[m];
    if (total > cap) throw Failure(PCS_ERR_CAPACITY, "idx buffer too small");
    uint32_t* didx = (uint32_t*)tg.alloc((total ? total : 1) * sizeof(uint32_t));
    PCSB_CUDA(cudaMemcpyAsync(dcnt, offsets, m * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
    launch_radius_dump<T>(tg.sorted, tg.order, tg.start, tg.g, dQ, (uint32_t)m, r, tg.s_pad, dcnt,
                          didx, s);
    if (total)
        PCSB_CUDA(cudaMemcpyAsync(idx, didx, total * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    PCSB_CUDA(cudaStreamSynchronize(s));
    PCSB_CUDA(cudaGetLastError());
    // hits ascending by index (proj/src/spatial.cpp:109-110)
    for (uint64_t i = 0; i < m; ++i) std::sort(idx + offsets[i], idx + offsets[i + 1]);
}

template <typename T>
void grid_sort_t(const double* C, uint64_t n, double support, uint32_t* keys_out,
                 uint32_t* order_out, cudaStream_t s) {
    TmpGrid<T> tg;
    tg.build(C, n, nullptr, nullptr, 0, support, s);
    PCSB_CUDA(cudaMemcpyAsync(keys_out, tg.skeys, n * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    PCSB_CUDA(cudaMemcpyAsync(order_out, tg.order, n * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    PCSB_CUDA(cudaStreamSynchronize(s));
    PCSB_CUDA(cudaGetLastError());
}

struct StreamGuard {
    cudaStream_t s = nullptr;
    StreamGuard() { PCSB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); }
    ~StreamGuard() {
        cudaStreamSynchronize(s);
        cudaStreamDestroy(s);
    }
};

}  // namespace

void radius_query_all(const pcs_lop_desc& d, const double* C, uint64_t n, const double* Q,
                      uint64_t m, double r, uint64_t* offsets, uint32_t* idx, uint64_t cap) {
    if (!(r > 0.0) || !std::isfinite(r))
        throw Failure(PCS_ERR_INVALID_PARAM, "radius_query requires finite r > 0");
    offsets[0] = 0;
    if (n == 0) {
        for (uint64_t i = 0; i < m; ++i) offsets[i + 1] = 0;
        return;
    }
    select_device(d.device);
    StreamGuard sg;
    if (d.precision == PCS_PREC_FP32) radius_query_t<float>(C, n, Q, m, r, offsets, idx, cap, sg.s);
    else radius_query_t<double>(C, n, Q, m, r, offsets, idx, cap, sg.s);
}

namespace {
template <typename T>
void density_weights_t(const pcs_lop_desc& d, const double* C, uint64_t n, double* v_out,
                       cudaStream_t s) {
    using V = typename Vec4<T>::type;
    const double support = d.h * d.cutoff_multiple;
    const double r2 = support * support;
    TmpGrid<T> tg;
    tg.build(C, n, nullptr, nullptr, 0, support, s);
    RunState* st = (RunState*)tg.alloc(sizeof(RunState));
    uint32_t* counter = (uint32_t*)tg.alloc(sizeof(uint32_t));
    PCSB_CUDA(cudaMemsetAsync(st, 0, sizeof(RunState), s));
    PCSB_CUDA(cudaMemsetAsync(counter, 0, sizeof(uint32_t), s));
    if (sizeof(T) == 4) {
        DensityArgs da{};
        uint32_t* pf = (uint32_t*)tg.alloc(n * sizeof(uint32_t));
        uint32_t* pfs = (uint32_t*)tg.alloc(n * sizeof(uint32_t));
        uint32_t* pq = (uint32_t*)tg.alloc(n * sizeof(uint32_t));
        RadixScratch rs;
        rs.keys_alt = (uint32_t*)tg.alloc(n * sizeof(uint32_t));
        rs.vals_alt = (uint32_t*)tg.alloc(n * sizeof(uint32_t));
        rs.blockhist = (uint32_t*)tg.alloc(radix_blockhist_entries((uint32_t)n) * sizeof(uint32_t));
        rs.capacity = (uint32_t)n;
        int bsh = 0;
        build_query_list((const float4*)tg.sorted, (uint32_t)n, tg.g, support, nullptr, 0, 0, pf, pfs,
                         pq, &bsh, rs, nullptr, s);
        const size_t cp_cap = pairs_capacity((uint32_t)n, tg.g);
        float4* cp = (float4*)tg.alloc(cp_cap * sizeof(float4));
        build_pairs((const float4*)tg.sorted, nullptr, nullptr, tg.skeys, (uint32_t)n, tg.g, tg.start, cp,
                    nullptr, s);
        da.C = (const float4*)tg.sorted;
        da.Cpairs = cp;
        da.Cpairs_cap = cp_cap;
        da.Cstart = tg.start;
        da.qlist = pq;
        da.qcodes = pfs;
        da.block_shift = bsh;
        da.nq = (uint32_t)n;
        da.g = tg.g;
        da.s_pad = tg.s_pad;
        da.r2 = r2;
        const F32Consts fc = fp32_consts(d.h, r2, tg.s_pad, tg.maxabs);
        da.scull2 = fc.scull2;
        da.kneg = fc.kneg;
        da.K0 = fc.K0;
        da.band = fc.band;
        da.inv_scale = fc.inv_scale;
        da.invert = 0;
        da.out_internal = (float4*)tg.unsorted;
        da.idx = tg.order;
        da.st = st;
        da.counter = counter;
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const int blocks = sms * fast_blocks_per_sm(4, true, false, 0);
        da.unit = work_unit_queries((uint32_t)n, blocks * 4);
        launch_density(da, blocks, s);
    } else {
        launch_exact_density<T>(tg.sorted, tg.start, tg.sorted, nullptr, (uint32_t)n, nullptr, tg.g,
                                tg.s_pad, r2, support, d.h, 0, tg.unsorted, tg.order, st, nullptr, s);
    }
    std::vector<V> h(n);
    PCSB_CUDA(cudaMemcpyAsync(h.data(), tg.unsorted, n * sizeof(V), cudaMemcpyDeviceToHost, s));
    PCSB_CUDA(cudaStreamSynchronize(s));
    PCSB_CUDA(cudaGetLastError());
    for (uint64_t i = 0; i < n; ++i) v_out[i] = (double)h[i].w;
}
}  // namespace

void density_weights(const pcs_lop_desc& d, const double* C, uint64_t n, double* v_out) {
    validate_desc(d);
    if (n == 0) return;
    select_device(d.device);
    StreamGuard sg;
    if (d.precision == PCS_PREC_FP32) density_weights_t<float>(d, C, n, v_out, sg.s);
    else density_weights_t<double>(d, C, n, v_out, sg.s);
}

void grid_sort(const pcs_lop_desc& d, const double* C, uint64_t n, double support,
               uint32_t* keys_out, uint32_t* order_out) {
    if (!(support > 0.0)) throw Failure(PCS_ERR_INVALID_PARAM, "support must be positive");
    if (n == 0) return;
    select_device(d.device);
    StreamGuard sg;
    if (d.precision == PCS_PREC_FP32) grid_sort_t<float>(C, n, support, keys_out, order_out, sg.s);
    else grid_sort_t<double>(C, n, support, keys_out, order_out, sg.s);
}

}  // namespace pcsb
