// plan.cuh — host-side orchestration of one LOP/WLOP run on one GPU (one rank).
//
// The plan owns every device buffer of a run, the stream it is issued on and
// (for multi-GPU) the NCCL communicator.  A sweep is a fixed sequence of
// launches (keys -> radix sort -> gather -> cell table -> [w_i] -> fused
// kernel -> deferred exact queries -> [all-gather X] -> finalize); all of them
// read a device "done" flag so sweeps after convergence cost a launch only.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/pcs_lop.h"
#include "common.cuh"
#include "comm.h"
#include "kernels.cuh"

namespace pcsb {

// Error carrying a pcs_status; converted at the C boundary.
struct Failure : std::runtime_error {
    pcs_status code;
    Failure(pcs_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void cuda_check(cudaError_t e, const char* what);
#define PCSB_CUDA(x) ::pcsb::cuda_check((x), #x)

// Derives the shared grid for a bounding box and a support radius.
GridGeom make_grid(const double lo[3], const double hi[3], double support, uint64_t npts);
// releases the reserved memory of the library's stream-ordered pool on `dev`
void trim_device_pool(int dev);
void* pool_alloc(int dev, size_t bytes, cudaStream_t s);
void pool_free(void* p, cudaStream_t s);
GridGeom make_grid_scaled(const double lo[3], const double hi[3], double support, double scale,
                          const GridGeom& base);
double x_cell_scale(uint64_t n, uint64_t m, const GridGeom& g);

void validate_desc(const pcs_lop_desc& d);  // throws Failure(INVALID_PARAM)
int select_device(int requested);           // throws Failure(NO_DEVICE)

class Plan {
public:
    explicit Plan(const pcs_lop_desc& d);
    ~Plan();
    Plan(const Plan&) = delete;
    Plan& operator=(const Plan&) = delete;

    void set_comm(const uint8_t id[128], int nranks, int rank);
    // In-process rank of a loopback group (comm.h): validation of the sharded path.
    void set_loopback(LoopbackGroup* g, int rank);
    void upload(const double* P, uint64_t n, const double* X0, uint64_t m);
    void reset();
    void set_positions(const double* X, uint64_t m);
    void run(int sweeps, bool sync);
    void synchronize();
    double last_run_ms() const { return last_run_ms_; }
    void download(double* X_out, pcs_lop_summary* s, uint32_t* iso, uint64_t cap);
    uint64_t launches() const { return launches_; }
    // CUDA-graph replay of sweeps 2, 3, ... in periods of kGraphPeriod (run()).
    void set_graphs(bool on);
    uint64_t graph_launches() const { return graph_launches_; }
    // Parity facility: per-query counts of every sweep (pcs_lop_plan_query_counts).
    void record_counts(bool on);
    void query_counts(int32_t* counts4, uint8_t* ever_flags, uint64_t m);

private:
    template <typename T> void upload_t(const double* P, uint64_t n, const double* X0, uint64_t m);
    template <typename T> void enqueue_sweep(int k);
    void enqueue_one(int k);
    // host state that enqueueing sweeps mutates (CUDA-graph capture / replay)
    struct HostSnap {
        uint32_t *qs, *ql, *qsa, *qla;
        int bs, bsa, since, issued, last;
        bool stale, next_ready;
        uint64_t launches;
        const void* counts;
    };
    HostSnap snapshot() const;
    void restore(const HostSnap& h);
    bool graph_matches() const;
    void replay_period();
    void capture_period(const HostSnap& at);
    void drop_graph();
    template <typename T> void density_pass_x(const uint32_t* qlist, uint32_t nq, void* Xcur);
    template <typename T> void grid_rebuild(const void* Xcur, cudaStream_t st);
    void allgather_x(void* X, bool fp32, cudaStream_t st = nullptr);
    bool gather_pending_ = false;  // sharded: X^k's all-gather runs at the start of sweep k
    void group_order(const void* cur, uint32_t* qlist, uint32_t* codes, uint32_t* tmp,
                     const uint32_t* done, cudaStream_t st);
    void free_all();
    void* dalloc(size_t bytes);
    void* talloc(size_t bytes);  // stream-ordered, from the device pool
    void tfree(void* p);

    pcs_lop_desc d_;
    bool fp32_;
    int device_ = 0;
    cudaStream_t stream_ = nullptr;
    cudaStream_t stream2_ = nullptr;  // projected-set grid, overlapped with the attraction pass
    cudaEvent_t ev_xready_ = nullptr;  // X^k final on stream_
    int nranks_ = 1, rank_ = 0;
    Collectives* coll_ = nullptr;  // owned; NCCL or loopback (comm.h)
    bool sharded() const { return coll_ != nullptr; }

    uint64_t n_ = 0, m_ = 0;
    uint32_t mpad_ = 0, chunk_ = 0, own_lo_ = 0, own_cnt_ = 0;
    GridGeom g_{};
    GridGeom gX_{};                 // grid of the projected set (make_grid_scaled)
    double support_ = 0, r2_ = 0, s_pad_ = 0;
    double maxabs_ = 0;               // largest |coordinate| at upload (fp32 rounding scale)
    int lanes_ = 4;
    int rep_lanes_ = 4;  // lanes per query of the repulsion pass
    int fast_grid_ = 0, exact_grid_ = 0, density_grid_ = 0;
    int attr_grid_ = 0;  // attraction pass blocks

    std::vector<void*> allocs_;
    size_t vec_bytes_ = 16;
    // data
    void* P_sorted_ = nullptr;
    uint32_t* P_order_ = nullptr;
    uint32_t* P_start_ = nullptr;
    float4* P_pairs_ = nullptr;      // fp32 candidate records (kernels.cuh)
    // projected set
    void* X_[2] = {nullptr, nullptr};
    void* X_init_ = nullptr;
    void* X_sorted_ = nullptr;
    uint32_t* X_keys_ = nullptr;
    uint32_t* X_skeys_ = nullptr;
    uint32_t* X_sidx_ = nullptr;
    uint32_t* X_start_ = nullptr;
    double* out_xyz_ = nullptr;       // download staging (original order, fp64)
    uint8_t* out_iso_ = nullptr;
    float4* X_pairs_ = nullptr;
    uint32_t* cell_scratch_ = nullptr;  // cell-table scan (build_cell_start)
    uint32_t* q_keys_ = nullptr;      // Morton codes of the query order (build_query_list)
    int block_shift_ = 0;
    // sweeps between query re-orderings (measured: 4 beats 1 by 3% on config 3 and
    // 12% per rank in the 8-GPU emulation; 15 loses group compactness)
    int reorder_every_ = 4;
    int sweeps_since_order_ = 0;
    bool q_stale_ = true;             // no order for the current X yet (upload / reset)
    uint32_t* q_skeys_ = nullptr;
    uint32_t* q_list_ = nullptr;
    // the next query order, built on stream2_ from X^k during sweep k (after the
    // projected-set grid) for the re-ordering sweep k+1, which swaps it in
    uint32_t* q_keys_alt_ = nullptr;
    uint32_t* q_skeys_alt_ = nullptr;
    uint32_t* q_list_alt_ = nullptr;
    int block_shift_alt_ = 0;
    bool q_next_ready_ = false;
    size_t P_pairs_cap_ = 0, X_pairs_cap_ = 0;  // float4 elements of the pair records
    bool fused_ = false;              // one pass (attraction + repulsion) after the X grid
    bool bisect_ = true;              // query groups by recursive bisection of 32-query units
    bool group_order_ = false;        // groups precomputed at each query-order rebuild (fp32)
    bool async_order_ = true;         // developer knob PCSB_ASYNC_ORDER=0: build in line
    int last_sweep_ = 0;              // last sweep index of the current run()
    cudaEvent_t ev_qready_ = nullptr;
    uint32_t* careful_list_ = nullptr;
    uint8_t* ever_iso_ = nullptr;
    uint32_t* orig_of_internal_ = nullptr;  // multi-GPU only
    bool record_counts_ = false;      // parity facility (record_counts)
    int4* qcounts_ = nullptr;         // last sweep, internal index
    uint8_t* qever_ = nullptr;        // flags OR-ed over the run
    RadixScratch rs_{};
    RadixScratch rs2_{};              // stream2_'s sorts
    float4* attr_ = nullptr;          // attraction sums per query-list position (PH_ATTR -> PH_REP)
    int2* attr_n_ = nullptr;
    static constexpr uint32_t kTailPlanes = 3;  // row-split tail units: up to 4 parts
    float4* attr_x_ = nullptr;  // kTailPlanes planes of tail_cap_ partial sums
    int2* attr_nx_ = nullptr;
    uint32_t tail_cap_ = 0;
    RunState* st_ = nullptr;
    SweepSlot* slots_ = nullptr;
    int slot_cap_ = 0;
    unsigned long long* bbox_slots_ = nullptr;

    int sweeps_issued_ = 0;
    bool uploaded_ = false;
    bool run_pending_ = false;
    unsigned long long setup_density_pairs_ = 0;
    uint64_t launches_ = 0;
    double setup_ms_ = 0, last_run_ms_ = 0, sweeps_ms_ = 0, kernel_ms_ = 0, sort_ms_ = 0;
    cudaEvent_t run_ev_[2] = {nullptr, nullptr};
    struct SweepEvents {
        // start | X grid begin, end (side stream) | queries | kernels | end | attraction end
        cudaEvent_t e[7];
    };
    std::vector<SweepEvents> pending_;  // per issued sweep in the current run
    std::vector<SweepEvents> event_pool_;
    // CUDA graph of kGraphPeriod sweeps.  A period starting at k0 = 2 (mod
    // kGraphPeriod) returns the host state (query-list buffers, reorder count) to
    // where it started and uses sweep slots 1..kGraphPeriod (mod kGraphPeriod),
    // so one capture is replayed for every later period with the same buffers.
    bool use_graphs_ = true;
    bool loopback_ = false;
    bool capturing_ = false;
    cudaGraph_t graph_ = nullptr;
    cudaGraphExec_t graph_exec_ = nullptr;
    uint64_t graph_period_launches_ = 0;  // kernels in one period
    uint64_t graph_launches_ = 0;         // replays
    HostSnap graph_snap_{};               // host state the captured period starts from
    HostSnap period_snap_{};              // a period start seen in the current run
    bool have_snap_ = false;
    uint32_t* q_home_[4] = {nullptr, nullptr, nullptr, nullptr};  // q_skeys_, q_list_, alts at upload
    std::vector<SweepEvents> capture_events_;
};

// Parity facilities (stateless).
void radius_query_all(const pcs_lop_desc& d, const double* C, uint64_t n, const double* Q,
                      uint64_t m, double r, uint64_t* offsets, uint32_t* idx, uint64_t cap);
void density_weights(const pcs_lop_desc& d, const double* C, uint64_t n, double* v_out);
void grid_sort(const pcs_lop_desc& d, const double* C, uint64_t n, double support,
               uint32_t* keys_out, uint32_t* order_out);

// Deviation metrics (nn.cu; proj/src/metrics.cpp, proj/src/spatial.cpp:119-158).
void nearest_all(const pcs_lop_desc& d, const double* C, uint64_t n, const double* Q, uint64_t m,
                 uint32_t* idx_out, double* dist_out);
void deviation(const pcs_lop_desc& d, const double* cloud, uint64_t m, const double* ref,
               uint64_t n, pcs_deviation_report* rep, double* distances_out);
void deviation_to_mesh(const pcs_lop_desc& d, const double* cloud, uint64_t m, const double* tri,
                       uint64_t ntri, pcs_deviation_report* rep, double* distances_out);


// MLS projection (mls.cu)
struct MlsIndex;
MlsIndex* mls_index_create(const double* xyz, uint64_t n, int device);
void mls_index_destroy(MlsIndex* ix);
void mls_index_radius(MlsIndex* ix, const double* centers, uint64_t m, double r, uint64_t* offsets,
                      uint32_t* idx, double* dist, uint64_t cap);
void mls_project(MlsIndex* ix, const pcs_mls_desc& d, const double* q, uint64_t m, int mode,
                 const double* frames, pcs_mls_result* out, double* centers_out);
void mls_smooth_outcomes(const pcs_mls_desc& d, const double* xyz, uint64_t n, double* out_xyz,
                         pcs_mls_outcome* outcomes, double* center_bounds);
void mls_last_device_ms(double out[2]);
void mls_smooth(const pcs_mls_desc& d, const double* xyz, uint64_t n, double* out_xyz,
                pcs_mls_result* results);
void mls_partition(const double* xyz, uint64_t n, uint64_t workers, double support, int32_t* axis,
                   double* cuts, uint32_t* worker_of);

}  // namespace pcsb
