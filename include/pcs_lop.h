/*
 * pcs_lop.h — C ABI of the B200-native LOP/WLOP operator.
 *
 * This is the drop-in boundary for the reference's hot path
 *
 *   std::pair<PointCloud, LopSummary>
 *   pcs::lop_project(const PointCloud& data, const PointCloud& initial,
 *                    const LopParams& params);
 *       /root/reference/proj/include/pcs/lop.hpp:51-53, src/lop.cpp:10-127
 *
 * Plain pointers and sizes only (no C++ or torch types).  The C++ header set
 * include/pcs/ (*.hpp) re-exposes pcs::lop_project with the reference's structs on
 * top of this ABI; Python binds it with ctypes (paper_2401_03365_b200/lop.py).
 *
 * Error model (mirrors proj/include/pcs/errors.hpp:9-53): every entry point
 * returns a pcs_status; the message of the last failure on the calling host
 * thread is available from pcs_last_error().  The reference's validation order
 * is kept: InvalidParam, then EmptyCloud(data), then an empty initial set
 * passes through (proj/src/lop.cpp:13-20).
 *
 * Threading: every call is synchronous with respect to the host buffers it is
 * given, re-entrant, and may be issued from any host thread; a plan object is
 * not thread-safe (one thread at a time per plan).
 */
#ifndef PCS_LOP_H
#define PCS_LOP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PCS_LOP_ABI_VERSION 1

typedef enum pcs_status {
    PCS_OK = 0,
    PCS_ERR_INVALID_PARAM = 1,  /* pcs::InvalidParam  (errors.hpp:23-26) */
    PCS_ERR_EMPTY_CLOUD = 2,    /* pcs::EmptyCloud    (errors.hpp:14-18) */
    PCS_ERR_NUMERICAL = 3,      /* pcs::NumericalFailure (errors.hpp:48-51) */
    PCS_ERR_CUDA = 4,           /* device / driver failure (reported as NumericalFailure in C++) */
    PCS_ERR_NCCL = 5,           /* collective failure */
    PCS_ERR_NO_DEVICE = 6,      /* no usable sm_100 device: there is no CPU fallback */
    PCS_ERR_CAPACITY = 7,       /* caller buffer too small; required size reported */
    PCS_ERR_EMPTY_MESH = 8,     /* pcs::EmptyMesh     (errors.hpp:20-23) */
    PCS_ERR_PARSE = 9           /* pcs::ParseError    (errors.hpp): see pcs_parse_error */
} pcs_status;

/* Repulsion penalty eta.  The reference hard-codes eta = 1/(3 r^3),
 * |eta'| = 1/r^4 (proj/src/kernels.cpp:17-29).  eta = -r (|eta'| = 1) is the
 * WLOP convention named by the benchmark configs; it is an extension. */
typedef enum pcs_eta_kind {
    PCS_ETA_INV_CUBE = 0,
    PCS_ETA_NEG_LINEAR = 1
} pcs_eta_kind;

typedef enum pcs_precision {
    PCS_PREC_FP64 = 0,  /* reference arithmetic: fp64 storage and math, exact predicate */
    PCS_PREC_FP32 = 1   /* fp32 storage, fused SFU/FP32 kernel; predicate re-decided in fp64 */
} pcs_precision;

/* LopParams (proj/include/pcs/lop.hpp:12-27) + KernelParams (kernels.hpp:12-24)
 * + the B200 extensions.  Initialise with pcs_lop_desc_default(). */
typedef struct pcs_lop_desc {
    uint32_t struct_size;      /* sizeof(pcs_lop_desc) — ABI guard */
    double h;                  /* KernelParams::h (Gaussian bandwidth) */
    double cutoff_multiple;    /* KernelParams::cutoff_multiple; support = h*cutoff */
    double mu;                 /* LopParams::mu in [0, 0.5) */
    int32_t iterations;        /* LopParams::iterations >= 1 */
    double convergence_tol;    /* LopParams::convergence_tol > 0 */
    int32_t eta_kind;          /* pcs_eta_kind */
    int32_t density_weights;   /* 0 = LOP, 1 = WLOP (v_j on data, w_i per sweep) */
    int32_t precision;         /* pcs_precision */
    int32_t device;            /* CUDA ordinal; -1 = current device */
    int32_t lanes_per_point;   /* fp32 kernel tuning: 0 = auto, else 2, 4, 8 */
    int32_t no_graphs;         /* 1: enqueue every sweep's launches; 0 (default): sweeps 2.. of
                                  unsharded plans are replayed as CUDA graphs of 8 sweeps */
    int32_t reserved[6];
} pcs_lop_desc;

/* LopSummary (proj/include/pcs/lop.hpp:29-35) + measured counters. */
typedef struct pcs_lop_summary {
    int32_t iterations_run;
    int32_t converged;
    uint64_t isolated_events;    /* per-sweep isolated count, summed over sweeps */
    uint64_t coincident_pairs;   /* ordered (i,i') pairs with d == 0 seen by repulsion */
    uint64_t n_isolated;         /* size of the unique ascending isolated index list */
    uint64_t interactions_attr;  /* evaluated (i,j) pairs with 0 < d <= support, all sweeps */
    uint64_t interactions_rep;   /* evaluated (i,i') pairs with 0 < d <= support, all sweeps */
    uint64_t density_pairs;      /* WLOP w_i / v_j pairs evaluated (0 < d <= support) */
    uint64_t careful_points;     /* points re-evaluated by the exact fp64 path (fp32 mode) */
    double last_max_disp;        /* max displacement of the last sweep */
    double setup_ms;             /* device time: upload conversion, data grid, v_j */
    double sweeps_ms;            /* device time of all sweeps (CUDA events) */
    double kernel_ms;            /* device time of the fused per-point kernel, all sweeps */
    double sort_ms;              /* device time of the per-sweep grid rebuild, all sweeps */
    uint64_t lane_candidates;    /* (point, candidate) evaluations of the fused kernel */
} pcs_lop_summary;

typedef struct pcs_lop_plan pcs_lop_plan;

/* ---- descriptor / errors ------------------------------------------------- */
void pcs_lop_desc_default(pcs_lop_desc* d);
const char* pcs_last_error(void);
int32_t pcs_lop_abi_version(void);
/* Validates exactly like LopParams::validate() (lop.hpp:18-26). */
pcs_status pcs_lop_validate(const pcs_lop_desc* d);

/* ---- one-shot drop-in call (replaces pcs::lop_project) ---------------------
 * P: n points as xyz doubles (PointCloud data), X0: m points (initial),
 * X_out: m points (the projected cloud).  isolated_out (capacity
 * isolated_cap, may be NULL) receives LopSummary::isolated_indices; if it is
 * too small the call still succeeds, summary->n_isolated reports the size and
 * only the first isolated_cap entries are written. */
pcs_status pcs_lop_run(const pcs_lop_desc* d, const double* P_xyz, uint64_t n,
                       const double* X0_xyz, uint64_t m, double* X_out_xyz,
                       pcs_lop_summary* summary, uint32_t* isolated_out,
                       uint64_t isolated_cap);

/* ---- plan API: device-resident runs (bench, multi-GPU) --------------------- */
pcs_status pcs_lop_plan_create(const pcs_lop_desc* d, pcs_lop_plan** out);
void pcs_lop_plan_destroy(pcs_lop_plan* p);
/* Uploads P and X0 (host doubles), builds the data grid (and v_j for WLOP). */
pcs_status pcs_lop_plan_upload(pcs_lop_plan* p, const double* P_xyz, uint64_t n,
                               const double* X0_xyz, uint64_t m);
/* Joins an NCCL clique (one process per GPU).  unique_id: 128 bytes from
 * pcs_nccl_unique_id() on rank 0, broadcast by the caller.  Must precede upload. */
pcs_status pcs_nccl_unique_id(uint8_t id_out[128]);
pcs_status pcs_lop_plan_set_comm(pcs_lop_plan* p, const uint8_t id[128], int32_t nranks,
                                 int32_t rank);
/* Loopback groups: nranks (<= 8) plans of ONE process on one device, each driven
 * by its own host thread, whose exchange step is a host rendezvous plus
 * device-to-device copies instead of NCCL.  A validation facility for the
 * sharded path on a single GPU (no kernel waits on another rank); not a
 * performance mode.  set_loopback must precede upload; destroy the group after
 * its plans. */
typedef struct pcs_loopback_group pcs_loopback_group;
pcs_status pcs_loopback_group_create(int32_t nranks, pcs_loopback_group** out);
void pcs_loopback_group_destroy(pcs_loopback_group* g);
pcs_status pcs_lop_plan_set_loopback(pcs_lop_plan* p, pcs_loopback_group* g, int32_t rank);
/* Restores X to X0 and clears the summary (P, grid and v_j are kept). */
pcs_status pcs_lop_plan_reset(pcs_lop_plan* p);
/* Runs `sweeps` further Jacobi sweeps (<= 0: the descriptor's iteration count),
 * stopping early on convergence.  Asynchronous unless sync != 0. */
pcs_status pcs_lop_plan_run(pcs_lop_plan* p, int32_t sweeps, int32_t sync);
pcs_status pcs_lop_plan_synchronize(pcs_lop_plan* p);
/* Device time of the last pcs_lop_plan_run (CUDA events on the plan stream). */
pcs_status pcs_lop_plan_last_run_ms(pcs_lop_plan* p, double* ms);
pcs_status pcs_lop_plan_download(pcs_lop_plan* p, double* X_out_xyz, pcs_lop_summary* summary,
                                 uint32_t* isolated_out, uint64_t isolated_cap);
/* Number of this process's kernel launches issued by the plan so far. */
uint64_t pcs_lop_plan_launches(const pcs_lop_plan* p);
/* Restart from the given positions (m points, original order; unsharded plans):
 * the next run starts its sweep 1 from X instead of X0.  The data grid and the
 * grid box of the upload are kept; positions may lie anywhere. */
pcs_status pcs_lop_plan_set_positions(pcs_lop_plan* p, const double* X_xyz, uint64_t m);
/* CUDA-graph replay of the sweeps on (1, the descriptor default unless
 * no_graphs) or off (0).  With graphs on, sweeps 2, 3, ... run as replays of one
 * captured graph of 8 sweeps (kernel_ms / sort_ms then cover only the sweeps
 * enqueued one by one); pcs_lop_plan_graph_launches counts the replays. */
pcs_status pcs_lop_plan_set_graphs(pcs_lop_plan* p, int32_t enable);
uint64_t pcs_lop_plan_graph_launches(const pcs_lop_plan* p);

/* Per-query evidence of the fused path (parity facility; off by default, call
 * after upload).  While enabled, every sweep records for each query of X^k:
 * {attraction interactions (0 < d <= support), repulsion interactions,
 * coincident pairs, flags} with flags 1 = isolated, 2 = anchored at a
 * zero-distance sample, 4 = deferred to the exact fp64 kernel.  These are the
 * per-point quantities of proj/src/lop.cpp:49-97 (hits of the two radius
 * queries :49,80 after the zero-distance and self rules).
 * pcs_lop_plan_query_counts returns the last sweep's records in original
 * order (counts4: 4*m int32; -1 for queries another rank owns) and, in
 * ever_flags (m bytes, may be NULL), the flags OR-ed over every sweep since
 * the last reset. */
pcs_status pcs_lop_plan_record_counts(pcs_lop_plan* p, int32_t enable);
pcs_status pcs_lop_plan_query_counts(pcs_lop_plan* p, int32_t* counts4, uint8_t* ever_flags,
                                     uint64_t m);
/* Returns the device memory the library keeps reserved between calls (its
 * stream-ordered pool on `device`, -1 = current) to the driver. */
pcs_status pcs_trim_device_pool(int32_t device);

/* ---- parity facilities ----------------------------------------------------
 * SpatialIndex::radius_query (proj/src/spatial.cpp:82-111) for every query, on
 * the device grid: CSR offsets (m+1) and hit indices ascending per query.
 * Call with idx == NULL to obtain offsets (total = offsets[m]) first.
 * Coordinates are rounded to fp32 first when precision == PCS_PREC_FP32
 * (the predicate is then the fp64 one over the rounded values). */
pcs_status pcs_radius_query_all(const pcs_lop_desc* d, const double* C_xyz, uint64_t n,
                                const double* Q_xyz, uint64_t m, double r,
                                uint64_t* offsets, uint32_t* idx, uint64_t idx_cap);
/* WLOP density weights over one cloud, v_j = 1 + sum_{j' != j, d <= support}
 * theta(d) (original order), evaluated exactly like the run does (fp32 fused
 * kernel or fp64 exact kernel per d->precision). */
pcs_status pcs_density_weights(const pcs_lop_desc* d, const double* C_xyz, uint64_t n,
                               double* v_out);
/* Grid sort order used by the device hash: sorted positions -> point index,
 * and the 32-bit cell keys, for a cloud (parity: stable sort by key). */
pcs_status pcs_grid_sort(const pcs_lop_desc* d, const double* C_xyz, uint64_t n, double support,
                         uint32_t* keys_out, uint32_t* order_out);

/* ---- deviation metrics (the next caller beside LOP) ---------
 * DeviationReport (proj/include/pcs/metrics.hpp:11-17): n, mean distance, RMS
 * ("std_deviation") and max distance of a cloud to a reference. */
typedef struct pcs_deviation_report {
    uint64_t n;
    double mean_distance;
    double std_deviation;
    double max_distance;
} pcs_deviation_report;

/* SpatialIndex::nearest (proj/src/spatial.cpp:119-158) for every query, on the
 * device: index of the nearest point of C (smallest index among equal squared
 * distances) and its distance sqrt(norm2(c - q)), bit-identical to the
 * reference.  n == 0 -> PCS_ERR_EMPTY_CLOUD. */
pcs_status pcs_nearest_all(const pcs_lop_desc* d, const double* C_xyz, uint64_t n,
                           const double* Q_xyz, uint64_t m, uint32_t* idx_out, double* dist_out);
/* pcs::deviation (proj/src/metrics.cpp:39-53): nearest-reference distance of
 * every cloud point (device), aggregated in index order as the reference does
 * (:11-37).  distances_out (m values) may be NULL.  Empty cloud, then empty
 * reference -> PCS_ERR_EMPTY_CLOUD. */
pcs_status pcs_deviation(const pcs_lop_desc* d, const double* cloud_xyz, uint64_t m,
                         const double* ref_xyz, uint64_t n, pcs_deviation_report* report,
                         double* distances_out);
/* pcs::deviation_to_mesh (proj/src/metrics.cpp:115-133): distance of every cloud
 * point to the nearest triangle of a triangle soup (9 doubles per triangle:
 * a, b, c), point_triangle_distance evaluated on the device with the
 * reference's operation order; aggregated like pcs_deviation.  Empty cloud ->
 * PCS_ERR_EMPTY_CLOUD, no triangles -> PCS_ERR_EMPTY_MESH. */
pcs_status pcs_deviation_to_mesh(const pcs_lop_desc* d, const double* cloud_xyz, uint64_t m,
                                 const double* tri_xyz, uint64_t ntri,
                                 pcs_deviation_report* report, double* distances_out);

/* ---- MLS projection ------------------------------------
 * Replaces the reference's per-point MLS solver (proj/src/wls.cpp:53-222,
 * proj/src/mls.cpp:28-93) and the spatial index it queries
 * (proj/include/pcs/spatial.hpp).  An index keeps a cloud resident on the
 * device; the grid for a query radius is built on first use and cached. */
typedef struct pcs_mls_index pcs_mls_index;

/* MlsParams (proj/include/pcs/mls.hpp:14-30) + the device. */
typedef struct pcs_mls_desc {
    uint32_t struct_size;      /* sizeof(pcs_mls_desc) */
    double h;                  /* KernelParams::h */
    double cutoff_multiple;    /* KernelParams::cutoff_multiple (support = h * cutoff) */
    int32_t degree;            /* polynomial degree in [1, 4] */
    double plane_tol;          /* plane fixed-point tolerance (> 0) */
    int32_t plane_max_iter;    /* >= 1 */
    int32_t device;            /* CUDA device, -1 = current */
} pcs_mls_desc;
void pcs_mls_desc_default(pcs_mls_desc* d); /* MlsParams defaults: h 1, cutoff 3, degree 2, 1e-10, 50 */

/* Mode of pcs_mls_project. */
typedef enum pcs_mls_mode {
    PCS_MLS_PROJECT = 0,  /* project_point_guarded without a guard (mls.cpp:28-69) */
    PCS_MLS_PLANE = 1,    /* fit_reference_plane (wls.cpp:53-147) */
    PCS_MLS_POLY = 2      /* fit_local_polynomial of degree d->degree over a given frame (wls.cpp:149-222) */
} pcs_mls_mode;

/* One query's outcome.  Status codes follow the reference enums:
 * status = ProjectionStatus (0 Full, 1 DegradedDegree, 2 PlaneOnly, 3 Skipped),
 * plane_status = PlaneFitStatus (0 Ok, 1 TooFewNeighbors, 2 DegenerateNeighborhood,
 * 3 NoConvergence), poly_status = PolyFitStatus of the last polynomial fit
 * (0 Ok, 1 TooFewNeighbors, 2 SingularSystem).  cmin/cmax bound every query
 * centre the computation used (plane iterates, frame origin) — a slab guard
 * (parallel_smooth) is decided from them exactly. */
typedef struct pcs_mls_result {
    double projected[3];
    double origin[3], normal[3], u[3], v[3];  /* LocalFrame */
    double coeffs[15];                        /* polynomial of degree_used (POLY: of d->degree) */
    double cmin[3], cmax[3];
    int32_t status;
    int32_t degree_used;
    int32_t iterations;
    int32_t plane_status;
    int32_t poly_status;
    int32_t pad;
} pcs_mls_result;

pcs_status pcs_mls_index_create(const double* xyz, uint64_t n, int32_t device, pcs_mls_index** out);
void pcs_mls_index_destroy(pcs_mls_index* index);
/* SpatialIndex::radius_query for m centres (proj/src/spatial.cpp:82-111): CSR of
 * the hits, ascending point index per centre, distances sqrt(norm2(p - c)) as
 * the reference computes them.  Query the total with idx/dist NULL first
 * (offsets[m] = total); PCS_ERR_CAPACITY when cap < total.  r must be finite > 0. */
pcs_status pcs_mls_index_radius(pcs_mls_index* index, const double* centers_xyz, uint64_t m,
                                double r, uint64_t* offsets, uint32_t* idx, double* dist,
                                uint64_t cap);
/* Per query: the projection / plane fit / polynomial fit, one warp per query.
 * frames (POLY only): 12 doubles per query, origin, normal, u, v.  centers_out
 * (may be NULL): (plane_max_iter + 1) x 3 doubles per query — the plane
 * iterates q_1..q_iterations, then the frame origin — so that a host-side
 * coverage predicate can be replayed in the reference's order. */
pcs_status pcs_mls_project(pcs_mls_index* index, const pcs_mls_desc* d, const double* q_xyz,
                           uint64_t m, int32_t mode, const double* frames, pcs_mls_result* out,
                           double* centers_out);
/* smooth_cloud (proj/src/mls.cpp:75-93) in one call: every point of the cloud
 * projected against the cloud itself; out_xyz (3n) and per-point results
 * (may be NULL). */
pcs_status pcs_mls_smooth(const pcs_mls_desc* d, const double* xyz, uint64_t n, double* out_xyz,
                          pcs_mls_result* results);
/* ProjectionOutcome without the point (proj/include/pcs/mls.hpp:38-44): what
 * smooth_cloud's SmoothingSummary::add consumes (proj/src/mls.cpp:5-16). */
typedef struct pcs_mls_outcome {
    int8_t status;        /* ProjectionStatus */
    int8_t degree_used;
    int8_t plane_status;  /* PlaneFitStatus */
    int8_t poly_status;   /* PolyFitStatus of the last fit tried */
    int32_t iterations;   /* plane-fit iterations */
} pcs_mls_outcome;
/* smooth_cloud as the reference returns it (the projected cloud and what the
 * summary needs): 32 bytes per point cross PCIe instead of the 312-byte
 * records of pcs_mls_smooth; the queries are the device index's own points. */
pcs_status pcs_mls_smooth_outcomes(const pcs_mls_desc* d, const double* xyz, uint64_t n,
                                   double* out_xyz, pcs_mls_outcome* outcomes);
/* The same with, per point, the bounds cmin[3], cmax[3] of the query centres its
 * projection used (plane iterates and frame origin: what a QueryCoverage guard
 * sees, proj/src/mls.cpp:28-47) in center_bounds (6n doubles): parallel_smooth
 * decides each worker point's coverage fallback from them
 * (proj/src/parallel.cpp:207-301). */
pcs_status pcs_mls_smooth_bounds(const pcs_mls_desc* d, const double* xyz, uint64_t n, double* out_xyz,
                                 pcs_mls_outcome* outcomes, double* center_bounds);
/* Measurement: device time (ms, CUDA events) of the plane-fit and the polynomial
 * launch of this process's last pcs_mls_smooth_outcomes call (bench.py). */
pcs_status pcs_mls_last_device_ms(double* plane_ms, double* poly_ms);
/* partition (proj/src/parallel.cpp:64-127), host only: axis, W-1 cuts, and the
 * worker of every point (counts differ by at most one). */
pcs_status pcs_mls_partition(const double* xyz, uint64_t n, uint64_t workers, double support,
                             int32_t* axis, double* cuts, uint32_t* worker_of);

/* ---- cloud IO (the data format either side of the path) -----
 * CloudFormat (proj/include/pcs/io.hpp): XYZ, or ASCII PLY. */
typedef enum pcs_cloud_format { PCS_FMT_XYZ = 0, PCS_FMT_PLY_ASCII = 1 } pcs_cloud_format;

/* Location and reason of a ParseError (the reference's "name:line: reason"). */
typedef struct pcs_parse_error {
    int64_t line;
    char reason[256];
} pcs_parse_error;

/* write_cloud_stream (proj/src/io.cpp:277-290): the file text of n points
 * (3 doubles each), coordinates in std::to_chars shortest round-trip form,
 * formatted on the device.  *len = bytes; out (cap bytes) may be NULL to size
 * the text first (PCS_ERR_CAPACITY when cap < *len). */
pcs_status pcs_format_cloud(const pcs_lop_desc* d, const double* xyz, uint64_t n, int32_t format,
                            char* out, uint64_t cap, uint64_t* len);
/* Same text in one pass, in a buffer the library allocates (release it with
 * pcs_free_buffer). */
pcs_status pcs_format_cloud_alloc(const pcs_lop_desc* d, const double* xyz, uint64_t n,
                                  int32_t format, char** out, uint64_t* len);
void pcs_free_buffer(void* p);
/* read_cloud_stream (proj/src/io.cpp:143-236, 260-264): parse a cloud file's text
 * on the device (lines the device cannot settle are re-read on the host with the
 * reference's rules).  *n_out = points; xyz_out receives 3*n doubles when
 * cap >= n (else PCS_ERR_CAPACITY, nothing written).  PCS_ERR_PARSE fills err
 * (may be NULL). */
pcs_status pcs_parse_cloud(const pcs_lop_desc* d, const char* text, uint64_t len, int32_t format,
                           double* xyz_out, uint64_t cap, uint64_t* n_out, pcs_parse_error* err);
/* read_mesh_stream (proj/src/io.cpp:306-325): triangles (9 doubles each) of an
 * ASCII PLY with a face element, fan-triangulated; host parser. */
pcs_status pcs_parse_mesh(const char* text, uint64_t len, double* tri_out, uint64_t cap,
                          uint64_t* ntri_out, pcs_parse_error* err);
/* format_double (proj/src/io.cpp:240-245): shortest round-trip text of v
 * (<= 32 bytes, not NUL-terminated); returns the length. */
int32_t pcs_format_double(double v, char* out32);

/* Multi-GPU ownership layout (host only, no device needed): shard r owns the
 * r-th contiguous range of `sorted_order` (the initial grid order of X0) and
 * occupies internal slots [r*chunk, r*chunk + counts[r]).  orig_of_internal
 * has nranks*chunk entries (0xFFFFFFFF for padding), internal_of_orig m. */
pcs_status pcs_shard_layout(const uint32_t* sorted_order, uint64_t m, int32_t nranks,
                            uint32_t* orig_of_internal, uint32_t* internal_of_orig,
                            uint32_t* chunk, uint32_t* counts);
/* Same, with the cuts at equal cumulative work: weights[o] = estimated work of
 * original point o (NULL = 1 each); chunk = the largest shard (the others are
 * padded).  Used by sharded plans with the data density around each X0 point. */
pcs_status pcs_shard_layout_weighted(const uint32_t* sorted_order, const float* weights,
                                     uint64_t m, int32_t nranks, uint32_t* orig_of_internal,
                                     uint32_t* internal_of_orig, uint32_t* chunk,
                                     uint32_t* counts);

/* ---- host generators (proj/include/pcs/rng.hpp, proj/src/bench.cpp:40-87) -- */
/* kind: 0 plane, 1 sphere, 2 torus(R=1,r=0.35), 3 gaussian bump */
pcs_status pcs_generate_surface(int32_t kind, uint64_t n, uint64_t seed, double* xyz);
pcs_status pcs_add_noise(double* xyz, uint64_t n, double sigma, uint64_t seed);
/* The benchmark configurations 1..5 (BASELINE.json), scaled by `scale` (1.0 =
 * full size).  Fills P (n_p points) and X0 (n_x points) — query the sizes with
 * P_xyz == NULL first.  Seeds: surface 0, noise 1, outliers/subset 2. */
pcs_status pcs_config_sizes(int32_t config, double scale, uint64_t* n_p, uint64_t* n_x);
pcs_status pcs_generate_config(int32_t config, double scale, double* P_xyz, double* X0_xyz);

#ifdef __cplusplus
}
#endif
#endif /* PCS_LOP_H */
