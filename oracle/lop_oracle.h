/*
 * lop_oracle.h — CPU restatement of the reference LOP path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2401_03365_b200/,
 * include/) links or calls this.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load it, and only as the
 * checker (never as the thing measured for the GPU arm).
 *
 * It restates, in plain C, the algorithm of
 *   /root/reference/proj/src/lop.cpp:10-127        (pcs::lop_project)
 *   /root/reference/proj/src/kernels.cpp:8-29      (theta, eta_derivative_magnitude)
 *   /root/reference/proj/src/spatial.cpp:82-111    (radius_query: d2 <= r*r, hits by index)
 *   /root/reference/proj/include/pcs/core.hpp:28-35 (dot/norm2/norm evaluation order)
 * with the same operation order, so that with eta = 1/(3 r^3) and no density
 * weights it is bit-identical to the reference (pinned in tests against
 * oracle/_ref, the reference compiled from its own sources).  It extends the
 * reference with two variants the reference does not implement (parity for
 * those is pinned only by this restatement — see DESIGN.md §Oracle):
 *   - eta(r) = -r  (|eta'| = 1)
 *   - WLOP density weights v_j (data, once) and w_i (projected set, per sweep).
 */
#ifndef PCS_LOP_ORACLE_H
#define PCS_LOP_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_ETA_INV_CUBE = 0, ORC_ETA_NEG_LINEAR = 1 };

enum {
    ORC_OK = 0,
    ORC_INVALID_PARAM = 1,
    ORC_EMPTY_CLOUD = 2,
    ORC_NO_MEMORY = 3,
    ORC_EMPTY_MESH = 4
};

typedef struct orc_params {
    double h;                /* KernelParams::h */
    double cutoff_multiple;  /* KernelParams::cutoff_multiple */
    double mu;               /* LopParams::mu in [0, 0.5) */
    int32_t iterations;      /* LopParams::iterations >= 1 */
    double convergence_tol;  /* LopParams::convergence_tol > 0 */
    int32_t eta_kind;        /* ORC_ETA_* */
    int32_t density_weights; /* 0 = LOP, 1 = WLOP */
    int32_t store_f32;       /* 1: round the iterate to fp32 after every sweep and the
                                data density weights to fp32 (mirrors the fp32 storage of
                                the B200 fp32 mode; 0 = the reference's fp64 storage) */
} orc_params;

typedef struct orc_summary {
    int32_t iterations_run;
    int32_t converged;
    uint64_t isolated_events;
    uint64_t coincident_pairs;
    uint64_t n_isolated;        /* entries written to isolated_out */
    uint64_t interactions_attr; /* evaluated (i,j) attraction pairs with d > 0, all sweeps */
    uint64_t interactions_rep;  /* evaluated (i,i') repulsion pairs with d > 0, all sweeps */
    uint64_t density_pairs_x;   /* w_i pairs (WLOP), all sweeps */
    uint64_t density_pairs_p;   /* v_j pairs (WLOP), once */
    double last_max_disp;
} orc_summary;

/* pcs::lop_project restated.  P: n*3 doubles, X0: m*3 doubles, out: m*3.
 * isolated_out (capacity m, may be NULL) receives the unique ascending
 * isolated indices.  threads <= 0 means "OpenMP default". */
int orc_lop_project(const double* P, size_t n, const double* X0, size_t m,
                    const orc_params* prm, double* out, orc_summary* sum,
                    uint32_t* isolated_out, int threads);

/* Same, and flags_out (m bytes, may be NULL) = per point, OR over sweeps >= 2 of
 * 1 isolated, 2 anchored, 8 a zero-distance data sample skipped (lop.cpp:55-61):
 * the discontinuities of the reference's update. */
int orc_lop_project_flags(const double* P, size_t n, const double* X0, size_t m,
                          const orc_params* prm, double* out, orc_summary* sum,
                          uint32_t* isolated_out, uint8_t* flags_out, int threads);

/* One sweep only, from X (m*3) to Xnext (m*3); per-point outputs optional.
 * Used by the per-sweep parity tests.  v (n, may be NULL) are data density
 * weights for WLOP (computed internally when NULL and density_weights). */
int orc_lop_sweep(const double* P, size_t n, const double* X, size_t m,
                  const orc_params* prm, double* Xnext, uint8_t* isolated,
                  uint32_t* coincident, double* max_disp, int threads);

/* One sweep from X evaluated for the queries rows[0..nrows) only (the whole X
 * is the repulsion candidate set): Xnext_rows (nrows*3) and, when counts is
 * not NULL, 4 int32 per row: attraction interactions (0 < d <= s), repulsion
 * interactions, coincident pairs, flags (1 isolated, 2 anchored, 8 a
 * zero-distance data sample was skipped).  Used by the
 * full-size per-query parity tests. */
int orc_lop_sweep_rows(const double* P, size_t n, const double* X, size_t m,
                       const orc_params* prm, const uint32_t* rows, size_t nrows,
                       double* Xnext_rows, int32_t* counts, int threads);

/* SpatialIndex::radius_query for every query: CSR output, hits ascending by
 * index.  offsets has m+1 entries.  If idx is NULL only offsets are filled.
 * dist (may be NULL) receives sqrt(d2) per hit. */
int orc_radius_query_all(const double* C, size_t n, const double* Q, size_t m,
                         double r, uint64_t* offsets, uint32_t* idx, double* dist,
                         int threads);

/* WLOP density weights over one cloud: v_j = 1 + sum_{j' != j, d2 <= s^2} theta(d). */
int orc_density_weights(const double* C, size_t n, double h, double cutoff,
                        double* v_out, int threads);

/* The pinned generators (same draw order as pcs::rng, proj/include/pcs/rng.hpp:16-46). */
void orc_add_noise(double* xyz, size_t n, double sigma, uint64_t seed);
void orc_plane(double* xyz, size_t n, uint64_t seed);
void orc_sphere(double* xyz, size_t n, uint64_t seed);
double orc_theta(double d, double h, double cutoff);
/* The benchmark configurations (same draws as pcs_generate_config): sizes, then
 * P (n_p*3) and X0 (n_x*3, may be NULL). */
int orc_config_sizes(int cfg, double scale, uint64_t* n_p, uint64_t* n_x);
int orc_generate_config(int cfg, double scale, double* P, double* X0);

/* Deviation metrics: proj/src/spatial.cpp:119-158 (nearest),
 * proj/src/metrics.cpp:11-133 (aggregate, deviation, point_triangle_distance,
 * deviation_to_mesh).  out = {n, mean, rms, max}. */
int orc_nearest_all(const double* C, size_t n, const double* Q, size_t m, uint32_t* idx_out,
                    double* dist_out, int threads);
int orc_deviation(const double* cloud, size_t m, const double* ref, size_t n, double out[4],
                  double* dist_out, int threads);
double orc_point_triangle_distance(const double p[3], const double tri[9]);
int orc_deviation_to_mesh(const double* cloud, size_t m, const double* tri, size_t ntri,
                          double out[4], double* dist_out, int threads);

/* MLS projection: proj/src/wls.cpp:53-222 (fit_reference_plane,
 * fit_local_polynomial), proj/src/mls.cpp:28-69 (project_point_guarded without
 * a guard).  Hits in ascending index order, weighted sums in that order (as the
 * reference); the eigen-solvers are restated, not Eigen's: the 3x3 covariance by
 * the closed form (trigonometric roots of the characteristic cubic, eigenvector
 * as the largest cross product of rows of A - l I), the K x K normal matrix by
 * cyclic Jacobi in long double.  Parity with the reference is pinned by the
 * reference's own tests (test_wls / test_mls properties), not by golden vectors:
 * Eigen is absent here, so the reference's MLS cannot be built. */
typedef struct orc_mls_params {
    double h, cutoff;
    int degree;
    double tol;
    int max_iter;
} orc_mls_params;
typedef struct orc_mls_result {
    double projected[3];
    double origin[3], normal[3], u[3], v[3];
    double coeffs[15];
    int status, degree_used, iterations, plane_status, poly_status;
} orc_mls_result;
enum { ORC_MLS_PROJECT = 0, ORC_MLS_PLANE = 1, ORC_MLS_POLY = 2 };
/* mode POLY: frames = 12 doubles per query (origin, normal, u, v). */
int orc_mls_project(const double* C, size_t n, const double* Q, size_t m, const orc_mls_params* prm,
                    int mode, const double* frames, orc_mls_result* out, int threads);

#ifdef __cplusplus
}
#endif
#endif
