// mls.cu — MLS projection on the device (the other
// per-point hot loop of the reference, beside LOP).
//
// Replaces, for a whole batch of query points at once:
//   fit_reference_plane    proj/src/wls.cpp:53-147   weighted-PCA fixed point
//   fit_local_polynomial   proj/src/wls.cpp:149-222  weighted normal equations
//   project_point_guarded  proj/src/mls.cpp:28-69    degree fallback ladder
//   smooth_cloud           proj/src/mls.cpp:75-93
//   SpatialIndex::radius_query  proj/src/spatial.cpp:82-111  (exact ball, CSR)
//
// B200 design: the cloud stays resident in HBM (fp64 double4) behind an index
// handle; for each support radius a uniform grid (cell side ~ support / 2, the
// LOP path's integer keys / radix sort / lower-bound cell table, grid_sort.cu)
// is built once and cached.  One warp per query point (persistent grid, atomic
// fetch): the candidate rows' bounds are loaded by the lanes at once and the
// candidates of up to 32 rows form one flat index space (row found by a binary
// search over shuffled prefix counts), so a radius query costs two dependent
// loads, not two per cell row.  Every weighted sum is lane-strided over that
// fixed enumeration and combined by a fixed xor tree: deterministic, but not
// the reference's index order, so results agree with it to rounding.
//
// Numerics (fp64 throughout, reference predicate and operation order):
//   hit        d2 = (dx*dx + dy*dy) + dz*dz <= r*r, no FMA; distance = sqrt(d2)
//   weight     theta(d) = d > support ? 0 : exp(-(d/h)^2)          (kernels.cpp:8-15)
//   plane      centroid, covariance about it, smallest-eigenvalue vector of
//              the 3x3 covariance (cyclic Jacobi; the reference uses Eigen's
//              closed-form solver), degenerate if l1 - l0 <= 1e-12 l2, move
//              q = r + <n, c - r> n, stop when |dq| < tol      (wls.cpp:75-135)
//   frame      normal flipped to <n, r - q> >= 0 (axis rule on a tie); u by
//              Gram-Schmidt against the least aligned axis, v = n x u (wls.cpp:12-35, 137-146)
//   polynomial normal matrix M = sum w b b^T, rhs sum w b f over the monomials
//              1, u, v, u^2, uv, v^2, ... (degree-major, a descending); eigen-
//              decomposition of M (cyclic Jacobi), singular if l_min <= 1e-12
//              l_max, solution V (V^T b / l) plus one refinement (wls.cpp:176-221)
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <numeric>
#include <vector>

#include "../../include/pcs_lop.h"
#include "host_io.h"
#include "kernels.cuh"
#include "plan.cuh"

namespace pcsb {

namespace {

constexpr int MLS_WARPS = 4;
constexpr int MLS_THREADS = MLS_WARPS * 32;
constexpr int KMAX = 15;   // coefficients of a degree-4 polynomial
constexpr int KS = 16;     // row stride of the per-warp matrices

enum : int { PS_FULL = 0, PS_DEGRADED = 1, PS_PLANE_ONLY = 2, PS_SKIPPED = 3 };
enum : int { PF_OK = 0, PF_TOO_FEW = 1, PF_DEGENERATE = 2, PF_NO_CONV = 3 };
enum : int { YF_OK = 0, YF_TOO_FEW = 1, YF_SINGULAR = 2 };

struct MlsArgs {
    const double4* pts;      // cloud in cell order
    const uint32_t* start;   // cell lower-bound table
    uint32_t n;              // cloud size (checked builds)
    GridGeom g;
    double s_pad, r2, support, h, inv_h;
    const double* q;         // queries, xyz
    uint32_t m;
    int mode;                // PCS_MLS_*
    int degree;
    double tol;
    int max_iter;
    const double* frames;    // POLY: 12 per query
    pcs_mls_result* out;
    double* centers;         // optional, (max_iter + 1) * 3 per query
    uint32_t* counter;
    // smooth_cloud (pcs_mls_smooth_outcomes): query i is the cloud's own sorted
    // point i (spatially coherent warps), results land at the point's original
    // index order[i] as xyz + the 8-byte outcome instead of the full record
    const uint32_t* order;
    double* lean_xyz;
    pcs_mls_outcome* lean_out;
    double* lean_bounds;     // optional: per point cmin[3], cmax[3] of the query centres used
    struct MlsMid* mid;      // plane-fit results between the two launches of the lean path
};

// What the polynomial launch of the lean path needs from the plane launch.
struct MlsMid {
    double o[3], n[3], u[3], v[3];
    double cmn[3], cmx[3];   // bounds of the plane iterates (the coverage guard's centres)
    int32_t iterations, plane_status, have_frame, pad;
};

struct WarpSmem {
    double A[KS * KS];   // matrix being diagonalised
    double M[KS * KS];   // copy of the normal matrix (refinement residual)
    double V[KS * KS];   // eigenvectors (columns)
    double b[KS], y[KS], x[KS], ev[KS];
    int perm[KS];
};

__device__ __noinline__ double wsum(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __noinline__ int wsumi(int v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// theta(d) = exp(-(d/h)^2) inside the support (proj/src/kernels.cpp:8-14); d/h as
// d * (1/h): one rounding apart from the reference's quotient
__device__ __forceinline__ double theta_k(double d, double support, double inv_h) {
    if (d > support) return 0.0;
    const double s = d * inv_h;
    return exp(-s * s);
}

// Calls f(k) for every candidate k (sorted position) of the cell rows within
// s_pad of c: batches of <= 32 rows, bounds loaded by the lanes at once,
// candidates flattened (each lane takes flat index lane, lane + 32, ...).
// Every lane calls f the same number of times per batch round (k = ~0u for
// padding), so f may use warp collectives.
template <typename F>
__device__ __forceinline__ void for_candidates(const MlsArgs& a, double cx, double cy, double cz,
                                               int lane, F&& f) {
    const GridGeom& g = a.g;
    const int lox = cell_coord(cx - a.s_pad, g.ox, g.inv_csx, g.gx);
    const int hix = cell_coord(cx + a.s_pad, g.ox, g.inv_csx, g.gx);
    const int loy = cell_coord(cy - a.s_pad, g.oy, g.inv_cs, g.gy);
    const int hiy = cell_coord(cy + a.s_pad, g.oy, g.inv_cs, g.gy);
    const int loz = cell_coord(cz - a.s_pad, g.oz, g.inv_cs, g.gz);
    const int hiz = cell_coord(cz + a.s_pad, g.oz, g.inv_cs, g.gz);
    const int ny = hiy - loy + 1;
    const int nrows = ny * (hiz - loz + 1);
    for (int r0 = 0; r0 < nrows; r0 += 32) {
        const int r = r0 + lane;
        uint32_t b = 0, cnt = 0;
        if (r < nrows) {
            const int yy = loy + r % ny, zz = loz + r / ny;
            const uint32_t base = ((uint32_t)zz * (uint32_t)g.gy + (uint32_t)yy) * (uint32_t)g.gx;
            PCSB_DCHECK((uint64_t)base + (uint64_t)hix + 1 <= (uint64_t)g.ncells);
            b = __ldg(&a.start[base + lox]);
            cnt = __ldg(&a.start[base + hix + 1]) - b;
            PCSB_DCHECK((uint64_t)b + cnt <= (uint64_t)a.n);
        }
        uint32_t incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        const uint32_t excl = incl - cnt;
        const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
        for (uint32_t j0 = 0; j0 < total; j0 += 32) {
            const uint32_t j = j0 + (uint32_t)lane;
            // the row holding flat index j: last lane with excl <= j
            int lo = 0;
#pragma unroll
            for (int step = 16; step; step >>= 1) {
                const uint32_t e = __shfl_sync(0xffffffffu, excl, lo + step);
                if (lo + step < 32 && e <= j) lo += step;
            }
            const uint32_t rb = __shfl_sync(0xffffffffu, b, lo);
            const uint32_t re = __shfl_sync(0xffffffffu, excl, lo);
            f(j < total ? rb + (j - re) : 0xFFFFFFFFu);
        }
    }
}

// Cyclic Jacobi eigen-decomposition of the symmetric K x K matrix in S.A
// (destroyed; its diagonal ends as the eigenvalues); eigenvectors -> S.V
// columns; sorted ascending into S.ev with S.V permuted accordingly.
__device__ __noinline__ void jacobi_eigen(WarpSmem& S, int K, int lane) {
    for (int i = lane; i < K * KS; i += 32) {
        const int r = i / KS, c = i % KS;
        if (c < K) S.V[i] = r == c ? 1.0 : 0.0;
    }
    __syncwarp();
    for (int sweep = 0; sweep < 60; ++sweep) {
        double off = 0.0, dia = 0.0;
        for (int i = lane; i < K * K; i += 32) {
            const int r = i / K, c = i % K;
            const double v = S.A[r * KS + c];
            if (r != c) off += v * v;
            else dia += v * v;
        }
        off = wsum(off);
        dia = wsum(dia);
        if (!(off > 1e-32 * dia)) break;  // off-diagonal mass at rounding level (or all zero)
        for (int p = 0; p < K - 1; ++p) {
            for (int q = p + 1; q < K; ++q) {
                const double apq = S.A[p * KS + q];
                if (apq == 0.0) continue;
                const double app = S.A[p * KS + p], aqq = S.A[q * KS + q];
                const double tau = (aqq - app) / (2.0 * apq);
                const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                const double c = 1.0 / sqrt(1.0 + t * t), s = t * c;
                __syncwarp();
                if (lane < K) {  // A <- A J (columns p, q)
                    const double akp = S.A[lane * KS + p], akq = S.A[lane * KS + q];
                    S.A[lane * KS + p] = c * akp - s * akq;
                    S.A[lane * KS + q] = s * akp + c * akq;
                    const double vkp = S.V[lane * KS + p], vkq = S.V[lane * KS + q];
                    S.V[lane * KS + p] = c * vkp - s * vkq;
                    S.V[lane * KS + q] = s * vkp + c * vkq;
                }
                __syncwarp();
                if (lane < K) {  // A <- J^T A (rows p, q)
                    const double apk = S.A[p * KS + lane], aqk = S.A[q * KS + lane];
                    S.A[p * KS + lane] = c * apk - s * aqk;
                    S.A[q * KS + lane] = s * apk + c * aqk;
                }
                __syncwarp();
                if (lane == 0) {
                    S.A[p * KS + q] = 0.0;
                    S.A[q * KS + p] = 0.0;
                }
                __syncwarp();
            }
        }
    }
    // ascending eigenvalues (stable selection by lane 0), eigenvectors permuted
    if (lane == 0) {
        for (int i = 0; i < K; ++i) S.perm[i] = i;
        for (int i = 0; i < K; ++i) {
            int best = i;
            for (int j = i + 1; j < K; ++j)
                if (S.A[S.perm[j] * KS + S.perm[j]] < S.A[S.perm[best] * KS + S.perm[best]]) best = j;
            const int t = S.perm[i];
            S.perm[i] = S.perm[best];
            S.perm[best] = t;
        }
        for (int i = 0; i < K; ++i) S.ev[i] = S.A[S.perm[i] * KS + S.perm[i]];
    }
    __syncwarp();
    // V columns in the sorted order (through A, which is free now)
    for (int i = lane; i < K * K; i += 32) {
        const int r = i / K, c = i % K;
        S.A[r * KS + c] = S.V[r * KS + S.perm[c]];
    }
    __syncwarp();
    for (int i = lane; i < K * K; i += 32) {
        const int r = i / K, c = i % K;
        S.V[r * KS + c] = S.A[r * KS + c];
    }
    __syncwarp();
}

// Symmetric 3 x 3 eigenproblem of the plane fit, every lane redundantly in
// registers (no shared memory, no warp barriers): cyclic Jacobi with the same
// rotation and stopping rule as jacobi_eigen.  a = {a00, a01, a02, a11, a12,
// a22}; returns the ascending eigenvalues and the eigenvector of the smallest.
struct Eig3 {
    double ev[3];
    double n[3];
};
template <int P, int Q, int R>
__device__ __forceinline__ void rot3(double (&A)[3][3], double (&V)[3][3]) {
    const double apq = A[P][Q];
    if (apq == 0.0) return;
    const double tau = (A[Q][Q] - A[P][P]) / (2.0 * apq);
    const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
    const double c = 1.0 / sqrt(1.0 + t * t), s = t * c;
    A[P][P] -= t * apq;
    A[Q][Q] += t * apq;
    A[P][Q] = A[Q][P] = 0.0;
    const double arp = A[R][P], arq = A[R][Q];
    A[R][P] = A[P][R] = c * arp - s * arq;
    A[R][Q] = A[Q][R] = s * arp + c * arq;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double vkp = V[k][P], vkq = V[k][Q];
        V[k][P] = c * vkp - s * vkq;
        V[k][Q] = s * vkp + c * vkq;
    }
}
// V: in, an orthonormal basis close to the eigenvectors (the previous plane
// iterate's; the identity at first) — the matrix is rotated into it, so the
// sweeps start from a nearly diagonal matrix (1-2 instead of ~5); out, the
// eigenvectors (columns).
__device__ __noinline__ Eig3 eig3(double a00, double a01, double a02, double a11, double a12,
                                  double a22, double (&V)[3][3]) {
    const double S[3][3] = {{a00, a01, a02}, {a01, a11, a12}, {a02, a12, a22}};
    double T[3][3], A[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)  // T = S V
#pragma unroll
        for (int j = 0; j < 3; ++j) T[i][j] = S[i][0] * V[0][j] + S[i][1] * V[1][j] + S[i][2] * V[2][j];
#pragma unroll
    for (int i = 0; i < 3; ++i)  // A = V^T T, symmetrised
#pragma unroll
        for (int j = i; j < 3; ++j)
            A[i][j] = A[j][i] = V[0][i] * T[0][j] + V[1][i] * T[1][j] + V[2][i] * T[2][j];
    for (int sweep = 0; sweep < 60; ++sweep) {
        const double off = 2.0 * (A[0][1] * A[0][1] + A[0][2] * A[0][2] + A[1][2] * A[1][2]);
        const double dia = A[0][0] * A[0][0] + A[1][1] * A[1][1] + A[2][2] * A[2][2];
        if (!(off > 1e-32 * dia)) break;
        rot3<0, 1, 2>(A, V);
        rot3<0, 2, 1>(A, V);
        rot3<1, 2, 0>(A, V);
    }
    // ascending eigenvalues, stable (ties keep the lower index first); selects, not
    // indexed reads, so that A and V stay in registers
    const double d0 = A[0][0], d1 = A[1][1], d2 = A[2][2];
    int i0 = 0;
    if (d1 < d0) i0 = 1;
    if (d2 < (i0 == 0 ? d0 : d1)) i0 = 2;
    const double lo = i0 == 0 ? d0 : (i0 == 1 ? d1 : d2);
    const double ra = i0 == 0 ? d1 : d0;  // the other two, lower index first
    const double rb = i0 == 2 ? d1 : d2;
    Eig3 e;
    e.ev[0] = lo;
    e.ev[1] = rb < ra ? rb : ra;
    e.ev[2] = rb < ra ? ra : rb;
#pragma unroll
    for (int k = 0; k < 3; ++k) e.n[k] = i0 == 0 ? V[k][0] : (i0 == 1 ? V[k][1] : V[k][2]);
    return e;
}

__device__ __forceinline__ void record_center(const MlsArgs& a, uint32_t qi, int slot, double x,
                                              double y, double z, double* cmn, double* cmx,
                                              int lane) {
    cmn[0] = fmin(cmn[0], x);
    cmn[1] = fmin(cmn[1], y);
    cmn[2] = fmin(cmn[2], z);
    cmx[0] = fmax(cmx[0], x);
    cmx[1] = fmax(cmx[1], y);
    cmx[2] = fmax(cmx[2], z);
    if (a.centers && lane == 0) {
        double* c = a.centers + ((size_t)qi * (size_t)(a.max_iter + 1) + (size_t)slot) * 3;
        c[0] = x;
        c[1] = y;
        c[2] = z;
    }
}

struct Frame {
    double o[3], n[3], u[3], v[3];
};

// Entry e of the packed normal system of a K-coefficient fit: the upper
// triangle of M row by row, then the right-hand side b (col -1).
__host__ __device__ constexpr int entry_row(int K, int e) {
    if (e >= K * (K + 1) / 2) return e - K * (K + 1) / 2;
    int r = 0;
    while (e >= K - r) {
        e -= K - r;
        ++r;
    }
    return r;
}
__host__ __device__ constexpr int entry_col(int K, int e) {
    if (e >= K * (K + 1) / 2) return -1;
    int r = 0;
    while (e >= K - r) {
        e -= K - r;
        ++r;
    }
    return r + e;
}

// The hit of candidate k for the frame F: local coordinates and weight
// (wls.cpp:183-188; distance = sqrt(norm2(p - origin))).
__device__ __forceinline__ bool frame_hit(const MlsArgs& a, const Frame& F, uint32_t k, double& ui,
                                          double& vi, double& fi, double& w) {
    if (k == 0xFFFFFFFFu) return false;
    const double4 p = a.pts[k];
    const double d2 = exact_d2(p.x, p.y, p.z, F.o[0], F.o[1], F.o[2]);
    if (!(d2 <= a.r2)) return false;
    const double dx = p.x - F.o[0], dy = p.y - F.o[1], dz = p.z - F.o[2];
    ui = __dadd_rn(__dadd_rn(__dmul_rn(dx, F.u[0]), __dmul_rn(dy, F.u[1])), __dmul_rn(dz, F.u[2]));
    vi = __dadd_rn(__dadd_rn(__dmul_rn(dx, F.v[0]), __dmul_rn(dy, F.v[1])), __dmul_rn(dz, F.v[2]));
    fi = __dadd_rn(__dadd_rn(__dmul_rn(dx, F.n[0]), __dmul_rn(dy, F.n[1])), __dmul_rn(dz, F.n[2]));
    w = theta_k(__dsqrt_rn(d2), a.support, a.inv_h);
    return true;
}

// Normal system of degree D <= 2 (K <= 6, 27 entries): every lane accumulates
// ITS hits into registers (entries fully unrolled), then one fixed xor-tree
// reduction per entry — no per-hit broadcast.  Returns the hit count.
template <int D>
__device__ __noinline__ int accum_lane(const MlsArgs& a, WarpSmem& S, const Frame& F, int lane) {
    constexpr int K = (D + 1) * (D + 2) / 2;
    constexpr int NE = K * (K + 1) / 2 + K;
    double acc[NE];
#pragma unroll
    for (int e = 0; e < NE; ++e) acc[e] = 0.0;
    int cnt = 0;
    for_candidates(a, F.o[0], F.o[1], F.o[2], lane, [&](uint32_t k) {
        double ui, vi, fi, w;
        if (!frame_hit(a, F, k, ui, vi, fi, w)) return;
        ++cnt;
        double up[D + 1], vp[D + 1], bs[K];
        up[0] = vp[0] = 1.0;
#pragma unroll
        for (int i = 1; i <= D; ++i) {
            up[i] = up[i - 1] * ui;
            vp[i] = vp[i - 1] * vi;
        }
        int kk = 0;
#pragma unroll
        for (int s = 0; s <= D; ++s)
#pragma unroll
            for (int e = s; e >= 0; --e) bs[kk++] = up[e] * vp[s - e];
#pragma unroll
        for (int e = 0; e < NE; ++e) {
            const int r = entry_row(K, e), c = entry_col(K, e);
            const double wb = w * bs[r];
            acc[e] += c >= 0 ? wb * bs[c] : wb * fi;
        }
    });
#pragma unroll
    for (int e = 0; e < NE; ++e) {
        const double v = wsum(acc[e]);
        const int r = entry_row(K, e), c = entry_col(K, e);
        if (lane == 0) {
            if (c >= 0) {
                S.M[r * KS + c] = v;
                S.M[c * KS + r] = v;
            } else {
                S.b[r] = v;
            }
        }
    }
    return wsumi(cnt);
}

// Normal system of degree 3 or 4 (K = 10, 15: up to 135 entries): each hit is
// broadcast to the warp and every lane accumulates the entries it owns.
__device__ __noinline__ int accum_bcast(const MlsArgs& a, WarpSmem& S, const Frame& F, int degree, int lane) {
    const int K = (degree + 1) * (degree + 2) / 2;
    const int NE = K * (K + 1) / 2 + K;  // packed upper triangle of M, then b
    // the entries this lane owns (e = lane + 32 t), as (row, col); col = -1: b[row]
    int er[5], ec[5];
#pragma unroll
    for (int t = 0; t < 5; ++t) {
        const int e = lane + 32 * t;
        er[t] = e < NE ? entry_row(K, e) : -1;
        ec[t] = e < NE ? entry_col(K, e) : -1;
    }
    double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    int cnt = 0;
    for_candidates(a, F.o[0], F.o[1], F.o[2], lane, [&](uint32_t k) {
        double ui = 0.0, vi = 0.0, fi = 0.0, w = 0.0;
        const bool hit = frame_hit(a, F, k, ui, vi, fi, w);
        cnt += hit ? 1 : 0;
        unsigned mask = __ballot_sync(0xffffffffu, hit);
        while (mask) {
            const int src = __ffs(mask) - 1;
            mask &= mask - 1;
            const double bu = __shfl_sync(0xffffffffu, ui, src);
            const double bv = __shfl_sync(0xffffffffu, vi, src);
            const double bf = __shfl_sync(0xffffffffu, fi, src);
            const double bw = __shfl_sync(0xffffffffu, w, src);
            double up[5], vp[5], basis[KMAX];
            up[0] = vp[0] = 1.0;
            for (int i = 1; i <= degree; ++i) {
                up[i] = up[i - 1] * bu;
                vp[i] = vp[i - 1] * bv;
            }
            int kk = 0;
            for (int s = 0; s <= degree; ++s)
                for (int e = s; e >= 0; --e) basis[kk++] = up[e] * vp[s - e];
#pragma unroll
            for (int t = 0; t < 5; ++t) {
                if (er[t] < 0) continue;
                const double wb = bw * basis[er[t]];
                acc[t] += ec[t] >= 0 ? wb * basis[ec[t]] : wb * bf;
            }
        }
    });
#pragma unroll
    for (int t = 0; t < 5; ++t) {
        if (er[t] < 0) continue;
        if (ec[t] >= 0) {
            S.M[er[t] * KS + ec[t]] = acc[t];
            S.M[ec[t] * KS + er[t]] = acc[t];
        } else {
            S.b[er[t]] = acc[t];
        }
    }
    return wsumi(cnt);
}

// fit_local_polynomial (wls.cpp:149-222) of `degree` over frame F; coefficients
// in S.x on success.
__device__ __noinline__ int poly_fit(const MlsArgs& a, WarpSmem& S, const Frame& F, int degree, int lane) {
    const int K = (degree + 1) * (degree + 2) / 2;
    const int cnt = degree == 1 ? accum_lane<1>(a, S, F, lane)
                  : degree == 2 ? accum_lane<2>(a, S, F, lane)
                                : accum_bcast(a, S, F, degree, lane);
    if (cnt < K) return YF_TOO_FEW;
    __syncwarp();
    for (int i = lane; i < K * KS; i += 32) S.A[i] = S.M[i];
    __syncwarp();
    jacobi_eigen(S, K, lane);
    const double lmax = S.ev[K - 1];
    if (!(lmax > 0.0) || S.ev[0] <= 1e-12 * lmax) return YF_SINGULAR;
    // coeffs = V (V^T b ./ l); one refinement with the residual b - M coeffs
    for (int pass = 0; pass < 2; ++pass) {
        double tmp = 0.0;
        if (lane < K) {  // (V^T rhs) ./ l, rhs = b, then the residual in S.y
            for (int k = 0; k < K; ++k) tmp += S.V[k * KS + lane] * (pass == 0 ? S.b[k] : S.y[k]);
            tmp = tmp / S.ev[lane];
        }
        __syncwarp();
        if (lane < K) S.A[lane] = tmp;
        __syncwarp();
        if (lane < K) {
            double s = 0.0;
            for (int j = 0; j < K; ++j) s += S.V[lane * KS + j] * S.A[j];
            S.x[lane] = pass == 0 ? s : S.x[lane] + s;
        }
        __syncwarp();
        if (pass == 0 && lane < K) {  // residual
            double s = 0.0;
            for (int j = 0; j < K; ++j) s += S.M[lane * KS + j] * S.x[j];
            S.y[lane] = S.b[lane] - s;
        }
        __syncwarp();
    }
    return YF_OK;
}

#ifndef PCSB_MLS_MINB
#define PCSB_MLS_MINB 8  // 64 registers: 233 -> 196 ms on the 1M-point sphere (6: 209, 5: 233)
#endif
// PH = 0: the whole projection in one launch.  The lean smooth_cloud path runs it
// as two launches — PH = 1: the plane fit (results to a.mid), PH = 2: the degree
// ladder over the stored frames — so that each launch's warps walk a code body
// half the size (the kernel's dominant stall is instruction fetch).
#ifndef PCSB_MLS_MINB_POLY
#define PCSB_MLS_MINB_POLY 5  // polynomial launch: 5 blocks/SM 35.8 ms, 4: 37.8, 8: 37.7, 3: 43.4
#endif
template <int PH>
__global__ void __launch_bounds__(MLS_THREADS, PH == 1 ? PCSB_MLS_MINB : PCSB_MLS_MINB_POLY)
mls_kernel(const MlsArgs a) {
    __shared__ WarpSmem smem[MLS_WARPS];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    WarpSmem& S = smem[warp];
    for (;;) {
        uint32_t qi = 0;
        if (lane == 0) qi = atomicAdd(a.counter, 1u);
        qi = __shfl_sync(0xffffffffu, qi, 0);
        if (qi >= a.m) break;
        double rx, ry, rz;
        if (PH != 0) {  // the lean path's launches: the cloud's own sorted points
            const double4 self = a.pts[qi];
            rx = self.x;
            ry = self.y;
            rz = self.z;
        } else {
            rx = a.q[3 * (size_t)qi];
            ry = a.q[3 * (size_t)qi + 1];
            rz = a.q[3 * (size_t)qi + 2];
        }
        pcs_mls_result R;
        memset(&R, 0, sizeof(R));
        R.projected[0] = rx;
        R.projected[1] = ry;
        R.projected[2] = rz;
        R.status = PS_SKIPPED;
        double cmn[3] = {INFINITY, INFINITY, INFINITY}, cmx[3] = {-INFINITY, -INFINITY, -INFINITY};
        Frame F;
        bool have_frame = false;

        if (PH == 2) {
            const MlsMid& M = a.mid[qi];
            for (int i = 0; i < 3; ++i) {
                F.o[i] = M.o[i];
                F.n[i] = M.n[i];
                F.u[i] = M.u[i];
                F.v[i] = M.v[i];
            }
            for (int i = 0; i < 3; ++i) {
                cmn[i] = M.cmn[i];
                cmx[i] = M.cmx[i];
            }
            R.iterations = M.iterations;
            R.plane_status = M.plane_status;
            have_frame = M.have_frame != 0;
        } else if (a.mode == PCS_MLS_POLY) {
            const double* fr = a.frames + 12 * (size_t)qi;
            for (int i = 0; i < 3; ++i) {
                F.o[i] = fr[i];
                F.n[i] = fr[3 + i];
                F.u[i] = fr[6 + i];
                F.v[i] = fr[9 + i];
            }
            have_frame = true;
        } else {
            // ---------------- reference plane (wls.cpp:53-147) ----------------
            double qx = rx, qy = ry, qz = rz;
            double nx = 0.0, ny = 0.0, nz = 0.0, t = 0.0;
            bool converged = false;
            int pstatus = PF_OK;
            double EV[3][3] = {{1.0, 0.0, 0.0}, {0.0, 1.0, 0.0}, {0.0, 0.0, 1.0}};  // eig3's basis
            for (int iter = 1; iter <= a.max_iter; ++iter) {
                R.iterations = iter;
                record_center(a, qi, iter - 1, qx, qy, qz, cmn, cmx, lane);
                // one pass over the neighbourhood: weight, first and second moments
                // about the iterate q; the covariance about the centroid c follows as
                // sum w (p-q)(p-q)^T - sw (c-q)(c-q)^T  (|c - q| is of the order of
                // the neighbourhood's spread, so nothing cancels beyond a few ulps;
                // wls.cpp:70-101 makes a centroid pass and a covariance pass)
                int cnt = 0;
                double sw = 0.0, sx = 0.0, sy = 0.0, sz = 0.0;
                double c00 = 0.0, c01 = 0.0, c02 = 0.0, c11 = 0.0, c12 = 0.0, c22 = 0.0;
                for_candidates(a, qx, qy, qz, lane, [&](uint32_t k) {
                    if (k == 0xFFFFFFFFu) return;
                    const double4 p = a.pts[k];
                    const double d2 = exact_d2(p.x, p.y, p.z, qx, qy, qz);
                    if (!(d2 <= a.r2)) return;
                    const double w = theta_k(__dsqrt_rn(d2), a.support, a.inv_h);
                    const double dx = p.x - qx, dy = p.y - qy, dz = p.z - qz;
                    const double wx = w * dx, wy = w * dy, wz = w * dz;
                    ++cnt;
                    sw += w;
                    sx += wx;
                    sy += wy;
                    sz += wz;
                    c00 += wx * dx;
                    c01 += wx * dy;
                    c02 += wx * dz;
                    c11 += wy * dy;
                    c12 += wy * dz;
                    c22 += wz * dz;
                });
                cnt = wsumi(cnt);
                sw = wsum(sw);
                if (cnt < 3 || !(sw > 0.0)) {
                    pstatus = PF_TOO_FEW;
                    break;
                }
                const double ox = wsum(sx) / sw, oy = wsum(sy) / sw, oz = wsum(sz) / sw;  // c - q
                const double cx = qx + ox, cy = qy + oy, cz = qz + oz;
                c00 = wsum(c00) - sw * ox * ox;
                c01 = wsum(c01) - sw * ox * oy;
                c02 = wsum(c02) - sw * ox * oz;
                c11 = wsum(c11) - sw * oy * oy;
                c12 = wsum(c12) - sw * oy * oz;
                c22 = wsum(c22) - sw * oz * oz;
                const Eig3 e3 = eig3(c00, c01, c02, c11, c12, c22, EV);
                if (e3.ev[1] - e3.ev[0] <= 1e-12 * e3.ev[2]) {
                    pstatus = PF_DEGENERATE;
                    break;
                }
                nx = e3.n[0];
                ny = e3.n[1];
                nz = e3.n[2];
                const double nn = sqrt(nx * nx + ny * ny + nz * nz);
                nx /= nn;
                ny /= nn;
                nz /= nn;
                t = nx * (cx - rx) + ny * (cy - ry) + nz * (cz - rz);
                const double qnx = rx + t * nx, qny = ry + t * ny, qnz = rz + t * nz;
                const double ddx = qnx - qx, ddy = qny - qy, ddz = qnz - qz;
                const double step = sqrt(ddx * ddx + ddy * ddy + ddz * ddz);
                qx = qnx;
                qy = qny;
                qz = qnz;
                if (step < a.tol) {
                    converged = true;
                    break;
                }
            }
            R.plane_status = pstatus;
            if (pstatus == PF_OK) {
                // <n, r - q> = -t: flip when t > 0; on a tie, positive z, then y, then x
                if (t > 0.0) {
                    nx = -nx;
                    ny = -ny;
                    nz = -nz;
                } else if (t == 0.0) {
                    const bool flip = nz != 0.0 ? nz < 0.0 : (ny != 0.0 ? ny < 0.0 : nx < 0.0);
                    if (flip) {
                        nx = -nx;
                        ny = -ny;
                        nz = -nz;
                    }
                }
                F.o[0] = qx; F.o[1] = qy; F.o[2] = qz;
                F.n[0] = nx; F.n[1] = ny; F.n[2] = nz;
                // u: Gram-Schmidt of the least aligned axis (ties x, y, z); v = n x u
                const double ax = fabs(nx), ay = fabs(ny), az = fabs(nz);
                double e0 = 1.0, e1 = 0.0, e2 = 0.0, best = ax;
                if (ay < best) { e0 = 0.0; e1 = 1.0; e2 = 0.0; best = ay; }
                if (az < best) { e0 = 0.0; e1 = 0.0; e2 = 1.0; }
                const double en = e0 * nx + e1 * ny + e2 * nz;
                double ux = e0 - en * nx, uy = e1 - en * ny, uz = e2 - en * nz;
                const double un = sqrt(ux * ux + uy * uy + uz * uz);
                ux /= un; uy /= un; uz /= un;
                F.u[0] = ux; F.u[1] = uy; F.u[2] = uz;
                F.v[0] = ny * uz - nz * uy;
                F.v[1] = nz * ux - nx * uz;
                F.v[2] = nx * uy - ny * ux;
                R.plane_status = converged ? PF_OK : PF_NO_CONV;
                have_frame = true;
            }
        }
        if (PH == 1) {
            if (lane == 0) {
                MlsMid M;
                for (int i = 0; i < 3; ++i) {
                    M.o[i] = have_frame ? F.o[i] : 0.0;
                    M.n[i] = have_frame ? F.n[i] : 0.0;
                    M.u[i] = have_frame ? F.u[i] : 0.0;
                    M.v[i] = have_frame ? F.v[i] : 0.0;
                    M.cmn[i] = cmn[i];
                    M.cmx[i] = cmx[i];
                }
                M.iterations = R.iterations;
                M.plane_status = R.plane_status;
                M.have_frame = have_frame ? 1 : 0;
                M.pad = 0;
                a.mid[qi] = M;
            }
            __syncwarp();
            continue;
        }
        if (have_frame) {
            if (PH != 2) {
                for (int i = 0; i < 3; ++i) {
                    R.origin[i] = F.o[i];
                    R.normal[i] = F.n[i];
                    R.u[i] = F.u[i];
                    R.v[i] = F.v[i];
                }
            }
            if (PH != 2 && a.mode == PCS_MLS_POLY) {
                record_center(a, qi, 0, F.o[0], F.o[1], F.o[2], cmn, cmx, lane);
                const int st = poly_fit(a, S, F, a.degree, lane);
                R.poly_status = st;
                if (st == YF_OK) {
                    R.degree_used = a.degree;
                    const int K = (a.degree + 1) * (a.degree + 2) / 2;
                    for (int k = 0; k < K; ++k) R.coeffs[k] = S.x[k];
                }
            } else if (PH == 2 || a.mode == PCS_MLS_PROJECT) {
                // ---------------- degree ladder (mls.cpp:48-68) ----------------
                record_center(a, qi, R.iterations, F.o[0], F.o[1], F.o[2], cmn, cmx, lane);
                R.projected[0] = F.o[0];
                R.projected[1] = F.o[1];
                R.projected[2] = F.o[2];
                R.status = PS_PLANE_ONLY;
                for (int deg = a.degree; deg >= 1; --deg) {
                    const int st = poly_fit(a, S, F, deg, lane);
                    R.poly_status = st;
                    if (st == YF_OK) {
                        if (PH != 2) {
                            const int K = (deg + 1) * (deg + 2) / 2;
                            for (int k = 0; k < K; ++k) R.coeffs[k] = S.x[k];
                        }
                        // evaluate_polynomial(poly, 0, 0) = c0 + c1*0 + ... = c0
                        const double hgt = S.x[0];
                        R.projected[0] = __dadd_rn(F.o[0], __dmul_rn(hgt, F.n[0]));
                        R.projected[1] = __dadd_rn(F.o[1], __dmul_rn(hgt, F.n[1]));
                        R.projected[2] = __dadd_rn(F.o[2], __dmul_rn(hgt, F.n[2]));
                        R.status = deg == a.degree ? PS_FULL : PS_DEGRADED;
                        R.degree_used = deg;
                        break;
                    }
                }
            }
        }
        for (int i = 0; i < 3; ++i) {
            R.cmin[i] = cmn[i];
            R.cmax[i] = cmx[i];
        }
        if (lane == 0) {
            if (PH == 2) {  // (R never leaves the registers in this launch)
                const size_t oi = a.order[qi];
                a.lean_xyz[3 * oi] = R.projected[0];
                a.lean_xyz[3 * oi + 1] = R.projected[1];
                a.lean_xyz[3 * oi + 2] = R.projected[2];
                pcs_mls_outcome o;
                o.status = (int8_t)R.status;
                o.degree_used = (int8_t)R.degree_used;
                o.plane_status = (int8_t)R.plane_status;
                o.poly_status = (int8_t)R.poly_status;
                o.iterations = R.iterations;
                a.lean_out[oi] = o;
                if (a.lean_bounds) {
                    for (int i = 0; i < 3; ++i) {
                        a.lean_bounds[6 * oi + i] = cmn[i];
                        a.lean_bounds[6 * oi + 3 + i] = cmx[i];
                    }
                }
            } else {
                a.out[qi] = R;
            }
        }
        __syncwarp();
    }
}

// Isotropic grid for radius queries of radius `support` over [lo, hi]: cell
// side support / 2, coarsened (doubled) until the table holds at most
// max(8n, 2^16) cells (<= 2^27).
GridGeom mls_grid(const double lo[3], const double hi[3], double support, uint64_t n) {
    double cs = support * 0.5;
    const double cap = std::min(std::max(8.0 * (double)n, 65536.0), (double)(1u << 27));
    auto cells = [&](double c) {
        double v = 1.0;
        for (int ax = 0; ax < 3; ++ax) v *= std::floor((hi[ax] - lo[ax]) / c) + 3.0;
        return v;
    };
    while (cells(cs) > cap) cs *= 2.0;
    GridGeom g{};
    g.cs = cs;
    g.inv_cs = 1.0 / cs;
    g.xsub = 1;
    g.csx = cs;
    g.inv_csx = g.inv_cs;
    g.ox = lo[0] - cs;
    g.oy = lo[1] - cs;
    g.oz = lo[2] - cs;
    g.gx = (int32_t)std::floor((hi[0] - g.ox) * g.inv_cs) + 2;
    g.gy = (int32_t)std::floor((hi[1] - g.oy) * g.inv_cs) + 2;
    g.gz = (int32_t)std::floor((hi[2] - g.oz) * g.inv_cs) + 2;
    g.sub_bits = 0;
    g.ncells = (uint32_t)g.gx * (uint32_t)g.gy * (uint32_t)g.gz;
    int b = 0;
    while (b < 32 && (1ull << b) < (uint64_t)g.ncells) ++b;
    g.key_bits = std::max(1, b);
    return g;
}

}  // namespace

// The device index of one cloud (pcs_mls_index).
struct MlsIndex {
    int device = 0;
    uint64_t n = 0;
    cudaStream_t s = nullptr;
    double* xyz = nullptr;      // original order
    double4* pts = nullptr;     // original order
    double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0}, maxabs = 0.0;
    std::vector<void*> allocs;  // the cached grid's buffers
    // cached grid
    double grid_support = -1.0;
    GridGeom g{};
    double4* sorted = nullptr;
    uint32_t* order = nullptr;
    uint32_t* start = nullptr;
    std::mutex mu;

    void* galloc(size_t b) {
        void* p = nullptr;
        p = pool_alloc(device, b, s);
        allocs.push_back(p);
        return p;
    }
    void free_grid() {
        for (void* p : allocs) pool_free(p, s);
        allocs.clear();
        grid_support = -1.0;
    }
    ~MlsIndex() {
        if (s) cudaStreamSynchronize(s);
        free_grid();
        pool_free(xyz, s);
        pool_free(pts, s);
        if (s) {
            cudaStreamSynchronize(s);
            cudaStreamDestroy(s);
        }
    }
    // the grid for radius `support` (built on first use, then cached)
    void ensure_grid(double support) {
        if (grid_support == support) return;
        free_grid();
        g = mls_grid(lo, hi, support, n);
        const uint32_t nn = (uint32_t)n;
        uint32_t* keys = (uint32_t*)galloc(n * 4);
        uint32_t* skeys = (uint32_t*)galloc(n * 4);
        order = (uint32_t*)galloc(n * 4);
        sorted = (double4*)galloc(n * sizeof(double4));
        start = (uint32_t*)galloc(((size_t)g.ncells + 1) * 4);
        RadixScratch rs;
        rs.keys_alt = (uint32_t*)galloc(n * 4);
        rs.vals_alt = (uint32_t*)galloc(n * 4);
        rs.blockhist = (uint32_t*)galloc(radix_blockhist_entries(nn) * 4);
        rs.capacity = nn;
        uint32_t* cscr = (uint32_t*)galloc(cell_scan_scratch_entries(g.ncells) * 4);
        launch_keys<double>(g, pts, nn, keys, nullptr, s);
        radix_sort(keys, nullptr, skeys, order, nn, g.key_bits, rs, nullptr, s);
        launch_gather<double>(pts, order, nn, sorted, nullptr, s);
        build_cell_start(skeys, nn, 0, g.ncells, start, cscr, nullptr, s);
        PCSB_CUDA(cudaStreamSynchronize(s));
        PCSB_CUDA(cudaGetLastError());
        grid_support = support;
    }
};

MlsIndex* mls_index_create(const double* xyz, uint64_t n, int device) {
    if (n > 0xFFFFFFFEull) throw Failure(PCS_ERR_INVALID_PARAM, "MLS index: at most 2^32-2 points");
    if (n && !xyz) throw Failure(PCS_ERR_INVALID_PARAM, "null buffer");
    std::unique_ptr<MlsIndex> ix(new MlsIndex);
    ix->device = select_device(device);
    ix->n = n;
    PCSB_CUDA(cudaStreamCreateWithFlags(&ix->s, cudaStreamNonBlocking));
    if (n) {
        ix->xyz = (double*)pool_alloc(ix->device, n * 3 * sizeof(double), ix->s);
        ix->pts = (double4*)pool_alloc(ix->device, n * sizeof(double4), ix->s);
        h2d_staged(ix->xyz, xyz, n * 3 * sizeof(double), ix->s);
        launch_convert_xyz<double>(ix->xyz, ix->pts, n, 1.0, ix->s);
        unsigned long long* slots =
            (unsigned long long*)pool_alloc(ix->device, 8 * sizeof(unsigned long long), ix->s);
        init_bbox_slots(slots, ix->s);
        launch_bbox<double>(ix->pts, n, slots, ix->s);
        unsigned long long hb[6];
        PCSB_CUDA(cudaMemcpyAsync(hb, slots, sizeof(hb), cudaMemcpyDeviceToHost, ix->s));
        PCSB_CUDA(cudaStreamSynchronize(ix->s));
        pool_free(slots, ix->s);
        for (int a = 0; a < 3; ++a) {
            ix->lo[a] = ordered_to_double(hb[a]);
            ix->hi[a] = ordered_to_double(hb[3 + a]);
            if (!std::isfinite(ix->lo[a]) || !std::isfinite(ix->hi[a]))
                throw Failure(PCS_ERR_INVALID_PARAM, "MLS index: coordinates must be finite");
            ix->maxabs = std::max(ix->maxabs, std::max(std::fabs(ix->lo[a]), std::fabs(ix->hi[a])));
        }
    }
    return ix.release();
}

void mls_index_destroy(MlsIndex* ix) { delete ix; }

namespace {
struct DevTmp {  // stream-ordered temporaries of one call (library pool)
    int dev;
    cudaStream_t s;
    std::vector<void*> p;
    DevTmp(int dev_, cudaStream_t s_) : dev(dev_), s(s_) {}
    ~DevTmp() {
        for (void* x : p) pool_free(x, s);
    }
    template <typename X>
    X* get(size_t count) {
        void* x = pool_alloc(dev, std::max<size_t>(count * sizeof(X), 16), s);
        p.push_back(x);
        return (X*)x;
    }
};
}  // namespace

void mls_index_radius(MlsIndex* ix, const double* centers, uint64_t m, double r, uint64_t* offsets,
                      uint32_t* idx, double* dist, uint64_t cap) {
    if (!(r > 0.0) || !std::isfinite(r))
        throw Failure(PCS_ERR_INVALID_PARAM, "radius_query requires finite r > 0");
    if (!offsets) throw Failure(PCS_ERR_INVALID_PARAM, "null buffer");
    std::lock_guard<std::mutex> lk(ix->mu);
    PCSB_CUDA(cudaSetDevice(ix->device));
    if (m == 0 || ix->n == 0) {
        for (uint64_t i = 0; i <= m; ++i) offsets[i] = 0;
        return;
    }
    if (m > 0xFFFFFFFEull) throw Failure(PCS_ERR_INVALID_PARAM, "radius_query: too many centres");
    ix->ensure_grid(r);
    DevTmp t(ix->device, ix->s);
    double* dQ = t.get<double>(m * 3);
    PCSB_CUDA(cudaMemcpyAsync(dQ, centers, m * 3 * sizeof(double), cudaMemcpyHostToDevice, ix->s));
    uint64_t* cnt = t.get<uint64_t>(m + 1);
    const double s_pad = r * (1.0 + 1e-12) + 4.0 * std::ldexp(ix->maxabs + r + 1.0, -52);
    launch_radius_dump<double>(ix->sorted, ix->order, ix->start, ix->g, dQ, (uint32_t)m, r, s_pad,
                               cnt, nullptr, ix->s);
    std::vector<uint64_t> hc(m);
    PCSB_CUDA(cudaMemcpyAsync(hc.data(), cnt, m * sizeof(uint64_t), cudaMemcpyDeviceToHost, ix->s));
    PCSB_CUDA(cudaStreamSynchronize(ix->s));
    offsets[0] = 0;
    for (uint64_t i = 0; i < m; ++i) offsets[i + 1] = offsets[i] + hc[i];
    const uint64_t total = offsets[m];
    if (!idx) return;
    if (cap < total) throw Failure(PCS_ERR_CAPACITY, "radius_query: idx capacity too small");
    if (total == 0) return;
    PCSB_CUDA(cudaMemcpyAsync(cnt, offsets, m * sizeof(uint64_t), cudaMemcpyHostToDevice, ix->s));
    uint32_t* didx = t.get<uint32_t>(total);
    launch_radius_dump<double>(ix->sorted, ix->order, ix->start, ix->g, dQ, (uint32_t)m, r, s_pad,
                               cnt, didx, ix->s);
    PCSB_CUDA(cudaMemcpyAsync(idx, didx, total * sizeof(uint32_t), cudaMemcpyDeviceToHost, ix->s));
    PCSB_CUDA(cudaStreamSynchronize(ix->s));
    PCSB_CUDA(cudaGetLastError());
}

void mls_project(MlsIndex* ix, const pcs_mls_desc& d, const double* q, uint64_t m, int mode,
                 const double* frames, pcs_mls_result* out, double* centers_out) {
    if (!(d.h > 0.0) || !std::isfinite(d.h))
        throw Failure(PCS_ERR_INVALID_PARAM, "KernelParams: h must be positive and finite");
    if (!(d.cutoff_multiple > 0.0) || !std::isfinite(d.cutoff_multiple))
        throw Failure(PCS_ERR_INVALID_PARAM, "KernelParams: cutoff_multiple must be positive and finite");
    if (d.degree < 1 || d.degree > 4)
        throw Failure(PCS_ERR_INVALID_PARAM, "MlsParams: degree must be in [1,4]");
    if (!(d.plane_tol > 0.0))
        throw Failure(PCS_ERR_INVALID_PARAM, "MlsParams: plane_tol must be positive");
    if (d.plane_max_iter < 1)
        throw Failure(PCS_ERR_INVALID_PARAM, "MlsParams: plane_max_iter must be >= 1");
    if (mode < PCS_MLS_PROJECT || mode > PCS_MLS_POLY)
        throw Failure(PCS_ERR_INVALID_PARAM, "pcs_mls_project: unknown mode");
    if (m == 0) return;
    if (!q || !out || (mode == PCS_MLS_POLY && !frames))
        throw Failure(PCS_ERR_INVALID_PARAM, "null buffer");
    if (m > 0xFFFFFFFEull) throw Failure(PCS_ERR_INVALID_PARAM, "pcs_mls_project: too many queries");
    std::lock_guard<std::mutex> lk(ix->mu);
    PCSB_CUDA(cudaSetDevice(ix->device));
    const double support = d.h * d.cutoff_multiple;
    if (ix->n == 0) {
        // no data: every query is skipped (TooFewNeighbors at iteration 1)
        for (uint64_t i = 0; i < m; ++i) {
            pcs_mls_result R;
            std::memset(&R, 0, sizeof(R));
            for (int a = 0; a < 3; ++a) {
                R.projected[a] = q[3 * i + a];
                R.cmin[a] = R.cmax[a] = mode == PCS_MLS_POLY ? frames[12 * i + a] : q[3 * i + a];
            }
            if (mode == PCS_MLS_POLY) {
                R.poly_status = YF_TOO_FEW;
            } else {
                R.status = PS_SKIPPED;
                R.iterations = 1;
                R.plane_status = PF_TOO_FEW;
                if (centers_out)
                    for (int a = 0; a < 3; ++a) centers_out[i * (size_t)(d.plane_max_iter + 1) * 3 + a] = q[3 * i + a];
            }
            out[i] = R;
        }
        return;
    }
    ix->ensure_grid(support);
    DevTmp t(ix->device, ix->s);
    MlsArgs a{};
    a.pts = ix->sorted;
    a.start = ix->start;
    a.n = (uint32_t)ix->n;
    a.g = ix->g;
    a.support = support;
    a.r2 = support * support;
    a.s_pad = support * (1.0 + 1e-12) + 4.0 * std::ldexp(ix->maxabs + support + 1.0, -52);
    a.h = d.h;
    a.inv_h = 1.0 / d.h;
    double* dq = t.get<double>(m * 3);
    PCSB_CUDA(cudaMemcpyAsync(dq, q, m * 3 * sizeof(double), cudaMemcpyHostToDevice, ix->s));
    a.q = dq;
    a.m = (uint32_t)m;
    a.mode = mode;
    a.degree = d.degree;
    a.tol = d.plane_tol;
    a.max_iter = d.plane_max_iter;
    if (mode == PCS_MLS_POLY) {
        double* df = t.get<double>(m * 12);
        PCSB_CUDA(cudaMemcpyAsync(df, frames, m * 12 * sizeof(double), cudaMemcpyHostToDevice, ix->s));
        a.frames = df;
    }
    a.out = t.get<pcs_mls_result>(m);
    const size_t ncen = (size_t)m * (size_t)(d.plane_max_iter + 1) * 3;
    if (centers_out) a.centers = t.get<double>(ncen);
    a.counter = t.get<uint32_t>(1);
    PCSB_CUDA(cudaMemsetAsync(a.counter, 0, sizeof(uint32_t), ix->s));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ix->device);
    const uint64_t want = (m + MLS_WARPS - 1) / MLS_WARPS;
    const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>(want, (uint64_t)sms * 8));
    mls_kernel<0><<<grid, MLS_THREADS, 0, ix->s>>>(a);
    PCSB_CUDA(cudaGetLastError());
    PCSB_CUDA(cudaMemcpyAsync(out, a.out, m * sizeof(pcs_mls_result), cudaMemcpyDeviceToHost, ix->s));
    if (centers_out)
        PCSB_CUDA(cudaMemcpyAsync(centers_out, a.centers, ncen * sizeof(double), cudaMemcpyDeviceToHost,
                                  ix->s));
    PCSB_CUDA(cudaStreamSynchronize(ix->s));
    PCSB_CUDA(cudaGetLastError());
}

namespace {
std::mutex g_last_mu;
double g_last_ms[2] = {0.0, 0.0};  // plane / polynomial launch of the last smooth_cloud call
}  // namespace

// smooth_cloud without the per-point records: the queries are the index's own
// sorted points (no second upload; consecutive warps work on neighbouring
// points), 32 bytes per point come back instead of 312.
void mls_smooth_outcomes(const pcs_mls_desc& d, const double* xyz, uint64_t n, double* out_xyz,
                         pcs_mls_outcome* outcomes, double* center_bounds) {
    if (n == 0) return;
    if (!xyz || !out_xyz || !outcomes) throw Failure(PCS_ERR_INVALID_PARAM, "null buffer");
    // parameter checks of mls_project (same messages): a zero-query call validates only
    mls_project(nullptr, d, nullptr, 0, PCS_MLS_PROJECT, nullptr, nullptr, nullptr);
    std::unique_ptr<MlsIndex> ix(mls_index_create(xyz, n, d.device));
    std::lock_guard<std::mutex> lk(ix->mu);
    PCSB_CUDA(cudaSetDevice(ix->device));
    const double support = d.h * d.cutoff_multiple;
    ix->ensure_grid(support);
    DevTmp t(ix->device, ix->s);
    MlsArgs a{};
    a.pts = ix->sorted;
    a.start = ix->start;
    a.n = (uint32_t)ix->n;
    a.g = ix->g;
    a.support = support;
    a.r2 = support * support;
    a.s_pad = support * (1.0 + 1e-12) + 4.0 * std::ldexp(ix->maxabs + support + 1.0, -52);
    a.h = d.h;
    a.inv_h = 1.0 / d.h;
    a.m = (uint32_t)n;
    a.mode = PCS_MLS_PROJECT;
    a.degree = d.degree;
    a.tol = d.plane_tol;
    a.max_iter = d.plane_max_iter;
    a.order = ix->order;
    a.lean_xyz = t.get<double>(n * 3);
    a.lean_out = t.get<pcs_mls_outcome>(n);
    a.lean_bounds = center_bounds ? t.get<double>(n * 6) : nullptr;
    a.counter = t.get<uint32_t>(1);
    PCSB_CUDA(cudaMemsetAsync(a.counter, 0, sizeof(uint32_t), ix->s));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ix->device);
    const uint64_t want = (n + MLS_WARPS - 1) / MLS_WARPS;
    const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>(want, (uint64_t)sms * 8));
    a.mid = t.get<MlsMid>(n);
    cudaEvent_t ev[3];
    for (auto& e : ev) PCSB_CUDA(cudaEventCreate(&e));
    PCSB_CUDA(cudaEventRecord(ev[0], ix->s));
    mls_kernel<1><<<grid, MLS_THREADS, 0, ix->s>>>(a);
    PCSB_CUDA(cudaEventRecord(ev[1], ix->s));
    PCSB_CUDA(cudaMemsetAsync(a.counter, 0, sizeof(uint32_t), ix->s));
    mls_kernel<2><<<grid, MLS_THREADS, 0, ix->s>>>(a);
    PCSB_CUDA(cudaEventRecord(ev[2], ix->s));
    PCSB_CUDA(cudaGetLastError());
    PCSB_CUDA(cudaMemcpyAsync(out_xyz, a.lean_xyz, n * 3 * sizeof(double), cudaMemcpyDeviceToHost, ix->s));
    PCSB_CUDA(cudaMemcpyAsync(outcomes, a.lean_out, n * sizeof(pcs_mls_outcome), cudaMemcpyDeviceToHost,
                              ix->s));
    if (center_bounds)
        PCSB_CUDA(cudaMemcpyAsync(center_bounds, a.lean_bounds, n * 6 * sizeof(double),
                                  cudaMemcpyDeviceToHost, ix->s));
    PCSB_CUDA(cudaStreamSynchronize(ix->s));
    PCSB_CUDA(cudaGetLastError());
    {   // device time of the two launches (pcs_mls_last_device_ms)
        float plane = 0.f, poly = 0.f;
        cudaEventElapsedTime(&plane, ev[0], ev[1]);
        cudaEventElapsedTime(&poly, ev[1], ev[2]);
        std::lock_guard<std::mutex> g(g_last_mu);
        g_last_ms[0] = plane;
        g_last_ms[1] = poly;
    }
    for (auto& e : ev) cudaEventDestroy(e);
}

void mls_last_device_ms(double out[2]) {
    std::lock_guard<std::mutex> g(g_last_mu);
    out[0] = g_last_ms[0];
    out[1] = g_last_ms[1];
}

void mls_smooth(const pcs_mls_desc& d, const double* xyz, uint64_t n, double* out_xyz,
                pcs_mls_result* results) {
    if (n == 0) return;
    if (!xyz || !out_xyz) throw Failure(PCS_ERR_INVALID_PARAM, "null buffer");
    if (!results) {  // only the cloud is wanted: the two-launch path (same projections)
        std::vector<pcs_mls_outcome> oc(n);
        mls_smooth_outcomes(d, xyz, n, out_xyz, oc.data(), nullptr);
        return;
    }
    std::unique_ptr<MlsIndex> ix(mls_index_create(xyz, n, d.device));
    pcs_mls_result* R = results;
    mls_project(ix.get(), d, xyz, n, PCS_MLS_PROJECT, nullptr, R, nullptr);
    for (uint64_t i = 0; i < n; ++i)
        for (int a = 0; a < 3; ++a) out_xyz[3 * i + a] = R[i].projected[a];
}

// partition (proj/src/parallel.cpp:64-127): longest bounding-box axis (ties
// keep the lower axis), points sorted by (coordinate, index), equal counts
// (the first N mod W slabs one larger), cuts midway between facing
// coordinates (the bbox edge for empty trailing slabs).
void mls_partition(const double* xyz, uint64_t n, uint64_t workers, double support, int32_t* axis_out,
                   double* cuts, uint32_t* worker_of) {
    if (workers < 1) throw Failure(PCS_ERR_INVALID_PARAM, "partition: workers must be >= 1");
    if (!(support > 0.0)) throw Failure(PCS_ERR_INVALID_PARAM, "partition: support must be positive");
    if (n == 0) throw Failure(PCS_ERR_EMPTY_CLOUD, "partition: cloud is empty");
    if (!xyz || !axis_out || (workers > 1 && !cuts) || !worker_of)
        throw Failure(PCS_ERR_INVALID_PARAM, "null buffer");
    if (n > 0xFFFFFFFFull) throw Failure(PCS_ERR_INVALID_PARAM, "partition: at most 2^32 points");
    double mn[3], mx[3];
    for (int a = 0; a < 3; ++a) mn[a] = mx[a] = xyz[a];
    for (uint64_t i = 0; i < n; ++i)
        for (int a = 0; a < 3; ++a) {
            mn[a] = std::fmin(mn[a], xyz[3 * i + a]);
            mx[a] = std::fmax(mx[a], xyz[3 * i + a]);
        }
    const double ext[3] = {mx[0] - mn[0], mx[1] - mn[1], mx[2] - mn[2]};
    int axis = 0;
    if (ext[1] > ext[axis]) axis = 1;
    if (ext[2] > ext[axis]) axis = 2;
    std::vector<uint32_t> order(n);
    std::iota(order.begin(), order.end(), 0u);
    std::sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) {
        const double ca = xyz[3 * (size_t)a + axis], cb = xyz[3 * (size_t)b + axis];
        if (ca != cb) return ca < cb;
        return a < b;
    });
    const uint64_t base = n / workers, rem = n % workers;
    uint64_t begin = 0;
    for (uint64_t u = 0; u < workers; ++u) {
        const uint64_t end = begin + base + (u < rem ? 1 : 0);
        for (uint64_t k = begin; k < end; ++k) worker_of[order[k]] = (uint32_t)u;
        if (u + 1 < workers) {
            if (end < n) {
                const double left = xyz[3 * (size_t)order[end - 1] + axis];
                const double right = xyz[3 * (size_t)order[end] + axis];
                cuts[u] = 0.5 * (left + right);
            } else {
                cuts[u] = mx[axis];
            }
        }
        begin = end;
    }
    *axis_out = axis;
}

}  // namespace pcsb
