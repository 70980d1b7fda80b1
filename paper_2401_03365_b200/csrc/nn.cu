// nn.cu — exact nearest-neighbour queries and the deviation metric on the device
// (SURVEY.md §8(f), row 2 — the next caller beside the LOP path).
//
// Replaces, for a whole query cloud at once:
//   SpatialIndex::nearest   proj/src/spatial.cpp:119-158   (kd-tree best-first
//       descent; smallest index on equal squared distance)
//   pcs::deviation          proj/src/metrics.cpp:39-53     (nearest distance of
//       every cloud point to the reference, then `aggregate` :11-37)
//
// B200 design: the reference cloud is hashed once into a uniform grid of cubic
// cells (the same integer key / radix sort / lower-bound cell table as the LOP
// data grid, grid_sort.cu), fp64 double4 in cell order.  One thread per query,
// queries visited in cell order (a radix sort of their keys) so neighbouring
// threads walk neighbouring cells through L1/L2.  A query scans Chebyshev shells
// of cells around its own (R = 0, 1, 2, ...); each shell row is one contiguous
// range of the sorted cloud.  After shell R the unvisited points all lie beyond
// the scanned block's faces; the walk stops once the best squared distance is
// strictly below the squared distance to the nearest interior face (minus a
// rounding slack), so neither a closer point nor an equal-distance point with a
// smaller index can remain.  Distances are the reference's exactly
// (`norm2(c - q)` with every fp64 operation individually rounded, then sqrt);
// the aggregate is summed on the host in index order, as the reference does.
#include "dev_knobs.h"
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "host_io.h"
#include "plan.cuh"
#include "ptri.h"

namespace pcsb {

namespace {

int bits_for(uint64_t v) {  // bits to hold 0..v-1
    int b = 0;
    while (b < 32 && (1ull << b) < v) ++b;
    return b;
}

double cubic_cells(const double lo[3], const double hi[3], double cs) {
    double c = 1.0;
    for (int a = 0; a < 3; ++a) c *= std::floor((hi[a] - lo[a]) / cs) + 3.0;
    return c;
}

// Isotropic grid over [lo, hi] with ~8 cells per reference point (a surface
// sample then shares its cell with O(10) others), at most 2^26 cells.
GridGeom nn_grid(const double lo[3], const double hi[3], uint64_t n) {
    double ext = 0.0;
    for (int a = 0; a < 3; ++a) ext = std::max(ext, hi[a] - lo[a]);
    if (!(ext > 0.0)) ext = 1.0;
    double target = std::min(8.0 * (double)n, (double)(1u << 26));
    if (const char* e = dev_knob("PCSB_NN_CELLS_PER_POINT"))  // developer knob
        target = std::min(std::atof(e) * (double)n, (double)(1u << 26));
    target = std::max(target, 1.0);
    // largest-first bisection on the cell side: cells_for is non-increasing in cs
    double a = ext * 1e-7, b = ext * 4.0;
    for (int it = 0; it < 80; ++it) {
        const double mid = std::sqrt(a * b);
        if (cubic_cells(lo, hi, mid) > target) a = mid;
        else b = mid;
    }
    const double cs = b;
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
    g.key_bits = std::max(1, bits_for((uint64_t)g.ncells));
    return g;
}

struct Best {
    double d2;
    uint32_t idx;
};

// Points [k0, k1) of the sorted cloud against q (proj/src/spatial.cpp:134-141).
__device__ __forceinline__ void scan_range(const double4* __restrict__ pts,
                                           const uint32_t* __restrict__ order, uint32_t k0,
                                           uint32_t k1, double qx, double qy, double qz, Best& b) {
    for (uint32_t k = k0; k < k1; ++k) {
        const double4 c = pts[k];
        const double d2 = exact_d2(c.x, c.y, c.z, qx, qy, qz);
        if (d2 <= b.d2) {
            const uint32_t idx = __ldg(&order[k]);
            if (d2 < b.d2 || idx < b.idx) {
                b.d2 = d2;
                b.idx = idx;
            }
        }
    }
}

__global__ void __launch_bounds__(128)
nn_kernel(const double4* __restrict__ pts, const uint32_t* __restrict__ order,
          const uint32_t* __restrict__ start, GridGeom g, const double4* __restrict__ Q,
          const uint32_t* __restrict__ qperm, uint32_t m, double slack,
          uint32_t* __restrict__ idx_out, double* __restrict__ dist_out) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= m) return;
    const uint32_t qi = qperm ? __ldg(&qperm[t]) : t;
    const double4 q = Q[qi];
    const int32_t cx = cell_coord(q.x, g.ox, g.inv_cs, g.gx);
    const int32_t cy = cell_coord(q.y, g.oy, g.inv_cs, g.gy);
    const int32_t cz = cell_coord(q.z, g.oz, g.inv_cs, g.gz);
    Best b{INFINITY, 0xFFFFFFFFu};
    const int32_t rmax = max(g.gx, max(g.gy, g.gz));
    for (int32_t R = 0; R <= rmax; ++R) {
        const int32_t z0 = max(cz - R, 0), z1 = min(cz + R, g.gz - 1);
        const int32_t y0 = max(cy - R, 0), y1 = min(cy + R, g.gy - 1);
        const int32_t x0 = max(cx - R, 0), x1 = min(cx + R, g.gx - 1);
        for (int32_t z = z0; z <= z1; ++z) {
            for (int32_t y = y0; y <= y1; ++y) {
                const uint32_t row = (uint32_t)g.gx * ((uint32_t)y + (uint32_t)g.gy * (uint32_t)z);
                if (abs(z - cz) == R || abs(y - cy) == R) {  // whole shell row
                    scan_range(pts, order, __ldg(&start[row + x0]), __ldg(&start[row + x1 + 1]),
                               q.x, q.y, q.z, b);
                } else {  // interior row: only its two end cells are on the shell
                    if (cx - R >= 0)
                        scan_range(pts, order, __ldg(&start[row + cx - R]),
                                   __ldg(&start[row + cx - R + 1]), q.x, q.y, q.z, b);
                    if (R > 0 && cx + R < g.gx)
                        scan_range(pts, order, __ldg(&start[row + cx + R]),
                                   __ldg(&start[row + cx + R + 1]), q.x, q.y, q.z, b);
                }
            }
        }
        // distance to the nearest face of the scanned block that has cells beyond it
        double gap = INFINITY;
        if (cx - R > 0) gap = fmin(gap, q.x - (g.ox + (double)(cx - R) * g.cs));
        if (cx + R < g.gx - 1) gap = fmin(gap, (g.ox + (double)(cx + R + 1) * g.cs) - q.x);
        if (cy - R > 0) gap = fmin(gap, q.y - (g.oy + (double)(cy - R) * g.cs));
        if (cy + R < g.gy - 1) gap = fmin(gap, (g.oy + (double)(cy + R + 1) * g.cs) - q.y);
        if (cz - R > 0) gap = fmin(gap, q.z - (g.oz + (double)(cz - R) * g.cs));
        if (cz + R < g.gz - 1) gap = fmin(gap, (g.oz + (double)(cz + R + 1) * g.cs) - q.z);
        if (gap == INFINITY) break;  // the whole grid has been scanned
        const double gg = gap - slack;
        if (gg > 0.0 && b.d2 < gg * gg) break;
    }
    idx_out[qi] = b.idx;
    dist_out[qi] = __dsqrt_rn(b.d2);
}

struct DevBuf {  // stream-ordered temporaries of one call, from the library's pool
    cudaStream_t s;
    int dev = 0;
    std::vector<void*> p;
    explicit DevBuf(cudaStream_t s_) : s(s_) { PCSB_CUDA(cudaGetDevice(&dev)); }
    ~DevBuf() {
        for (void* x : p) pool_free(x, s);
    }
    template <typename X>
    X* get(size_t count) {
        void* x = pool_alloc(dev, std::max<size_t>(count * sizeof(X), 16), s);
        p.push_back(x);
        return (X*)x;
    }
};

struct Stream {
    cudaStream_t s = nullptr;
    Stream() { PCSB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); }
    ~Stream() {
        cudaStreamSynchronize(s);
        cudaStreamDestroy(s);
    }
};

// Nearest reference point of every query (original indices, exact distances).
void nearest_device(const double* C, uint64_t n, const double* Qh, uint64_t m, uint32_t* idx,
                    double* dist, cudaStream_t s) {
    if (n > 0xFFFFFFFEull || m > 0xFFFFFFFEull)
        throw Failure(PCS_ERR_INVALID_PARAM, "nearest: clouds are limited to 2^32-2 points");
    DevBuf mem(s);
    const uint32_t nn = (uint32_t)n, mm = (uint32_t)m;
    double* dC = mem.get<double>(n * 3);
    double* dQ = mem.get<double>(m * 3);
    h2d_staged(dC, C, n * 3 * sizeof(double), s);
    h2d_staged(dQ, Qh, m * 3 * sizeof(double), s);
    double4* Cv = mem.get<double4>(n);
    double4* Qv = mem.get<double4>(m);
    launch_convert_xyz<double>(dC, Cv, n, 1.0, s);
    launch_convert_xyz<double>(dQ, Qv, m, 0.0, s);
    unsigned long long* slots = mem.get<unsigned long long>(8);
    init_bbox_slots(slots, s);
    launch_bbox<double>(Cv, n, slots, s);
    launch_bbox<double>(Qv, m, slots, s);
    unsigned long long hb[6];
    PCSB_CUDA(cudaMemcpyAsync(hb, slots, sizeof(hb), cudaMemcpyDeviceToHost, s));
    PCSB_CUDA(cudaStreamSynchronize(s));
    double lo[3], hi[3], maxabs = 0.0;
    for (int a = 0; a < 3; ++a) {
        lo[a] = ordered_to_double(hb[a]);
        hi[a] = ordered_to_double(hb[3 + a]);
        if (!std::isfinite(lo[a]) || !std::isfinite(hi[a]))
            throw Failure(PCS_ERR_INVALID_PARAM, "clouds must have finite coordinates");
        maxabs = std::max(maxabs, std::max(std::fabs(lo[a]), std::fabs(hi[a])));
    }
    const GridGeom g = nn_grid(lo, hi, n);
    const uint32_t cap = std::max(nn, mm);
    uint32_t* keys = mem.get<uint32_t>(cap);
    uint32_t* skeys = mem.get<uint32_t>(cap);
    uint32_t* order = mem.get<uint32_t>(nn);
    uint32_t* qperm = mem.get<uint32_t>(mm);
    double4* sorted = mem.get<double4>(n);
    uint32_t* start = mem.get<uint32_t>((size_t)g.ncells + 1);
    RadixScratch rs;
    rs.keys_alt = mem.get<uint32_t>(cap);
    rs.vals_alt = mem.get<uint32_t>(cap);
    rs.blockhist = mem.get<uint32_t>(radix_blockhist_entries(cap));
    rs.capacity = cap;
    uint32_t* cscr = mem.get<uint32_t>(cell_scan_scratch_entries(g.ncells));
    // reference cloud: cell keys -> stable sort -> gather -> lower-bound table
    launch_keys<double>(g, Cv, nn, keys, nullptr, s);
    radix_sort(keys, nullptr, skeys, order, nn, g.key_bits, rs, nullptr, s);
    launch_gather<double>(Cv, order, nn, sorted, nullptr, s);
    build_cell_start(skeys, nn, 0, g.ncells, start, cscr, nullptr, s);
    // queries in cell order
    launch_keys<double>(g, Qv, mm, keys, nullptr, s);
    radix_sort(keys, nullptr, skeys, qperm, mm, g.key_bits, rs, nullptr, s);
    uint32_t* didx = mem.get<uint32_t>(mm);
    double* ddist = mem.get<double>(m);
    // rounding slack of the face distances: cell coordinates are fp64 products of
    // magnitude <= maxabs + a few cells (a few ulps each)
    const double slack = 8.0 * std::ldexp(maxabs + 4.0 * g.cs + 1.0, -52);
    nn_kernel<<<(mm + 127) / 128, 128, 0, s>>>(sorted, order, start, g, Qv, qperm, mm, slack, didx,
                                              ddist);
    PCSB_CUDA(cudaGetLastError());
    PCSB_CUDA(cudaMemcpyAsync(idx, didx, m * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    PCSB_CUDA(cudaMemcpyAsync(dist, ddist, m * sizeof(double), cudaMemcpyDeviceToHost, s));
    PCSB_CUDA(cudaStreamSynchronize(s));
    PCSB_CUDA(cudaGetLastError());
}

// Mesh deviation (proj/src/metrics.cpp:115-133): one thread per cloud point,
// the triangle soup streamed through shared memory in tiles; the minimum over
// triangles is order-free, so the result is the reference's exactly.
constexpr int MESH_THREADS = 128;
constexpr int MESH_TILE = 128;  // triangles per shared-memory tile (9 KB)

__global__ void __launch_bounds__(MESH_THREADS)
mesh_kernel(const double* __restrict__ P, uint32_t m, const double* __restrict__ T, uint32_t nt,
            double* __restrict__ dist_out) {
    __shared__ double tile[MESH_TILE * 9];
    const uint32_t i = blockIdx.x * MESH_THREADS + threadIdx.x;
    const bool live = i < m;
    ptri::V3 p{0.0, 0.0, 0.0};
    if (live) p = {P[3 * (size_t)i], P[3 * (size_t)i + 1], P[3 * (size_t)i + 2]};
    double best = INFINITY;
    bool first = true;
    for (uint32_t t0 = 0; t0 < nt; t0 += MESH_TILE) {
        const uint32_t cnt = min((uint32_t)MESH_TILE, nt - t0);
        __syncthreads();
        for (uint32_t k = threadIdx.x; k < cnt * 9; k += MESH_THREADS) tile[k] = T[(size_t)t0 * 9 + k];
        __syncthreads();
        if (live) {
            for (uint32_t t = 0; t < cnt; ++t) {
                const double* q = tile + 9 * t;
                const double d = ptri::distance(p, {q[0], q[1], q[2]}, {q[3], q[4], q[5]},
                                                {q[6], q[7], q[8]});
                // best = min(best, d) with best seeded by triangle 0 (std::min keeps
                // the current value unless the new one is smaller)
                if (first) {
                    best = d;
                    first = false;
                } else if (d < best) {
                    best = d;
                }
            }
        }
    }
    if (live) dist_out[i] = best;
}

// Index-order aggregation of proj/src/metrics.cpp:11-37.
void aggregate(const double* dist, uint64_t m, pcs_deviation_report* rep) {
    double sum = 0.0, sum_sq = 0.0, max_d = 0.0;
    for (uint64_t i = 0; i < m; ++i) {
        const double v = dist[i];
        sum += v;
        const volatile double sq = v * v;  // no contraction into an fma
        sum_sq += sq;
        max_d = std::max(max_d, v);
    }
    const double nd = (double)m;
    rep->n = m;
    rep->mean_distance = sum / nd;
    rep->std_deviation = std::sqrt(sum_sq / nd);
    rep->max_distance = max_d;
    if (rep->std_deviation < rep->mean_distance * (1.0 - 1e-12))
        throw Failure(PCS_ERR_NUMERICAL, "internal: RMS deviation fell below mean distance");
}

}  // namespace

void nearest_all(const pcs_lop_desc& d, const double* C, uint64_t n, const double* Q, uint64_t m,
                 uint32_t* idx_out, double* dist_out) {
    if (n == 0) throw Failure(PCS_ERR_EMPTY_CLOUD, "nearest: index built over an empty cloud");
    if (m == 0) return;
    if (!C || !Q || !idx_out || !dist_out) throw Failure(PCS_ERR_INVALID_PARAM, "null buffer");
    select_device(d.device);
    Stream st;
    nearest_device(C, n, Q, m, idx_out, dist_out, st.s);
}

// proj/src/metrics.cpp:39-53 + aggregate (:11-37): the distances come from the
// device; the sums run here in index order, exactly as the reference's loop.
void deviation(const pcs_lop_desc& d, const double* cloud, uint64_t m, const double* ref,
               uint64_t n, pcs_deviation_report* rep, double* distances_out) {
    if (m == 0) throw Failure(PCS_ERR_EMPTY_CLOUD, "deviation: cloud is empty");
    if (n == 0) throw Failure(PCS_ERR_EMPTY_CLOUD, "deviation: reference cloud is empty");
    if (!cloud || !ref || !rep) throw Failure(PCS_ERR_INVALID_PARAM, "null buffer");
    select_device(d.device);
    std::vector<uint32_t> idx(m);
    std::vector<double> own;
    double* dist = distances_out;
    if (!dist) {
        own.resize(m);
        dist = own.data();
    }
    {
        Stream st;
        nearest_device(ref, n, cloud, m, idx.data(), dist, st.s);
    }
    aggregate(dist, m, rep);
}

void deviation_to_mesh(const pcs_lop_desc& d, const double* cloud, uint64_t m, const double* tri,
                       uint64_t ntri, pcs_deviation_report* rep, double* distances_out) {
    if (m == 0) throw Failure(PCS_ERR_EMPTY_CLOUD, "deviation_to_mesh: cloud is empty");
    if (ntri == 0) throw Failure(PCS_ERR_EMPTY_MESH, "deviation_to_mesh: mesh has no triangles");
    if (!cloud || !tri || !rep) throw Failure(PCS_ERR_INVALID_PARAM, "null buffer");
    if (m > 0xFFFFFFFEull || ntri > 0xFFFFFFFEull)
        throw Failure(PCS_ERR_INVALID_PARAM, "deviation_to_mesh: sizes are limited to 2^32-2");
    select_device(d.device);
    std::vector<double> own;
    double* dist = distances_out;
    if (!dist) {
        own.resize(m);
        dist = own.data();
    }
    {
        Stream st;
        DevBuf mem(st.s);
        double* dP = mem.get<double>(m * 3);
        double* dT = mem.get<double>(ntri * 9);
        double* dD = mem.get<double>(m);
        PCSB_CUDA(cudaMemcpyAsync(dP, cloud, m * 3 * sizeof(double), cudaMemcpyHostToDevice, st.s));
        PCSB_CUDA(cudaMemcpyAsync(dT, tri, ntri * 9 * sizeof(double), cudaMemcpyHostToDevice, st.s));
        mesh_kernel<<<(uint32_t)((m + MESH_THREADS - 1) / MESH_THREADS), MESH_THREADS, 0, st.s>>>(
            dP, (uint32_t)m, dT, (uint32_t)ntri, dD);
        PCSB_CUDA(cudaGetLastError());
        PCSB_CUDA(cudaMemcpyAsync(dist, dD, m * sizeof(double), cudaMemcpyDeviceToHost, st.s));
        PCSB_CUDA(cudaStreamSynchronize(st.s));
        PCSB_CUDA(cudaGetLastError());
    }
    aggregate(dist, m, rep);
}

}  // namespace pcsb
