// common.cuh — shared device-side types for the B200 LOP/WLOP path.
//
// HBM layout (see DESIGN.md §Data layout):
//   data P      : vec4[N] in grid-sorted order, .w = 1/v_j (WLOP, fp32) | v_j (fp64) | 1
//   P order     : uint32[N] sorted position -> original data index
//   X (two)     : vec4[Mpad] in internal index order (ping-pong across sweeps)
//   X sorted    : vec4[M] gathered per sweep, .w = w_i (WLOP) ; uint32 slot -> internal index
//   cell start  : uint32[ncells+1] lower-bound table per grid (P static, X per sweep)
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

// Checked builds (-DPCSB_CHECKS, tools/build_variant.sh checked ...): device-
// side bounds / invariant assertions that trap the kernel (the launch then
// fails loudly); compiled out of the shipped library.
#ifdef PCSB_CHECKS
#include <cstdio>
#define PCSB_DCHECK(c)                                                                     \
    do {                                                                                   \
        if (!(c)) {                                                                        \
            printf("PCSB_CHECKS failed at %s:%d: %s\n", __FILE__, __LINE__, #c);          \
            __trap();                                                                      \
        }                                                                                  \
    } while (0)
#else
#define PCSB_DCHECK(c) \
    do {               \
    } while (0)
#endif

namespace pcsb {

// Uniform grid shared by the data and the projected set.  Cells are cubes of
// side cs; points outside the box clamp into the boundary cells (a clamp is a
// 1-Lipschitz map of cell coordinates, so no neighbour is ever lost).  The sort
// key is  linear_cell << (3*sub_bits) | morton(sub-cell)  so that every row of
// cells (fixed y,z, a run of x) is one contiguous range of the sorted array and
// points inside a cell are ordered along a Z-curve (compact query groups).
// Cells may be finer along x (the row direction): csx = cs / xsub.
struct GridGeom {
    double ox, oy, oz;   // origin
    double cs, inv_cs;   // y/z cell side and its inverse
    double csx, inv_csx; // x cell side (cs / xsub) and its inverse
    int32_t xsub;        // x cells per y/z cell side
    int32_t gx, gy, gz;  // cells per axis
    int32_t sub_bits;    // morton bits per axis inside a cell
    uint32_t ncells;     // gx*gy*gz
    int32_t key_bits;    // radix bits of the key
};

// Per-run device state (one allocation, zero-initialised at reset).
struct RunState {
    uint32_t done;            // converged -> later sweeps are no-ops
    int32_t iterations_run;
    uint32_t converged;
    uint32_t pad0;
    unsigned long long isolated_events;
    unsigned long long coincident_pairs;
    unsigned long long interactions_attr;
    unsigned long long interactions_rep;
    unsigned long long density_pairs;
    unsigned long long careful_points;
    unsigned long long lane_candidates;  // (query, buffered candidate) evaluations, fused kernel
    double last_max_disp;
};

// Per-sweep scratch slots (indexed by sweep number, zeroed at reset).
struct SweepSlot {
    unsigned long long max_disp_bits;  // max displacement (non-negative double bits)
    uint32_t group_counter;            // dynamic group fetch of the fused kernel
    uint32_t careful_count;            // queries deferred to the exact path
    uint32_t density_counter;          // dynamic group fetch of the w_i pass
    uint32_t exact_counter;            // dynamic fetch of the exact kernel
    uint32_t group_counter2;           // dynamic group fetch of the repulsion pass
    uint32_t pad_;
};

template <typename T> struct Vec4;
template <> struct Vec4<float> { using type = float4; };
template <> struct Vec4<double> { using type = double4; };

__host__ __device__ inline uint32_t morton3_spread(uint32_t v) {
    // spreads the low 3 bits of v to positions 0,3,6
    return (v & 1u) | ((v & 2u) << 2) | ((v & 4u) << 4);
}

// Clamped cell coordinate along one axis, computed in fp64 (no rounding can
// push a point two cells away from a neighbour).
__device__ __forceinline__ int32_t cell_coord(double x, double o, double inv, int32_t g) {
    const double u = floor((x - o) * inv);
    if (!(u >= 0.0)) return 0;  // also NaN
    if (u >= (double)(g - 1)) return g - 1;
    return (int32_t)u;
}

__device__ __forceinline__ uint32_t point_key(const GridGeom& g, double x, double y, double z) {
    const double ux = (x - g.ox) * g.inv_csx, uy = (y - g.oy) * g.inv_cs, uz = (z - g.oz) * g.inv_cs;
    const double fx = floor(ux), fy = floor(uy), fz = floor(uz);
    int32_t cx = (fx >= 0.0) ? (fx >= (double)(g.gx - 1) ? g.gx - 1 : (int32_t)fx) : 0;
    int32_t cy = (fy >= 0.0) ? (fy >= (double)(g.gy - 1) ? g.gy - 1 : (int32_t)fy) : 0;
    int32_t cz = (fz >= 0.0) ? (fz >= (double)(g.gz - 1) ? g.gz - 1 : (int32_t)fz) : 0;
    const uint32_t cell = (uint32_t)cx + (uint32_t)g.gx * ((uint32_t)cy + (uint32_t)g.gy * (uint32_t)cz);
    if (g.sub_bits == 0) return cell;
    const int32_t ns = 1 << g.sub_bits;
    auto sub = [&](double u, int32_t c) -> uint32_t {
        int32_t s = (int32_t)floor((u - (double)c) * (double)ns);
        s = s < 0 ? 0 : (s >= ns ? ns - 1 : s);
        return (uint32_t)s;
    };
    const uint32_t m = morton3_spread(sub(ux, cx)) | (morton3_spread(sub(uy, cy)) << 1) |
                       (morton3_spread(sub(uz, cz)) << 2);
    return (cell << (3 * g.sub_bits)) | m;
}

// Pair-record layout (kernels.cuh): the first point of grid row `row` sits at
// record slot start[row*gx] + pair_row_delta(row) — even, and rows never
// overlap (the delta grows by 0..2 per row).  start = the sorted cloud's cell table.
__device__ __forceinline__ uint32_t pair_row_delta(const uint32_t* __restrict__ start, uint32_t row,
                                                   uint32_t gx) {
    const uint32_t rs = __ldg(&start[(size_t)row * gx]);
    return row + ((rs + row) & 1u);
}

// MUFU.EX2 / MUFU.RSQ, flush-to-zero forms (one SFU op each, no range fix-up).
// Hits have arg >= -band (ex2 >= ~1) and d2 >= FLT_MIN unless the pair is
// (nearly) coincident, which surfaces as a non-finite sum and is deferred to
// the exact fp64 path.
__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float rsqrt_approx(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Exact reference squared distance: norm2(p - c) = (dx*dx + dy*dy) + dz*dz with
// every operation individually rounded (no FMA contraction), as x86-64 does for
// proj/include/pcs/core.hpp:28,34 and proj/src/spatial.cpp:100.
__device__ __forceinline__ double exact_d2(double px, double py, double pz, double cx, double cy,
                                           double cz) {
    const double dx = __dsub_rn(px, cx), dy = __dsub_rn(py, cy), dz = __dsub_rn(pz, cz);
    return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
}

__device__ __forceinline__ void atomic_max_nonneg_double(unsigned long long* slot, double v) {
    // non-negative doubles order like their bit patterns
    atomicMax(slot, (unsigned long long)__double_as_longlong(v));
}

}  // namespace pcsb
