// kernels.cuh — launcher declarations for the sm_100a kernels.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"

namespace pcsb {

// ---- grid / sort (grid_sort.cu) ---------------------------------------------
template <typename T>
void launch_convert_xyz(const double* xyz, typename Vec4<T>::type* out, uint64_t n, T w,
                        cudaStream_t s);
// bbox accumulated into 6 ordered-uint64 slots: min xyz, max xyz
template <typename T>
void launch_bbox(const typename Vec4<T>::type* pts, uint64_t n, unsigned long long* slots,
                 cudaStream_t s);
void init_bbox_slots(unsigned long long* slots, cudaStream_t s);
double ordered_to_double(unsigned long long v);

template <typename T>
void launch_keys(const GridGeom& g, const typename Vec4<T>::type* pts, uint32_t n,
                 uint32_t* keys, const uint32_t* done, cudaStream_t s);

struct RadixScratch {
    uint32_t* keys_alt = nullptr;
    uint32_t* vals_alt = nullptr;
    uint32_t* blockhist = nullptr;  // 256 * nblocks
    uint32_t capacity = 0;
};
size_t radix_blockhist_entries(uint32_t n);
// Stable LSD sort of (keys, values = 0..n-1 when vals_in == nullptr) on the low
// key_bits bits.  Results land in keys_out / vals_out.  Returns kernel count.
// (values = val_base + i when vals_in == nullptr)
int radix_sort(const uint32_t* keys_in, const uint32_t* vals_in, uint32_t* keys_out,
               uint32_t* vals_out, uint32_t n, int key_bits, RadixScratch& scr,
               const uint32_t* done, cudaStream_t s, uint32_t val_base = 0);

template <typename T>
void launch_gather(const typename Vec4<T>::type* src, const uint32_t* idx, uint32_t n,
                   typename Vec4<T>::type* dst, const uint32_t* done, cudaStream_t s);

// Query list of the fused kernels: the sorted slots in Morton (Z-curve) order of
// their half-cell coordinates (<= 10 bits per axis, per-axis bit counts;
// keys_sorted_tmp keeps the codes), so that consecutive queries are spatially
// close; a query group never crosses a Morton block of side ~2 support (code >>
// block_shift changes), which bounds its box.  With sorted_idx, the queries
// whose internal index lies in [own_lo, own_hi) come first (multi-GPU
// ownership).  Returns kernel count.
// pts[0..n) are the queries; qlist receives val_base + their positions.
template <typename V>
int build_query_list(const V* sorted_pts, uint32_t n, const GridGeom& g, double support,
                     const uint32_t* sorted_idx, uint32_t own_lo, uint32_t own_hi, uint32_t* keys_tmp,
                     uint32_t* keys_sorted_tmp, uint32_t* qlist, int* block_shift,
                     RadixScratch& scr, const uint32_t* done, cudaStream_t s,
                     uint32_t val_base = 0);
// Work unit of the fused kernels: `unit` (<= 32) consecutive entries of the query
// list, fetched with one atomic.
uint32_t work_unit_queries(uint32_t nq, int total_warps);

// cell_start[c] = first sorted position whose cell >= c, c in [0, ncells]
// (marks + prefix max; scratch: cell_scan_scratch_entries(ncells) words).
size_t cell_scan_scratch_entries(uint32_t ncells);
int build_cell_start(const uint32_t* sorted_keys, uint32_t n, int sub_shift, uint32_t ncells,
                     uint32_t* cell_start, uint32_t* scratch, const uint32_t* done,
                     cudaStream_t s);

// Pair records: the fp32 candidate layout of the fused kernels.  A sorted cloud
// is re-laid as records of two consecutive slots, record r = float4 pairs[2r] =
// (x0 x1 y0 y1) and pairs[2r+1] = (z0 z1 w0 w1), with every grid row (fixed
// y, z) starting at an even slot (slot = sorted position + pair_row_delta(row),
// common.cuh), so any x-range of a row is a contiguous, 32-byte aligned byte
// range (one bulk copy).  The slots between rows hold far points of weight 0.
size_t pairs_capacity(uint32_t n, const GridGeom& g);  // float4 elements
// Packs the sorted cloud src[0..n) — or, with idx, gathers src[idx[i]] and also
// writes sorted_out[i] — into records; cell_start = the sorted cloud's cell table.
int build_pairs(const float4* src, const uint32_t* idx, float4* sorted_out,
                const uint32_t* sorted_keys, uint32_t n, const GridGeom& g,
                const uint32_t* cell_start, float4* pairs, const uint32_t* done, cudaStream_t s);

// ---- fused fp32 kernels (lop_fast.cu) ---------------------------------------
struct FastArgs {
    const float4* Ppairs;     // data, pair records; w = 1/v_j (WLOP) or 1
    size_t Ppairs_cap;        // float4 elements of Ppairs (checked builds)
    const uint32_t* Pstart;   // cell table of the sorted data (+ row delta = record slot)
    const float4* Xq;         // projected set X^k, internal index order (queries)
    const float4* Xpairs;     // projected set, pair records; w = w_i (WLOP)
    size_t Xpairs_cap;        // float4 elements of Xpairs (checked builds)
    const uint32_t* Xstart;   // cell table of the sorted projected set
    const uint32_t* qlist;    // queries (internal indices, build_query_list order)
    const uint32_t* qcodes;   // their Morton codes
    int block_shift;          // groups stay inside one (code >> block_shift) block
    uint32_t nq;
    uint32_t unit;            // queries per work unit (work_unit_queries)
    uint32_t tail_start;      // list position (multiple of unit) where short units begin
    uint32_t tail_unit;       // queries per unit from tail_start (raised to one group)
    uint32_t tail_parts;      // attraction pass: warps sharing a tail unit's candidate rows (1 = off)
    uint32_t tail_cap;        // entries per plane of attr_x / attr_nx (positions from tail_start)
    int bisect;               // 1: groups by recursive bisection of each unit (bisect_unit)
    GridGeom gP, gX;          // grids of the data and of the projected set
    double s_pad;             // support with margin (cell ranges)
    double r2;                // support^2 in fp64: exact re-decision of borderline pairs
    float scull2;             // row trimming radius^2 (s_pad + fp32 slack)
    float kneg;               // -log2(e)/h^2
    float K0;                 // log2(e) * r2f / h^2  (hit <=> fma(d2,kneg,K0) >= 0)
    float band;               // |arg| <= band -> borderline, re-decided in fp64
    float support;            // s (fp32), repulsion scale
    float mu;
    float4* Xnext;            // internal index order
    uint32_t* careful_list;   // deferred queries (internal indices)
    float4* attr;             // PH_ATTR -> PH_REP: per list position (sum w, sum w d)
    int2* attr_n;             //   (hits, zero-distance candidates)
    float4* attr_x;           // parts 1.. of row-split tail units: tail_parts - 1 planes
    int2* attr_nx;
    uint8_t* ever_isolated;   // internal index
    int4* qcounts;            // parity facility (nullptr = off), internal index: per query
                              // {attraction hits, repulsion hits, coincident, flags}
    uint8_t* qever;           // with qcounts: OR of the flags over all sweeps
    RunState* st;
    SweepSlot* slot;
    const uint32_t* done;
};

// flags of FastArgs::qcounts / ExactArgs::qcounts (pcs_lop_plan_query_counts)
enum : int { QC_ISOLATED = 1, QC_ANCHORED = 2, QC_DEFERRED = 4 };

// rep_mode: 0 = attraction only (mu == 0), 1 = inv-cube repulsion, 2 = neg-linear.
// phase: 0 = fused, 1 = attraction pass (writes attr), 2 = repulsion + update.
void launch_fast(const FastArgs& a, int lanes_per_point, bool wlop, bool check_zero,
                 int rep_mode, int phase, int grid_blocks, cudaStream_t s);
int fast_blocks_per_sm(int lanes_per_point, bool wlop, bool check_zero, int rep_mode);

struct DensityArgs {
    const float4* C;          // cloud, sorted (queries)
    const float4* Cpairs;     // cloud, pair records (candidates)
    size_t Cpairs_cap;        // float4 elements of Cpairs (checked builds)
    const uint32_t* Cstart;   // cell table of the sorted cloud
    const uint32_t* qlist;    // queries (sorted slots, build_query_list order)
    const uint32_t* qcodes;
    int block_shift;
    uint32_t nq;
    uint32_t unit;
    GridGeom g;
    double s_pad, r2;
    float scull2, kneg, K0, band;
    float inv_scale;          // 2^-K0 (undo the theta scaling)
    int invert;               // 1: write 1/(density) (data v_j), 0: write density (w_i)
    float4* out_sorted;       // if non-null: .w of this sorted array
    float4* out_internal;     // else: .w of this internal-order array, index via idx
    const uint32_t* idx;      // sorted slot -> internal index
    RunState* st;
    uint32_t* counter;
    const uint32_t* done;
};
void launch_density(const DensityArgs& a, int grid_blocks, cudaStream_t s);
// Query groups of the curve-ordered list qin[0, nq) (internal indices into Xq):
// bisected 8-query groups of every 32-position unit, cut where consecutive
// queries are farther apart than sqrt(jump2); writes the permuted list to qout
// and, per position, the first position of its group to codes (the fused
// kernels then group by equal codes, block_shift = 0).
void launch_group_order(const uint32_t* qin, const float4* Xq, uint32_t nq, float jump2,
                        uint32_t* qout, uint32_t* codes, const uint32_t* done, cudaStream_t s);

// ---- exact fp64 path (lop_exact.cu) -----------------------------------------
template <typename T>
struct ExactArgs {
    using V = typename Vec4<T>::type;
    const V* P;               // sorted data; .w = v_j (fp64) or 1/v_j (fp32), 1 if LOP
    const uint32_t* Porder;   // sorted -> original data index (anchor tie-break)
    const uint32_t* Pstart;
    const V* Xs;              // sorted projected set; .w = w_i (WLOP)
    const uint32_t* Xstart;
    const uint32_t* Xs_idx;   // sorted slot -> internal index (self exclusion)
    const V* Xq;              // X^k, internal order (query positions)
    const uint32_t* qlist;    // queries (internal indices); nullptr = 0..nq-1
    const uint32_t* nq_dev;   // if non-null, the query count lives on the device
    uint32_t nq;
    GridGeom g, gX;           // grids of the data and of the projected set
    double s_pad, r2, support, h, mu;
    int eta_kind;             // 0 inv-cube, 1 neg-linear
    int wlop;
    V* Xnext;
    uint8_t* ever_isolated;
    int4* qcounts;            // as FastArgs::qcounts (nullptr = off)
    uint8_t* qever;
    RunState* st;
    SweepSlot* slot;
    const uint32_t* done;
    int count_careful;        // add processed queries to st->careful_points
};
template <typename T>
void launch_exact(const ExactArgs<T>& a, int grid_blocks, cudaStream_t s);

// Exact (fp64) density weights: for query q = qlist[i] (or i) at Cq[q],
// v = 1 + sum theta over the sorted cloud C (cell table Cstart) minus the query
// itself (candidate k is the query when (qself ? qself[k] : k) == q); written to
// out[out_idx ? out_idx[q] : q].w (inverted if invert).
template <typename T>
void launch_exact_density(const typename Vec4<T>::type* C, const uint32_t* Cstart,
                          const typename Vec4<T>::type* Cq, const uint32_t* qlist, uint32_t nq,
                          const uint32_t* qself, const GridGeom& g, double s_pad, double r2,
                          double support, double h, int invert, typename Vec4<T>::type* out,
                          const uint32_t* out_idx, RunState* st, const uint32_t* done,
                          cudaStream_t s);

// Radius queries (parity facility): count (idx == nullptr) or fill CSR (unsorted).
template <typename T>
void launch_radius_dump(const typename Vec4<T>::type* C, const uint32_t* Corder,
                        const uint32_t* Cstart, const GridGeom& g, const double* Q, uint32_t m,
                        double r, double s_pad, uint64_t* offsets_or_counts, uint32_t* idx,
                        cudaStream_t s);

// ---- sweep bookkeeping --------------------------------------------------------
void launch_finalize_sweep(RunState* st, SweepSlot* slot, SweepSlot* next, double tol,
                           cudaStream_t s);
template <typename T>
void launch_unpermute(const typename Vec4<T>::type* X, const uint32_t* orig_of_internal,
                      uint32_t mpad, double* out_xyz, cudaStream_t s);
void launch_iso_to_orig(const uint8_t* ever_iso, const uint32_t* orig_of_internal, uint32_t mpad,
                        uint8_t* iso_orig, cudaStream_t s);
template <typename T>
void launch_scatter_init(const typename Vec4<T>::type* X0, const uint32_t* internal_of_orig,
                         uint32_t m, typename Vec4<T>::type* X, cudaStream_t s);
// work estimate per X0 point (data points its own row-trimmed ball stages + 64), sharded layout
template <typename T>
void launch_shard_work(const typename Vec4<T>::type* X0, uint32_t m, const GridGeom& g,
                       double s_pad, const uint32_t* Pstart, float* w, cudaStream_t s);
template <typename T>
void launch_fill_invalid(typename Vec4<T>::type* X, uint32_t mpad, const uint32_t* orig_of_internal,
                         cudaStream_t s);

}  // namespace pcsb
