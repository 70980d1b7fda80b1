// grid_sort.cu — the spatial hash: fp64 cell keys, a hand-written stable LSD
// radix sort of (key, index), the gather into sorted order and the cell
// lower-bound table.  Replaces the reference's kd-tree build + radius query
// (proj/src/spatial.cpp:32-111) with integer work that is HBM/L2-bound.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

namespace pcsb {

namespace {

constexpr int RS_THREADS = 256;
constexpr int RS_ITEMS = 8;
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;
constexpr int RS_WARPS = RS_THREADS / 32;

__device__ __forceinline__ unsigned long long double_to_ordered(double v) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}

template <typename V, typename T>
__global__ void convert_xyz_kernel(const double* __restrict__ xyz, V* __restrict__ out, uint64_t n,
                                   T w) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        V v;
        v.x = (T)xyz[3 * i];
        v.y = (T)xyz[3 * i + 1];
        v.z = (T)xyz[3 * i + 2];
        v.w = w;
        out[i] = v;
    }
}

template <typename V>
__global__ void bbox_kernel(const V* __restrict__ pts, uint64_t n, unsigned long long* slots) {
    double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const V p = pts[i];
        const double c[3] = {(double)p.x, (double)p.y, (double)p.z};
        if (!(c[0] == c[0])) continue;  // NaN marks an unused padding slot
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            mn[a] = fmin(mn[a], c[a]);
            mx[a] = fmax(mx[a], c[a]);
        }
    }
#pragma unroll
    for (int a = 0; a < 3; ++a)
        for (int o = 16; o; o >>= 1) {
            mn[a] = fmin(mn[a], __shfl_xor_sync(0xffffffffu, mn[a], o));
            mx[a] = fmax(mx[a], __shfl_xor_sync(0xffffffffu, mx[a], o));
        }
    if ((threadIdx.x & 31) == 0) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            if (mn[a] <= mx[a]) {
                atomicMin(&slots[a], double_to_ordered(mn[a]));
                atomicMax(&slots[3 + a], double_to_ordered(mx[a]));
            }
        }
    }
}

__global__ void init_bbox_kernel(unsigned long long* slots) {
    if (threadIdx.x < 3) slots[threadIdx.x] = ~0ULL;
    else if (threadIdx.x < 6) slots[threadIdx.x] = 0ULL;
}

template <typename V>
__global__ void keys_kernel(GridGeom g, const V* __restrict__ pts, uint32_t n,
                            uint32_t* __restrict__ keys, const uint32_t* done) {
    if (done && *done) return;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const V p = pts[i];
        const double x = (double)p.x;
        keys[i] = (x == x) ? point_key(g, x, (double)p.y, (double)p.z) : 0xFFFFFFFFu;
    }
}

// ---- radix sort -------------------------------------------------------------

__global__ void __launch_bounds__(RS_THREADS)
rs_hist_kernel(const uint32_t* __restrict__ keys, uint32_t n, int shift, uint32_t mask,
               uint32_t* __restrict__ blockhist, uint32_t nblocks, const uint32_t* done) {
    if (done && *done) return;
    __shared__ uint32_t h[RS_WARPS][256];
    for (int i = threadIdx.x; i < RS_WARPS * 256; i += RS_THREADS) (&h[0][0])[i] = 0;
    __syncthreads();
    const int warp = threadIdx.x >> 5;
    const uint32_t base = blockIdx.x * RS_TILE;
#pragma unroll
    for (int r = 0; r < RS_ITEMS; ++r) {
        const uint32_t i = base + r * RS_THREADS + threadIdx.x;
        if (i < n) atomicAdd(&h[warp][(keys[i] >> shift) & mask], 1u);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < 256; d += RS_THREADS) {
        uint32_t s = 0;
#pragma unroll
        for (int w = 0; w < RS_WARPS; ++w) s += h[w][d];
        blockhist[(size_t)d * nblocks + blockIdx.x] = s;
    }
}

// Exclusive scan of the digit-major block histograms, one block per digit row
// (row d = the counts of digit d in every tile); the row totals land in
// `totals` and are scanned by rs_scan_totals_kernel.
constexpr int RS_ROW_THREADS = 256;

__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* sh, uint32_t* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) sh[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0u;
        uint32_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += t;
        }
        if (lane < (int)(blockDim.x >> 5)) sh[lane] = wi - w;
        if (lane == 31) sh[32] = wi;
    }
    __syncthreads();
    const uint32_t r = sh[warp] + incl - v;
    if (total) *total = sh[32];
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(RS_ROW_THREADS)
rs_scan_rows_kernel(uint32_t* __restrict__ a, uint32_t nblocks, uint32_t* __restrict__ totals,
                    const uint32_t* done) {
    if (done && *done) return;
    __shared__ uint32_t sh[33];
    uint32_t* row = a + (size_t)blockIdx.x * nblocks;
    const uint32_t chunk = (nblocks + RS_ROW_THREADS - 1) / RS_ROW_THREADS;
    const uint32_t b = threadIdx.x * chunk;
    const uint32_t e = min(b + chunk, nblocks);
    uint32_t s = 0;
    for (uint32_t i = b; i < e; ++i) s += row[i];
    uint32_t tot = 0;
    uint32_t run = block_exclusive_scan(s, sh, &tot);
    for (uint32_t i = b; i < e; ++i) {
        const uint32_t v = row[i];
        row[i] = run;
        run += v;
    }
    if (threadIdx.x == 0) totals[blockIdx.x] = tot;
}

// Exclusive scan of the 256 digit totals -> digit bases (in place).
__global__ void __launch_bounds__(256) rs_scan_totals_kernel(uint32_t* __restrict__ totals,
                                                            const uint32_t* done) {
    if (done && *done) return;
    __shared__ uint32_t sh[33];
    const uint32_t v = totals[threadIdx.x];
    const uint32_t ex = block_exclusive_scan(v, sh, nullptr);
    totals[threadIdx.x] = ex;
}

// Stable scatter: within a tile elements keep their order (round-major,
// warp-major, lane-minor), ranks inside a warp come from __match_any_sync.
__global__ void __launch_bounds__(RS_THREADS)
rs_scatter_kernel(const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin,
                  uint32_t* __restrict__ kout, uint32_t* __restrict__ vout, uint32_t n, int shift,
                  uint32_t mask, const uint32_t* __restrict__ blockoff, uint32_t nblocks,
                  const uint32_t* __restrict__ digit_base, const uint32_t* done) {
    if (done && *done) return;
    __shared__ uint32_t run[256];
    __shared__ uint32_t wcnt[RS_WARPS][256];
    __shared__ uint32_t woff[RS_WARPS][256];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int d = threadIdx.x; d < 256; d += RS_THREADS) {
        run[d] = digit_base[d] + blockoff[(size_t)d * nblocks + blockIdx.x];
#pragma unroll
        for (int w = 0; w < RS_WARPS; ++w) wcnt[w][d] = 0;
    }
    __syncthreads();
    const uint32_t base = blockIdx.x * RS_TILE;
    const unsigned lt = (1u << lane) - 1u;
    for (int r = 0; r < RS_ITEMS; ++r) {
        const uint32_t i = base + r * RS_THREADS + threadIdx.x;
        const bool valid = i < n;
        const uint32_t key = valid ? kin[i] : 0u;
        const uint32_t val = valid ? (vin ? vin[i] : i) : 0u;
        const uint32_t d = valid ? ((key >> shift) & mask) : 256u;
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const uint32_t rank = __popc(peers & lt);
        if (valid && (__ffs(peers) - 1) == lane) wcnt[warp][d] = __popc(peers);
        __syncthreads();
        for (int dd = threadIdx.x; dd < 256; dd += RS_THREADS) {
            uint32_t acc = run[dd];
#pragma unroll
            for (int w = 0; w < RS_WARPS; ++w) {
                const uint32_t c = wcnt[w][dd];
                woff[w][dd] = acc;
                acc += c;
                wcnt[w][dd] = 0;
            }
            run[dd] = acc;
        }
        __syncthreads();
        if (valid) {
            const uint32_t pos = woff[warp][d] + rank;
            kout[pos] = key;
            vout[pos] = val;
        }
    }
}

template <typename V>
__global__ void gather_kernel(const V* __restrict__ src, const uint32_t* __restrict__ idx,
                              uint32_t n, V* __restrict__ dst, const uint32_t* done) {
    if (done && *done) return;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        dst[i] = src[idx[i]];
}

// Query order of the fused kernels (kernels.cuh build_query_list): Morton
// (Z-curve) code of the point's sub-cell, decoded from its grid key.
__device__ __forceinline__ uint32_t compact3(uint32_t m) {  // bits 0,3,6,.. -> 0,1,2,..
    m &= 0x09249249u;
    m = (m ^ (m >> 2)) & 0x030C30C3u;
    m = (m ^ (m >> 4)) & 0x0300F00Fu;
    m = (m ^ (m >> 8)) & 0x030000FFu;
    m = (m ^ (m >> 16)) & 0x000003FFu;
    return m;
}
__device__ __forceinline__ uint32_t spread3(uint32_t v) {  // 10 bits -> 0,3,6,..
    v &= 0x3FFu;
    v = (v | (v << 16)) & 0x030000FFu;
    v = (v | (v << 8)) & 0x0300F00Fu;
    v = (v | (v << 4)) & 0x030C30C3u;
    v = (v | (v << 2)) & 0x09249249u;
    return v;
}

__global__ void morton_keys_kernel(const uint32_t* __restrict__ skeys, uint32_t n, int sb, uint32_t gx,
                                   uint32_t gy, int shift, const uint32_t* __restrict__ sidx,
                                   uint32_t lo, uint32_t hi, uint32_t owner_bit,
                                   uint32_t* __restrict__ keys, const uint32_t* done) {
    if (done && *done) return;
    const uint32_t smask = (1u << (3 * sb)) - 1u;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t k = skeys[i];
        const uint32_t cell = k >> (3 * sb), sub = k & smask;
        const uint32_t cx = cell % gx, r = cell / gx;
        const uint32_t cy = r % gy, cz = r / gy;
        const uint32_t fx = ((cx << sb) | compact3(sub)) >> shift;
        const uint32_t fy = ((cy << sb) | compact3(sub >> 1)) >> shift;
        const uint32_t fz = ((cz << sb) | compact3(sub >> 2)) >> shift;
        uint32_t key = spread3(fx) | (spread3(fy) << 1) | (spread3(fz) << 2);
        if (sidx) {
            const uint32_t o = sidx[i];
            if (o < lo || o >= hi) key |= owner_bit;  // not owned: after the owned queries
        }
        keys[i] = key;
    }
}

constexpr uint32_t kShortGap = 64;

// Thread k (0..n) owns the cells in (cell[k-1], cell[k]]: their lower bound is k.
__global__ void cell_start_kernel(const uint32_t* __restrict__ skeys, uint32_t n, int sub_shift,
                                  uint32_t ncells, uint32_t* __restrict__ start,
                                  uint32_t* __restrict__ gaps, uint32_t* gap_count,
                                  const uint32_t* done) {
    if (done && *done) return;
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k <= n; k += gridDim.x * blockDim.x) {
        const int64_t cur = (k < n) ? (int64_t)(skeys[k] >> sub_shift) : (int64_t)ncells;
        const int64_t prev = (k > 0) ? (int64_t)(skeys[k - 1] >> sub_shift) : -1;
        const int64_t lo = prev + 1, hi = cur;
        if (lo > hi) continue;
        if (hi - lo < (int64_t)kShortGap) {
            for (int64_t c = lo; c <= hi; ++c) start[c] = k;
        } else {
            const uint32_t g = atomicAdd(gap_count, 1u);
            gaps[3 * g] = (uint32_t)lo;
            gaps[3 * g + 1] = (uint32_t)hi;
            gaps[3 * g + 2] = k;
        }
    }
}

__global__ void gap_fill_kernel(uint32_t* __restrict__ start, const uint32_t* __restrict__ gaps,
                                const uint32_t* gap_count, const uint32_t* done) {
    if (done && *done) return;
    const uint32_t ng = *gap_count;
    for (uint32_t g = blockIdx.x; g < ng; g += gridDim.x) {
        const uint32_t lo = gaps[3 * g], hi = gaps[3 * g + 1], v = gaps[3 * g + 2];
        for (uint32_t c = lo + threadIdx.x; c <= hi; c += blockDim.x) start[c] = v;
    }
}

// ---- pair records (kernels.cuh) ----------------------------------------------
// Slot of the first point of grid row `row` is start[row*gx] + row_delta(row):
// even, and rows never overlap (delta grows by at most 2 per row).
__device__ __forceinline__ uint32_t row_delta(const uint32_t* __restrict__ start, uint32_t row,
                                              uint32_t gx) {
    const uint32_t rs = start[(size_t)row * gx];
    return row + ((rs + row) & 1u);
}

__device__ __forceinline__ void write_slot(float* __restrict__ pairs, uint32_t p, float x, float y,
                                           float z, float w) {
    float* r = pairs + 8 * (size_t)(p >> 1) + (p & 1u);
    r[0] = x;
    r[2] = y;
    r[4] = z;
    r[6] = w;
}

constexpr float kPadFar = 1.0e18f;  // padding slot: far from everything, weight 0

// start_pad[c] = start[c] + row_delta(row of c); the slots between two rows
// (and after the last) become far padding points.
__global__ void pad_table_kernel(const uint32_t* __restrict__ start, uint32_t ncells, uint32_t gx,
                                 uint32_t* __restrict__ start_pad, float* __restrict__ pairs,
                                 const uint32_t* done) {
    if (done && *done) return;
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c <= ncells;
         c += gridDim.x * blockDim.x) {
        const uint32_t row = c / gx;
        const uint32_t d = row_delta(start, row, gx);
        const uint32_t v = start[c];
        start_pad[c] = v + d;
        if (c == row * gx && row > 0) {
            const uint32_t dp = row_delta(start, row - 1, gx);
            for (uint32_t p = v + dp; p < v + d; ++p) write_slot(pairs, p, kPadFar, kPadFar, kPadFar, 0.f);
        }
    }
}

__global__ void pack_pairs_kernel(const float4* __restrict__ sorted, const uint32_t* __restrict__ skeys,
                                  uint32_t n, int sub_shift, uint32_t gx,
                                  const uint32_t* __restrict__ start, float* __restrict__ pairs,
                                  const uint32_t* done) {
    if (done && *done) return;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const float4 c = sorted[i];
        const uint32_t row = (skeys[i] >> sub_shift) / gx;
        write_slot(pairs, i + row_delta(start, row, gx), c.x, c.y, c.z, c.w);
    }
}

int grid_for(uint64_t n, int threads, int max_blocks = 148 * 16) {
    uint64_t b = (n + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > (uint64_t)max_blocks) b = max_blocks;
    return (int)b;
}

}  // namespace

double ordered_to_double(unsigned long long v) {
    const unsigned long long b = (v >> 63) ? (v & 0x7FFFFFFFFFFFFFFFULL) : ~v;
    double d;
    memcpy(&d, &b, sizeof(d));
    return d;
}

template <typename T>
void launch_convert_xyz(const double* xyz, typename Vec4<T>::type* out, uint64_t n, T w,
                        cudaStream_t s) {
    if (!n) return;
    convert_xyz_kernel<typename Vec4<T>::type, T><<<grid_for(n, 256), 256, 0, s>>>(xyz, out, n, w);
}

template <typename T>
void launch_bbox(const typename Vec4<T>::type* pts, uint64_t n, unsigned long long* slots,
                 cudaStream_t s) {
    if (!n) return;
    bbox_kernel<typename Vec4<T>::type><<<grid_for(n, 256, 148 * 4), 256, 0, s>>>(pts, n, slots);
}

void init_bbox_slots(unsigned long long* slots, cudaStream_t s) {
    init_bbox_kernel<<<1, 32, 0, s>>>(slots);
}

template <typename T>
void launch_keys(const GridGeom& g, const typename Vec4<T>::type* pts, uint32_t n, uint32_t* keys,
                 const uint32_t* done, cudaStream_t s) {
    if (!n) return;
    keys_kernel<typename Vec4<T>::type><<<grid_for(n, 256), 256, 0, s>>>(g, pts, n, keys, done);
}

size_t radix_blockhist_entries(uint32_t n) {
    const size_t nb = (n + RS_TILE - 1) / RS_TILE;
    return 256 * (nb ? nb : 1) + 256;  // + the digit totals / bases
}

int radix_sort(const uint32_t* keys_in, const uint32_t* vals_in, uint32_t* keys_out,
               uint32_t* vals_out, uint32_t n, int key_bits, RadixScratch& scr,
               const uint32_t* done, cudaStream_t s) {
    if (n == 0) return 0;
    const uint32_t nblocks = (n + RS_TILE - 1) / RS_TILE;
    const int passes = key_bits <= 0 ? 1 : (key_bits + 7) / 8;
    // ping-pong so that the last pass writes keys_out/vals_out
    const uint32_t* kin = keys_in;
    const uint32_t* vin = vals_in;
    int launches = 0;
    for (int p = 0; p < passes; ++p) {
        const int shift = 8 * p;
        const int bits = (key_bits - shift) < 8 ? (key_bits - shift) : 8;
        const uint32_t mask = bits <= 0 ? 0u : ((1u << bits) - 1u);
        const bool last = (p == passes - 1);
        // pass parity: the final pass targets *_out
        const bool to_out = ((passes - 1 - p) % 2) == 0;
        uint32_t* ko = to_out ? keys_out : scr.keys_alt;
        uint32_t* vo = to_out ? vals_out : scr.vals_alt;
        rs_hist_kernel<<<nblocks, RS_THREADS, 0, s>>>(kin, n, shift, mask, scr.blockhist, nblocks,
                                                      done);
        uint32_t* totals = scr.blockhist + 256 * (size_t)nblocks;
        rs_scan_rows_kernel<<<256, RS_ROW_THREADS, 0, s>>>(scr.blockhist, nblocks, totals, done);
        rs_scan_totals_kernel<<<1, 256, 0, s>>>(totals, done);
        rs_scatter_kernel<<<nblocks, RS_THREADS, 0, s>>>(kin, vin, ko, vo, n, shift, mask,
                                                         scr.blockhist, nblocks, totals, done);
        launches += 4;
        kin = ko;
        vin = vo;
        (void)last;
    }
    return launches;
}

template <typename T>
void launch_gather(const typename Vec4<T>::type* src, const uint32_t* idx, uint32_t n,
                   typename Vec4<T>::type* dst, const uint32_t* done, cudaStream_t s) {
    if (!n) return;
    gather_kernel<typename Vec4<T>::type><<<grid_for(n, 256), 256, 0, s>>>(src, idx, n, dst, done);
}

int build_query_list(const uint32_t* sorted_keys, uint32_t n, const GridGeom& g, double support,
                     const uint32_t* sorted_idx, uint32_t own_lo, uint32_t own_hi, uint32_t* keys_tmp,
                     uint32_t* keys_sorted_tmp, uint32_t* qlist, int* block_shift,
                     RadixScratch& scr, const uint32_t* done, cudaStream_t s) {
    const int sb = g.sub_bits;
    uint32_t fmax = (uint32_t)std::max(g.gx, std::max(g.gy, g.gz)) << sb;
    int bits = 0;
    while (bits < 32 && (1ull << bits) < fmax) ++bits;
    const int shift = bits > 10 ? bits - 10 : 0;
    // Morton blocks of side ~2 support: 2^k code units per axis (measured best on
    // the height-field config: fuller groups outweigh their larger boxes)
    const double unit = g.cs * std::ldexp(1.0, shift - sb);
    int k = (int)std::floor(std::log2(2.0 * support / unit) + 0.5);
    if (const char* e = std::getenv("PCSB_BLOCK_ADJ")) k += std::atoi(e);  // developer knob
    k = std::max(0, std::min(k, 10));
    *block_shift = 3 * k;
    if (!n) return 0;
    // the ownership flag sits right above the Morton code, inside the sorted bits
    const int mbits = 3 * std::min(bits, 10);
    morton_keys_kernel<<<grid_for(n, 256), 256, 0, s>>>(sorted_keys, n, sb, (uint32_t)g.gx,
                                                        (uint32_t)g.gy, shift, sorted_idx, own_lo,
                                                        own_hi, 1u << mbits, keys_tmp, done);
    const int key_bits = mbits + (sorted_idx ? 1 : 0);
    return 1 + radix_sort(keys_tmp, nullptr, keys_sorted_tmp, qlist, n, std::max(key_bits, 1), scr,
                          done, s);
}

int build_cell_start(const uint32_t* sorted_keys, uint32_t n, int sub_shift, uint32_t ncells,
                     uint32_t* cell_start, uint32_t* gap_list, uint32_t* gap_count,
                     const uint32_t* done, cudaStream_t s) {
    cudaMemsetAsync(gap_count, 0, sizeof(uint32_t), s);
    cell_start_kernel<<<grid_for((uint64_t)n + 1, 256), 256, 0, s>>>(
        sorted_keys, n, sub_shift, ncells, cell_start, gap_list, gap_count, done);
    gap_fill_kernel<<<148 * 2, 256, 0, s>>>(cell_start, gap_list, gap_count, done);
    return 2;
}

size_t pairs_capacity(uint32_t n, const GridGeom& g) {
    const size_t rows = (size_t)g.gy * (size_t)g.gz;
    return (size_t)n + 2 * rows + 4;
}

int build_pairs(const float4* sorted, const uint32_t* sorted_keys, uint32_t n, const GridGeom& g,
                const uint32_t* cell_start, uint32_t* start_pad, float4* pairs, bool table,
                const uint32_t* done, cudaStream_t s) {
    int k = 0;
    if (table) {
        pad_table_kernel<<<grid_for((uint64_t)g.ncells + 1, 256), 256, 0, s>>>(
            cell_start, g.ncells, (uint32_t)g.gx, start_pad, (float*)pairs, done);
        ++k;
    }
    if (n) {
        pack_pairs_kernel<<<grid_for(n, 256), 256, 0, s>>>(sorted, sorted_keys, n, 3 * g.sub_bits,
                                                          (uint32_t)g.gx, cell_start,
                                                          (float*)pairs, done);
        ++k;
    }
    return k;
}

template void launch_convert_xyz<float>(const double*, float4*, uint64_t, float, cudaStream_t);
template void launch_convert_xyz<double>(const double*, double4*, uint64_t, double, cudaStream_t);
template void launch_bbox<float>(const float4*, uint64_t, unsigned long long*, cudaStream_t);
template void launch_bbox<double>(const double4*, uint64_t, unsigned long long*, cudaStream_t);
template void launch_keys<float>(const GridGeom&, const float4*, uint32_t, uint32_t*,
                                 const uint32_t*, cudaStream_t);
template void launch_keys<double>(const GridGeom&, const double4*, uint32_t, uint32_t*,
                                  const uint32_t*, cudaStream_t);
template void launch_gather<float>(const float4*, const uint32_t*, uint32_t, float4*,
                                   const uint32_t*, cudaStream_t);
template void launch_gather<double>(const double4*, const uint32_t*, uint32_t, double4*,
                                    const uint32_t*, cudaStream_t);

}  // namespace pcsb
