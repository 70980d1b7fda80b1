// grid_sort.cu — the spatial hash: fp64 cell keys, a hand-written stable LSD
// radix sort of (key, index), the gather into sorted order and the cell
// lower-bound table.  Replaces the reference's kd-tree build + radius query
// (proj/src/spatial.cpp:32-111) with integer work that is HBM/L2-bound.
#include "dev_knobs.h"
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>

#include <cooperative_groups.h>

#include "common.cuh"
#include "host_io.h"
#include "kernels.cuh"

namespace pcsb {

namespace cg = cooperative_groups;

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

// Histogram of tile `tile` (digit-major layout: blockhist[d * ntiles + tile]).
__device__ __forceinline__ void hist_tile(const uint32_t* __restrict__ keys, uint32_t n, int shift,
                                          uint32_t mask, uint32_t* __restrict__ blockhist,
                                          uint32_t ntiles, uint32_t tile, uint32_t (*h)[256]) {
    for (int i = threadIdx.x; i < RS_WARPS * 256; i += RS_THREADS) (&h[0][0])[i] = 0;
    __syncthreads();
    const int warp = threadIdx.x >> 5;
    const uint32_t base = tile * RS_TILE;
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
        blockhist[(size_t)d * ntiles + tile] = s;
    }
    __syncthreads();
}

__global__ void __launch_bounds__(RS_THREADS)
rs_hist_kernel(const uint32_t* __restrict__ keys, uint32_t n, int shift, uint32_t mask,
               uint32_t* __restrict__ blockhist, uint32_t nblocks, const uint32_t* done) {
    if (done && *done) return;
    __shared__ uint32_t h[RS_WARPS][256];
    hist_tile(keys, n, shift, mask, blockhist, nblocks, blockIdx.x, h);
}

// Exclusive scan of the digit-major block histograms, one block per digit row
// (row d = the counts of digit d in every tile); the row totals land in
// `totals` and are scanned by rs_scan_totals_kernel.
constexpr int RS_ROW_THREADS = 1024;

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

// Exclusive scan of digit row d across the tiles; the row total goes to totals[d].
__device__ __forceinline__ void scan_row(uint32_t* __restrict__ a, uint32_t ntiles,
                                         uint32_t* __restrict__ totals, uint32_t d, uint32_t* sh) {
    uint32_t* row = a + (size_t)d * ntiles;
    const uint32_t chunk = (ntiles + blockDim.x - 1) / blockDim.x;
    const uint32_t b = min(threadIdx.x * chunk, ntiles);
    const uint32_t e = min(b + chunk, ntiles);
    uint32_t s = 0;
#pragma unroll 8
    for (uint32_t i = b; i < e; ++i) s += row[i];
    uint32_t tot = 0;
    uint32_t run = block_exclusive_scan(s, sh, &tot);
#pragma unroll 8
    for (uint32_t i = b; i < e; ++i) {
        const uint32_t v = row[i];
        row[i] = run;
        run += v;
    }
    if (threadIdx.x == 0) totals[d] = tot;
    __syncthreads();
}

// Exclusive scan of digit row d by ONE thread (rows of a few tiles).
constexpr uint32_t kSerialScanTiles = 16;
__device__ __forceinline__ void serial_scan_row(uint32_t* __restrict__ a, uint32_t ntiles,
                                                uint32_t* __restrict__ totals, uint32_t d) {
    uint32_t* row = a + (size_t)d * ntiles;
    uint32_t run = 0;
    for (uint32_t t0 = 0; t0 < ntiles; t0 += 16) {
        uint32_t v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = t0 + i < ntiles ? row[t0 + i] : 0u;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            if (t0 + i < ntiles) row[t0 + i] = run;
            run += v[i];
        }
    }
    totals[d] = run;
}

__global__ void __launch_bounds__(RS_ROW_THREADS)
rs_scan_rows_kernel(uint32_t* __restrict__ a, uint32_t nblocks, uint32_t* __restrict__ totals,
                    const uint32_t* done) {
    if (done && *done) return;
    __shared__ uint32_t sh[33];
    scan_row(a, nblocks, totals, blockIdx.x, sh);
}

// Stable scatter: within a tile elements keep their order (warp-major, then
// round, then lane: each warp owns 256 consecutive keys), ranks inside a warp
// come from __match_any_sync and a per-warp running digit count.  The tile is
// first reordered by digit in shared memory, then written out as contiguous
// digit runs (~8 keys = one 32-byte sector per run for 8-bit digits and
// 2048-key tiles), instead of 4-byte writes scattered over 256 buckets.
struct ScatterSmem {
    uint32_t run[256];    // tile-local running offset per digit
    uint32_t gbase[256];  // global position = gbase[d] + tile-local position
    uint32_t wcnt[RS_WARPS][256];
    uint32_t woff[RS_WARPS][256];
    uint32_t skey[RS_TILE];
    uint32_t sval[RS_TILE];
    uint32_t sh[33];
};

// kKeepVals: hold the tile's values in registers between ranking and placement
// (the multi-kernel sort); else re-read them (the cooperative sort, which must
// stay within 48 registers)
template <bool kKeepVals>
__device__ __forceinline__ void scatter_tile(const uint32_t* __restrict__ kin,
                                             const uint32_t* __restrict__ vin,
                                             uint32_t* __restrict__ kout, uint32_t* __restrict__ vout,
                                             uint32_t n, int shift, uint32_t mask,
                                             const uint32_t* __restrict__ blockoff, uint32_t ntiles,
                                             const uint32_t* __restrict__ digit_totals,
                                             uint32_t val_base, uint32_t tile, ScatterSmem& S) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int d0 = threadIdx.x;  // RS_THREADS == 256: one digit per thread
    // digit bases (exclusive scan of the digit totals) and this tile's digit counts
    const uint32_t tot = digit_totals[d0];
    const uint32_t dbase = block_exclusive_scan(tot, S.sh, nullptr);
    const uint32_t boff = blockoff[(size_t)d0 * ntiles + tile];
    const uint32_t bnext = tile + 1 < ntiles ? blockoff[(size_t)d0 * ntiles + tile + 1] : tot;
    const uint32_t tstart = block_exclusive_scan(bnext - boff, S.sh, nullptr);
    S.run[d0] = tstart;
    S.gbase[d0] = dbase + boff - tstart;
#pragma unroll
    for (int w = 0; w < RS_WARPS; ++w) S.wcnt[w][d0] = 0;
    __syncthreads();
    // warp w ranks the tile's keys [w*256, (w+1)*256) in rounds of 32 consecutive
    // keys (so warp, round, lane is the input order), keeping a per-warp running
    // count per digit: one block barrier for the whole tile
    const uint32_t base = tile * RS_TILE;
    const uint32_t wbase = base + (uint32_t)warp * (RS_ITEMS * 32);
    const unsigned lt = (1u << lane) - 1u;
    uint32_t keys[RS_ITEMS], vals[RS_ITEMS], rk[RS_ITEMS];
#pragma unroll
    for (int r = 0; r < RS_ITEMS; ++r) {
        const uint32_t i = wbase + r * 32 + lane;
        keys[r] = i < n ? kin[i] : 0u;
        if (kKeepVals) vals[r] = i < n ? (vin ? vin[i] : val_base + i) : 0u;
    }
#pragma unroll
    for (int r = 0; r < RS_ITEMS; ++r) {
        const bool valid = wbase + r * 32 + lane < n;
        const uint32_t d = valid ? ((keys[r] >> shift) & mask) : 256u;
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const uint32_t before = valid ? S.wcnt[warp][d] : 0u;
        rk[r] = valid ? before + __popc(peers & lt) : 0xFFFFFFFFu;
        __syncwarp();
        if (valid && (__ffs(peers) - 1) == lane) S.wcnt[warp][d] = before + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    {
        uint32_t acc = S.run[d0];
#pragma unroll
        for (int w = 0; w < RS_WARPS; ++w) {
            const uint32_t c = S.wcnt[w][d0];
            S.woff[w][d0] = acc;
            acc += c;
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < RS_ITEMS; ++r) {
        if (rk[r] != 0xFFFFFFFFu) {
            const uint32_t pos = S.woff[warp][(keys[r] >> shift) & mask] + rk[r];  // tile-local
            const uint32_t i = wbase + r * 32 + lane;
            S.skey[pos] = keys[r];
            S.sval[pos] = kKeepVals ? vals[r] : (vin ? vin[i] : val_base + i);
        }
    }
    __syncthreads();
    const uint32_t cnt = min((uint32_t)RS_TILE, n - base);
    for (uint32_t p = threadIdx.x; p < cnt; p += RS_THREADS) {
        const uint32_t key = S.skey[p];
        const uint32_t g = S.gbase[(key >> shift) & mask] + p;
        kout[g] = key;
        vout[g] = S.sval[p];
    }
    __syncthreads();
}

// Stable scatter: within a tile elements keep their order (round-major,
// warp-major, lane-minor), ranks inside a warp come from __match_any_sync.  The
// tile is first reordered by digit in shared memory, then written out as
// contiguous digit runs (~8 keys = one 32-byte sector per run for 8-bit digits
// and 2048-key tiles), instead of 4-byte writes scattered over 256 buckets.
__global__ void __launch_bounds__(RS_THREADS)
rs_scatter_kernel(const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin,
                  uint32_t* __restrict__ kout, uint32_t* __restrict__ vout, uint32_t n, int shift,
                  uint32_t mask, const uint32_t* __restrict__ blockoff, uint32_t nblocks,
                  const uint32_t* __restrict__ digit_totals, uint32_t val_base,
                  const uint32_t* done) {
    if (done && *done) return;
    __shared__ ScatterSmem S;
    scatter_tile<true>(kin, vin, kout, vout, n, shift, mask, blockoff, nblocks, digit_totals, val_base,
                 blockIdx.x, S);
}

// The whole LSD sort in ONE cooperative launch (per pass: histograms, row
// scans, scatters, separated by grid-wide barriers; tiles and digit rows are
// looped over the co-resident grid).  For the per-sweep sorts (<= a few M
// keys) the multi-kernel version is launch/latency-bound.
// (<= 48 registers: it must fit beside 5 blocks of the attraction pass, whose
// SM slots it shares when it sorts the projected set on the side stream)
__global__ void __launch_bounds__(RS_THREADS, 5)
rs_coop_kernel(const uint32_t* keys_in, const uint32_t* vals_in, uint32_t* keys_out,
               uint32_t* vals_out, uint32_t* keys_alt, uint32_t* vals_alt, uint32_t n, int key_bits,
               uint32_t* blockhist, uint32_t ntiles, uint32_t val_base, const uint32_t* done) {
    if (done && *done) return;  // the flag is constant during the launch: uniform exit
    cg::grid_group grid = cg::this_grid();
    __shared__ ScatterSmem S;
    __shared__ uint32_t h[RS_WARPS][256];
    const int passes = key_bits <= 0 ? 1 : (key_bits + 7) / 8;
    const uint32_t* kin = keys_in;
    const uint32_t* vin = vals_in;
    uint32_t* totals = blockhist + 256 * (size_t)ntiles;
    for (int p = 0; p < passes; ++p) {
        const int shift = 8 * p;
        const int bits = (key_bits - shift) < 8 ? (key_bits - shift) : 8;
        const uint32_t mask = bits <= 0 ? 0u : ((1u << bits) - 1u);
        const bool to_out = ((passes - 1 - p) % 2) == 0;
        uint32_t* ko = to_out ? keys_out : keys_alt;
        uint32_t* vo = to_out ? vals_out : vals_alt;
        for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x)
            hist_tile(kin, n, shift, mask, blockhist, ntiles, t, h);
        grid.sync();
        if (ntiles <= kSerialScanTiles) {
            // few tiles (the grid is then only a few blocks): one thread per digit
            // row, 16 entries per L2 round trip, no block barriers (a 1-tile sort
            // spent 430 us here scanning 256 rows one after another)
            if (blockIdx.x == 0) serial_scan_row(blockhist, ntiles, totals, threadIdx.x);
        } else {
            for (uint32_t d = blockIdx.x; d < 256; d += gridDim.x) scan_row(blockhist, ntiles, totals, d, S.sh);
        }
        grid.sync();
        for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x)
            scatter_tile<false>(kin, vin, ko, vo, n, shift, mask, blockhist, ntiles, totals,
                         p == 0 ? val_base : 0u, t, S);
        grid.sync();
        kin = ko;
        vin = vo;
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
// (Z-curve) code of the point's half-cell coordinates, with per-axis bit counts
// (an axis with fewer cells drops out of the top levels), computed from the
// sorted positions.
// x extent in y/z-sized cells (the Morton code is isotropic)
__host__ __device__ inline int32_t gx_iso(const GridGeom& g) { return (g.gx + g.xsub - 1) / g.xsub; }

struct MortonAxes {
    int bits[3];  // code bits per axis (after coarsening by `shift`)
    int shift;
    int hilbert;  // 1: Hilbert index over max(bits) bits per axis, 0: Morton interleave
};

// 3-D Hilbert index of (x, y, z), B bits each (Skilling's transpose algorithm,
// "Programming the Hilbert curve", AIP Conf. Proc. 707, 2004): undo the excess
// rotations level by level, Gray-encode, interleave.  Consecutive indices are
// face-adjacent cells, so runs of the order stay more compact than Z-curve runs
// (which jump across blocks); the top 3k bits still name aligned blocks of 2^k
// cells.
__device__ __forceinline__ uint32_t hilbert3(uint32_t x, uint32_t y, uint32_t z, int B) {
    uint32_t X[3] = {x, y, z};
    const uint32_t M = 1u << (B - 1);
    for (uint32_t Q = M; Q > 1; Q >>= 1) {
        const uint32_t P = Q - 1;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            if (X[i] & Q) {
                X[0] ^= P;
            } else {
                const uint32_t t = (X[0] ^ X[i]) & P;
                X[0] ^= t;
                X[i] ^= t;
            }
        }
    }
    X[1] ^= X[0];
    X[2] ^= X[1];
    uint32_t t = 0;
    for (uint32_t Q = M; Q > 1; Q >>= 1)
        if (X[2] & Q) t ^= Q - 1;
#pragma unroll
    for (int i = 0; i < 3; ++i) X[i] ^= t;
    uint32_t key = 0;
    for (int b = B - 1; b >= 0; --b)
#pragma unroll
        for (int i = 0; i < 3; ++i) key = (key << 1) | ((X[i] >> b) & 1u);
    return key;
}

__device__ __forceinline__ uint32_t half_cell(double x, double o, double inv2, int32_t g2) {
    const double u = floor((x - o) * inv2);
    if (!(u >= 0.0)) return 0u;
    if (u >= (double)(g2 - 1)) return (uint32_t)(g2 - 1);
    return (uint32_t)u;
}

template <typename V>
__global__ void morton_keys_kernel(const V* __restrict__ pts, uint32_t n, GridGeom g, MortonAxes ax,
                                   const uint32_t* __restrict__ sidx, uint32_t lo, uint32_t hi,
                                   uint32_t owner_bit, uint32_t* __restrict__ keys,
                                   const uint32_t* done) {
    if (done && *done) return;
    const double inv2 = 2.0 * g.inv_cs;
    const int top = max(ax.bits[0], max(ax.bits[1], ax.bits[2]));
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const V p = pts[i];
        const uint32_t f[3] = {half_cell((double)p.x, g.ox, inv2, 2 * gx_iso(g)) >> ax.shift,
                               half_cell((double)p.y, g.oy, inv2, 2 * g.gy) >> ax.shift,
                               half_cell((double)p.z, g.oz, inv2, 2 * g.gz) >> ax.shift};
        uint32_t key = 0;
        if (ax.hilbert) {
            key = top > 0 ? hilbert3(f[0], f[1], f[2], top) : 0u;
        } else {
            for (int l = top - 1; l >= 0; --l)
#pragma unroll
                for (int a = 2; a >= 0; --a)
                    if (l < ax.bits[a]) key = (key << 1) | ((f[a] >> l) & 1u);
        }
        if (sidx) {
            const uint32_t o = sidx[i];
            if (o < lo || o >= hi) key |= owner_bit;  // not owned: after the owned queries
        }
        keys[i] = key;
    }
}

// ---- cell table: start[c] = #points with cell < c = a prefix maximum of marks ----
// mark: for every boundary between two consecutive sorted points (and after the
// last), start[cell(k) + 1] = k + 1; all other entries 0; then an inclusive
// prefix-max over [0, ncells] fills every empty cell with the next start.  The
// prefix entering each 4096-entry tile comes from a binary search over the keys
// (cell_tile_prefix_kernel), so the table is read and written once after the
// marks, through shared memory, in coalesced 16-byte accesses.
constexpr int CS_THREADS = 256;
constexpr int CS_ITEMS = 16;
constexpr int CS_TILE = CS_THREADS * CS_ITEMS;

__global__ void cell_mark_kernel(const uint32_t* __restrict__ skeys, uint32_t n, int sub_shift,
                                 uint32_t* __restrict__ start, const uint32_t* done) {
    if (done && *done) return;
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const uint32_t c = skeys[k] >> sub_shift;
        if (k + 1 == n || (skeys[k + 1] >> sub_shift) != c) start[c + 1] = k + 1;
    }
}

// exclusive prefix max of the marks before each tile, without reading the table:
// marks grow with the cell index (the keys are sorted), so the maximum over the
// entries before tile b (indices <= T - 1, T = b * CS_TILE) is start[T - 1] =
// #points with cell < T - 1, one binary search over the sorted keys per tile
__global__ void cell_tile_prefix_kernel(const uint32_t* __restrict__ skeys, uint32_t n,
                                        int sub_shift, uint32_t ntiles,
                                        uint32_t* __restrict__ tprefix, const uint32_t* done) {
    if (done && *done) return;
    const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= ntiles) return;
    if (b == 0) {
        tprefix[0] = 0;
        return;
    }
    const uint32_t target = b * (uint32_t)CS_TILE - 1;
    uint32_t lo = 0, hi = n;  // first k with cell(k) >= target
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if ((skeys[mid] >> sub_shift) < target) lo = mid + 1;
        else hi = mid;
    }
    tprefix[b] = lo;
}

__global__ void __launch_bounds__(CS_THREADS)
cell_apply_kernel(uint32_t* __restrict__ a, uint32_t count, const uint32_t* __restrict__ tprefix,
                  const uint32_t* done) {
    if (done && *done) return;
    __shared__ uint32_t sh[CS_THREADS / 32];
    // the tile passes through shared memory (one word of padding per 32) so that
    // global loads and stores are coalesced while each thread scans CS_ITEMS
    // consecutive entries without bank conflicts
    __shared__ uint32_t tile[CS_TILE + CS_TILE / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const size_t tbase = (size_t)blockIdx.x * CS_TILE;
    const bool full = tbase + CS_TILE <= count;
    if (full) {
        const uint4* src = reinterpret_cast<const uint4*>(a + tbase);
#pragma unroll
        for (int i = 0; i < CS_ITEMS / 4; ++i) {
            const int j = i * CS_THREADS + threadIdx.x;  // uint4 index in the tile
            const uint4 q = src[j];
            const int w = 4 * j;
            tile[w + (w >> 5)] = q.x;
            tile[w + 1 + (w >> 5)] = q.y;
            tile[w + 2 + (w >> 5)] = q.z;
            tile[w + 3 + (w >> 5)] = q.w;
        }
    } else {
        for (int i = 0; i < CS_ITEMS; ++i) {
            const int w = i * CS_THREADS + threadIdx.x;
            tile[w + (w >> 5)] = (tbase + w < count) ? a[tbase + w] : 0u;
        }
    }
    __syncthreads();
    // thread t owns CS_ITEMS consecutive entries of the tile
    const int own = threadIdx.x * CS_ITEMS;
    uint32_t v[CS_ITEMS];
    uint32_t run = 0;
#pragma unroll
    for (int i = 0; i < CS_ITEMS; ++i) {
        v[i] = tile[own + i + ((own + i) >> 5)];
        run = max(run, v[i]);
        v[i] = run;
    }
    uint32_t incl = run;  // inclusive max over the warp's threads
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl = max(incl, t);
    }
    if (lane == 31) sh[warp] = incl;
    const uint32_t left = __shfl_up_sync(0xffffffffu, incl, 1);
    __syncthreads();
    uint32_t pre = tprefix[blockIdx.x];
    for (int w = 0; w < warp; ++w) pre = max(pre, sh[w]);
    if (lane > 0) pre = max(pre, left);
#pragma unroll
    for (int i = 0; i < CS_ITEMS; ++i) tile[own + i + ((own + i) >> 5)] = max(pre, v[i]);
    __syncthreads();
    if (full) {
        uint4* dst = reinterpret_cast<uint4*>(a + tbase);
#pragma unroll
        for (int i = 0; i < CS_ITEMS / 4; ++i) {
            const int j = i * CS_THREADS + threadIdx.x;
            const int w = 4 * j;
            dst[j] = make_uint4(tile[w + (w >> 5)], tile[w + 1 + (w >> 5)], tile[w + 2 + (w >> 5)],
                                tile[w + 3 + (w >> 5)]);
        }
    } else {
        for (int i = 0; i < CS_ITEMS; ++i) {
            const int w = i * CS_THREADS + threadIdx.x;
            if (tbase + w < count) a[tbase + w] = tile[w + (w >> 5)];
        }
    }
}

// ---- pair records (kernels.cuh) ----------------------------------------------
__device__ __forceinline__ void write_slot(float* __restrict__ pairs, uint32_t p, float x, float y,
                                          float z, float w) {
    float* r = pairs + 8 * (size_t)(p >> 1) + (p & 1u);
    r[0] = x;
    r[2] = y;
    r[4] = z;
    r[6] = w;
}

constexpr float kPadFar = 1.0e18f;  // padding slot: far from everything, weight 0

// Point i (sorted order) -> its record slot; the last point of a row also
// writes the padding slots up to the next point's slot (or the even end).
// With idx, the point is gathered from src[idx[i]] and also stored to sorted_out[i].
__global__ void pack_pairs_kernel(const float4* __restrict__ src, const uint32_t* __restrict__ idx,
                                  float4* __restrict__ sorted_out,
                                  const uint32_t* __restrict__ skeys, uint32_t n, int sub_shift,
                                  uint32_t gx, const uint32_t* __restrict__ start,
                                  float* __restrict__ pairs, const uint32_t* done) {
    if (done && *done) return;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const float4 c = src[idx ? idx[i] : i];
        if (sorted_out) sorted_out[i] = c;
        const uint32_t row = (skeys[i] >> sub_shift) / gx;
        const uint32_t p = i + pair_row_delta(start, row, gx);
        write_slot(pairs, p, c.x, c.y, c.z, c.w);
        uint32_t next;
        if (i + 1 < n) {
            const uint32_t nrow = (skeys[i + 1] >> sub_shift) / gx;
            next = nrow == row ? p + 1 : (i + 1) + pair_row_delta(start, nrow, gx);
        } else {
            next = (p + 2) & ~1u;
        }
        for (uint32_t q = p + 1; q < next; ++q) write_slot(pairs, q, kPadFar, kPadFar, kPadFar, 0.f);
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

#ifdef PCSB_CHECKS
// Checked builds: the lower-bound table is non-decreasing and ends at n; the
// radix sort's output keys are non-decreasing in the sorted bits.
__global__ void check_cell_table_kernel(const uint32_t* start, uint32_t ncells, uint32_t n,
                                        const uint32_t* done) {
    if (done && *done) return;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < ncells; i += gridDim.x * blockDim.x)
        PCSB_DCHECK(start[i] <= start[i + 1]);
    if (blockIdx.x == 0 && threadIdx.x == 0) PCSB_DCHECK(start[0] == 0 && start[ncells] == n);
}
__global__ void check_sorted_kernel(const uint32_t* keys, uint32_t n, uint32_t mask,
                                    const uint32_t* done) {
    if (done && *done) return;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i + 1 < n; i += gridDim.x * blockDim.x)
        PCSB_DCHECK((keys[i] & mask) <= (keys[i + 1] & mask));
}
#endif

static int radix_sort_impl(const uint32_t* keys_in, const uint32_t* vals_in, uint32_t* keys_out,
                           uint32_t* vals_out, uint32_t n, int key_bits, RadixScratch& scr,
                           const uint32_t* done, cudaStream_t s, uint32_t val_base);

int radix_sort(const uint32_t* keys_in, const uint32_t* vals_in, uint32_t* keys_out,
               uint32_t* vals_out, uint32_t n, int key_bits, RadixScratch& scr,
               const uint32_t* done, cudaStream_t s, uint32_t val_base) {
    const int k = radix_sort_impl(keys_in, vals_in, keys_out, vals_out, n, key_bits, scr, done, s, val_base);
#ifdef PCSB_CHECKS
    if (n > 1) {
        const uint32_t mask = key_bits >= 32 ? 0xFFFFFFFFu : ((1u << (key_bits > 0 ? key_bits : 1)) - 1u);
        check_sorted_kernel<<<grid_for(n, 256), 256, 0, s>>>(keys_out, n, mask, done);
    }
#endif
    return k;
}

static int radix_sort_impl(const uint32_t* keys_in, const uint32_t* vals_in, uint32_t* keys_out,
                           uint32_t* vals_out, uint32_t n, int key_bits, RadixScratch& scr,
                           const uint32_t* done, cudaStream_t s, uint32_t val_base) {
    if (n == 0) return 0;
    static const int coop_blocks = [] {
        int dev = 0, sms = 0, per = 0, ok = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&ok, cudaDevAttrCooperativeLaunch, dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, rs_coop_kernel, RS_THREADS, 0);
        if (const char* e = dev_knob("PCSB_COOP_SORT"))  // developer knob: 0 disables
            if (std::atoi(e) == 0) ok = 0;
        return ok ? sms * per : 0;
    }();
    const uint32_t ntiles = (n + RS_TILE - 1) / RS_TILE;
    // measured: one cooperative launch wins for small sorts (config 2's 100K keys:
    // 0.14 -> 0.10 ms per query order) and loses from ~1M keys on
    static const uint32_t coop_max = [] {
        const char* e = dev_knob("PCSB_COOP_MAX");  // developer knob (keys)
        return e ? (uint32_t)std::atol(e) : (256u << 10);
    }();
    if (coop_blocks > 0 && n <= coop_max) {
        // half the co-resident capacity: the two per-sweep sorts (query order on
        // the main stream, projected-set grid on the side stream) can co-run
        const int grid = (int)std::min<uint32_t>(ntiles, (uint32_t)std::max(1, coop_blocks / 2));
        const uint32_t* ki = keys_in;
        const uint32_t* vi = vals_in;
        uint32_t* ka = scr.keys_alt;
        uint32_t* va = scr.vals_alt;
        uint32_t* bh = scr.blockhist;
        uint32_t nn = n, nt = ntiles, vb = val_base;
        int kb = key_bits;
        void* args[] = {(void*)&ki, (void*)&vi, (void*)&keys_out, (void*)&vals_out, (void*)&ka,
                        (void*)&va, (void*)&nn, (void*)&kb, (void*)&bh, (void*)&nt, (void*)&vb,
                        (void*)&done};
        if (cudaLaunchCooperativeKernel((const void*)rs_coop_kernel, grid, RS_THREADS, args, 0, s) ==
            cudaSuccess)
            return 1;
        cudaGetLastError();  // fall through to the multi-kernel sort
    }
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
        rs_scan_rows_kernel<<<256, nblocks >= 16384 ? RS_ROW_THREADS : 256, 0, s>>>(scr.blockhist, nblocks, totals, done);
        rs_scatter_kernel<<<nblocks, RS_THREADS, 0, s>>>(kin, vin, ko, vo, n, shift, mask,
                                                         scr.blockhist, nblocks, totals, val_base,
                                                         done);
        launches += 3;
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

template <typename V>
int build_query_list(const V* sorted_pts, uint32_t n, const GridGeom& g, double support,
                     const uint32_t* sorted_idx, uint32_t own_lo, uint32_t own_hi, uint32_t* keys_tmp,
                     uint32_t* keys_sorted_tmp, uint32_t* qlist, int* block_shift,
                     RadixScratch& scr, const uint32_t* done, cudaStream_t s, uint32_t val_base) {
    auto width = [](uint64_t v) {  // bits to represent 0..v-1
        int b = 0;
        while (b < 32 && (1ull << b) < v) ++b;
        return b;
    };
    const int full[3] = {width(2ull * gx_iso(g)), width(2ull * g.gy), width(2ull * g.gz)};
    MortonAxes ax;
    ax.shift = std::max(0, std::max(full[0], std::max(full[1], full[2])) - 10);
    int mbits = 0;
    for (int a = 0; a < 3; ++a) {
        ax.bits[a] = std::max(0, full[a] - ax.shift);
        mbits += ax.bits[a];
    }
    // query curve: Hilbert (measured tighter groups than the Z-curve) unless the
    // developer knob PCSB_CURVE=morton
    static const int hilbert = [] {
        const char* e = dev_knob("PCSB_CURVE");
        return (e && std::string(e) == "morton") ? 0 : 1;
    }();
    ax.hilbert = hilbert;
    const int hb = std::max(ax.bits[0], std::max(ax.bits[1], ax.bits[2]));
    if (ax.hilbert) mbits = 3 * hb;
    // Morton blocks of side ~2 support: 2^k code units per axis (measured best on
    // the height-field config: fuller groups outweigh their larger boxes)
    const double unit = 0.5 * g.cs * std::ldexp(1.0, ax.shift);
    int k = (int)std::floor(std::log2(2.0 * support / unit) + 0.5);
    if (const char* e = dev_knob("PCSB_BLOCK_ADJ")) k += std::atoi(e);  // developer knob
    k = std::max(0, std::min(k, 10));
    *block_shift = 0;
    if (ax.hilbert) *block_shift = 3 * std::min(k, hb);
    else
        for (int a = 0; a < 3; ++a) *block_shift += std::min(k, ax.bits[a]);
    if (!n) return 0;
    // the ownership flag sits right above the Morton code, inside the sorted bits
    morton_keys_kernel<V><<<grid_for(n, 256), 256, 0, s>>>(sorted_pts, n, g, ax, sorted_idx, own_lo,
                                                           own_hi, 1u << mbits, keys_tmp, done);
    const int key_bits = mbits + (sorted_idx ? 1 : 0);
    return 1 + radix_sort(keys_tmp, nullptr, keys_sorted_tmp, qlist, n, std::max(key_bits, 1), scr,
                          done, s, val_base);
}

template int build_query_list<float4>(const float4*, uint32_t, const GridGeom&, double,
                                      const uint32_t*, uint32_t, uint32_t, uint32_t*, uint32_t*,
                                      uint32_t*, int*, RadixScratch&, const uint32_t*, cudaStream_t,
                                      uint32_t);
template int build_query_list<double4>(const double4*, uint32_t, const GridGeom&, double,
                                       const uint32_t*, uint32_t, uint32_t, uint32_t*, uint32_t*,
                                       uint32_t*, int*, RadixScratch&, const uint32_t*, cudaStream_t,
                                       uint32_t);

namespace {
__global__ void widen_f32x3_kernel(const float* __restrict__ src, float4* __restrict__ dst,
                                   uint64_t n, float w) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        dst[i] = make_float4(src[3 * i], src[3 * i + 1], src[3 * i + 2], w);
}
}  // namespace

void launch_widen_f32x3(const float* src, float4* dst, size_t n, float w, cudaStream_t s) {
    if (n) widen_f32x3_kernel<<<grid_for(n, 256), 256, 0, s>>>(src, dst, n, w);
}

size_t cell_scan_scratch_entries(uint32_t ncells) {
    return ((size_t)ncells + 1 + CS_TILE - 1) / CS_TILE + 1;
}

int build_cell_start(const uint32_t* sorted_keys, uint32_t n, int sub_shift, uint32_t ncells,
                     uint32_t* cell_start, uint32_t* scratch, const uint32_t* done,
                     cudaStream_t s) {
    const uint32_t count = ncells + 1;
    const uint32_t ntiles = (count + CS_TILE - 1) / CS_TILE;
    cudaMemsetAsync(cell_start, 0, (size_t)count * sizeof(uint32_t), s);
    if (n) cell_mark_kernel<<<grid_for(n, 256), 256, 0, s>>>(sorted_keys, n, sub_shift, cell_start, done);
    cell_tile_prefix_kernel<<<grid_for(ntiles, 256), 256, 0, s>>>(sorted_keys, n, sub_shift, ntiles,
                                                                  scratch, done);
    cell_apply_kernel<<<ntiles, CS_THREADS, 0, s>>>(cell_start, count, scratch, done);
#ifdef PCSB_CHECKS
    check_cell_table_kernel<<<grid_for(count, 256), 256, 0, s>>>(cell_start, ncells, n, done);
#endif
    return n ? 3 : 2;
}

size_t pairs_capacity(uint32_t n, const GridGeom& g) {
    const size_t rows = (size_t)g.gy * (size_t)g.gz;
    return (size_t)n + 2 * rows + 4;
}

int build_pairs(const float4* src, const uint32_t* idx, float4* sorted_out,
                const uint32_t* sorted_keys, uint32_t n, const GridGeom& g,
                const uint32_t* cell_start, float4* pairs, const uint32_t* done, cudaStream_t s) {
    if (!n) return 0;
    pack_pairs_kernel<<<grid_for(n, 256), 256, 0, s>>>(src, idx, sorted_out, sorted_keys, n,
                                                      3 * g.sub_bits, (uint32_t)g.gx, cell_start,
                                                      (float*)pairs, done);
    return 1;
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
