#include "dev_knobs.h"
#include <cstdlib>
// lop_exact.cu — the exact-arithmetic path (fp64 math, reference predicate).
//
// One warp per query (a block per query for the fp32 path's deferred queries);
// its threads stride over the candidates of the cell rows that can hold a point
// within the support.  Every decision follows the reference
// literally:
//   membership   d2 = (dx*dx + dy*dy) + dz*dz <= r*r, no FMA  (spatial.cpp:89,100-101, core.hpp:28)
//   distance     sqrt(d2)                                       (spatial.cpp:102)
//   theta        d > support ? 0 : exp(-(d/h)^2)               (kernels.cpp:8-15)
//   |eta'|       1/(d^2)^2 (inv-cube) | 1 (neg-linear)          (kernels.cpp:23-29)
//   attraction   d == 0 -> anchor candidate (smallest index), else w = theta/d  (lop.cpp:54-65)
//   isolation    !(sum w > 0): anchored -> anchor, else held + flagged         (lop.cpp:67-75)
//   repulsion    skip self, d == 0 -> coincident++, w = theta*|eta'|/d         (lop.cpp:79-97)
// Only the summation order differs from the reference (thread-strided partial
// sums combined by a fixed xor tree and warp order — deterministic, but not index order), so the
// result agrees to a few ulp rather than bit-for-bit.
//
// It is the whole computation in PCS_PREC_FP64 mode and the deferred-query path
// of the fp32 fused kernel.
#include <algorithm>
#include <cfloat>

#include "common.cuh"
#include "kernels.cuh"

namespace pcsb {

namespace {

constexpr int EX_WARPS = 4;
constexpr int EX_THREADS = EX_WARPS * 32;

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ unsigned long long warp_sum_u(unsigned long long v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ unsigned long long warp_min_u(unsigned long long v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w < v ? w : v;
    }
    return v;
}

// A team of NW warps evaluates one query: NW = 1 (a warp per query: the fp64
// path over all queries) or a whole block (the few deferred queries of the fp32
// path, whose latency would otherwise end each sweep).  Team reductions combine
// the warps' partial sums in a fixed order, so results stay deterministic.
template <int NW>
struct Team {
    static constexpr int kSize = 32 * NW;
    double* sh;  // NW words of block shared memory (NW > 1)
    __device__ __forceinline__ int rank() const { return NW == 1 ? (int)(threadIdx.x & 31) : (int)threadIdx.x; }
    __device__ __forceinline__ double sum(double v) const {
        v = warp_sum_d(v);
        if (NW == 1) return v;
        __syncthreads();
        if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
        __syncthreads();
        double r = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) r += sh[w];
        return r;
    }
    __device__ __forceinline__ unsigned long long sum(unsigned long long v) const {
        v = warp_sum_u(v);
        if (NW == 1) return v;
        unsigned long long* u = reinterpret_cast<unsigned long long*>(sh);
        __syncthreads();
        if ((threadIdx.x & 31) == 0) u[threadIdx.x >> 5] = v;
        __syncthreads();
        unsigned long long r = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) r += u[w];
        return r;
    }
    __device__ __forceinline__ unsigned long long min(unsigned long long v) const {
        v = warp_min_u(v);
        if (NW == 1) return v;
        unsigned long long* u = reinterpret_cast<unsigned long long*>(sh);
        __syncthreads();
        if ((threadIdx.x & 31) == 0) u[threadIdx.x >> 5] = v;
        __syncthreads();
        unsigned long long r = ~0ull;
#pragma unroll
        for (int w = 0; w < NW; ++w) r = u[w] < r ? u[w] : r;
        return r;
    }
};
constexpr int EX_TEAM_WARPS = 8;  // deferred queries: one 256-thread block per query

__device__ __forceinline__ double theta_ref(double d, double support, double h) {
    if (d > support) return 0.0;
    const double s = d / h;
    return exp(-s * s);
}

__device__ __forceinline__ double etad_ref(double d, int kind) {
    if (kind == 1) return 1.0;
    const double d2 = __dmul_rn(d, d);
    return 1.0 / __dmul_rn(d2, d2);
}

struct Rows {
    int lox, hix, loy, ny, loz, nrows;
};

__device__ __forceinline__ Rows rows_around(const GridGeom& g, double x, double y, double z,
                                            double s_pad) {
    Rows r;
    r.lox = cell_coord(x - s_pad, g.ox, g.inv_csx, g.gx);
    r.hix = cell_coord(x + s_pad, g.ox, g.inv_csx, g.gx);
    r.loy = cell_coord(y - s_pad, g.oy, g.inv_cs, g.gy);
    const int hiy = cell_coord(y + s_pad, g.oy, g.inv_cs, g.gy);
    r.loz = cell_coord(z - s_pad, g.oz, g.inv_cs, g.gz);
    const int hiz = cell_coord(z + s_pad, g.oz, g.inv_cs, g.gz);
    r.ny = hiy - r.loy + 1;
    r.nrows = r.ny * (hiz - r.loz + 1);
    return r;
}

// Calls f(k) for every sorted position k of the rows, strided over `stride`
// threads (a warp's lanes, or a team's threads).
template <typename F>
__device__ __forceinline__ void for_each_candidate(const uint32_t* __restrict__ start,
                                                   const GridGeom& g, const Rows& rw, int lane,
                                                   F&& f, int stride = 32) {
    for (int r = 0; r < rw.nrows; ++r) {
        const int yy = rw.loy + r % rw.ny;
        const int zz = rw.loz + r / rw.ny;
        const uint32_t base = ((uint32_t)zz * (uint32_t)g.gy + (uint32_t)yy) * (uint32_t)g.gx;
        PCSB_DCHECK((uint64_t)base + (uint64_t)rw.hix + 1 <= (uint64_t)g.ncells);
        const uint32_t b = __ldg(&start[base + rw.lox]);
        const uint32_t e = __ldg(&start[base + rw.hix + 1]);
        PCSB_DCHECK(b <= e);
        for (uint32_t k = b + lane; k < e; k += stride) f(k);
    }
}

// Team version of for_each_candidate: for a block team the row bounds are
// loaded in parallel and the candidates of all rows form one flat index space
// (row found by binary search over the rows' prefix counts in shared memory),
// so a query costs a few dependent loads instead of ~2 per row.
constexpr int EX_TEAM_MAXR = 256;
struct TeamRows {
    uint32_t b[EX_TEAM_MAXR];
    uint32_t pre[EX_TEAM_MAXR + 1];
    uint32_t wtot[32];
};

template <int NW, typename F>
__device__ __forceinline__ void team_for_each(const uint32_t* __restrict__ start, const GridGeom& g,
                                              const Rows& rw, const Team<NW>& team, TeamRows* tr,
                                              F&& f) {
    if (NW == 1 || rw.nrows > EX_TEAM_MAXR || rw.nrows > Team<NW>::kSize) {
        for_each_candidate(start, g, rw, team.rank(), f, Team<NW>::kSize);
        return;
    }
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    uint32_t cnt = 0;
    if (t < rw.nrows) {
        const int yy = rw.loy + t % rw.ny;
        const int zz = rw.loz + t / rw.ny;
        const uint32_t base = ((uint32_t)zz * (uint32_t)g.gy + (uint32_t)yy) * (uint32_t)g.gx;
        PCSB_DCHECK((uint64_t)base + (uint64_t)rw.hix + 1 <= (uint64_t)g.ncells);
        const uint32_t b = __ldg(&start[base + rw.lox]);
        cnt = __ldg(&start[base + rw.hix + 1]) - b;
        PCSB_DCHECK(cnt <= 0x7FFFFFFFu);
        tr->b[t] = b;
    }
    uint32_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    __syncthreads();  // the previous query's readers of tr are done
    if (lane == 31) tr->wtot[w] = incl;
    __syncthreads();
    uint32_t before = 0;
    for (int i = 0; i < w; ++i) before += tr->wtot[i];
    if (t < rw.nrows) tr->pre[t] = before + incl - cnt;
    if (t == rw.nrows - 1) tr->pre[rw.nrows] = before + incl;
    __syncthreads();
    const uint32_t total = tr->pre[rw.nrows];
    for (uint32_t j = t; j < total; j += Team<NW>::kSize) {
        int lo = 0, hi = rw.nrows - 1;  // last row with pre <= j
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (tr->pre[mid] <= j) lo = mid;
            else hi = mid - 1;
        }
        f(tr->b[lo] + (j - tr->pre[lo]));
    }
}

template <typename T, bool kWlop, int NW>
__global__ void __launch_bounds__(NW == 1 ? EX_THREADS : 32 * NW) exact_kernel(const ExactArgs<T> a) {
    using V = typename Vec4<T>::type;
    if (a.done && *a.done) return;
    __shared__ double team_sh[NW];
    __shared__ uint32_t team_q;
    __shared__ TeamRows team_rows[1];
    const Team<NW> team{team_sh};
    const int lane = team.rank();  // this thread's rank in the query's team
    const uint32_t nq = a.nq_dev ? *a.nq_dev : a.nq;
    uint32_t* counter = &a.slot->exact_counter;
    for (;;) {
        uint32_t qn = 0;
        if (NW == 1) {
            if (lane == 0) qn = atomicAdd(counter, 1u);
            qn = __shfl_sync(0xffffffffu, qn, 0);
        } else {
            __syncthreads();
            if (threadIdx.x == 0) team_q = atomicAdd(counter, 1u);
            __syncthreads();
            qn = team_q;
        }
        if (qn >= nq) break;
        const uint32_t q_int = a.qlist ? a.qlist[qn] : qn;  // internal index
        const V qv = a.Xq[q_int];
        const double x = (double)qv.x, y = (double)qv.y, z = (double)qv.z;
        const Rows rw = rows_around(a.g, x, y, z, a.s_pad);

        // ---- attraction over the data (lop.cpp:49-65) ----
        double sw = 0.0, nx = 0.0, ny = 0.0, nz = 0.0;
        unsigned long long cnt = 0;
        unsigned long long anchor = ~0ull;  // (original index << 32) | sorted position
        team_for_each(a.Pstart, a.g, rw, team, team_rows, [&](uint32_t k) {
            const V p = a.P[k];
            const double px = (double)p.x, py = (double)p.y, pz = (double)p.z;
            const double d2 = exact_d2(px, py, pz, x, y, z);
            if (!(d2 <= a.r2)) return;
            const double d = __dsqrt_rn(d2);
            if (d == 0.0) {
                const unsigned long long key =
                    ((unsigned long long)a.Porder[k] << 32) | (unsigned long long)k;
                anchor = key < anchor ? key : anchor;
                return;
            }
            double w = theta_ref(d, a.support, a.h) / d;
            if (kWlop) w = (sizeof(T) == 8) ? w / (double)p.w : w * (double)p.w;
            sw += w;
            nx += w * px;
            ny += w * py;
            nz += w * pz;
            ++cnt;
        });
        sw = team.sum(sw);
        nx = team.sum(nx);
        ny = team.sum(ny);
        nz = team.sum(nz);
        cnt = team.sum(cnt);
        anchor = team.min(anchor);

        double ux, uy, uz;
        bool isolated = false, attracted = sw > 0.0;
        unsigned long long rcnt = 0, coinc = 0;
        if (!attracted) {
            if (anchor != ~0ull) {
                const V p = a.P[(uint32_t)(anchor & 0xFFFFFFFFull)];
                ux = (double)p.x;
                uy = (double)p.y;
                uz = (double)p.z;
            } else {
                isolated = true;
                ux = x;
                uy = y;
                uz = z;
            }
        } else {
            ux = nx / sw;
            uy = ny / sw;
            uz = nz / sw;
            // ---- repulsion over the projected set (lop.cpp:79-97) ----
            if (a.mu > 0.0) {
                double rs = 0.0, rx = 0.0, ry = 0.0, rz = 0.0;
                const Rows rx_ = rows_around(a.gX, x, y, z, a.s_pad);
                team_for_each(a.Xstart, a.gX, rx_, team, team_rows, [&](uint32_t k) {
                    if (a.Xs_idx[k] == q_int) return;
                    const V c = a.Xs[k];
                    const double cx = (double)c.x, cy = (double)c.y, cz = (double)c.z;
                    const double d2 = exact_d2(cx, cy, cz, x, y, z);
                    if (!(d2 <= a.r2)) return;
                    const double d = __dsqrt_rn(d2);
                    if (d == 0.0) {
                        ++coinc;
                        return;
                    }
                    double w = theta_ref(d, a.support, a.h) * etad_ref(d, a.eta_kind) / d;
                    if (kWlop) w = w * (double)c.w;
                    rs += w;
                    rx += w * (x - cx);
                    ry += w * (y - cy);
                    rz += w * (z - cz);
                    ++rcnt;
                });
                rs = team.sum(rs);
                rx = team.sum(rx);
                ry = team.sum(ry);
                rz = team.sum(rz);
                rcnt = team.sum(rcnt);
                coinc = team.sum(coinc);
                if (rs > 0.0) {
                    ux += a.mu * (rx / rs);
                    uy += a.mu * (ry / rs);
                    uz += a.mu * (rz / rs);
                }
            }
        }
        if (lane == 0) {
            V out;
            out.x = (T)ux;
            out.y = (T)uy;
            out.z = (T)uz;
            out.w = (T)0;
            a.Xnext[q_int] = out;
            const double dx = (double)out.x - x, dy = (double)out.y - y, dz = (double)out.z - z;
            const double disp = sqrt(dx * dx + dy * dy + dz * dz);
            if (disp > 0.0) atomic_max_nonneg_double(&a.slot->max_disp_bits, disp);
            if (isolated) {
                a.ever_isolated[q_int] = 1;
                atomicAdd(&a.st->isolated_events, 1ull);
            }
            if (attracted) {
                if (cnt) atomicAdd(&a.st->interactions_attr, cnt);
                if (rcnt) atomicAdd(&a.st->interactions_rep, rcnt);
                if (coinc) atomicAdd(&a.st->coincident_pairs, coinc);
            }
            if (a.count_careful) atomicAdd(&a.st->careful_points, 1ull);
            if (a.qcounts) {
                const int fl = (isolated ? QC_ISOLATED : (attracted ? 0 : QC_ANCHORED)) |
                               (a.count_careful ? QC_DEFERRED : 0);
                a.qcounts[q_int] = make_int4(attracted ? (int)cnt : 0, attracted ? (int)rcnt : 0,
                                             attracted ? (int)coinc : 0, fl);
                a.qever[q_int] |= (uint8_t)fl;
            }
        }
    }
}

template <typename T>
__global__ void __launch_bounds__(EX_THREADS)
exact_density_kernel(const typename Vec4<T>::type* __restrict__ C, const uint32_t* __restrict__ Cstart,
                     const typename Vec4<T>::type* __restrict__ Cq,
                     const uint32_t* __restrict__ qlist, uint32_t nq,
                     const uint32_t* __restrict__ qself, GridGeom g, double s_pad, double r2,
                     double support, double h, int invert, typename Vec4<T>::type* out,
                     const uint32_t* __restrict__ out_idx, RunState* st, const uint32_t* done) {
    using V = typename Vec4<T>::type;
    if (done && *done) return;
    const int lane = threadIdx.x & 31;
    const uint32_t wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t qn = wid; qn < nq; qn += nw) {
        const uint32_t qid = qlist ? qlist[qn] : qn;
        const V qv = Cq[qid];
        const double x = (double)qv.x, y = (double)qv.y, z = (double)qv.z;
        const Rows rw = rows_around(g, x, y, z, s_pad);
        double acc = 0.0;
        unsigned long long pairs = 0;
        for_each_candidate(Cstart, g, rw, lane, [&](uint32_t k) {
            if ((qself ? qself[k] : k) == qid) return;
            const V c = C[k];
            const double d2 = exact_d2((double)c.x, (double)c.y, (double)c.z, x, y, z);
            if (!(d2 <= r2)) return;
            const double d = __dsqrt_rn(d2);
            acc += theta_ref(d, support, h);
            if (d > 0.0) ++pairs;
        });
        acc = warp_sum_d(acc);
        pairs = warp_sum_u(pairs);
        if (lane == 0) {
            const double dens = 1.0 + acc;
            const T val = invert ? (T)(1.0 / dens) : (T)dens;
            out[out_idx ? out_idx[qid] : qid].w = val;
            if (pairs) atomicAdd(&st->density_pairs, pairs);
        }
    }
}

template <typename T>
__global__ void __launch_bounds__(EX_THREADS)
radius_dump_kernel(const typename Vec4<T>::type* __restrict__ C, const uint32_t* __restrict__ Corder,
                   const uint32_t* __restrict__ Cstart, GridGeom g, const double* __restrict__ Q,
                   uint32_t m, double r2, double s_pad, uint64_t* offsets_or_counts,
                   uint32_t* idx) {
    using V = typename Vec4<T>::type;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const uint32_t wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t qn = wid; qn < m; qn += nw) {
        // queries are rounded exactly like the cloud (fp32 mode compares fp32 values)
        const double x = (double)(T)Q[3 * (size_t)qn], y = (double)(T)Q[3 * (size_t)qn + 1],
                     z = (double)(T)Q[3 * (size_t)qn + 2];
        const Rows rw = rows_around(g, x, y, z, s_pad);
        uint64_t pos = idx ? offsets_or_counts[qn] : 0;
        for (int rr = 0; rr < rw.nrows; ++rr) {
            const int yy = rw.loy + rr % rw.ny;
            const int zz = rw.loz + rr / rw.ny;
            const uint32_t base = ((uint32_t)zz * (uint32_t)g.gy + (uint32_t)yy) * (uint32_t)g.gx;
            const uint32_t b = Cstart[base + rw.lox];
            const uint32_t e = Cstart[base + rw.hix + 1];
            for (uint32_t k0 = b; k0 < e; k0 += 32) {
                const uint32_t k = k0 + lane;
                bool hit = false;
                if (k < e) {
                    const V c = C[k];
                    hit = exact_d2((double)c.x, (double)c.y, (double)c.z, x, y, z) <= r2;
                }
                const unsigned msk = __ballot_sync(0xffffffffu, hit);
                if (idx && hit) idx[pos + __popc(msk & lt)] = Corder[k];
                pos += __popc(msk);
            }
        }
        if (!idx && lane == 0) offsets_or_counts[qn] = pos;
    }
}

// Sweep epilogue (lop.cpp:102-119).  The sweep count lives on the device
// (iterations_run += 1 per executed sweep), so the launch has no per-sweep
// argument and replays identically inside a CUDA graph.
__global__ void finalize_kernel(RunState* st, SweepSlot* slot, SweepSlot* next, double tol) {
    if (st->done) return;
    if (next != slot) *next = SweepSlot{};  // recycled slot of the next sweep
    const unsigned long long b = slot->max_disp_bits;
    const double md = __longlong_as_double((long long)b);
    st->iterations_run += 1;
    st->last_max_disp = md;
    if (md < tol) {  // lop.cpp:116-119
        st->converged = 1;
        st->done = 1;
    }
}

template <typename V>
__global__ void unpermute_kernel(const V* __restrict__ X, const uint32_t* __restrict__ orig,
                                 uint32_t mpad, double* __restrict__ out) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < mpad; i += gridDim.x * blockDim.x) {
        const uint32_t o = orig ? orig[i] : i;
        if (o == 0xFFFFFFFFu) continue;
        const V v = X[i];
        out[3 * (size_t)o] = (double)v.x;
        out[3 * (size_t)o + 1] = (double)v.y;
        out[3 * (size_t)o + 2] = (double)v.z;
    }
}

__global__ void iso_to_orig_kernel(const uint8_t* __restrict__ ever, const uint32_t* __restrict__ orig,
                                   uint32_t mpad, uint8_t* __restrict__ out) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < mpad; i += gridDim.x * blockDim.x) {
        const uint32_t o = orig ? orig[i] : i;
        if (o == 0xFFFFFFFFu) continue;
        out[o] = ever[i];
    }
}


template <typename V>
__global__ void scatter_init_kernel(const V* __restrict__ X0, const uint32_t* __restrict__ iof,
                                    uint32_t m, V* __restrict__ X) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
        X[iof ? iof[i] : i] = X0[i];
}

template <typename V, typename T>
__global__ void fill_invalid_kernel(V* __restrict__ X, uint32_t mpad, const uint32_t* __restrict__ orig) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < mpad; i += gridDim.x * blockDim.x) {
        if (orig[i] == 0xFFFFFFFFu) {
            V v;
            v.x = (T)NAN;
            v.y = (T)NAN;
            v.z = (T)NAN;
            v.w = (T)0;
            X[i] = v;
        }
    }
}

int blocks_for(uint64_t n, int threads) {
    uint64_t b = (n + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > 148 * 16) b = 148 * 16;
    return (int)b;
}

}  // namespace

template <typename T>
void launch_exact(const ExactArgs<T>& a, int grid_blocks, cudaStream_t s) {
    if (a.count_careful) {  // the fp32 path's deferred queries: a block per query
        constexpr int NT = 32 * EX_TEAM_WARPS;
        if (a.wlop) exact_kernel<T, true, EX_TEAM_WARPS><<<grid_blocks, NT, 0, s>>>(a);
        else exact_kernel<T, false, EX_TEAM_WARPS><<<grid_blocks, NT, 0, s>>>(a);
    } else if (a.nq <= 32768u) {
        // few queries (config 1: 2,000): a 128-thread team per query with its
        // rows' bounds loaded at once and the candidates flattened — the latency of
        // a few dependent loads per query instead of ~2 per cell row
        const int blocks = (int)std::min<uint32_t>(std::max(a.nq, 1u), (uint32_t)grid_blocks * 2u);
        if (a.wlop) exact_kernel<T, true, 4><<<blocks, 128, 0, s>>>(a);
        else exact_kernel<T, false, 4><<<blocks, 128, 0, s>>>(a);
    } else {
        if (a.wlop) exact_kernel<T, true, 1><<<grid_blocks, EX_THREADS, 0, s>>>(a);
        else exact_kernel<T, false, 1><<<grid_blocks, EX_THREADS, 0, s>>>(a);
    }
}

template <typename T>
void launch_exact_density(const typename Vec4<T>::type* C, const uint32_t* Cstart,
                          const typename Vec4<T>::type* Cq, const uint32_t* qlist, uint32_t nq,
                          const uint32_t* qself, const GridGeom& g, double s_pad, double r2,
                          double support, double h, int invert, typename Vec4<T>::type* out,
                          const uint32_t* out_idx, RunState* st, const uint32_t* done,
                          cudaStream_t s) {
    if (!nq) return;
    exact_density_kernel<T><<<blocks_for((uint64_t)nq * 32, EX_THREADS), EX_THREADS, 0, s>>>(
        C, Cstart, Cq, qlist, nq, qself, g, s_pad, r2, support, h, invert, out, out_idx, st, done);
}

template <typename T>
void launch_radius_dump(const typename Vec4<T>::type* C, const uint32_t* Corder,
                        const uint32_t* Cstart, const GridGeom& g, const double* Q, uint32_t m,
                        double r, double s_pad, uint64_t* offsets_or_counts, uint32_t* idx,
                        cudaStream_t s) {
    if (!m) return;
    const double r2 = r * r;
    radius_dump_kernel<T><<<blocks_for((uint64_t)m * 32, EX_THREADS), EX_THREADS, 0, s>>>(
        C, Corder, Cstart, g, Q, m, r2, s_pad, offsets_or_counts, idx);
}

void launch_finalize_sweep(RunState* st, SweepSlot* slot, SweepSlot* next, double tol,
                           cudaStream_t s) {
    finalize_kernel<<<1, 1, 0, s>>>(st, slot, next, tol);
}

template <typename T>
void launch_unpermute(const typename Vec4<T>::type* X, const uint32_t* orig, uint32_t mpad,
                      double* out, cudaStream_t s) {
    if (!mpad) return;
    unpermute_kernel<typename Vec4<T>::type><<<blocks_for(mpad, 256), 256, 0, s>>>(X, orig, mpad, out);
}

void launch_iso_to_orig(const uint8_t* ever, const uint32_t* orig, uint32_t mpad, uint8_t* out,
                        cudaStream_t s) {
    if (!mpad) return;
    iso_to_orig_kernel<<<blocks_for(mpad, 256), 256, 0, s>>>(ever, orig, mpad, out);
}


template <typename T>
void launch_scatter_init(const typename Vec4<T>::type* X0, const uint32_t* iof, uint32_t m,
                         typename Vec4<T>::type* X, cudaStream_t s) {
    if (!m) return;
    scatter_init_kernel<typename Vec4<T>::type><<<blocks_for(m, 256), 256, 0, s>>>(X0, iof, m, X);
}

template <typename T>
void launch_fill_invalid(typename Vec4<T>::type* X, uint32_t mpad, const uint32_t* orig,
                         cudaStream_t s) {
    if (!mpad) return;
    fill_invalid_kernel<typename Vec4<T>::type, T><<<blocks_for(mpad, 256), 256, 0, s>>>(X, mpad, orig);
}

// Work estimate of an X0 point for the sharded layout: the data points the
// fused kernel would stage for this point alone — every grid row (y, z) within
// the support, trimmed in x to the point's ball chord through the row (the
// kernel's per-row trimming, lop_fast.cu row_range, for a group of one) — plus
// a per-query constant for the group setup.  Unlike a plain density count it
// sees the surface's slope against the rows (measured: config 3's middle
// z-slab costs ~6% more per interaction than the others).
template <typename V>
__global__ void shard_work_kernel(const V* __restrict__ X0, uint32_t m, GridGeom g, double s_pad,
                                  float per_query, const uint32_t* __restrict__ Pstart,
                                  float* __restrict__ w) {
    const int R = (int)ceil(s_pad * g.inv_cs);
    const double r2 = s_pad * s_pad;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
        const V p = X0[i];
        const double px = (double)p.x, py = (double)p.y, pz = (double)p.z;
        const int cy = cell_coord(py, g.oy, g.inv_cs, g.gy);
        const int cz = cell_coord(pz, g.oz, g.inv_cs, g.gz);
        uint32_t cnt = 0;
        for (int z = max(cz - R, 0); z <= min(cz + R, g.gz - 1); ++z) {
            const double z0 = g.oz + g.cs * (double)z, z1 = z0 + g.cs;
            const double gz = fmax(0.0, fmax(z0 - pz, pz - z1));
            for (int y = max(cy - R, 0); y <= min(cy + R, g.gy - 1); ++y) {
                const double y0 = g.oy + g.cs * (double)y, y1 = y0 + g.cs;
                const double gy = fmax(0.0, fmax(y0 - py, py - y1));
                const double rem = r2 - gy * gy - gz * gz;
                if (rem < 0.0) continue;
                const double hx = sqrt(rem);
                const int lx = cell_coord(px - hx, g.ox, g.inv_csx, g.gx);
                const int hxc = cell_coord(px + hx, g.ox, g.inv_csx, g.gx);
                const uint32_t base = ((uint32_t)z * (uint32_t)g.gy + (uint32_t)y) * (uint32_t)g.gx;
                cnt += Pstart[base + hxc + 1] - Pstart[base + lx];
            }
        }
        w[i] = per_query + (float)cnt;
    }
}

template <typename T>
void launch_shard_work(const typename Vec4<T>::type* X0, uint32_t m, const GridGeom& g,
                       double s_pad, const uint32_t* Pstart, float* w, cudaStream_t s) {
    if (!m) return;
    static const float per_query = [] {  // developer knob: per-query constant of the estimate
        const char* e = dev_knob("PCSB_SHARD_C");
        return e ? (float)std::atof(e) : 64.0f;
    }();
    shard_work_kernel<typename Vec4<T>::type><<<blocks_for(m, 256), 256, 0, s>>>(
        X0, m, g, s_pad, per_query, Pstart, w);
}

#define PCSB_INST(T)                                                                              \
    template void launch_exact<T>(const ExactArgs<T>&, int, cudaStream_t);                       \
    template void launch_shard_work<T>(const Vec4<T>::type*, uint32_t, const GridGeom&, double,   \
                                       const uint32_t*, float*, cudaStream_t);                    \
    template void launch_exact_density<T>(const Vec4<T>::type*, const uint32_t*,                 \
                                          const Vec4<T>::type*, const uint32_t*, uint32_t,        \
                                          const uint32_t*, const GridGeom&, double, double,       \
                                          double, double, int, Vec4<T>::type*, const uint32_t*,   \
                                          RunState*, const uint32_t*, cudaStream_t);              \
    template void launch_radius_dump<T>(const Vec4<T>::type*, const uint32_t*, const uint32_t*,   \
                                        const GridGeom&, const double*, uint32_t, double, double, \
                                        uint64_t*, uint32_t*, cudaStream_t);                      \
    template void launch_unpermute<T>(const Vec4<T>::type*, const uint32_t*, uint32_t, double*,   \
                                      cudaStream_t);                                              \
    template void launch_scatter_init<T>(const Vec4<T>::type*, const uint32_t*, uint32_t,         \
                                         Vec4<T>::type*, cudaStream_t);                           \
    template void launch_fill_invalid<T>(Vec4<T>::type*, uint32_t, const uint32_t*, cudaStream_t);
PCSB_INST(float)
PCSB_INST(double)
#undef PCSB_INST

}  // namespace pcsb
