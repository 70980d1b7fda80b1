// lop_fast.cu — the fused per-point LOP/WLOP kernel (fp32, SFU/FP32-bound).
//
// Replaces the per-point body of the reference sweep, proj/src/lop.cpp:41-100
// (attraction :49-65, isolation/anchor :67-75, Weiszfeld quotient :77,
// repulsion :79-97), with one persistent warp-cooperative kernel:
//
//  * A warp owns a GROUP of Q = 32/L consecutive queries of the cell-sorted
//    projected set (L lanes per query).  Groups are fetched dynamically
//    (atomic counter) so density imbalance self-schedules.
//  * The warp computes the group's bounding box, walks the cell rows that can
//    hold a point within the support of that box (each row is ONE contiguous
//    run of the sorted array), streams the run with coalesced float4 loads,
//    culls every candidate against the box once, and compacts the survivors
//    into a per-warp shared-memory buffer (ballot + popc).
//  * Each lane then evaluates its query against every L-th buffered candidate
//    (shared-memory broadcast, one wavefront per LDS.128): d2 with FFMA,
//    theta with MUFU.EX2, 1/d with MUFU.RSQ, predicated accumulation.
//  * The exact neighbour predicate of the reference (fp64, d2 <= r*r,
//    proj/src/spatial.cpp:89,101) is reproduced by deciding in fp32 with a
//    guard band: a query that sees any candidate inside the band, a
//    zero-distance attraction candidate (sweeps >= 2), a coincident projected
//    pair or a non-finite sum is deferred to the exact fp64 kernel
//    (lop_exact.cu), so the neighbour SET is always the reference's.
//
// Accumulation is relative to the query (sum alpha*(p - x)), which keeps the
// fp32 rounding error proportional to the support radius rather than to |x|.
#include <cfloat>

#include "common.cuh"
#include "kernels.cuh"

namespace pcsb {

namespace {

constexpr int FAST_WARPS = 4;
constexpr int FAST_THREADS = FAST_WARPS * 32;
constexpr int BUF = 256;     // staged candidates per warp (float4)
constexpr int UNROLL = 4;
constexpr float kFar = 1.0e18f;

struct Box {
    float mnx, mny, mnz, mxx, mxy, mxz;
};

struct CellRange {
    int lox, loy, loz, hix, hiy, hiz;
};

__device__ __forceinline__ float warp_min(float v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

template <int L>
__device__ __forceinline__ float group_sum(float v) {
#pragma unroll
    for (int o = 1; o < L; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
template <int L>
__device__ __forceinline__ int group_or(int v) {
#pragma unroll
    for (int o = 1; o < L; o <<= 1) v |= __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ CellRange cell_range(const GridGeom& g, const Box& b, double s_pad) {
    CellRange r;
    r.lox = cell_coord((double)b.mnx - s_pad, g.ox, g.inv_cs, g.gx);
    r.loy = cell_coord((double)b.mny - s_pad, g.oy, g.inv_cs, g.gy);
    r.loz = cell_coord((double)b.mnz - s_pad, g.oz, g.inv_cs, g.gz);
    r.hix = cell_coord((double)b.mxx + s_pad, g.ox, g.inv_cs, g.gx);
    r.hiy = cell_coord((double)b.mxy + s_pad, g.oy, g.inv_cs, g.gy);
    r.hiz = cell_coord((double)b.mxz + s_pad, g.oz, g.inv_cs, g.gz);
    return r;
}

// Streams every candidate of the rows covered by `cr`, culls it against the
// group box and hands full buffers to `eval(count)`.  Warp-uniform control.
template <typename Eval>
__device__ __forceinline__ void stream_candidates(const float4* __restrict__ src,
                                                  const uint32_t* __restrict__ start,
                                                  const GridGeom& g, const CellRange& cr,
                                                  const Box& b, float scull2, float4* buf,
                                                  int lane, Eval&& eval) {
    const int ny = cr.hiy - cr.loy + 1;
    const int nrows = ny * (cr.hiz - cr.loz + 1);
    const unsigned lt = (1u << lane) - 1u;
    int count = 0;
    for (int r0 = 0; r0 < nrows; r0 += 32) {
        uint32_t rb = 0, re = 0;
        const int r = r0 + lane;
        if (r < nrows) {
            const int yy = cr.loy + r % ny;
            const int zz = cr.loz + r / ny;
            const uint32_t base = ((uint32_t)zz * (uint32_t)g.gy + (uint32_t)yy) * (uint32_t)g.gx;
            rb = __ldg(&start[base + cr.lox]);
            re = __ldg(&start[base + cr.hix + 1]);
        }
        const int nr = min(32, nrows - r0);
        for (int j = 0; j < nr; ++j) {
            const uint32_t b0 = __shfl_sync(0xffffffffu, rb, j);
            const uint32_t e0 = __shfl_sync(0xffffffffu, re, j);
            for (uint32_t k = b0; k < e0; k += 32) {
                const uint32_t idx = k + lane;
                float4 c = make_float4(kFar, kFar, kFar, 0.f);
                const bool in = idx < e0;
                if (in) c = __ldg(&src[idx]);
                const float ex = fmaxf(fmaxf(b.mnx - c.x, c.x - b.mxx), 0.f);
                const float ey = fmaxf(fmaxf(b.mny - c.y, c.y - b.mxy), 0.f);
                const float ez = fmaxf(fmaxf(b.mnz - c.z, c.z - b.mxz), 0.f);
                const bool keep = in && (fmaf(ez, ez, fmaf(ey, ey, ex * ex)) <= scull2);
                const unsigned m = __ballot_sync(0xffffffffu, keep);
                if (keep) buf[count + __popc(m & lt)] = c;
                count += __popc(m);
                if (count > BUF - 32) {
                    __syncwarp();
                    eval(count);
                    __syncwarp();
                    count = 0;
                }
            }
        }
    }
    if (count) {
        __syncwarp();
        eval(count);
        __syncwarp();
    }
}

// Pads the buffer to a multiple of L*UNROLL with far-away dummies.
template <int L>
__device__ __forceinline__ int pad_buffer(float4* buf, int count, int lane) {
    constexpr int STEP = L * UNROLL;
    const int padded = (count + STEP - 1) / STEP * STEP;
    for (int i = count + lane; i < padded; i += 32) buf[i] = make_float4(kFar, kFar, kFar, 0.f);
    __syncwarp();
    return padded;
}

struct AttrAcc {
    float sa, cnt, sx, sy, sz, nr;
    int band;
};

struct RepAcc {
    float sb, cnt, sx, sy, sz, nr;
    int band;
};

template <int L, bool kWlop, bool kCheckZero, int kRep>
__global__ void __launch_bounds__(FAST_THREADS)
fast_kernel(const FastArgs a) {
    constexpr int Q = 32 / L;
    __shared__ float4 smem[FAST_WARPS * BUF];
    if (*a.done) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float4* buf = smem + warp * BUF;
    const int qi = lane / L, sub = lane % L;
    const uint32_t ngroups = (a.nq + Q - 1) / Q;

    for (;;) {
        uint32_t grp = 0;
        if (lane == 0) grp = atomicAdd(&a.slot->group_counter, 1u);
        grp = __shfl_sync(0xffffffffu, grp, 0);
        if (grp >= ngroups) break;

        const uint32_t qpos = grp * Q + qi;
        const bool qvalid = qpos < a.nq;
        const uint32_t qp = qvalid ? qpos : grp * Q;  // duplicates keep the box tight
        const uint32_t qslot = a.qlist ? __ldg(&a.qlist[qp]) : qp;
        const float4 q = __ldg(&a.Xs[qslot]);

        Box box;
        box.mnx = warp_min(q.x); box.mny = warp_min(q.y); box.mnz = warp_min(q.z);
        box.mxx = warp_max(q.x); box.mxy = warp_max(q.y); box.mxz = warp_max(q.z);
        const CellRange cr = cell_range(a.g, box, a.s_pad);

        // ---------------- attraction: data candidates ----------------
        AttrAcc at{0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0};
        auto eval_attr = [&](int count) {
            const int padded = pad_buffer<L>(buf, count, lane);
            for (int k = sub; k < padded; k += L * UNROLL) {
#pragma unroll
                for (int u = 0; u < UNROLL; ++u) {
                    const float4 c = buf[k + u * L];
                    const float dx = c.x - q.x, dy = c.y - q.y, dz = c.z - q.z;
                    const float d2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
                    const float arg = fmaf(d2, a.kneg, a.K0);  // log2 theta + K0; >= 0 <=> hit
                    at.band |= (fabsf(arg) <= a.band);
                    const float rs = rsqrt_approx(d2);
                    float al = ex2_approx(arg) * rs;
                    if (kWlop) al *= c.w;
                    bool hit = arg >= 0.f;
                    if (kCheckZero) {
                        at.nr += hit ? 1.f : 0.f;
                        hit = hit && (d2 > 0.f);
                    }
                    if (hit) {
                        at.sa += al;
                        at.cnt += 1.f;
                        at.sx = fmaf(al, dx, at.sx);
                        at.sy = fmaf(al, dy, at.sy);
                        at.sz = fmaf(al, dz, at.sz);
                    }
                }
            }
        };
        stream_candidates(a.P, a.Pstart, a.g, cr, box, a.scull2, buf, lane, eval_attr);

        // ---------------- repulsion: projected-set candidates ----------------
        RepAcc rp{0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0};
        if (kRep != 0) {
            auto eval_rep = [&](int count) {
                const int padded = pad_buffer<L>(buf, count, lane);
                for (int k = sub; k < padded; k += L * UNROLL) {
#pragma unroll
                    for (int u = 0; u < UNROLL; ++u) {
                        const float4 c = buf[k + u * L];
                        const float dx = c.x - q.x, dy = c.y - q.y, dz = c.z - q.z;
                        const float d2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
                        const float arg = fmaf(d2, a.kneg, a.K0);
                        rp.band |= (fabsf(arg) <= a.band);
                        const float rs = rsqrt_approx(d2);
                        float be;
                        if (kRep == 1) {
                            // theta/d^5, scaled by s^5: theta * (s/d)^5 (no fp32 overflow)
                            const float th = ex2_approx(d2 * a.kneg);
                            const float u1 = rs * a.support;
                            const float u2 = u1 * u1;
                            be = th * u2 * u2 * u1;
                        } else {
                            be = ex2_approx(arg) * rs;  // theta/d (scaled by 2^K0)
                        }
                        if (kWlop) be *= c.w;
                        const bool inr = arg >= 0.f;
                        rp.nr += inr ? 1.f : 0.f;
                        if (inr && d2 > 0.f) {
                            rp.sb += be;
                            rp.cnt += 1.f;
                            rp.sx = fmaf(be, dx, rp.sx);
                            rp.sy = fmaf(be, dy, rp.sy);
                            rp.sz = fmaf(be, dz, rp.sz);
                        }
                    }
                }
            };
            stream_candidates(a.Xs, a.Xstart, a.g, cr, box, a.scull2, buf, lane, eval_rep);
        }

        // ---------------- per-query reduction over its L lanes ----------------
        at.sa = group_sum<L>(at.sa);
        at.cnt = group_sum<L>(at.cnt);
        at.sx = group_sum<L>(at.sx);
        at.sy = group_sum<L>(at.sy);
        at.sz = group_sum<L>(at.sz);
        if (kCheckZero) at.nr = group_sum<L>(at.nr);
        int band = group_or<L>(at.band);
        if (kRep != 0) {
            rp.sb = group_sum<L>(rp.sb);
            rp.cnt = group_sum<L>(rp.cnt);
            rp.sx = group_sum<L>(rp.sx);
            rp.sy = group_sum<L>(rp.sy);
            rp.sz = group_sum<L>(rp.sz);
            rp.nr = group_sum<L>(rp.nr);
            band |= group_or<L>(rp.band);
        }

        // ---------------- finalize (lane sub == 0 of each valid query) ----------------
        const bool leader = qvalid && sub == 0;
        bool isolated = false;
        float disp = 0.f;
        unsigned long long n_attr = 0, n_rep = 0;
        if (leader) {
            const uint32_t qi_int = __ldg(&a.Xs_idx[qslot]);
            bool bad = band != 0 || !isfinite(at.sa) || !isfinite(at.sx) || !isfinite(at.sy) ||
                       !isfinite(at.sz);
            const float zeros = kCheckZero ? (at.nr - at.cnt) : 0.f;
            if (kCheckZero && zeros > 0.f) {
                // d2 == 0 in fp32 could be a distinct pair only if a coordinate is tiny
                const float tiny = 0x1p-50f;
                if (fabsf(q.x) < tiny || fabsf(q.y) < tiny || fabsf(q.z) < tiny) bad = true;
            }
            const bool attracted = at.sa > 0.f;
            if (kRep != 0 && attracted) {
                // exactly one zero-distance candidate must remain: the query itself;
                // any other is a coincident pair, counted by the exact path
                const float z = rp.nr - rp.cnt;
                bad = bad || !isfinite(rp.sb) || !isfinite(rp.sx) || !isfinite(rp.sy) ||
                      !isfinite(rp.sz) || z > 1.5f || z < 0.5f;
            }
            if (bad) {
                const uint32_t pos = atomicAdd(&a.slot->careful_count, 1u);
                a.careful_list[pos] = qslot;
            } else {
                float nx = q.x, ny = q.y, nz = q.z;
                if (!attracted) {
                    // zeros > 0: anchored at the coincident sample, which IS q
                    // (lop.cpp:67-69); otherwise isolated and held (lop.cpp:70-73)
                    if (!(kCheckZero && zeros > 0.f)) isolated = true;
                } else {
                    const float inv = 1.0f / at.sa;
                    nx = q.x + at.sx * inv;
                    ny = q.y + at.sy * inv;
                    nz = q.z + at.sz * inv;
                    n_attr = (unsigned long long)at.cnt;
                    if (kRep != 0 && rp.sb > 0.f) {
                        const float f = a.mu / rp.sb;
                        nx = fmaf(-f, rp.sx, nx);
                        ny = fmaf(-f, rp.sy, ny);
                        nz = fmaf(-f, rp.sz, nz);
                    }
                    if (kRep != 0) n_rep = (unsigned long long)rp.cnt;
                }
                a.Xnext[qi_int] = make_float4(nx, ny, nz, 0.f);
                const float ddx = nx - q.x, ddy = ny - q.y, ddz = nz - q.z;
                disp = sqrtf(fmaf(ddz, ddz, fmaf(ddy, ddy, ddx * ddx)));
                if (isolated) {
                    a.ever_isolated[qi_int] = 1;
                    atomicAdd(&a.st->isolated_events, 1ull);
                }
            }
        }
        // warp aggregation of the per-group statistics
        float md = disp;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            md = fmaxf(md, __shfl_xor_sync(0xffffffffu, md, o));
            n_attr += __shfl_xor_sync(0xffffffffu, n_attr, o);
            n_rep += __shfl_xor_sync(0xffffffffu, n_rep, o);
        }
        if (lane == 0) {
            if (md > 0.f) atomic_max_nonneg_double(&a.slot->max_disp_bits, (double)md);
            if (n_attr) atomicAdd(&a.st->interactions_attr, n_attr);
            if (n_rep) atomicAdd(&a.st->interactions_rep, n_rep);
        }
    }
}

// ---------------------------------------------------------------------------
// WLOP density pass: dens_i = 1 + sum_{i' != i, d <= s} theta(d)  (fp32).
// ---------------------------------------------------------------------------
constexpr int DL = 4;  // lanes per point

__global__ void __launch_bounds__(FAST_THREADS)
density_kernel(const DensityArgs a) {
    constexpr int Q = 32 / DL;
    __shared__ float4 smem[FAST_WARPS * BUF];
    if (a.done && *a.done) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float4* buf = smem + warp * BUF;
    const int qi = lane / DL, sub = lane % DL;
    const uint32_t ngroups = (a.nq + Q - 1) / Q;
    for (;;) {
        uint32_t grp = 0;
        if (lane == 0) grp = atomicAdd(a.counter, 1u);
        grp = __shfl_sync(0xffffffffu, grp, 0);
        if (grp >= ngroups) break;
        const uint32_t qpos = grp * Q + qi;
        const bool qvalid = qpos < a.nq;
        const uint32_t qp = qvalid ? qpos : grp * Q;
        const uint32_t qslot = a.qlist ? __ldg(&a.qlist[qp]) : qp;
        const float4 q = __ldg(&a.C[qslot]);
        Box box;
        box.mnx = warp_min(q.x); box.mny = warp_min(q.y); box.mnz = warp_min(q.z);
        box.mxx = warp_max(q.x); box.mxy = warp_max(q.y); box.mxz = warp_max(q.z);
        const CellRange cr = cell_range(a.g, box, a.s_pad);
        float st = 0.f, nr = 0.f, cnt = 0.f;
        auto eval = [&](int count) {
            const int padded = pad_buffer<DL>(buf, count, lane);
            for (int k = sub; k < padded; k += DL * UNROLL) {
#pragma unroll
                for (int u = 0; u < UNROLL; ++u) {
                    const float4 c = buf[k + u * DL];
                    const float dx = c.x - q.x, dy = c.y - q.y, dz = c.z - q.z;
                    const float d2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
                    const float arg = fmaf(d2, a.kneg, a.K0);
                    const float th = ex2_approx(arg);
                    const bool inr = arg >= 0.f;
                    nr += inr ? 1.f : 0.f;
                    if (inr && d2 > 0.f) {
                        st += th;
                        cnt += 1.f;
                    }
                }
            }
        };
        stream_candidates(a.C, a.Cstart, a.g, cr, box, a.scull2, buf, lane, eval);
        st = group_sum<DL>(st);
        nr = group_sum<DL>(nr);
        cnt = group_sum<DL>(cnt);
        unsigned long long pairs = 0;
        if (qvalid && sub == 0) {
            // theta(0) = 1 for coincident duplicates; minus one for the point itself
            const float dens = 1.0f + st * a.inv_scale + (nr - cnt - 1.0f);
            const float val = a.invert ? 1.0f / dens : dens;
            if (a.out_sorted) a.out_sorted[qslot].w = val;
            else a.out_internal[__ldg(&a.idx[qslot])].w = val;
            pairs = (unsigned long long)cnt;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) pairs += __shfl_xor_sync(0xffffffffu, pairs, o);
        if (lane == 0 && pairs) atomicAdd(&a.st->density_pairs, pairs);
    }
}

template <int L, bool W, bool Z, int R>
void launch_one(const FastArgs& a, int grid, cudaStream_t s) {
    fast_kernel<L, W, Z, R><<<grid, FAST_THREADS, 0, s>>>(a);
}

template <int L>
void launch_l(const FastArgs& a, bool wlop, bool cz, int rep, int grid, cudaStream_t s) {
#define PCSB_DISPATCH(W, Z, R) \
    if (wlop == W && cz == Z && rep == R) return launch_one<L, W, Z, R>(a, grid, s);
    PCSB_DISPATCH(false, false, 0)
    PCSB_DISPATCH(false, false, 1)
    PCSB_DISPATCH(false, false, 2)
    PCSB_DISPATCH(false, true, 0)
    PCSB_DISPATCH(false, true, 1)
    PCSB_DISPATCH(false, true, 2)
    PCSB_DISPATCH(true, false, 0)
    PCSB_DISPATCH(true, false, 1)
    PCSB_DISPATCH(true, false, 2)
    PCSB_DISPATCH(true, true, 0)
    PCSB_DISPATCH(true, true, 1)
    PCSB_DISPATCH(true, true, 2)
#undef PCSB_DISPATCH
}

template <int L, bool W, bool Z, int R>
int occ_one() {
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fast_kernel<L, W, Z, R>, FAST_THREADS, 0);
    return b;
}

}  // namespace

void launch_fast(const FastArgs& a, int lanes_per_point, bool wlop, bool check_zero, int rep_mode,
                 int grid_blocks, cudaStream_t s) {
    switch (lanes_per_point) {
        case 1: return launch_l<1>(a, wlop, check_zero, rep_mode, grid_blocks, s);
        case 2: return launch_l<2>(a, wlop, check_zero, rep_mode, grid_blocks, s);
        case 8: return launch_l<8>(a, wlop, check_zero, rep_mode, grid_blocks, s);
        default: return launch_l<4>(a, wlop, check_zero, rep_mode, grid_blocks, s);
    }
}

int fast_blocks_per_sm(int lanes_per_point, bool wlop, bool check_zero, int rep_mode) {
    (void)lanes_per_point;
    (void)check_zero;
    (void)wlop;
    (void)rep_mode;
    int b = occ_one<4, false, false, 2>();
    return b > 0 ? b : 1;
}

void launch_density(const DensityArgs& a, int grid_blocks, cudaStream_t s) {
    density_kernel<<<grid_blocks, FAST_THREADS, 0, s>>>(a);
}

}  // namespace pcsb
