// lop_fast.cu — the fused per-point LOP/WLOP kernel (fp32, SFU/FP32-bound).
//
// Replaces the per-point body of the reference sweep, proj/src/lop.cpp:41-100
// (attraction :49-65, isolation/anchor :67-75, Weiszfeld quotient :77,
// repulsion :79-97), with one persistent warp-cooperative kernel:
//
//  * A warp takes a GROUP of Q = 32/L consecutive queries of the cell-sorted
//    projected set (L lanes per query).  Groups are fetched dynamically
//    (atomic counter) so density imbalance self-schedules.  A group is split
//    into SEGMENTS of queries that sit in one cell row and in adjacent cells,
//    so a segment's bounding box is at most a few cells wide.
//  * For each segment the warp walks the cell rows that can hold a point within
//    the support of the box (each row is ONE contiguous run of the sorted
//    array), streams the run with coalesced float4 loads, culls every
//    candidate against the box once, and compacts the survivors into a
//    per-warp shared-memory buffer (ballot + popc).
//  * Each lane then evaluates its query against every L-th buffered candidate
//    (shared-memory broadcast, one wavefront per LDS.128): d2 with FFMA,
//    theta with MUFU.EX2, 1/d with MUFU.RSQ, predicated accumulation.
//  * The reference's exact neighbour predicate (fp64, d2 <= r*r,
//    proj/src/spatial.cpp:89,101) is reproduced by deciding in fp32 and
//    re-deciding in fp64, in-kernel, every pair that falls in a guard band
//    around the support (a warp vote keeps that path off the common case).
//    Queries that meet an exact zero distance in the attraction (sweeps >= 2),
//    a coincident projected pair, or a non-finite sum are deferred to the exact
//    fp64 kernel (lop_exact.cu).  The neighbour SET is always the reference's.
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

// Bounding box over the member lanes of the current segment.
__device__ __forceinline__ Box member_box(const float4& q, bool member) {
    Box b;
    b.mnx = warp_min(member ? q.x : INFINITY);
    b.mny = warp_min(member ? q.y : INFINITY);
    b.mnz = warp_min(member ? q.z : INFINITY);
    b.mxx = warp_max(member ? q.x : -INFINITY);
    b.mxy = warp_max(member ? q.y : -INFINITY);
    b.mxz = warp_max(member ? q.z : -INFINITY);
    return b;
}

// Query group of Q = 32/L consecutive sorted slots, split into segments of
// queries in the same cell row whose x cells are at most one apart.
template <int L>
struct Group {
    uint32_t qslot;
    float4 q;
    bool qvalid;
    int seg;
    int nseg;
};

template <int L>
__device__ __forceinline__ Group<L> load_group(uint32_t grp, uint32_t nq, const uint32_t* qlist,
                                               const float4* __restrict__ pts,
                                               const uint32_t* __restrict__ skeys,
                                               const GridGeom& g, int lane) {
    constexpr int Q = 32 / L;
    Group<L> G;
    const int qi = lane / L, sub = lane % L;
    const uint32_t qpos = grp * Q + qi;
    G.qvalid = qpos < nq;
    const uint32_t qp = G.qvalid ? qpos : grp * Q;  // padding lanes duplicate query 0
    G.qslot = qlist ? __ldg(&qlist[qp]) : qp;
    G.q = __ldg(&pts[G.qslot]);
    const uint32_t cell = __ldg(&skeys[G.qslot]) >> (3 * g.sub_bits);
    const uint32_t row = cell / (uint32_t)g.gx;
    const uint32_t cx = cell - row * (uint32_t)g.gx;
    const int src = qi > 0 ? (qi - 1) * L : 0;
    const uint32_t prow = __shfl_sync(0xffffffffu, row, src);
    const uint32_t pcx = __shfl_sync(0xffffffffu, cx, src);
    const bool start = G.qvalid && (qi == 0 || row != prow || cx > pcx + 1 || cx < pcx);
    const unsigned smask = __ballot_sync(0xffffffffu, start && sub == 0);
    G.nseg = __popc(smask);
    G.seg = __popc(smask & (unsigned)((2ull << (qi * L)) - 1ull)) - 1;
    return G;
}

// Streams every candidate of the rows covered by `cr`, culls it against the
// box and hands full buffers to `eval(count)`.  Warp-uniform control flow.
// The next 32-candidate chunk of a row is loaded before the current one is
// culled (one chunk of prefetch per lane hides most of the L2 latency).
template <typename Eval>
__device__ __forceinline__ void stream_candidates(const float4* __restrict__ src,
                                                  const uint32_t* __restrict__ start,
                                                  const GridGeom& g, const CellRange& cr,
                                                  const Box& b, float scull2, float4* buf,
                                                  int lane, Eval&& eval) {
    const int ny = cr.hiy - cr.loy + 1;
    const int nrows = ny * (cr.hiz - cr.loz + 1);
    const unsigned lt = (1u << lane) - 1u;
    const float4 far4 = make_float4(kFar, kFar, kFar, 0.f);
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
            if (b0 >= e0) continue;
            float4 c = (b0 + lane < e0) ? __ldg(&src[b0 + lane]) : far4;
            for (uint32_t k = b0; k < e0; k += 32) {
                const uint32_t kn = k + 32 + lane;
                const float4 cn = (kn < e0) ? __ldg(&src[kn]) : far4;
                const float ex = fmaxf(fmaxf(b.mnx - c.x, c.x - b.mxx), 0.f);
                const float ey = fmaxf(fmaxf(b.mny - c.y, c.y - b.mxy), 0.f);
                const float ez = fmaxf(fmaxf(b.mnz - c.z, c.z - b.mxz), 0.f);
                const bool keep = fmaf(ez, ez, fmaf(ey, ey, ex * ex)) <= scull2;
                const unsigned m = __ballot_sync(0xffffffffu, keep);
                if (keep) buf[count + __popc(m & lt)] = c;
                count += __popc(m);
                if (count > BUF - 32) {
                    __syncwarp();
                    eval(count);
                    __syncwarp();
                    count = 0;
                }
                c = cn;
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

// Accumulators of one query (per lane partial sums).
struct Acc {
    float s, n, x, y, z;  // sum w, #hits, sum w*(c - q)
    float nr;             // candidates with d2 <= r2 (incl. zero distance)
};

// The kernel of every pass: the in-range decision is made in fp32 on
// arg = fma(d2, kneg, K0) >= 0.  `bmin` tracks min |arg| so that, once per
// buffer, pairs inside the guard band can be re-decided exactly in fp64 (rare).
template <int L, typename Weight>
__device__ __forceinline__ void eval_buffer(const float4* buf, int padded, int sub,
                                            const float4& q, float kneg, float K0,
                                            bool count_range, Acc& A, float& bmin, Weight&& wfn) {
    for (int k = sub; k < padded; k += L * UNROLL) {
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            const float4 c = buf[k + u * L];
            const float dx = c.x - q.x, dy = c.y - q.y, dz = c.z - q.z;
            const float d2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
            const float arg = fmaf(d2, kneg, K0);
            bmin = fminf(bmin, fabsf(arg));
            const float w = wfn(c, d2, arg);
            if (arg >= 0.f) {
                if (count_range) A.nr += 1.f;
                if (!count_range || d2 > 0.f) {
                    A.s += w;
                    A.n += 1.f;
                    A.x = fmaf(w, dx, A.x);
                    A.y = fmaf(w, dy, A.y);
                    A.z = fmaf(w, dz, A.z);
                }
            }
        }
    }
}

// Exact fp64 re-decision of the guard-band pairs of one buffer: a pair whose
// fp32 decision differs from the reference predicate (d2 <= r*r in fp64,
// proj/src/spatial.cpp:89,101) has its contribution added or removed.
template <int L, typename Weight>
__device__ __forceinline__ void fix_band(const float4* buf, int padded, int sub, const float4& q,
                                         float kneg, float K0, float band, double r2,
                                         bool count_range, Acc& A, Weight&& wfn) {
    for (int k = sub; k < padded; k += L) {
        const float4 c = buf[k];
        const float dx = c.x - q.x, dy = c.y - q.y, dz = c.z - q.z;
        const float d2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
        const float arg = fmaf(d2, kneg, K0);
        if (!(fabsf(arg) <= band)) continue;
        const bool exact = exact_d2(c.x, c.y, c.z, q.x, q.y, q.z) <= r2;
        const bool fp32 = arg >= 0.f;
        if (exact == fp32) continue;
        const float sgn = exact ? 1.f : -1.f;
        const float w = wfn(c, d2, arg) * sgn;
        if (count_range) A.nr += sgn;
        if (!count_range || d2 > 0.f) {
            A.s += w;
            A.n += sgn;
            A.x = fmaf(w, dx, A.x);
            A.y = fmaf(w, dy, A.y);
            A.z = fmaf(w, dz, A.z);
        }
    }
}

template <int L>
__device__ __forceinline__ void group_reduce(Acc& A, bool with_nr) {
    A.s = group_sum<L>(A.s);
    A.n = group_sum<L>(A.n);
    A.x = group_sum<L>(A.x);
    A.y = group_sum<L>(A.y);
    A.z = group_sum<L>(A.z);
    if (with_nr) A.nr = group_sum<L>(A.nr);
}

template <int L, bool kWlop, bool kCheckZero, int kRep>
__global__ void __launch_bounds__(FAST_THREADS)
fast_kernel(const FastArgs a) {
    constexpr int Q = 32 / L;
    __shared__ float4 smem[FAST_WARPS * BUF];
    if (*a.done) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float4* buf = smem + warp * BUF;
    const int sub = lane % L;
    const uint32_t ngroups = (a.nq + Q - 1) / Q;
    const float kneg = a.kneg, K0 = a.K0;

    // alpha = theta/d (scaled by 2^K0), x (1/v_j) for WLOP     (lop.cpp:62)
    auto w_attr = [&](const float4& c, float d2, float arg) {
        float w = ex2_approx(arg) * rsqrt_approx(d2);
        if (kWlop) w *= c.w;
        return w;
    };
    // beta = theta |eta'| / d, x w_i' for WLOP                   (lop.cpp:90-91)
    auto w_rep = [&](const float4& c, float d2, float arg) {
        const float rs = rsqrt_approx(d2);
        float w;
        if (kRep == 1) {
            // theta/d^5, scaled by s^5: theta * (s/d)^5 (no fp32 overflow)
            const float th = ex2_approx(d2 * kneg);
            const float u1 = rs * a.support;
            const float u2 = u1 * u1;
            w = th * u2 * u2 * u1;
        } else {
            w = ex2_approx(arg) * rs;  // theta/d, scaled by 2^K0
        }
        if (kWlop) w *= c.w;
        return w;
    };

    for (;;) {
        uint32_t grp = 0;
        if (lane == 0) grp = atomicAdd(&a.slot->group_counter, 1u);
        grp = __shfl_sync(0xffffffffu, grp, 0);
        if (grp >= ngroups) break;
        const Group<L> G = load_group<L>(grp, a.nq, a.qlist, a.Xs, a.Xskeys, a.g, lane);
        const float4 q = G.q;

        for (int sg = 0; sg < G.nseg; ++sg) {
            const bool member = G.qvalid && G.seg == sg;
            const Box box = member_box(q, member);
            const CellRange cr = cell_range(a.g, box, a.s_pad);

            // ---------------- attraction: data candidates ----------------
            Acc at{0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            stream_candidates(a.P, a.Pstart, a.g, cr, box, a.scull2, buf, lane, [&](int count) {
                const int padded = pad_buffer<L>(buf, count, lane);
                float bmin = INFINITY;
                eval_buffer<L>(buf, padded, sub, q, kneg, K0, kCheckZero, at, bmin, w_attr);
                if (__any_sync(0xffffffffu, bmin <= a.band))
                    fix_band<L>(buf, padded, sub, q, kneg, K0, a.band, a.r2, kCheckZero, at, w_attr);
            });

            // ---------------- repulsion: projected-set candidates ----------------
            Acc rp{0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            if (kRep != 0) {
                stream_candidates(a.Xs, a.Xstart, a.g, cr, box, a.scull2, buf, lane, [&](int count) {
                    const int padded = pad_buffer<L>(buf, count, lane);
                    float bmin = INFINITY;
                    eval_buffer<L>(buf, padded, sub, q, kneg, K0, true, rp, bmin, w_rep);
                    if (__any_sync(0xffffffffu, bmin <= a.band))
                        fix_band<L>(buf, padded, sub, q, kneg, K0, a.band, a.r2, true, rp, w_rep);
                });
            }

            // ---------------- per-query reduction over its L lanes ----------------
            group_reduce<L>(at, kCheckZero);
            if (kRep != 0) group_reduce<L>(rp, true);

            // ---------------- finalize (lane sub == 0 of each member query) ----------------
            float disp = 0.f;
            unsigned long long n_attr = 0, n_rep = 0;
            if (member && sub == 0) {
                const uint32_t qi_int = __ldg(&a.Xs_idx[G.qslot]);
                bool bad = !isfinite(at.s) || !isfinite(at.x) || !isfinite(at.y) || !isfinite(at.z);
                const float zeros = kCheckZero ? (at.nr - at.n) : 0.f;
                if (kCheckZero && zeros > 0.f) {
                    // an fp32 d2 of 0 could hide a distinct pair only for tiny coordinates
                    const float tiny = 0x1p-50f;
                    if (fabsf(q.x) < tiny || fabsf(q.y) < tiny || fabsf(q.z) < tiny) bad = true;
                }
                const bool attracted = at.s > 0.f;
                if (kRep != 0 && attracted) {
                    // exactly one zero-distance candidate must remain: the query itself;
                    // any other is a coincident pair, counted by the exact path
                    const float z = rp.nr - rp.n;
                    bad = bad || !isfinite(rp.s) || !isfinite(rp.x) || !isfinite(rp.y) ||
                          !isfinite(rp.z) || z > 1.5f || z < 0.5f;
                }
                if (bad) {
                    const uint32_t pos = atomicAdd(&a.slot->careful_count, 1u);
                    a.careful_list[pos] = G.qslot;
                } else {
                    float nx = q.x, ny = q.y, nz = q.z;
                    bool isolated = false;
                    if (!attracted) {
                        // zeros > 0: anchored at the coincident sample, which IS q
                        // (lop.cpp:67-69); otherwise isolated and held (lop.cpp:70-73)
                        isolated = !(kCheckZero && zeros > 0.f);
                    } else {
                        const float inv = 1.0f / at.s;  // Weiszfeld quotient (lop.cpp:77)
                        nx = q.x + at.x * inv;
                        ny = q.y + at.y * inv;
                        nz = q.z + at.z * inv;
                        n_attr = (unsigned long long)at.n;
                        if (kRep != 0) {
                            n_rep = (unsigned long long)rp.n;
                            if (rp.s > 0.f) {  // lop.cpp:95-96, x - x' = -(c - q)
                                const float f = a.mu / rp.s;
                                nx = fmaf(-f, rp.x, nx);
                                ny = fmaf(-f, rp.y, ny);
                                nz = fmaf(-f, rp.z, nz);
                            }
                        }
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
            // warp aggregation of the per-segment statistics
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
}

// ---------------------------------------------------------------------------
// WLOP density pass: dens_i = 1 + sum_{i' != i, d <= s} theta(d)  (fp32,
// exact neighbour set via the same fp64 re-decision of guard-band pairs).
// ---------------------------------------------------------------------------
constexpr int DL = 4;  // lanes per point

__global__ void __launch_bounds__(FAST_THREADS)
density_kernel(const DensityArgs a) {
    __shared__ float4 smem[FAST_WARPS * BUF];
    constexpr int Q = 32 / DL;
    if (a.done && *a.done) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float4* buf = smem + warp * BUF;
    const int sub = lane % DL;
    const uint32_t ngroups = (a.nq + Q - 1) / Q;
    auto w_theta = [&](const float4&, float, float arg) { return ex2_approx(arg); };
    for (;;) {
        uint32_t grp = 0;
        if (lane == 0) grp = atomicAdd(a.counter, 1u);
        grp = __shfl_sync(0xffffffffu, grp, 0);
        if (grp >= ngroups) break;
        const Group<DL> G = load_group<DL>(grp, a.nq, a.qlist, a.C, a.Cskeys, a.g, lane);
        const float4 q = G.q;
        for (int sg = 0; sg < G.nseg; ++sg) {
            const bool member = G.qvalid && G.seg == sg;
            const Box box = member_box(q, member);
            const CellRange cr = cell_range(a.g, box, a.s_pad);
            Acc A{0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            stream_candidates(a.C, a.Cstart, a.g, cr, box, a.scull2, buf, lane, [&](int count) {
                const int padded = pad_buffer<DL>(buf, count, lane);
                float bmin = INFINITY;
                eval_buffer<DL>(buf, padded, sub, q, a.kneg, a.K0, true, A, bmin, w_theta);
                if (__any_sync(0xffffffffu, bmin <= a.band))
                    fix_band<DL>(buf, padded, sub, q, a.kneg, a.K0, a.band, a.r2, true, A, w_theta);
            });
            A.s = group_sum<DL>(A.s);
            A.n = group_sum<DL>(A.n);
            A.nr = group_sum<DL>(A.nr);
            unsigned long long pairs = 0;
            if (member && sub == 0) {
                // theta(0) = 1 for coincident duplicates; minus one for the point itself
                const float dens = 1.0f + A.s * a.inv_scale + (A.nr - A.n - 1.0f);
                const float val = a.invert ? 1.0f / dens : dens;
                if (a.out_sorted) a.out_sorted[G.qslot].w = val;
                else a.out_internal[__ldg(&a.idx[G.qslot])].w = val;
                pairs = (unsigned long long)A.n;
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) pairs += __shfl_xor_sync(0xffffffffu, pairs, o);
            if (lane == 0 && pairs) atomicAdd(&a.st->density_pairs, pairs);
        }
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
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fast_kernel<4, false, false, 2>,
                                                  FAST_THREADS, 0);
    return b > 0 ? b : 1;
}

void launch_density(const DensityArgs& a, int grid_blocks, cudaStream_t s) {
    density_kernel<<<grid_blocks, FAST_THREADS, 0, s>>>(a);
}

}  // namespace pcsb
