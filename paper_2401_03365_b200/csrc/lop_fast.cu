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

#ifndef PCSB_FAST_MINB
#define PCSB_FAST_MINB 6
#endif
constexpr int FAST_WARPS = 4;
constexpr int FAST_THREADS = FAST_WARPS * 32;
constexpr int BUF = 256;     // staged candidates per warp (float4)
constexpr int RING = 4;      // cp.async pipeline depth: 32-candidate chunks in flight per warp
// Unrolled pairs per lane step: L*UNROLL = 16 pairs, so the bank swizzle of the
// staging layout (bit 3 of the pair index) is a compile-time constant per step.
template <int L> struct Unroll { static constexpr int value = 16 / L; };
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

// Staging layout (per warp, BUF candidates): PAIR-INTERLEAVED so that one lane
// evaluates two candidates with packed fp32x2 instructions, and BANK-SWIZZLED so
// that the scalar stores of 32 consecutive candidates hit 32 distinct banks:
//   AX = float4[BUF/2]: pair j = (x0 x1 y0 y1), BZ = float4[BUF/2]: (z0 z1 w0 w1),
//   with the two halves swapped when bit 3 of j is set.
__device__ __forceinline__ int stage_word(int k, int comp) {
    const int j = k >> 1;
    return j * 4 + 2 * (comp ^ ((j >> 3) & 1)) + (k & 1);
}

__device__ __forceinline__ void stage_store(float4* buf, int k, const float4& c) {
    float* ax = reinterpret_cast<float*>(buf);
    float* bz = reinterpret_cast<float*>(buf + BUF / 2);
    ax[stage_word(k, 0)] = c.x;
    ax[stage_word(k, 1)] = c.y;
    bz[stage_word(k, 0)] = c.z;
    bz[stage_word(k, 1)] = c.w;
}

__device__ __forceinline__ float4 stage_load(const float4* buf, int k) {
    const float* ax = reinterpret_cast<const float*>(buf);
    const float* bz = reinterpret_cast<const float*>(buf + BUF / 2);
    return make_float4(ax[stage_word(k, 0)], ax[stage_word(k, 1)], bz[stage_word(k, 0)],
                       bz[stage_word(k, 1)]);
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
                                                  float4* /*ring*/, int lane, Eval&& eval) {
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
                if (keep) stage_store(buf, count + __popc(m & lt), c);
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

// ---------------------------------------------------------------------------
// Evaluation of a staged buffer.  Candidates sit in PAIR-INTERLEAVED layout
// (pair j = 32 bytes: x0 x1 y0 y1 | z0 z1 w0 w1) so that one lane evaluates two
// candidates per iteration with packed fp32x2 instructions (FADD2/FMUL2/FFMA2:
// half the issue slots of scalar FP32).  Per pair: 2 LDS.128, 3+3 packed ops
// for d2, 1 FFMA2 for the exponent, 4 MUFU (2x EX2, 2x RSQ), 2 FSETP + 2 FSEL
// for the hit mask, 1 FMUL2 and 4 packed accumulations.
// ---------------------------------------------------------------------------
enum : int { K_ATTR = 0, K_REP_INVCUBE = 1, K_REP_NEGLIN = 2, K_DENSITY = 3 };

struct Acc {
    float2 s, x, y, z;  // sum w, sum w*(c - q), per candidate parity
    float2 n2;          // hits, per candidate parity
    float n, nr;        // hits (after reduction), candidates in range (incl. zero distance)
};

__device__ __forceinline__ Acc acc_zero() {
    Acc A;
    A.s = A.x = A.y = A.z = A.n2 = make_float2(0.f, 0.f);
    A.n = A.nr = 0.f;
    return A;
}

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }

struct EvalConsts {
    float2 nqx, nqy, nqz;  // -q
    float2 kneg, K0;
    float support;
};

// Pads the buffer (count candidates) to a multiple of 32 (16 pairs) with far
// dummies; returns the number of pairs.
__device__ __forceinline__ int pad_pairs(float4* buf, int count, int lane) {
    const int padded = (count + 31) & ~31;
    if (count + lane < padded) stage_store(buf, count + lane, make_float4(kFar, kFar, kFar, 0.f));
    __syncwarp();
    return padded >> 1;
}

// weight of one candidate given its hit predicate (kind-specific); vectorised over a pair
template <int KIND, bool kWlop, bool kZero>
__device__ __forceinline__ float2 pair_weight(const float2& d2, const float2& arg, bool px, bool py,
                                              const float4& B, const EvalConsts& ec) {
    float2 w;
    if (KIND == K_DENSITY) {
        w = f2(px ? ex2_approx(arg.x) : 0.f, py ? ex2_approx(arg.y) : 0.f);
        return w;
    }
    // kZero: zero-distance candidates are masked out, so keep their rsqrt finite
    // (0 * inf would poison the sums); otherwise a zero distance is a hit whose
    // infinite weight surfaces as a non-finite sum and defers the query
    const float2 d2s = kZero ? f2(fmaxf(d2.x, 1e-37f), fmaxf(d2.y, 1e-37f)) : d2;
    const float2 rs = f2(rsqrt_approx(d2s.x), rsqrt_approx(d2s.y));
    if (KIND == K_REP_INVCUBE) {
        // theta/d^5 scaled by s^5 = theta * (s/d)^5 (no fp32 overflow)
        const float2 a2 = __fmul2_rn(d2, ec.kneg);
        const float2 th = f2(px ? ex2_approx(a2.x) : 0.f, py ? ex2_approx(a2.y) : 0.f);
        const float2 u = __fmul2_rn(rs, f2(ec.support, ec.support));
        const float2 u2 = __fmul2_rn(u, u);
        w = __fmul2_rn(__fmul2_rn(__fmul2_rn(th, u2), u2), u);
    } else {
        // alpha = theta/d (attraction) or beta = theta*1/d (eta = -r), theta scaled by 2^K0
        const float2 th = f2(px ? ex2_approx(arg.x) : 0.f, py ? ex2_approx(arg.y) : 0.f);
        w = __fmul2_rn(th, rs);
    }
    if (kWlop) w = __fmul2_rn(w, f2(B.z, B.w));  // 1/v_j (attraction) | w_i' (repulsion)
    return w;
}

// kZero: exclude d2 == 0 from the hits (and count in-range candidates in nr).
template <int L, int KIND, bool kWlop, bool kZero>
__device__ __forceinline__ void eval_pairs(const float4* __restrict__ pb, int npairs, int sub,
                                           const EvalConsts& ec, Acc& A, float& bmin) {
    constexpr int U = Unroll<L>::value;
    const float4* ax = pb;
    const float4* bz = pb + BUF / 2;
    for (int j0 = sub; j0 < npairs; j0 += L * U) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int j = j0 + u * L;
            // j0 = sub + 16 t with sub < L, so bit 3 of j is that of u*L: a constant
            constexpr bool kSw = false;
            const bool sw = kSw || (((u * L) >> 3) & 1);
            const float4 Ar = ax[j], Br = bz[j];
            const float4 Apos = sw ? make_float4(Ar.z, Ar.w, Ar.x, Ar.y) : Ar;
            const float4 B = sw ? make_float4(Br.z, Br.w, Br.x, Br.y) : Br;
            const float2 dx = __fadd2_rn(f2(Apos.x, Apos.y), ec.nqx);
            const float2 dy = __fadd2_rn(f2(Apos.z, Apos.w), ec.nqy);
            const float2 dz = __fadd2_rn(f2(B.x, B.y), ec.nqz);
            float2 d2 = __fmul2_rn(dx, dx);
            d2 = __ffma2_rn(dy, dy, d2);
            d2 = __ffma2_rn(dz, dz, d2);
            const float2 arg = __ffma2_rn(d2, ec.kneg, ec.K0);  // >= 0 <=> d2 <= r2 (fp32)
            bmin = fminf(bmin, fminf(fabsf(arg.x), fabsf(arg.y)));
            bool px = arg.x >= 0.f, py = arg.y >= 0.f;
            if (kZero) {
                A.nr += (px ? 1.f : 0.f) + (py ? 1.f : 0.f);
                px = px && d2.x > 0.f;
                py = py && d2.y > 0.f;
            }
            const float2 w = pair_weight<KIND, kWlop, kZero>(d2, arg, px, py, B, ec);
            A.n2 = __fadd2_rn(A.n2, f2(px ? 1.f : 0.f, py ? 1.f : 0.f));
            A.s = __fadd2_rn(A.s, w);
            if (KIND != K_DENSITY) {
                A.x = __ffma2_rn(w, dx, A.x);
                A.y = __ffma2_rn(w, dy, A.y);
                A.z = __ffma2_rn(w, dz, A.z);
            }
        }
    }
}

// Exact fp64 re-decision of the guard-band pairs of one buffer: a candidate
// whose fp32 decision differs from the reference predicate (d2 <= r*r in fp64,
// proj/src/spatial.cpp:89,101) has its contribution added or removed.  The
// weights are recomputed with the very same fp32 operations as eval_pairs.
template <int L, int KIND, bool kWlop, bool kZero>
__device__ __forceinline__ void fix_band(const float4* buf, int npairs, int sub, const float4& q,
                                         const EvalConsts& ec, float band, double r2, Acc& A) {
    // candidate k sits in pair k/2, evaluated by lane sub == (k/2) % L
    for (int j = sub; j < npairs; j += L)
        for (int h = 0; h < 2; ++h) {
        const float4 cc = stage_load(buf, 2 * j + h);
        const float cx = cc.x, cy = cc.y, cz = cc.z, cw = cc.w;
        const float dx = cx - q.x, dy = cy - q.y, dz = cz - q.z;
        const float d2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
        const float arg = fmaf(d2, ec.kneg.x, ec.K0.x);
        if (!(fabsf(arg) <= band)) continue;
        const bool exact = exact_d2(cx, cy, cz, q.x, q.y, q.z) <= r2;
        const bool fp32 = arg >= 0.f;
        if (exact == fp32) continue;
        // (the accumulators are per candidate parity h; any slot of the lane works)
        const float sgn = exact ? 1.f : -1.f;
        const float4 B = make_float4(cz, cz, cw, cw);
        const float2 w2 = pair_weight<KIND, kWlop, kZero>(f2(d2, d2), f2(arg, arg), true, true, B, ec);
        if (kZero) A.nr += sgn;
        if (!kZero || d2 > 0.f) {
            const float w = w2.x * sgn;
            A.n2.x += sgn;
            A.s.x += w;
            if (KIND != K_DENSITY) {
                A.x.x = fmaf(w, dx, A.x.x);
                A.y.x = fmaf(w, dy, A.y.x);
                A.z.x = fmaf(w, dz, A.z.x);
            }
        }
        }
}

// One buffer: pad, evaluate, re-decide the band if any lane saw a band pair.
template <int L, int KIND, bool kWlop, bool kZero>
__device__ __forceinline__ int eval_buffer(float4* buf, int count, int lane, int sub,
                                           const float4& q, const EvalConsts& ec, float band,
                                           double r2, Acc& A) {
    const int npairs = pad_pairs(buf, count, lane);
    float bmin = INFINITY;
    eval_pairs<L, KIND, kWlop, kZero>(buf, npairs, sub, ec, A, bmin);
    if (__any_sync(0xffffffffu, bmin <= band))
        fix_band<L, KIND, kWlop, kZero>(buf, npairs, sub, q, ec, band, r2, A);
    return 2 * npairs;
}

template <int L>
__device__ __forceinline__ void group_reduce(Acc& A, bool with_nr) {
    A.s.x = group_sum<L>(A.s.x + A.s.y);
    A.x.x = group_sum<L>(A.x.x + A.x.y);
    A.y.x = group_sum<L>(A.y.x + A.y.y);
    A.z.x = group_sum<L>(A.z.x + A.z.y);
    A.n = group_sum<L>(A.n2.x + A.n2.y);
    if (with_nr) A.nr = group_sum<L>(A.nr);
}

__device__ __forceinline__ EvalConsts make_consts(const float4& q, float kneg, float K0,
                                                  float support) {
    EvalConsts ec;
    ec.nqx = f2(-q.x, -q.x);
    ec.nqy = f2(-q.y, -q.y);
    ec.nqz = f2(-q.z, -q.z);
    ec.kneg = f2(kneg, kneg);
    ec.K0 = f2(K0, K0);
    ec.support = support;
    return ec;
}

template <int L, bool kWlop, bool kCheckZero, int kRep>
__global__ void __launch_bounds__(FAST_THREADS, PCSB_FAST_MINB)
fast_kernel(const FastArgs a) {
    constexpr int Q = 32 / L;
    constexpr int KREP = kRep == 1 ? K_REP_INVCUBE : K_REP_NEGLIN;
    __shared__ float4 smem[FAST_WARPS * (BUF + RING * 32)];
    if (*a.done) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float4* buf = smem + warp * (BUF + RING * 32);
    float4* ring = buf + BUF;
    const int sub = lane % L;
    const uint32_t ngroups = (a.nq + Q - 1) / Q;

    for (;;) {
        uint32_t grp = 0;
        if (lane == 0) grp = atomicAdd(&a.slot->group_counter, 1u);
        grp = __shfl_sync(0xffffffffu, grp, 0);
        if (grp >= ngroups) break;
        const Group<L> G = load_group<L>(grp, a.nq, a.qlist, a.Xs, a.Xskeys, a.g, lane);
        const float4 q = G.q;
        const EvalConsts ec = make_consts(q, a.kneg, a.K0, a.support);

        for (int sg = 0; sg < G.nseg; ++sg) {
            const bool member = G.qvalid && G.seg == sg;
            const Box box = member_box(q, member);
            const CellRange cr = cell_range(a.g, box, a.s_pad);

            // ---------------- attraction: data candidates (lop.cpp:49-65) ----------------
            Acc at = acc_zero();
            uint32_t evals = 0;  // buffered candidates evaluated by this segment (x Q queries)
            stream_candidates(a.P, a.Pstart, a.g, cr, box, a.scull2, buf, ring, lane, [&](int count) {
                evals += eval_buffer<L, K_ATTR, kWlop, kCheckZero>(buf, count, lane, sub, q, ec,
                                                                   a.band, a.r2, at);
            });

            // ---------------- repulsion: projected-set candidates (lop.cpp:79-97) ----------------
            Acc rp = acc_zero();
            if (kRep != 0) {
                stream_candidates(a.Xs, a.Xstart, a.g, cr, box, a.scull2, buf, ring, lane, [&](int count) {
                    evals += eval_buffer<L, KREP, kWlop, true>(buf, count, lane, sub, q, ec, a.band,
                                                               a.r2, rp);
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
                const float sa = at.s.x;
                bool bad = !isfinite(sa) || !isfinite(at.x.x) || !isfinite(at.y.x) ||
                           !isfinite(at.z.x);
                const float zeros = kCheckZero ? (at.nr - at.n) : 0.f;
                if (kCheckZero && zeros > 0.f) {
                    // an fp32 d2 of 0 could hide a distinct pair only for tiny coordinates
                    const float tiny = 0x1p-40f;
                    if (fabsf(q.x) < tiny || fabsf(q.y) < tiny || fabsf(q.z) < tiny) bad = true;
                }
                const bool attracted = sa > 0.f;
                if (kRep != 0 && attracted) {
                    // exactly one zero-distance candidate must remain: the query itself;
                    // any other is a coincident pair, counted by the exact path
                    const float z = rp.nr - rp.n;
                    bad = bad || !isfinite(rp.s.x) || !isfinite(rp.x.x) || !isfinite(rp.y.x) ||
                          !isfinite(rp.z.x) || z > 1.5f || z < 0.5f;
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
                        const float inv = 1.0f / sa;  // Weiszfeld quotient (lop.cpp:77)
                        nx = q.x + at.x.x * inv;
                        ny = q.y + at.y.x * inv;
                        nz = q.z + at.z.x * inv;
                        n_attr = (unsigned long long)at.n;
                        if (kRep != 0) {
                            n_rep = (unsigned long long)rp.n;
                            if (rp.s.x > 0.f) {  // lop.cpp:95-96, x - x' = -(c - q)
                                const float f = a.mu / rp.s.x;
                                nx = fmaf(-f, rp.x.x, nx);
                                ny = fmaf(-f, rp.y.x, ny);
                                nz = fmaf(-f, rp.z.x, nz);
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
                atomicAdd(&a.st->lane_candidates, (unsigned long long)evals * Q);
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
    __shared__ float4 smem[FAST_WARPS * (BUF + RING * 32)];
    constexpr int Q = 32 / DL;
    if (a.done && *a.done) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float4* buf = smem + warp * (BUF + RING * 32);
    float4* ring = buf + BUF;
    const int sub = lane % DL;
    const uint32_t ngroups = (a.nq + Q - 1) / Q;
    for (;;) {
        uint32_t grp = 0;
        if (lane == 0) grp = atomicAdd(a.counter, 1u);
        grp = __shfl_sync(0xffffffffu, grp, 0);
        if (grp >= ngroups) break;
        const Group<DL> G = load_group<DL>(grp, a.nq, a.qlist, a.C, a.Cskeys, a.g, lane);
        const float4 q = G.q;
        const EvalConsts ec = make_consts(q, a.kneg, a.K0, 0.f);
        for (int sg = 0; sg < G.nseg; ++sg) {
            const bool member = G.qvalid && G.seg == sg;
            const Box box = member_box(q, member);
            const CellRange cr = cell_range(a.g, box, a.s_pad);
            Acc A = acc_zero();
            stream_candidates(a.C, a.Cstart, a.g, cr, box, a.scull2, buf, ring, lane, [&](int count) {
                eval_buffer<DL, K_DENSITY, false, true>(buf, count, lane, sub, q, ec, a.band, a.r2, A);
            });
            A.s.x = group_sum<DL>(A.s.x + A.s.y);
            A.n = group_sum<DL>(A.n2.x + A.n2.y);
            A.nr = group_sum<DL>(A.nr);
            unsigned long long pairs = 0;
            if (member && sub == 0) {
                // theta(0) = 1 for coincident duplicates; minus one for the point itself
                const float dens = 1.0f + A.s.x * a.inv_scale + (A.nr - A.n - 1.0f);
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
