// lop_fast.cu — the fused per-point LOP/WLOP kernel (fp32, SFU/FP32-bound).
//
// Replaces the per-point body of the reference sweep, proj/src/lop.cpp:41-100
// (attraction :49-65, isolation/anchor :67-75, Weiszfeld quotient :77,
// repulsion :79-97), with one persistent warp-cooperative kernel:
//
//  * Work unit = 16 (or 32) consecutive queries of the Hilbert-ordered query list
//    (build_query_list), fetched by an atomic counter so density imbalance
//    self-schedules; the pass ends on one-group units.  A warp splits its unit
//    into GROUPS of Q = 32/L queries (L lanes per query): runs of the curve cut
//    at curve blocks, or (single-GPU LOP) a recursive bisection of the unit
//    along the longest axis (bisect_unit) — either way a compact box.
//  * Candidates: the cell rows (fixed y, z) within the support of the box, each
//    trimmed in x to the union of the group's queries' ball chords through the
//    row (row_range; no per-candidate cull).  Each row is one contiguous range
//    of 32-byte pair records; a warp streams its rows back to back into one half
//    of a per-warp double buffer with one cp.async.bulk (TMA) per row piece
//    while the other half is evaluated.
//  * Evaluation: two candidates per lane with packed fp32x2 (FADD2/FMUL2/FFMA2),
//    theta on MUFU.EX2, 1/d on MUFU.RSQ, predicated accumulation of
//    sum w (c - q) relative to the query (fp32 error ~ support, not ~ |x|).
//  * The reference's exact neighbour predicate (fp64, d2 <= r*r,
//    proj/src/spatial.cpp:89,101) is reproduced by deciding in fp32 and
//    re-deciding in fp64, in-kernel, every pair within a guard band of the
//    support (a warp vote keeps that path off the common case).  Queries that
//    meet an exact zero distance in the attraction (sweeps >= 2), a coincident
//    projected pair or a non-finite sum are deferred to the exact fp64 kernel
//    (lop_exact.cu).  The neighbour SET is always the reference's.
#include "dev_knobs.h"
#include <algorithm>
#include <cfloat>
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

#ifndef PCSB_FAST_MINB
#define PCSB_FAST_MINB 6
#endif

namespace pcsb {

namespace {

constexpr int FAST_WARPS = 4;
constexpr int FAST_THREADS = FAST_WARPS * 32;
#ifndef PCSB_HR
#define PCSB_HR 128
#endif
constexpr int HR = PCSB_HR;  // pair records per half (2 candidates each; per warp: 2 halves)

constexpr float kFar = 1.0e18f;

// Unrolled records per lane step: L*U = STEP records per warp step.
#ifndef PCSB_STEP
#define PCSB_STEP 16
#endif
constexpr int STEP = PCSB_STEP;
static_assert(HR % STEP == 0, "a half holds whole eval steps");
template <int L> struct Unroll { static constexpr int value = STEP / L; };

struct Box {
    float mnx, mny, mnz, mxx, mxy, mxz;
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

// ---------------------------------------------------------------------------
// Staging: per warp a ring of two halves of HR pair records (kernels.cuh:
// record = (x0 x1 y0 y1)(z0 z1 w0 w1)), filled by bulk asynchronous copies
// (cp.async.bulk, the TMA engine's linear mode) that complete on one mbarrier
// per half.  A candidate row is ONE contiguous range of records, so a row
// costs one copy instruction regardless of its length.  Eval reads records
// with two LDS.128; the L lanes of a query read L consecutive records (32-byte
// stride: conflict-free for L <= 4).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() {
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_LOOP:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_LOOP;\n\t}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}
// generic-proxy accesses of a half before the async proxy rewrites it
__device__ __forceinline__ void fence_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

// Checked builds poison a half with far records once it has been evaluated:
// a later evaluation that reads the half before its bulk copies landed then
// sees points that are never hits, and the exact per-query interaction counts
// of the parity tests expose the missing neighbours.
__device__ __forceinline__ void poison_half(float4* half, int lane) {
#ifdef PCSB_CHECKS
    for (int t = lane; t < 2 * HR; t += 32)
        half[t] = (t & 1) ? make_float4(kFar, kFar, 0.f, 0.f) : make_float4(kFar, kFar, kFar, kFar);
    __syncwarp();
#else
    (void)half;
    (void)lane;
#endif
}

struct Stage {
    float4* ring;     // 2 halves x HR records x 2 float4
    uint32_t ring_s;  // its shared-window address
    uint32_t bar_s;   // two mbarriers (one per half)
    uint32_t phase;   // bit h: parity of the next completion of half h
};

__device__ __forceinline__ Stage make_stage(float4* ring, uint64_t* bars, int lane) {
    Stage S;
    S.ring = ring;
    S.ring_s = (uint32_t)__cvta_generic_to_shared(ring);
    S.bar_s = (uint32_t)__cvta_generic_to_shared(bars);
    S.phase = 0;
    poison_half(ring, lane);
    poison_half(ring + 2 * HR, lane);
    if (lane == 0) {
        mbar_init(S.bar_s, 1);
        mbar_init(S.bar_s + 8, 1);
        mbar_init_fence();
    }
    __syncwarp();
    return S;
}

// candidate k of a staged half (fix-up path)
__device__ __forceinline__ float4 stage_load(const float4* half, int k) {
    const float4 A = half[2 * (k >> 1)];
    const float4 B = half[2 * (k >> 1) + 1];
    return (k & 1) ? make_float4(A.y, A.w, B.y, B.w) : make_float4(A.x, A.z, B.x, B.z);
}

// ---------------------------------------------------------------------------
// Candidate rows of a group: every cell row (y, z) within the support of the
// group's box, each trimmed in x to the union of its queries' ball chords
// (row_range).  A superset of the union of the queries' neighbourhoods.
// ---------------------------------------------------------------------------
struct RowSpan {
    int loy, ny, loz, nrows;
};

__device__ __forceinline__ RowSpan row_span(const GridGeom& g, const Box& b, double s_pad) {
    RowSpan r;
    r.loy = cell_coord((double)b.mny - s_pad, g.oy, g.inv_cs, g.gy);
    const int hiy = cell_coord((double)b.mxy + s_pad, g.oy, g.inv_cs, g.gy);
    r.loz = cell_coord((double)b.mnz - s_pad, g.oz, g.inv_cs, g.gz);
    const int hiz = cell_coord((double)b.mxz + s_pad, g.oz, g.inv_cs, g.gz);
    r.ny = hiy - r.loy + 1;
    r.nrows = r.ny * (hiz - r.loz + 1);
    return r;
}

// The queries of the current group (shared memory) and the squared radius the
// rows are trimmed with: (s_pad + 16 ulp(max |coord|))^2, so that the fp32
// interval arithmetic below stays a superset of the exact neighbourhoods.
struct GroupQ {
    const float4* q;
    int n;
    float cull2;
};

// (begin, end) of row r of the span, in record-slot units; begin == end if the row is
// empty.  The row's x range is the union over the group's queries of the chord
// of each query's ball through the row (gaps to the row's y/z cell intervals;
// boundary cells, which also hold clamped outside points, are unbounded).
__device__ __forceinline__ void row_range(const uint32_t* __restrict__ start, const GridGeom& g,
                                          const GroupQ& G, const RowSpan& rs, int r, uint32_t& rb,
                                          uint32_t& re) {
    rb = re = 0;
    if (r >= rs.nrows) return;
    const int yy = rs.loy + r % rs.ny;
    const int zz = rs.loz + r / rs.ny;
    const float y0 = yy == 0 ? -INFINITY : (float)(g.oy + g.cs * (double)yy);
    const float y1 = yy == g.gy - 1 ? INFINITY : (float)(g.oy + g.cs * (double)(yy + 1));
    const float z0 = zz == 0 ? -INFINITY : (float)(g.oz + g.cs * (double)zz);
    const float z1 = zz == g.gz - 1 ? INFINITY : (float)(g.oz + g.cs * (double)(zz + 1));
    float lo = INFINITY, hi = -INFINITY;
    for (int k = 0; k < G.n; ++k) {
        const float4 q = G.q[k];
        const float gy = fmaxf(0.f, fmaxf(y0 - q.y, q.y - y1));
        const float gz = fmaxf(0.f, fmaxf(z0 - q.z, q.z - z1));
        const float rem = fmaf(-gz, gz, fmaf(-gy, gy, G.cull2));
        if (rem >= 0.f) {
            const float hx = rem > 0.f ? rem * rsqrt_approx(rem) : 0.f;
            lo = fminf(lo, q.x - hx);
            hi = fmaxf(hi, q.x + hx);
        }
    }
    if (!(lo <= hi)) return;
    const int lox = cell_coord((double)lo, g.ox, g.inv_csx, g.gx);
    const int hix = cell_coord((double)hi, g.ox, g.inv_csx, g.gx);
    const uint32_t row = (uint32_t)zz * (uint32_t)g.gy + (uint32_t)yy;
    const uint32_t base = row * (uint32_t)g.gx;
    PCSB_DCHECK(lox <= hix && (uint64_t)base + (uint64_t)hix + 1 <= (uint64_t)g.ncells);
    const uint32_t delta = pair_row_delta(start, row, (uint32_t)g.gx);  // record-slot shift
    rb = __ldg(&start[base + lox]) + delta;
    re = __ldg(&start[base + hix + 1]) + delta;
    PCSB_DCHECK(rb <= re);
}

// Streams every record of the trimmed rows through the double buffer and calls
// eval(half_ptr, nrec) on each full half (nrec = HR) and on the final partial
// one (padded with far records to a multiple of STEP).  The rows of a batch (<=
// 32, one per lane) are laid end to end (warp scan of their record counts);
// each lane copies the part of its row that falls in the current half with ONE
// cp.async.bulk (expect_tx on the half's mbarrier first); lane 0 arrives once
// the half is full.  A half is evaluated after the other half has been filled,
// so its copies had that long to land.
template <typename Eval>
__device__ __forceinline__ void gather_eval(const float4* __restrict__ pairs, size_t pairs_cap,
                                            const uint32_t* __restrict__ start, const GridGeom& g,
                                            const Box& b, double s_pad, const GroupQ& G, Stage& S,
                                            int lane, int rfirst, int rstride, Eval&& eval) {
    (void)pairs_cap;
    const RowSpan rs = row_span(g, b, s_pad);
    uint32_t cur = 0, fill = 0;
    int pending = -1;
    auto finish = [&](uint32_t h, int nrec) {
        PCSB_DCHECK(nrec >= 0 && nrec <= HR && nrec % STEP == 0);
#ifndef PCSB_MUTATE_NO_WAIT  // detector self-test only (tools/gpu_checked.sh): a missing wait
        mbar_wait(S.bar_s + 8u * h, (S.phase >> h) & 1u);
#endif
        S.phase ^= 1u << h;
        eval(S.ring + h * (2 * HR), nrec);
        __syncwarp();
        poison_half(S.ring + h * (2 * HR), lane);
    };
    // rows rfirst, rfirst + rstride, ...: all of them (0, 1), or this warp's share
    // of a tail group whose rows are dealt round robin to rstride warps
    for (int r0 = rfirst; r0 < rs.nrows; r0 += 32 * rstride) {
        uint32_t rb, re;
        row_range(start, g, G, rs, r0 + lane * rstride, rb, re);
        const uint32_t rec0 = rb >> 1;
        const uint32_t nrec = re > rb ? ((re + 1) >> 1) - rec0 : 0u;
        uint32_t incl = nrec;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
        const uint32_t mine0 = incl - nrec;  // my row: batch offsets [mine0, incl)
        for (uint32_t w0 = 0; w0 < total;) {
            const uint32_t w1 = min(total, w0 + (uint32_t)HR - fill);
            const uint32_t lo = max(mine0, w0), hi = min(incl, w1);
            if (lo < hi) {
                PCSB_DCHECK(fill + (lo - w0) + (hi - lo) <= (uint32_t)HR);
                PCSB_DCHECK(2 * ((size_t)rec0 + (hi - mine0)) <= pairs_cap);
                const uint32_t bar = S.bar_s + 8u * cur;
                mbar_expect_tx(bar, (hi - lo) * 32u);
                bulk_g2s(S.ring_s + (cur * HR + fill + (lo - w0)) * 32u,
                         pairs + 2 * (size_t)(rec0 + (lo - mine0)), (hi - lo) * 32u, bar);
            }
            fill += w1 - w0;
            w0 = w1;
            if (fill == HR) {
                __syncwarp();
                if (lane == 0) mbar_arrive(S.bar_s + 8u * cur);
                if (pending >= 0) finish((uint32_t)pending, HR);
                pending = (int)cur;
                cur ^= 1u;
                fill = 0;
                fence_async_smem();
            }
        }
    }
    if (fill > 0) {
        const uint32_t padded = (fill + STEP - 1) / STEP * STEP;
        float4* h = S.ring + cur * (2 * HR);
        for (uint32_t t = 2 * fill + lane; t < 2 * padded; t += 32)
            h[t] = (t & 1) ? make_float4(kFar, kFar, 0.f, 0.f) : make_float4(kFar, kFar, kFar, kFar);
        __syncwarp();
        if (lane == 0) mbar_arrive(S.bar_s + 8u * cur);
        if (pending >= 0) finish((uint32_t)pending, HR);
        finish(cur, (int)padded);
    } else if (pending >= 0) {
        finish((uint32_t)pending, HR);
    }
    fence_async_smem();
}

// ---------------------------------------------------------------------------
// Evaluation of a staged half.  Per record (two candidates, one query): 2 LDS,
// 3+3 packed ops for d2, one FFMA2 for the exponent, 4 MUFU (2x EX2, 2x RSQ),
// one FMUL2 for the weight and 4 packed accumulations — 12 FMA-pipe ops; the
// hit masks, their count and the guard-band minimum run on the integer/ALU
// pipe (FSET, LOP3, IADD3, FMNMX3), which the packed-FMA/MUFU mix leaves idle
// (tools/mix_bench.cu: each packed op removed from the mix is ~0.4 ns/record).
// ---------------------------------------------------------------------------
enum : int { K_ATTR = 0, K_REP_INVCUBE = 1, K_REP_NEGLIN = 2, K_DENSITY = 3 };

struct Acc {
    float2 s, x, y, z;  // sum w, sum w*(c - q), per candidate parity
    int miss;           // -(fp32 decisions "out of range", re-decided in the band)
    int zero;           // -(zero-distance candidates) (kZero)
    int evald;          // candidates evaluated by this lane
    int hneg, rneg;     // after group_reduce: hits (d > 0), in range (incl. d == 0)
};

__device__ __forceinline__ Acc acc_zero() {
    Acc A;
    A.s = A.x = A.y = A.z = make_float2(0.f, 0.f);
    A.miss = A.zero = A.evald = A.hneg = A.rneg = 0;
    return A;
}

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }

__device__ __forceinline__ float2 and2(const float2& v, const uint2& m) {
    return f2(__uint_as_float(__float_as_uint(v.x) & m.x), __uint_as_float(__float_as_uint(v.y) & m.y));
}

struct EvalConsts {
    float2 nqx, nqy, nqz;  // -q
    float2 kneg, K0;
    float support;
};

// The hit mask m (all-ones / zero per candidate) clears theta's bits, so MUFU
// runs unpredicated and a miss contributes exactly +0.
template <int KIND, bool kWlop, bool kZero>
__device__ __forceinline__ float2 pair_weight(const float2& d2, const float2& arg, const uint2& m,
                                              const float4& B, const EvalConsts& ec) {
    float2 w;
    if (KIND == K_DENSITY) return and2(f2(ex2_approx(arg.x), ex2_approx(arg.y)), m);
    // kZero: zero-distance candidates are masked out, so keep their rsqrt finite
    // (0 * inf would poison the sums); otherwise a zero distance is a hit whose
    // infinite weight surfaces as a non-finite sum and defers the query
    const float2 d2s = kZero ? f2(fmaxf(d2.x, 1e-37f), fmaxf(d2.y, 1e-37f)) : d2;
    const float2 rs = f2(rsqrt_approx(d2s.x), rsqrt_approx(d2s.y));
    if (KIND == K_REP_INVCUBE) {
        // theta/d^5 scaled by s^5 = theta * (s/d)^5 (no fp32 overflow)
        const float2 a2 = __fmul2_rn(d2, ec.kneg);
        const float2 th = and2(f2(ex2_approx(a2.x), ex2_approx(a2.y)), m);
        const float2 u = __fmul2_rn(rs, f2(ec.support, ec.support));
        const float2 u2 = __fmul2_rn(u, u);
        w = __fmul2_rn(__fmul2_rn(__fmul2_rn(th, u2), u2), u);
    } else {
        // alpha = theta/d (attraction) or beta = theta*1/d (eta = -r), theta scaled by 2^K0
        w = __fmul2_rn(and2(f2(ex2_approx(arg.x), ex2_approx(arg.y)), m), rs);
    }
    if (kWlop) w = __fmul2_rn(w, f2(B.z, B.w));  // 1/v_j (attraction) | w_i' (repulsion)
    return w;
}

// All-ones iff v < 0: the sign bit spread by one arithmetic shift (inline PTX so
// that it is not turned back into compare + select).  For arg = fma(d2, kneg,
// K0), K0 > 0, this is exactly "arg < 0": arg is never -0 (an exactly
// cancelling fma rounds to +0) and never NaN (candidates and padding are finite).
__device__ __forceinline__ uint32_t sign_mask(float v) {
    uint32_t m;
    asm("shr.s32 %0, %1, 31;" : "=r"(m) : "r"(__float_as_uint(v)));
    return m;
}
// All-ones iff d2 == +0 (d2 >= 0 is a sum of squares).
__device__ __forceinline__ uint32_t zero_mask(float d2) {
    uint32_t m;
    asm("{\n\t.reg .u32 t;\n\tadd.u32 t, %1, 0xffffffff;\n\tshr.s32 %0, t, 31;\n\t}"
        : "=r"(m)
        : "r"(__float_as_uint(d2)));
    return m;
}


// kZero: exclude d2 == 0 from the hits (and count in-range candidates in rneg).
template <int L, int KIND, bool kWlop, bool kZero>
__device__ __forceinline__ void eval_pairs(const float4* __restrict__ pb, int nrec, int sub,
                                           const EvalConsts& ec, Acc& A, float& bmin) {
    constexpr int U = Unroll<L>::value;
    for (int j0 = sub; j0 < nrec; j0 += L * U) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int j = j0 + u * L;
            const float4 Apos = pb[2 * j];
            const float4 B = pb[2 * j + 1];
            const float2 dx = __fadd2_rn(f2(Apos.x, Apos.y), ec.nqx);
            const float2 dy = __fadd2_rn(f2(Apos.z, Apos.w), ec.nqy);
            const float2 dz = __fadd2_rn(f2(B.x, B.y), ec.nqz);
            float2 d2 = __fmul2_rn(dx, dx);
            d2 = __ffma2_rn(dy, dy, d2);
            d2 = __ffma2_rn(dz, dz, d2);
            const float2 arg = __ffma2_rn(d2, ec.kneg, ec.K0);  // >= 0 <=> d2 <= r2 (fp32)
            bmin = fminf(bmin, fminf(fabsf(arg.x), fabsf(arg.y)));
            const uint2 sg = make_uint2(sign_mask(arg.x), sign_mask(arg.y));  // -1: out
            uint2 m = make_uint2(~sg.x, ~sg.y);  // weight mask (folds into LOP3)
            A.miss += (int)sg.x + (int)sg.y;
            if (kZero) {
                const uint2 z = make_uint2(zero_mask(d2.x), zero_mask(d2.y));
                A.zero += (int)z.x + (int)z.y;
                m.x &= ~z.x;
                m.y &= ~z.y;
            }
            const float2 w = pair_weight<KIND, kWlop, kZero>(d2, arg, m, B, ec);
            A.s = __fadd2_rn(A.s, w);
            if (KIND != K_DENSITY) {
                A.x = __ffma2_rn(w, dx, A.x);
                A.y = __ffma2_rn(w, dy, A.y);
                A.z = __ffma2_rn(w, dz, A.z);
            }
        }
    }
}

// Exact fp64 re-decision of the guard-band pairs of one half: a candidate
// whose fp32 decision differs from the reference predicate (d2 <= r*r in fp64,
// proj/src/spatial.cpp:89,101) has its contribution added or removed.  The
// weights are recomputed with the very same fp32 operations as eval_pairs.
template <int L, int KIND, bool kWlop, bool kZero>
__device__ __forceinline__ void fix_band(const float4* buf, int nrec, int sub, const float4& q,
                                         const EvalConsts& ec, float band, double r2, Acc& A) {
    for (int j = sub; j < nrec; j += L) {  // candidate k sits in record k/2, lane (k/2) % L
        for (int h = 0; h < 2; ++h) {
            const float4 cc = stage_load(buf, 2 * j + h);
            const float dx = cc.x - q.x, dy = cc.y - q.y, dz = cc.z - q.z;
            const float d2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
            const float arg = fmaf(d2, ec.kneg.x, ec.K0.x);
            if (!(fabsf(arg) <= band)) continue;
            const bool exact = exact_d2(cc.x, cc.y, cc.z, q.x, q.y, q.z) <= r2;
            const bool fp32 = arg >= 0.f;
            if (exact == fp32) continue;
            const int sgn = exact ? 1 : -1;
            const float4 B = make_float4(cc.z, cc.z, cc.w, cc.w);
            const float2 w2 = pair_weight<KIND, kWlop, kZero>(f2(d2, d2), f2(arg, arg),
                                                              make_uint2(~0u, ~0u), B, ec);
            A.miss += sgn;  // the fast path counted the fp32 decision
            if (!kZero || d2 > 0.f) {
                const float w = w2.x * (float)sgn;
                A.s.x += w;
                if (KIND != K_DENSITY) {
                    A.x.x = fmaf(w, dx, A.x.x);
                    A.y.x = fmaf(w, dy, A.y.x);
                    A.z.x = fmaf(w, dz, A.z.x);
                }
            }
        }
    }
}

// One staged half: evaluate, re-decide the band if any lane saw a band pair.
template <int L, int KIND, bool kWlop, bool kZero>
__device__ __forceinline__ void eval_half(const float4* half, int nrec, int sub, const float4& q,
                                          const EvalConsts& ec, float band, double r2, Acc& A) {
    float bmin = INFINITY;
    eval_pairs<L, KIND, kWlop, kZero>(half, nrec, sub, ec, A, bmin);
    A.evald += 2 * nrec / L;  // nrec is a multiple of STEP = L * U: every lane the same
    if (__any_sync(0xffffffffu, bmin <= band))
        fix_band<L, KIND, kWlop, kZero>(half, nrec, sub, q, ec, band, r2, A);
}

template <int L>
__device__ __forceinline__ int group_isum(int v) {
#pragma unroll
    for (int o = 1; o < L; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Per-query totals over its L lanes; afterwards hneg = hits, rneg = in range.
template <int L>
__device__ __forceinline__ void group_reduce(Acc& A, bool with_nr) {
    A.s.x = group_sum<L>(A.s.x + A.s.y);
    A.x.x = group_sum<L>(A.x.x + A.x.y);
    A.y.x = group_sum<L>(A.y.x + A.y.y);
    A.z.x = group_sum<L>(A.z.x + A.z.y);
    (void)with_nr;
    const int ev = group_isum<L>(A.evald), miss = group_isum<L>(A.miss);
    A.rneg = ev + miss;                          // in range (d2 <= r2)
    A.hneg = A.rneg + group_isum<L>(A.zero);     // hits (and d > 0 when kZero)
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

// The next work unit for this warp: [r0, r1) positions in the query list.
// Units of `unit` queries up to tail_start, then units of tail_unit (one query
// group) so that the pass ends on short units (the tail of a persistent pass).
//
// With parts > 1 every tail unit is handed out `parts` times: part p takes the
// candidate rows p, p + parts, ... of the unit's groups (the attraction pass
// of a short query list ends on fractions of a group; the partial sums are
// combined in part order by the repulsion pass).
__device__ __forceinline__ bool next_unit(uint32_t* counter, uint32_t nq, uint32_t unit,
                                          uint32_t tail_start, uint32_t tail_unit, uint32_t parts,
                                          int lane, uint32_t& r0, uint32_t& r1, uint32_t& part) {
    uint32_t u = 0;
    if (lane == 0) u = atomicAdd(counter, 1u);
    u = __shfl_sync(0xffffffffu, u, 0);
    const uint32_t n1 = tail_start / unit;  // tail_start is a multiple of unit
    uint32_t len = unit;
    part = 0;
    if (u < n1) {
        r0 = u * unit;
    } else {
        const uint32_t t = u - n1;
        r0 = tail_start + (t / parts) * tail_unit;
        part = t % parts;
        len = tail_unit;
    }
    if (r0 >= nq) return false;
    r1 = min(r0 + len, nq);
    return true;
}

// Group starts inside a unit (bit i: a group must start at r0 + i): Morton
// block changes.
__device__ __forceinline__ unsigned group_breaks(const uint32_t* __restrict__ qcodes, int shift,
                                                 uint32_t r0, uint32_t r1, int lane) {
    const uint32_t pos = r0 + lane;
    const uint32_t code = pos < r1 ? (__ldg(&qcodes[pos]) >> shift) : 0xFFFFFFFFu;
    const uint32_t prev = __shfl_up_sync(0xffffffffu, code, 1);
    return __ballot_sync(0xffffffffu, lane == 0 || (pos < r1 && code != prev));
}

// End of the group starting at g0: the next break, at most Q queries.
__device__ __forceinline__ uint32_t group_end(unsigned brk, uint32_t r0, uint32_t r1, uint32_t g0,
                                              uint32_t Q) {
    const uint32_t rel = g0 - r0;
    const unsigned later = brk & ~((2u << rel) - 1u);
    const uint32_t e = later ? r0 + (uint32_t)(__ffs(later) - 1) : r1;
    return min(e, min(g0 + Q, r1));
}

// Groups of a unit by recursive bisection (FastArgs::bisect): the unit's (<= 32)
// queries, one per lane, are sorted along the longest axis of their box and
// halved, then each half along its own longest axis, down to groups of Q — a k-d
// split, so a group is compact in every direction (modelled on config 3:
// candidates per interaction -4% vs runs of Q consecutive curve positions).
// Returns, for slot `lane` of the sorted order, the query's position in the
// unit; positions >= n (padding) sort last.  Ties break on the position, so the
// grouping is deterministic.
template <int Q>
__device__ __forceinline__ uint32_t bisect_unit(const uint32_t* __restrict__ qlist,
                                                const float4* __restrict__ Xq, uint32_t r0,
                                                uint32_t n, int lane) {
    uint32_t idx = (uint32_t)lane;
    float4 p = make_float4(INFINITY, INFINITY, INFINITY, 0.f);
    if (idx < n) p = __ldg(&Xq[__ldg(&qlist[r0 + idx])]);
#pragma unroll
    for (int S = 32; S > Q; S >>= 1) {
        const bool valid = idx < n;
        float mnx = valid ? p.x : INFINITY, mny = valid ? p.y : INFINITY, mnz = valid ? p.z : INFINITY;
        float mxx = valid ? p.x : -INFINITY, mxy = valid ? p.y : -INFINITY, mxz = valid ? p.z : -INFINITY;
#pragma unroll
        for (int o = 1; o < S; o <<= 1) {
            mnx = fminf(mnx, __shfl_xor_sync(0xffffffffu, mnx, o));
            mny = fminf(mny, __shfl_xor_sync(0xffffffffu, mny, o));
            mnz = fminf(mnz, __shfl_xor_sync(0xffffffffu, mnz, o));
            mxx = fmaxf(mxx, __shfl_xor_sync(0xffffffffu, mxx, o));
            mxy = fmaxf(mxy, __shfl_xor_sync(0xffffffffu, mxy, o));
            mxz = fmaxf(mxz, __shfl_xor_sync(0xffffffffu, mxz, o));
        }
        const float ex = mxx - mnx, ey = mxy - mny, ez = mxz - mnz;
        const int axis = (ex >= ey && ex >= ez) ? 0 : (ey >= ez ? 1 : 2);
        float key = valid ? (axis == 0 ? p.x : (axis == 1 ? p.y : p.z)) : INFINITY;
        // bitonic sort of (key, idx) ascending inside aligned segments of S lanes
#pragma unroll
        for (int k = 2; k <= S; k <<= 1) {
#pragma unroll
            for (int j = k >> 1; j > 0; j >>= 1) {
                const float ok = __shfl_xor_sync(0xffffffffu, key, j);
                const uint32_t oi = __shfl_xor_sync(0xffffffffu, idx, j);
                float4 op;
                op.x = __shfl_xor_sync(0xffffffffu, p.x, j);
                op.y = __shfl_xor_sync(0xffffffffu, p.y, j);
                op.z = __shfl_xor_sync(0xffffffffu, p.z, j);
                op.w = 0.f;
                const bool up = k == S ? true : ((lane & k) == 0);
                const bool lower = (lane & j) == 0;
                const bool less = ok < key || (ok == key && oi < idx);  // other before mine
                if (lower ? (up ? less : !less) : (up ? !less : less)) {
                    key = ok;
                    idx = oi;
                    p = op;
                }
            }
        }
    }
    return idx;
}

// Phases of the per-point update.  PH_ALL: attraction, repulsion and the update
// in one pass.  PH_ATTR: attraction only; the per-query sums go to a.attr (the
// projected set's grid is rebuilt meanwhile on another stream).  PH_REP:
// repulsion, then the update from a.attr.  PH_ATTR and PH_REP form the same
// groups (same list, same cuts), so a.attr is indexed by list position.
enum : int { PH_ALL = 0, PH_ATTR = 1, PH_REP = 2 };

template <int L, bool kWlop, bool kCheckZero, int kRep, int PH>
__global__ void __launch_bounds__(FAST_THREADS, PCSB_FAST_MINB)
fast_kernel(const FastArgs a) {
    constexpr int Q = 32 / L;
    constexpr int KREP = kRep == 1 ? K_REP_INVCUBE : K_REP_NEGLIN;
    constexpr bool kAttr = PH != PH_REP;
    constexpr bool kRepul = kRep != 0 && PH != PH_ATTR;
    __shared__ __align__(128) float4 smem[FAST_WARPS * 4 * HR];
    __shared__ __align__(8) uint64_t bars[FAST_WARPS * 2];
    __shared__ float4 qsh[FAST_WARPS][Q];
    if (*a.done) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    Stage S = make_stage(smem + warp * 4 * HR, bars + 2 * warp, lane);
    const int qi = lane / L, sub = lane % L;
    uint32_t* counter = PH == PH_REP ? &a.slot->group_counter2 : &a.slot->group_counter;

    uint32_t r0, r1, part;
    const uint32_t tail_unit = max(a.tail_unit, (uint32_t)Q);
    // only the attraction pass splits its tail units by rows (FastArgs::tail_parts)
    const uint32_t parts = PH == PH_ATTR ? max(a.tail_parts, 1u) : 1u;
    while (next_unit(counter, a.nq, a.unit, a.tail_start, tail_unit, parts, lane, r0, r1, part)) {
        const int rfirst = (int)part, rstride = r0 >= a.tail_start ? (int)parts : 1;
        const bool bis = a.bisect != 0;
        const unsigned brk = bis ? 0u : group_breaks(a.qcodes, a.block_shift, r0, r1, lane);
        const uint32_t slotpos = bis ? bisect_unit<Q>(a.qlist, a.Xq, r0, r1 - r0, lane) : (uint32_t)lane;
        for (uint32_t g0 = r0, g1; g0 < r1; g0 = g1) {
            g1 = bis ? min(g0 + (uint32_t)Q, r1) : group_end(brk, r0, r1, g0, Q);
            const bool member = g0 + qi < g1;
            // the list position of this lane's query (slot -> position in the unit)
            const uint32_t pos = __shfl_sync(0xffffffffu, slotpos,
                                             (int)(member ? g0 - r0 + qi : g0 - r0));
            const uint32_t qpos = r0 + pos;
            const uint32_t qp = qpos;  // padding lanes duplicate the group's first query
            const uint32_t qint = __ldg(&a.qlist[qp]);  // internal index
            const float4 q = __ldg(&a.Xq[qint]);
            const EvalConsts ec = make_consts(q, a.kneg, a.K0, a.support);
            const Box box = member_box(q, member);
            if (member && sub == 0) qsh[warp][qi] = q;
            __syncwarp();
            const GroupQ G{qsh[warp], (int)(g1 - g0), a.scull2};
            uint32_t evals = 0;  // staged candidates evaluated (x Q queries)

            // ---------------- attraction: data candidates (lop.cpp:49-65) ----------------
            Acc at = acc_zero();
            if (kAttr) {
                gather_eval(a.Ppairs, a.Ppairs_cap, a.Pstart, a.gP, box, a.s_pad, G, S, lane,
                            rfirst, rstride, [&](const float4* half, int nrec) {
                                eval_half<L, K_ATTR, kWlop, kCheckZero>(half, nrec, sub, q, ec,
                                                                      a.band, a.r2, at);
                                evals += 2 * nrec;
                            });
                group_reduce<L>(at, kCheckZero);
            }
            if (PH == PH_ATTR) {
                if (member && sub == 0) {
                    // part p > 0 of a row-split tail unit: plane p - 1 of the extra sums
                    const size_t o = part == 0 ? (size_t)qpos
                                               : (size_t)(part - 1) * a.tail_cap + (qpos - a.tail_start);
                    (part == 0 ? a.attr : a.attr_x)[o] = make_float4(at.s.x, at.x.x, at.y.x, at.z.x);
                    (part == 0 ? a.attr_n : a.attr_nx)[o] =
                        make_int2(at.hneg, kCheckZero ? at.rneg - at.hneg : 0);
                }
                if (lane == 0) atomicAdd(&a.st->lane_candidates, (unsigned long long)evals * Q);
                continue;
            }
            if (PH == PH_REP && member && sub == 0) {
                float4 v = a.attr[qpos];
                int2 c = a.attr_n[qpos];
                if (a.tail_parts > 1 && qpos >= a.tail_start) {
                    // row-split tail units of the attraction pass: partial sums in part order
                    for (uint32_t p = 1; p < a.tail_parts; ++p) {
                        const size_t o = (size_t)(p - 1) * a.tail_cap + (qpos - a.tail_start);
                        const float4 w = a.attr_x[o];
                        const int2 d = a.attr_nx[o];
                        v.x += w.x;
                        v.y += w.y;
                        v.z += w.z;
                        v.w += w.w;
                        c.x += d.x;
                        c.y += d.y;
                    }
                }
                at.s.x = v.x;
                at.x.x = v.y;
                at.y.x = v.z;
                at.z.x = v.w;
                at.hneg = c.x;
                at.rneg = c.x + c.y;
            }

            // ---------------- repulsion: projected-set candidates (lop.cpp:79-97) ----------------
            Acc rp = acc_zero();
            if (kRepul) {
                gather_eval(a.Xpairs, a.Xpairs_cap, a.Xstart, a.gX, box, a.s_pad, G, S, lane, 0, 1,
                            [&](const float4* half, int nrec) {
                                eval_half<L, KREP, kWlop, true>(half, nrec, sub, q, ec, a.band,
                                                                a.r2, rp);
                                evals += 2 * nrec;
                            });
                group_reduce<L>(rp, true);
            }

            // ---------------- update (lane sub == 0 of each member query) ----------------
            float disp = 0.f;
            unsigned long long n_attr = 0, n_rep = 0;
            if (member && sub == 0) {
                const float sa = at.s.x;
                bool bad = !isfinite(sa) || !isfinite(at.x.x) || !isfinite(at.y.x) ||
                           !isfinite(at.z.x);
                const int zeros = kCheckZero ? (at.rneg - at.hneg) : 0;
                if (kCheckZero && zeros > 0) {
                    // an fp32 d2 of 0 could hide a distinct pair only for tiny coordinates
                    const float tiny = 0x1p-40f;
                    if (fabsf(q.x) < tiny || fabsf(q.y) < tiny || fabsf(q.z) < tiny) bad = true;
                }
                const bool attracted = sa > 0.f;
                if (kRep != 0 && attracted) {
                    // exactly one zero-distance candidate must remain: the query itself;
                    // any other is a coincident pair, counted by the exact path
                    const int z = rp.rneg - rp.hneg;
                    bad = bad || !isfinite(rp.s.x) || !isfinite(rp.x.x) || !isfinite(rp.y.x) ||
                          !isfinite(rp.z.x) || z != 1;
                }
                if (bad) {
#ifdef PCSB_CAREFUL_DIAG  // developer diagnostic (tools/build_variant.sh)
                    printf("careful q=%u (%.9g %.9g %.9g) w=%g sa=%g hits=%d zeros=%d rp.s=%g rz=%d\n",
                           qint, q.x, q.y, q.z, q.w, sa, at.hneg, zeros, rp.s.x,
                           rp.rneg - rp.hneg);
#endif
                    const uint32_t pos = atomicAdd(&a.slot->careful_count, 1u);
                    a.careful_list[pos] = qint;  // counts: written by the exact kernel
                } else {
                    float nx = q.x, ny = q.y, nz = q.z;
                    bool isolated = false;
                    if (!attracted) {
                        // zeros > 0: anchored at the coincident sample, which IS q
                        // (lop.cpp:67-69); otherwise isolated and held (lop.cpp:70-73)
                        isolated = !(kCheckZero && zeros > 0);
                    } else {
                        const float inv = 1.0f / sa;  // Weiszfeld quotient (lop.cpp:77)
                        nx = q.x + at.x.x * inv;
                        ny = q.y + at.y.x * inv;
                        nz = q.z + at.z.x * inv;
                        n_attr = (unsigned long long)at.hneg;
                        if (kRep != 0) {
                            n_rep = (unsigned long long)rp.hneg;
                            if (rp.s.x > 0.f) {  // lop.cpp:95-96, x - x' = -(c - q)
                                const float f = a.mu / rp.s.x;
                                nx = fmaf(-f, rp.x.x, nx);
                                ny = fmaf(-f, rp.y.x, ny);
                                nz = fmaf(-f, rp.z.x, nz);
                            }
                        }
                    }
                    a.Xnext[qint] = make_float4(nx, ny, nz, 0.f);
                    if (a.qcounts) {
                        const int fl = isolated ? QC_ISOLATED : (attracted ? 0 : QC_ANCHORED);
                        a.qcounts[qint] = make_int4((int)n_attr, (int)n_rep, 0, fl);
                        a.qever[qint] |= (uint8_t)fl;
                    }
                    const float ddx = nx - q.x, ddy = ny - q.y, ddz = nz - q.z;
                    disp = sqrtf(fmaf(ddz, ddz, fmaf(ddy, ddy, ddx * ddx)));
                    if (isolated) {
                        a.ever_isolated[qint] = 1;
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
#ifdef PCSB_COUNT_MEMBERS
                atomicAdd(&a.st->lane_candidates,
                          (unsigned long long)evals * (unsigned long long)(g1 - g0));
#else
                atomicAdd(&a.st->lane_candidates, (unsigned long long)evals * Q);
#endif
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Query groups, computed once per query-order rebuild (every few sweeps) rather
// than by the fused passes of every sweep: each 32-position unit of the curve-
// ordered list is cut where the curve jumps (farther than sqrt(jump2) between
// consecutive queries: the curve leaving a rank's slab or a cluster), and every
// piece is bisected recursively along its longest axis (bisect_unit).  The list
// is permuted into that order and the code of every position becomes the first
// position of its group, so the fused kernels' curve-run grouping
// (group_breaks / group_end with block_shift = 0) reproduces the bisected groups.
// ---------------------------------------------------------------------------
template <int Q>
__global__ void __launch_bounds__(128)
group_order_kernel(const uint32_t* __restrict__ qin, const float4* __restrict__ Xq, uint32_t nq,
                   float jump2, uint32_t* __restrict__ qout, uint32_t* __restrict__ codes,
                   const uint32_t* done) {
    if (done && *done) return;
    const int lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t u = warp; (uint64_t)u * 32 < nq; u += nw) {
        const uint32_t r0 = u * 32, r1 = min(nq, r0 + 32);
        for (uint32_t s0 = r0, s1; s0 < r1; s0 = s1) {
            const uint32_t pos = s0 + (uint32_t)lane;
            float4 p = make_float4(0.f, 0.f, 0.f, 0.f);
            if (pos < r1) p = __ldg(&Xq[__ldg(&qin[pos])]);
            const float px = __shfl_up_sync(0xffffffffu, p.x, 1);
            const float py = __shfl_up_sync(0xffffffffu, p.y, 1);
            const float pz = __shfl_up_sync(0xffffffffu, p.z, 1);
            const float dx = p.x - px, dy = p.y - py, dz = p.z - pz;
            const bool jump = lane > 0 && pos < r1 && fmaf(dz, dz, fmaf(dy, dy, dx * dx)) > jump2;
            const unsigned m = __ballot_sync(0xffffffffu, jump);
            s1 = m ? s0 + (uint32_t)(__ffs(m) - 1) : r1;
            const uint32_t n = s1 - s0;
            const uint32_t slot = bisect_unit<Q>(qin, Xq, s0, n, lane);
            if ((uint32_t)lane < n) {
                qout[s0 + lane] = __ldg(&qin[s0 + slot]);
                codes[s0 + lane] = s0 + ((uint32_t)lane / Q) * Q;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// WLOP density pass: dens_i = 1 + sum_{i' != i, d <= s} theta(d)  (fp32,
// exact neighbour set via the same fp64 re-decision of guard-band pairs).
// ---------------------------------------------------------------------------
constexpr int DL = 4;  // lanes per point

__global__ void __launch_bounds__(FAST_THREADS, PCSB_FAST_MINB)
density_kernel(const DensityArgs a) {
    constexpr int Q = 32 / DL;
    __shared__ __align__(128) float4 smem[FAST_WARPS * 4 * HR];
    __shared__ __align__(8) uint64_t bars[FAST_WARPS * 2];
    __shared__ float4 qsh[FAST_WARPS][Q];
    if (a.done && *a.done) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    Stage S = make_stage(smem + warp * 4 * HR, bars + 2 * warp, lane);
    const int qi = lane / DL, sub = lane % DL;
    uint32_t r0, r1;
    uint32_t part;
    while (next_unit(a.counter, a.nq, a.unit, a.nq / a.unit * a.unit, a.unit, 1u, lane, r0, r1, part)) {
        const unsigned brk = group_breaks(a.qcodes, a.block_shift, r0, r1, lane);
        for (uint32_t g0 = r0, g1; g0 < r1; g0 = g1) {
            g1 = group_end(brk, r0, r1, g0, Q);
            const uint32_t qpos = g0 + qi;
            const bool member = qpos < g1;
            const uint32_t qp = member ? qpos : g0;
            const uint32_t qslot = __ldg(&a.qlist[qp]);
            const float4 q = __ldg(&a.C[qslot]);
            const EvalConsts ec = make_consts(q, a.kneg, a.K0, 0.f);
            const Box box = member_box(q, member);
            if (member && sub == 0) qsh[warp][qi] = q;
            __syncwarp();
            const GroupQ G{qsh[warp], (int)(g1 - g0), a.scull2};
            Acc A = acc_zero();
            gather_eval(a.Cpairs, a.Cpairs_cap, a.Cstart, a.g, box, a.s_pad, G, S, lane, 0, 1,
                        [&](const float4* half, int nrec) {
                            eval_half<DL, K_DENSITY, false, true>(half, nrec, sub, q, ec, a.band,
                                                                 a.r2, A);
                        });
            group_reduce<DL>(A, true);
            unsigned long long pairs = 0;
            if (member && sub == 0) {
                // theta(0) = 1 for coincident duplicates; minus one for the point itself
                const float dens = 1.0f + A.s.x * a.inv_scale + (float)(A.rneg - A.hneg - 1);
                const float val = a.invert ? 1.0f / dens : dens;
                if (a.out_sorted) a.out_sorted[qslot].w = val;
                else a.out_internal[__ldg(&a.idx[qslot])].w = val;
                pairs = (unsigned long long)A.hneg;
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) pairs += __shfl_xor_sync(0xffffffffu, pairs, o);
            if (lane == 0 && pairs) atomicAdd(&a.st->density_pairs, pairs);
        }
    }
}

template <int L, bool W, bool Z, int R>
void launch_one(const FastArgs& a, int phase, int grid, cudaStream_t s) {
    if (phase == PH_ATTR) fast_kernel<L, W, Z, R, PH_ATTR><<<grid, FAST_THREADS, 0, s>>>(a);
    else if (phase == PH_REP) fast_kernel<L, W, Z, R, PH_REP><<<grid, FAST_THREADS, 0, s>>>(a);
    else fast_kernel<L, W, Z, R, PH_ALL><<<grid, FAST_THREADS, 0, s>>>(a);
}

template <int L>
void launch_l(const FastArgs& a, bool wlop, bool cz, int rep, int phase, int grid, cudaStream_t s) {
#define PCSB_DISPATCH(W, Z, R) \
    if (wlop == W && cz == Z && rep == R) return launch_one<L, W, Z, R>(a, phase, grid, s);
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
                 int phase, int grid_blocks, cudaStream_t s) {
    switch (lanes_per_point) {
        case 2: return launch_l<2>(a, wlop, check_zero, rep_mode, phase, grid_blocks, s);
        case 8: return launch_l<8>(a, wlop, check_zero, rep_mode, phase, grid_blocks, s);
        default: return launch_l<4>(a, wlop, check_zero, rep_mode, phase, grid_blocks, s);
    }
}

int fast_blocks_per_sm(int lanes_per_point, bool wlop, bool check_zero, int rep_mode) {
    (void)lanes_per_point;
    (void)check_zero;
    (void)wlop;
    (void)rep_mode;
    static int cached = 0;  // same for every variant (launch bounds + static smem)
    if (!cached) {
        int b = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fast_kernel<4, false, false, 2, PH_ALL>,
                                                      FAST_THREADS, 0);
        cached = b > 0 ? b : 1;
    }
    return cached;
}

uint32_t work_unit_queries(uint32_t nq, int total_warps) {
    // measured (config 3, tools/unit_probe.py, tools/scaling_probe.py): 16 beats 32
    // (shorter tail) and 8 (more fetches and partial groups), at 1/1, 1/4 and 1/8 of X
    (void)nq;
    (void)total_warps;
    static const uint32_t u = [] {
        const char* e = dev_knob("PCSB_UNIT");  // developer knob (1..32)
        const int v = e ? std::atoi(e) : 16;
        return (uint32_t)(v >= 1 && v <= 32 ? v : 16);
    }();
    return u;
}

void launch_group_order(const uint32_t* qin, const float4* Xq, uint32_t nq, float jump2,
                        uint32_t* qout, uint32_t* codes, const uint32_t* done, cudaStream_t s) {
    if (!nq) return;
    const uint32_t units = (nq + 31) / 32;
    const int blocks = (int)std::min<uint32_t>((units + 3) / 4, 148u * 16u);
    group_order_kernel<8><<<blocks, 128, 0, s>>>(qin, Xq, nq, jump2, qout, codes, done);
}

void launch_density(const DensityArgs& a, int grid_blocks, cudaStream_t s) {
    density_kernel<<<grid_blocks, FAST_THREADS, 0, s>>>(a);
}

}  // namespace pcsb
