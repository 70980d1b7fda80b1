// ptri.h — exact point-to-triangle distance shared by the host API
// (pcs::point_triangle_distance) and the device mesh-deviation kernel (nn.cu).
//
// Follows the reference's evaluation, proj/src/metrics.cpp:55-113: the Voronoi-
// region walk of Ericson's "Real-Time Collision Detection" (vertex regions a,
// b, c, edge regions ab, ac, bc, then the face), with the degenerate-triangle
// fallback to the three clamped segment distances.  Every fp64 operation is
// written out in the reference's association order and rounded individually
// (device: __d*_rn intrinsics; host: plain operators on x86-64, which has no
// fused multiply-add to contract into), so host and device agree bit for bit
// with the reference build.
#pragma once

#include <cmath>

#if defined(__CUDACC__)
#define PCSB_HD __host__ __device__ __forceinline__
#else
#define PCSB_HD inline
#endif

namespace pcsb {
namespace ptri {

PCSB_HD double mul(double a, double b) {
#if defined(__CUDA_ARCH__)
    return __dmul_rn(a, b);
#else
    return a * b;
#endif
}
PCSB_HD double add(double a, double b) {
#if defined(__CUDA_ARCH__)
    return __dadd_rn(a, b);
#else
    return a + b;
#endif
}
PCSB_HD double sub(double a, double b) {
#if defined(__CUDA_ARCH__)
    return __dsub_rn(a, b);
#else
    return a - b;
#endif
}
PCSB_HD double div(double a, double b) {
#if defined(__CUDA_ARCH__)
    return __ddiv_rn(a, b);
#else
    return a / b;
#endif
}
PCSB_HD double root(double a) {
#if defined(__CUDA_ARCH__)
    return __dsqrt_rn(a);
#else
    return std::sqrt(a);
#endif
}

struct V3 {
    double x, y, z;
};

PCSB_HD V3 vsub(V3 a, V3 b) { return {sub(a.x, b.x), sub(a.y, b.y), sub(a.z, b.z)}; }
PCSB_HD V3 vadd(V3 a, V3 b) { return {add(a.x, b.x), add(a.y, b.y), add(a.z, b.z)}; }
PCSB_HD V3 vscale(double s, V3 a) { return {mul(s, a.x), mul(s, a.y), mul(s, a.z)}; }
// a.x*b.x + a.y*b.y + a.z*b.z, left to right (core.hpp dot)
PCSB_HD double vdot(V3 a, V3 b) { return add(add(mul(a.x, b.x), mul(a.y, b.y)), mul(a.z, b.z)); }
PCSB_HD double vnorm(V3 a) { return root(vdot(a, a)); }

// distance from p to the segment [s0, s1], the parameter clamped to [0, 1]
PCSB_HD double segment(V3 p, V3 s0, V3 s1) {
    const V3 d = vsub(s1, s0);
    const double len2 = vdot(d, d);
    if (len2 == 0.0) return vnorm(vsub(p, s0));
    double t = div(vdot(vsub(p, s0), d), len2);
    t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
    return vnorm(vsub(p, vadd(s0, vscale(t, d))));
}

PCSB_HD double distance(V3 p, V3 a, V3 b, V3 c) {
    const V3 ab = vsub(b, a), ac = vsub(c, a);
    const V3 ap = vsub(p, a);
    const double d1 = vdot(ab, ap), d2 = vdot(ac, ap);
    if (d1 <= 0.0 && d2 <= 0.0) return vnorm(vsub(p, a));  // vertex a
    const V3 bp = vsub(p, b);
    const double d3 = vdot(ab, bp), d4 = vdot(ac, bp);
    if (d3 >= 0.0 && d4 <= d3) return vnorm(vsub(p, b));  // vertex b
    const double vc = sub(mul(d1, d4), mul(d3, d2));
    if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) {  // edge ab
        const double v = div(d1, sub(d1, d3));
        return vnorm(vsub(p, vadd(a, vscale(v, ab))));
    }
    const V3 cp = vsub(p, c);
    const double d5 = vdot(ab, cp), d6 = vdot(ac, cp);
    if (d6 >= 0.0 && d5 <= d6) return vnorm(vsub(p, c));  // vertex c
    const double vb = sub(mul(d5, d2), mul(d1, d6));
    if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {  // edge ac
        const double w = div(d2, sub(d2, d6));
        return vnorm(vsub(p, vadd(a, vscale(w, ac))));
    }
    const double va = sub(mul(d3, d6), mul(d5, d4));
    const double e43 = sub(d4, d3), e56 = sub(d5, d6);
    if (va <= 0.0 && e43 >= 0.0 && e56 >= 0.0) {  // edge bc
        const double w = div(e43, add(e43, e56));
        return vnorm(vsub(p, vadd(b, vscale(w, vsub(c, b)))));
    }
    const double sum = add(add(va, vb), vc);
    if (!(sum > 0.0)) {  // zero-area triangle: the nearest point is on an edge
        const double s_ab = segment(p, a, b), s_bc = segment(p, b, c), s_ac = segment(p, a, c);
        double best = s_ab;
        if (s_bc < best) best = s_bc;
        if (s_ac < best) best = s_ac;
        return best;
    }
    const double denom = div(1.0, sum);
    const double v = mul(vb, denom), w = mul(vc, denom);
    return vnorm(vsub(p, vadd(vadd(a, vscale(v, ab)), vscale(w, ac))));
}

}  // namespace ptri
}  // namespace pcsb
