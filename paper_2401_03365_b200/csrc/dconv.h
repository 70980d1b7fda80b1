// dconv.h — double <-> decimal text conversions for the cloud IO kernels
// (io.cu), byte-compatible with the reference's writer and reader
// (proj/src/io.cpp:36-48 parse_double = std::from_chars, :240-245 format_double =
// std::to_chars shortest round-trip).  __host__ __device__: the same code runs in
// the GPU kernels and in the host-side tests against libstdc++.
//
// * format: shortest round-trip digits by the Ryu algorithm (U. Adams, "Ryū: fast
//   float-to-string conversion", PLDI 2018) over exact 125-bit power-of-five
//   tables (dconv_tables.h, generated with big integers by
//   tools/gen_dconv_tables.py), laid out as libstdc++'s std::to_chars(double)
//   does: fixed or scientific, whichever is shorter (fixed on a tie), the
//   exponent with at least two digits, and a fixed-notation integer printed
//   with the double's exact integer digits.
// * parse: the from_chars grammar ([-]digits[.digits][(e|E)[+|-]digits]);
//   decimal significands of up to 19 digits with |decimal exponent| <= 27 are
//   rounded to nearest-even by exact 128-bit integer arithmetic (the product
//   w*5^q, or the quotient of w*2^s by 5^-q with its remainder).  Anything else
//   reports "not handled" and the caller parses that token with std::from_chars
//   on the host.
#pragma once

#include <cstdint>

#include "dconv_tables.h"

#if defined(__CUDACC__)
#define DCONV_HD __host__ __device__ __forceinline__
#else
#define DCONV_HD inline
#endif

namespace pcsb {
namespace dconv {

// ---- 64/128-bit helpers --------------------------------------------------------
struct U128 {
    uint64_t lo, hi;
};

DCONV_HD U128 mul64(uint64_t a, uint64_t b) {
#if defined(__CUDA_ARCH__)
    return {a * b, __umul64hi(a, b)};
#else
    const unsigned __int128 p = (unsigned __int128)a * b;
    return {(uint64_t)p, (uint64_t)(p >> 64)};
#endif
}

DCONV_HD int clz64(uint64_t x) {
#if defined(__CUDA_ARCH__)
    return __clzll((long long)x);
#else
    return x ? __builtin_clzll(x) : 64;
#endif
}

DCONV_HD const uint64_t* pow5inv(int i) {
#if defined(__CUDA_ARCH__)
    return kPow5InvDev[i];
#else
    return kPow5InvHost[i];
#endif
}
DCONV_HD const uint64_t* pow5(int i) {
#if defined(__CUDA_ARCH__)
    return kPow5Dev[i];
#else
    return kPow5Host[i];
#endif
}

// ---- Ryu: shortest decimal digits of a finite, non-zero double ------------------
DCONV_HD int pow5bits(int e) { return (int)(((uint32_t)e * 1217359u) >> 19) + 1; }
DCONV_HD uint32_t log10pow2(int e) { return ((uint32_t)e * 78913u) >> 18; }
DCONV_HD uint32_t log10pow5(int e) { return ((uint32_t)e * 732923u) >> 20; }

DCONV_HD uint32_t pow5factor(uint64_t v) {
    uint32_t c = 0;
    while (v % 5 == 0) {
        v /= 5;
        ++c;
    }
    return c;
}
DCONV_HD bool multiple_of_pow5(uint64_t v, uint32_t p) { return pow5factor(v) >= p; }
DCONV_HD bool multiple_of_pow2(uint64_t v, uint32_t p) { return (v & ((1ull << p) - 1)) == 0; }

// (m * mul) >> j for a 128-bit multiplier, j >= 64
DCONV_HD uint64_t mul_shift(uint64_t m, const uint64_t* mul, int j) {
    const U128 b0 = mul64(m, mul[0]);
    const U128 b2 = mul64(m, mul[1]);
    // (b0 >> 64) + b2, then >> (j - 64)
    uint64_t lo = b2.lo + b0.hi;
    uint64_t hi = b2.hi + (lo < b0.hi ? 1u : 0u);
    const int s = j - 64;
    if (s == 0) return lo;
    if (s >= 64) return hi >> (s - 64);
    return (lo >> s) | (hi << (64 - s));
}

struct Decimal {
    uint64_t digits;  // shortest significand
    int32_t exp10;    // value = digits * 10^exp10
};

DCONV_HD Decimal shortest(uint64_t ieee_mant, uint32_t ieee_exp) {
    int32_t e2;
    uint64_t m2;
    if (ieee_exp == 0) {
        e2 = 1 - 1023 - 52 - 2;
        m2 = ieee_mant;
    } else {
        e2 = (int32_t)ieee_exp - 1023 - 52 - 2;
        m2 = (1ull << 52) | ieee_mant;
    }
    const bool even = (m2 & 1) == 0;
    const bool accept = even;
    const uint64_t mv = 4 * m2;
    const uint32_t mm_shift = (ieee_mant != 0 || ieee_exp <= 1) ? 1u : 0u;

    uint64_t vr, vp, vm;
    int32_t e10;
    bool vm_tz = false, vr_tz = false;
    if (e2 >= 0) {
        const uint32_t q = log10pow2(e2) - (e2 > 3 ? 1u : 0u);
        e10 = (int32_t)q;
        const int k = kPow5InvBits + pow5bits((int)q) - 1;
        const int i = -e2 + (int)q + k;
        const uint64_t* mul = pow5inv((int)q);
        vr = mul_shift(4 * m2, mul, i);
        vp = mul_shift(4 * m2 + 2, mul, i);
        vm = mul_shift(4 * m2 - 1 - mm_shift, mul, i);
        if (q <= 21) {
            const uint32_t mv_mod5 = (uint32_t)(mv % 5);
            if (mv_mod5 == 0) {
                vr_tz = multiple_of_pow5(mv, q);
            } else if (accept) {
                vm_tz = multiple_of_pow5(mv - 1 - mm_shift, q);
            } else {
                vp -= multiple_of_pow5(mv + 2, q) ? 1u : 0u;
            }
        }
    } else {
        const uint32_t q = log10pow5(-e2) - (-e2 > 1 ? 1u : 0u);
        e10 = (int32_t)q + e2;
        const int i = -e2 - (int)q;
        const int k = pow5bits(i) - kPow5Bits;
        const int j = (int)q - k;
        const uint64_t* mul = pow5(i);
        vr = mul_shift(4 * m2, mul, j);
        vp = mul_shift(4 * m2 + 2, mul, j);
        vm = mul_shift(4 * m2 - 1 - mm_shift, mul, j);
        if (q <= 1) {
            vr_tz = true;
            if (accept) vm_tz = mm_shift == 1;
            else --vp;
        } else if (q < 63) {
            vr_tz = multiple_of_pow2(mv, q);
        }
    }

    int32_t removed = 0;
    uint8_t last = 0;
    uint64_t out;
    if (vm_tz || vr_tz) {
        while (vp / 10 > vm / 10) {
            vm_tz &= vm % 10 == 0;
            vr_tz &= last == 0;
            last = (uint8_t)(vr % 10);
            vr /= 10;
            vp /= 10;
            vm /= 10;
            ++removed;
        }
        if (vm_tz) {
            while (vm % 10 == 0) {
                vr_tz &= last == 0;
                last = (uint8_t)(vr % 10);
                vr /= 10;
                vp /= 10;
                vm /= 10;
                ++removed;
            }
        }
        if (vr_tz && last == 5 && vr % 2 == 0) last = 4;  // exact half: round to even
        out = vr + (((vr == vm && (!accept || !vm_tz)) || last >= 5) ? 1u : 0u);
    } else {
        bool round_up = false;
        while (vp / 10 > vm / 10) {
            round_up = vr % 10 >= 5;
            vr /= 10;
            vp /= 10;
            vm /= 10;
            ++removed;
        }
        out = vr + ((vr == vm || round_up) ? 1u : 0u);
    }
    return {out, e10 + removed};
}

DCONV_HD int ndigits(uint64_t v) {
    int n = 1;
    while (v >= 10) {
        v /= 10;
        ++n;
    }
    return n;
}

// Writes v with std::to_chars(double) layout into out (>= 32 bytes); returns
// the character count.
DCONV_HD int format(double v, char* out) {
    uint64_t bits;
#if defined(__CUDA_ARCH__)
    bits = (uint64_t)__double_as_longlong(v);
#else
    __builtin_memcpy(&bits, &v, 8);
#endif
    const bool neg = (bits >> 63) != 0;
    const uint64_t mant = bits & ((1ull << 52) - 1);
    const uint32_t ex = (uint32_t)((bits >> 52) & 0x7FF);
    int n = 0;
    if (ex == 0x7FF) {
        if (neg) out[n++] = '-';
        if (mant) {
            out[n++] = 'n', out[n++] = 'a', out[n++] = 'n';
        } else {
            out[n++] = 'i', out[n++] = 'n', out[n++] = 'f';
        }
        return n;
    }
    if (neg) out[n++] = '-';
    if (ex == 0 && mant == 0) {
        out[n++] = '0';
        return n;
    }
    const Decimal d = shortest(mant, ex);
    char dig[20];
    const int nd = ndigits(d.digits);
    {
        uint64_t t = d.digits;
        for (int k = nd - 1; k >= 0; --k) {
            dig[k] = (char)('0' + t % 10);
            t /= 10;
        }
    }
    const int sexp = d.exp10 + nd - 1;  // scientific exponent
    const int aexp = sexp < 0 ? -sexp : sexp;
    const int sci_len = nd + (nd > 1 ? 1 : 0) + 2 + (aexp >= 100 ? 3 : 2);
    int fix_len;
    if (sexp < 0) fix_len = nd + 1 - sexp;
    else if (sexp < nd - 1) fix_len = nd + 1;
    else fix_len = sexp + 1;
    if (sci_len < fix_len) {
        out[n++] = dig[0];
        if (nd > 1) {
            out[n++] = '.';
            for (int k = 1; k < nd; ++k) out[n++] = dig[k];
        }
        out[n++] = 'e';
        out[n++] = sexp < 0 ? '-' : '+';
        if (aexp >= 100) out[n++] = (char)('0' + aexp / 100);
        out[n++] = (char)('0' + (aexp / 10) % 10);
        out[n++] = (char)('0' + aexp % 10);
        return n;
    }
    if (sexp < 0) {
        out[n++] = '0';
        out[n++] = '.';
        for (int k = 0; k < -sexp - 1; ++k) out[n++] = '0';
        for (int k = 0; k < nd; ++k) out[n++] = dig[k];
        return n;
    }
    if (sexp < nd - 1) {
        for (int k = 0; k <= sexp; ++k) out[n++] = dig[k];
        out[n++] = '.';
        for (int k = sexp + 1; k < nd; ++k) out[n++] = dig[k];
        return n;
    }
    // an integer: the double's exact integer digits (it is m * 2^e2 with e2 >= 0
    // here, below 2^128 because fixed only wins up to ~24 digits)
    {
        const uint64_t m2 = ex == 0 ? mant : ((1ull << 52) | mant);
        const int e2 = (ex == 0 ? 1 : (int)ex) - 1023 - 52;
        if (e2 <= 0) {  // < 2^53: the shortest digits are exact
            for (int k = 0; k < nd; ++k) out[n++] = dig[k];
            for (int k = nd; k <= sexp; ++k) out[n++] = '0';
            return n;
        }
        uint64_t hi = e2 >= 64 ? (m2 << (e2 - 64)) : (e2 ? (m2 >> (64 - e2)) : 0);
        uint64_t lo = e2 >= 64 ? 0 : (m2 << e2);
        char tmp[48];
        int t = 0;
        while (hi || lo) {  // 128-bit division by 10, 32 bits at a time
            uint64_t r = 0;
            uint32_t part[4] = {(uint32_t)(hi >> 32), (uint32_t)hi, (uint32_t)(lo >> 32), (uint32_t)lo};
            for (int k = 0; k < 4; ++k) {
                const uint64_t cur = (r << 32) | part[k];
                part[k] = (uint32_t)(cur / 10);
                r = cur % 10;
            }
            hi = ((uint64_t)part[0] << 32) | part[1];
            lo = ((uint64_t)part[2] << 32) | part[3];
            tmp[t++] = (char)('0' + r);
        }
        while (t) out[n++] = tmp[--t];
        return n;
    }
}

// ---- parsing --------------------------------------------------------------------
DCONV_HD double make_double(bool neg, uint64_t mant53, int exp2) {
    // mant53 in [2^52, 2^53): value = mant53 * 2^exp2, a normal double
    const uint64_t be = (uint64_t)(exp2 + 52 + 1023);
    const uint64_t bits = ((uint64_t)neg << 63) | (be << 52) | (mant53 & ((1ull << 52) - 1));
#if defined(__CUDA_ARCH__)
    return __longlong_as_double((long long)bits);
#else
    double d;
    __builtin_memcpy(&d, &bits, 8);
    return d;
#endif
}

// Round the 128-bit integer (hi, lo) * 2^exp2 (plus a sticky bit) to a double.
DCONV_HD bool round128(bool neg, uint64_t hi, uint64_t lo, int exp2, bool sticky, double* out) {
    const int lz = hi ? clz64(hi) : 64 + clz64(lo);
    const int bl = 128 - lz;  // bit length >= 1
    int shift = bl - 53;      // bits below the 53-bit mantissa
    uint64_t mant;
    bool half = false, below = sticky;
    if (shift <= 0) {
        mant = lo << (-shift);  // bl <= 53: exact, fits in lo
    } else {
        // mant = (hi:lo) >> shift, rest bits decide the rounding
        if (shift >= 64) {
            mant = hi >> (shift - 64);
            const uint64_t rhi = shift == 64 ? 0 : (hi & ((1ull << (shift - 64)) - 1));
            const int hb = shift - 1;  // half bit index
            if (hb >= 64) {
                half = (hi >> (hb - 64)) & 1;
                below = below || lo != 0 || (rhi & ((1ull << (hb - 64)) - 1)) != 0;
            } else {
                half = (lo >> hb) & 1;
                below = below || (lo & ((1ull << hb) - 1)) != 0;
            }
        } else {
            mant = (lo >> shift) | (hi << (64 - shift));
            const int hb = shift - 1;
            half = (lo >> hb) & 1;
            below = below || (hb > 0 && (lo & ((1ull << hb) - 1)) != 0);
        }
        if (half && (below || (mant & 1))) ++mant;
        if (mant == (1ull << 53)) {
            mant >>= 1;
            ++shift;
        }
    }
    const int e = exp2 + shift;
    const int eb = e + 52 + 1023;
    if (eb <= 0 || eb >= 0x7FF) return false;  // subnormal or overflow: not handled here
    *out = make_double(neg, mant, e);
    return true;
}

DCONV_HD bool is_digit(char c) { return c >= '0' && c <= '9'; }

// 10^k, k <= 19
DCONV_HD uint64_t pow10u(int k) {
    uint64_t p = 1;
    for (int i = 0; i < k; ++i) p *= 10;
    return p;
}

// (hi:lo) / d for d < 2^64 with hi < d: quotient and remainder, long division
// in 32-bit digits.
DCONV_HD uint64_t div128(uint64_t hi, uint64_t lo, uint64_t d, uint64_t* rem) {
    // normalise
    const int s = clz64(d);
    d <<= s;
    if (s) {
        hi = (hi << s) | (lo >> (64 - s));
        lo <<= s;
    }
    const uint64_t dh = d >> 32, dl = d & 0xFFFFFFFFull;
    uint64_t q[2];
    uint64_t r = hi;
    for (int k = 0; k < 2; ++k) {
        const uint64_t nxt = (lo >> (32 * (1 - k))) & 0xFFFFFFFFull;
        // divide (r:nxt) (96 bits, r < d) by d -> 32-bit quotient digit
        uint64_t qh = r / dh;
        uint64_t rh = r - qh * dh;
        while (qh >> 32 || qh * dl > ((rh << 32) | nxt)) {
            --qh;
            rh += dh;
            if (rh >> 32) break;
        }
        r = ((r << 32) | nxt) - qh * d;
        q[k] = qh;
    }
    *rem = r >> s;
    return (q[0] << 32) | q[1];
}

// Parses [p, e) entirely as a from_chars double; false = not handled (the caller
// re-parses on the host: syntax errors, > 19 significant digits, |exp| > 27,
// subnormal/overflowing results, "inf"/"nan").
DCONV_HD bool parse(const char* p, const char* e, double* out) {
    bool neg = false;
    if (p < e && *p == '-') {
        neg = true;
        ++p;
    }
    uint64_t w = 0;
    int nd = 0, dexp = 0;
    bool any = false;
    while (p < e && is_digit(*p)) {
        any = true;
        if (w == 0 && *p == '0') {  // leading zeros
            ++p;
            continue;
        }
        if (nd >= 19) return false;
        w = w * 10 + (uint64_t)(*p - '0');
        ++nd;
        ++p;
    }
    if (p < e && *p == '.') {
        ++p;
        while (p < e && is_digit(*p)) {
            any = true;
            if (w == 0 && *p == '0') {
                --dexp;
                ++p;
                continue;
            }
            if (nd >= 19) return false;
            w = w * 10 + (uint64_t)(*p - '0');
            ++nd;
            --dexp;
            ++p;
        }
    }
    if (!any) return false;
    if (p < e && (*p == 'e' || *p == 'E')) {
        ++p;
        bool eneg = false;
        if (p < e && (*p == '+' || *p == '-')) {
            eneg = *p == '-';
            ++p;
        }
        if (p >= e || !is_digit(*p)) return false;
        int x = 0;
        while (p < e && is_digit(*p)) {
            if (x > 100000) return false;
            x = x * 10 + (*p - '0');
            ++p;
        }
        dexp += eneg ? -x : x;
    }
    if (p != e) return false;
    if (w == 0) {
        *out = neg ? -0.0 : 0.0;
        return true;
    }
    if (dexp > 27 || dexp < -27) return false;
    if (dexp >= 0) {
        // w * 5^q * 2^q, exact
        const U128 a = mul64(w, pow10u(dexp > 19 ? 19 : dexp) / (1ull << (dexp > 19 ? 19 : dexp)));
        // 5^q for q <= 27 exceeds 64 bits past q = 27: split 5^q = 5^a * 5^b
        uint64_t hi = a.hi, lo = a.lo;
        if (dexp > 19) {
            const uint64_t f = pow10u(dexp - 19) >> (dexp - 19);  // 5^(q-19)
            const U128 l2 = mul64(lo, f), h2 = mul64(hi, f);
            if (h2.hi) return false;
            lo = l2.lo;
            hi = l2.hi + h2.lo;
            if (hi < h2.lo) return false;
        }
        return round128(neg, hi, lo, dexp, false, out);
    }
    // w / (5^q * 2^q), q = -dexp <= 27: quotient of (w << s) by 5^q with >= 64
    // significant bits, the remainder as a sticky bit
    const int q = -dexp;
    const uint64_t d = pow10u(q > 19 ? 19 : q) >> (q > 19 ? 19 : q);  // 5^min(q,19)
    uint64_t dd = d;
    if (q > 19) {
        const uint64_t f = pow10u(q - 19) >> (q - 19);
        const U128 t = mul64(dd, f);
        if (t.hi) return false;  // 5^q >= 2^64 (q >= 28)
        dd = t.lo;
    }
    // Q = floor(w * 2^t / 5^q) with 62..64 significant bits: t = 63 - len(w) + len(5^q)
    // keeps the 128-bit numerator's high word below the divisor
    const int t = 63 - (64 - clz64(w)) + (64 - clz64(dd));
    uint64_t nh, nl;
    if (t >= 64) {
        nh = w << (t - 64);
        nl = 0;
    } else {
        nh = t ? (w >> (64 - t)) : 0;
        nl = w << t;
    }
    uint64_t rem;
    const uint64_t quo = div128(nh, nl, dd, &rem);
    // w / 10^q = (w * 2^t / 5^q) * 2^(-t - q)
    return round128(neg, 0, quo, -t - q, rem != 0, out);
}

}  // namespace dconv
}  // namespace pcsb
