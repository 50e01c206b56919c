// girg_device.cuh -- device primitives of the B200 GIRG generator (sm_100a).
//
// Philox4x32-10 counter-based randomness, 53-bit uniforms, Morton interleave and the canonical
// double-precision model arithmetic (no FMA contraction: the library is compiled with
// -fmad=false so every product and sum rounds separately, as in DESIGN.md "Canonical
// arithmetic").  Citations "P:NNN" refer to lines of PAPER.md (arXiv:1905.06706).
#pragma once
#include <math_constants.h>
#include <cstdint>
#include <cuda_runtime.h>

namespace girg {

// ---------------------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al., SC'11).  Key = (lo32(seed), hi32(seed)).  Each round is two
// 32x32->64 multiplies (IMAD.WIDE / IMAD.HI) and two 3-input XORs (LOP3).
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1)
{
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
        c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    }
    return c;
}

// uniform on the 2^-53 grid in [0,1) from words (hi, lo): exact conversion
__device__ __forceinline__ double u53(uint32_t hi, uint32_t lo)
{
    const unsigned long long b = ((((unsigned long long)hi) << 32) | lo) >> 11;
    return __dmul_rn(__ull2double_rn(b), 0x1p-53);
}

// ---------------------------------------------------------------------------------------
// Morton code: bit interleave, coordinate 0 most significant in each
// d-bit group.  `lvl` bits per coordinate, d*lvl <= 31.
// ---------------------------------------------------------------------------------------
template <int D>
__device__ __forceinline__ uint32_t spread_bits(uint32_t c)
{
    if constexpr (D == 1) {
        return c;
    } else if constexpr (D == 2) {
        c &= 0x0000ffffu;
        c = (c | (c << 8)) & 0x00ff00ffu;
        c = (c | (c << 4)) & 0x0f0f0f0fu;
        c = (c | (c << 2)) & 0x33333333u;
        c = (c | (c << 1)) & 0x55555555u;
        return c;
    } else if constexpr (D == 3) {
        c &= 0x000003ffu;
        c = (c | (c << 16)) & 0x030000ffu;
        c = (c | (c << 8)) & 0x0300f00fu;
        c = (c | (c << 4)) & 0x030c30c3u;
        c = (c | (c << 2)) & 0x09249249u;
        return c;
    } else {
        uint32_t r = 0;
#pragma unroll
        for (int b = 0; b < 32 / D; ++b) r |= ((c >> b) & 1u) << (b * D);
        return r;
    }
}

template <int D>
__device__ __forceinline__ uint32_t gather_bits(uint32_t m)
{
    if constexpr (D == 1) {
        return m;
    } else if constexpr (D == 2) {
        m &= 0x55555555u;
        m = (m | (m >> 1)) & 0x33333333u;
        m = (m | (m >> 2)) & 0x0f0f0f0fu;
        m = (m | (m >> 4)) & 0x00ff00ffu;
        m = (m | (m >> 8)) & 0x0000ffffu;
        return m;
    } else if constexpr (D == 3) {
        m &= 0x09249249u;
        m = (m | (m >> 2)) & 0x030c30c3u;
        m = (m | (m >> 4)) & 0x0300f00fu;
        m = (m | (m >> 8)) & 0x030000ffu;
        m = (m | (m >> 16)) & 0x000003ffu;
        return m;
    } else {
        uint32_t r = 0;
#pragma unroll
        for (int b = 0; b < 32 / D; ++b) r |= ((m >> (b * D)) & 1u) << b;
        return r;
    }
}

template <int D>
__device__ __forceinline__ uint32_t morton_encode(const uint32_t (&c)[D])
{
    uint32_t code = 0;
#pragma unroll
    for (int k = 0; k < D; ++k) code |= spread_bits<D>(c[k]) << (D - 1 - k);
    return code;
}

template <int D>
__device__ __forceinline__ void morton_decode(uint32_t code, uint32_t (&c)[D])
{
#pragma unroll
    for (int k = 0; k < D; ++k) c[k] = gather_bits<D>(code >> (D - 1 - k));
}

// ---------------------------------------------------------------------------------------
// Canonical model arithmetic: torus L-inf distance, D = dist^d left
// to right, q = (w_u*w_v)*s, p = min(1, (q/D)^(1/T)) (Eq. 1 P:277 in kappa form), threshold
// D <= q.
// ---------------------------------------------------------------------------------------
// ---------------------------------------------------------------------------------------
// R26: the log / exp / pow of the edge decisions, written with + - * / and bit
// operations only (no libdevice), the formulas the oracle states: both sides compute identical
// bits, so a T > 0 decision cannot differ by a library ulp.  (-fmad=false: no contraction.)
//   log: x = m 2^k, m in [sqrt(1/2), sqrt(2)), s = (m-1)/(m+1),
//        log m = 2s (1 + s^2/3 + ... + s^22/23), log x = k ln2_hi + (k ln2_lo + log m)
//   exp: k = rint(t / ln2), r = (t - k ln2_hi) - k ln2_lo, sum_{i<=13} r^i/i!, times 2^k
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ double pow2i(int k)  // 2^k, -1022 <= k <= 1023
{
    return __longlong_as_double((long long)((unsigned long long)(k + 1023) << 52));
}

__device__ __forceinline__ double det_log(double x)
{
    if (!(x > 0.0)) return x == 0.0 ? -CUDART_INF : CUDART_NAN;
    if (isinf(x)) return x;
    int k = 0;
    unsigned long long b = (unsigned long long)__double_as_longlong(x);
    if (((b >> 52) & 0x7ff) == 0) {
        x = x * 0x1p54;
        k = -54;
        b = (unsigned long long)__double_as_longlong(x);
    }
    k += (int)((b >> 52) & 0x7ff) - 1023;
    double m = __longlong_as_double((long long)((b & 0x000fffffffffffffull) | 0x3ff0000000000000ull));
    if (m > 0x1.6a09e667f3bcdp+0) {
        m = m * 0.5;
        k += 1;
    }
    const double f = m - 1.0;
    const double sv = f / (m + 1.0);
    const double z = sv * sv;
    double p = 0x1.642c8590b2164p-5;
    p = p * z + 0x1.8618618618618p-5;
    p = p * z + 0x1.af286bca1af28p-5;
    p = p * z + 0x1.e1e1e1e1e1e1ep-5;
    p = p * z + 0x1.1111111111111p-4;
    p = p * z + 0x1.3b13b13b13b14p-4;
    p = p * z + 0x1.745d1745d1746p-4;
    p = p * z + 0x1.c71c71c71c71cp-4;
    p = p * z + 0x1.2492492492492p-3;
    p = p * z + 0x1.999999999999ap-3;
    p = p * z + 0x1.5555555555555p-2;
    const double logm = (2.0 * sv) + (2.0 * sv) * (z * p);
    const double kd = (double)k;
    return kd * 0x1.62e42fee00000p-1 + (kd * 0x1.a39ef35793c76p-33 + logm);
}

__device__ __forceinline__ double det_exp(double t)
{
    if (isnan(t)) return t;
    if (t > 709.78) return CUDART_INF;
    if (t < -745.2) return 0.0;
    const double kd = rint(t * 0x1.71547652b82fep+0);
    const int k = (int)kd;
    const double r = (t - kd * 0x1.62e42fee00000p-1) - kd * 0x1.a39ef35793c76p-33;
    double p = 0x1.6124613a86d09p-33;
    p = p * r + 0x1.1eed8eff8d898p-29;
    p = p * r + 0x1.ae64567f544e4p-26;
    p = p * r + 0x1.27e4fb7789f5cp-22;
    p = p * r + 0x1.71de3a556c734p-19;
    p = p * r + 0x1.a01a01a01a01ap-16;
    p = p * r + 0x1.a01a01a01a01ap-13;
    p = p * r + 0x1.6c16c16c16c17p-10;
    p = p * r + 0x1.1111111111111p-7;
    p = p * r + 0x1.5555555555555p-5;
    p = p * r + 0x1.5555555555555p-3;
    p = p * r + 0.5;
    p = p * r + 1.0;
    p = p * r + 1.0;
    if (k >= -1022 && k <= 1023) return p * pow2i(k);
    if (k > 1023) return (p * pow2i(1023)) * pow2i(k - 1023);
    return (p * pow2i(k + 200)) * pow2i(-200);
}

__device__ __forceinline__ double det_pow(double x, double y) { return det_exp(y * det_log(x)); }

template <int D>
__device__ __forceinline__ double dist_pow(const double (&xu)[D], const double (&xv)[D])
{
    double dist = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) {
        const double a = fabs(__dsub_rn(xu[k], xv[k]));
        const double t = fmin(a, __dsub_rn(1.0, a));
        dist = fmax(dist, t);
    }
    double P = dist;
#pragma unroll
    for (int k = 1; k < D; ++k) P = __dmul_rn(P, dist);
    return P;
}

__device__ __forceinline__ double prob_uv(double wu, double wv, double s, double Dp, double invT)
{
    const double q = __dmul_rn(__dmul_rn(wu, wv), s);
    const double ratio = __ddiv_rn(q, Dp);
    if (ratio >= 1.0) return 1.0;
    return det_pow(ratio, invT);  // R26
}

// ---------------------------------------------------------------------------------------
// Fast decisions.  Each returns a decision only when it provably
// equals the one of the canonical double-precision arithmetic above; otherwise it reports
// "undecided" and the caller evaluates the canonical expression.  log2 of a double is taken as
// exponent (exact) + MUFU lg2 of the top 23 mantissa bits: |error| <= 2^-20 + 2^-22.5 < 1.3e-6.
// ---------------------------------------------------------------------------------------
// log2(x) = e + f for a positive normal double; false for 0, subnormal, inf, nan
__device__ __forceinline__ bool log2_split(double x, int& e, float& f)
{
    const unsigned long long b = (unsigned long long)__double_as_longlong(x);
    const int ex = (int)((b >> 52) & 0x7ffu);
    e = ex - 1023;
    f = __log2f(__int_as_float(0x3f800000 | (unsigned)((b >> 29) & 0x7fffffu)));
    return ex != 0 && ex != 0x7ff && (b >> 63) == 0;
}

// r < min(1, (q / D)^invT) with q = (wu*wv)*s (canonical, double) ?  1 / 0, or -1 when the float
// estimate cannot decide.  log2 ratio = log2 q - log2 D (error <= 2 * 1.3e-6 + float rounding
// 2.4e-7 < 3e-6); log2 r error <= 1.3e-6; margins 1e-5 (ratio vs 1) and 1e-5 * invT + 2e-6.
__device__ __forceinline__ int fast_lt_prob(double r, double q, double Dp, double invT)
{
    int e1, e4, e5;
    float f1, f4, f5;
    bool ok = log2_split(q, e1, f1);
    ok &= log2_split(Dp, e4, f4);
    ok &= log2_split(r, e5, f5);
    if (!ok) return -1;
    const double lr = (double)(e1 - e4) + (double)(f1 - f4);
    if (lr > 1e-5) return 1;   // ratio > 1: p = 1 > r
    if (lr > -1e-5) return -1;
    const double diff = invT * lr - ((double)e5 + (double)f5);  // log2 p - log2 r
    const double margin = 1e-5 * invT + 2e-6;
    if (diff > margin) return 1;
    if (diff < -margin) return 0;
    return -1;
}

// geometric jump (R10): z = log(1-rj)/log1p(-pbar) = log2(y)/log2(1-pbar), y = 1-rj in (0,1),
// il2 = 1/log2(1-pbar) < 0.  Returns 1: stop (z >= remaining), 0: land at skip k = floor(z),
// -1: undecided.  |z error| <= 1.3e-6 |il2| (+ rounding): margin 2e-6 |il2| + 1e-12 z + 1e-12.
__device__ __forceinline__ int fast_jump(double y, double il2, long long remaining, long long& k)
{
    int e;
    float f;
    if (!log2_split(y, e, f)) return -1;
    const double z = ((double)e + (double)f) * il2;
    const double margin = 2e-6 * fabs(il2) + 1e-12 * z + 1e-12;
    const double rem = (double)remaining;
    if (z - margin >= rem) return 1;
    if (z + margin >= rem) return -1;
    const double lo = floor(z - margin), hi = floor(z + margin);
    if (lo != hi || lo < 0.0) return -1;
    k = (long long)lo;
    return 0;
}

}  // namespace girg
