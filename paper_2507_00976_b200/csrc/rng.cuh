// rng.cuh — device implementation of the sketch RNG spec.
//
// The paper draws the sketching operator S (d x m, iid N(0,1)) once from a counter-based
// generator (P:293 Random123; P:476 step bqrrp:sample; §3.2; variance-one reading Z3).
// This is the CUDA side's own implementation of the written spec (Philox4x32-10 + Box-Muller with
// self-written log and cos(2*pi*u)).  Every floating-point operation is an explicitly rounded
// intrinsic (__dadd_rn / __dmul_rn / __ddiv_rn / __dsqrt_rn), so no FMA contraction can occur and
// each entry is bit-identical to any other IEEE implementation of the same sequence of operations.
#pragma once
#include <cstdint>

namespace bqrrp {

__device__ __forceinline__ void philox4x32_10(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t& c3, uint32_t k0,
                                              uint32_t k1)
{
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
        uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
        uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}

// log(x), x in (0,1]: x = 2^e f, f in [sqrt2/2, sqrt2), s = (f-1)/(f+1), log f = 2 atanh s.
__device__ __forceinline__ double rng_log(double x)
{
    const double inv_odd[12] = {0x1.5555555555555p-2, 0x1.999999999999ap-3, 0x1.2492492492492p-3,
                                0x1.c71c71c71c71cp-4, 0x1.745d1745d1746p-4, 0x1.3b13b13b13b14p-4,
                                0x1.1111111111111p-4, 0x1.e1e1e1e1e1e1ep-5, 0x1.af286bca1af28p-5,
                                0x1.8618618618618p-5, 0x1.642c8590b2164p-5, 0x1.47ae147ae147bp-5};
    const double ln2_hi = 0x1.62e42fee00000p-1, ln2_lo = 0x1.a39ef35793c76p-33, sqrt2 = 0x1.6a09e667f3bcdp+0;
    unsigned long long bits = (unsigned long long)__double_as_longlong(x);
    int e = (int)((bits >> 52) & 0x7ff) - 1023;
    double f = __longlong_as_double((long long)((bits & 0x000fffffffffffffull) | 0x3ff0000000000000ull));
    if (f > sqrt2) { f = __dmul_rn(f, 0.5); e += 1; }
    double s = __ddiv_rn(__dsub_rn(f, 1.0), __dadd_rn(f, 1.0));
    double s2 = __dmul_rn(s, s);
    double p = inv_odd[11];
#pragma unroll
    for (int k = 10; k >= 0; --k) p = __dadd_rn(__dmul_rn(p, s2), inv_odd[k]);
    double two_s = __dmul_rn(2.0, s);
    double lf = __dadd_rn(two_s, __dmul_rn(two_s, __dmul_rn(s2, p)));
    double ed = (double)e;
    return __dadd_rn(__dmul_rn(ed, ln2_hi), __dadd_rn(__dmul_rn(ed, ln2_lo), lf));
}

__device__ __forceinline__ double rng_poly_sin(double x)
{
    const double c[9] = {-0x1.5555555555555p-3, 0x1.1111111111111p-7, -0x1.a01a01a01a01ap-13,
                         0x1.71de3a556c734p-19, -0x1.ae64567f544e4p-26, 0x1.6124613a86d09p-33,
                         -0x1.ae7f3e733b81fp-41, 0x1.952c77030ad4ap-49, -0x1.2f49b46814157p-57};
    double x2 = __dmul_rn(x, x), p = c[8];
#pragma unroll
    for (int k = 7; k >= 0; --k) p = __dadd_rn(__dmul_rn(p, x2), c[k]);
    return __dadd_rn(x, __dmul_rn(x, __dmul_rn(x2, p)));
}
__device__ __forceinline__ double rng_poly_cos(double x)
{
    const double c[9] = {-0x1.0000000000000p-1, 0x1.5555555555555p-5, -0x1.6c16c16c16c17p-10,
                         0x1.a01a01a01a01ap-16, -0x1.27e4fb7789f5cp-22, 0x1.1eed8eff8d898p-29,
                         -0x1.93974a8c07c9dp-37, 0x1.ae7f3e733b81fp-45, -0x1.6827863b97d97p-53};
    double x2 = __dmul_rn(x, x), p = c[8];
#pragma unroll
    for (int k = 7; k >= 0; --k) p = __dadd_rn(__dmul_rn(p, x2), c[k]);
    return __dadd_rn(1.0, __dmul_rn(x2, p));
}

// cos(2 pi u), u in [0,1): t = 4u = q + r exactly, fold r to [0, 1/2].
__device__ __forceinline__ double rng_cos2pi(double u)
{
    const double half_pi = 0x1.921fb54442d18p+0;
    double t = __dmul_rn(4.0, u);
    int q = (int)t;
    double r = __dsub_rn(t, (double)q);
    double cr, sr;
    if (r <= 0.5) {
        double x = __dmul_rn(half_pi, r);
        cr = rng_poly_cos(x);
        sr = rng_poly_sin(x);
    } else {
        double x = __dmul_rn(half_pi, __dsub_rn(1.0, r));
        cr = rng_poly_sin(x);
        sr = rng_poly_cos(x);
    }
    switch (q & 3) {
    case 0: return cr;
    case 1: return -sr;
    case 2: return -cr;
    default: return sr;
    }
}

// N(0,1) entry (i, j) of stream `stream` (0 = sketch S, 1 = test matrices).
__device__ __forceinline__ double rng_gauss(uint64_t seed, uint32_t stream, uint64_t i, uint64_t j)
{
    uint32_t c0 = (uint32_t)i, c1 = (uint32_t)j, c2 = (uint32_t)(j >> 32), c3 = stream;
    philox4x32_10(c0, c1, c2, c3, (uint32_t)seed, (uint32_t)(seed >> 32));
    unsigned long long a = ((unsigned long long)c0 << 32) | c1;
    unsigned long long c = ((unsigned long long)c2 << 32) | c3;
    double u1 = __dmul_rn(__dadd_rn((double)(a >> 12), 0.5), 0x1p-52);
    double u2 = __dmul_rn((double)(c >> 11), 0x1p-53);
    return __dmul_rn(__dsqrt_rn(__dmul_rn(-2.0, rng_log(u1))), rng_cos2pi(u2));
}

}  // namespace bqrrp
