// numerics.cuh — the bit-exact numerics contract as
// sm_100a device functions.  Every floating-point expression of the reference
// that feeds a scheduling decision is reproduced here with explicit
// round-to-nearest intrinsics (no FMA contraction regardless of --fmad), IEEE
// division, half-even rounding and exact integer arithmetic.
#pragma once
#include <stdint.h>

#define SLOSIM_INF64 0x7fffffffffffffffLL

namespace slosim {

__device__ __forceinline__ double xadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double xsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double xmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double xdiv(double a, double b) { return __ddiv_rn(a, b); }

// RN(a/x) > RN(b/y) for a > b >= 1 small integers and x, y > 0 finite (the
// throughput test of decode_sched.py:87-89).  The products a*y and b*x carry
// at most 2^-53 relative error each; when they differ by more than 2^-50
// relative, the exact quotients differ by more than the two roundings can
// close, so the product comparison decides; otherwise divide exactly.
__device__ __forceinline__ bool quot_gt(double a, double x, double b, double y) {
    double p = __dmul_rn(a, y), q = __dmul_rn(b, x);
    if (p > __dmul_rn(q, 1.0 + 0x1p-50)) return true;
    if (p < __dmul_rn(q, 1.0 - 0x1p-50)) return false;
    return __ddiv_rn(a, x) > __ddiv_rn(b, y);
}

// Python round(x) for floats: half-to-even (engine.py:183,192; costmodel.py:303).
__device__ __forceinline__ int64_t rint_i64(double x) { return __double2ll_rn(x); }

__device__ __forceinline__ int bitlen_u128(unsigned __int128 x) {
    uint64_t h = (uint64_t)(x >> 64), l = (uint64_t)x;
    return h ? 128 - __clzll((long long)h) : (l ? 64 - __clzll((long long)l) : 0);
}

// Python int/int true division of 128-bit operands: the correctly rounded
// double (long division with a sticky bit, half-even on the 53-bit mantissa).
__device__ __noinline__ double idiv128(__int128 p, __int128 q) {
    bool neg = (p < 0) != (q < 0);
    unsigned __int128 a = p < 0 ? (unsigned __int128)(-p) : (unsigned __int128)p;
    unsigned __int128 b = q < 0 ? (unsigned __int128)(-q) : (unsigned __int128)q;
    if (a == 0) return neg ? -0.0 : 0.0;
    int s = 55 - (bitlen_u128(a) - bitlen_u128(b));
    unsigned __int128 num = a, den = b;
    if (s >= 0) num <<= s; else den <<= -s;
    unsigned __int128 Q = num / den, R = num % den;
    int drop = bitlen_u128(Q) - 53;
    unsigned __int128 mant = Q >> drop;
    unsigned __int128 low = Q & ((((unsigned __int128)1) << drop) - 1);
    unsigned __int128 half = ((unsigned __int128)1) << (drop - 1);
    if (low > half || (low == half && (R != 0 || (mant & 1)))) mant++;
    double r = scalbn((double)(uint64_t)mant, drop - s);
    return neg ? -r : r;
}

// Python int/int true division (correctly rounded).  Fast path when both
// operands convert to double exactly: IEEE division is then correctly rounded.
__device__ __forceinline__ double idiv(int64_t p, int64_t q) {
    const int64_t lim = (int64_t)1 << 53;
    if (p > -lim && p < lim && q > -lim && q < lim) return xdiv((double)p, (double)q);
    return idiv128((__int128)p, (__int128)q);
}

// (a*b)/c with the exact integer product (curve arithmetic, engine.py:167,172).
__device__ __forceinline__ double idiv_prod(int64_t a, int64_t b, int64_t c) {
    __int128 p = (__int128)a * (__int128)b;
    const __int128 lim = ((__int128)1) << 53;
    if (p > -lim && p < lim && c > -(1LL << 53) && c < (1LL << 53)) return xdiv((double)(int64_t)p, (double)c);
    return idiv128(p, (__int128)c);
}

// ceil(tokens * busy / total), exact (costmodel.py:267-268).  The quotient is
// estimated with one f64 division and corrected with the exact integer
// remainder (|error| <= 1 unit for the operand ranges of the engine); a
// 128-bit long division handles products >= 2^62.
__device__ __noinline__ int64_t ceil_muldiv_slow(int64_t tokens, int64_t busy, int64_t total) {
    unsigned __int128 num = (unsigned __int128)(uint64_t)tokens * (uint64_t)busy;
    return (int64_t)((num + (unsigned __int128)total - 1) / (unsigned __int128)total);
}

__device__ __forceinline__ int64_t ceil_muldiv(int64_t tokens, int64_t busy, int64_t total) {
    if (tokens == 0) return 0;
    uint64_t hi = __umul64hi((uint64_t)tokens, (uint64_t)busy);
    uint64_t n = (uint64_t)tokens * (uint64_t)busy;
    if (hi != 0 || n >= (1ULL << 62)) return ceil_muldiv_slow(tokens, busy, total);
    uint64_t d = (uint64_t)total;
    uint64_t q = (uint64_t)__ddiv_rz((double)n, (double)d);
    int64_t r = (int64_t)(n - q * d);
    int guard = 0;
    while (r < 0) { q--; r += (int64_t)d; if (++guard > 4) return ceil_muldiv_slow(tokens, busy, total); }
    while (r >= (int64_t)d) { q++; r -= (int64_t)d; if (++guard > 4) return ceil_muldiv_slow(tokens, busy, total); }
    return (int64_t)(q + (r != 0));
}

// Decision digest: D <- fold((D ^ x) * phi64),
// and a 32-bit per-member hash summed over a decode batch (order-free).
__device__ __forceinline__ uint64_t dstep(uint64_t D, uint64_t x) {
    uint64_t z = (D ^ x) * 0x9E3779B97F4A7C15ULL;
    return z ^ (z >> 32);
}
__device__ __forceinline__ uint32_t member_hash(uint32_t pos) { return (pos + 1u) * 0x9E3779B1u; }

// splitmix64 finalizer.
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x ^= x >> 30; x *= 0xbf58476d1ce4e5b9ULL;
    x ^= x >> 27; x *= 0x94d049bb133111ebULL;
    x ^= x >> 31;
    return x;
}

// Orderable key of a double: ascending u64 order == ascending value, -0.0 == +0.0.
__device__ __forceinline__ uint64_t dkey(double x) {
    if (x == 0.0) x = 0.0;
    uint64_t b = (uint64_t)__double_as_longlong(x);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}

// numpy PCG64 (XSL-RR 128/64): step then output (engine.py:191, 225).
struct Pcg64 { uint64_t shi, slo, ihi, ilo; };
__device__ __forceinline__ uint64_t pcg_next(Pcg64& g) {
    const uint64_t mh = 0x2360ED051FC65DA4ULL, ml = 0x4385DF649FCCF645ULL;
    uint64_t lo = g.slo * ml;
    uint64_t hi = __umul64hi(g.slo, ml) + g.slo * mh + g.shi * ml;
    uint64_t nlo = lo + g.ilo;
    uint64_t carry = nlo < lo ? 1ULL : 0ULL;
    uint64_t nhi = hi + g.ihi + carry;
    g.slo = nlo; g.shi = nhi;
    unsigned rot = (unsigned)(nhi >> 58);
    uint64_t x = nhi ^ nlo;
    return (x >> rot) | (x << ((64u - rot) & 63u));
}
// Generator.uniform(low, high) = low + (high - low) * next_double
__device__ __forceinline__ double pcg_uniform(Pcg64& g, double low, double high) {
    double u = xmul((double)(pcg_next(g) >> 11), 1.0 / 9007199254740992.0);
    return xadd(low, xmul(xsub(high, low), u));
}

}  // namespace slosim
