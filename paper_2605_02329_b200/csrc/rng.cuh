// rng.cuh — the reference's workload generator on the device.
//
// gen_longtail (/root/reference/pkg/src/slosim/workload.py:88-112) draws every trace from
// numpy's default_rng(seed): SeedSequence -> PCG64, then exponential gaps, uniforms, two
// lognormal series and bounded integers.  This header restates, operation for operation,
// the code those calls execute in numpy 2.3.5 and in the glibc 2.39 libm it calls:
//
//   SeedSequence            numpy/random/bit_generator.pyx (mix_entropy, generate_state)
//   PCG64                   numpy/random/src/pcg64/pcg64.h (XSL-RR 128/64, buffered 32-bit half)
//   next_double             (x >> 11) * 2^-53
//   standard_exponential    distributions.c random_standard_exponential (256-level ziggurat)
//   standard_normal         distributions.c random_standard_normal (256-level ziggurat)
//   lognormal               exp(mean + sigma * standard_normal)
//   integers (int64)        random_bounded_uint64_fill -> buffered_bounded_lemire_uint32
//   exp, log1p              glibc's x86-64 FMA variants (__exp_fma, __log1p_fma), the ones the
//                           dynamic linker selects on every FMA-capable x86-64 host: the fused
//                           operations below are the vfmadd/vfnmadd/vfmsub of that code
//
// Every operation is an explicit IEEE double add/sub/mul/div or fma (the library is compiled
// with --fmad=false, host builds with -ffp-contract=off), so the device produces the same bits
// as numpy on the host.  The header compiles both for the device and as host C++ (the test
// harness tools/rng_host), like tengine.cuh.
#pragma once
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "../../include/slosim_b200.h"
#include "rng_tables.h"

#ifdef __CUDACC__
#define RNG_HD __host__ __device__ __forceinline__
#else
#define RNG_HD inline
#endif

namespace slosim {
namespace rng {

typedef unsigned __int128 u128;

RNG_HD uint64_t asu64(double x) {
#ifdef __CUDA_ARCH__
    return (uint64_t)__double_as_longlong(x);
#else
    uint64_t u;
    memcpy(&u, &x, 8);
    return u;
#endif
}
RNG_HD double asf64(uint64_t u) {
#ifdef __CUDA_ARCH__
    return __longlong_as_double((long long)u);
#else
    double x;
    memcpy(&x, &u, 8);
    return x;
#endif
}

// ------------------------------------------------------------------ SeedSequence
// bit_generator.pyx: entropy = the seed as little-endian 32-bit words ([0] for 0), pool of 4.
constexpr uint32_t INIT_A = 0x43b0d7e5u, MULT_A = 0x931e8875u, INIT_B = 0x8b51f9ddu, MULT_B = 0x58f38dedu;
constexpr uint32_t MIX_MULT_L = 0xca01f9ddu, MIX_MULT_R = 0x4973f715u;

RNG_HD uint32_t hashmix(uint32_t v, uint32_t& hc) {
    v ^= hc;
    hc *= MULT_A;
    v *= hc;
    return v ^ (v >> 16);
}
RNG_HD uint32_t mix(uint32_t x, uint32_t y) {
    uint32_t r = MIX_MULT_L * x - MIX_MULT_R * y;
    return r ^ (r >> 16);
}

// generate_state(4, uint64) of SeedSequence(seed): words[0..3].
RNG_HD void seed_sequence(uint64_t seed, uint64_t out[4]) {
    uint32_t ent[2];
    int n_ent = 0;
    if (seed == 0) {
        ent[n_ent++] = 0;
    } else {
        while (seed) { ent[n_ent++] = (uint32_t)seed; seed >>= 32; }
    }
    uint32_t pool[4];
    uint32_t hc = INIT_A;
    for (int i = 0; i < 4; i++) pool[i] = hashmix(i < n_ent ? ent[i] : 0u, hc);
    for (int s = 0; s < 4; s++)
        for (int d = 0; d < 4; d++)
            if (s != d) pool[d] = mix(pool[d], hashmix(pool[s], hc));
    // (entropy beyond the pool size: at most 2 words here, never)
    uint32_t hb = INIT_B;
    uint32_t w[8];
    for (int i = 0; i < 8; i++) {
        uint32_t v = pool[i & 3];
        v ^= hb;
        hb *= MULT_B;
        v *= hb;
        w[i] = v ^ (v >> 16);
    }
    for (int k = 0; k < 4; k++) out[k] = (uint64_t)w[2 * k] | ((uint64_t)w[2 * k + 1] << 32);
}

// ------------------------------------------------------------------ PCG64
constexpr uint64_t PCG_MULT_HI = 0x2360ED051FC65DA4ULL, PCG_MULT_LO = 0x4385DF649FCCF645ULL;

struct Pcg {
    u128 state, inc;
    uint32_t u32;
    bool has32;
};

RNG_HD void pcg_step(Pcg& g) {
    const u128 mult = ((u128)PCG_MULT_HI << 64) | PCG_MULT_LO;
    g.state = g.state * mult + g.inc;
}

// default_rng(seed): PCG64(SeedSequence(seed)), pcg64_set_seed -> pcg_setseq_128_srandom_r.
RNG_HD void pcg_seed(Pcg& g, uint64_t seed) {
    uint64_t v[4];
    seed_sequence(seed, v);
    const u128 initstate = ((u128)v[0] << 64) | v[1];
    const u128 initseq = ((u128)v[2] << 64) | v[3];
    g.state = 0;
    g.inc = (initseq << 1) | 1;
    pcg_step(g);
    g.state += initstate;
    pcg_step(g);
    g.u32 = 0;
    g.has32 = false;
}

RNG_HD uint64_t next_u64(Pcg& g) {
    pcg_step(g);
    const uint64_t hi = (uint64_t)(g.state >> 64), lo = (uint64_t)g.state;
    const unsigned rot = (unsigned)(hi >> 58);
    const uint64_t x = hi ^ lo;
    return (x >> rot) | (x << ((64u - rot) & 63u));
}

// pcg64_next32: the low half now, the high half buffered for the next call.
RNG_HD uint32_t next_u32(Pcg& g) {
    if (g.has32) {
        g.has32 = false;
        return g.u32;
    }
    const uint64_t x = next_u64(g);
    g.has32 = true;
    g.u32 = (uint32_t)(x >> 32);
    return (uint32_t)x;
}

RNG_HD double next_double(Pcg& g) { return (double)(next_u64(g) >> 11) * (1.0 / 9007199254740992.0); }

// ------------------------------------------------------------------ libm: exp (__exp_fma)
// exp(x) = 2^(k/128) * exp(r), |r| <= ln2/256: table scale + tail, degree-5 polynomial.
constexpr double EXP_INVLN2N = 0x1.71547652b82fep7, EXP_SHIFT = 0x1.8p52;
constexpr double EXP_NEGLN2HIN = -0x1.62e42fefa0000p-8, EXP_NEGLN2LON = -0x1.cf79abc9e3b3ap-47;
constexpr double EXP_C2 = 0x1.ffffffffffdbdp-2, EXP_C3 = 0x1.555555555543cp-3;
constexpr double EXP_C4 = 0x1.55555cf172b91p-5, EXP_C5 = 0x1.1111167a4d017p-7;

// Returns false when x is outside the range this restatement covers (|x| >= 512, inf, nan):
// glibc's special-case scaling is not restated; no draw of gen_longtail's defaults comes near.
RNG_HD bool gexp(double x, double& y) {
    const uint32_t abstop = (uint32_t)(asu64(x) >> 52) & 0x7ff;
    if (abstop - 0x3c9u > 0x3eu) {
        if ((int32_t)(abstop - 0x3c9u) < 0) {  // |x| < 2^-54
            y = 1.0 + x;
            return true;
        }
        return false;
    }
    double kd = fma(x, EXP_INVLN2N, EXP_SHIFT);
    const uint64_t ki = asu64(kd);
    kd = kd - EXP_SHIFT;
    double r = fma(kd, EXP_NEGLN2HIN, x);
    r = fma(kd, EXP_NEGLN2LON, r);
    const uint32_t idx = 2u * (uint32_t)(ki & 127u);
    const uint64_t top = ki << 45;
    const double tail = asf64(exp_tab[idx]);
    const uint64_t sbits = exp_tab[idx + 1] + top;
    const double r2 = r * r;
    const double p23 = fma(r, EXP_C3, EXP_C2);
    const double t0 = r + tail;
    const double p45 = fma(r, EXP_C5, EXP_C4);
    double tmp = fma(p23, r2, t0);
    const double r4 = r2 * r2;
    tmp = fma(r4, p45, tmp);
    const double scale = asf64(sbits);
    y = fma(scale, tmp, scale);
    return true;
}

// ------------------------------------------------------------------ libm: log1p (__log1p_fma)
// fdlibm's log1p (k, f with 1+x = 2^k (1+f), s = f/(2+f), degree-14 even polynomial).
constexpr double L_LN2_HI = 0x1.62e42feep-1, L_LN2_LO = 0x1.a39ef35793c76p-33;
constexpr double Lp1 = 0x1.5555555555593p-1, Lp2 = 0x1.999999997fa04p-2, Lp3 = 0x1.2492494229359p-2;
constexpr double Lp4 = 0x1.c71c51d8e78afp-3, Lp5 = 0x1.7466496cb03dep-3, Lp6 = 0x1.39a09d078c69fp-3;
constexpr double Lp7 = 0x1.2f112df3e5244p-3;

RNG_HD double set_high(double u, uint32_t hi) { return asf64(((uint64_t)hi << 32) | (asu64(u) & 0xffffffffULL)); }

// For x > -1 (finite).  Returns false outside that domain.
RNG_HD bool glog1p(double x, double& y) {
    const int32_t hx = (int32_t)(asu64(x) >> 32);
    const uint32_t ax = (uint32_t)hx & 0x7fffffffu;
    int k;
    double f, c = 0.0, hfsq;
    uint32_t hu;
    if (hx <= 0x3fda8279) {  // x < 0.41422, including every negative x
        if (ax > 0x3fefffffu) return false;  // x <= -1
        if (ax <= 0x3e1fffffu) {              // |x| < 2^-29
            if (ax <= 0x3c8fffffu) { y = x; return true; }
            y = fma(-(x * x), 0.5, x);
            return true;
        }
        if ((uint32_t)hx + 0x402d413cu > 0x402d413cu) {  // -0.2929 < x < 0.41422: k = 0, f = x
            k = 0;
            f = x;
            hfsq = (x * 0.5) * x;
            hu = 1;
            goto poly;
        }
    } else if (hx > 0x7fefffff) {
        return false;  // inf / nan
    } else if (hx > 0x433fffff) {  // x >= 2^53: 1 + x == x
        k = (hx >> 20) - 1023;
        hu = (uint32_t)hx;
        double u = x;
        c = 0.0;
        hu &= 0x000fffffu;
        if (hu > 0x6a09du) {
            k += 1;
            u = set_high(u, hu | 0x3fe00000u);
            hu = (0x00100000u - hu) >> 2;
        } else {
            u = set_high(u, hu | 0x3ff00000u);
        }
        f = u - 1.0;
        hfsq = (f * 0.5) * f;
        goto small_f;
    }
    {
        double u = x + 1.0;
        hu = (uint32_t)(asu64(u) >> 32);
        k = (int32_t)(hu >> 20) - 1023;
        c = k > 0 ? 1.0 - (u - x) : x - (u - 1.0);  // correction term
        c = c / u;
        hu &= 0x000fffffu;
        if (hu > 0x6a09du) {
            k += 1;
            u = set_high(u, hu | 0x3fe00000u);  // normalize u/2
            hu = (0x00100000u - hu) >> 2;
        } else {
            u = set_high(u, hu | 0x3ff00000u);  // normalize u
        }
        f = u - 1.0;
        hfsq = (f * 0.5) * f;
    }
small_f:
    if (hu == 0) {  // |f| < 2^-20
        if (f == 0.0) {
            if (k == 0) { y = 0.0; return true; }
            const double kd = (double)k;
            y = fma(kd, L_LN2_HI, fma(kd, L_LN2_LO, c));
            return true;
        }
        const double R = fma(-f, 0.66666666666666666, 1.0) * hfsq;
        if (k == 0) { y = f - R; return true; }
        const double kd = (double)k;
        y = fma(kd, L_LN2_HI, -((R - fma(kd, L_LN2_LO, c)) - f));
        return true;
    }
poly : {
    const double s = f / (f + 2.0);
    const double z = s * s;
    const double R2 = fma(z, Lp3, Lp2);
    const double R3 = fma(z, Lp5, Lp4);
    const double R4 = fma(z, Lp7, Lp6);
    const double z2 = z * z;
    const double z4 = z2 * z2;
    const double z6 = z2 * z4;
    double R = fma(z, Lp1, z2 * R2);
    R = fma(z4, R3, R);
    R = fma(z6, R4, R);
    const double q = s * (R + hfsq);
    if (k == 0) { y = f - (hfsq - q); return true; }
    const double kd = (double)k;
    double w = fma(kd, L_LN2_LO, c);
    w = w + q;
    w = hfsq - w;
    w = w - f;
    y = fma(kd, L_LN2_HI, -w);
    return true;
}
}

// ------------------------------------------------------------------ distributions
// `ok` is cleared when a libm call leaves the restated domain (never for gen_longtail's defaults).
RNG_HD double standard_exponential(Pcg& g, bool& ok) {
    for (;;) {
        uint64_t ri = next_u64(g);
        ri >>= 3;
        const uint32_t idx = (uint32_t)(ri & 0xff);
        ri >>= 8;
        const double x = (double)ri * we_double[idx];
        if (ri < ke_double[idx]) return x;  // 98.9% of draws
        if (idx == 0) {
            double l;
            ok &= glog1p(-next_double(g), l);
            return ZIG_EXP_R - l;
        }
        double e;
        ok &= gexp(-x, e);
        if ((fe_double[idx - 1] - fe_double[idx]) * next_double(g) + fe_double[idx] < e) return x;
    }
}

RNG_HD double standard_normal(Pcg& g, bool& ok) {
    for (;;) {
        uint64_t r = next_u64(g);
        const uint32_t idx = (uint32_t)(r & 0xff);
        r >>= 8;
        const uint64_t sign = r & 0x1;
        const uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
        double x = (double)rabs * wi_double[idx];
        if (sign & 0x1) x = -x;
        if (rabs < ki_double[idx]) return x;  // 99.3% of draws
        if (idx == 0) {
            for (;;) {
                double l1, l2;
                ok &= glog1p(-next_double(g), l1);
                const double xx = -ZIG_NOR_INV_R * l1;
                ok &= glog1p(-next_double(g), l2);
                const double yy = -l2;
                if (yy + yy > xx * xx) return ((rabs >> 8) & 0x1) ? -(ZIG_NOR_R + xx) : ZIG_NOR_R + xx;
            }
        }
        double e;
        ok &= gexp(-0.5 * x * x, e);
        if ((fi_double[idx - 1] - fi_double[idx]) * next_double(g) + fi_double[idx] < e) return x;
    }
}

RNG_HD double lognormal(Pcg& g, double mean, double sigma, bool& ok) {
    double y;
    ok &= gexp(mean + sigma * standard_normal(g, ok), y);
    return y;
}

// buffered_bounded_lemire_uint32 (rng = high - low, 0 < rng < 2^32 - 1).
RNG_HD uint32_t bounded_lemire32(Pcg& g, uint32_t rng) {
    const uint32_t rng_excl = rng + 1u;
    uint64_t m = (uint64_t)next_u32(g) * rng_excl;
    uint32_t leftover = (uint32_t)m;
    if (leftover < rng_excl) {
        const uint32_t threshold = (0xffffffffu - rng) % rng_excl;
        while (leftover < threshold) {
            m = (uint64_t)next_u32(g) * rng_excl;
            leftover = (uint32_t)m;
        }
    }
    return (uint32_t)(m >> 32);
}

// Generator.integers(low, high_exclusive) for int64 with a range below 2^32 - 1.
RNG_HD int64_t integers(Pcg& g, int64_t low, int64_t high_excl) {
    const uint64_t rng = (uint64_t)(high_excl - 1 - low);
    if (rng == 0) return low;
    return low + (int64_t)bounded_lemire32(g, (uint32_t)rng);
}

RNG_HD int64_t rint64(double x) {
#ifdef __CUDA_ARCH__
    return __double2ll_rn(x);
#else
    return (int64_t)nearbyint(x);
#endif
}

// ------------------------------------------------------------------ gen_longtail (workload.py:88-112)
// LongTailSpec.__post_init__ (workload.py:73-85), plus what the restatement covers: a tail range
// below 2^32 - 1 (numpy's 32-bit Lemire path) and the trace inside the output table.
RNG_HD bool spec_ok(const slosim_longtail_spec_t& s, int64_t n_total) {
    return s.qps > 0 && s.n_requests >= 0 && s.p_long >= 0.0 && s.p_long <= 1.0 &&
           s.long_len_min <= s.long_len_max && s.long_len_min >= 1 && s.short_len_log_sigma >= 0 &&
           s.out_len_log_sigma >= 0 && s.long_len_max - s.long_len_min < 0xFFFFFFFELL &&
           s.long_len_max <= 0x7FFFFFFFLL && s.offset >= 0 && s.offset <= n_total - s.n_requests;
}

RNG_HD int gen_longtail_one(const slosim_longtail_spec_t& s, int64_t* arr, int32_t* inp, int32_t* out, int32_t* hit,
                       int32_t* idr) {
    Pcg g;
    pcg_seed(g, s.seed);
    const int64_t n = s.n_requests;
    bool ok = true;
    // gaps = exponential(1/qps, n); arrivals_s = cumsum(gaps)
    const double scale = 1.0 / s.qps;
    double acc = 0.0;
    for (int64_t k = 0; k < n; k++) {
        acc = acc + scale * standard_exponential(g, ok);
        arr[k] = rint64(acc * 1000000.0);
        hit[k] = 0;
        idr[k] = (int32_t)k;
    }
    // is_long = random(n) < p_long (kept as a mark in input_len until the tail draws)
    for (int64_t k = 0; k < n; k++) inp[k] = next_double(g) < s.p_long ? -1 : 0;
    // body = lognormal(short mean, short sigma, n): input = max(1, round(body)) when not long
    for (int64_t k = 0; k < n; k++) {
        const double b = lognormal(g, s.short_len_log_mean, s.short_len_log_sigma, ok);
        if (inp[k] == 0) {
            const double r = b < 2147483647.0 ? b : 2147483647.0;
            if (!(b < 2147483647.5)) ok = false;  // token counts exceed int32 (TraceArrays raises)
            const int64_t v = rint64(r);
            inp[k] = (int32_t)(v < 1 ? 1 : v);
        }
    }
    // tail = integers(long_min, long_max + 1, n)
    for (int64_t k = 0; k < n; k++) {
        const int64_t t = integers(g, s.long_len_min, s.long_len_max + 1);
        if (inp[k] == -1) inp[k] = (int32_t)t;
    }
    // outputs = lognormal(out mean, out sigma, n): output = max(1, round(outputs))
    for (int64_t k = 0; k < n; k++) {
        const double o = lognormal(g, s.out_len_log_mean, s.out_len_log_sigma, ok);
        if (!(o < 2147483647.5)) ok = false;
        const int64_t v = rint64(o < 2147483647.0 ? o : 2147483647.0);
        out[k] = (int32_t)(v < 1 ? 1 : v);
    }
    return ok ? SLOSIM_OK : SLOSIM_ERANGE;
}

}  // namespace rng
}  // namespace slosim
