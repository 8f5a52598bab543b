// Host build of the device workload generator (paper_2605_02329_b200/csrc/rng.cuh): the same
// source compiled as plain C++ (-ffp-contract=off), so the CPU test suite checks the restated
// numpy/glibc algorithms against numpy itself without a GPU (tests/test_rng_host.py).
#include <stdint.h>

#include "../../include/slosim_b200.h"
#include "../../paper_2605_02329_b200/csrc/rng.cuh"

using namespace slosim;

extern "C" void rng_host_seed_state(uint64_t seed, uint64_t out[4]) {
    rng::Pcg g;
    rng::pcg_seed(g, seed);
    out[0] = (uint64_t)(g.state >> 64); out[1] = (uint64_t)g.state;
    out[2] = (uint64_t)(g.inc >> 64); out[3] = (uint64_t)g.inc;
}

extern "C" int rng_host_libm(int fn, int64_t n, const double* x, double* y, uint8_t* ok) {
    for (int64_t i = 0; i < n; i++) {
        double v = 0.0;
        ok[i] = fn == 0 ? rng::gexp(x[i], v) : rng::glog1p(x[i], v);
        y[i] = v;
    }
    return 0;
}

extern "C" int rng_host_draws(int kind, const uint64_t* seeds, int64_t n_seeds, int64_t n, double p0, double p1,
                              uint64_t* out, int32_t* status) {
    for (int64_t i = 0; i < n_seeds; i++) {
        rng::Pcg g;
        rng::pcg_seed(g, seeds[i]);
        bool ok = true;
        uint64_t* o = out + i * n;
        for (int64_t k = 0; k < n; k++) {
            double v = 0.0;
            switch (kind) {
                case SLOSIM_DRAW_RAW: o[k] = rng::next_u64(g); continue;
                case SLOSIM_DRAW_RANDOM: v = rng::next_double(g); break;
                case SLOSIM_DRAW_STD_EXPONENTIAL: v = rng::standard_exponential(g, ok); break;
                case SLOSIM_DRAW_EXPONENTIAL: v = p0 * rng::standard_exponential(g, ok); break;
                case SLOSIM_DRAW_STD_NORMAL: v = rng::standard_normal(g, ok); break;
                case SLOSIM_DRAW_LOGNORMAL: v = rng::lognormal(g, p0, p1, ok); break;
                case SLOSIM_DRAW_INTEGERS: o[k] = (uint64_t)rng::integers(g, (int64_t)p0, (int64_t)p1); continue;
                default: ok = false; break;
            }
            o[k] = rng::asu64(v);
        }
        status[i] = ok ? 0 : SLOSIM_ERANGE;
    }
    return 0;
}

extern "C" int rng_host_gen_longtail(const slosim_longtail_spec_t* specs, int64_t n_specs, int64_t* arr, int32_t* inp,
                                     int32_t* out, int32_t* hit, int32_t* idr, int64_t n_total, int32_t* status) {
    for (int64_t i = 0; i < n_specs; i++) {
        const slosim_longtail_spec_t& s = specs[i];
        if (!rng::spec_ok(s, n_total)) { status[i] = SLOSIM_EINVAL; continue; }
        const int64_t o = s.offset;
        status[i] = rng::gen_longtail_one(s, arr + o, inp + o, out + o, hit + o, idr + o);
    }
    return 0;
}
