// longtail.cu — gen_longtail on the device (workload.py:88-112).
//
// One thread generates one trace: the draws of a trace form one sequential PCG64 stream
// (exponential gaps, then uniforms, lognormal bodies, bounded integers and lognormal outputs,
// each series over all n requests), so a trace is the unit of parallelism.  The arrival
// cumsum is the sequential left-to-right f64 sum numpy.cumsum computes; each value is written
// once, as the integer microseconds seconds_to_us makes of it (domain.py:20-25).  Requests
// come out in position order: ids r{k:0w} sort by position and arrivals never decrease, so
// the reference's sort by (arrival, id) (workload.py:111) is the identity and id_rank = k.
#include <cuda_runtime.h>

#include "../../include/slosim_b200.h"
#include "rng.cuh"

using namespace slosim;

int slosim_internal_fail(int code, const char* what, cudaError_t e);  // capi.cu (slosim_last_error)

#define LCK(call)                                                              \
    do {                                                                       \
        cudaError_t e_ = (call);                                               \
        if (e_ != cudaSuccess) return slosim_internal_fail(SLOSIM_ECUDA, #call, e_); \
    } while (0)

namespace {

__global__ void k_gen_longtail(const slosim_longtail_spec_t* specs, int64_t n_specs, int64_t* arrival, int32_t* inp,
                               int32_t* out, int32_t* hit, int32_t* idr, int64_t n_total, int32_t* status) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_specs) return;
    const slosim_longtail_spec_t s = specs[i];
    if (!rng::spec_ok(s, n_total)) {
        status[i] = SLOSIM_EINVAL;
        return;
    }
    const int64_t o = s.offset;
    status[i] = rng::gen_longtail_one(s, arrival + o, inp + o, out + o, hit + o, idr + o);
}

// Test entry point: n draws per seed of one numpy Generator method.
__global__ void k_rng_draws(int32_t kind, const uint64_t* seeds, int64_t n_seeds, int64_t n, double p0, double p1,
                            uint64_t* out, int32_t* status) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_seeds) return;
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
    status[i] = ok ? SLOSIM_OK : SLOSIM_ERANGE;
}

__global__ void k_libm(int32_t fn, int64_t n, const double* x, double* y, uint8_t* ok) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double v = 0.0;
    const bool g = fn == 0 ? rng::gexp(x[i], v) : rng::glog1p(x[i], v);
    y[i] = v;
    ok[i] = g;
}

template <class T>
struct DevBuf {
    T* p = nullptr;
    ~DevBuf() { if (p) cudaFree(p); }
    cudaError_t alloc(int64_t n) { return cudaMalloc(&p, (size_t)(n > 0 ? n : 1) * sizeof(T)); }
};

}  // namespace

extern "C" int slosim_gen_longtail(const slosim_longtail_spec_t* d_specs, int64_t n_specs, int64_t* d_arrival_us,
                                   int32_t* d_input_len, int32_t* d_output_len, int32_t* d_prefix_hit_len,
                                   int32_t* d_id_rank, int64_t n_total, int32_t* d_status, void* stream) {
    if (n_specs < 0 || n_total < 0 || (n_specs > 0 && (!d_specs || !d_status)) ||
        (n_total > 0 && (!d_arrival_us || !d_input_len || !d_output_len || !d_prefix_hit_len || !d_id_rank)))
        return SLOSIM_EINVAL;
    if (n_specs == 0) return SLOSIM_OK;
    const int threads = 32;
    k_gen_longtail<<<(unsigned)((n_specs + threads - 1) / threads), threads, 0, (cudaStream_t)stream>>>(
        d_specs, n_specs, d_arrival_us, d_input_len, d_output_len, d_prefix_hit_len, d_id_rank, n_total, d_status);
    LCK(cudaGetLastError());
    return SLOSIM_OK;
}

extern "C" int slosim_gen_longtail_host(const slosim_longtail_spec_t* specs, int64_t n_specs, int64_t* arrival_us,
                                        int32_t* input_len, int32_t* output_len, int32_t* prefix_hit_len,
                                        int32_t* id_rank, int64_t n_total, int32_t* status) {
    if (n_specs < 0 || n_total < 0 || (n_specs > 0 && (!specs || !status)) ||
        (n_total > 0 && (!arrival_us || !input_len || !output_len || !prefix_hit_len || !id_rank)))
        return SLOSIM_EINVAL;
    if (n_specs == 0) return SLOSIM_OK;
    DevBuf<slosim_longtail_spec_t> ds;
    DevBuf<int64_t> da;
    DevBuf<int32_t> di, dout, dh, dr, dst;
    LCK(ds.alloc(n_specs)); LCK(da.alloc(n_total)); LCK(di.alloc(n_total)); LCK(dout.alloc(n_total));
    LCK(dh.alloc(n_total)); LCK(dr.alloc(n_total)); LCK(dst.alloc(n_specs));
    LCK(cudaMemcpy(ds.p, specs, n_specs * sizeof(*specs), cudaMemcpyHostToDevice));
    // positions no spec covers come back as they went in
    LCK(cudaMemcpy(da.p, arrival_us, n_total * 8, cudaMemcpyHostToDevice));
    LCK(cudaMemcpy(di.p, input_len, n_total * 4, cudaMemcpyHostToDevice));
    LCK(cudaMemcpy(dout.p, output_len, n_total * 4, cudaMemcpyHostToDevice));
    LCK(cudaMemcpy(dh.p, prefix_hit_len, n_total * 4, cudaMemcpyHostToDevice));
    LCK(cudaMemcpy(dr.p, id_rank, n_total * 4, cudaMemcpyHostToDevice));
    int rc = slosim_gen_longtail(ds.p, n_specs, da.p, di.p, dout.p, dh.p, dr.p, n_total, dst.p, nullptr);
    if (rc != SLOSIM_OK) return rc;
    LCK(cudaDeviceSynchronize());
    LCK(cudaMemcpy(arrival_us, da.p, n_total * 8, cudaMemcpyDeviceToHost));
    LCK(cudaMemcpy(input_len, di.p, n_total * 4, cudaMemcpyDeviceToHost));
    LCK(cudaMemcpy(output_len, dout.p, n_total * 4, cudaMemcpyDeviceToHost));
    LCK(cudaMemcpy(prefix_hit_len, dh.p, n_total * 4, cudaMemcpyDeviceToHost));
    LCK(cudaMemcpy(id_rank, dr.p, n_total * 4, cudaMemcpyDeviceToHost));
    LCK(cudaMemcpy(status, dst.p, n_specs * 4, cudaMemcpyDeviceToHost));
    return SLOSIM_OK;
}

extern "C" int slosim_rng_draws(int32_t kind, const uint64_t* seeds, int64_t n_seeds, int64_t n_per_seed, double p0,
                                double p1, uint64_t* out, int32_t* status) {
    if (n_seeds < 0 || n_per_seed < 0 || kind < 0 || kind > SLOSIM_DRAW_INTEGERS) return SLOSIM_EINVAL;
    if (kind == SLOSIM_DRAW_INTEGERS && !(p1 - p0 >= 1.0 && p1 - p0 <= 4294967295.0)) return SLOSIM_EINVAL;
    if (n_seeds == 0) return SLOSIM_OK;
    DevBuf<uint64_t> dseed, dout;
    DevBuf<int32_t> dst;
    LCK(dseed.alloc(n_seeds)); LCK(dout.alloc(n_seeds * n_per_seed)); LCK(dst.alloc(n_seeds));
    LCK(cudaMemcpy(dseed.p, seeds, n_seeds * 8, cudaMemcpyHostToDevice));
    k_rng_draws<<<(unsigned)((n_seeds + 63) / 64), 64>>>(kind, dseed.p, n_seeds, n_per_seed, p0, p1, dout.p, dst.p);
    LCK(cudaGetLastError());
    LCK(cudaDeviceSynchronize());
    LCK(cudaMemcpy(out, dout.p, n_seeds * n_per_seed * 8, cudaMemcpyDeviceToHost));
    LCK(cudaMemcpy(status, dst.p, n_seeds * 4, cudaMemcpyDeviceToHost));
    return SLOSIM_OK;
}

extern "C" int slosim_libm(int32_t fn, int64_t n, const double* x, double* y, uint8_t* ok) {
    if (n < 0 || fn < 0 || fn > 1) return SLOSIM_EINVAL;
    if (n == 0) return SLOSIM_OK;
    DevBuf<double> dx, dy;
    DevBuf<uint8_t> dok;
    LCK(dx.alloc(n)); LCK(dy.alloc(n)); LCK(dok.alloc(n));
    LCK(cudaMemcpy(dx.p, x, n * 8, cudaMemcpyHostToDevice));
    k_libm<<<(unsigned)((n + 255) / 256), 256>>>(fn, n, dx.p, dy.p, dok.p);
    LCK(cudaGetLastError());
    LCK(cudaMemcpy(y, dy.p, n * 8, cudaMemcpyDeviceToHost));
    LCK(cudaMemcpy(ok, dok.p, n, cudaMemcpyDeviceToHost));
    return SLOSIM_OK;
}
