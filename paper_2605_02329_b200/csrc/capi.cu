// capi.cu — the C-ABI of include/slosim_b200.h: host entry points, device
// workspace management and the single-snapshot kernels (K7) that expose the
// policies and cost models of the engine one decision at a time.  The snapshot
// kernels call the very same device functions as the batched engine.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <mutex>
#include <vector>

#include "engine.cuh"
#include "tengine.cuh"

using namespace slosim;

// engine_lat.cu: the engine built for one block per SM (no spills), for small batches
cudaError_t slosim_launch_latency_engine(int grid, const void* cx, char* ws, size_t stride, int64_t cap,
                                         unsigned long long* work, cudaStream_t st);

namespace {

thread_local char g_err[512];
std::mutex g_mu;

int fail_cuda(cudaError_t e, const char* what) {
    snprintf(g_err, sizeof(g_err), "%s: %s", what, cudaGetErrorString(e));
    return SLOSIM_ECUDA;
}

#define CK(call)                                              \
    do {                                                      \
        cudaError_t e_ = (call);                              \
        if (e_ != cudaSuccess) return fail_cuda(e_, #call);   \
    } while (0)

// Grow-only device arena per purpose (the engine workspace, profile tables,
// work counter, snapshot scratch, host-entry staging), one set per device.
struct Arena {
    void* ptr = nullptr;
    size_t size = 0;
    // `busy`: last stream work that used the arena (waited on before it is freed)
    cudaError_t reserve(size_t bytes, cudaEvent_t busy = nullptr) {
        if (ptr && size >= bytes) return cudaSuccess;
        if (ptr) {
            if (busy) cudaEventSynchronize(busy);
            cudaFree(ptr);
        }
        ptr = nullptr;
        size = 0;
        size_t want = std::max(bytes, (size_t)1 << 20);
        cudaError_t e = cudaMalloc(&ptr, want);
        if (e != cudaSuccess) { ptr = nullptr; return e; }
        // zero once per allocation: the engine's branch-free LUT update reads (and discards) the
        // neighbour of an edge cell, which may lie outside the live part of a workspace LUT
        e = cudaMemset(ptr, 0, want);
        if (e != cudaSuccess) { cudaFree(ptr); ptr = nullptr; return e; }
        size = want;
        return cudaSuccess;
    }
};

// Per-device library state.  Engine launches on one device are serialised in
// stream order: each launch waits for the previous launch's `done` event
// (whatever stream it ran on) before it rewrites the shared workspace, profile
// tables and work counter, so concurrent callers on different streams get the
// results of sequential calls.
constexpr int kMaxDevices = 64;
struct DevState {
    Arena ws, tabs, work, snap, io, lws, defer;
    int sms = 0, blocks_per_sm = 0, lane_blocks_per_sm = 0;
    cudaEvent_t done = nullptr;
};
DevState g_dev[kMaxDevices];

int current_device(int* dev) {
    CK(cudaGetDevice(dev));
    if (*dev < 0 || *dev >= kMaxDevices) {
        snprintf(g_err, sizeof(g_err), "device %d beyond the library limit (%d)", *dev, kMaxDevices);
        return SLOSIM_ECUDA;
    }
    return SLOSIM_OK;
}

DevState& dev_state(int dev) { return g_dev[dev]; }

int launch_geometry(DevState& ds, int dev, int64_t n_instances, int* grid) {
    if (!ds.sms) {
        CK(cudaDeviceGetAttribute(&ds.sms, cudaDevAttrMultiProcessorCount, dev));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ds.blocks_per_sm, sim_kernel, 128, 0));
        if (ds.blocks_per_sm < 1) ds.blocks_per_sm = 1;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ds.lane_blocks_per_sm, lane::lane_kernel, 128, 0));
        if (ds.lane_blocks_per_sm < 1) ds.lane_blocks_per_sm = 1;
        if (const char* e = getenv("SLOSIM_LANE_BLOCKS_PER_SM")) {
            int v = atoi(e);
            if (v >= 1 && v < ds.lane_blocks_per_sm) ds.lane_blocks_per_sm = v;
        }
        // experiment knob: fewer resident blocks per SM (occupancy studies)
        if (const char* e = getenv("SLOSIM_BLOCKS_PER_SM")) {
            int v = atoi(e);
            if (v >= 1 && v < ds.blocks_per_sm) ds.blocks_per_sm = v;
        }
    }
    int64_t warps_needed = n_instances;
    int64_t blocks = (warps_needed + 3) / 4;
    int64_t full = (int64_t)ds.sms * ds.blocks_per_sm;
    *grid = (int)std::max<int64_t>(1, std::min<int64_t>(blocks, full));
    return SLOSIM_OK;
}

}  // namespace

// ------------------------------------------------------------------ engine --
extern "C" int64_t slosim_workspace_bytes(const slosim_batch_t* b) {
    if (!b || b->n_instances < 0) return -1;
    int dev = 0, grid = 0;
    if (current_device(&dev) != SLOSIM_OK) return -1;
    if (launch_geometry(dev_state(dev), dev, b->n_instances, &grid) != SLOSIM_OK) return -1;
    return (int64_t)grid * 4 * (int64_t)ws_bytes(b->max_requests) +
           (int64_t)b->n_profiles * 2 * (int64_t)sizeof(LutMem);
}

extern "C" int slosim_run_batch(const slosim_batch_t* b, void* stream) {
    if (!b || b->n_instances < 0 || b->n_profiles < 1 || !b->profiles || !b->instances || !b->summaries ||
        b->traces.n_total < 0)
        return SLOSIM_EINVAL;
    if (b->n_instances == 0) return SLOSIM_OK;
    if (b->traces.n_total > 0 && (!b->traces.arrival_us || !b->traces.input_len || !b->traces.output_len ||
                                  !b->traces.prefix_hit_len || !b->traces.id_rank))
        return SLOSIM_EINVAL;
    if ((b->flags & SLOSIM_F_ROWS) &&
        (!b->rows.ttft_us || !b->rows.mean_tpot_us || !b->rows.decode_tps || !b->rows.met_flags ||
         !b->rows.deadline_misses || !b->rows.t_prefill_finish || !b->rows.t_first_token ||
         !b->rows.t_last_token || !b->rows.first_sched_us))
        return SLOSIM_EINVAL;
    if ((b->flags & SLOSIM_F_EXPORT_LUT) && (!b->lut_out_sums || !b->lut_out_counts)) return SLOSIM_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    std::lock_guard<std::mutex> lock(g_mu);
    int dev = 0;
    int rc = current_device(&dev);
    if (rc) return rc;
    DevState& ds = dev_state(dev);
    if (!ds.done) CK(cudaEventCreateWithFlags(&ds.done, cudaEventDisableTiming));
    int64_t cap = b->max_requests;
    if (cap <= 0) {
        std::vector<slosim_instance_t> h((size_t)b->n_instances);
        CK(cudaMemcpyAsync(h.data(), b->instances, h.size() * sizeof(slosim_instance_t), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        for (auto& x : h) cap = std::max<int64_t>(cap, x.n_requests);
    }
    if (cap > INT32_MAX) return SLOSIM_EINVAL;
    int grid = 0;
    rc = launch_geometry(ds, dev, b->n_instances, &grid);
    if (rc) return rc;
    size_t stride = ws_bytes(cap);
    size_t total = stride * (size_t)grid * 4;
    CK(ds.ws.reserve(total, ds.done));
    CK(ds.tabs.reserve(sizeof(LutMem) * 2 * (size_t)b->n_profiles, ds.done));
    CK(ds.work.reserve(64, ds.done));
    // the previous launch on this device (any stream) owns the arenas until it completes
    CK(cudaStreamWaitEvent(st, ds.done, 0));
    LutMem* sched = (LutMem*)ds.tabs.ptr;
    LutMem* frozen = sched + b->n_profiles;
    build_profile_tables<<<b->n_profiles, 32, 0, st>>>(b->profiles, b->n_profiles, sched, frozen);
    CK(cudaGetLastError());
    CK(cudaMemsetAsync(ds.work.ptr, 0, 8, st));
    Ctx cx;
    cx.B = *b;
    cx.B.max_requests = cap;
    cx.sched_tab = sched;
    cx.frozen_tab = frozen;
    cx.dyn_n = nullptr;
    const bool force_lat = getenv("SLOSIM_FORCE_LATENCY_ENGINE") != nullptr;  // experiment knob
    const bool full = (b->flags & (SLOSIM_F_ROWS | SLOSIM_F_EXPORT_LUT)) || b->trace_buf;
    // Lane engine (tengine.cuh, one instance per thread) for throughput batches; the instances it
    // does not cover are appended to a deferred list that the warp engine then runs in the same stream.
    // One instance per thread pays off once the batch fills every lane slot of the GPU at least
    // once (sms x resident blocks x 128 lanes, 37,888 on a B200); smaller batches run faster as
    // one instance per warp.
    const int64_t lane_slots = (int64_t)ds.sms * ds.lane_blocks_per_sm * 128;
    const bool lane_path = !full && !force_lat && !getenv("SLOSIM_NO_LANE_ENGINE") &&
                           (b->n_instances >= lane_slots || getenv("SLOSIM_FORCE_LANE_ENGINE"));
    // experiment knob: lane engine with k live lanes per warp (k = 1: one instance per warp)
    int lpw = 32;
    if (const char* e = getenv("SLOSIM_LANE_LPW")) lpw = std::max(1, std::min(32, atoi(e)));
    const bool narrow = lpw < 32 && !full && !force_lat;
    if (lane_path || narrow) {
        const int64_t per_block = 4 * (int64_t)lpw;
        int64_t lblocks = std::min<int64_t>((b->n_instances + per_block - 1) / per_block,
                                            (int64_t)ds.sms * ds.lane_blocks_per_sm);
        size_t lstride = lane::lws_bytes(cap, LUT_CELLS);
        CK(ds.lws.reserve(lstride * (size_t)lblocks * 4, ds.done));
        CK(ds.defer.reserve(sizeof(int64_t) * (size_t)b->n_instances + 256, ds.done));
        unsigned long long* ctr = (unsigned long long*)ds.work.ptr;  // [0] lane work, [1] deferred count, [2] warp work
        CK(cudaMemsetAsync(ctr, 0, 24, st));
        lane::LCtx lc;
        lc.B = cx.B;
        lc.sched_tab = sched;
        lc.deferred = (int64_t*)ds.defer.ptr;
        lc.n_deferred = ctr + 1;
        lane::lane_kernel<<<(int)lblocks, 128, 0, st>>>(lc, (char*)ds.lws.ptr, cap, LUT_CELLS, ctr, lpw);
        CK(cudaGetLastError());
        cx.B.order = (const int64_t*)ds.defer.ptr;
        cx.dyn_n = ctr + 1;
        sim_kernel<<<grid, 128, 0, st>>>(cx, (char*)ds.ws.ptr, stride, cap, ctr + 2);
        CK(cudaGetLastError());
        CK(cudaEventRecord(ds.done, st));
        return SLOSIM_OK;
    }
    if ((b->n_instances <= (int64_t)ds.sms * 4 || force_lat) && !getenv("SLOSIM_NO_LATENCY_ENGINE")) {
        // at most one 4-warp block per SM: the spill-free latency build (engine_lat.cu)
        CK(slosim_launch_latency_engine(grid, &cx, (char*)ds.ws.ptr, stride, cap, (unsigned long long*)ds.work.ptr,
                                        st));
    } else {
        sim_kernel<<<grid, 128, 0, st>>>(cx, (char*)ds.ws.ptr, stride, cap, (unsigned long long*)ds.work.ptr);
        CK(cudaGetLastError());
    }
    CK(cudaEventRecord(ds.done, st));
    return SLOSIM_OK;
}

namespace {
// Device staging for the host-buffer entry point: one grow-only arena per
// device carved into 256-byte-aligned pieces (no cudaMalloc/cudaFree per call,
// so a call costs its copies and kernels only).
std::mutex g_io_mu;
struct Carve {
    char* base = nullptr;
    size_t off = 0;
    template <class T>
    T* take(size_t n) {
        if (n == 0) return nullptr;
        T* p = base ? (T*)(base + off) : nullptr;
        off += (n * sizeof(T) + 255) & ~(size_t)255;
        return p;
    }
};
template <class T>
cudaError_t up(T* d, const T* h, size_t n) {
    if (!d || !h || n == 0) return cudaSuccess;
    return cudaMemcpyAsync(d, h, n * sizeof(T), cudaMemcpyHostToDevice, 0);
}
}  // namespace

// Default processing order of the persistent work queue (same rule as
// batch.schedule_order): group by decode policy (slack-guided first), then by
// prefill policy, so each SM runs one specialised engine loop and prefill
// handler at a time; longest-first inside a group (cost = n_requests x
// arrival stretch factor).
static void default_order(const slosim_batch_t* hb, std::vector<int64_t>& order) {
    size_t n = (size_t)hb->n_instances;
    order.resize(n);
    std::vector<double> cost(n);
    for (size_t i = 0; i < n; i++) {
        order[i] = (int64_t)i;
        const slosim_instance_t& x = hb->instances[i];
        cost[i] = (double)x.n_requests * (x.rescale_factor > 0 ? x.rescale_factor : 1.0);
    }
    std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
        int da = hb->instances[a].decode_policy, db = hb->instances[b].decode_policy;
        if (da != db) return da > db;
        int pa = hb->instances[a].prefill_policy, pb = hb->instances[b].prefill_policy;
        if (pa != pb) return pa > pb;
        return cost[a] > cost[b];
    });
}

extern "C" int slosim_run_batch_host(const slosim_batch_t* hb, float* elapsed_ms) {
    if (!hb) return SLOSIM_EINVAL;
    std::lock_guard<std::mutex> lock(g_io_mu);
    int dev = 0;
    if (int rc0 = current_device(&dev)) return rc0;
    Arena& io = dev_state(dev).io;
    slosim_batch_t d = *hb;
    size_t nt = (size_t)hb->traces.n_total, ni = (size_t)hb->n_instances;
    int64_t rows_n = 0, tb_n = 0;
    for (size_t i = 0; i < ni; i++) {
        const slosim_instance_t& x = hb->instances[i];
        rows_n = std::max<int64_t>(rows_n, x.row_offset + x.n_requests);
        if (x.trace_buf_offset >= 0) tb_n = std::max<int64_t>(tb_n, x.trace_buf_offset + x.trace_buf_words);
        d.max_requests = std::max<int64_t>(d.max_requests, x.n_requests);
    }
    const bool rows = (hb->flags & SLOSIM_F_ROWS) != 0;
    const size_t rn = rows ? (size_t)rows_n : 0;
    const size_t tbn = hb->trace_buf ? (size_t)tb_n : 0;
    const size_t FR = SLOSIM_MAX_BSZ_BUCKETS * SLOSIM_MAX_SEQ_BUCKETS;
    const bool lut = (hb->flags & SLOSIM_F_EXPORT_LUT) && hb->lut_out_sums;
    std::vector<int64_t> order;
    if (hb->order) order.assign(hb->order, hb->order + ni);
    else default_order(hb, order);
    // pass 0 sizes the arena, pass 1 carves it
    for (int pass = 0; pass < 2; pass++) {
        Carve c;
        if (pass == 1) {
            CK(io.reserve(0));
            c.base = (char*)io.ptr;
        }
        d.traces.arrival_us = c.take<int64_t>(nt);
        d.traces.input_len = c.take<int32_t>(nt);
        d.traces.output_len = c.take<int32_t>(nt);
        d.traces.prefix_hit_len = c.take<int32_t>(nt);
        d.traces.id_rank = c.take<int32_t>(nt);
        d.profiles = c.take<slosim_profile_t>((size_t)hb->n_profiles);
        d.instances = c.take<slosim_instance_t>(ni);
        d.summaries = c.take<slosim_summary_t>(ni);
        d.rows.ttft_us = c.take<int64_t>(rn);
        d.rows.mean_tpot_us = c.take<double>(rn);
        d.rows.decode_tps = c.take<double>(rn);
        d.rows.met_flags = c.take<uint8_t>(rn);
        d.rows.deadline_misses = c.take<int32_t>(rn);
        d.rows.t_prefill_finish = c.take<int64_t>(rn);
        d.rows.t_first_token = c.take<int64_t>(rn);
        d.rows.t_last_token = c.take<int64_t>(rn);
        d.rows.first_sched_us = c.take<int64_t>(rn);
        d.trace_buf = c.take<int64_t>(tbn);
        d.lut_out_sums = c.take<double>(lut ? ni * FR : 0);
        d.lut_out_counts = c.take<int32_t>(lut ? ni * FR : 0);
        d.order = c.take<int64_t>(ni);
        if (pass == 0) CK(io.reserve(c.off));
    }
    CK(up((int64_t*)d.traces.arrival_us, hb->traces.arrival_us, nt));
    CK(up((int32_t*)d.traces.input_len, hb->traces.input_len, nt));
    CK(up((int32_t*)d.traces.output_len, hb->traces.output_len, nt));
    CK(up((int32_t*)d.traces.prefix_hit_len, hb->traces.prefix_hit_len, nt));
    CK(up((int32_t*)d.traces.id_rank, hb->traces.id_rank, nt));
    CK(up((slosim_profile_t*)d.profiles, hb->profiles, (size_t)hb->n_profiles));
    CK(up((slosim_instance_t*)d.instances, hb->instances, ni));
    CK(up((int64_t*)d.order, order.data(), ni));
    if (!hb->trace_buf) d.trace_buf = nullptr;
    struct Events {  // destroyed on every return path
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        ~Events() {
            if (e0) cudaEventDestroy(e0);
            if (e1) cudaEventDestroy(e1);
        }
    } ev;
    CK(cudaEventCreate(&ev.e0));
    CK(cudaEventCreate(&ev.e1));
    CK(cudaEventRecord(ev.e0, 0));
    int rc = slosim_run_batch(&d, nullptr);
    CK(cudaEventRecord(ev.e1, 0));
    if (rc) {
        cudaEventSynchronize(ev.e1);
        return rc;
    }
    CK(cudaMemcpyAsync(hb->summaries, d.summaries, ni * sizeof(slosim_summary_t), cudaMemcpyDeviceToHost, 0));
    if (rows) {
        const slosim_rows_t& R = hb->rows;
#define COPYROW(f, T) \
    if (R.f) CK(cudaMemcpyAsync(R.f, d.rows.f, rn * sizeof(T), cudaMemcpyDeviceToHost, 0))
        COPYROW(ttft_us, int64_t); COPYROW(mean_tpot_us, double); COPYROW(decode_tps, double);
        COPYROW(met_flags, uint8_t); COPYROW(deadline_misses, int32_t); COPYROW(t_prefill_finish, int64_t);
        COPYROW(t_first_token, int64_t); COPYROW(t_last_token, int64_t); COPYROW(first_sched_us, int64_t);
#undef COPYROW
    }
    if (tbn) CK(cudaMemcpyAsync(hb->trace_buf, d.trace_buf, tbn * sizeof(int64_t), cudaMemcpyDeviceToHost, 0));
    if (lut) {
        CK(cudaMemcpyAsync(hb->lut_out_sums, d.lut_out_sums, ni * FR * sizeof(double), cudaMemcpyDeviceToHost, 0));
        CK(cudaMemcpyAsync(hb->lut_out_counts, d.lut_out_counts, ni * FR * sizeof(int32_t), cudaMemcpyDeviceToHost, 0));
    }
    CK(cudaStreamSynchronize(0));
    if (elapsed_ms) cudaEventElapsedTime(elapsed_ms, ev.e0, ev.e1);
    return SLOSIM_OK;
}

// ------------------------------------------------------- snapshot kernels --
namespace {

struct SnapLut {
    int nb, ns;
    int32_t bb[SLOSIM_MAX_BSZ_BUCKETS];
    int32_t sb[SLOSIM_MAX_SEQ_BUCKETS];
};

__global__ void k_lut_lookup(SnapLut sl, const double* fsums, const int32_t* fcounts, LutMem* tab, int64_t n,
                             const int64_t* bsz, const int64_t* seq, double* out) {
    if (threadIdx.x < 32) lut_build(tab, sl.nb, sl.ns, sl.bb, sl.sb, fsums, fcounts, threadIdx.x);
    __syncthreads();
    for (int64_t k = threadIdx.x; k < n; k += blockDim.x) out[k] = lut_lookup(tab, bsz[k], seq[k]);
}

__global__ void k_formula(int nbase, const int64_t* bx, const double* by, double gamma, int64_t n, const int64_t* bsz,
                          const int64_t* seq, double* out) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) out[k] = decode_formula(nbase, bx, by, gamma, bsz[k], seq[k]);
}

__global__ void k_estimate(int64_t tok, int64_t busy, int64_t n, const int64_t* tokens, int64_t* out) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) out[k] = ceil_muldiv(tokens[k], busy, tok);
}

__global__ void k_predict(int n, const int64_t* arr, const int64_t* rem, int64_t t_now, int64_t tok, int64_t busy,
                          int64_t* out) {
    int lane = threadIdx.x;
    int64_t cursor = t_now;
    for (int base = 0; base < n; base += 32) {
        int k = base + lane;
        bool v = k < n;
        int64_t a = v ? arr[k] : 0;
        int64_t d = v ? ceil_muldiv(rem[k], busy, tok) : 0;
        int nvalid = n - base < 32 ? n - base : 32;
        int64_t fin = fcfs_walk_chunk(v, a, d, cursor, nvalid, lane);
        if (v) out[k] = fin;
    }
}

// Sort snapshot entries by (arrival, id_rank) into a queue workspace (one warp).
__device__ void snap_queue(int n, const int64_t* arr, const int32_t* inp, const int64_t* rem, const int32_t* idr,
                           const WS& w, int lane) {
    for (int i0 = 0; i0 < n; i0 += 32) {
        int i = i0 + lane;
        int rank = 0;
        if (i < n) {
            for (int j = 0; j < n; j++) {
                bool less = arr[j] < arr[i] || (arr[j] == arr[i] && idr[j] < idr[i]);
                rank += less;
            }
            w.i32(Q_POS)[rank] = i;
            w.i64(Q_ARR)[rank] = arr[i];
            w.i32(Q_INP)[rank] = inp[i];
            w.i32(Q_REM)[rank] = (int32_t)rem[i];
            w.i32(Q_FULL)[rank] = (int32_t)rem[i];
        }
    }
    __syncwarp();
}

__global__ void k_select_prefill(int policy, int n, const int64_t* arr, const int32_t* inp, const int64_t* rem,
                                 const int32_t* idr, int64_t budget, int64_t t_now, int64_t tok, int64_t busy,
                                 int64_t ttft, char* wsb, int64_t cap, int32_t* out_index, int64_t* out_take,
                                 int32_t* n_out, double* out_scores) {
    int lane = threadIdx.x;
    WS w = make_ws(wsb, cap);
    snap_queue(n, arr, inp, rem, idr, w, lane);
    int k = prefill_select(policy, w, 0, n, budget, t_now, tok, busy, ttft, lane);
    const int32_t* q_pos = w.i32(Q_POS);
    for (int e = lane; e < k; e += 32) { out_index[e] = q_pos[w.i32(PF_QIDX)[e]]; out_take[e] = w.i32(PF_TAKE)[e]; }
    if (policy == SLOSIM_PREFILL_KAIROS_URGENCY && out_scores)
        for (int q = lane; q < n; q += 32) out_scores[q_pos[q]] = w.f64(Q_SCORE)[q];
    if (lane == 0) *n_out = k;
}

__global__ void k_select_decode(int policy, int n, const int64_t* seq, const int32_t* idr, const int64_t* ngen,
                                const double* tfirst, double t_now, int64_t tpot, SnapLut sl, const double* fsums,
                                const int32_t* fcounts, LutMem* tab, char* wsb, int64_t cap, int32_t* out_batch,
                                int32_t* n_batch, int32_t* out_delayed, int32_t* n_delayed, double* out_times,
                                double* out_pred, double* out_smin, int32_t* out_fb) {
    int lane = threadIdx.x;
    lut_build(tab, sl.nb, sl.ns, sl.bb, sl.sb, fsums, fcounts, lane);
    const LutMem* L = tab;
    WS w = make_ws(wsb, cap);
    int32_t* a_seq = w.i32(A_SEQ);
    int32_t* a_idr = w.i32(A_IDR);
    int32_t* a_flag = w.i32(A_FLAG);
    int32_t* a_ord = w.i32(A_ORD);
    int64_t mx = 0;
    for (int i = lane; i < n; i += 32) {
        a_seq[i] = (int32_t)seq[i];
        a_idr[i] = idr[i];
        a_flag[i] = 0;
        mx = seq[i] > mx ? seq[i] : mx;
    }
    mx = wmax64(mx);
    __syncwarp();
    decode_order(n, a_seq, a_idr, a_ord, lane);
    double fallback = lut_lookup(L, n, mx);
    if (policy == SLOSIM_DECODE_CONTINUOUS) {
        for (int r = lane; r < n; r += 32) out_batch[r] = a_ord[r];
        if (lane == 0) {
            *n_batch = n; *n_delayed = 0; *out_pred = fallback;
            *out_smin = __longlong_as_double(0x7ff0000000000000LL);
            *out_fb = 0;
        }
        return;
    }
    // compute_slack with the full-batch step cost (decode_sched.py:36-57, :75-79), f64 times
    double smin = __longlong_as_double(0x7ff0000000000000LL);
    for (int i = lane; i < n; i += 32) {
        double sl2 = xsub(xsub((double)(tpot * (ngen[i] + 1)), xsub(t_now, tfirst[i])), fallback);
        smin = sl2 < smin ? sl2 : smin;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) { double x = __shfl_xor_sync(FULLMASK, smin, o); smin = x < smin ? x : smin; }
    double tcur;
    int64_t ms;
    int nd = 0;
    int b = decode_scan(L, n, a_ord, a_seq, a_flag, smin, &tcur, &ms, out_batch, out_delayed, out_times, &nd, lane);
    __syncwarp();
    if (b == 0) {
        for (int r = lane; r < n; r += 32) out_batch[r] = a_ord[r];
        if (lane == 0) { *n_batch = n; *n_delayed = 0; *out_pred = fallback; *out_smin = smin; *out_fb = 1; }
    } else if (lane == 0) {
        *n_batch = b; *n_delayed = nd; *out_pred = tcur; *out_smin = smin; *out_fb = 0;
    }
}

__global__ void k_prefill_gt(int nc, const int64_t* cx, const int64_t* cy, int k, const int64_t* done,
                             const int64_t* take, int64_t* out) {
    __shared__ int64_t sx[SLOSIM_MAX_CURVE_POINTS], sy[SLOSIM_MAX_CURVE_POINTS];
    if (threadIdx.x < nc) { sx[threadIdx.x] = cx[threadIdx.x]; sy[threadIdx.x] = cy[threadIdx.x]; }
    __syncthreads();
    if (threadIdx.x != 0) return;
    double total = 0.0;
    for (int e = 0; e < k; e++)
        total = xadd(total, xsub(curve_at(nc, sx, sy, done[e] + take[e]), curve_at(nc, sx, sy, done[e])));
    int64_t d = rint_i64(total);
    *out = d < 1 ? 1 : d;
}

__global__ void k_request_metrics(int64_t n, const double* arr, const int64_t* outl, const int64_t* off,
                                  const double* ts, int64_t ttft_slo, int64_t tpot_slo, double* ttft, double* tpot,
                                  double* tps, uint8_t* flags, int32_t* misses) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const double* tk = ts + off[k];
    int64_t m = off[k + 1] - off[k];
    double tf = tk[0];
    // ttft_metric metrics.py:30-35
    double v = xsub(tf, arr[k]);
    bool tm = v <= (double)ttft_slo;
    double tp = 0.0, tr = __longlong_as_double(0x7ff8000000000000LL);
    bool pm = true;
    if (outl[k] != 1) {
        // tpot_metric :38-46, decode_throughput :49-54
        double span = xsub(tk[m - 1], tf);
        tp = xdiv(span, (double)(outl[k] - 1));
        pm = tp <= (double)tpot_slo;
        tr = xdiv((double)(outl[k] - 1), xdiv(span, 1e6));
    }
    // deadline_misses :57-69: token j due at t_first + j * tpot
    int32_t mi = 0;
    for (int64_t j = 1; j < m; j++) mi += tk[j] > xadd(tf, (double)(j * tpot_slo));
    ttft[k] = v; tpot[k] = tp; tps[k] = tr;
    flags[k] = (uint8_t)((tm ? 1 : 0) | (pm ? 2 : 0) | ((tm && pm) ? 4 : 0));
    misses[k] = mi;
}

__global__ void k_aggregate(int64_t n, const uint8_t* flags, const double* tps, double* scratch, double* agg) {
    int lane = threadIdx.x;
    int64_t c0 = 0, c1 = 0, c2 = 0;
    int cnt = 0;
    for (int64_t base = 0; base < n; base += 32) {
        int64_t k = base + lane;
        bool v = k < n;
        uint8_t f = v ? flags[k] : 0;
        c0 += f & 1; c1 += (f >> 1) & 1; c2 += (f >> 2) & 1;
        bool has = v && tps[k] == tps[k];
        unsigned m = __ballot_sync(FULLMASK, has);
        if (has) scratch[cnt + __popc(m & ((1u << lane) - 1u))] = tps[k];
        cnt += __popc(m);
    }
    c0 = wsum64(c0); c1 = wsum64(c1); c2 = wsum64(c2);
    __syncwarp();
    double p50 = __longlong_as_double(0x7ff8000000000000LL), p90 = p50;
    if (cnt > 0) {
        int64_t r50 = (int64_t)ceil(xmul(50 / 100.0, (double)cnt));
        int64_t r90 = (int64_t)ceil(xmul(90 / 100.0, (double)cnt));
        p50 = radix_select(scratch, cnt, r50 < 1 ? 1 : r50, lane);
        p90 = radix_select(scratch, cnt, r90 < 1 ? 1 : r90, lane);
    }
    if (lane == 0) {
        agg[0] = idiv(c0, n); agg[1] = idiv(c1, n); agg[2] = idiv(c2, n); agg[3] = p50; agg[4] = p90;
    }
}

__global__ void k_synth(slosim_profile_t* P, int na, const int64_t* ab, const int64_t* as, const double* aus,
                        double gamma, int64_t w) {
    __shared__ int64_t bx[SLOSIM_MAX_BASE_POINTS];
    __shared__ double by[SLOSIM_MAX_BASE_POINTS];
    __shared__ int nbase;
    if (threadIdx.x == 0) {
        // base = sorted((seq, float(us)) for bsz == 1)  (costmodel.py:290)
        int m = 0;
        for (int k = 0; k < na; k++) {
            if (ab[k] != 1) continue;
            int b = m++;
            while (b > 0 && (bx[b - 1] > as[k] || (bx[b - 1] == as[k] && by[b - 1] > aus[k]))) {
                bx[b] = bx[b - 1]; by[b] = by[b - 1]; b--;
            }
            bx[b] = as[k]; by[b] = aus[k];
        }
        nbase = m;
    }
    __syncthreads();
    const int FR = SLOSIM_MAX_BSZ_BUCKETS * SLOSIM_MAX_SEQ_BUCKETS;
    for (int c = threadIdx.x; c < FR; c += blockDim.x) {
        int i = c / SLOSIM_MAX_SEQ_BUCKETS, j = c % SLOSIM_MAX_SEQ_BUCKETS;
        double s = 0.0;
        int32_t n = 0;
        if (i < P->nb && j < P->ns && w != 0) {
            // round(decode_step_formula(...)) then max(1, .) (costmodel.py:301-304)
            int64_t v = rint_i64(decode_formula(nbase, bx, by, gamma, P->bsz_buckets[i], P->seq_buckets[j]));
            if (v < 1) v = 1;
            s = (double)(v * w);
            n = (int32_t)w;
        }
        P->lut_sums[c] = s;
        P->lut_counts[c] = n;
    }
    __syncthreads();
    if (threadIdx.x == 0 && w != 0) {
        // anchors pinned in order (costmodel.py:305-308)
        for (int k = 0; k < na; k++) {
            int i = bucket_index(P->bsz_buckets, P->nb, ab[k]), j = bucket_index(P->seq_buckets, P->ns, as[k]);
            P->lut_sums[i * SLOSIM_MAX_SEQ_BUCKETS + j] = xmul(aus[k], (double)w);
            P->lut_counts[i * SLOSIM_MAX_SEQ_BUCKETS + j] = (int32_t)w;
        }
    }
}

// Snapshot scratch: carve typed buffers from one grow-only allocation.
struct Bump {
    char* base;
    size_t off = 0;
    template <class T>
    T* take(size_t n) {
        T* p = (T*)(base + off);
        off += (n * sizeof(T) + 255) & ~(size_t)255;
        return p;
    }
};

// Snapshot scratch of the current device (snapshot calls are synchronous).
char* g_snap_ptr = nullptr;
cudaError_t snap_reserve(size_t bytes) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
    Arena& a = g_dev[dev].snap;
    e = a.reserve(bytes);
    g_snap_ptr = (char*)a.ptr;
    return e;
}

SnapLut make_snaplut(int32_t nb, const int32_t* bb, int32_t ns, const int32_t* sb) {
    SnapLut s{};
    s.nb = nb; s.ns = ns;
    for (int i = 0; i < nb; i++) s.bb[i] = bb[i];
    for (int j = 0; j < ns; j++) s.sb[j] = sb[j];
    return s;
}

void frame(int32_t nb, int32_t ns, const double* sums, const int32_t* counts, std::vector<double>& fs,
           std::vector<int32_t>& fc) {
    const size_t FR = SLOSIM_MAX_BSZ_BUCKETS * SLOSIM_MAX_SEQ_BUCKETS;
    fs.assign(FR, 0.0);
    fc.assign(FR, 0);
    for (int i = 0; i < nb; i++)
        for (int j = 0; j < ns; j++) {
            fs[i * SLOSIM_MAX_SEQ_BUCKETS + j] = sums[i * ns + j];
            fc[i * SLOSIM_MAX_SEQ_BUCKETS + j] = counts[i * ns + j];
        }
}

bool lut_dims_ok(int32_t nb, int32_t ns) {
    return nb >= 1 && nb <= SLOSIM_MAX_BSZ_BUCKETS && ns >= 1 && ns <= SLOSIM_MAX_SEQ_BUCKETS;
}

}  // namespace

#define H2D(dst, src, n) CK(cudaMemcpy(dst, src, (n) * sizeof(*(src)), cudaMemcpyHostToDevice))
#define D2H(dst, src, n) CK(cudaMemcpy(dst, src, (n) * sizeof(*(dst)), cudaMemcpyDeviceToHost))

extern "C" int slosim_lut_lookup(int32_t nb, const int32_t* bb, int32_t ns, const int32_t* sb, const double* sums,
                                 const int32_t* counts, int64_t n, const int64_t* bsz, const int64_t* seq,
                                 double* out) {
    if (!lut_dims_ok(nb, ns) || n < 0) return SLOSIM_EINVAL;
    bool any = false;
    for (int c = 0; c < nb * ns; c++) any |= counts[c] > 0;
    if (!any) return SLOSIM_ECONFIG;
    for (int64_t k = 0; k < n; k++) if (bsz[k] < 1 || seq[k] < 1) return SLOSIM_EINVAL;
    if (n == 0) return SLOSIM_OK;
    std::lock_guard<std::mutex> lock(g_mu);
    std::vector<double> fs;
    std::vector<int32_t> fc;
    frame(nb, ns, sums, counts, fs, fc);
    CK(snap_reserve(sizeof(LutMem) + fs.size() * 12 + (size_t)n * 24 + 4096));
    Bump bp{g_snap_ptr};
    LutMem* tab = bp.take<LutMem>(1);
    double* dfs = bp.take<double>(fs.size());
    int32_t* dfc = bp.take<int32_t>(fc.size());
    int64_t* db = bp.take<int64_t>(n);
    int64_t* dsq = bp.take<int64_t>(n);
    double* dout = bp.take<double>(n);
    H2D(dfs, fs.data(), fs.size()); H2D(dfc, fc.data(), fc.size()); H2D(db, bsz, n); H2D(dsq, seq, n);
    k_lut_lookup<<<1, 256>>>(make_snaplut(nb, bb, ns, sb), dfs, dfc, tab, n, db, dsq, dout);
    CK(cudaGetLastError());
    D2H(out, dout, n);
    return SLOSIM_OK;
}

extern "C" int slosim_decode_formula(int32_t n_base, const int64_t* bx, const double* by, double gamma, int64_t n,
                                     const int64_t* bsz, const int64_t* seq, double* out) {
    if (n_base < 1 || n_base > SLOSIM_MAX_BASE_POINTS || n < 0) return SLOSIM_EINVAL;
    if (n == 0) return SLOSIM_OK;
    std::lock_guard<std::mutex> lock(g_mu);
    CK(snap_reserve((size_t)n * 24 + 4096));
    Bump bp{g_snap_ptr};
    int64_t* dbx = bp.take<int64_t>(n_base);
    double* dby = bp.take<double>(n_base);
    int64_t* db = bp.take<int64_t>(n);
    int64_t* dsq = bp.take<int64_t>(n);
    double* dout = bp.take<double>(n);
    H2D(dbx, bx, n_base); H2D(dby, by, n_base); H2D(db, bsz, n); H2D(dsq, seq, n);
    k_formula<<<(unsigned)((n + 255) / 256), 256>>>(n_base, dbx, dby, gamma, n, db, dsq, dout);
    CK(cudaGetLastError());
    D2H(out, dout, n);
    return SLOSIM_OK;
}

extern "C" int slosim_estimate_duration(int64_t total_tokens, int64_t total_busy_us, int64_t n,
                                        const int64_t* tokens, int64_t* out) {
    if (total_busy_us <= 0 || total_tokens <= 0) return SLOSIM_ECONFIG;
    for (int64_t k = 0; k < n; k++) if (tokens[k] < 0) return SLOSIM_EINVAL;
    if (n == 0) return SLOSIM_OK;
    std::lock_guard<std::mutex> lock(g_mu);
    CK(snap_reserve((size_t)n * 16 + 4096));
    Bump bp{g_snap_ptr};
    int64_t* dt = bp.take<int64_t>(n);
    int64_t* dout = bp.take<int64_t>(n);
    H2D(dt, tokens, n);
    k_estimate<<<(unsigned)((n + 255) / 256), 256>>>(total_tokens, total_busy_us, n, dt, dout);
    CK(cudaGetLastError());
    D2H(out, dout, n);
    return SLOSIM_OK;
}

extern "C" int slosim_predict_finish(int32_t n, const int64_t* arrival, const int64_t* remaining, int64_t t_now,
                                     int64_t est_tokens, int64_t est_busy, int64_t* out_finish) {
    if (n < 0) return SLOSIM_EINVAL;
    if (est_busy <= 0 || est_tokens <= 0) return SLOSIM_ECONFIG;
    if (n == 0) return SLOSIM_OK;
    std::lock_guard<std::mutex> lock(g_mu);
    CK(snap_reserve((size_t)n * 24 + 4096));
    Bump bp{g_snap_ptr};
    int64_t* da = bp.take<int64_t>(n);
    int64_t* dr = bp.take<int64_t>(n);
    int64_t* dout = bp.take<int64_t>(n);
    H2D(da, arrival, n); H2D(dr, remaining, n);
    k_predict<<<1, 32>>>(n, da, dr, t_now, est_tokens, est_busy, dout);
    CK(cudaGetLastError());
    D2H(out_finish, dout, n);
    return SLOSIM_OK;
}

extern "C" int slosim_select_prefill(int32_t policy, int32_t n, const int64_t* arrival, const int32_t* input_len,
                                     const int64_t* remaining, const int32_t* id_rank, int64_t budget, int64_t t_now,
                                     int64_t est_tokens, int64_t est_busy, int64_t ttft_slo_us, int32_t* out_index,
                                     int64_t* out_take, int32_t* n_out, double* out_scores) {
    if (budget < 1 || n < 0 || policy < 0 || policy > 2) return SLOSIM_EINVAL;
    if (policy == SLOSIM_PREFILL_KAIROS_URGENCY && n > 0 && (est_busy <= 0 || est_tokens <= 0)) return SLOSIM_ECONFIG;
    if (n == 0) { *n_out = 0; return SLOSIM_OK; }
    std::lock_guard<std::mutex> lock(g_mu);
    size_t wsb = ws_bytes(n);
    CK(snap_reserve(wsb + (size_t)n * 64 + 8192));
    Bump bp{g_snap_ptr};
    char* dws = bp.take<char>(wsb);
    int64_t* da = bp.take<int64_t>(n);
    int32_t* di = bp.take<int32_t>(n);
    int64_t* dr = bp.take<int64_t>(n);
    int32_t* dk = bp.take<int32_t>(n);
    int32_t* doi = bp.take<int32_t>(n);
    int64_t* dot = bp.take<int64_t>(n);
    int32_t* dno = bp.take<int32_t>(1);
    double* dsc = bp.take<double>(n);
    H2D(da, arrival, n); H2D(di, input_len, n); H2D(dr, remaining, n); H2D(dk, id_rank, n);
    k_select_prefill<<<1, 32>>>(policy, n, da, di, dr, dk, budget, t_now, est_tokens, est_busy, ttft_slo_us, dws, n,
                                doi, dot, dno, dsc);
    CK(cudaGetLastError());
    D2H(n_out, dno, 1);
    D2H(out_index, doi, *n_out);
    D2H(out_take, dot, *n_out);
    if (out_scores && policy == SLOSIM_PREFILL_KAIROS_URGENCY) D2H(out_scores, dsc, n);
    return SLOSIM_OK;
}

extern "C" int slosim_select_decode(int32_t policy, int32_t n, const int64_t* seq_len, const int32_t* id_rank,
                                    const int64_t* n_gen, const double* t_first, double t_now, int64_t tpot_slo_us,
                                    int32_t nb, const int32_t* bb, int32_t ns, const int32_t* sb, const double* sums,
                                    const int32_t* counts, int32_t* out_batch, int32_t* n_batch, int32_t* out_delayed,
                                    int32_t* n_delayed, double* out_admit_times, double* out_pred, double* out_smin,
                                    int32_t* out_fallback) {
    if (n < 1 || policy < 0 || policy > 1 || !lut_dims_ok(nb, ns)) return SLOSIM_EINVAL;
    bool any = false;
    for (int c = 0; c < nb * ns; c++) any |= counts[c] > 0;
    if (!any) return SLOSIM_ECONFIG;
    std::lock_guard<std::mutex> lock(g_mu);
    std::vector<double> fs;
    std::vector<int32_t> fc;
    frame(nb, ns, sums, counts, fs, fc);
    size_t wsb = ws_bytes(n);
    CK(snap_reserve(wsb + sizeof(LutMem) + fs.size() * 12 + (size_t)n * 64 + 8192));
    Bump bp{g_snap_ptr};
    char* dws = bp.take<char>(wsb);
    LutMem* tab = bp.take<LutMem>(1);
    double* dfs = bp.take<double>(fs.size());
    int32_t* dfc = bp.take<int32_t>(fc.size());
    int64_t* dseq = bp.take<int64_t>(n);
    int32_t* didr = bp.take<int32_t>(n);
    int64_t* dng = bp.take<int64_t>(n);
    double* dtf = bp.take<double>(n);
    int32_t* db = bp.take<int32_t>(n);
    int32_t* dd = bp.take<int32_t>(n);
    double* dt = bp.take<double>(n);
    int32_t* dnb = bp.take<int32_t>(4);
    double* dsc = bp.take<double>(2);
    H2D(dfs, fs.data(), fs.size()); H2D(dfc, fc.data(), fc.size());
    H2D(dseq, seq_len, n); H2D(didr, id_rank, n); H2D(dng, n_gen, n); H2D(dtf, t_first, n);
    k_select_decode<<<1, 32>>>(policy, n, dseq, didr, dng, dtf, t_now, tpot_slo_us, make_snaplut(nb, bb, ns, sb), dfs,
                               dfc, tab, dws, n, db, dnb, dd, dnb + 1, dt, dsc, dsc + 1, dnb + 2);
    CK(cudaGetLastError());
    int32_t hn[4];
    D2H(hn, dnb, 3);
    double hs[2];
    D2H(hs, dsc, 2);
    *n_batch = hn[0]; *n_delayed = hn[1]; *out_fallback = hn[2]; *out_pred = hs[0]; *out_smin = hs[1];
    D2H(out_batch, db, hn[0]);
    if (hn[1]) D2H(out_delayed, dd, hn[1]);
    if (out_admit_times && !hn[2] && policy == SLOSIM_DECODE_KAIROS_SLACK) D2H(out_admit_times, dt, hn[0]);
    return SLOSIM_OK;
}

extern "C" int slosim_prefill_batch_us(int32_t n_curve, const int64_t* cx, const int64_t* cy, int32_t k,
                                       const int64_t* done_before, const int64_t* take, int64_t* out_us) {
    if (n_curve < 2 || n_curve > SLOSIM_MAX_CURVE_POINTS || k < 0) return SLOSIM_EINVAL;
    std::lock_guard<std::mutex> lock(g_mu);
    CK(snap_reserve((size_t)(k + 1) * 16 + 8192));
    Bump bp{g_snap_ptr};
    int64_t* dx = bp.take<int64_t>(n_curve);
    int64_t* dy = bp.take<int64_t>(n_curve);
    int64_t* dd = bp.take<int64_t>(k + 1);
    int64_t* dt = bp.take<int64_t>(k + 1);
    int64_t* dout = bp.take<int64_t>(1);
    H2D(dx, cx, n_curve); H2D(dy, cy, n_curve);
    if (k) { H2D(dd, done_before, k); H2D(dt, take, k); }
    k_prefill_gt<<<1, 32>>>(n_curve, dx, dy, k, dd, dt, dout);
    CK(cudaGetLastError());
    D2H(out_us, dout, 1);
    return SLOSIM_OK;
}

extern "C" int slosim_request_metrics(int64_t n, const double* arrival, const int64_t* output_len,
                                      const int64_t* ts_offsets, const double* ts, int64_t ttft_slo_us,
                                      int64_t tpot_slo_us, double* ttft_us, double* mean_tpot, double* tps,
                                      uint8_t* met_flags, int32_t* misses, double* agg) {
    if (n < 0) return SLOSIM_EINVAL;
    if (n == 0) {
        if (agg) { agg[0] = agg[1] = agg[2] = 1.0; agg[3] = agg[4] = NAN; }
        return SLOSIM_OK;
    }
    int64_t nts = ts_offsets[n];
    for (int64_t k = 0; k < n; k++) if (ts_offsets[k + 1] - ts_offsets[k] < 1) return SLOSIM_EINVAL;
    std::lock_guard<std::mutex> lock(g_mu);
    CK(snap_reserve((size_t)n * 80 + (size_t)nts * 8 + 8192));
    Bump bp{g_snap_ptr};
    double* da = bp.take<double>(n);
    int64_t* dol = bp.take<int64_t>(n);
    int64_t* doff = bp.take<int64_t>(n + 1);
    double* dts = bp.take<double>(nts);
    double* dtt = bp.take<double>(n);
    double* dtp = bp.take<double>(n);
    double* dtr = bp.take<double>(n);
    uint8_t* dfl = bp.take<uint8_t>(n);
    int32_t* dmi = bp.take<int32_t>(n);
    double* dscr = bp.take<double>(n);
    double* dagg = bp.take<double>(5);
    H2D(da, arrival, n); H2D(dol, output_len, n); H2D(doff, ts_offsets, n + 1); H2D(dts, ts, nts);
    k_request_metrics<<<(unsigned)((n + 127) / 128), 128>>>(n, da, dol, doff, dts, ttft_slo_us, tpot_slo_us, dtt, dtp,
                                                            dtr, dfl, dmi);
    CK(cudaGetLastError());
    k_aggregate<<<1, 32>>>(n, dfl, dtr, dscr, dagg);
    CK(cudaGetLastError());
    if (ttft_us) D2H(ttft_us, dtt, n);
    if (mean_tpot) D2H(mean_tpot, dtp, n);
    if (tps) D2H(tps, dtr, n);
    if (met_flags) D2H(met_flags, dfl, n);
    if (misses) D2H(misses, dmi, n);
    if (agg) D2H(agg, dagg, 5);
    return SLOSIM_OK;
}

extern "C" int slosim_synth_profile(slosim_profile_t* profile, int32_t n_anchors, const int64_t* anchor_bsz,
                                    const int64_t* anchor_seq, const double* anchor_us, double batch_growth,
                                    int64_t prior_weight) {
    if (!profile || !lut_dims_ok(profile->nb, profile->ns) || n_anchors < 1 || batch_growth < 0 || prior_weight < 0)
        return SLOSIM_EINVAL;
    int nbase = 0;
    for (int k = 0; k < n_anchors; k++) nbase += anchor_bsz[k] == 1;
    if (nbase == 0 || nbase > SLOSIM_MAX_BASE_POINTS) return SLOSIM_EINVAL;
    std::lock_guard<std::mutex> lock(g_mu);
    CK(snap_reserve(sizeof(slosim_profile_t) + (size_t)n_anchors * 24 + 8192));
    Bump bp{g_snap_ptr};
    slosim_profile_t* dp = bp.take<slosim_profile_t>(1);
    int64_t* dab = bp.take<int64_t>(n_anchors);
    int64_t* das = bp.take<int64_t>(n_anchors);
    double* dau = bp.take<double>(n_anchors);
    H2D(dp, profile, 1); H2D(dab, anchor_bsz, n_anchors); H2D(das, anchor_seq, n_anchors);
    H2D(dau, anchor_us, n_anchors);
    k_synth<<<1, 256>>>(dp, n_anchors, dab, das, dau, batch_growth, prior_weight);
    CK(cudaGetLastError());
    D2H(profile, dp, 1);
    return SLOSIM_OK;
}

// K6 (pre-collective): per-cell histograms of e2e-met counts, accumulated on the device.
__global__ void k_histogram(int64_t n, const slosim_summary_t* s, const int32_t* cell, int32_t n_bins,
                            unsigned long long* hist) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n || cell[k] < 0) return;
    int b = s[k].e2e_met;
    b = b < 0 ? 0 : (b >= n_bins ? n_bins - 1 : b);
    atomicAdd(hist + (int64_t)cell[k] * n_bins + b, 1ULL);
}

extern "C" int slosim_histogram(int64_t n, const slosim_summary_t* d_summaries, const int32_t* d_cell,
                                int32_t n_bins, int64_t* d_hist, void* stream) {
    if (n < 0 || n_bins < 1) return SLOSIM_EINVAL;
    if (n == 0) return SLOSIM_OK;
    k_histogram<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(n, d_summaries, d_cell, n_bins,
                                                                              (unsigned long long*)d_hist);
    CK(cudaGetLastError());
    return SLOSIM_OK;
}

extern "C" int slosim_abi_version(void) { return SLOSIM_ABI_VERSION; }

extern "C" int slosim_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

extern "C" const char* slosim_build_info(void) {
    return "slosim_b200 abi=2 arch=sm_100a fmad=false";
}

extern "C" const char* slosim_last_error(void) { return g_err; }

// For the other translation units (longtail.cu): record a CUDA error for slosim_last_error.
int slosim_internal_fail(int code, const char* what, cudaError_t e) {
    fail_cuda(e, what);
    return code;
}

// ---------------------------------------------------------------- exchange --
namespace {
// NCCL entry points resolved at run time (no link-time dependency; an already
// loaded libnccl.so.2, e.g. PyTorch's, is reused).  Enum values per nccl.h.
typedef int (*nccl_allreduce_fn)(const void*, void*, size_t, int, int, void*, cudaStream_t);
typedef int (*nccl_allgather_fn)(const void*, void*, size_t, int, void*, cudaStream_t);
typedef const char* (*nccl_errstr_fn)(int);
constexpr int kNcclUint8 = 1, kNcclInt64 = 4, kNcclSum = 0;
struct Nccl {
    nccl_allreduce_fn all_reduce = nullptr;
    nccl_allgather_fn all_gather = nullptr;
    nccl_errstr_fn err = nullptr;
    bool tried = false;
};
Nccl& nccl() {
    static Nccl n;
    std::lock_guard<std::mutex> lock(g_mu);
    if (!n.tried) {
        n.tried = true;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
        if (h) {
            n.all_reduce = (nccl_allreduce_fn)dlsym(h, "ncclAllReduce");
            n.all_gather = (nccl_allgather_fn)dlsym(h, "ncclAllGather");
            n.err = (nccl_errstr_fn)dlsym(h, "ncclGetErrorString");
        }
    }
    return n;
}
}  // namespace

extern "C" int slosim_exchange(void* nccl_comm, const slosim_summary_t* d_mine, int64_t n_mine, slosim_summary_t* d_all,
                               int64_t* d_hist, int64_t n_hist, void* stream) {
    if (!nccl_comm || n_mine < 0 || n_hist < 0 || (n_mine && (!d_mine || !d_all)) || (n_hist && !d_hist))
        return SLOSIM_EINVAL;
    Nccl& n = nccl();
    if (!n.all_reduce || !n.all_gather) {
        snprintf(g_err, sizeof(g_err), "slosim_exchange: libnccl.so.2 not loadable");
        return SLOSIM_ECUDA;
    }
    cudaStream_t st = (cudaStream_t)stream;
    int r = 0;
    if (n_hist) r = n.all_reduce(d_hist, d_hist, (size_t)n_hist, kNcclInt64, kNcclSum, nccl_comm, st);
    if (!r && n_mine)
        r = n.all_gather(d_mine, d_all, (size_t)n_mine * sizeof(slosim_summary_t), kNcclUint8, nccl_comm, st);
    if (r) {
        snprintf(g_err, sizeof(g_err), "slosim_exchange: NCCL error %d (%s)", r, n.err ? n.err(r) : "?");
        return SLOSIM_ECUDA;
    }
    return SLOSIM_OK;
}

#ifdef SLOSIM_PROF
cudaError_t slosim_lat_prof_read(unsigned long long* out16, int reset);
// Debug builds only: read (and optionally reset) the section-profile counters of both engine builds.
extern "C" int slosim_prof_read(unsigned long long* out16, int reset) {
    unsigned long long lat[16];
    CK(cudaMemcpyFromSymbol(out16, slosim::g_prof, 16 * sizeof(unsigned long long)));
    CK(slosim_lat_prof_read(lat, reset));
    for (int k = 0; k < 16; k++) out16[k] += lat[k];
    if (reset) {
        unsigned long long z[16] = {0};
        CK(cudaMemcpyToSymbol(slosim::g_prof, z, sizeof(z)));
    }
    return 0;
}
#endif
