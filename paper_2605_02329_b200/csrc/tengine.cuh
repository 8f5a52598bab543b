// tengine.cuh — the lane engine: one simulated instance per THREAD.
//
// The warp engine (engine.cuh) gives each instance a whole warp; with 3-4
// requests active on average (config 5) most lanes idle while the warp walks
// a long chain of shuffles and reductions per decode step, and the kernel is
// bound by instruction issue and fetch.  Here every lane runs its own
// instance of the same event loop (engine.py:261-302) with its scalar state in
// registers and its request sets in a per-warp workspace, so one warp
// instruction advances up to 32 instances.  The loop is flattened: each trip is
// one instant of the lane's instance, and a lane whose instance has finished
// writes its summary and pulls the next instance from the work queue in the
// same trip, so the warp stays full until the queue drains.
//
// Work whose size is the prefill queue (the urgency scores of every queued
// request, the policy's packing) would serialise a warp behind one lane, so a
// prefill step starts warp-cooperatively: every lane that needs one is served
// in turn by all 32 lanes through the warp engine's prefill_select
// (warpops.cuh) on that lane's queue.
//
// Workspace (per warp):
//   active set, lane-interleaved (element k of lane l at [k * 32 + l]): the
//     decode loops walk it from the start in lockstep, one line per load;
//   LUT cells, lane-interleaved;
//   per lane, contiguous: the prefill queue, prefill batch, pending-admission
//     and transfer lists and tps values, in the warp engine's workspace layout
//     (warpops.cuh WS), so prefill_select runs on one lane's queue unchanged.
//
// Scope: instances whose profile has the power-of-two LUT geometry (the
// reference defaults, costmodel.py:26-27), a fully populated LUT, the plain
// ground-truth decode formula (no frozen file LUT, no noise), in batches
// without per-request rows, event trace or LUT export.  capi.cu routes other
// batches to the warp engine, and the lane kernel defers other instances to
// it.  Decisions, counters and digests are identical to the warp engine's and
// the oracle's.
//
// Reference mapping: same as engine.cuh (engine.py:198-413, prefill_sched.py,
// decode_sched.py:60-124, costmodel.py:118-187, metrics.py:30-144).
#pragma once
#include "../../include/slosim_b200.h"
#include "lut.cuh"
#include "warpops.cuh"

#if defined(SLOSIM_LANE_NO_PREFETCH) && !defined(SLOSIM_LANE_NO_VBASE)
#define SLOSIM_LANE_NO_VBASE  // the slack base is kept by the software-pipelined member loop only
#endif

namespace slosim {
namespace lane {

constexpr int WL = 32;

#ifndef LANE_HOOK_DECODE  // test harness hook (tools/lane_host): called at every decode step start
#define LANE_HOOK_DECODE(S, w)
#endif

// Element k of a lane's array: lane-interleaved (stride 32) or contiguous (stride 1).
template <class T, int STRIDE>
struct Arr {
    T* p;  // element 0 of this lane
    __device__ __forceinline__ T& operator[](int k) const { return p[(size_t)k * STRIDE]; }
};

// Active set (interleaved), capacity `cap` requests: entry k of lane l is the 16-byte element
// [k * 32 + l] of each of two vector arrays, V0 = {seq, flag, id_rank, pos} and
// V1 = {input, output, misses, -}, plus t_first in an i64 array, so the member loop moves an
// entry with three loads.  A_FLAG bit 0: member of the running Alg. 3 batch; bit 1: TTFT met.
enum A32 { A_SEQ, A_FLAG, A_IDR, A_POS, A_INP, A_OUT, A_MISS, N_A32 };  // V0.x..w, V1.x..z
enum A64 { A_TF, N_A64 };
constexpr int A_VEC_BYTES = 2 * 16 + 8;  // per entry and lane

__host__ __device__ inline size_t lws_lane_bytes(size_t c) {
    return N_WS_I32 * ws_align(4 * c) + N_WS_I64 * ws_align(8 * c);
}
__host__ __device__ inline size_t lws_bytes(int64_t cap, int cells) {
    size_t c = (size_t)(cap > 0 ? cap : 1);
    return (size_t)WL * (c * A_VEC_BYTES + (size_t)cells * (8 + 8 + 4) + lws_lane_bytes(c));
}

// One warp's workspace: [active set, interleaved][LUT, interleaved][32 per-lane WS regions].
struct LWs {
    char* wb;  // warp base
    size_t c;
    int cells, lane;
    __device__ __forceinline__ int4* v0() const { return (int4*)wb + lane; }
    __device__ __forceinline__ int4* v1() const { return (int4*)(wb + (size_t)WL * 16 * c) + lane; }
    // one field of the vector arrays (stride 4 ints per entry slot)
    __device__ __forceinline__ Arr<int32_t, WL * 4> a32(int k) const {
        return Arr<int32_t, WL * 4>{(int32_t*)(k < 4 ? v0() : v1()) + (k & 3)};
    }
    __device__ __forceinline__ Arr<int64_t, WL> a64(int k) const {
        return Arr<int64_t, WL>{(int64_t*)(wb + (size_t)WL * 32 * c + (size_t)k * WL * 8 * c) + lane};
    }
    __device__ __forceinline__ char* lut_base() const { return wb + (size_t)WL * c * A_VEC_BYTES; }
    __device__ __forceinline__ Arr<double, WL> mean() const { return Arr<double, WL>{(double*)lut_base() + lane}; }
    __device__ __forceinline__ Arr<double, WL> sum() const {
        return Arr<double, WL>{(double*)(lut_base() + (size_t)WL * 8 * cells) + lane};
    }
    __device__ __forceinline__ Arr<int32_t, WL> cnt() const {
        return Arr<int32_t, WL>{(int32_t*)(lut_base() + (size_t)WL * 16 * cells) + lane};
    }
    __device__ __forceinline__ WS ws() const {
        char* b = lut_base() + (size_t)WL * 20 * cells + (size_t)lane * lws_lane_bytes(c);
        return WS{b, (uint32_t)ws_align(4 * c), (uint32_t)ws_align(8 * c)};
    }
    __device__ __forceinline__ Arr<int32_t, 1> r32(int k) const { return Arr<int32_t, 1>{ws().i32(k)}; }
    __device__ __forceinline__ Arr<int64_t, 1> r64(int k) const { return Arr<int64_t, 1>{ws().i64(k)}; }
    __device__ __forceinline__ Arr<double, 1> r64f(int k) const { return Arr<double, 1>{ws().f64(k)}; }
    __device__ __forceinline__ LWs for_lane(int l) const { return LWs{wb, c, cells, l}; }
};

// Python-form row interpolation on the power-of-two grid (lut.cuh lut_eval<true> / geval_p):
// value of row r at column selection (c, dx) from the stored means; the np.interp slope of a
// populated column pair is (m[c+1] - m[c]) * 2^-wsh, exactly as stored by lut_build / gupdate.
// Scaling by a power of two is exact, so slope * dx = RN((m[c+1] - m[c]) * (dx * 2^-wsh)) with
// dx * 2^-wsh exact: one rounding, one multiply (dxw below); likewise the weight across rows,
// (bsz - 2^lo) * 2^-lo, is formed exactly and applied with one multiply.
struct LGeo { int nb, ns, wsh; double inv_w; };

__device__ __forceinline__ double lrow(const Arr<double, WL>& M, const LGeo& g, int r, int c, double dxw) {
    const int k = r * g.ns + c;
    const double m0 = M[k];
    if (dxw == 0.0) return m0;
    return xadd(xmul(xsub(M[k + 1], m0), dxw), m0);
}

// DecodeStepLUT.lookup (costmodel.py:157-187) on the full power-of-two grid.
__device__ __forceinline__ double llookup(const Arr<double, WL>& M, const LGeo& g, int bsz, int seq) {
    // column selection (lut_col<true>)
    const int w = 1 << g.wsh;
    int c = (seq >> g.wsh) - 1;
    const bool in = seq > w && c < g.ns - 1;
    c = in ? c : (seq <= w ? 0 : g.ns - 1);
    const double dxw = in ? (double)(seq & (w - 1)) * g.inv_w : 0.0;
    // row selection (lut_rows_nb<true>)
    const int i = gbidx(bsz);
    const bool single = (i == 0) | (i >= g.nb) | ((1u << i) == (unsigned)bsz);
    const int lo = i >= g.nb ? g.nb - 1 : (i == 0 ? 0 : i - 1);
    const int r1 = single ? (i >= g.nb ? g.nb - 1 : i) : lo;
    const double v1 = lrow(M, g, r1, c, dxw);
    if (single) return v1;
    const double v2 = lrow(M, g, i, c, dxw);
    return xadd(v1, xmul(xsub(v2, v1), (double)(bsz - (1 << lo)) * pow2_neg(lo)));
}

// llookup with a one-entry memo: within one Alg. 3 scan the LUT is fixed, and consecutive candidates
// often share the (|B|+1, column) key (sequences below the first bucket edge all select column 0).
struct LMemo { int bsz, c; double dx, v; };
__device__ __forceinline__ double llookup_memo(const Arr<double, WL>& M, const LGeo& g, int bsz, int seq, LMemo& mm) {
    const int w = 1 << g.wsh;
    int c = (seq >> g.wsh) - 1;
    const bool in = seq > w && c < g.ns - 1;
    c = in ? c : (seq <= w ? 0 : g.ns - 1);
    const double dx = in ? (double)(seq & (w - 1)) * g.inv_w : 0.0;
    if (bsz == mm.bsz && c == mm.c && dx == mm.dx) return mm.v;
    const int i = gbidx(bsz);
    const bool single = (i == 0) | (i >= g.nb) | ((1u << i) == (unsigned)bsz);
    const int lo = i >= g.nb ? g.nb - 1 : (i == 0 ? 0 : i - 1);
    const int r1 = single ? (i >= g.nb ? g.nb - 1 : i) : lo;
    double v = lrow(M, g, r1, c, dx);
    if (!single) {
        const double v2 = lrow(M, g, i, c, dx);
        v = xadd(v, xmul(xsub(v2, v), (double)(bsz - (1 << lo)) * pow2_neg(lo)));
    }
    mm = LMemo{bsz, c, dx, v};
    return v;
}

// RN(a/x) > RN(b/y) (decode_sched.py:87-89), see numerics.cuh quot_gt.
__device__ __noinline__ bool lquot_exact(double a, double x, double b, double y) { return __ddiv_rn(a, x) > __ddiv_rn(b, y); }
__device__ __forceinline__ bool lquot_gt(double a, double x, double b, double y) {
    const double p = __dmul_rn(a, y), q = __dmul_rn(b, x);
    if (p > __dmul_rn(q, 1.0 + 0x1p-50)) return true;
    if (p < __dmul_rn(q, 1.0 - 0x1p-50)) return false;
    return lquot_exact(a, x, b, y);
}

// Nearest-rank selection (metrics.py:87-92): the r-th smallest (1-based) of a[lo..hi) by quickselect
// (positive doubles; ties are equal values, so any partition order gives the same value).
__device__ __noinline__ double lselect(const Arr<double, 1>& a, int lo, int hi, int r) {
    int k = lo + r - 1;
    while (hi - lo > 1) {
        const double piv = a[lo + ((hi - lo) >> 1)];
        int i = lo, j = hi - 1;
        while (i <= j) {
            while (a[i] < piv) i++;
            while (a[j] > piv) j--;
            if (i <= j) { double x = a[i]; a[i] = a[j]; a[j] = x; i++; j--; }
        }
        if (k <= j) hi = j + 1;
        else if (k >= i) lo = i;
        else return a[k];
    }
    return a[k];
}

struct LCtx {
    slosim_batch_t B;
    const LutMem* sched_tab;
    int64_t* deferred;                 // instances this engine does not cover (run by the warp engine after)
    unsigned long long* n_deferred;
};

// Instances outside the lane engine's scope (see the header comment) go to the warp engine.
__device__ __forceinline__ bool lane_eligible(const LCtx& cx, int64_t ii) {
    const int pid = cx.B.instances[ii].profile_id;
    if (pid < 0 || pid >= cx.B.n_profiles) return true;  // invalid: linit reports EINVAL
    const LutMem* T = cx.sched_tab + pid;
    const slosim_profile_t* P = cx.B.profiles + pid;
    return T->bad || (T->geo && T->full && P->gt_frozen == 0 && !(P->noise_eps > 0.0));
}

// Per-lane instance state (registers; never address-taken).
struct St {
    int64_t ii;
    int64_t off;  // trace offset
    const slosim_profile_t* P;
    int64_t ttft_slo, tpot_slo;
    int n;
    int8_t ppol, dpol;
    bool use_lut, gline;
    LGeo g;
    GtLine gl;
    // event state
    int ai, qh, qt, pf_k, ph, pt, trn, an;
    int64_t next_arr, pf_end, pf_dur, tr_min, dc_end, dc_dur, amax, kv, est_tok, est_busy;
    int dc_bsz, dc_max;
    int dc_prefix;  // continuous batching: the running batch is active entries [0, dc_prefix)
                    // (admissions append); Alg. 3: -1, members carry A_FLAG bit 0
    int32_t c_ttft, c_tpot, c_e2e, ntps, max_q, max_a, finished;
    int64_t misses, worst_wait, psteps, dsteps, v_dec, b_dec, v_pre, t_end;
    uint64_t D;
#ifndef SLOSIM_LANE_NO_VBASE
    // Alg. 3 slack base: min over the active set of tpot*(n_gen+1) + t_first, so that the slack
    // minimum at time t (decode_sched.py:36-57, 89-90) is vbase - t - fallback; kept by the
    // member loop, admission and retirement instead of a pass over the active set per step
    int64_t vbase;
#endif
};

// Rarely used per-instance parameters are read from the descriptor (not kept in registers).
__device__ __forceinline__ const slosim_instance_t& linst(const LCtx& cx, const St& S) { return cx.B.instances[S.ii]; }

__device__ __forceinline__ int64_t larrival(const LCtx& cx, const St& S, int p) {
    const int64_t a = cx.B.traces.arrival_us[S.off + p];
    const double fac = linst(cx, S).rescale_factor;
    return fac > 0 ? rint_i64(xmul((double)a, fac)) : a;
}

__device__ __forceinline__ bool linstance_ok(const slosim_batch_t* B, const slosim_instance_t* I, const LutMem* tabs) {
    const int64_t n = I->n_requests, off = I->trace_offset;
    bool ok = n >= 0 && n <= B->max_requests && I->profile_id >= 0 && I->profile_id < B->n_profiles && off >= 0 &&
              off <= B->traces.n_total - n && I->prefill_policy >= 0 && I->prefill_policy <= 2 &&
              I->decode_policy >= 0 && I->decode_policy <= 1 && I->chunk_budget >= 1 && I->ttft_slo_us > 0 &&
              I->tpot_slo_us > 0 && I->kv_capacity_tokens >= 1 && I->transfer_base_us >= 0 &&
              I->transfer_per_token_us >= 0.0 && !(I->rescale_factor != I->rescale_factor);
    if (ok) ok = tabs[I->profile_id].bad == 0;
    return ok;
}

__device__ void lwrite_status(slosim_summary_t* out, int n, int status) {
    slosim_summary_t s = {};
    s.status = status;
    s.n = n;
    s.tps_p50 = __longlong_as_double(0x7ff8000000000000LL);
    s.tps_p90 = s.tps_p50;
    *out = s;
}

// Start instance ii on this lane (Simulation.__init__ engine.py:198-246).  Returns false when the
// instance finished immediately (invalid or unrunnable: its summary is written).
__device__ __forceinline__ bool linit(St& S, const LCtx& cx, const LWs& w, int64_t ii) {
    const slosim_batch_t* B = &cx.B;
    const slosim_instance_t* I = B->instances + ii;
    S.ii = ii;
    S.n = I->n_requests;
    if (!linstance_ok(B, I, cx.sched_tab)) {
        lwrite_status(B->summaries + ii, S.n, SLOSIM_EINVAL);
        return false;
    }
    const int pid = I->profile_id;
    S.P = B->profiles + pid;
    S.off = I->trace_offset;
    S.ttft_slo = I->ttft_slo_us;
    S.tpot_slo = I->tpot_slo_us;
    S.ppol = I->prefill_policy;
    S.dpol = I->decode_policy;
    const LutMem* ST = cx.sched_tab + pid;
    // KV reservation check (engine.py:227-232)
    const int32_t* Tinp = B->traces.input_len + S.off;
    const int32_t* Tout = B->traces.output_len + S.off;
    int64_t worst = 0;
    for (int p = 0; p < S.n; p++) {
        const int64_t need = (int64_t)Tinp[p] + Tout[p];
        worst = need > worst ? need : worst;
    }
    if (worst > I->kv_capacity_tokens || ST->rowmask == 0) {
        lwrite_status(B->summaries + ii, S.n, SLOSIM_ECONFIG);
        return false;
    }
    S.use_lut = S.dpol == SLOSIM_DECODE_KAIROS_SLACK || (B->flags & SLOSIM_F_ALWAYS_LUT);
    S.g = LGeo{ST->nb, ST->ns, ST->wsh, pow2_neg(ST->wsh)};
    if (S.use_lut) {
        const auto M = w.mean(), Su = w.sum();
        const auto C = w.cnt();
        const int K = ST->nb * ST->ns;
        for (int k = 0; k < K; k++) { M[k] = ST->mean[k]; Su[k] = ST->sum[k]; C[k] = ST->cnt[k]; }
    }
    S.gline = gt_line_make(S.P->n_base, S.P->base_x, S.P->base_y, S.P->gamma, S.gl);
    S.est_tok = S.P->est_tokens;
    S.est_busy = S.P->est_busy_us;
    S.ai = S.qh = S.qt = S.pf_k = S.ph = S.pt = S.trn = S.an = 0;
    S.next_arr = S.n > 0 ? larrival(cx, S, 0) : SLOSIM_INF64;
    S.pf_end = S.tr_min = S.dc_end = SLOSIM_INF64;
    S.pf_dur = S.dc_dur = S.amax = S.kv = 0;
    S.dc_bsz = S.dc_max = 0;
    S.dc_prefix = 0;
    S.c_ttft = S.c_tpot = S.c_e2e = S.ntps = S.max_q = S.max_a = S.finished = 0;
    S.misses = S.worst_wait = S.psteps = S.dsteps = S.v_dec = S.b_dec = S.v_pre = S.t_end = 0;
    S.D = 0;
#ifndef SLOSIM_LANE_NO_VBASE
    S.vbase = SLOSIM_INF64;
#endif
    return true;
}

// metrics aggregate (metrics.py:109-144) + summary row.
__device__ __forceinline__ void lfinalize(const St& S, const LCtx& cx, const LWs& w) {
    double p50 = __longlong_as_double(0x7ff8000000000000LL), p90 = p50;
    if (S.ntps > 0) {
        const auto T = w.r64f(TPS);
        int64_t r50 = (int64_t)ceil(xmul(50 / 100.0, (double)S.ntps));
        int64_t r90 = (int64_t)ceil(xmul(90 / 100.0, (double)S.ntps));
        r50 = r50 < 1 ? 1 : r50;
        r90 = r90 < 1 ? 1 : r90;
        // after selecting rank r50, a[r50..] holds the values >= it: select r90 there
        p50 = lselect(T, 0, S.ntps, (int)r50);
        p90 = r90 == r50 ? p50 : lselect(T, (int)r50, S.ntps, (int)(r90 - r50));
    }
    slosim_summary_t s;
    s.status = S.finished == S.n ? SLOSIM_OK : -1;
    s.n = S.n;
    s.ttft_met = S.c_ttft; s.tpot_met = S.c_tpot; s.e2e_met = S.c_e2e; s.n_tps = S.ntps;
    s.tps_p50 = p50; s.tps_p90 = p90;
    s.worst_queue_wait_us = S.worst_wait;
    s.prefill_steps = S.psteps; s.decode_steps = S.dsteps;
    s.digest = S.D;
    s.v_dec = S.v_dec; s.b_dec = S.b_dec; s.v_pre = S.v_pre;
    s.deadline_misses = S.misses;
    s.t_end_us = S.t_end;
    s.est_tokens = S.est_tok; s.est_busy_us = S.est_busy;
    s.max_queue = S.max_q; s.max_active = S.max_a;
    s.sim_cycles = 0;
    cx.B.summaries[S.ii] = s;
}

// Pending list insert keeping (tpf, id_rank) order (engine.py:358).
__device__ __forceinline__ void lpending_insert(St& S, const LWs& w, int64_t tpf, int32_t idr, int64_t ttr, int32_t pos) {
    const auto PT = w.r64(PD_TPF), PR = w.r64(PD_TTR);
    const auto PP = w.r32(PD_POS), PI = w.r32(PD_IDR);
    int k = S.pt;
    while (k > S.ph && (PT[k - 1] > tpf || (PT[k - 1] == tpf && PI[k - 1] > idr))) {
        PT[k] = PT[k - 1]; PR[k] = PR[k - 1]; PP[k] = PP[k - 1]; PI[k] = PI[k - 1];
        k--;
    }
    PT[k] = tpf; PR[k] = ttr; PP[k] = pos; PI[k] = idr;
    S.pt++;
}

// ---- rare events (arrivals, transfers, prefill completion) at instant t (engine.py:286-350)
__device__ __forceinline__ void lrare(St& S, const LCtx& cx, const LWs& w, int64_t t) {
    const int32_t* Tinp = cx.B.traces.input_len + S.off;
    const int32_t* Tidr = cx.B.traces.id_rank + S.off;
    if (S.next_arr == t) {  // arrivals (engine.py:288-291): a contiguous run of the trace
        const int32_t* Thit = cx.B.traces.prefix_hit_len + S.off;
        const auto QP = w.r32(Q_POS), QR = w.r32(Q_REM), QF = w.r32(Q_FULL), QI = w.r32(Q_INP);
        const auto QA = w.r64(Q_ARR);
        int64_t a = t;
        while (a == t) {
            const int p = S.ai;
            const int32_t inp = Tinp[p], full = inp - Thit[p];
            QP[S.qt] = p; QA[S.qt] = t; QI[S.qt] = inp; QF[S.qt] = full; QR[S.qt] = full;
            S.qt++;
            S.ai++;
            a = S.ai < S.n ? larrival(cx, S, S.ai) : SLOSIM_INF64;
        }
        S.next_arr = a;
    }
    if (S.tr_min == t) {  // transfers pushed at earlier instants (engine.py:294-298)
        const auto TT = w.r64(TR_T), TF = w.r64(TR_TPF);
        const auto TP = w.r32(TR_POS);
        int m = 0;
        int64_t mn = SLOSIM_INF64;
        for (int k = 0; k < S.trn; k++) {
            const int64_t tt = TT[k], tpf = TF[k];
            const int32_t pos = TP[k];
            if (tt == t) {
                lpending_insert(S, w, tpf, Tidr[pos], t, pos);
            } else {
                TT[m] = tt; TF[m] = tpf; TP[m] = pos; m++;
                mn = tt < mn ? tt : mn;
            }
        }
        S.trn = m;
        S.tr_min = mn;
    }
    if (S.pf_end == t) {  // prefill step completion (engine.py:327-350)
        const auto QP = w.r32(Q_POS), QR = w.r32(Q_REM), QF = w.r32(Q_FULL), QI = w.r32(Q_INP);
        const auto QA = w.r64(Q_ARR);
        const auto FQ = w.r32(PF_QIDX), FT = w.r32(PF_TAKE);
        int64_t tot = 0;
        uint64_t h = dstep(S.D, (uint64_t)t ^ 0xA5A5A5A5A5A5A5A5ULL);
        int ncomp = 0;
        for (int e = 0; e < S.pf_k; e++) {
            const int qi = FQ[e];
            const int32_t take = FT[e];
            const int32_t rem = QR[qi] - take;
            QR[qi] = rem;
            const int32_t pos = QP[qi];
            tot += take;
            h = dstep(h, ((uint64_t)(uint32_t)pos << 32) | (uint32_t)take);
            if (rem == 0) {  // completed: leaves the queue, KV transfer in batch order
                ncomp++;
                const slosim_instance_t& I = linst(cx, S);
                const int64_t delay = I.transfer_base_us + rint_i64(xmul((double)QI[qi], I.transfer_per_token_us));
                if (delay == 0) {
                    lpending_insert(S, w, t, Tidr[pos], t, pos);
                } else {
                    const auto TT = w.r64(TR_T), TF = w.r64(TR_TPF);
                    TT[S.trn] = t + delay; TF[S.trn] = t; w.r32(TR_POS)[S.trn] = pos;
                    S.trn++;
                    S.tr_min = t + delay < S.tr_min ? t + delay : S.tr_min;
                }
            }
        }
        S.est_tok += tot;
        S.est_busy += S.pf_dur;
        S.psteps++;
        S.D = dstep(h, (uint64_t)S.pf_dur);
        if (S.ppol == SLOSIM_PREFILL_FCFS) {
            S.qh += ncomp;  // FCFS completes a prefix of the queue
        } else if (ncomp) {
            int o = S.qh;
            for (int qi = S.qh; qi < S.qt; qi++) {
                const int32_t rem = QR[qi];
                if (rem > 0) {
                    if (o != qi) { QP[o] = QP[qi]; QR[o] = rem; QF[o] = QF[qi]; QI[o] = QI[qi]; QA[o] = QA[qi]; }
                    o++;
                }
            }
            S.qt = o;
        }
        S.pf_end = SLOSIM_INF64;
    }
}

// ---- admission under the KV reservation (engine.py:355-375)
__device__ __forceinline__ void ladmit(St& S, const LCtx& cx, const LWs& w) {
    const int32_t* Tinp = cx.B.traces.input_len + S.off;
    const int32_t* Tout = cx.B.traces.output_len + S.off;
    const auto PR = w.r64(PD_TTR);
    const auto PP = w.r32(PD_POS), PI = w.r32(PD_IDR);
    const auto AT = w.a64(A_TF);
    const int64_t kv_cap = linst(cx, S).kv_capacity_tokens;
    while (S.pt > S.ph) {
        const int32_t pos = PP[S.ph];
        const int32_t outl = Tout[pos], inp = Tinp[pos];
        const int64_t need = (int64_t)inp + outl;
        if (S.kv + need > kv_cap) break;  // head-of-line blocking
        const int64_t ttr = PR[S.ph];
        const int32_t idr = PI[S.ph];
        S.ph++;
        const bool ttm = ttr - larrival(cx, S, pos) <= S.ttft_slo;
        S.c_ttft += ttm;
        if (outl == 1) {  // finishes at its first token, holds no KV
            S.c_tpot++;
            S.c_e2e += ttm;
            S.finished++;
            continue;
        }
        S.kv += need;
        // kairos: keep the active set in (seq_len, id) order (decode_sched.py:74)
        int k = S.an;
        if (S.dpol == SLOSIM_DECODE_KAIROS_SLACK) {
            // shift the entries that sort after the new one up by one (three loads and stores per
            // entry); entry k-2 is loaded while entry k-1 is stored at k
            int4* V0 = w.v0();
            int4* V1 = w.v1();
            if (k > 0) {
                int4 a_ = V0[(k - 1) * WL], b_ = V1[(k - 1) * WL];
                int64_t t_ = AT[k - 1];
                while (k > 0 && (a_.x > inp || (a_.x == inp && a_.z > idr))) {
                    int4 a2 = make_int4(0, 0, 0, 0), b2 = make_int4(0, 0, 0, 0);
                    int64_t t2 = 0;
                    if (k > 1) { a2 = V0[(k - 2) * WL]; b2 = V1[(k - 2) * WL]; t2 = AT[k - 2]; }
                    V0[k * WL] = a_; V1[k * WL] = b_; AT[k] = t_;
                    a_ = a2; b_ = b2; t_ = t2;
                    k--;
                }
            }
        }
        w.v0()[k * WL] = make_int4(inp, ttm ? 2 : 0, idr, pos);
        w.v1()[k * WL] = make_int4(inp, outl, 0, 0);
        AT[k] = ttr;
#ifndef SLOSIM_LANE_NO_VBASE
        S.vbase = min(S.vbase, ttr + S.tpot_slo);
#endif
        S.an++;
        S.amax = inp > S.amax ? inp : S.amax;
    }
}

// ---- start a prefill step on this lane alone (engine.py:307-325, prefill_sched.py:93-145); the
// host test harness uses it, the kernel starts prefill steps cooperatively (coop_prefill_start).
__device__ __forceinline__ void lprefill_start(St& S, const LCtx& cx, const LWs& w, int64_t t) {
    const auto QR = w.r32(Q_REM), QF = w.r32(Q_FULL), QI = w.r32(Q_INP);
    const auto QA = w.r64(Q_ARR);
    const auto QK = w.r64f(Q_SCORE);
    const auto FQ = w.r32(PF_QIDX), FT = w.r32(PF_TAKE);
    const int qlen = S.qt - S.qh;
    S.v_pre += qlen;
    S.max_q = qlen > S.max_q ? qlen : S.max_q;
    int k = 0;
    int64_t left = linst(cx, S).chunk_budget;
    if (S.ppol == SLOSIM_PREFILL_FCFS) {
        for (int qi = S.qh; qi < S.qt && left > 0; qi++) {
            const int64_t rem = QR[qi];
            const int64_t take = rem < left ? rem : left;
            FQ[k] = qi; FT[k] = (int32_t)take; k++;
            left -= take;
        }
    } else {
        if (S.ppol == SLOSIM_PREFILL_KAIROS_URGENCY) {
            // predict_finish_times (prefill_sched.py:39-56) + _selection_score (:82-90), FCFS order
            int64_t cursor = t;
            for (int qi = S.qh; qi < S.qt; qi++) {
                const int64_t a = QA[qi];
                cursor = (cursor > a ? cursor : a) + ceil_muldiv(QR[qi], S.est_busy, S.est_tok);
                QK[qi] = selection_score(S.ttft_slo, cursor, a, QI[qi]);
            }
        }
        // repeated arg-best strictly after the previous pick:
        //   sjf (remaining, arrival, id) -> (rem, qi); kairos (-score, arrival, id) -> (~dkey(score), qi)
        uint64_t pk = 0;
        int pq = -1;
        const bool sjf = S.ppol == SLOSIM_PREFILL_SJF;
        while (left > 0) {
            uint64_t bk = ~0ULL;
            int bq = -1;
            for (int qi = S.qh; qi < S.qt; qi++) {
                const uint64_t key = sjf ? (uint64_t)(uint32_t)QR[qi] : ~dkey(QK[qi]);
                const bool after = key > pk || (key == pk && qi > pq);
                if (after && (key < bk || (key == bk && qi < bq) || bq < 0)) { bk = key; bq = qi; }
            }
            if (bq < 0) break;
            const int64_t rem = QR[bq];
            const int64_t take = rem < left ? rem : left;
            FQ[k] = bq; FT[k] = (int32_t)take; k++;
            left -= take;
            pk = bk;
            pq = bq;
        }
    }
    S.pf_k = k;
    // ground-truth duration: ordered sum of curve increments (engine.py:175-183)
    const slosim_profile_t* P = S.P;
    double total = 0.0;
    int64_t ww = 0;
    for (int e = 0; e < k; e++) {
        const int qi = FQ[e];
        const int64_t take = FT[e];
        const int64_t done = (int64_t)QF[qi] - QR[qi];
        total = xadd(total, xsub(curve_at(P->n_curve, P->curve_x, P->curve_y, done + take),
                                 curve_at(P->n_curve, P->curve_x, P->curve_y, done)));
        if (done == 0) {  // first time scheduled (engine.py:322)
            const int64_t wt = t - QA[qi];
            ww = wt > ww ? wt : ww;
        }
    }
    S.worst_wait = ww > S.worst_wait ? ww : S.worst_wait;
    const int64_t d = rint_i64(total);
    S.pf_dur = d < 1 ? 1 : d;
    S.pf_end = t + S.pf_dur;
}

// ---- start a prefill step warp-cooperatively on lane L's queue.  Every lane calls this with the
// same L and L's scalars (broadcast by the caller); it returns the step's entry count, duration and
// first-schedule wait, which lane L folds into its state.  The policies of prefill_sched.py run
// through prefill_select (warpops.cuh); the duration is the in-order ground-truth sum
// (engine.py:175-183).
struct PfOut { int k; int64_t dur, ww; };
__device__ __noinline__ PfOut coop_prefill_start(const WS& ws, int ppol, int qh, int qt, int64_t budget, int64_t t,
                                                  int64_t est_tok, int64_t est_busy, int64_t ttft_slo,
                                                  const slosim_profile_t* P, int lane) {
    const int k = prefill_select(ppol, ws, qh, qt, budget, t, est_tok, est_busy, ttft_slo, lane);
    const int32_t* pf_qidx = ws.i32(PF_QIDX);
    const int32_t* pf_take = ws.i32(PF_TAKE);
    const int32_t* q_full = ws.i32(Q_FULL);
    const int32_t* q_rem = ws.i32(Q_REM);
    const int64_t* q_arr = ws.i64(Q_ARR);
    const int n_curve = P->n_curve;
    double total = 0.0;
    int64_t ww = 0;
    for (int base = 0; base < k; base += 32) {
        const int e = base + lane;
        double term = 0.0;
        if (e < k) {
            const int qi = pf_qidx[e];
            const int64_t take = pf_take[e];
            const int64_t done = (int64_t)q_full[qi] - q_rem[qi];
            term = xsub(curve_at(n_curve, P->curve_x, P->curve_y, done + take),
                        curve_at(n_curve, P->curve_x, P->curve_y, done));
            if (done == 0) {  // first time scheduled (engine.py:322)
                const int64_t wt = t - q_arr[qi];
                ww = wt > ww ? wt : ww;
            }
        }
        const int lim = k - base < 32 ? k - base : 32;
        for (int j = 0; j < lim; j++) total = xadd(total, __shfl_sync(FULLMASK, term, j));
    }
    const int64_t d = rint_i64(total);
    return PfOut{k, d < 1 ? 1 : d, wmax64(ww)};
}

// ---- decode step completion (engine.py:394-413): token, per-token deadline (metrics.py:57-69),
// retirement (request_metrics metrics.py:72-84), LUT update (costmodel.py:118-128), digest.
__device__ __forceinline__ void ldecode_done(St& S, const LWs& w, int64_t t) {
    const auto AP = w.a32(A_POS), AS = w.a32(A_SEQ), AI = w.a32(A_IDR), AO = w.a32(A_OUT), AN = w.a32(A_INP),
               AM = w.a32(A_MISS), AF = w.a32(A_FLAG);
    const auto AT = w.a64(A_TF);
    const auto TP = w.r64f(TPS);
    uint32_t hs = 0;
    int o = 0;
    int64_t mx = 0, kv_rel = 0;
    const int an = S.an, pre = S.dc_prefix;
    const bool kairos = S.dpol == SLOSIM_DECODE_KAIROS_SLACK;
    bool moved = false;  // a member now sorts before an earlier entry (kairos order repair below)
    int32_t pseq = -1, pidr = -1;
#ifndef SLOSIM_LANE_NO_PREFETCH
    // software-pipelined: entry k+1 is loaded while entry k is processed (stores go to o <= k)
    int4* const V0 = w.v0();
    int4* const V1 = w.v1();
    int4 na = make_int4(0, 0, 0, 0), nb = make_int4(0, 0, 0, 0);
    int64_t n_tf = 0;
    if (an > 0) { na = V0[0]; nb = V1[0]; n_tf = AT[0]; }
#ifndef SLOSIM_LANE_NO_VBASE
    int64_t vb = SLOSIM_INF64;
#endif
    for (int k = 0; k < an; k++) {
        int32_t seq = na.x;
        const int32_t fl = na.y, idr = na.z, pos = na.w, inp = nb.x, outl = nb.y, miss0 = nb.z;
        const int64_t tf = n_tf;
        if (k + 1 < an) { na = V0[(k + 1) * WL]; nb = V1[(k + 1) * WL]; n_tf = AT[k + 1]; }
        if (pre >= 0 ? k < pre : (fl & 1)) {
            seq += 1;
            const int ngen = seq - inp;
            hs += member_hash((uint32_t)pos);
            const int64_t dl = tf + (int64_t)ngen * S.tpot_slo;  // this token's deadline (metrics.py:57-69)
            const int32_t miss = miss0 + (t > dl ? 1 : 0);
#ifndef SLOSIM_LANE_NO_VBASE
            if (ngen != outl - 1) vb = min(vb, dl + S.tpot_slo);
#endif
            if (ngen == outl - 1) {  // retires: request_metrics (metrics.py:72-84)
                const int64_t span = t - tf;
                const double tpot = idiv(span, (int64_t)(outl - 1));
                const bool tpm = tpot <= (double)S.tpot_slo;
                TP[S.ntps] = xdiv((double)(outl - 1), xdiv((double)span, 1e6));
                S.ntps++;
                S.misses += miss;
                S.c_tpot += tpm;
                S.c_e2e += tpm && (fl & 2);
                S.finished++;
                kv_rel += (int64_t)inp + outl;
                continue;
            }
            if (o != k) {
                V0[o * WL] = make_int4(seq, fl & ~1, idr, pos);
                V1[o * WL] = make_int4(inp, outl, miss, 0);
                AT[o] = tf;
            } else {
                *(int2*)&V0[o * WL] = make_int2(seq, fl & ~1);
                AM[o] = miss;
            }
        } else {
#ifndef SLOSIM_LANE_NO_VBASE
            vb = min(vb, tf + ((int64_t)(seq - inp) + 1) * S.tpot_slo);
#endif
            if (o != k) {
                V0[o * WL] = make_int4(seq, fl, idr, pos);
                V1[o * WL] = make_int4(inp, outl, miss0, 0);
                AT[o] = tf;
            }
        }
        if (kairos) moved |= seq < pseq || (seq == pseq && idr < pidr);
        pseq = seq;
        pidr = idr;
        mx = seq > mx ? seq : mx;
        o++;
    }
#else
    for (int k = 0; k < an; k++) {
        int32_t seq = AS[k];
        const int32_t fl = AF[k];
        const int32_t idr = AI[k];
        if (pre >= 0 ? k < pre : (fl & 1)) {
            const int32_t pos = AP[k], inp = AN[k], outl = AO[k];
            const int64_t tf = AT[k];
            seq += 1;
            const int ngen = seq - inp;
            hs += member_hash((uint32_t)pos);
            const int32_t miss = AM[k] + (t > tf + (int64_t)ngen * S.tpot_slo ? 1 : 0);
            if (ngen == outl - 1) {  // retires: request_metrics (metrics.py:72-84)
                const int64_t span = t - tf;
                const double tpot = idiv(span, (int64_t)(outl - 1));
                const bool tpm = tpot <= (double)S.tpot_slo;
                TP[S.ntps] = xdiv((double)(outl - 1), xdiv((double)span, 1e6));
                S.ntps++;
                S.misses += miss;
                S.c_tpot += tpm;
                S.c_e2e += tpm && (fl & 2);
                S.finished++;
                kv_rel += (int64_t)inp + outl;
                continue;
            }
            if (o != k) { AP[o] = pos; AN[o] = inp; AO[o] = outl; AT[o] = tf; AI[o] = idr; }
            AM[o] = miss;
            AS[o] = seq;
            AF[o] = fl & ~1;
        } else if (o != k) {
            AP[o] = AP[k]; AN[o] = AN[k]; AO[o] = AO[k]; AT[o] = AT[k]; AI[o] = idr; AM[o] = AM[k]; AS[o] = seq;
            AF[o] = fl;
        }
        if (kairos) moved |= seq < pseq || (seq == pseq && idr < pidr);
        pseq = seq;
        pidr = idr;
        mx = seq > mx ? seq : mx;
        o++;
    }
#endif
    S.an = o;
    S.amax = mx;
    S.kv -= kv_rel;
#ifndef SLOSIM_LANE_NO_VBASE
    S.vbase = vb;
#endif
    if (moved) {
        // members moved up by one token: restore (seq_len, id) order by insertion
        int4* const V0 = w.v0();
        int4* const V1 = w.v1();
        for (int k = 1; k < o; k++) {
            const int4 a = V0[k * WL];
            if (!(AS[k - 1] > a.x || (AS[k - 1] == a.x && AI[k - 1] > a.z))) continue;
            const int4 b = V1[k * WL];
            const int64_t tf = AT[k];
            int j = k;
            while (j > 0 && (AS[j - 1] > a.x || (AS[j - 1] == a.x && AI[j - 1] > a.z))) {
                V0[j * WL] = V0[(j - 1) * WL]; V1[j * WL] = V1[(j - 1) * WL]; AT[j] = AT[j - 1];
                j--;
            }
            V0[j * WL] = a; V1[j * WL] = b; AT[j] = tf;
        }
    }
#ifdef SLOSIM_LANE_LATE_LUT
    if (S.use_lut) {
        // DecodeStepLUT.update on the full power-of-two grid: cell sum/count/mean (slopes follow the means)
        const LGeo& g = S.g;
        const int i = min(gbidx(S.dc_bsz), g.nb - 1);
        const int j = min(((S.dc_max + (1 << g.wsh) - 1) >> g.wsh) - 1, g.ns - 1);
        const int c = i * g.ns + j;
        const auto M = w.mean(), Su = w.sum();
        const auto C = w.cnt();
        const double sum = xadd(Su[c], (double)S.dc_dur);
        const int32_t cnt = C[c] + 1;
        Su[c] = sum;
        C[c] = cnt;
        M[c] = xdiv(sum, (double)cnt);
    }
#endif
    S.dsteps++;
    uint64_t D = dstep(S.D, (uint64_t)t ^ 0x5A5A5A5A5A5A5A5AULL);
    D = dstep(D, ((uint64_t)hs << 32) | (uint32_t)S.dc_bsz);
    S.D = dstep(D, (uint64_t)S.dc_dur);
    S.dc_end = SLOSIM_INF64;
}

// FCFS-prefill instances fast-forward at every trip by default.  Alone, fcfs + continuous is faster with
// its runs confined to the launch's tail (299 -> 130M req/s with them everywhere, 243M in the tail only),
// but in the config-5 mix the warp's other lanes gain more than it loses: on 131,072-instance slices
// 48.4M (tail only, quorum 5/8) -> 50.6-51.3M req/s (always, quorum 1/8), `profiles/r2p_ff_quorum_ab.log`.
#ifdef SLOSIM_LANE_FF_FCFS_TAIL_ONLY
#define LFF_PREFILL_EXCLUDED(S, tail) ((S).ppol == SLOSIM_PREFILL_FCFS && !(tail))
#else
#define LFF_PREFILL_EXCLUDED(S, tail) false
#endif
#ifndef SLOSIM_LANE_FF_QUORUM8  // eighths of the live lanes that must be able to fast-forward
#define SLOSIM_LANE_FF_QUORUM8 1
#endif
#ifndef SLOSIM_LANE_FF_MAX
#define SLOSIM_LANE_FF_MAX 64
#endif
// ---- continuous batching (decode_sched.py:114-124) between other events, on the lane.  The step just
// started batches the whole active set; so does every following decode start until an arrival,
// transfer or prefill completion (the next rare instant), an admission (which needs one of those or a
// retirement) or a retirement.  Completions that end before the next rare instant, retire nobody and
// miss no per-token deadline (metrics.py:57-69) are applied here in step order: the digest fold of
// each completion, the next step's ground-truth duration (engine.py:185-192) and start.  The step
// after the run is left in progress for the loop.  The engine's counters and the members' token
// counts advance by the number of completions.
#ifndef SLOSIM_LANE_NO_VBASE
__device__ __forceinline__ void lff_continuous(St& S, const LWs& w) {
    int64_t tr = min(S.next_arr, S.pf_end);
    tr = min(tr, S.tr_min);
    const int an = S.an;
    const int64_t tpot = S.tpot_slo;
    // the earliest next-token deadline of the active set (the slack base, kept by the member pass and
    // admission, less one TPOT): no member misses at completion m iff e_m - (m+1)*tpot <= cmin
    const int64_t cmin = S.vbase - tpot;  // (lff_ok: the in-progress step's completion is pure)
    const int4* const V0 = w.v0();
    const int4* const V1 = w.v1();
    uint32_t hs = 0;
    int r = 0x7fffffff;
    for (int k = 0; k < an; k++) {
        const int4 a = V0[k * WL], b = V1[k * WL];
        hs += member_hash((uint32_t)a.w);
        r = min(r, b.y - 2 - (a.x - b.x));
    }
    const uint64_t mid = ((uint64_t)hs << 32) | (uint32_t)an;
    int m = 0, bmax = S.dc_max;
    int64_t e = S.dc_end, d = S.dc_dur;
    uint64_t D = S.D;
    // completion m: before the next rare instant, nobody retires (m < r), nobody misses a deadline
    // (e_m - (m+1)*tpot <= tf + n_gen*tpot for every member)
    // (at most SLOSIM_LANE_FF_MAX per call: a lane alone in a long quiet stretch would otherwise hold
    // its warp while the other lanes wait at the reconvergence point)
    const int mmax = min(r, SLOSIM_LANE_FF_MAX);
    while (m < mmax && e < tr && e - (int64_t)(m + 1) * tpot <= cmin) {
        D = dstep(D, (uint64_t)e ^ 0x5A5A5A5A5A5A5A5AULL);
        D = dstep(D, mid);
        D = dstep(D, (uint64_t)d);
        m++;
        bmax++;
        const double val = S.gline ? gt_line_eval(S.gl, an, bmax)
                                   : decode_formula(S.P->n_base, S.P->base_x, S.P->base_y, S.P->gamma, an, bmax);
        d = rint_i64(val);
        d = d < 1 ? 1 : d;
        e += d;
    }
    if (m == 0) return;
    const auto AS = w.a32(A_SEQ);
    for (int k = 0; k < an; k++) AS[k] = AS[k] + m;
    S.D = D;
    S.dsteps += m;
    S.v_dec += (int64_t)m * an;
    S.b_dec += (int64_t)m * an;
    S.amax += m;
    S.dc_max = bmax;
    S.dc_dur = d;
    S.dc_end = e;
}

// A continuous-batching step in progress that batches the whole active set (no admission since its
// start) and ends before the next rare instant with no member missing its deadline at it.
__device__ __forceinline__ bool lff_ok(const St& S, bool tail) {
    if (S.dpol != SLOSIM_DECODE_CONTINUOUS || S.use_lut || S.dc_end == SLOSIM_INF64 || S.dc_prefix != S.an ||
        S.an < 1 || LFF_PREFILL_EXCLUDED(S, tail))
        return false;
    const int64_t tr = min(min(S.next_arr, S.pf_end), S.tr_min);
    return S.dc_end < tr && S.dc_end <= S.vbase;
}
#endif

// ---- start a decode step (engine.py:377-392; decode_sched.py:60-124)
__device__ __forceinline__ void ldecode_start(St& S, const LWs& w, int64_t t) {
    const int an = S.an;
    S.v_dec += an;
    S.max_a = an > S.max_a ? an : S.max_a;
    int bsz = an, bmax = (int)S.amax;
    if (S.dpol == SLOSIM_DECODE_KAIROS_SLACK) {
        // Alg. 3 (select_decode_batch decode_sched.py:60-111) over the (seq_len, id)-ordered active set.
        // With one active request both outcomes (admit it / fall back) are the same batch.
        const auto AS = w.a32(A_SEQ), AN = w.a32(A_INP), AF = w.a32(A_FLAG);
        const auto AT = w.a64(A_TF);
        S.dc_prefix = -1;
        int b = 0, ms = 0;
        if (an > 1) {
            const auto M = w.mean();
            const LGeo& g = S.g;
#ifndef SLOSIM_LANE_NO_VBASE
            const int64_t vmin = S.vbase - t;
#else
            int64_t vmin = SLOSIM_INF64;
            for (int k = 0; k < an; k++) {
                const int64_t v = S.tpot_slo * ((int64_t)(AS[k] - AN[k]) + 1) - (t - AT[k]);
                vmin = v < vmin ? v : vmin;
            }
#endif
            const double smin = xsub((double)vmin, llookup(M, g, an, bmax));
            double tcur = 0.0;
            LMemo mm{-1, -1, 0.0, 0.0};
#ifndef SLOSIM_LANE_NO_SCAN_FLAGS
            // candidate k+1's key and flag word (one 8-byte load) are loaded while candidate k is decided
            const int2* const V0 = (const int2*)w.v0();
            int2 nv = V0[0];
            for (int k = 0; k < an; k++) {
                const int seq = nv.x, fl = nv.y;
                if (k + 1 < an) nv = V0[(k + 1) * WL * 2];
                const double ts = llookup_memo(M, g, b + 1, seq, mm);
                if (ts <= smin && (b == 0 || lquot_gt((double)(b + 1), ts, (double)b, tcur))) {
                    AF[k] = fl | 1;
                    b++;
                    tcur = ts;
                    ms = seq;
                }
            }
#else
            int nseq = AS[0];
            for (int k = 0; k < an; k++) {
                const int seq = nseq;
                if (k + 1 < an) nseq = AS[k + 1];
                const double ts = llookup_memo(M, g, b + 1, seq, mm);
                if (ts <= smin && (b == 0 || lquot_gt((double)(b + 1), ts, (double)b, tcur))) {
                    AF[k] |= 1;
                    b++;
                    tcur = ts;
                    ms = seq;
                }
            }
#endif
        }
        if (b > 0) {
            bsz = b;
            bmax = ms;
        } else {
#ifndef SLOSIM_LANE_NO_SCAN_FLAGS
            int fl = AF[0];  // fallback: the whole active set
            for (int k = 0; k < an; k++) {
                const int f = fl;
                if (k + 1 < an) fl = AF[k + 1];
                AF[k] = f | 1;
            }
#else
            for (int k = 0; k < an; k++) AF[k] |= 1;  // fallback: the whole active set
#endif
        }
    } else {
        S.dc_prefix = an;
    }
    S.b_dec += bsz;
    // _GroundTruth.decode_step_us (engine.py:185-192), plain formula
    const double val = S.gline ? gt_line_eval(S.gl, bsz, bmax)
                               : decode_formula(S.P->n_base, S.P->base_x, S.P->base_y, S.P->gamma, bsz, bmax);
    const int64_t d = rint_i64(val);
    S.dc_dur = d < 1 ? 1 : d;
    S.dc_bsz = bsz;
    S.dc_max = bmax;
    S.dc_end = t + S.dc_dur;
#ifndef SLOSIM_LANE_LATE_LUT
    if (S.use_lut) {
        // DecodeStepLUT.update (costmodel.py:118-128) of this step's completion, applied as soon as its
        // ground-truth duration is known: nothing reads the LUT before the next decode start, which
        // follows the completion, so the state every lookup sees is the reference's.  In the same
        // block as the ground-truth division, so the two divisions overlap.
        const LGeo& g = S.g;
        const int i = min(gbidx(bsz), g.nb - 1);
        const int j = min(((bmax + (1 << g.wsh) - 1) >> g.wsh) - 1, g.ns - 1);
        const int c = i * g.ns + j;
        const auto M = w.mean(), Su = w.sum();
        const auto C = w.cnt();
        const double sum = xadd(Su[c], (double)S.dc_dur);
        const int32_t cnt = C[c] + 1;
        Su[c] = sum;
        C[c] = cnt;
        M[c] = xdiv(sum, (double)cnt);
    }
#endif
    LANE_HOOK_DECODE(S, w);
}

// One instant of the lane's instance (the instant loop engine.py:264-271), in two parts around the
// prefill start: lstep_a applies every event at the instant and the admissions and reports whether a
// prefill step is to start (need_pf); lstep_c then starts a decode step.  lstep_a returns false,
// after writing the summary row, once the instance is quiescent.
__device__ __forceinline__ bool lstep_a(St& S, const LCtx& cx, const LWs& w, int64_t& t, bool& need_pf) {
    const int64_t t_rare = min(min(S.next_arr, S.pf_end), S.tr_min);
    t = min(S.dc_end, t_rare);
    need_pf = false;
    if (t == SLOSIM_INF64) {
        lfinalize(S, cx, w);
        return false;
    }
    S.t_end = t;
    if (t_rare == t) lrare(S, cx, w, t);
    if (S.dc_end == t) ldecode_done(S, w, t);
    if (S.pt > S.ph) ladmit(S, cx, w);
    need_pf = S.pf_end == SLOSIM_INF64 && S.qt > S.qh;
    return true;
}

__device__ __forceinline__ void lstep_c(St& S, const LWs& w, int64_t t) {
    if (S.dc_end == SLOSIM_INF64 && S.an > 0) ldecode_start(S, w, t);
}

// Single-lane form (host test harness): the prefill step starts on this lane alone.
__device__ __forceinline__ bool lstep(St& S, const LCtx& cx, const LWs& w) {
    int64_t t;
    bool need_pf;
    if (!lstep_a(S, cx, w, t, need_pf)) return false;
    if (need_pf) lprefill_start(S, cx, w, t);
    lstep_c(S, w, t);
    return true;
}

#ifndef SLOSIM_LANE_MIN_BLOCKS
#define SLOSIM_LANE_MIN_BLOCKS 2
#endif

// Urgency/SJF prefill starts over a queue of at most this many requests run on the lane itself
// (quadratic in the queue length, but every such lane proceeds at once); longer queues go to the
// warp-cooperative path
#ifndef SLOSIM_LANE_SERIAL_PF_MAX
#define SLOSIM_LANE_SERIAL_PF_MAX 8
#endif

// Persistent lane engine: each lane pulls instances (in `order`) from the work counter.
__global__ void __launch_bounds__(128, SLOSIM_LANE_MIN_BLOCKS)
    lane_kernel(const __grid_constant__ LCtx cx, char* ws_base, int64_t cap, int cells, unsigned long long* work,
                int lanes_per_warp) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const size_t warp_bytes = lws_bytes(cap, cells);
    const LWs w{ws_base + (size_t)gw * warp_bytes, (size_t)(cap > 0 ? cap : 1), cells, lane};
    const int64_t N = cx.B.n_instances;
    St S;
    S.ii = 0;
    // live: an instance in progress; done: the work queue is drained.  Launches of small batches,
    // where per-instance latency decides, use only lanes [0, lanes_per_warp) of each warp.
    bool live = false, done = lane >= lanes_per_warp;
    for (;;) {
        if (!live && !done) {
            // pull the next instance (one atomic per warp for all lanes that need work)
            const unsigned need = __activemask();
            const int leader = __ffs(need) - 1;
            const int rank = __popc(need & ((1u << lane) - 1u));
            unsigned long long base = 0;
            if (lane == leader) base = atomicAdd(work, (unsigned long long)__popc(need));
            base = __shfl_sync(need, base, leader);
            const unsigned long long k = base + rank;
            if ((int64_t)k >= N) {
                done = true;
            } else {
                const int64_t ii = cx.B.order ? cx.B.order[k] : (int64_t)k;
                if (ii >= 0 && ii < N) {
                    if (!lane_eligible(cx, ii)) cx.deferred[atomicAdd(cx.n_deferred, 1ULL)] = ii;
                    else live = linit(S, cx, w, ii);
                }
            }
        }
        int64_t t = 0;
        bool need_pf = false;
        if (live) live = lstep_a(S, cx, w, t, need_pf);
        // prefill starts: FCFS packs a prefix of the queue, cheap on the lane itself; the urgency and
        // SJF policies order the whole queue, so one lane's queue at a time, all lanes cooperating
        if (need_pf && (S.ppol == SLOSIM_PREFILL_FCFS || S.qt - S.qh <= SLOSIM_LANE_SERIAL_PF_MAX)) {
            lprefill_start(S, cx, w, t);
            need_pf = false;
        }
        const int64_t budget = need_pf ? (int64_t)linst(cx, S).chunk_budget : 0;  // lanes with a queue only
        __syncwarp();
        for (unsigned m = __ballot_sync(FULLMASK, need_pf); m; m &= m - 1) {
            const int L = __ffs((int)m) - 1;
            const PfOut r = coop_prefill_start(
                w.for_lane(L).ws(), __shfl_sync(FULLMASK, (int)S.ppol, L), __shfl_sync(FULLMASK, S.qh, L),
                __shfl_sync(FULLMASK, S.qt, L), __shfl_sync(FULLMASK, budget, L),
                __shfl_sync(FULLMASK, t, L), __shfl_sync(FULLMASK, S.est_tok, L),
                __shfl_sync(FULLMASK, S.est_busy, L), __shfl_sync(FULLMASK, S.ttft_slo, L),
                (const slosim_profile_t*)__shfl_sync(FULLMASK, (unsigned long long)S.P, L), lane);
            if (lane == L) {
                const int qlen = S.qt - S.qh;
                S.v_pre += qlen;
                S.max_q = qlen > S.max_q ? qlen : S.max_q;
                S.pf_k = r.k;
                S.worst_wait = r.ww > S.worst_wait ? r.ww : S.worst_wait;
                S.pf_dur = r.dur;
                S.pf_end = t + r.dur;
            }
        }
        if (live) lstep_c(S, w, t);
#if !defined(SLOSIM_LANE_NO_FF) && !defined(SLOSIM_LANE_NO_VBASE)
        // continuous-batching runs are fast-forwarded on the lanes only when (nearly) every live lane of
        // the warp has one: a lone lane's run would hold the warp while the others wait
        {
            const bool drained = __any_sync(FULLMASK, done);  // the work queue is empty (every lane takes part)
            const bool ffc = live && lff_ok(S, drained);
            const unsigned cm = __ballot_sync(FULLMASK, ffc), lm = __ballot_sync(FULLMASK, live);
            if (ffc && __popc(cm) * 8 >= __popc(lm) * SLOSIM_LANE_FF_QUORUM8) lff_continuous(S, w);
        }
#endif
        if (__all_sync(FULLMASK, done && !live)) break;
    }
}

}  // namespace lane
}  // namespace slosim
