// tengine.cuh — the lane engine: one simulated instance per THREAD.
//
// The warp engine (engine.cuh) gives each instance a whole warp; with 3-4
// requests active on average (config 5) most lanes idle while the warp walks
// a long chain of shuffles and reductions per decode step, and the kernel is
// bound by instruction issue and fetch.  Here every lane runs its own
// instance of the same event loop (engine.py:261-302) with scalar state in
// registers and its request sets in a per-lane workspace, so one warp
// instruction advances 32 instances.  The loop is flattened: each trip is one
// instant of the lane's instance, and a lane whose instance has finished
// writes its summary and pulls the next instance from the work queue in the
// same trip, so the warp stays full until the queue drains.
//
// Workspace: per warp, every array is lane-interleaved (element k of lane l
// at [k * 32 + l]), so the loops that walk the active set from its start —
// the hot ones — load one line per warp instruction.
//
// Scope: batches whose profiles all have the power-of-two LUT geometry
// (the reference defaults, costmodel.py:26-27), a fully populated LUT, the
// plain ground-truth decode formula (no frozen file LUT, no noise), and no
// per-request rows, event trace or LUT export.  capi.cu routes every other
// batch to the warp engine.  Decisions, counters and digests are identical to
// the warp engine and the oracle.
//
// Reference mapping: same as engine.cuh (engine.py:198-413, prefill_sched.py,
// decode_sched.py:60-124, costmodel.py:118-187, metrics.py:30-144).
#pragma once
#include "../../include/slosim_b200.h"
#include "lut.cuh"

namespace slosim {
namespace lane {

constexpr int WL = 32;

#ifndef LANE_HOOK_DECODE  // test harness hook (tools/lane_host): called at every decode step start
#define LANE_HOOK_DECODE(S, w)
#endif

template <class T>
struct Arr {
    T* p;  // element 0 of this lane
    __device__ __forceinline__ T& operator[](int k) const { return p[(size_t)k * WL]; }
};

// Per-lane arrays, capacity `cap` requests (LUT arrays: `cells`).
//   A_RT   decode tokens still to generate (output_len - 1 - n_generated)
//   A_DL   deadline of the next token: t_first + (n_generated + 1) * tpot_slo (metrics.py:57-69); the
//          Eq. 2 slack of decode_sched.py:36-57 is A_DL - t_now
//   A_FLAG bit 0: admitted by this step's Alg. 3 scan; bit 1: TTFT met; bits 2..: admission stamp
//          (decode steps started before the request joined; the Alg. 3 fallback batch is every
//          entry whose stamp <= the step's index)
enum LI32 { Q_POS, Q_REM, Q_FULL, Q_INP, PF_Q, PF_TAKE, PD_POS, PD_IDR, TR_POS, A_POS, A_SEQ, A_IDR, A_OUT, A_INP,
            A_MISS, A_FLAG, A_RT, N_LI32 };
enum LI64 { Q_ARR, Q_KEY, PD_TPF, PD_TTR, TR_T, TR_TPF, A_TF, A_DL, TPS, N_LI64 };

__host__ __device__ inline size_t lws_bytes(int64_t cap, int cells) {
    size_t c = (size_t)(cap > 0 ? cap : 1);
    return (size_t)WL * (N_LI32 * 4 * c + N_LI64 * 8 * c + (size_t)cells * (8 + 8 + 4));
}

// One warp's workspace: region r of element type T holds [capacity][32 lanes].
struct LWs {
    char* wb;  // warp base
    size_t c;
    int cells, lane;
    __device__ __forceinline__ Arr<int32_t> i32(int k) const {
        return Arr<int32_t>{(int32_t*)(wb + (size_t)k * WL * 4 * c) + lane};
    }
    __device__ __forceinline__ Arr<int64_t> i64(int k) const {
        return Arr<int64_t>{(int64_t*)(wb + (size_t)N_LI32 * WL * 4 * c + (size_t)k * WL * 8 * c) + lane};
    }
    __device__ __forceinline__ Arr<double> f64(int k) const { return Arr<double>{(double*)i64(k).p}; }
    // LUT cells: mean, sum (f64), count (i32)
    __device__ __forceinline__ char* lut_base() const { return wb + (size_t)WL * (N_LI32 * 4 * c + N_LI64 * 8 * c); }
    __device__ __forceinline__ Arr<double> mean() const { return Arr<double>{(double*)lut_base() + lane}; }
    __device__ __forceinline__ Arr<double> sum() const {
        return Arr<double>{(double*)(lut_base() + (size_t)WL * 8 * cells) + lane};
    }
    __device__ __forceinline__ Arr<int32_t> cnt() const {
        return Arr<int32_t>{(int32_t*)(lut_base() + (size_t)WL * 16 * cells) + lane};
    }
};

// Python-form row interpolation on the power-of-two grid (lut.cuh lut_eval<true> / geval_p):
// value of row r at column selection (c, dx) from the stored means; the np.interp
// slope of a populated column pair is (m[c+1] - m[c]) * 2^-wsh, exactly as stored by
// lut_build / gupdate.
struct LGeo { int nb, ns, wsh; double inv_w; };

__device__ __forceinline__ double lrow(const Arr<double>& M, const LGeo& g, int r, int c, double dx) {
    const int k = r * g.ns + c;
    const double m0 = M[k];
    if (dx == 0.0) return m0;
    const double slope = xmul(xsub(M[k + 1], m0), g.inv_w);
    return xadd(xmul(slope, dx), m0);
}

__device__ __forceinline__ double llookup(const Arr<double>& M, const LGeo& g, int bsz, int seq) {
    // column selection (lut_col<true>)
    const int w = 1 << g.wsh;
    int c = (seq >> g.wsh) - 1;
    const bool in = seq > w && c < g.ns - 1;
    c = in ? c : (seq <= w ? 0 : g.ns - 1);
    const double dx = in ? (double)(seq & (w - 1)) : 0.0;
    // row selection (lut_rows_nb<true>)
    const int i = gbidx(bsz);
    const bool single = (i == 0) | (i >= g.nb) | ((1u << i) == (unsigned)bsz);
    const int lo = i >= g.nb ? g.nb - 1 : (i == 0 ? 0 : i - 1);
    const int r1 = single ? (i >= g.nb ? g.nb - 1 : i) : lo;
    const double v1 = lrow(M, g, r1, c, dx);
    if (single) return v1;
    const double v2 = lrow(M, g, i, c, dx);
    return xadd(v1, xmul(xmul(xsub(v2, v1), (double)(bsz - (1 << lo))), pow2_neg(lo)));
}

// (a, x, b, y): RN(a/x) > RN(b/y) (decode_sched.py:87-89), see numerics.cuh quot_gt.
__device__ __noinline__ bool lquot_exact(double a, double x, double b, double y) { return __ddiv_rn(a, x) > __ddiv_rn(b, y); }
__device__ __forceinline__ bool lquot_gt(double a, double x, double b, double y) {
    const double p = __dmul_rn(a, y), q = __dmul_rn(b, x);
    if (p > __dmul_rn(q, 1.0 + 0x1p-50)) return true;
    if (p < __dmul_rn(q, 1.0 - 0x1p-50)) return false;
    return lquot_exact(a, x, b, y);
}

// Nearest-rank selection (metrics.py:87-92): the r-th smallest (1-based) of a[lo..hi) by quickselect
// (positive doubles; ties are equal values so any partition order gives the same value).
__device__ __noinline__ double lselect(const Arr<double>& a, int lo, int hi, int r) {
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

// Per-lane instance state that only the rare events touch; it lives in local memory (the rare
// handlers take it by reference).  The decode hot path keeps its own state in registers (Hot) and
// the two are synchronised around the rare handlers.
struct St {
    int64_t ii;
    int64_t off;  // trace offset
    const slosim_profile_t* P;
    double fac, tpt;
    int64_t ttft_slo, kv_cap, tr_base;
    int n, budget;
    int ppol;
    bool gline;
    GtLine gl;
    int ai, qh, qt, pf_k, ph, pt, trn;
    int64_t next_arr, pf_end, pf_dur, tr_min, kv, est_tok, est_busy;
    int32_t c_ttft, c_tpot, c_e2e, ntps, max_q, finished;
    int64_t misses, worst_wait, psteps, v_pre;
    // synchronised with Hot around the rare handlers / at the end
    int an, amax, steps_started;
    uint64_t D;
    int64_t dsteps, v_dec, b_dec, t_end;
    int max_a;
};

// Decode hot-path state (registers).
struct Hot {
    int64_t dc_end, t_rare, dc_dur, tpot, t_end, dsteps, v_dec, b_dec;
    uint64_t D;
    int an, amax, dc_bsz, dc_max, mode, max_a;  // mode: >= 0 prefix batch, -1 flag bit 0, -2 stamp (fallback)
    bool pend, kairos, use_lut;
    int nb, ns, wsh;
};

__device__ __forceinline__ int64_t larrival(const LCtx& cx, const St& S, int p) {
    const int64_t a = cx.B.traces.arrival_us[S.off + p];
    return S.fac > 0 ? rint_i64(xmul((double)a, S.fac)) : a;
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
__device__ __noinline__ bool linit(St& S, const LCtx& cx, const LWs& w, int64_t ii) {
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
    S.fac = I->rescale_factor;
    S.ttft_slo = I->ttft_slo_us;
    S.kv_cap = I->kv_capacity_tokens;
    S.tr_base = I->transfer_base_us;
    S.tpt = I->transfer_per_token_us;
    S.budget = I->chunk_budget;
    S.ppol = I->prefill_policy;
    const LutMem* ST = cx.sched_tab + pid;
    // KV reservation check (engine.py:227-232)
    const int32_t* Tinp = B->traces.input_len + S.off;
    const int32_t* Tout = B->traces.output_len + S.off;
    int64_t worst = 0;
    for (int p = 0; p < S.n; p++) {
        const int64_t need = (int64_t)Tinp[p] + Tout[p];
        worst = need > worst ? need : worst;
    }
    if (worst > S.kv_cap || ST->rowmask == 0) {
        lwrite_status(B->summaries + ii, S.n, SLOSIM_ECONFIG);
        return false;
    }
    if (I->decode_policy == SLOSIM_DECODE_KAIROS_SLACK || (B->flags & SLOSIM_F_ALWAYS_LUT)) {
        const Arr<double> M = w.mean(), Su = w.sum();
        const Arr<int32_t> C = w.cnt();
        const int K = ST->nb * ST->ns;
        for (int k = 0; k < K; k++) { M[k] = ST->mean[k]; Su[k] = ST->sum[k]; C[k] = ST->cnt[k]; }
    }
    S.gline = gt_line_make(S.P->n_base, S.P->base_x, S.P->base_y, S.P->gamma, S.gl);
    S.est_tok = S.P->est_tokens;
    S.est_busy = S.P->est_busy_us;
    S.ai = S.qh = S.qt = S.pf_k = S.ph = S.pt = S.trn = 0;
    S.next_arr = S.n > 0 ? larrival(cx, S, 0) : SLOSIM_INF64;
    S.pf_end = S.tr_min = SLOSIM_INF64;
    S.pf_dur = S.kv = 0;
    S.c_ttft = S.c_tpot = S.c_e2e = S.ntps = S.max_q = S.finished = 0;
    S.misses = S.worst_wait = S.psteps = S.v_pre = 0;
    S.an = S.amax = S.steps_started = 0;
    S.D = 0;
    return true;
}

// Hot state of a freshly started instance.
__device__ __forceinline__ void lhot_init(Hot& H, const St& S, const LCtx& cx) {
    const slosim_instance_t* I = cx.B.instances + S.ii;
    const LutMem* ST = cx.sched_tab + I->profile_id;
    H.dc_end = SLOSIM_INF64;
    H.t_rare = S.next_arr;
    H.dc_dur = 0;
    H.tpot = I->tpot_slo_us;
    H.t_end = H.dsteps = H.v_dec = H.b_dec = 0;
    H.D = 0;
    H.an = H.amax = H.dc_bsz = H.dc_max = H.max_a = 0;
    H.mode = 0;
    H.pend = false;
    H.kairos = I->decode_policy == SLOSIM_DECODE_KAIROS_SLACK;
    H.use_lut = H.kairos || (cx.B.flags & SLOSIM_F_ALWAYS_LUT);
    H.nb = ST->nb;
    H.ns = ST->ns;
    H.wsh = ST->wsh;
}

__device__ __forceinline__ void lhot_out(const Hot& H, St& S) {
    S.an = H.an;
    S.amax = H.amax;
    S.D = H.D;
    S.steps_started = (int)H.dsteps + (H.dc_end != SLOSIM_INF64 ? 1 : 0);
}
__device__ __forceinline__ void lhot_in(Hot& H, const St& S) {
    H.an = S.an;
    H.amax = S.amax;
    H.D = S.D;
    int64_t tr = S.next_arr < S.pf_end ? S.next_arr : S.pf_end;
    H.t_rare = S.tr_min < tr ? S.tr_min : tr;
    H.pend = S.pt > S.ph || (S.pf_end == SLOSIM_INF64 && S.qt > S.qh);
}

// metrics aggregate (metrics.py:109-144) + summary row.
__device__ __noinline__ void lfinalize(St& S, const LCtx& cx, const LWs& w) {
    double p50 = __longlong_as_double(0x7ff8000000000000LL), p90 = p50;
    if (S.ntps > 0) {
        const Arr<double> T = w.f64(TPS);
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
    const Arr<int64_t> PT = w.i64(PD_TPF), PR = w.i64(PD_TTR);
    const Arr<int32_t> PP = w.i32(PD_POS), PI = w.i32(PD_IDR);
    int k = S.pt;
    while (k > S.ph && (PT[k - 1] > tpf || (PT[k - 1] == tpf && PI[k - 1] > idr))) {
        PT[k] = PT[k - 1]; PR[k] = PR[k - 1]; PP[k] = PP[k - 1]; PI[k] = PI[k - 1];
        k--;
    }
    PT[k] = tpf; PR[k] = ttr; PP[k] = pos; PI[k] = idr;
    S.pt++;
}

// ---- rare events (arrivals, transfers, prefill completion) at instant t (engine.py:286-350)
__device__ __noinline__ void lrare(St& S, const LCtx& cx, const LWs& w, int64_t t) {
    const int32_t* Tinp = cx.B.traces.input_len + S.off;
    const int32_t* Tidr = cx.B.traces.id_rank + S.off;
    if (S.next_arr == t) {  // arrivals (engine.py:288-291): a contiguous run of the trace
        const int32_t* Thit = cx.B.traces.prefix_hit_len + S.off;
        const Arr<int32_t> QP = w.i32(Q_POS), QR = w.i32(Q_REM), QF = w.i32(Q_FULL), QI = w.i32(Q_INP);
        const Arr<int64_t> QA = w.i64(Q_ARR);
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
        const Arr<int64_t> TT = w.i64(TR_T), TF = w.i64(TR_TPF);
        const Arr<int32_t> TP = w.i32(TR_POS);
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
        const Arr<int32_t> QP = w.i32(Q_POS), QR = w.i32(Q_REM), QF = w.i32(Q_FULL), QI = w.i32(Q_INP);
        const Arr<int64_t> QA = w.i64(Q_ARR);
        const Arr<int32_t> FQ = w.i32(PF_Q), FT = w.i32(PF_TAKE);
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
                const int64_t delay = S.tr_base + rint_i64(xmul((double)QI[qi], S.tpt));
                if (delay == 0) {
                    lpending_insert(S, w, t, Tidr[pos], t, pos);
                } else {
                    const Arr<int64_t> TT = w.i64(TR_T), TF = w.i64(TR_TPF);
                    TT[S.trn] = t + delay; TF[S.trn] = t; w.i32(TR_POS)[S.trn] = pos;
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
__device__ __forceinline__ void ladmit(St& S, const LCtx& cx, const LWs& w, int64_t t, int64_t tpot, bool kairos) {
    const int32_t* Tinp = cx.B.traces.input_len + S.off;
    const int32_t* Tout = cx.B.traces.output_len + S.off;
    const Arr<int64_t> PR = w.i64(PD_TTR);
    const Arr<int32_t> PP = w.i32(PD_POS), PI = w.i32(PD_IDR);
    const Arr<int32_t> AP = w.i32(A_POS), AS = w.i32(A_SEQ), AI = w.i32(A_IDR), AO = w.i32(A_OUT), AN = w.i32(A_INP),
                       AM = w.i32(A_MISS), AF = w.i32(A_FLAG), AR = w.i32(A_RT);
    const Arr<int64_t> AT = w.i64(A_TF), AD = w.i64(A_DL);
    const int stamp = S.steps_started << 2;
    while (S.pt > S.ph) {
        const int32_t pos = PP[S.ph];
        const int32_t outl = Tout[pos], inp = Tinp[pos];
        const int64_t need = (int64_t)inp + outl;
        if (S.kv + need > S.kv_cap) break;  // head-of-line blocking
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
        if (kairos) {
            while (k > 0 && (AS[k - 1] > inp || (AS[k - 1] == inp && AI[k - 1] > idr))) {
                AP[k] = AP[k - 1]; AS[k] = AS[k - 1]; AI[k] = AI[k - 1]; AO[k] = AO[k - 1]; AN[k] = AN[k - 1];
                AM[k] = AM[k - 1]; AF[k] = AF[k - 1]; AR[k] = AR[k - 1]; AT[k] = AT[k - 1]; AD[k] = AD[k - 1];
                k--;
            }
        }
        AP[k] = pos; AS[k] = inp; AI[k] = idr; AO[k] = outl; AN[k] = inp; AM[k] = 0; AF[k] = (ttm ? 2 : 0) | stamp;
        AR[k] = outl - 1; AT[k] = ttr; AD[k] = ttr + tpot;
        S.an++;
        S.amax = inp > S.amax ? inp : S.amax;
    }
}

// ---- start a prefill step (engine.py:307-325, prefill_sched.py:93-145)
__device__ __forceinline__ void lprefill_start(St& S, const LWs& w, int64_t t) {
    const Arr<int32_t> QR = w.i32(Q_REM), QF = w.i32(Q_FULL), QI = w.i32(Q_INP);
    const Arr<int64_t> QA = w.i64(Q_ARR), QK = w.i64(Q_KEY);
    const Arr<int32_t> FQ = w.i32(PF_Q), FT = w.i32(PF_TAKE);
    const int qlen = S.qt - S.qh;
    S.v_pre += qlen;
    S.max_q = qlen > S.max_q ? qlen : S.max_q;
    int k = 0;
    int64_t left = S.budget;
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
                const int64_t slack = S.ttft_slo - (cursor - a);
                const double u = idiv(slack, S.ttft_slo);
                const double sc = u >= 0 ? xdiv(u, (double)QI[qi]) : xmul(u, (double)QI[qi]);
                QK[qi] = (int64_t)~dkey(sc);
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
                const uint64_t key = sjf ? (uint64_t)(uint32_t)QR[qi] : (uint64_t)QK[qi];
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

// ---- admission then a new prefill step (out of line)
__device__ __noinline__ void lafter(St& S, const LCtx& cx, const LWs& w, int64_t t, int64_t tpot, bool kairos) {
    if (S.pt > S.ph) ladmit(S, cx, w, t, tpot, kairos);
    if (S.pf_end == SLOSIM_INF64 && S.qt > S.qh) lprefill_start(S, w, t);
}

// request_metrics (metrics.py:72-84) of a request retiring at t; returns its KV reservation.
__device__ __noinline__ int64_t lretire(St& S, const LWs& w, int k, int64_t t, int64_t tpot, int32_t fl) {
    const int32_t outl = w.i32(A_OUT)[k], inp = w.i32(A_INP)[k];
    const int64_t span = t - w.i64(A_TF)[k];
    const double tp = idiv(span, (int64_t)(outl - 1));
    const bool tpm = tp <= (double)tpot;
    w.f64(TPS)[S.ntps] = xdiv((double)(outl - 1), xdiv((double)span, 1e6));
    S.ntps++;
    S.c_tpot += tpm;
    S.c_e2e += tpm && (fl & 2);
    S.finished++;
    return (int64_t)inp + outl;
}

// ---- decode step completion (engine.py:394-413): token, per-token deadline
// (metrics.py:57-69), retirement, LUT update (costmodel.py:118-128), digest.
__device__ __forceinline__ void ldecode_done(Hot& H, St& S, const LWs& w, int64_t t) {
    const Arr<int32_t> AP = w.i32(A_POS), AS = w.i32(A_SEQ), AI = w.i32(A_IDR), AO = w.i32(A_OUT), AN = w.i32(A_INP),
                       AM = w.i32(A_MISS), AF = w.i32(A_FLAG), AR = w.i32(A_RT);
    const Arr<int64_t> AT = w.i64(A_TF), AD = w.i64(A_DL);
    uint32_t hs = 0;
    int o = 0, mx = 0;
    int64_t kv_rel = 0;
    const int an = H.an, mode = H.mode;
    const int sid = (int)H.dsteps;  // this step's index
    bool moved = false;  // a member now sorts before an earlier entry (kairos order repair below)
    int32_t pseq = -1;
    for (int k = 0; k < an; k++) {
        int32_t seq = AS[k];
        const int32_t fl = AF[k];
        const bool member = mode >= 0 ? k < mode : (mode == -1 ? (fl & 1) != 0 : (fl >> 2) <= sid);
        if (member) {
            const int32_t pos = AP[k];
            const int64_t dl = AD[k];
            const int32_t rt = AR[k] - 1;
            seq += 1;
            hs += member_hash((uint32_t)pos);
            const int32_t late = t > dl ? 1 : 0;
            if (rt == 0) {  // retires
                S.misses += AM[k] + late;
                kv_rel += lretire(S, w, k, t, H.tpot, fl);
                continue;
            }
            if (o != k) {
                AP[o] = pos; AN[o] = AN[k]; AO[o] = AO[k]; AT[o] = AT[k]; AI[o] = AI[k]; AM[o] = AM[k] + late;
            } else if (late) {
                AM[o] = AM[k] + 1;
            }
            AS[o] = seq;
            AR[o] = rt;
            AD[o] = dl + H.tpot;
            AF[o] = fl & ~1;
        } else if (o != k) {
            AP[o] = AP[k]; AN[o] = AN[k]; AO[o] = AO[k]; AT[o] = AT[k]; AI[o] = AI[k]; AM[o] = AM[k]; AS[o] = seq;
            AF[o] = fl; AR[o] = AR[k]; AD[o] = AD[k];
        }
        if (H.kairos && seq <= pseq) moved = moved || seq < pseq || AI[o] < AI[o - 1];
        pseq = seq;
        mx = seq > mx ? seq : mx;
        o++;
    }
    H.an = o;
    H.amax = mx;
    if (kv_rel) S.kv -= kv_rel;
    if (moved && H.kairos) {
        // members moved up by one token: restore (seq_len, id) order by insertion
        for (int k = 1; k < o; k++) {
            const int32_t sk = AS[k], ik = AI[k];
            if (!(AS[k - 1] > sk || (AS[k - 1] == sk && AI[k - 1] > ik))) continue;
            const int32_t p = AP[k], n_ = AN[k], ou = AO[k], mi = AM[k], fl = AF[k], r = AR[k];
            const int64_t tf = AT[k], dl = AD[k];
            int j = k;
            while (j > 0 && (AS[j - 1] > sk || (AS[j - 1] == sk && AI[j - 1] > ik))) {
                AP[j] = AP[j - 1]; AS[j] = AS[j - 1]; AI[j] = AI[j - 1]; AO[j] = AO[j - 1]; AN[j] = AN[j - 1];
                AM[j] = AM[j - 1]; AF[j] = AF[j - 1]; AR[j] = AR[j - 1]; AT[j] = AT[j - 1]; AD[j] = AD[j - 1];
                j--;
            }
            AP[j] = p; AS[j] = sk; AI[j] = ik; AO[j] = ou; AN[j] = n_; AM[j] = mi; AF[j] = fl; AR[j] = r; AT[j] = tf;
            AD[j] = dl;
        }
    }
    if (H.use_lut) {
        // DecodeStepLUT.update on the full power-of-two grid: cell sum/count/mean (slopes follow the means)
        const int i = min(gbidx(H.dc_bsz), H.nb - 1);
        const int j = min(((H.dc_max + (1 << H.wsh) - 1) >> H.wsh) - 1, H.ns - 1);
        const int c = i * H.ns + j;
        const Arr<double> M = w.mean(), Su = w.sum();
        const Arr<int32_t> C = w.cnt();
        const double sum = xadd(Su[c], (double)H.dc_dur);
        const int32_t cnt = C[c] + 1;
        Su[c] = sum;
        C[c] = cnt;
        M[c] = xdiv(sum, (double)cnt);
    }
    H.dsteps++;
    uint64_t D = dstep(H.D, (uint64_t)t ^ 0x5A5A5A5A5A5A5A5AULL);
    D = dstep(D, ((uint64_t)hs << 32) | (uint32_t)H.dc_bsz);
    H.D = dstep(D, (uint64_t)H.dc_dur);
    H.dc_end = SLOSIM_INF64;
}

// ---- start a decode step (engine.py:377-392; decode_sched.py:60-124)
__device__ __forceinline__ void ldecode_start(Hot& H, const St& S, const LWs& w, int64_t t) {
    const int an = H.an;
    H.v_dec += an;
    H.max_a = an > H.max_a ? an : H.max_a;
    int bsz = an, bmax = H.amax;
    if (H.kairos) {
        // Alg. 3 (select_decode_batch decode_sched.py:60-111) over the (seq_len, id)-ordered active set.
        // With one active request both outcomes (admit it / fall back) are the same batch.
        int b = 0, ms = 0;
        if (an > 1) {
            const Arr<int32_t> AS = w.i32(A_SEQ), AF = w.i32(A_FLAG);
            const Arr<int64_t> AD = w.i64(A_DL);
            const Arr<double> M = w.mean();
            const LGeo g{H.nb, H.ns, H.wsh, pow2_neg(H.wsh)};
            int64_t dmin = SLOSIM_INF64;
            for (int k = 0; k < an; k++) {
                const int64_t d = AD[k];
                dmin = d < dmin ? d : dmin;
            }
            const double smin = xsub((double)(dmin - t), llookup(M, g, an, H.amax));
            double tcur = 0.0;
            for (int k = 0; k < an; k++) {
                const int seq = AS[k];
                const double ts = llookup(M, g, b + 1, seq);
                if (ts <= smin && (b == 0 || lquot_gt((double)(b + 1), ts, (double)b, tcur))) {
                    AF[k] |= 1;
                    b++;
                    tcur = ts;
                    ms = seq;
                }
            }
        }
        if (b > 0) { bsz = b; bmax = ms; H.mode = -1; }
        else H.mode = -2;  // the whole active set
    } else {
        H.mode = an;
    }
    H.b_dec += bsz;
    // _GroundTruth.decode_step_us (engine.py:185-192), plain formula
    const double val = S.gline ? gt_line_eval(S.gl, bsz, bmax)
                               : decode_formula(S.P->n_base, S.P->base_x, S.P->base_y, S.P->gamma, bsz, bmax);
    const int64_t d = rint_i64(val);
    H.dc_dur = d < 1 ? 1 : d;
    H.dc_bsz = bsz;
    H.dc_max = bmax;
    H.dc_end = t + H.dc_dur;
    LANE_HOOK_DECODE(H, w);
}

// One instant of the lane's instance (the instant loop engine.py:264-271): all events at the
// instant, then admission, a new prefill step and a new decode step.  Returns false, after
// writing the summary row, once the instance is quiescent.
__device__ __forceinline__ bool lstep(Hot& H, St& S, const LCtx& cx, const LWs& w) {
    const int64_t t = min(H.dc_end, H.t_rare);
    if (t == SLOSIM_INF64) {
        lhot_out(H, S);
        S.dsteps = H.dsteps; S.v_dec = H.v_dec; S.b_dec = H.b_dec; S.t_end = H.t_end; S.max_a = H.max_a;
        lfinalize(S, cx, w);
        return false;
    }
    H.t_end = t;
    if (H.t_rare == t) {
        lhot_out(H, S);
        lrare(S, cx, w, t);
        lhot_in(H, S);
    }
    if (H.dc_end == t) ldecode_done(H, S, w, t);
    if (H.pend) {
        lhot_out(H, S);
        lafter(S, cx, w, t, H.tpot, H.kairos);
        lhot_in(H, S);
    }
    if (H.dc_end == SLOSIM_INF64 && H.an > 0) ldecode_start(H, S, w, t);
    return true;
}

#ifndef SLOSIM_LANE_MIN_BLOCKS
#define SLOSIM_LANE_MIN_BLOCKS 4
#endif

// Persistent lane engine: each lane pulls instances (in `order`) from the work counter.
__global__ void __launch_bounds__(128, SLOSIM_LANE_MIN_BLOCKS)
    lane_kernel(const __grid_constant__ LCtx cx, char* ws_base, int64_t cap, int cells, unsigned long long* work) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const size_t warp_bytes = lws_bytes(cap, cells);
    const LWs w{ws_base + (size_t)gw * warp_bytes, (size_t)(cap > 0 ? cap : 1), cells, lane};
    const int64_t N = cx.B.n_instances;
    St S;
    Hot H;
    bool live = false;  // this lane has an instance in progress
    for (;;) {
        if (!live) {
            // pull the next instance (one atomic per warp for all lanes that need work)
            const unsigned need = __activemask();
            const int leader = __ffs(need) - 1;
            const int rank = __popc(need & ((1u << lane) - 1u));
            unsigned long long base = 0;
            if (lane == leader) base = atomicAdd(work, (unsigned long long)__popc(need));
            base = __shfl_sync(need, base, leader);
            const unsigned long long k = base + rank;
            if ((int64_t)k >= N) break;
            const int64_t ii = cx.B.order ? cx.B.order[k] : (int64_t)k;
            if (ii < 0 || ii >= N) continue;
            if (!lane_eligible(cx, ii)) {
                cx.deferred[atomicAdd(cx.n_deferred, 1ULL)] = ii;
                continue;
            }
            live = linit(S, cx, w, ii);
            if (live) lhot_init(H, S, cx);
            continue;
        }
        live = lstep(H, S, cx, w);
    }
}

}  // namespace lane
}  // namespace slosim
