// engine.cuh — the batched discrete-event simulator (K1-K5 of SURVEY §2).
//
// One warp simulates one instance (one ClusterConfig x workload, engine.py:195-413)
// from first arrival to quiescence; a persistent grid of warps pulls instances
// from an atomic work counter.  All control flow is warp-uniform: every lane
// holds the same scalar state (time, pool status, counters) and the lanes
// cooperate on the per-request sets (prefill queue, pending admission list,
// active decode set), which live in a per-warp SoA workspace that stays
// L1-resident for the life of an instance; up to 32 active decode requests
// live in the lanes' registers (Slot).  Decode steps between rare events are
// applied in bulk where the batch cannot change (ff_steps), and the LUT has a
// power-of-two geometry path (lut.cuh).  The kernel is instruction-fetch
// bound, so the hot loop is kept short and every rare event runs out of line
// (DESIGN.md §5).
//
// Reference mapping (engine.py):
//   instant loop :264-271                      -> simulate() main loop
//   _dispatch :286-302                         -> arrival / transfer / completion blocks
//   _start_prefill / _finish_prefill_step :307-350
//   _admit :355-375, _start_decode / _finish_decode_step :377-413
//   metrics :274-284 -> metrics.py:30-144      (per-request rows at retirement, finalize)
#pragma once
#include "../../include/slosim_b200.h"
#include "lut.cuh"
#include "warpops.cuh"

namespace slosim {

// Per-profile LUT tables (scheduler seed + frozen ground truth), built once per launch.
#ifndef SLOSIM_ENGINE_ONLY
__global__ void build_profile_tables(const slosim_profile_t* profiles, int n_profiles, LutMem* sched,
                                     LutMem* frozen) {
    int lane = threadIdx.x & 31;
    int p = blockIdx.x;
    if (p >= n_profiles) return;
    const slosim_profile_t* P = profiles + p;
    // a malformed profile (grid or curve sizes beyond the frame) is marked bad: its instances get EINVAL
    const bool ok = P->nb >= 1 && P->nb <= SLOSIM_MAX_BSZ_BUCKETS && P->ns >= 1 && P->ns <= SLOSIM_MAX_SEQ_BUCKETS &&
                    P->n_curve >= 2 && P->n_curve <= SLOSIM_MAX_CURVE_POINTS && P->n_base >= 0 &&
                    P->n_base <= SLOSIM_MAX_BASE_POINTS && (P->n_base >= 1 || P->gt_frozen);
    if (!ok) {
        if (lane == 0) { sched[p].bad = 1; frozen[p].bad = 1; }
        return;
    }
    lut_build(sched + p, P->nb, P->ns, P->bsz_buckets, P->seq_buckets, P->lut_sums, P->lut_counts, lane);
    lut_build(frozen + p, P->nb, P->ns, P->bsz_buckets, P->seq_buckets, P->gt_sums, P->gt_counts, lane);
}
#endif

// ------------------------------------------------------------ trace writer --
struct TraceW {
    int64_t* buf;
    int64_t cap;
    int64_t used;
    __device__ __forceinline__ void put(int64_t idx, int64_t v) const {
        if (buf && idx < cap - 2) buf[idx] = v;
    }
};

// ---------------------------------------------------- decode policy (K3) --
// Orders the active set by (seq_len, id) (decode_sched.py:74) into ord[0..an).
__device__ __noinline__ void decode_order_wide(int an, const int32_t* a_seq, const int32_t* a_idr, int32_t* ord,
                                              int lane);

__device__ __forceinline__ void decode_order(int an, const int32_t* a_seq, const int32_t* a_idr, int32_t* ord,
                                             int lane) {
    if (an <= 32) {
        uint64_t key = lane < an ? (((uint64_t)(uint32_t)a_seq[lane] << 32) | (uint32_t)a_idr[lane]) : ~0ULL;
        int rank = 0;
        for (int j = 0; j < an; j++) {
            uint64_t kj = __shfl_sync(FULLMASK, key, j);
            rank += kj < key;
        }
        if (lane < an) ord[rank] = lane;
        __syncwarp();
    } else {
        decode_order_wide(an, a_seq, a_idr, ord, lane);
    }
}

__device__ __noinline__ void decode_order_wide(int an, const int32_t* a_seq, const int32_t* a_idr, int32_t* ord,
                                              int lane) {
    {
        for (int i0 = 0; i0 < an; i0 += 32) {
            int i = i0 + lane;
            uint64_t key = i < an ? (((uint64_t)(uint32_t)a_seq[i] << 32) | (uint32_t)a_idr[i]) : ~0ULL;
            int rank = 0;
            for (int j0 = 0; j0 < an; j0 += 32) {
                int jj = j0 + lane;
                uint64_t mine = jj < an ? (((uint64_t)(uint32_t)a_seq[jj] << 32) | (uint32_t)a_idr[jj]) : ~0ULL;
                int lim = an - j0 < 32 ? an - j0 : 32;
                for (int j = 0; j < lim; j++) {
                    uint64_t kj = __shfl_sync(FULLMASK, mine, j);
                    rank += kj < key;
                }
            }
            if (i < an) ord[rank] = i;
        }
    }
    __syncwarp();
}

// Alg. 3 greedy scan (select_decode_batch decode_sched.py:80-111) over the
// ordered active set.  Lanes test 32 consecutive candidates speculatively
// against the current (|B|, t_cur); the first admissible one is admitted and
// the scan restarts right after it; a round with no admissible lane rejects
// all remaining candidates of the window at once.  On a fully populated LUT
// the per-candidate column selection is computed once and each round only
// selects the rows for |B|+1.  Sets a_flag bit0 of admitted entries; returns
// |B| (0 = fallback).  Optional audit outputs (snapshot API): admitted order,
// delayed order, admission times.
__device__ __noinline__ int decode_scan_general(const LutMem* L, int an, const int32_t* ord, const int32_t* a_seq,
                                                int32_t* a_flag, double smin, double* tcur_out, int64_t* maxseq_out,
                                                int32_t* audit_batch, int32_t* audit_delayed, double* audit_times,
                                                int* n_delayed, int lane);

__device__ __forceinline__ int decode_scan(const LutMem* L, int an, const int32_t* ord, const int32_t* a_seq,
                                           int32_t* a_flag, double smin, double* tcur_out, int64_t* maxseq_out,
                                           int32_t* audit_batch, int32_t* audit_delayed, double* audit_times,
                                           int* n_delayed, int lane) {
    int b = 0;
    double tcur = 0.0;
    int64_t mseq = 0;
    if (L->full && an <= 32 && !audit_delayed) {
        // Dual-hypothesis rounds.  X: every candidate from s on is admitted, so
        // lane r tests with |B| = b + (r - s) and t_cur = x[r-1]; the first lane
        // whose test fails ends an admitted run (all X tests before it used the
        // true state).  If that lane is s itself (nothing admitted this round),
        // hypothesis Y (state unchanged) resolves the rest of the window: the
        // first Y-admissible lane is admitted, or the window is rejected whole.
        bool have = lane < an;
        int i = have ? ord[lane] : 0;
        int64_t seq = have ? a_seq[i] : 1;
        ColSel cs = lut_col(L, seq);
        int s = 0;
        while (s < an) {
            bool valid = have && lane >= s;
            int64_t bx = b + (lane - s) + 1;
            double x = valid ? lut_eval(L, lut_rows_nb(L, bx), cs) : 0.0;
            double xprev = __shfl_up_sync(FULLMASK, x, 1);
            double tprev = lane == s ? tcur : xprev;
            int64_t bprev = bx - 1;
            bool okx = valid && x <= smin && (bprev == 0 || xdiv((double)(bprev + 1), x) > xdiv((double)bprev, tprev));
            unsigned failm = __ballot_sync(FULLMASK, valid && !okx);
            int f = failm ? __ffs((int)failm) - 1 : an;
            if (valid && lane < f) a_flag[i] |= 1;
            if (f > s) {
                b += f - s;
                tcur = __shfl_sync(FULLMASK, x, f - 1);
                mseq = __shfl_sync(FULLMASK, seq, f - 1);
                s = f + 1;  // candidate f is rejected under the now-current state
                continue;
            }
            // nothing admitted: candidate s rejected; test the rest with the unchanged state
            RowSel rs = lut_rows(L, b + 1);
            double thr = b ? xdiv((double)b, tcur) : 0.0;
            bool vy = have && lane > s;
            double y = vy ? lut_eval(L, rs, cs) : 0.0;
            bool oky = vy && y <= smin && (b == 0 || xdiv((double)(b + 1), y) > thr);
            unsigned m = __ballot_sync(FULLMASK, oky);
            if (!m) break;
            int j = __ffs((int)m) - 1;
            if (lane == j) a_flag[i] |= 1;
            tcur = __shfl_sync(FULLMASK, y, j);
            mseq = __shfl_sync(FULLMASK, seq, j);
            b++;
            s = j + 1;
        }
        __syncwarp();
        *tcur_out = tcur;
        *maxseq_out = mseq;
        return b;
    }
    return decode_scan_general(L, an, ord, a_seq, a_flag, smin, tcur_out, maxseq_out, audit_batch, audit_delayed,
                               audit_times, n_delayed, lane);
}

__device__ __noinline__ int decode_scan_general(const LutMem* L, int an, const int32_t* ord, const int32_t* a_seq,
                                                int32_t* a_flag, double smin, double* tcur_out, int64_t* maxseq_out,
                                                int32_t* audit_batch, int32_t* audit_delayed, double* audit_times,
                                                int* n_delayed, int lane) {
    int b = 0;
    double tcur = 0.0;
    int64_t mseq = 0;
    int nd = 0;
    int s = 0;
    while (s < an) {
        int r = s + lane;
        bool valid = r < an;
        int i = valid ? ord[r] : 0;
        int64_t seq = valid ? a_seq[i] : 1;
        double ts = 0.0;
        bool cond = false;
        if (valid) {
            ts = lut_lookup(L, b + 1, seq);
            cond = ts <= smin && (b == 0 || xdiv((double)(b + 1), ts) > xdiv((double)b, tcur));
        }
        unsigned m = __ballot_sync(FULLMASK, cond);
        int j = m ? __ffs((int)m) - 1 : 32;
        int lim = an - s < 32 ? an - s : 32;
        if (audit_delayed) {
            if (lane < j && lane < lim) audit_delayed[nd + lane] = i;
            nd += (j < lim ? j : lim);
        }
        if (!m) { s += 32; continue; }
        if (lane == j) {
            a_flag[i] |= 1;
            if (audit_batch) { audit_batch[b] = i; audit_times[b] = ts; }
        }
        tcur = __shfl_sync(FULLMASK, ts, j);
        mseq = __shfl_sync(FULLMASK, seq, j);
        b++;
        s += j + 1;
        __syncwarp();
    }
    if (n_delayed) *n_delayed = nd;
    *tcur_out = tcur;
    *maxseq_out = mseq;
    return b;
}


// --------------------------------------------------------------- engine --
struct Ctx {
    slosim_batch_t B;  // by value: lives in the kernel parameter (constant) bank
    const LutMem* sched_tab;
    const LutMem* frozen_tab;
    const unsigned long long* dyn_n;  // non-null: the instance count is *dyn_n (instances deferred by the lane engine)
};

__device__ __forceinline__ int64_t arrival_of(const int64_t* Tarr, double fac, int p) {
    int64_t a = Tarr[p];
    return fac > 0 ? rint_i64(xmul((double)a, fac)) : a;
}

// Pending list insert keeping (tpf, id_rank) order (engine.py:358).
__device__ __noinline__ void pending_insert(const WS& w, int ph, int& pt, int64_t tpf, int32_t idr, int64_t ttr, int32_t pos,
                               int lane) {
    int64_t* pd_tpf = w.i64(PD_TPF);
    int64_t* pd_ttr = w.i64(PD_TTR);
    int32_t* pd_pos = w.i32(PD_POS);
    int32_t* pd_idr = w.i32(PD_IDR);
    int at = pt;
    if (pt > ph && (pd_tpf[pt - 1] > tpf || (pd_tpf[pt - 1] == tpf && pd_idr[pt - 1] > idr))) {
        int cnt = 0;
        for (int base = ph; base < pt; base += 32) {
            int k = base + lane;
            bool less = k < pt && (pd_tpf[k] < tpf || (pd_tpf[k] == tpf && pd_idr[k] < idr));
            cnt += __popc(__ballot_sync(FULLMASK, less));
        }
        at = ph + cnt;
        for (int hi = pt; hi > at; hi -= 32) {
            int lo = hi - 32 > at ? hi - 32 : at;
            int k = lo + lane;
            int64_t a = 0, b = 0;
            int32_t c = 0, d = 0;
            bool v = k < hi;
            if (v) { a = pd_tpf[k]; b = pd_ttr[k]; c = pd_pos[k]; d = pd_idr[k]; }
            __syncwarp();
            if (v) { pd_tpf[k + 1] = a; pd_ttr[k + 1] = b; pd_pos[k + 1] = c; pd_idr[k + 1] = d; }
            __syncwarp();
        }
    }
    if (lane == 0) { pd_tpf[at] = tpf; pd_ttr[at] = ttr; pd_pos[at] = pos; pd_idr[at] = idr; }
    pt++;
    __syncwarp();
}

// Exact nearest-rank selection (metrics.py:87-92) of the r-th smallest of
// n positive doubles by a bitwise radix descent on their IEEE bit patterns.
__device__ __noinline__ double radix_select(const double* v, int n, int64_t r, int lane) {
    uint64_t prefix = 0;
    int64_t need = r;
    for (int bit = 63; bit >= 0; bit--) {
        uint64_t hi_mask = bit == 63 ? 0ULL : (~0ULL << (bit + 1));
        int64_t c = 0;
        for (int k = lane; k < n; k += 32) {
            uint64_t x = (uint64_t)__double_as_longlong(v[k]);
            c += ((x & hi_mask) == prefix) && !((x >> bit) & 1ULL);
        }
        c = wsum64(c);
        if (need > c) { need -= c; prefix |= 1ULL << bit; }
    }
    return __longlong_as_double((long long)prefix);
}

__device__ void write_status(slosim_summary_t* out, int n, int status) {
    slosim_summary_t s = {};
    s.status = status;
    s.n = n;
    s.tps_p50 = __longlong_as_double(0x7ff8000000000000LL);
    s.tps_p90 = s.tps_p50;
    *out = s;
}

// ------------------------------------------------------ instance state --
// One active decode request held in a lane's registers (engine.py:374 _active).
struct Slot {
    int32_t pos, seq, idr, out, inp, miss, flag;  // flag bit1: TTFT met
    int64_t tf;                                   // t_first_token
};

// All per-instance state of one simulation.  It lives in registers inside the
// hot decode loop of simulate(); the rare per-request events (arrival,
// transfer, prefill completion/start, admission) are out-of-line functions
// that take it by reference, so their code stays out of the hot loop's
// instruction working set (the SM instruction cache is ~32 KB).
struct Sim {
    const slosim_batch_t* B;
    const slosim_instance_t* I;
    const slosim_profile_t* P;
    const int64_t* Tarr;
    const int32_t *Tinp, *Tout, *Thit, *Tidr;
    LutMem* L;
    WS w;
    double fac;
    int64_t ii, row0, tpot_slo, ttft_slo, kv_cap;
    int n, ppol;
    bool rows;
    // event state
    int ai, qh, qt, pf_k, trn, ph, pt, an, dc_prefix, finished;
    int64_t next_arr, pf_end, pf_dur, tr_min, dc_end, dc_dur, dc_bsz, dc_max, amax, kv, est_tok, est_busy;
    // active-set representation: register slots (lane i holds slot i, occupancy
    // mask `amask`, running batch `dc_mask`) while <= 32 requests are active,
    // the workspace arrays (A_*) otherwise
    bool regmode;
    uint32_t amask, dc_mask;
    // counters (l_*: per-lane partials, reduced at the end)
    int32_t c_ttft, c_tpot, c_e2e, ntps, max_q, max_a, l_tpot, l_e2e;
    int64_t misses, worst_wait, psteps, dsteps, v_dec, b_dec, v_pre, t_end, l_miss;
    uint64_t D;
    TraceW T;
    Pcg64 rng;  // decode noise (engine.py:191), drawn only when noise_eps > 0
    // the lane's slot, handed to out-of-line code by reference; the hot loop
    // keeps its own copy in registers (never address-taken)
    Slot sl;
    // results of the memory-mode decode handlers
    int sel_bsz, sel_nmem;
    int64_t sel_max;
    uint32_t sel_hash;
};


// Section profiling (debug builds with -DSLOSIM_PROF only): per-instance clock64
// totals of the loop sections, summed over instances into g_prof (slosim_prof_read).
#ifdef SLOSIM_PROF
__device__ unsigned long long g_prof[16];
#define PROF_DECL long long pf_acc[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0}; long long pf_t = clock64()
#define PROF_MARK(k) do { long long pf_n = clock64(); pf_acc[k] += pf_n - pf_t; pf_t = pf_n; } while (0)
#define PROF_COUNT(k, v) (pf_acc[k] += (v))
#define PROF_FLUSH() do { if (lane == 0) for (int pk = 0; pk < 10; pk++) atomicAdd(&g_prof[pk], (unsigned long long)pf_acc[pk]); } while (0)
#else
#define PROF_DECL
#define PROF_MARK(k)
#define PROF_COUNT(k, v)
#define PROF_FLUSH()
#endif

// 64-bit signed warp minimum from two 32-bit REDUX operations.
__device__ __forceinline__ int64_t wmin64_redux(int64_t v) {
    int hi = (int)(v >> 32);
    int mh = __reduce_min_sync(FULLMASK, hi);
    unsigned lo = hi == mh ? (unsigned)(uint64_t)v : 0xffffffffu;
    unsigned ml = __reduce_min_sync(FULLMASK, lo);
    return (int64_t)(((uint64_t)(uint32_t)mh << 32) | ml);
}

// register slots -> workspace arrays (compacted, slot order); running-batch membership
// moves to the flag bit0 representation of memory mode
__device__ __noinline__ void to_memory_mode(Sim& S, Slot& sl, int lane) {
    bool occ = (S.amask >> lane) & 1u;
    int d = __popc(S.amask & lanemask_lt(lane));
    if (occ) {
        S.w.i32(A_POS)[d] = sl.pos; S.w.i32(A_SEQ)[d] = sl.seq; S.w.i32(A_IDR)[d] = sl.idr; S.w.i32(A_OUT)[d] = sl.out;
        S.w.i32(A_INP)[d] = sl.inp; S.w.i32(A_MISS)[d] = sl.miss; S.w.i64(A_TFIRST)[d] = sl.tf;
        S.w.i32(A_FLAG)[d] = (sl.flag & 2) | (int)((S.dc_mask >> lane) & 1u);
    }
    __syncwarp();
    S.an = __popc(S.amask);
    S.dc_prefix = -1;
    S.regmode = false;
}

// workspace arrays -> register slots (when <= 32 are active and no decode step is running)
__device__ __noinline__ void to_register_mode(Sim& S, Slot& sl, int lane) {
    if (lane < S.an) {
        sl.pos = S.w.i32(A_POS)[lane]; sl.seq = S.w.i32(A_SEQ)[lane]; sl.idr = S.w.i32(A_IDR)[lane];
        sl.out = S.w.i32(A_OUT)[lane]; sl.inp = S.w.i32(A_INP)[lane]; sl.miss = S.w.i32(A_MISS)[lane];
        sl.flag = S.w.i32(A_FLAG)[lane] & 2; sl.tf = S.w.i64(A_TFIRST)[lane];
    }
    S.amask = S.an >= 32 ? 0xffffffffu : ((1u << S.an) - 1u);
    S.dc_mask = 0;
    S.regmode = true;
}

// ---- arrivals (engine.py:288-291): a contiguous run of the trace
template <bool FULL>
__device__ __noinline__ void on_arrivals(Sim& S, int64_t t, int lane) {
    int32_t* q_pos = S.w.i32(Q_POS);
    int32_t* q_rem = S.w.i32(Q_REM);
    int32_t* q_full = S.w.i32(Q_FULL);
    int32_t* q_inp = S.w.i32(Q_INP);
    int64_t* q_arr = S.w.i64(Q_ARR);
    for (;;) {
        int p = S.ai + lane;
        int64_t a = p < S.n ? arrival_of(S.Tarr, S.fac, p) : SLOSIM_INF64;
        unsigned m = __ballot_sync(FULLMASK, a == t);
        int cnt = __popc(m);
        if (lane < cnt) {
            int qi = S.qt + lane;
            int32_t inp = S.Tinp[p];
            int32_t full = inp - S.Thit[p];
            q_pos[qi] = p; q_arr[qi] = a; q_inp[qi] = inp; q_full[qi] = full; q_rem[qi] = full;
            if (FULL && S.T.buf) {
                int64_t o = S.T.used + 3 * lane;
                S.T.put(o, SLOSIM_EV_ARRIVAL); S.T.put(o + 1, t); S.T.put(o + 2, p);
            }
        }
        S.T.used += 3 * cnt;
        S.qt += cnt;
        S.ai += cnt;
        if (cnt < 32) { S.next_arr = __shfl_sync(FULLMASK, a, cnt); break; }
    }
    __syncwarp();
}

// ---- transfers due now that were pushed at earlier instants (engine.py:294-298)
template <bool FULL>
__device__ __noinline__ void on_transfers(Sim& S, int64_t t, int lane) {
    int64_t* tr_t = S.w.i64(TR_T);
    int64_t* tr_tpf = S.w.i64(TR_TPF);
    int32_t* tr_pos = S.w.i32(TR_POS);
    int m_keep = 0;
    for (int base = 0; base < S.trn; base += 32) {
        int k = base + lane;
        bool v = k < S.trn;
        int64_t tt = v ? tr_t[k] : 0, tpf = v ? tr_tpf[k] : 0;
        int32_t pos = v ? tr_pos[k] : 0;
        bool due = v && tt == t;
        unsigned dm = __ballot_sync(FULLMASK, due);
        unsigned km = __ballot_sync(FULLMASK, v && !due);
        __syncwarp();
        if (v && !due) {
            int o = m_keep + __popc(km & lanemask_lt(lane));
            tr_t[o] = tt; tr_tpf[o] = tpf; tr_pos[o] = pos;
        }
        m_keep += __popc(km);
        __syncwarp();
        while (dm) {
            int j = __ffs((int)dm) - 1;
            dm &= dm - 1;
            int64_t jtpf = __shfl_sync(FULLMASK, tpf, j);
            int32_t jpos = __shfl_sync(FULLMASK, pos, j);
            pending_insert(S.w, S.ph, S.pt, jtpf, S.Tidr[jpos], t, jpos, lane);
            if (FULL && S.T.buf && lane == 0) {
                S.T.put(S.T.used, SLOSIM_EV_TRANSFER_DONE); S.T.put(S.T.used + 1, t); S.T.put(S.T.used + 2, jpos);
            }
            S.T.used += 3;
        }
    }
    S.trn = m_keep;
    int64_t mn = SLOSIM_INF64;
    for (int k = lane; k < S.trn; k += 32) { int64_t tt = tr_t[k]; mn = tt < mn ? tt : mn; }
    S.tr_min = wmin64(mn);
}

// ---- prefill step completion (engine.py:327-350)
template <bool FULL>
__device__ __noinline__ void on_prefill_done(Sim& S, int64_t t, int lane) {
    const slosim_instance_t* I = S.I;
    int32_t* q_pos = S.w.i32(Q_POS);
    int32_t* q_rem = S.w.i32(Q_REM);
    int32_t* q_full = S.w.i32(Q_FULL);
    int32_t* q_inp = S.w.i32(Q_INP);
    int64_t* q_arr = S.w.i64(Q_ARR);
    const int32_t* pf_qidx = S.w.i32(PF_QIDX);
    const int32_t* pf_take = S.w.i32(PF_TAKE);
    const int pf_k = S.pf_k;
    int64_t tot = 0;
    uint64_t h = dstep(S.D, (uint64_t)t ^ 0xA5A5A5A5A5A5A5A5ULL);
    if (FULL && S.T.buf && lane == 0) {
        S.T.put(S.T.used, SLOSIM_EV_PREFILL_DONE); S.T.put(S.T.used + 1, t); S.T.put(S.T.used + 2, S.pf_dur);
        S.T.put(S.T.used + 3, pf_k);
    }
    S.T.used += 4;
    int64_t tw_transfers = S.T.used + pf_k;  // delay-0 TransferDone records follow the batch list
    int ncomp = 0, n0 = 0;
    for (int base = 0; base < pf_k; base += 32) {
        int e = base + lane;
        bool v = e < pf_k;
        int64_t take = 0;
        int32_t pos = 0, inp = 0;
        bool comp = false;
        uint64_t word = 0;
        if (v) {
            int qi = pf_qidx[e];
            take = pf_take[e];
            int32_t rem = q_rem[qi] - (int32_t)take;
            q_rem[qi] = rem;
            pos = q_pos[qi];
            inp = q_inp[qi];
            comp = rem == 0;
            word = ((uint64_t)(uint32_t)pos << 32) | (uint32_t)take;
            if (FULL) S.T.put(S.T.used + e, (int64_t)word);
        }
        tot += take;
        int lim = pf_k - base < 32 ? pf_k - base : 32;
        for (int j = 0; j < lim; j++) h = dstep(h, __shfl_sync(FULLMASK, word, j));
        // completed requests leave the queue and start their KV transfer, batch order
        int64_t delay = comp ? I->transfer_base_us + rint_i64(xmul((double)inp, I->transfer_per_token_us)) : 0;
        unsigned cm = __ballot_sync(FULLMASK, comp);
        unsigned zm = __ballot_sync(FULLMASK, comp && delay == 0);
        if (FULL && S.T.buf && comp && delay == 0) {
            int64_t o = tw_transfers + 3 * (n0 + __popc(zm & lanemask_lt(lane)));
            S.T.put(o, SLOSIM_EV_TRANSFER_DONE); S.T.put(o + 1, t); S.T.put(o + 2, pos);
        }
        n0 += __popc(zm);
        ncomp += __popc(cm);
        if (FULL && S.rows && comp) S.B->rows.t_prefill_finish[S.row0 + pos] = t;
        while (cm) {
            int j = __ffs((int)cm) - 1;
            cm &= cm - 1;
            int32_t jpos = __shfl_sync(FULLMASK, pos, j);
            int64_t jdel = __shfl_sync(FULLMASK, delay, j);
            if (jdel == 0) {
                pending_insert(S.w, S.ph, S.pt, t, S.Tidr[jpos], t, jpos, lane);
            } else {
                if (lane == 0) { S.w.i64(TR_T)[S.trn] = t + jdel; S.w.i64(TR_TPF)[S.trn] = t; S.w.i32(TR_POS)[S.trn] = jpos; }
                S.trn++;
                S.tr_min = t + jdel < S.tr_min ? t + jdel : S.tr_min;
            }
        }
    }
    S.T.used += pf_k + 3 * n0;
    tot = wsum64(tot);
    S.est_tok += tot;
    S.est_busy += S.pf_dur;
    S.psteps++;
    S.D = dstep(h, (uint64_t)S.pf_dur);
    __syncwarp();
    if (S.ppol == SLOSIM_PREFILL_FCFS) {
        S.qh += ncomp;  // FCFS completes a prefix of the queue
    } else if (ncomp) {
        int o = S.qh;
        for (int base = S.qh; base < S.qt; base += 32) {
            int qi = base + lane;
            bool v = qi < S.qt;
            int32_t pos = 0, rem = 0, full = 0, inp = 0;
            int64_t a = 0;
            if (v) { pos = q_pos[qi]; rem = q_rem[qi]; full = q_full[qi]; inp = q_inp[qi]; a = q_arr[qi]; }
            bool keep = v && rem > 0;
            unsigned km = __ballot_sync(FULLMASK, keep);
            __syncwarp();
            if (keep) {
                int d = o + __popc(km & lanemask_lt(lane));
                q_pos[d] = pos; q_rem[d] = rem; q_full[d] = full; q_inp[d] = inp; q_arr[d] = a;
            }
            o += __popc(km);
            __syncwarp();
        }
        S.qt = o;
    }
    S.pf_end = SLOSIM_INF64;
}

// ---- admission under the KV reservation (engine.py:355-375)
template <bool FULL>
__device__ __noinline__ void on_admit(Sim& S, Slot& sl, int64_t t, int lane) {
    const slosim_batch_t* B = S.B;
    while (S.pt > S.ph) {
        int k = S.ph + lane;
        bool v = k < S.pt;
        int32_t pos = v ? S.w.i32(PD_POS)[k] : 0;
        int32_t outl = v ? S.Tout[pos] : 0, inp = v ? S.Tinp[pos] : 0;
        int64_t need = (int64_t)inp + outl;
        int64_t held = (v && outl > 1) ? need : 0;
        int64_t excl = wscan_incl64(held, lane) - held;
        bool ok = v && S.kv + excl + need <= S.kv_cap;
        unsigned vm = __ballot_sync(FULLMASK, v);
        unsigned okm = __ballot_sync(FULLMASK, ok);
        unsigned fail = vm & ~okm;
        int cnt = fail ? __ffs((int)fail) - 1 : __popc(vm);
        bool adm = lane < cnt;
        int64_t ttr = adm ? S.w.i64(PD_TTR)[k] : 0;
        int32_t idr = adm ? S.w.i32(PD_IDR)[k] : 0;
        bool ttm = false;
        if (adm) {
            int64_t ttft = ttr - arrival_of(S.Tarr, S.fac, pos);
            ttm = ttft <= S.ttft_slo;
            if (FULL && S.T.buf) {
                int64_t o2 = S.T.used + 4 * lane;
                S.T.put(o2, SLOSIM_EV_ADMIT); S.T.put(o2 + 1, t); S.T.put(o2 + 2, pos); S.T.put(o2 + 3, ttr);
            }
            if (FULL && S.rows) {
                int64_t g = S.row0 + pos;
                B->rows.ttft_us[g] = ttft;
                B->rows.t_first_token[g] = ttr;
                if (outl == 1) {
                    B->rows.mean_tpot_us[g] = 0.0;
                    B->rows.decode_tps[g] = __longlong_as_double(0x7ff8000000000000LL);
                    B->rows.met_flags[g] = (uint8_t)((ttm ? 1 : 0) | 2 | (ttm ? 4 : 0));
                    B->rows.deadline_misses[g] = 0;
                    B->rows.t_last_token[g] = ttr;
                }
            }
        }
        S.T.used += 4 * cnt;
        S.c_ttft += __popc(__ballot_sync(FULLMASK, adm && ttm));
        unsigned one = __ballot_sync(FULLMASK, adm && outl == 1);
        S.c_tpot += __popc(one);
        S.c_e2e += __popc(__ballot_sync(FULLMASK, adm && outl == 1 && ttm));
        S.finished += __popc(one);
        unsigned dec = __ballot_sync(FULLMASK, adm && outl > 1);
        int ndec = __popc(dec);
        if (S.regmode && __popc(S.amask) + ndec > 32) to_memory_mode(S, sl, lane);
        if (S.regmode) {
            // the r-th admitted decoding request takes the r-th lowest free slot
            unsigned freem = ~S.amask;
            int fr = __popc(freem & lanemask_lt(lane));
            bool take = ((freem >> lane) & 1u) && fr < ndec;
            int src = ndec ? (int)__fns(dec, 0, (fr < ndec ? fr : 0) + 1) : 0;
            int32_t npos = __shfl_sync(FULLMASK, pos, src), ninp = __shfl_sync(FULLMASK, inp, src);
            int32_t nout = __shfl_sync(FULLMASK, outl, src), nidr = __shfl_sync(FULLMASK, idr, src);
            int64_t ntf = __shfl_sync(FULLMASK, ttr, src);
            bool nttm = __shfl_sync(FULLMASK, ttm, src);
            if (take) {
                sl.pos = npos; sl.seq = ninp; sl.idr = nidr; sl.out = nout; sl.inp = ninp; sl.miss = 0;
                sl.flag = nttm ? 2 : 0; sl.tf = ntf;
            }
            S.amask |= __ballot_sync(FULLMASK, take);
            S.an = __popc(S.amask);
        } else {
            if (adm && outl > 1) {
                int d = S.an + __popc(dec & lanemask_lt(lane));
                S.w.i32(A_POS)[d] = pos; S.w.i32(A_SEQ)[d] = inp; S.w.i32(A_IDR)[d] = idr;
                S.w.i32(A_OUT)[d] = outl; S.w.i32(A_INP)[d] = inp; S.w.i32(A_MISS)[d] = 0; S.w.i64(A_TFIRST)[d] = ttr;
                S.w.i32(A_FLAG)[d] = ttm ? 2 : 0;
            }
            S.an += ndec;
        }
        S.amax = __reduce_max_sync(FULLMASK, (int)(adm && outl > 1 && inp > S.amax ? (int64_t)inp : S.amax));
        S.kv += wsum64(adm ? held : 0);
        S.ph += cnt;
        __syncwarp();
        if (cnt < 32) break;
    }
}

// ---- start a prefill step (engine.py:307-325)
template <bool FULL>
__device__ __noinline__ void on_prefill_start(Sim& S, int64_t t, int lane) {
    const slosim_profile_t* P = S.P;
    int qlen = S.qt - S.qh;
    S.v_pre += qlen;
    S.max_q = qlen > S.max_q ? qlen : S.max_q;
    S.pf_k = prefill_select(S.ppol, S.w, S.qh, S.qt, S.I->chunk_budget, t, S.est_tok, S.est_busy, S.ttft_slo, lane);
    if (S.pf_k <= 0) return;
    // ground-truth duration: ordered sum of curve increments (engine.py:175-183)
    const int32_t* pf_qidx = S.w.i32(PF_QIDX);
    const int32_t* pf_take = S.w.i32(PF_TAKE);
    const int32_t* q_full = S.w.i32(Q_FULL);
    const int32_t* q_rem = S.w.i32(Q_REM);
    const int64_t* q_arr = S.w.i64(Q_ARR);
    const int n_curve = P->n_curve;
    double total = 0.0;
    int64_t ww = 0;
    for (int base = 0; base < S.pf_k; base += 32) {
        int e = base + lane;
        double term = 0.0;
        if (e < S.pf_k) {
            int qi = pf_qidx[e];
            int64_t take = pf_take[e];
            int64_t done = (int64_t)q_full[qi] - q_rem[qi];
            term = xsub(curve_at(n_curve, P->curve_x, P->curve_y, done + take),
                        curve_at(n_curve, P->curve_x, P->curve_y, done));
            if (done == 0) {  // first time scheduled (engine.py:322)
                int64_t wt = t - q_arr[qi];
                ww = wt > ww ? wt : ww;
                if (FULL && S.rows) S.B->rows.first_sched_us[S.row0 + S.w.i32(Q_POS)[qi]] = t;
            }
        }
        int lim = S.pf_k - base < 32 ? S.pf_k - base : 32;
        for (int j = 0; j < lim; j++) total = xadd(total, __shfl_sync(FULLMASK, term, j));
    }
    ww = wmax64(ww);
    S.worst_wait = ww > S.worst_wait ? ww : S.worst_wait;
    int64_t d = rint_i64(total);
    S.pf_dur = d < 1 ? 1 : d;
    S.pf_end = t + S.pf_dur;
}

// ---- finalize: aggregate (metrics.py:109-144)
template <bool FULL>
__device__ __noinline__ void on_finalize(Sim& S, long long c0, int lane) {
    const slosim_batch_t* B = S.B;
    double p50 = __longlong_as_double(0x7ff8000000000000LL), p90 = p50;
    __syncwarp();
    S.c_tpot += __reduce_add_sync(FULLMASK, (unsigned)S.l_tpot);
    S.c_e2e += __reduce_add_sync(FULLMASK, (unsigned)S.l_e2e);
    S.misses += wsum64(S.l_miss);
    if (S.ntps > 0) {
        int64_t r50 = (int64_t)ceil(xmul(50 / 100.0, (double)S.ntps));
        int64_t r90 = (int64_t)ceil(xmul(90 / 100.0, (double)S.ntps));
        p50 = radix_select(S.w.f64(TPS), S.ntps, r50 < 1 ? 1 : r50, lane);
        p90 = radix_select(S.w.f64(TPS), S.ntps, r90 < 1 ? 1 : r90, lane);
    }
    if (FULL && (B->flags & SLOSIM_F_EXPORT_LUT) && B->lut_out_sums) {
        const int FR = LUT_CELLS;
        const int nb = S.P->nb, ns = S.P->ns;
        for (int c = lane; c < FR; c += 32) {
            int i = c / SLOSIM_MAX_SEQ_BUCKETS, j = c % SLOSIM_MAX_SEQ_BUCKETS;
            bool in = i < nb && j < ns;
            B->lut_out_sums[S.ii * FR + c] = in ? S.L->sum[i * ns + j] : 0.0;
            B->lut_out_counts[S.ii * FR + c] = in ? S.L->cnt[i * ns + j] : 0;
        }
    }
    const TraceW& T = S.T;
    if (FULL && T.buf && lane == 0 && T.used + 2 <= T.cap) { T.buf[T.used] = SLOSIM_EV_END; T.buf[T.used + 1] = T.used + 2; }
    if (lane == 0) {
        slosim_summary_t s;
        s.status = (S.finished == S.n ? SLOSIM_OK : -1) | ((FULL && T.buf && T.used + 2 > T.cap) ? 0x100 : 0);
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
        s.sim_cycles = clock64() - c0;
        B->summaries[S.ii] = s;
    }
}

// ---- memory-mode decode step completion (> 32 active; engine.py:394-413)
template <bool FULL>
__device__ __noinline__ void on_decode_done_mem(Sim& S, Slot& sl, int64_t t, int lane) {
    uint32_t& s_out = S.sel_hash;
    int& nmem_out = S.sel_nmem;
    const WS& w = S.w;
    int32_t* a_pos = w.i32(A_POS);
    int32_t* a_seq = w.i32(A_SEQ);
    int32_t* a_idr = w.i32(A_IDR);
    int32_t* a_out = w.i32(A_OUT);
    int32_t* a_inp = w.i32(A_INP);
    int32_t* a_miss = w.i32(A_MISS);
    int32_t* a_flag = w.i32(A_FLAG);
    int64_t* a_tf = w.i64(A_TFIRST);
    uint32_t s = 0;
    int64_t kv_rel = 0, mx = 0;
    int o = 0;
    int64_t tw0 = S.T.used + 5;
    int nmem = 0;
    const int an = S.an, dc_prefix = S.dc_prefix;
    const int64_t tpot_slo = S.tpot_slo;
    for (int base = 0; base < an; base += 32) {
        int i = base + lane;
        bool v = i < an;
        int32_t flag = 0, pos = 0, seq = 0, idr = 0, outl = 0, inp = 0, miss = 0;
        int64_t tf = 0;
        if (v) {
            flag = a_flag[i]; pos = a_pos[i]; seq = a_seq[i]; idr = a_idr[i]; outl = a_out[i]; inp = a_inp[i];
            miss = a_miss[i]; tf = a_tf[i];
        }
        bool inb = v && (dc_prefix >= 0 ? i < dc_prefix : (flag & 1));
        bool retire = false, tpm = false;
        double tps = 0.0;
        if (inb) {
            seq += 1;
            int64_t ngen = seq - inp;
            s += member_hash((uint32_t)pos);
            if (t > tf + ngen * tpot_slo) miss++;  // deadline_misses metrics.py:57-69
            if (ngen == outl - 1) {
                retire = true;
                int64_t span = t - tf;
                double tpot = idiv(span, (int64_t)(outl - 1));
                tpm = tpot <= (double)tpot_slo;
                tps = xdiv((double)(outl - 1), xdiv((double)span, 1e6));
                kv_rel += (int64_t)inp + outl;
                if (FULL && S.rows) {
                    bool ttm = (flag & 2) != 0;
                    int64_t g = S.row0 + pos;
                    S.B->rows.mean_tpot_us[g] = tpot;
                    S.B->rows.decode_tps[g] = tps;
                    S.B->rows.met_flags[g] = (uint8_t)((ttm ? 1 : 0) | (tpm ? 2 : 0) | ((ttm && tpm) ? 4 : 0));
                    S.B->rows.deadline_misses[g] = miss;
                    S.B->rows.t_last_token[g] = t;
                }
            }
        }
        unsigned rmask = __ballot_sync(FULLMASK, retire);
        if (retire) {
            S.w.f64(TPS)[S.ntps + __popc(rmask & lanemask_lt(lane))] = tps;
            S.l_miss += miss;
            S.l_tpot += tpm;
            S.l_e2e += tpm && (flag & 2);
        }
        S.ntps += __popc(rmask);
        S.finished += __popc(rmask);
        if (FULL && S.T.buf) {
            unsigned bm = __ballot_sync(FULLMASK, inb);
            if (inb) S.T.put(tw0 + nmem + __popc(bm & lanemask_lt(lane)), pos);
            nmem += __popc(bm);
        }
        bool keep = v && !retire;
        unsigned km = __ballot_sync(FULLMASK, keep);
        __syncwarp();
        if (keep) {
            int d = o + __popc(km & lanemask_lt(lane));
            a_pos[d] = pos; a_seq[d] = seq; a_idr[d] = idr; a_out[d] = outl; a_inp[d] = inp;
            a_miss[d] = miss; a_tf[d] = tf; a_flag[d] = flag & ~1;
            mx = seq > mx ? seq : mx;
        }
        o += __popc(km);
        __syncwarp();
    }
    S.an = o;
    S.amax = __reduce_max_sync(FULLMASK, (int)mx);
    S.kv -= wsum64(kv_rel);
    s_out = __reduce_add_sync(FULLMASK, s);
    nmem_out = nmem;
    if (S.an <= 32) to_register_mode(S, sl, lane);
}

// ---- memory-mode decode start (> 32 active; engine.py:377-392, decode_sched.py:60-124)
template <int DP>
__device__ __noinline__ void on_decode_start_mem(Sim& S, int64_t t, int lane) {
    const WS& w = S.w;
    const int an = S.an;
    int& bsz = S.sel_bsz;
    int64_t& bmax = S.sel_max;
    bsz = an;
    bmax = S.amax;
    S.dc_prefix = an;
    if (DP == SLOSIM_DECODE_KAIROS_SLACK) {
        const int32_t* a_seq = w.i32(A_SEQ);
        const int32_t* a_inp = w.i32(A_INP);
        const int64_t* a_tf = w.i64(A_TFIRST);
        double fallback = lut_lookup(S.L, an, S.amax);
        int64_t sl = SLOSIM_INF64;
        for (int i = lane; i < an; i += 32) {
            int64_t ngen = (int64_t)a_seq[i] - a_inp[i];
            int64_t v = S.tpot_slo * (ngen + 1) - (t - a_tf[i]);
            sl = v < sl ? v : sl;
        }
        sl = wmin64(sl);
        double smin = xsub((double)sl, fallback);
        decode_order(an, a_seq, w.i32(A_IDR), w.i32(A_ORD), lane);
        double tcur;
        int64_t ms;
        int b = decode_scan(S.L, an, w.i32(A_ORD), a_seq, w.i32(A_FLAG), smin, &tcur, &ms, nullptr, nullptr, nullptr,
                            nullptr, lane);
        if (b > 0) { bsz = b; bmax = ms; S.dc_prefix = -1; }
    }
}

// Alg. 3 (select_decode_batch decode_sched.py:60-111) on register slots, fully
// populated LUT: dual-hypothesis rounds in rank space.  Lane i knows the rank
// of its slot in (seq_len, id) order and the lane of its rank predecessor.
// X: all candidates from rank s on are admitted (|B| = b + rank - s); the lowest
// failing rank ends the admitted run.  If rank s itself fails, Y tests the rest
// with the unchanged (|B|, t_cur) and admits the lowest admissible rank.
// Returns |B| (0 = fallback) and the admitted slot mask.
// The fallback cost lookup(|A|, max_seq) (decode_sched.py:75) is the first
// round's evaluation of the last-ranked slot (|B| = an at its seq_len = max_seq),
// so s_min = min(v) - that value is formed after the first evaluation.
template <bool G>
__device__ __forceinline__ int scan_slots(const LutMem* L, uint32_t amask, int an, const Slot& sl, int64_t vmin,
                                          uint32_t& adm, int64_t& mseq, int lane) {
    bool occ = (amask >> lane) & 1u;
    int rank = 0, pred = lane;
    uint64_t key = occ ? (((uint64_t)(uint32_t)sl.seq << 32) | (uint32_t)sl.idr) : ~0ULL;
    uint64_t best = 0;
    for (uint32_t m = amask; m; m &= m - 1) {
        int j = __ffs((int)m) - 1;
        uint64_t kj = __shfl_sync(FULLMASK, key, j);
        if (kj < key) {
            rank++;
            if (kj >= best) { best = kj; pred = j; }
        }
    }
    ColSel cs = lut_col<G>(L, occ ? sl.seq : 1);
    int b = 0, s = 0;
    double tcur = 0.0;
    adm = 0;
    mseq = 0;
    double x = occ ? lut_eval<G>(L, lut_rows_nb<G>(L, rank + 1), cs) : 0.0;
    const double smin = xsub((double)vmin, __shfl_sync(FULLMASK, x, __ffs((int)__ballot_sync(FULLMASK, occ && rank == an - 1)) - 1));
    bool fresh = true;
    while (s < an) {
        bool valid = occ && rank >= s;
        int64_t bx = b + (rank - s) + 1;
        if (!fresh) x = valid ? lut_eval<G>(L, lut_rows_nb<G>(L, bx), cs) : 0.0;
        fresh = false;
        double xprev = __shfl_sync(FULLMASK, x, pred);
        double tprev = rank == s ? tcur : xprev;
        int64_t bprev = bx - 1;
        bool okx = valid && x <= smin && (bprev == 0 || quot_gt((double)(bprev + 1), x, (double)bprev, tprev));
        int f = __reduce_min_sync(FULLMASK, (valid && !okx) ? rank : an);
        adm |= __ballot_sync(FULLMASK, valid && rank < f);
        if (f > s) {
            int lf = __ffs((int)__ballot_sync(FULLMASK, occ && rank == f - 1)) - 1;
            tcur = __shfl_sync(FULLMASK, x, lf);
            mseq = __shfl_sync(FULLMASK, sl.seq, lf);
            b += f - s;
            s = f + 1;  // rank f is rejected under the now-current state
            continue;
        }
        RowSel rs = lut_rows<G>(L, b + 1);
        bool vy = occ && rank > s;
        double y = vy ? lut_eval<G>(L, rs, cs) : 0.0;
        bool oky = vy && y <= smin && (b == 0 || quot_gt((double)(b + 1), y, (double)b, tcur));
        int g = __reduce_min_sync(FULLMASK, oky ? rank : an);
        if (g >= an) break;
        int lg = __ffs((int)__ballot_sync(FULLMASK, occ && rank == g)) - 1;
        adm |= 1u << lg;
        tcur = __shfl_sync(FULLMASK, y, lg);
        mseq = __shfl_sync(FULLMASK, sl.seq, lg);
        b++;
        s = g + 1;
    }
    return b;
}

// quot_gt (numerics.cuh) split for the hot scan: the product test decides
// unless the two products are within 2^-50 of each other (`tie`), in which
// case the caller divides exactly out of line.
__device__ __forceinline__ bool quot_gt_fast(double a, double x, double b, double y, bool& tie) {
    const double p = __dmul_rn(a, y), q = __dmul_rn(b, x);
    const bool gt = p > __dmul_rn(q, 1.0 + 0x1p-50);
    tie = !gt && !(p < __dmul_rn(q, 1.0 - 0x1p-50));
    return gt;
}
__device__ __noinline__ bool quot_gt_exact(double a, double x, double b, double y) {
    return __ddiv_rn(a, x) > __ddiv_rn(b, y);
}

// scan_slots on the power-of-two geometry (the benchmark's hot path), same
// decisions with fewer dependent steps: ranks are found two slots per
// iteration, and every round evaluates both hypotheses (X: the run from rank s
// on is admitted; Y: state unchanged) so that a round resolves with one
// uniform branch whichever applies.
// The (seq_len, id) ranks of the previous step are kept (rk_rank, rk_pred for
// the occupied-lane set rk_mask) and reused when the slot set is unchanged and
// every slot still compares above its rank predecessor: the old rank order is
// then still sorted, so the ranks are unchanged.
__device__ __forceinline__ int scan_geo(const LutMem* L, const Geo& g, const RowP* rowtab, uint32_t amask, int an,
                                        const Slot& sl, int64_t vmin, uint32_t& adm, int& mseq, int& rk_rank,
                                        int& rk_pred, uint32_t& rk_mask, int lane) {
    const bool occ = (amask >> lane) & 1u;
    const uint64_t key = occ ? (((uint64_t)(uint32_t)sl.seq << 32) | (uint32_t)sl.idr) : ~0ULL;
    int rank = rk_rank, pred = rk_pred;
    const uint64_t kp = __shfl_sync(FULLMASK, key, pred);
    if (rk_mask != amask || __any_sync(FULLMASK, occ && rank > 0 && !(kp < key))) {
        rank = 0;
        pred = lane;
        uint64_t best = 0;
        for (uint32_t m = amask; m;) {
            const int j1 = __ffs((int)m) - 1;
            m &= m - 1;
            const int j2 = m ? __ffs((int)m) - 1 : j1;
            m &= m - 1;
            const uint64_t k1 = __shfl_sync(FULLMASK, key, j1), k2 = __shfl_sync(FULLMASK, key, j2);
            const bool l1 = k1 < key, l2 = k2 < key && j2 != j1;
            rank += (int)l1 + (int)l2;
            if (l1 && k1 >= best) { best = k1; pred = j1; }
            if (l2 && k2 >= best) { best = k2; pred = j2; }
        }
        rk_rank = rank;
        rk_pred = pred;
        rk_mask = amask;
    }
    const ColSel cs = gcol(g, occ ? sl.seq : 1);
    int b = 0, s = 0;
    double tcur = 0.0;
    adm = 0;
    mseq = 0;
    double x = geval_p(L, g, rowtab[occ ? rank + 1 : 1], cs);
    const int llast = __ffs((int)__ballot_sync(FULLMASK, occ && rank == an - 1)) - 1;
    const double smin = xsub((double)vmin, __shfl_sync(FULLMASK, x, llast));
    bool first = true;
    for (;;) {
        const bool valid = occ && rank >= s;
        const int bx = b + (rank - s) + 1;
        if (!first) x = geval_p(L, g, rowtab[valid ? bx : 1], cs);
        first = false;
        const double xprev = __shfl_sync(FULLMASK, x, pred);
        const double tprev = rank == s ? tcur : xprev;
        const int bprev = bx - 1;
        bool tx;
        bool qx = quot_gt_fast((double)(bprev + 1), x, (double)bprev, tprev, tx);
        const bool ex = valid && x <= smin && bprev != 0 && tx;
        if (__any_sync(FULLMASK, ex))
            if (ex) qx = quot_gt_exact((double)(bprev + 1), x, (double)bprev, tprev);
        const bool okx = valid && x <= smin && (bprev == 0 || qx);
        const int f = __reduce_min_sync(FULLMASK, (valid && !okx) ? rank : an);
        int last, cnt;
        double tsel;
        if (f > s) {  // X: ranks [s, f) admitted, rank f rejected under the new state
            last = f - 1;
            cnt = f - s;
            tsel = x;
            adm |= __ballot_sync(FULLMASK, valid && rank < f);
        } else {      // Y: rank s rejected; the lowest rank admissible under the unchanged state
            const bool vy = occ && rank > s;
            const double y = geval_p(L, g, rowtab[b + 1], cs);
            bool ty;
            bool qy = quot_gt_fast((double)(b + 1), y, (double)b, tcur, ty);
            const bool ey = vy && y <= smin && b != 0 && ty;
            if (__any_sync(FULLMASK, ey))
                if (ey) qy = quot_gt_exact((double)(b + 1), y, (double)b, tcur);
            const bool oky = vy && y <= smin && (b == 0 || qy);
            const int gy = __reduce_min_sync(FULLMASK, oky ? rank : an);
            if (gy >= an) break;  // the window is rejected
            last = gy;
            cnt = 1;
            tsel = y;
            adm |= __ballot_sync(FULLMASK, occ && rank == gy);
        }
        const int ll = __ffs((int)__ballot_sync(FULLMASK, occ && rank == last)) - 1;
        tcur = __shfl_sync(FULLMASK, tsel, ll);
        mseq = __shfl_sync(FULLMASK, sl.seq, ll);
        s = f > s ? f + 1 : last + 1;
        b += cnt;
        if (s >= an) break;
    }
    return b;
}

// Ground-truth decode step for frozen (file-backed) profiles and/or noise
// (engine.py:185-192): out of the hot loop, which then carries neither the
// general LUT lookup nor the PCG64 state.
__device__ __noinline__ double gt_decode_cold(Sim& S, const LutMem* frozen, int64_t bsz, int64_t bmax) {
    const slosim_profile_t* P = S.P;
    double val = P->gt_frozen ? lut_lookup(frozen, bsz, bmax)
                              : decode_formula(P->n_base, P->base_x, P->base_y, P->gamma, bsz, bmax);
    double eps = P->noise_eps;
    if (eps > 0) val = xmul(val, pcg_uniform(S.rng, xsub(1.0, eps), xadd(1.0, eps)));
    return val;
}

// request_metrics (metrics.py:72-84) for the requests retiring at t, one per
// lane with `retire` set; appends their decode tps at tps_buf[ntps..] in lane
// order and returns the warp's released KV reservation.
template <bool FULL>
__device__ __noinline__ int64_t on_retire(Sim& S, const Slot sl, int64_t t, bool retire, int ntps, int lane) {
    unsigned rmask = __ballot_sync(FULLMASK, retire);
    int64_t kv_rel = 0;
    if (retire) {
        int64_t span = t - sl.tf;
        double tpot = idiv(span, (int64_t)(sl.out - 1));
        bool tpm = tpot <= (double)S.tpot_slo;
        double tps = xdiv((double)(sl.out - 1), xdiv((double)span, 1e6));
        kv_rel = (int64_t)sl.inp + sl.out;
        if (FULL && S.rows) {
            bool ttm = (sl.flag & 2) != 0;
            int64_t g = S.row0 + sl.pos;
            S.B->rows.mean_tpot_us[g] = tpot;
            S.B->rows.decode_tps[g] = tps;
            S.B->rows.met_flags[g] = (uint8_t)((ttm ? 1 : 0) | (tpm ? 2 : 0) | ((ttm && tpm) ? 4 : 0));
            S.B->rows.deadline_misses[g] = sl.miss;
            S.B->rows.t_last_token[g] = t;
        }
        S.w.f64(TPS)[ntps + __popc(rmask & lanemask_lt(lane))] = tps;
        S.l_miss += sl.miss;
        S.l_tpot += tpm;
        S.l_e2e += tpm && (sl.flag & 2);
    }
    return wsum64(kv_rel);
}

// DecodeStepLUT.lookup (costmodel.py:157-187) on the full power-of-two grid from the cell means,
// with cell c0's mean replaced by m0 (ff_verify): the np.interp slope of a column pair is formed
// from the means exactly as lut_build/gupdate store it, RN((m[c+1] - m[c]) * 2^-wsh), and the
// rows combine as in geval_p.
__device__ __forceinline__ double ff_row(const double* M, const Geo& g, double inv_w, int r, const ColSel& cs, int c0,
                                         double m0) {
    const int k = r * g.ns + cs.c;
    const double a = k == c0 ? m0 : M[k];
    if (cs.dx == 0.0) return a;
    const double b = k + 1 == c0 ? m0 : M[k + 1];
    return xadd(xmul(xsub(b, a), cs.dx * inv_w), a);  // = slope * dx, slope = (b - a) * 2^-wsh (exact scaling)
}
__device__ __forceinline__ double ff_lookup(const LutMem* L, const Geo& g, double inv_w, const RowP& rp, int seq,
                                            int c0, double m0) {
    const ColSel cs = gcol(g, seq);
    const double v1 = ff_row(L->mean, g, inv_w, rp.r1, cs, c0, m0);
    const double v2 = rp.r2 == rp.r1 ? v1 : ff_row(L->mean, g, inv_w, rp.r2, cs, c0, m0);
    return xadd(v1, xmul(xsub(v2, v1), rp.wgt));
}
__device__ __forceinline__ bool ff_quot_gt(double a, double x, double b, double y) {
    bool tie;
    const bool gt = quot_gt_fast(a, x, b, y, tie);
    return tie ? quot_gt_exact(a, x, b, y) : gt;
}

// ff_steps<.., V = true>: lane k runs select_decode_batch for the step started at e_k (after
// completions 0..k of the run, each of them batching the whole active set A) and returns the batch
// as a mask over A's (seq_len, id) ranks: all of A when the greedy scan admits every candidate or
// none (the fallback), 0 when the run's LUT cell leaves the exact integer range.  `e` is this
// lane's e_k; `rank` the lane's rank among A at time t (scan_geo's cache).
__device__ __noinline__ uint32_t ff_verify(const Sim& S, const Slot& sl, int64_t t, int64_t e, int lane,
                                           const RowP* rowtab, int rank) {
    const bool occ = (S.amask >> lane) & 1u;
    const int an = S.an;
    const int64_t tpot = S.tpot_slo;
    // the active set's sequence lengths in rank order (per-warp shared memory)
    __shared__ int32_t ff_seq[4][32];
    int32_t* rs = ff_seq[threadIdx.x >> 5];
    __syncwarp();
    if (occ) rs[rank] = sl.seq;
    // slack (decode_sched.py:36-57) at step k+1: tpot*(n_gen + k + 2) - (e_k - t_first)
    const int64_t v0 = wmin64_redux(occ ? tpot * ((int64_t)(sl.seq - sl.inp) + 1) + sl.tf : SLOSIM_INF64);
    __syncwarp();
    const LutMem* L = S.L;
    const Geo g = geo_of(L);
    const double inv_w = pow2_neg(g.wsh);
    const int kk = lane + 1;  // completions applied before step k+1 starts
    // cell c0 after kk completions: exact integer sum (checked integral by the caller's commit) over count
    const int i0 = min(gbidx(an), g.nb - 1);
    const int j0 = min((int)((S.dc_max + (1 << g.wsh) - 1) >> g.wsh) - 1, g.ns - 1);
    const int c0 = i0 * g.ns + j0;
    const double s0 = L->sum[c0];
    if (!(s0 == rint(s0) && fabs(s0) + (double)(e - t) < 0x1p53)) return 0u;
    const double m0 = xdiv(xadd(s0, (double)(e - t)), (double)(L->cnt[c0] + kk));
    const int64_t vmin = v0 + (int64_t)kk * tpot - e;
    const double fb = ff_lookup(L, g, inv_w, rowtab[an], (int)S.amax + kk, c0, m0);
    const double smin = xsub((double)vmin, fb);
    // the greedy scan in (seq_len, id) order (decode_sched.py:84-95)
    const uint32_t full = an >= 32 ? ~0u : (1u << an) - 1u;
    uint32_t adm = 0;
    int b = 0;
    double tcur = 0.0;
#pragma unroll 1
    for (int r = 0; r < an; r++) {
        const double x = ff_lookup(L, g, inv_w, rowtab[b + 1], rs[r] + kk, c0, m0);
        if (x <= smin && (b == 0 || ff_quot_gt((double)(b + 1), x, (double)b, tcur))) {
            adm |= 1u << r;
            b++;
            tcur = x;
        }
    }
    return b == 0 ? full : adm;  // nothing admitted: the fallback decodes all of A
}

// Decode steps between rare events, applied in bulk.  Under continuous
// batching (decode_sched.py:114-124) the batch is the whole active set; under
// Alg. 3 with a single active request it is that request whatever the scan
// decides.  Either way consecutive decode steps (engine.py:377-413) differ
// only in max_seq (+1 per step) until an arrival, transfer or prefill
// completion arrives or a member retires.  Lane k evaluates the ground-truth
// duration of the k-th step from now (k = 0: the step just started), a warp
// scan gives the step end times, and the leading run of m steps that end
// strictly before the next rare event with no member retiring is applied at
// once: per-token deadlines (metrics.py:57-69) and the decision digest, folded
// in step order, and (LUTUPD) the m DecodeStepLUT.update calls
// (costmodel.py:118-128).  Nothing reads the LUT inside the run, and the m
// steps are kept to one cell, so the updates collapse into one: the cell sum
// grows by the exact integer total (the cell sum must be an integer below
// 2^53, so every intermediate f64 sum is exact in any grouping), the count by
// m, and the mean and slopes are recomputed once from the final sums.  Step m
// is left in progress exactly as the loop would have started it.  Returns m.
// Preconditions (checked by the caller): register mode, plain formula ground
// truth, no per-step trace, no pending prefill start; LUTUPD: a fully
// populated LUT and either one active request or (V) a batch that is the whole
// active set.
//
// V (Alg. 3 with |A| > 1, the step just started batching all of A): the
// decision of every later step in the run is verified instead of assumed.
// Lane k re-runs select_decode_batch (decode_sched.py:60-111) for step k+1 as
// the loop would see it at time e_k: every request advanced by k+1 tokens (so
// the (seq_len, id) order is unchanged), the slack minimum shifted by
// (k+1)*tpot - (e_k - t), and the LUT as the k+1 earlier completions leave it
// (only cell c0 differs: its exact integer sum over its count; lookups read
// means and form the np.interp slopes as the stored slopes are formed).  The
// step batches A again iff the greedy scan admits every candidate, or none
// (the fallback).  The run is the leading prefix of steps whose completion is
// pure and whose successor's decision is verified.
template <bool LUTUPD, bool G, bool V = false>
__device__ __noinline__ int ff_steps(Sim& S, Slot& sl, int64_t t, int lane, const RowP* rowtab = nullptr,
                                     int rank = 0) {
    const bool occ = (S.amask >> lane) & 1u;  // every active request is in the batch
    const int64_t ng = (int64_t)sl.seq - sl.inp;  // tokens generated before step 0
    const int r = __reduce_min_sync(FULLMASK, occ ? (int)(sl.out - 2 - ng) : 0x7fffffff);
    if (r < 1) return 0;
    int64_t tr = S.next_arr;
    tr = S.tr_min < tr ? S.tr_min : tr;
    tr = S.pf_end < tr ? S.pf_end : tr;
    const int64_t bsz = S.dc_bsz, bmax = S.dc_max;
    const slosim_profile_t* P = S.P;
    int64_t d = rint_i64(decode_formula(P->n_base, P->base_x, P->base_y, P->gamma, bsz, bmax + lane));
    d = d < 1 ? 1 : d;
    const int64_t e = t + wscan_incl64(d, lane);
    bool pure = e < tr && lane < r && lane < 31;
    LutMem* L = S.L;
    if (LUTUPD) {
        // the LUT cell of step k (bucket of (bsz, max_seq)); j is nondecreasing in k
        const int ns = L->ns;
        int j = G ? geo_sidx(L, bmax + lane) : lut_sidx(L, bmax + lane);
        j = j < ns - 1 ? j : ns - 1;
        const int j0 = __shfl_sync(FULLMASK, j, 0);  // unconditional: every lane takes part
        pure = pure && j == j0;
    }
    uint32_t vmask = 0;
    bool tail = false;
    int m;
    if (V) {  // every lane takes part in the verification's collectives
        vmask = ff_verify(S, sl, t, e, lane, rowtab, rank);
        const uint32_t full = S.an >= 32 ? ~0u : (1u << S.an) - 1u;
        // the leading run of verified steps; when the step after it batches a proper subset of A
        // and the run's last completion is pure, that step is started here too (the tail)
        const unsigned pm = __ballot_sync(FULLMASK, pure && vmask == full);
        m = __ffs((int)~pm) - 1;
        tail = __shfl_sync(FULLMASK, pure && vmask != 0u && vmask != full, m & 31) && m < 31;
        vmask = __shfl_sync(FULLMASK, vmask, m & 31);
        m += tail ? 1 : 0;
    } else {
        // end times increase and the other bounds are thresholds, so the pure steps form a prefix
        m = __popc(__ballot_sync(FULLMASK, pure));
    }
    if (m <= 0) return 0;
    if (LUTUPD) {
        const int64_t dsum = wsum64(lane < m ? d : 0);
        const int nb = L->nb, ns = L->ns;
        int i = G ? geo_bidx(bsz) : lut_bidx(L, bsz), j = G ? geo_sidx(L, bmax) : lut_sidx(L, bmax);
        i = i < nb - 1 ? i : nb - 1;
        j = j < ns - 1 ? j : ns - 1;
        const double s0 = L->sum[i * ns + j];
        if (!(s0 == rint(s0) && fabs(s0) + (double)dsum < 0x1p53)) return 0;
        lut_update_warp<G>(L, bsz, bmax, dsum, lane, m);
        __syncwarp();
    }
    const uint32_t s = __reduce_add_sync(FULLMASK, occ ? member_hash((uint32_t)sl.pos) : 0u);
    const uint64_t mid = ((uint64_t)s << 32) | (uint32_t)bsz;
    const int64_t tpot = S.tpot_slo;
    const int64_t c = sl.tf + ng * tpot;
    uint64_t D = S.D;
    int miss = 0;
#pragma unroll 1
    for (int k = 0; k < m; k++) {
        const int64_t ek = __shfl_sync(FULLMASK, e, k);
        const int64_t dk = __shfl_sync(FULLMASK, d, k);
        miss += ek > c + (int64_t)(k + 1) * tpot;
        D = dstep(D, (uint64_t)ek ^ 0x5A5A5A5A5A5A5A5AULL);
        D = dstep(D, mid);
        D = dstep(D, (uint64_t)dk);
    }
    if (occ) { sl.seq += m; sl.miss += miss; }
    S.D = D;
    S.amax += m;
    if (V && tail) {
        // step m batches the ranks in vmask: membership, its max_seq and ground-truth duration
        const bool in = occ && ((vmask >> rank) & 1u);
        S.dc_mask = __ballot_sync(FULLMASK, in);
        const int tb = __popc(vmask);
        const int tmax = __reduce_max_sync(FULLMASK, in ? sl.seq : 0);
        int64_t td = rint_i64(decode_formula(P->n_base, P->base_x, P->base_y, P->gamma, tb, tmax));
        td = td < 1 ? 1 : td;
        S.dc_end = __shfl_sync(FULLMASK, e, m - 1) + td;
        S.dc_dur = td;
        S.dc_bsz = tb;
        S.dc_max = tmax;
        return m;
    }
    S.dc_end = __shfl_sync(FULLMASK, e, m);
    S.dc_dur = __shfl_sync(FULLMASK, d, m);
    S.dc_max = bmax + m;
    return m;
}

// Verified multi-step fast-forward of Alg. 3 runs: a latency-build feature.  In the throughput
// build the other resident warps use the issue slots the verifications cost (configs 3 and 4:
// 213 -> 230 ms and 673 -> 727 ms with it, attempts gated by FF_MIN_STREAK; 265 and 1045 ms
// ungated), in the latency build nothing else would (config 2: 6.78 -> 4.07 s, config 1: 83 ->
// 50 ms).  SLOSIM_FF_MULTI_ALL compiles it into the throughput build too (experiments).
#if defined(SLOSIM_NO_FF_MULTI) || ((!defined(SLOSIM_MIN_BLOCKS) || SLOSIM_MIN_BLOCKS != 1) && !defined(SLOSIM_FF_MULTI_ALL))
#define FF_MULTI false
#else
#define FF_MULTI true
#endif

#ifndef FF_MIN_STREAK
#define FF_MIN_STREAK 3
#endif

#ifdef SLOSIM_NO_FF_KAIROS
#define FF_KAIROS false
#else
#define FF_KAIROS true
#endif

#ifdef SLOSIM_NO_SKIP1
#define SKIP_SINGLE(an) true
#else
#define SKIP_SINGLE(an) ((an) > 1)
#endif

// Descriptor validation (include/slosim_b200.h): everything the engine indexes
// with must lie inside the buffers the batch describes.
__device__ __noinline__ bool instance_ok(const slosim_batch_t* B, const slosim_instance_t* I, const LutMem* tabs) {
    const int64_t n = I->n_requests, off = I->trace_offset;
    bool ok = n >= 0 && n <= B->max_requests && I->profile_id >= 0 && I->profile_id < B->n_profiles &&
              off >= 0 && off <= B->traces.n_total - n && I->prefill_policy >= 0 && I->prefill_policy <= 2 &&
              I->decode_policy >= 0 && I->decode_policy <= 1 && I->chunk_budget >= 1 && I->ttft_slo_us > 0 &&
              I->tpot_slo_us > 0 && I->kv_capacity_tokens >= 1 && I->transfer_base_us >= 0 &&
              I->transfer_per_token_us >= 0.0 && !(I->rescale_factor != I->rescale_factor);
    if (ok) ok = tabs[I->profile_id].bad == 0;
    if (ok && (B->flags & SLOSIM_F_ROWS))
        ok = I->row_offset >= 0 && (B->rows_capacity <= 0 || I->row_offset <= B->rows_capacity - n);
    if (ok && B->trace_buf && I->trace_buf_offset >= 0)
        ok = I->trace_buf_words >= 0 &&
             (B->trace_buf_capacity <= 0 || I->trace_buf_offset <= B->trace_buf_capacity - I->trace_buf_words);
    return ok;
}

// DP: decode policy (compile-time), FULL: event trace / per-request rows / LUT
// export compiled in, G: power-of-two LUT geometry.  The throughput path runs
// simulate<DP, false, G>, whose hot loop carries no tracing or row-output code.
#ifdef SLOSIM_SIM_NOINLINE
#define SIM_INLINE __noinline__
#else
#define SIM_INLINE __forceinline__
#endif
template <int DP, bool FULL, bool G>
__device__ SIM_INLINE void simulate(const Ctx& cx, int64_t ii, const WS& w, int lane) {
    const long long c0 = clock64();
    Sim S;
    S.B = &cx.B;
    S.ii = ii;
    S.I = S.B->instances + ii;
    const slosim_instance_t* I = S.I;
    S.n = I->n_requests;
    const int pid = I->profile_id;
    const int64_t off = I->trace_offset;
    // C-ABI contract: a malformed descriptor gets SLOSIM_EINVAL and touches nothing else
    if (!instance_ok(S.B, I, cx.sched_tab)) {
        if (lane == 0) write_status(S.B->summaries + ii, S.n, SLOSIM_EINVAL);
        return;
    }
    S.P = S.B->profiles + pid;
    S.Tarr = S.B->traces.arrival_us + off;
    S.Tinp = S.B->traces.input_len + off;
    S.Tout = S.B->traces.output_len + off;
    S.Thit = S.B->traces.prefix_hit_len + off;
    S.Tidr = S.B->traces.id_rank + off;
    S.fac = I->rescale_factor;
    S.rows = FULL && (S.B->flags & SLOSIM_F_ROWS) != 0;
    S.tpot_slo = I->tpot_slo_us;
    S.ttft_slo = I->ttft_slo_us;
    S.kv_cap = I->kv_capacity_tokens;
    S.ppol = I->prefill_policy;
    S.row0 = I->row_offset;
    S.w = w;

    // ---- Simulation.__init__ checks (engine.py:218-232)
    int64_t worst = 0;
#pragma unroll 1
    for (int p = lane; p < S.n; p += 32) {
        int64_t need = (int64_t)S.Tinp[p] + S.Tout[p];
        worst = need > worst ? need : worst;
    }
    worst = wmax64(worst);
    const LutMem* ST = cx.sched_tab + pid;
    if (worst > S.kv_cap || ST->rowmask == 0) {
        if (lane == 0) write_status(S.B->summaries + ii, S.n, SLOSIM_ECONFIG);
        return;
    }
    const bool use_lut = DP == SLOSIM_DECODE_KAIROS_SLACK || (S.B->flags & (SLOSIM_F_ALWAYS_LUT | SLOSIM_F_EXPORT_LUT));
    S.L = w.lut();
    LutMem* L = S.L;
    if (use_lut) lut_copy(L, ST, lane);
    bool lut_full = use_lut && L->full != 0;
    int rk_rank = 0, rk_pred = lane;  // cached slot ranks of the kairos scan (scan_geo)
    uint32_t rk_mask = 0;
    int ff_streak = 0;
    const Geo geo = G ? geo_of(ST) : Geo{0, 0, 0};
    // row selections of batch sizes 1..32 for the register-mode scan (per warp)
    __shared__ RowP row_tabs[4][33];
    RowP* const rowtab = row_tabs[threadIdx.x >> 5];
    if (G) {
        rowtab[lane + 1] = rowp_of(geo, lane + 1);
        if (lane == 0) rowtab[0] = rowp_of(geo, 1);
        __syncwarp();
    }
    S.est_tok = S.P->est_tokens;
    S.est_busy = S.P->est_busy_us;
    S.rng = Pcg64{I->rng_state_hi, I->rng_state_lo, I->rng_inc_hi, I->rng_inc_lo};
    S.T = TraceW{nullptr, 0, 0};
    if (FULL && S.B->trace_buf && I->trace_buf_offset >= 0) {
        S.T.buf = S.B->trace_buf + I->trace_buf_offset;
        S.T.cap = I->trace_buf_words;
    }
    S.ai = 0;
    S.next_arr = S.n > 0 ? arrival_of(S.Tarr, S.fac, 0) : SLOSIM_INF64;
    S.qh = S.qt = S.pf_k = S.trn = S.ph = S.pt = S.an = S.finished = 0;
    S.pf_end = S.tr_min = S.dc_end = SLOSIM_INF64;
    S.pf_dur = S.dc_dur = S.dc_bsz = S.dc_max = S.amax = S.kv = 0;
    S.dc_prefix = -1;
    S.regmode = true;
    S.amask = S.dc_mask = 0;
    S.c_ttft = S.c_tpot = S.c_e2e = S.ntps = S.max_q = S.max_a = S.l_tpot = S.l_e2e = 0;
    S.misses = S.worst_wait = S.psteps = S.dsteps = S.v_dec = S.b_dec = S.v_pre = S.t_end = S.l_miss = 0;
    S.D = 0;
    Slot sl{0, 0, 0, 0, 0, 0, 0, 0};
    const int64_t tpot_slo = S.tpot_slo;
    const bool gt_plain = S.P->gt_frozen == 0 && S.P->noise_eps <= 0.0;
    // one- or two-anchor ground-truth decode curve staged in shared memory (per warp)
    __shared__ GtLine gt_lines[4];
    GtLine* const gtl = gt_lines + (threadIdx.x >> 5);
    bool gt_fast = false;
    if (lane == 0) gt_fast = gt_line_make(S.P->n_base, S.P->base_x, S.P->base_y, S.P->gamma, *gtl);
    gt_fast = __shfl_sync(FULLMASK, gt_fast, 0);
    __syncwarp();

    // hot state in registers; synced with S around the (rare) out-of-line calls.
    // The rare-event clocks (next arrival, prefill end, first transfer) and the
    // queue/pending cursors change only inside those calls, so the hot loop
    // keeps just their minimum (t_rare) and two derived flags.
    int64_t dc_end, dc_dur, dc_bsz, dc_max, amax, kv, t_end = 0;
    int64_t t_rare;
    bool adm_pend, pf_wait;
    int an, ntps, finished;
    uint32_t amask, dc_mask;
    bool regmode;
    uint64_t D;
    int64_t dsteps = 0, v_dec = 0, b_dec = 0;
    int32_t max_a = 0;
#define SIM_SYNC_IN()                                                                                          \
    dc_end = S.dc_end; dc_dur = S.dc_dur; dc_bsz = S.dc_bsz; dc_max = S.dc_max; amax = S.amax; kv = S.kv;     \
    an = S.an; ntps = S.ntps; finished = S.finished; amask = S.amask; dc_mask = S.dc_mask;                    \
    regmode = S.regmode; D = S.D;                                                                              \
    t_rare = S.next_arr < S.pf_end ? S.next_arr : S.pf_end;                                                    \
    t_rare = S.tr_min < t_rare ? S.tr_min : t_rare;                                                            \
    adm_pend = S.pt > S.ph;                                                                                    \
    pf_wait = S.pf_end == SLOSIM_INF64 && S.qt > S.qh
#define SIM_SYNC_OUT()                                                                                         \
    S.dc_end = dc_end; S.dc_dur = dc_dur; S.dc_bsz = dc_bsz; S.dc_max = dc_max; S.amax = amax; S.kv = kv;     \
    S.an = an; S.ntps = ntps; S.finished = finished; S.amask = amask; S.dc_mask = dc_mask;                    \
    S.regmode = regmode; S.D = D
    SIM_SYNC_IN();
    PROF_DECL;

    for (;;) {
        PROF_MARK(5);
        const int64_t t = dc_end < t_rare ? dc_end : t_rare;
        if (t == SLOSIM_INF64) break;
        t_end = t;

        // rare events (a few per request) run out of line, in the reference's order
        if (__builtin_expect(t_rare == t, 0)) {
            SIM_SYNC_OUT();
            if (S.next_arr == t) on_arrivals<FULL>(S, t, lane);
            if (S.tr_min == t) on_transfers<FULL>(S, t, lane);
            if (S.pf_end == t) on_prefill_done<FULL>(S, t, lane);
            SIM_SYNC_IN();
        }
        PROF_MARK(0);

        // ---- decode step completion (engine.py:394-413): the hot path
        if (dc_end == t) {
            uint32_t s = 0;
            int nmem = 0;
            if (__builtin_expect(regmode, 1)) {
                // branch-free member update: token time, per-token deadline
                // (deadline_misses metrics.py:57-69), retirement test
                const bool inb = (dc_mask >> lane) & 1u;
                sl.seq += inb ? 1 : 0;
                const int ngen = sl.seq - sl.inp;
                const uint32_t hsh = inb ? member_hash((uint32_t)sl.pos) : 0u;
                sl.miss += (inb && t > sl.tf + (int64_t)ngen * tpot_slo) ? 1 : 0;
                const bool retire = inb && ngen == sl.out - 1;
                unsigned rmask = __ballot_sync(FULLMASK, retire);
                if (__builtin_expect(rmask != 0, 0)) {
                    kv -= on_retire<FULL>(S, sl, t, retire, ntps, lane);
                    ntps += __popc(rmask);
                    finished += __popc(rmask);
                    amask &= ~rmask;
                }
                if (FULL && S.T.buf) {
                    if (inb) S.T.put(S.T.used + 5 + __popc(dc_mask & lanemask_lt(lane)), sl.pos);
                    nmem = __popc(dc_mask);
                }
                amax = __reduce_max_sync(FULLMASK, ((amask >> lane) & 1u) ? sl.seq : 0);
                s = __reduce_add_sync(FULLMASK, hsh);
                an = __popc(amask);
            } else {
                SIM_SYNC_OUT();
                S.sl = sl;
                on_decode_done_mem<FULL>(S, S.sl, t, lane);
                sl = S.sl;
                s = S.sel_hash;
                nmem = S.sel_nmem;
                SIM_SYNC_IN();
            }
            if (use_lut) {
                if (G && lut_full) {
                    gupdate(L, geo, (int)dc_bsz, (int)dc_max, dc_dur, lane);
                    __syncwarp();
                } else {
                    lut_update_warp<G>(L, dc_bsz, dc_max, dc_dur, lane);
                    __syncwarp();
                    lut_full = L->full != 0;
                }
            }
            dsteps++;
            D = dstep(D, (uint64_t)t ^ 0x5A5A5A5A5A5A5A5AULL);
            D = dstep(D, ((uint64_t)s << 32) | (uint32_t)dc_bsz);
            D = dstep(D, (uint64_t)dc_dur);
            if (FULL && S.T.buf && lane == 0) {
                S.T.put(S.T.used, SLOSIM_EV_DECODE_DONE); S.T.put(S.T.used + 1, t); S.T.put(S.T.used + 2, dc_dur);
                S.T.put(S.T.used + 3, dc_bsz); S.T.put(S.T.used + 4, dc_max);
            }
            if (FULL) S.T.used += 5 + nmem;
            dc_end = SLOSIM_INF64;
            // no step runs now: an admission that switches to memory mode before the next decode
            // start must not carry this batch's membership into the flag bits (to_memory_mode)
            dc_mask = 0;
        }

        PROF_MARK(1);
        // admission, then a new prefill step (out of line)
        if (__builtin_expect(adm_pend || pf_wait, 0)) {
            SIM_SYNC_OUT();
            if (S.pt > S.ph) {
                S.sl = sl;
                on_admit<FULL>(S, S.sl, t, lane);
                sl = S.sl;
            }
            if (S.pf_end == SLOSIM_INF64 && S.qt > S.qh) on_prefill_start<FULL>(S, t, lane);
            SIM_SYNC_IN();
        }

        PROF_MARK(2);
        // ---- start a decode step (engine.py:377-392): the hot path
        if (dc_end == SLOSIM_INF64 && an > 0) {
            PROF_COUNT(7, an == 1);
            PROF_COUNT(6, an > 16 ? (an > 32 ? 1000000 : 1) : 0);
            v_dec += an;
            max_a = an > max_a ? an : max_a;
            int bsz = an;
            int64_t bmax = amax;
            if (__builtin_expect(regmode, 1)) {
                dc_mask = amask;
                // With one active request both outcomes of Alg. 3 (admit it, or fall
                // back to the whole active set) are the same batch: skip the scan.
                if (DP == SLOSIM_DECODE_KAIROS_SLACK && SKIP_SINGLE(an)) {
                    dc_mask = 0;  // set below from the selection
                    // select_decode_batch decode_sched.py:60-111
                    bool occ = (amask >> lane) & 1u;
                    int64_t v = occ ? tpot_slo * ((int64_t)(sl.seq - sl.inp) + 1) - (t - sl.tf) : SLOSIM_INF64;
                    uint32_t adm;
                    int64_t ms;
                    int b;
                    if (G && __builtin_expect(lut_full, 1)) {
                        int msq;
                        b = scan_geo(L, geo, rowtab, amask, an, sl, wmin64_redux(v), adm, msq, rk_rank, rk_pred,
                                     rk_mask, lane);
                        ms = msq;
                    } else if (__builtin_expect(lut_full, 1)) {
                        b = scan_slots<G>(L, amask, an, sl, wmin64_redux(v), adm, ms, lane);
                    } else {
                        // general LUT: memory-mode selection on a spilled copy
                        SIM_SYNC_OUT();
                        S.sl = sl;
                        to_memory_mode(S, S.sl, lane);
                        on_decode_start_mem<DP>(S, t, lane);
                        bsz = S.sel_bsz;
                        bmax = S.sel_max;
                        // map the flag bits back to slots (slot order == compacted order)
                        int d = __popc(amask & lanemask_lt(lane));
                        bool f = ((amask >> lane) & 1u) && (S.w.i32(A_FLAG)[d] & 1);
                        adm = __ballot_sync(FULLMASK, f);
                        b = S.dc_prefix >= 0 ? 0 : bsz;
                        ms = bmax;
                        S.regmode = true;
                        S.dc_prefix = -1;
                        SIM_SYNC_IN();
                    }
                    if (b > 0) { bsz = b; bmax = ms; dc_mask = adm; }
                    else { bsz = an; bmax = amax; dc_mask = amask; }
                }
            } else {
                SIM_SYNC_OUT();
                on_decode_start_mem<DP>(S, t, lane);
                SIM_SYNC_IN();
                bsz = S.sel_bsz;
                bmax = S.sel_max;
            }
            b_dec += bsz;
            // _GroundTruth.decode_step_us engine.py:185-192 (frozen profiles and noise out of line)
            const slosim_profile_t* P = S.P;
            double val;
            if (__builtin_expect(gt_plain && gt_fast, 1))
                val = gt_line_eval(*gtl, bsz, bmax);
            else if (gt_plain)
                val = decode_formula(P->n_base, P->base_x, P->base_y, P->gamma, bsz, bmax);
            else
                val = gt_decode_cold(S, cx.frozen_tab + pid, bsz, bmax);
            int64_t d = rint_i64(val);
            dc_dur = d < 1 ? 1 : d;
            dc_bsz = bsz;
            dc_max = bmax;
            dc_end = t + dc_dur;
#ifndef SLOSIM_NO_FF
            // Alg. 3 runs that repeat a batch (|A| > 1) are verified step by step (ff_steps<.., V>);
            // the geometry scan keeps the ranks they need
            // when the step batches the whole active set (a verifier for repeated partial batches,
            // merging the advanced members into the others' order, was exact but slower: config 2
            // 5.72 s with whole-set runs only, 6.10 s with partial batches the previous step also
            // ran, 6.93 s with every batch, 6.04 s general verifier on whole-set runs)
            // and the steps before it did too (ff_streak: consecutive steps batching the whole active
            // set, FF_MIN_STREAK of them before an attempt): an attempt whose first step fails costs
            // about one step, and a partial batch tends to follow a partial batch
            const bool whole = bsz == an;
            const bool ff_multi = DP == SLOSIM_DECODE_KAIROS_SLACK && FF_MULTI && G && an > 1 && whole &&
                                  ff_streak >= FF_MIN_STREAK;
            ff_streak = whole ? ff_streak + 1 : 0;
            if ((DP == SLOSIM_DECODE_CONTINUOUS ? !use_lut : (FF_KAIROS && (an == 1 || ff_multi))) &&
                (DP == SLOSIM_DECODE_CONTINUOUS || lut_full) && regmode && gt_plain && !(FULL && S.T.buf) &&
                dc_end < t_rare && !pf_wait) {
                PROF_MARK(3);
                SIM_SYNC_OUT();
                S.sl = sl;
                const int m = DP == SLOSIM_DECODE_CONTINUOUS ? ff_steps<false, false>(S, S.sl, t, lane)
                              : an == 1                      ? ff_steps<true, G>(S, S.sl, t, lane)
                                                             : ff_steps<true, G, FF_MULTI>(S, S.sl, t, lane, rowtab, rk_rank);
                sl = S.sl;
                SIM_SYNC_IN();
                PROF_MARK(4);
                PROF_COUNT(8, 1);
                PROF_COUNT(9, m);
                dsteps += m;
                v_dec += (int64_t)m * an;
                ff_streak = dc_bsz == bsz ? ff_streak + m : 0;  // a trailing partial step ends the streak
                // the run's last step may batch a subset of A (ff_steps<.., V> tail): dc_bsz
                b_dec += m > 0 ? (int64_t)(m - 1) * bsz + dc_bsz : 0;
            }
#endif
        }
        PROF_MARK(3);
    }
    PROF_FLUSH();
    SIM_SYNC_OUT();
#undef SIM_SYNC_IN
#undef SIM_SYNC_OUT
    S.t_end = t_end;
    S.dsteps = dsteps;
    S.v_dec = v_dec;
    S.b_dec = b_dec;
    S.max_a = max_a;
    on_finalize<FULL>(S, c0, lane);
}

#ifndef SLOSIM_MIN_BLOCKS
#define SLOSIM_MIN_BLOCKS 4
#endif

__global__ void __launch_bounds__(128, SLOSIM_MIN_BLOCKS)
    sim_kernel(const __grid_constant__ Ctx cx, char* ws_base, size_t ws_stride, int64_t cap, unsigned long long* work) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    WS w = make_ws(ws_base + (size_t)gw * ws_stride, cap);
    const int64_t N = cx.dyn_n ? (int64_t)*cx.dyn_n : cx.B.n_instances;
    const int64_t N_ids = cx.B.n_instances;  // instance ids range over the whole batch
    const bool full = (cx.B.flags & (SLOSIM_F_ROWS | SLOSIM_F_EXPORT_LUT)) || cx.B.trace_buf;
    for (;;) {
        unsigned long long k = 0;
        if (lane == 0) k = atomicAdd(work, 1ULL);
        k = __shfl_sync(FULLMASK, k, 0);
        if ((int64_t)k >= N) break;
        const int64_t ii = cx.B.order ? cx.B.order[k] : (int64_t)k;
        if (ii < 0 || ii >= N_ids) continue;  // not a permutation entry: skipped (C-ABI contract)
        const slosim_instance_t* I = cx.B.instances + ii;
        const bool kairos = I->decode_policy == SLOSIM_DECODE_KAIROS_SLACK;
        const bool pid_ok = I->profile_id >= 0 && I->profile_id < cx.B.n_profiles;
        // power-of-two LUT geometry: index arithmetic and exact power-of-two divisions
#ifdef SLOSIM_NO_GEO
        const bool geo = false;
#else
        const bool geo = pid_ok && cx.sched_tab[I->profile_id].geo != 0;
#endif
        if (full) {
            if (kairos) {
                if (geo) simulate<SLOSIM_DECODE_KAIROS_SLACK, true, true>(cx, ii, w, lane);
                else simulate<SLOSIM_DECODE_KAIROS_SLACK, true, false>(cx, ii, w, lane);
            } else {
                simulate<SLOSIM_DECODE_CONTINUOUS, true, false>(cx, ii, w, lane);
            }
        } else {
            if (kairos) {
                if (geo) simulate<SLOSIM_DECODE_KAIROS_SLACK, false, true>(cx, ii, w, lane);
                else simulate<SLOSIM_DECODE_KAIROS_SLACK, false, false>(cx, ii, w, lane);
            } else {
                simulate<SLOSIM_DECODE_CONTINUOUS, false, false>(cx, ii, w, lane);
            }
        }
        __syncwarp();
    }
}

}  // namespace slosim
