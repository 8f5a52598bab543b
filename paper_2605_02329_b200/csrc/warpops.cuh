// warpops.cuh — warp-cooperative building blocks shared by the warp engine
// (engine.cuh) and the lane engine's cooperative rare-event handlers
// (tengine.cuh): warp reductions/scans, the per-warp SoA workspace layout, and
// the prefill policies of prefill_sched.py (FCFS finish-time walk, urgency
// score, budget packing) over one instance's queue.
#pragma once
#include "../../include/slosim_b200.h"
#include "lut.cuh"

namespace slosim {

#define FULLMASK 0xffffffffu

// ------------------------------------------------------------ warp helpers --
__device__ __forceinline__ int64_t wsum64(int64_t v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULLMASK, v, o);
    return v;
}
__device__ __forceinline__ uint64_t wsumu64(uint64_t v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULLMASK, v, o);
    return v;
}
__device__ __forceinline__ int64_t wmax64(int64_t v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) { int64_t w = __shfl_xor_sync(FULLMASK, v, o); v = w > v ? w : v; }
    return v;
}
__device__ __forceinline__ int64_t wmin64(int64_t v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) { int64_t w = __shfl_xor_sync(FULLMASK, v, o); v = w < v ? w : v; }
    return v;
}
__device__ __forceinline__ uint64_t wminu64(uint64_t v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) { uint64_t w = __shfl_xor_sync(FULLMASK, v, o); v = w < v ? w : v; }
    return v;
}
__device__ __forceinline__ int64_t wscan_incl64(int64_t v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) { int64_t w = __shfl_up_sync(FULLMASK, v, o); if (lane >= o) v += w; }
    return v;
}
__device__ __forceinline__ unsigned lanemask_lt(int lane) { return (1u << lane) - 1u; }

// ------------------------------------------------------------- workspace --
// Per-warp SoA workspace of capacity `cap` requests, addressed as base + fixed
// multiples of the two aligned array sizes (so it costs 3 live registers).
enum WsI32 { Q_POS, Q_REM, Q_FULL, Q_INP, PF_QIDX, PF_TAKE, TR_POS, PD_POS, PD_IDR,
             A_POS, A_SEQ, A_IDR, A_OUT, A_INP, A_MISS, A_FLAG, A_ORD, N_WS_I32 };
enum WsI64 { Q_ARR, Q_SCORE, TR_T, TR_TPF, PD_TPF, PD_TTR, A_TFIRST, TPS, N_WS_I64 };

__host__ __device__ inline size_t ws_align(size_t x) { return (x + 127) & ~(size_t)127; }

struct WS {
    char* base;
    uint32_t a4, a8;
    __device__ __forceinline__ int32_t* i32(int k) const { return (int32_t*)(base + (size_t)k * a4); }
    __device__ __forceinline__ int64_t* i64(int k) const {
        return (int64_t*)(base + (size_t)N_WS_I32 * a4 + (size_t)k * a8);
    }
    __device__ __forceinline__ double* f64(int k) const { return (double*)i64(k); }
    __device__ __forceinline__ LutMem* lut() const {
        return (LutMem*)(base + (size_t)N_WS_I32 * a4 + (size_t)N_WS_I64 * a8);
    }
};

__host__ __device__ inline size_t ws_bytes(int64_t cap) {
    size_t c = (size_t)(cap > 0 ? cap : 1);
    return N_WS_I32 * ws_align(4 * c) + N_WS_I64 * ws_align(8 * c) + ws_align(sizeof(LutMem));
}

__device__ __forceinline__ WS make_ws(char* base, int64_t cap) {
    size_t c = (size_t)(cap > 0 ? cap : 1);
    return WS{base, (uint32_t)ws_align(4 * c), (uint32_t)ws_align(8 * c)};
}


// --------------------------------------------------- prefill policy (K2) --
// FCFS finish-time walk (predict_finish_times prefill_sched.py:39-56) over one
// chunk of 32 queue entries as a max-plus scan: entry k maps the cursor
// c -> max(c, a_k) + d_k = max(c + d_k, a_k + d_k); compositions are
// (A, B) pairs with (A1,B1) then (A2,B2) = (A1+A2, max(B1+A2, B2)).
// Returns this lane's finish time and updates the carried cursor.
__device__ __forceinline__ int64_t fcfs_walk_chunk(bool valid, int64_t arrival, int64_t d, int64_t& cursor,
                                                   int nvalid, int lane) {
    int64_t A = valid ? d : 0;
    int64_t Bv = valid ? arrival + d : (INT64_MIN / 4);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int64_t a2 = __shfl_up_sync(FULLMASK, A, o);
        int64_t b2 = __shfl_up_sync(FULLMASK, Bv, o);
        if (lane >= o) {
            int64_t nb = b2 + A;
            Bv = nb > Bv ? nb : Bv;
            A = a2 + A;
        }
    }
    int64_t c = cursor + A;
    int64_t fin = c > Bv ? c : Bv;
    cursor = __shfl_sync(FULLMASK, fin, nvalid - 1);
    return fin;
}

// _selection_score prefill_sched.py:68-90 (urgency, then /len or *len by sign).
__device__ __forceinline__ double selection_score(int64_t ttft_slo, int64_t finish, int64_t arrival, int32_t inp) {
    int64_t slack = ttft_slo - (finish - arrival);
    double u = idiv(slack, ttft_slo);
    return u >= 0 ? xdiv(u, (double)inp) : xmul(u, (double)inp);
}

// Packs the chunk budget from the queue [qh, qt) per policy (prefill_sched.py:93-145).
// Writes (queue index, take) in batch order; returns the number of entries.
__device__ __noinline__ int prefill_select(int policy, const WS& w, int qh, int qt, int64_t budget, int64_t t_now,
                              int64_t est_tok, int64_t est_busy, int64_t ttft_slo, int lane) {
    int32_t* pf_qidx = w.i32(PF_QIDX);
    int32_t* pf_take = w.i32(PF_TAKE);
    const int32_t* q_rem = w.i32(Q_REM);
    int k = 0;
    int64_t left = budget;
    if (policy == SLOSIM_PREFILL_FCFS) {
        // fcfs_select_prefill :130-131 — the queue is already in FCFS order
        for (int base = qh; base < qt && left > 0; base += 32) {
            int qi = base + lane;
            bool valid = qi < qt;
            int64_t rem = valid ? q_rem[qi] : 0;
            int64_t incl = wscan_incl64(rem, lane);
            int64_t excl = incl - rem;
            int64_t take = (valid && excl < left) ? (rem < left - excl ? rem : left - excl) : 0;
            unsigned m = __ballot_sync(FULLMASK, take > 0);
            if (take > 0) {
                int d = k + __popc(m & lanemask_lt(lane));
                pf_qidx[d] = qi;
                pf_take[d] = (int32_t)take;
            }
            k += __popc(m);
            left -= wsum64(take);
        }
        __syncwarp();
        return k;
    }
    double* q_score = w.f64(Q_SCORE);
    if (policy == SLOSIM_PREFILL_KAIROS_URGENCY) {
        // predict_finish_times + _selection_score for every queued request
        const int64_t* q_arr = w.i64(Q_ARR);
        const int32_t* q_inp = w.i32(Q_INP);
        int64_t cursor = t_now;
        for (int base = qh; base < qt; base += 32) {
            int qi = base + lane;
            bool valid = qi < qt;
            int64_t a = valid ? q_arr[qi] : 0;
            int64_t rem = valid ? q_rem[qi] : 0;
            int64_t d = valid ? ceil_muldiv(rem, est_busy, est_tok) : 0;
            int nvalid = qt - base < 32 ? qt - base : 32;
            int64_t fin = fcfs_walk_chunk(valid, a, d, cursor, nvalid, lane);
            if (valid) q_score[qi] = selection_score(ttft_slo, fin, a, q_inp[qi]);
        }
        __syncwarp();
    }
    // repeated arg-best in the policy order, strictly after the previous pick:
    //   sjf    key (remaining, arrival, id)   -> (rem, qi)
    //   kairos key (-score, arrival, id)       -> (~dkey(score), qi)
    uint64_t pk = 0;
    int pq = -1;
    while (left > 0) {
        uint64_t bk = ~0ULL;
        int bq = 0x7fffffff;
        for (int base = qh; base < qt; base += 32) {
            int qi = base + lane;
            if (qi < qt) {
                uint64_t key = policy == SLOSIM_PREFILL_SJF ? (uint64_t)(uint32_t)q_rem[qi] : ~dkey(q_score[qi]);
                bool after = key > pk || (key == pk && qi > pq);
                if (after && (key < bk || (key == bk && qi < bq))) { bk = key; bq = qi; }
            }
        }
        uint64_t mk = wminu64(bk);
        int cand = (bk == mk) ? bq : 0x7fffffff;
        int mq = __reduce_min_sync(FULLMASK, cand);
        if (mq == 0x7fffffff) break;
        int64_t rem = q_rem[mq];
        int64_t take = rem < left ? rem : left;
        if (take > 0) {
            if (lane == 0) { pf_qidx[k] = mq; pf_take[k] = (int32_t)take; }
            k++;
            left -= take;
        }
        pk = mk;
        pq = mq;
    }
    __syncwarp();
    return k;
}

}  // namespace slosim
