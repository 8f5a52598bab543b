// lane_host.cpp — CPU harness of the lane engine (TEST INFRASTRUCTURE): runs the per-lane
// simulation code of csrc/tengine.cuh, compiled as host C++, one instance at a time on a host
// batch, so its decisions can be compared with the C oracle without a GPU.
// Build: g++ -O2 -std=c++17 -ffp-contract=off -fPIC -shared (tools/lane_host/build.sh).
#include "hostcompat.h"

#include <vector>

// decode-step log of the last instance run (debugging aid: t_end, duration, bsz, max_seq per step)
static std::vector<int64_t> g_log;
#define LANE_HOOK_DECODE(S, w)                                                                    \
    do {                                                                                          \
        g_log.push_back((S).dc_end); g_log.push_back((S).dc_dur); g_log.push_back((S).dc_bsz);    \
        g_log.push_back((S).dc_max); g_log.push_back((S).an);                                     \
        for (int q = 0; q < (S).an; q++) { g_log.push_back((w).a32(A_POS)[q]); g_log.push_back((w).a32(A_SEQ)[q]); } \
    } while (0)

#include "../../paper_2605_02329_b200/csrc/tengine.cuh"

using namespace slosim;
using namespace slosim::lane;

// The scheduler LUT table build_profile_tables makes (lut.cuh lut_build), for the fields the lane
// engine reads.
static void host_table(LutMem* L, const slosim_profile_t* P) {
    memset(L, 0, sizeof(*L));
    const int nb = P->nb, ns = P->ns;
    L->nb = nb;
    L->ns = ns;
    int cells = 0;
    uint32_t rm = 0;
    for (int i = 0; i < nb; i++)
        for (int j = 0; j < ns; j++) {
            const int c = i * ns + j;
            L->sum[c] = P->lut_sums[i * SLOSIM_MAX_SEQ_BUCKETS + j];
            L->cnt[c] = P->lut_counts[i * SLOSIM_MAX_SEQ_BUCKETS + j];
            L->mean[c] = L->cnt[c] > 0 ? L->sum[c] / (double)L->cnt[c] : 0.0;
            if (L->cnt[c] > 0) { cells++; rm |= 1u << i; }
        }
    int wsh = 0;
    while (wsh < 30 && (1 << wsh) < P->seq_buckets[0]) wsh++;
    bool geo = nb <= 16 && (1 << wsh) == P->seq_buckets[0];
    for (int i = 0; i < nb; i++) geo = geo && P->bsz_buckets[i] == (1 << i);
    for (int j = 0; j < ns; j++) geo = geo && (int64_t)P->seq_buckets[j] == ((int64_t)(j + 1) << wsh);
    L->rowmask = rm;
    L->populated = cells;
    L->full = cells == nb * ns;
    L->geo = geo;
    L->wsh = wsh;
    L->bad = 0;
}

// Runs every instance of a HOST batch; instances outside the lane engine's scope get status -99.
extern "C" int lane_host_run_batch(const slosim_batch_t* B) {
    std::vector<LutMem> tabs((size_t)B->n_profiles);
    for (int p = 0; p < B->n_profiles; p++) host_table(&tabs[p], B->profiles + p);
    int64_t cap = 1;
    for (int64_t i = 0; i < B->n_instances; i++) cap = std::max<int64_t>(cap, B->instances[i].n_requests);
    LCtx cx{};
    cx.B = *B;
    cx.B.max_requests = cap;
    cx.sched_tab = tabs.data();
    std::vector<char> ws(lws_bytes(cap, LUT_CELLS));
    const LWs w{ws.data(), (size_t)cap, LUT_CELLS, 0};
    for (int64_t ii = 0; ii < B->n_instances; ii++) {
        if (!lane_eligible(cx, ii)) {
            B->summaries[ii].status = -99;
            continue;
        }
        St S;
        g_log.clear();
        if (!linit(S, cx, w, ii)) continue;
        while (lstep(S, cx, w)) {
        }
    }
    return 0;
}

// copies up to `cap` words of the decode-step log of the last instance; returns its length
extern "C" int64_t lane_host_decode_log(int64_t* out, int64_t cap) {
    const int64_t n = (int64_t)g_log.size();
    for (int64_t k = 0; k < n && k < cap; k++) out[k] = g_log[k];
    return n;
}
