/*
 * slosim_oracle.c — CPU ORACLE (test infrastructure, NOT the product).
 *
 * A single-threaded plain-C restatement of the reference simulator
 * /root/reference/pkg/src/slosim (engine.py, prefill_sched.py, decode_sched.py,
 * costmodel.py, metrics.py), used only by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg as the checker and CPU
 * baseline.  It is pinned against golden vectors produced by the Python
 * reference itself (tests/golden/make_golden.py) — see tests/test_oracle_golden.py.
 *
 * Arithmetic follows the reference's formula shapes exactly:
 * compile with -ffp-contract=off (no FMA), half-even rounding via rint(),
 * correctly-rounded int/int true division, 128-bit ceil-div for the estimator.
 * It deliberately shares no code with the CUDA path; only the packed
 * input/output layouts of include/slosim_b200.h.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/slosim_b200.h"

#define INF64 INT64_MAX

/* ------------------------------------------------------------ numerics ---- */

static int bitlen_u128(unsigned __int128 x) {
    int n = 0;
    while (x) { n++; x >>= 1; }
    return n;
}

/* Python int/int true division: the correctly rounded double of p/q. */
static double idiv(__int128 p, __int128 q) {
    int neg = (p < 0) != (q < 0);
    unsigned __int128 a = p < 0 ? (unsigned __int128)(-p) : (unsigned __int128)p;
    unsigned __int128 b = q < 0 ? (unsigned __int128)(-q) : (unsigned __int128)q;
    const unsigned __int128 lim = (unsigned __int128)1 << 53;
    double r;
    if (a < lim && b < lim) {
        r = (double)(uint64_t)a / (double)(uint64_t)b;
    } else {
        int s = 55 - (bitlen_u128(a) - bitlen_u128(b));
        unsigned __int128 num = a, den = b;
        if (s >= 0) num <<= s; else den <<= -s;
        unsigned __int128 Q = num / den, R = num % den;
        int nq = bitlen_u128(Q), drop = nq - 53;
        unsigned __int128 mant = Q >> drop, low = Q & ((((unsigned __int128)1) << drop) - 1);
        unsigned __int128 half = ((unsigned __int128)1) << (drop - 1);
        if (low > half || (low == half && (R != 0 || (mant & 1)))) mant++;
        r = ldexp((double)(uint64_t)mant, drop - s);
    }
    return neg ? -r : r;
}

static int64_t round_half_even(double x) { return (int64_t)rint(x); }

static int bisect_left_i32(const int32_t* a, int n, int64_t x) {
    int lo = 0, hi = n;
    while (lo < hi) { int mid = (lo + hi) / 2; if (a[mid] < x) lo = mid + 1; else hi = mid; }
    return lo;
}

/* ----------------------------------------------------------- cost models --- */

typedef struct {
    int nb, ns;
    const int32_t* bb;
    const int32_t* sb;
    double* sums;   /* [nb*ns] in a 16x64 frame: index i*SLOSIM_MAX_SEQ_BUCKETS+j */
    int32_t* counts;
} OLut;

#define CELL(i, j) ((i) * SLOSIM_MAX_SEQ_BUCKETS + (j))

/* DecodeStepLUT._bucket_index costmodel.py:99-103 */
static int bucket_index(const int32_t* b, int n, int64_t v) {
    int i = bisect_left_i32(b, n, v);
    return i < n - 1 ? i : n - 1;
}

/* np.interp over the populated columns of row i (costmodel.py:143-155). */
static double row_eval(const OLut* L, int i, int64_t seq) {
    int cols[SLOSIM_MAX_SEQ_BUCKETS], m = 0;
    for (int j = 0; j < L->ns; j++) if (L->counts[CELL(i, j)] > 0) cols[m++] = j;
    double x = (double)seq;
    double ys[SLOSIM_MAX_SEQ_BUCKETS], xs[SLOSIM_MAX_SEQ_BUCKETS];
    for (int k = 0; k < m; k++) {
        xs[k] = (double)L->sb[cols[k]];
        ys[k] = L->sums[CELL(i, cols[k])] / (double)L->counts[CELL(i, cols[k])];
    }
    if (m == 1) return ys[0];
    if (x <= xs[0]) return ys[0];
    if (x >= xs[m - 1]) return ys[m - 1];
    int j = 0;
    while (!(xs[j] <= x && x < xs[j + 1])) j++;
    if (xs[j] == x) return ys[j];
    double slope = (ys[j + 1] - ys[j]) / (xs[j + 1] - xs[j]);
    return slope * (x - xs[j]) + ys[j];
}

/* DecodeStepLUT.lookup costmodel.py:157-187 (caller guarantees non-empty, bsz,seq >= 1) */
static double lut_lookup(const OLut* L, int64_t bsz, int64_t seq) {
    int i = bisect_left_i32(L->bb, L->nb, bsz);
    int j = bisect_left_i32(L->sb, L->ns, seq);
    int exact_b = i < L->nb && L->bb[i] == bsz;
    int exact_s = j < L->ns && L->sb[j] == seq;
    if (exact_b && exact_s && L->counts[CELL(i, j)] > 0)
        return L->sums[CELL(i, j)] / (double)L->counts[CELL(i, j)];
    int rows[SLOSIM_MAX_BSZ_BUCKETS], nr = 0;
    int32_t rb[SLOSIM_MAX_BSZ_BUCKETS];
    for (int r = 0; r < L->nb; r++) {
        int any = 0;
        for (int c = 0; c < L->ns; c++) if (L->counts[CELL(r, c)] > 0) { any = 1; break; }
        if (any) { rb[nr] = L->bb[r]; rows[nr++] = r; }
    }
    int k = bisect_left_i32(rb, nr, bsz);
    if (k == 0) return row_eval(L, rows[0], seq);
    if (k == nr) return row_eval(L, rows[nr - 1], seq);
    if (rb[k] == bsz) return row_eval(L, rows[k], seq);
    double v_lo = row_eval(L, rows[k - 1], seq);
    double v_hi = row_eval(L, rows[k], seq);
    int64_t b_lo = rb[k - 1], b_hi = rb[k];
    return v_lo + (v_hi - v_lo) * (double)(bsz - b_lo) / (double)(b_hi - b_lo);
}

static int lut_empty(const OLut* L) {
    for (int i = 0; i < L->nb; i++)
        for (int j = 0; j < L->ns; j++) if (L->counts[CELL(i, j)] > 0) return 0;
    return 1;
}

/* DecodeStepLUT.update costmodel.py:118-128 */
static void lut_update(OLut* L, int64_t bsz, int64_t max_seq, int64_t obs) {
    int i = bucket_index(L->bb, L->nb, bsz), j = bucket_index(L->sb, L->ns, max_seq);
    L->sums[CELL(i, j)] += (double)obs;
    L->counts[CELL(i, j)] += 1;
}

/* _interp_clamped costmodel.py:32-47 (ys floats, x int) */
static double interp_clamped(int n, const int64_t* px, const double* py, int64_t x) {
    if (x <= px[0]) return py[0];
    if (x >= px[n - 1]) return py[n - 1];
    int k = 0;
    while (k + 1 < n && px[k + 1] <= x) k++; /* bisect_right(xs, x) - 1 */
    double y0 = py[k], y1 = py[k + 1];
    return y0 + (y1 - y0) * (double)(x - px[k]) / (double)(px[k + 1] - px[k]);
}

/* decode_step_formula costmodel.py:50-58 */
static double decode_formula(const slosim_profile_t* P, int64_t bsz, int64_t seq) {
    return interp_clamped(P->n_base, P->base_x, P->base_y, seq) * (1.0 + P->gamma * (double)(bsz - 1));
}

/* PrefillThroughputEstimator.estimate_duration_us costmodel.py:261-268 */
static int64_t est_duration(int64_t total, int64_t busy, int64_t tokens) {
    if (tokens == 0) return 0;
    __int128 num = (__int128)tokens * busy;
    return (int64_t)((num + total - 1) / total);
}

/* _GroundTruth._curve_at engine.py:161-173 (integer points) */
static double curve_at(const slosim_profile_t* P, int64_t tokens) {
    int n = P->n_curve;
    const int64_t* x = P->curve_x;
    const int64_t* y = P->curve_y;
    if (tokens >= x[n - 1]) {
        int64_t x0 = x[n - 2], y0 = y[n - 2], x1 = x[n - 1], y1 = y[n - 1];
        return (double)y1 + idiv((__int128)(y1 - y0) * (tokens - x1), x1 - x0);
    }
    for (int k = 0; k < n - 1; k++) {
        if (tokens <= x[k + 1]) {
            int64_t x0 = x[k], y0 = y[k], x1 = x[k + 1], y1 = y[k + 1];
            return (double)y0 + idiv((__int128)(y1 - y0) * (tokens - x0), x1 - x0);
        }
    }
    return NAN;
}

/* _GroundTruth.prefill_batch_us engine.py:175-183 */
static int64_t prefill_gt(const slosim_profile_t* P, int k, const int64_t* done, const int64_t* take) {
    double total = 0.0;
    for (int e = 0; e < k; e++) total += curve_at(P, done[e] + take[e]) - curve_at(P, done[e]);
    int64_t r = round_half_even(total);
    return r < 1 ? 1 : r;
}

/* numpy PCG64 (XSL-RR 128/64) + Generator.uniform, engine.py:191 */
typedef struct { unsigned __int128 state, inc; } Pcg64;
static uint64_t pcg_next(Pcg64* g) {
    const unsigned __int128 mult = (((unsigned __int128)0x2360ED051FC65DA4ULL) << 64) | 0x4385DF649FCCF645ULL;
    g->state = g->state * mult + g->inc;
    uint64_t hi = (uint64_t)(g->state >> 64), lo = (uint64_t)g->state;
    unsigned rot = (unsigned)(g->state >> 122);
    uint64_t x = hi ^ lo;
    return (x >> rot) | (x << ((64 - rot) & 63));
}
static double pcg_uniform(Pcg64* g, double low, double high) {
    double u = (double)(pcg_next(g) >> 11) * (1.0 / 9007199254740992.0);
    return low + (high - low) * u;
}

/* _GroundTruth.decode_step_us engine.py:185-192 */
static int64_t decode_gt(const slosim_profile_t* P, const OLut* frozen, Pcg64* g, int64_t bsz, int64_t max_seq) {
    double v = P->gt_frozen ? lut_lookup(frozen, bsz, max_seq) : decode_formula(P, bsz, max_seq);
    if (P->noise_eps > 0) v *= pcg_uniform(g, 1.0 - P->noise_eps, 1.0 + P->noise_eps);
    int64_t r = round_half_even(v);
    return r < 1 ? 1 : r;
}

/* ------------------------------------------------------------- digest ----
 * D <- fold((D ^ x) * phi64); decode members: sum of 32-bit (pos+1)*phi32. */
static uint64_t dstep(uint64_t D, uint64_t x) {
    uint64_t z = (D ^ x) * 0x9E3779B97F4A7C15ULL;
    return z ^ (z >> 32);
}
static uint64_t mix64(uint64_t x) {
    x ^= x >> 30; x *= 0xbf58476d1ce4e5b9ULL;
    x ^= x >> 27; x *= 0x94d049bb133111ebULL;
    x ^= x >> 31;
    return x;
}

/* ---------------------------------------------------------- simulation ---- */

typedef struct { int64_t tpf; int32_t idr; int64_t ttr; int32_t pos; } Pend;

typedef struct {
    int64_t* buf; int64_t cap; int64_t used; int overflow;
} Tr;

static void tr_put(Tr* T, const int64_t* w, int64_t k) {
    if (!T->buf) return;
    if (T->used + k > T->cap - 2) { T->overflow = 1; T->used += k; return; }
    memcpy(T->buf + T->used, w, (size_t)k * 8); T->used += k;
}

typedef struct {
    const slosim_profile_t* P;
    const slosim_instance_t* I;
    int n;
    int64_t* arr; const int32_t* inp; const int32_t* out; const int32_t* hit; const int32_t* idr;
    int32_t* done; int32_t* ngen; int64_t* tpf; int64_t* tfirst; int64_t* tlast; int64_t* fsched; int32_t* miss;
    OLut lut, frozen;
    int64_t est_tok, est_busy;
} Sim;

static int64_t rem_of(const Sim* S, int p) { return (int64_t)S->inp[p] - S->hit[p] - S->done[p]; }

/* key (arrival, id) of _fcfs_order prefill_sched.py:35-36 */
static int fcfs_less(const Sim* S, int a, int b) {
    if (S->arr[a] != S->arr[b]) return S->arr[a] < S->arr[b];
    return S->idr[a] < S->idr[b];
}

/* _pack prefill_sched.py:93-106 over an ordered candidate list */
static int pack(const Sim* S, const int* cand, int nc, int64_t budget, int* out_pos, int64_t* out_take) {
    int k = 0; int64_t left = budget;
    for (int c = 0; c < nc; c++) {
        if (left == 0) break;
        int64_t r = rem_of(S, cand[c]);
        int64_t take = r < left ? r : left;
        if (take <= 0) continue;
        out_pos[k] = cand[c]; out_take[k] = take; k++; left -= take;
    }
    return k;
}

static __thread const Sim* t_sim;
static __thread const double* t_score;
static __thread const int64_t* t_seq;

static int cmp_fcfs(const void* a, const void* b) {
    int x = *(const int*)a, y = *(const int*)b;
    return fcfs_less(t_sim, x, y) ? -1 : (fcfs_less(t_sim, y, x) ? 1 : 0);
}
/* sjf key (remaining, arrival, id) prefill_sched.py:134-138 */
static int cmp_sjf(const void* a, const void* b) {
    int x = *(const int*)a, y = *(const int*)b;
    int64_t rx = rem_of(t_sim, x), ry = rem_of(t_sim, y);
    if (rx != ry) return rx < ry ? -1 : 1;
    return cmp_fcfs(a, b);
}

/* kairos key (-score, arrival, id) prefill_sched.py:123-126; t_score indexed by pos */
static int cmp_kairos(const void* a, const void* b) {
    int x = *(const int*)a, y = *(const int*)b;
    double nx = -t_score[x], ny = -t_score[y];
    if (!(nx == ny)) return nx < ny ? -1 : 1;
    return cmp_fcfs(a, b);
}

/* decode order (seq_len, id) decode_sched.py:74 */
static int cmp_decode(const void* a, const void* b) {
    int x = *(const int*)a, y = *(const int*)b;
    if (t_seq[x] != t_seq[y]) return t_seq[x] < t_seq[y] ? -1 : 1;
    return t_sim->idr[x] < t_sim->idr[y] ? -1 : (t_sim->idr[x] > t_sim->idr[y]);
}

static int cmp_pend(const void* a, const void* b) {
    const Pend* x = (const Pend*)a; const Pend* y = (const Pend*)b;
    if (x->tpf != y->tpf) return x->tpf < y->tpf ? -1 : 1;
    return x->idr < y->idr ? -1 : (x->idr > y->idr);
}

static int cmp_dbl(const void* a, const void* b) {
    double x = *(const double*)a, y = *(const double*)b;
    return x < y ? -1 : (x > y);
}

/* Simulation.run engine.py:261-284 for one instance. */
static void run_instance(const slosim_batch_t* B, int64_t ii) {
    const slosim_instance_t* I = &B->instances[ii];
    const slosim_profile_t* P = &B->profiles[I->profile_id];
    slosim_summary_t* O = &B->summaries[ii];
    memset(O, 0, sizeof(*O));
    Sim S; memset(&S, 0, sizeof(S));
    S.P = P; S.I = I;
    int n = S.n = I->n_requests;
    int64_t off = I->trace_offset;
    S.inp = B->traces.input_len + off; S.out = B->traces.output_len + off;
    S.hit = B->traces.prefix_hit_len + off; S.idr = B->traces.id_rank + off;
    size_t nn = (size_t)(n > 0 ? n : 1);
    S.arr = malloc(nn * 8);
    for (int p = 0; p < n; p++) {
        int64_t a = B->traces.arrival_us[off + p];
        /* rescale_qps workload.py:175-182: round(arrival * factor) */
        S.arr[p] = I->rescale_factor > 0 ? round_half_even((double)a * I->rescale_factor) : a;
    }
    O->n = n;
    O->tps_p50 = NAN; O->tps_p90 = NAN;
    /* KV reservation check engine.py:227-232 */
    int64_t worst = 0;
    for (int p = 0; p < n; p++) { int64_t w = (int64_t)S.inp[p] + S.out[p]; if (w > worst) worst = w; }
    double lsums[SLOSIM_MAX_BSZ_BUCKETS * SLOSIM_MAX_SEQ_BUCKETS];
    int32_t lcounts[SLOSIM_MAX_BSZ_BUCKETS * SLOSIM_MAX_SEQ_BUCKETS];
    memcpy(lsums, P->lut_sums, sizeof(lsums)); memcpy(lcounts, P->lut_counts, sizeof(lcounts));
    S.lut = (OLut){P->nb, P->ns, P->bsz_buckets, P->seq_buckets, lsums, lcounts};
    S.frozen = (OLut){P->nb, P->ns, P->bsz_buckets, P->seq_buckets, (double*)P->gt_sums, (int32_t*)P->gt_counts};
    if (worst > I->kv_capacity_tokens || lut_empty(&S.lut)) { O->status = SLOSIM_ECONFIG; free(S.arr); return; }
    S.est_tok = P->est_tokens; S.est_busy = P->est_busy_us;
    Pcg64 rng = {(((unsigned __int128)I->rng_state_hi) << 64) | I->rng_state_lo,
                 (((unsigned __int128)I->rng_inc_hi) << 64) | I->rng_inc_lo};

    S.done = calloc(nn, 4); S.ngen = calloc(nn, 4); S.miss = calloc(nn, 4);
    S.tpf = malloc(nn * 8); S.tfirst = malloc(nn * 8); S.tlast = malloc(nn * 8); S.fsched = malloc(nn * 8);
    for (int p = 0; p < n; p++) S.tpf[p] = S.tfirst[p] = S.tlast[p] = S.fsched[p] = -1;
    int* queue = malloc(nn * sizeof(int)); int qn = 0;
    int* pf_pos = malloc(nn * sizeof(int)); int64_t* pf_take = malloc(nn * 8); int pf_k = 0;
    int64_t* pf_done = malloc(nn * 8);
    int64_t pf_end = -1, pf_dur = 0;
    int64_t* tr_t = malloc(nn * 8); int* tr_p = malloc(nn * sizeof(int)); int trn = 0;
    Pend* pend = malloc(nn * sizeof(Pend)); int pdn = 0;
    int* act = malloc(nn * sizeof(int)); int an = 0;
    int* dcb = malloc(nn * sizeof(int)); int dck = 0;
    int64_t* seqv = malloc(nn * 8);
    int* cand = malloc(nn * sizeof(int));
    double* score = malloc(nn * sizeof(double));
    int64_t dc_end = -1, dc_dur = 0, dc_bsz = 0, dc_max = 0;
    int64_t kv = 0; int finished = 0; int ai = 0;
    uint64_t D = 0;
    Tr T = {0};
    if (B->trace_buf && I->trace_buf_offset >= 0) { T.buf = B->trace_buf + I->trace_buf_offset; T.cap = I->trace_buf_words; }
    const int use_lut = I->decode_policy == SLOSIM_DECODE_KAIROS_SLACK || (B->flags & (SLOSIM_F_ALWAYS_LUT | SLOSIM_F_EXPORT_LUT));
    t_sim = &S;

    for (;;) {
        int64_t t = INF64;
        if (ai < n) t = S.arr[ai];
        if (pf_end >= 0 && pf_end < t) t = pf_end;
        if (dc_end >= 0 && dc_end < t) t = dc_end;
        for (int k = 0; k < trn; k++) if (tr_t[k] < t) t = tr_t[k];
        if (t == INF64) break;
        O->t_end_us = t;
        /* arrivals engine.py:288-291 */
        while (ai < n && S.arr[ai] == t) {
            int64_t w[3] = {SLOSIM_EV_ARRIVAL, t, ai}; tr_put(&T, w, 3);
            queue[qn++] = ai++;
        }
        /* transfers pushed earlier, in push order engine.py:294-298 */
        { int m = 0;
          for (int k = 0; k < trn; k++) {
              if (tr_t[k] == t) {
                  int p = tr_p[k];
                  pend[pdn++] = (Pend){S.tpf[p], S.idr[p], t, p};
                  int64_t w[3] = {SLOSIM_EV_TRANSFER_DONE, t, p}; tr_put(&T, w, 3);
              } else { tr_t[m] = tr_t[k]; tr_p[m] = tr_p[k]; m++; }
          }
          trn = m; }
        /* prefill completion engine.py:327-350 */
        if (pf_end == t) {
            int64_t tot = 0;
            for (int e = 0; e < pf_k; e++) { S.done[pf_pos[e]] += (int32_t)pf_take[e]; tot += pf_take[e]; }
            S.est_tok += tot; S.est_busy += pf_dur;
            O->prefill_steps++;
            D = dstep(D, (uint64_t)t ^ 0xA5A5A5A5A5A5A5A5ULL);
            for (int e = 0; e < pf_k; e++) D = dstep(D, ((uint64_t)pf_pos[e] << 32) | (uint64_t)pf_take[e]);
            D = dstep(D, (uint64_t)pf_dur);
            if (T.buf) {
                int64_t w[4] = {SLOSIM_EV_PREFILL_DONE, t, pf_dur, pf_k}; tr_put(&T, w, 4);
                for (int e = 0; e < pf_k; e++) { int64_t x = ((int64_t)pf_pos[e] << 32) | pf_take[e]; tr_put(&T, &x, 1); }
            }
            for (int e = 0; e < pf_k; e++) {
                int p = pf_pos[e];
                if (rem_of(&S, p) == 0 && S.tpf[p] < 0) {
                    S.tpf[p] = t;
                    int m = 0; for (int k = 0; k < qn; k++) if (queue[k] != p) queue[m++] = queue[k];
                    qn = m;
                    int64_t delay = I->transfer_base_us + round_half_even((double)S.inp[p] * I->transfer_per_token_us);
                    if (delay == 0) {
                        pend[pdn++] = (Pend){t, S.idr[p], t, p};
                        int64_t w[3] = {SLOSIM_EV_TRANSFER_DONE, t, p}; tr_put(&T, w, 3);
                    } else { tr_t[trn] = t + delay; tr_p[trn] = p; trn++; }
                }
            }
            pf_end = -1;
        }
        /* decode completion engine.py:394-413 */
        if (dc_end == t) {
            uint32_t s = 0;
            for (int b = 0; b < dck; b++) {
                int p = dcb[b];
                s += ((uint32_t)p + 1u) * 0x9E3779B1u;
                S.ngen[p] += 1;
                if (t > S.tfirst[p] + (int64_t)S.ngen[p] * I->tpot_slo_us) S.miss[p]++;
                S.tlast[p] = t;
                if (S.ngen[p] == S.out[p] - 1) {
                    finished++; kv -= (int64_t)S.inp[p] + S.out[p];
                    int m = 0; for (int k = 0; k < an; k++) if (act[k] != p) act[m++] = act[k];
                    an = m;
                }
            }
            if (use_lut) lut_update(&S.lut, dc_bsz, dc_max, dc_dur);
            O->decode_steps++;
            D = dstep(D, (uint64_t)t ^ 0x5A5A5A5A5A5A5A5AULL);
            D = dstep(D, ((uint64_t)s << 32) | (uint32_t)dck);
            D = dstep(D, (uint64_t)dc_dur);
            if (T.buf) {
                int64_t w[5] = {SLOSIM_EV_DECODE_DONE, t, dc_dur, dc_bsz, dc_max}; tr_put(&T, w, 5);
                for (int b = 0; b < dck; b++) { int64_t x = dcb[b]; tr_put(&T, &x, 1); }
            }
            dc_end = -1;
        }
        /* _admit engine.py:355-375 */
        if (pdn > 1) qsort(pend, (size_t)pdn, sizeof(Pend), cmp_pend);
        { int h0 = 0;
          while (h0 < pdn) {
              int p = pend[h0].pos;
              int64_t need = (int64_t)S.inp[p] + S.out[p];
              if (kv + need > I->kv_capacity_tokens) break;
              h0++;
              S.tfirst[p] = pend[h0 - 1].ttr; S.tlast[p] = pend[h0 - 1].ttr;
              int64_t w[4] = {SLOSIM_EV_ADMIT, t, p, S.tfirst[p]}; tr_put(&T, w, 4);
              if (S.out[p] == 1) finished++;
              else { act[an++] = p; kv += need; }
          }
          if (h0) { memmove(pend, pend + h0, (size_t)(pdn - h0) * sizeof(Pend)); pdn -= h0; } }
        /* _start_prefill engine.py:307-325 */
        if (pf_end < 0 && qn > 0) {
            int nc = qn;
            memcpy(cand, queue, (size_t)qn * sizeof(int));
            if (I->prefill_policy == SLOSIM_PREFILL_FCFS) {
                qsort(cand, (size_t)nc, sizeof(int), cmp_fcfs);
            } else if (I->prefill_policy == SLOSIM_PREFILL_SJF) {
                qsort(cand, (size_t)nc, sizeof(int), cmp_sjf);
            } else {
                /* predict_finish_times prefill_sched.py:39-56 + _selection_score :82-90 */
                qsort(cand, (size_t)nc, sizeof(int), cmp_fcfs);
                int64_t cursor = t;
                for (int c = 0; c < nc; c++) {
                    int p = cand[c];
                    int64_t a = S.arr[p];
                    cursor = (cursor > a ? cursor : a) + est_duration(S.est_tok, S.est_busy, rem_of(&S, p));
                    int64_t slack = I->ttft_slo_us - (cursor - a);
                    double u = idiv(slack, I->ttft_slo_us);
                    score[p] = u >= 0 ? u / (double)S.inp[p] : u * (double)S.inp[p];
                }
                t_score = score;
                qsort(cand, (size_t)nc, sizeof(int), cmp_kairos);
            }
            pf_k = pack(&S, cand, nc, I->chunk_budget, pf_pos, pf_take);
            if (pf_k > 0) {
                for (int e = 0; e < pf_k; e++) {
                    int p = pf_pos[e];
                    pf_done[e] = S.done[p];
                    if (S.fsched[p] < 0) S.fsched[p] = t;
                }
                pf_dur = prefill_gt(P, pf_k, pf_done, pf_take);
                pf_end = t + pf_dur;
                O->v_pre += qn;
                if (qn > O->max_queue) O->max_queue = qn;
            }
        }
        /* _start_decode engine.py:377-392 */
        if (dc_end < 0 && an > 0) {
            for (int k = 0; k < an; k++) seqv[act[k]] = (int64_t)S.inp[act[k]] + S.ngen[act[k]];
            memcpy(cand, act, (size_t)an * sizeof(int));
            t_seq = seqv;
            qsort(cand, (size_t)an, sizeof(int), cmp_decode);
            if (I->decode_policy == SLOSIM_DECODE_CONTINUOUS) {
                /* continuous_batching_select decode_sched.py:114-124 */
                memcpy(dcb, cand, (size_t)an * sizeof(int)); dck = an;
            } else {
                /* select_decode_batch decode_sched.py:60-111 */
                int64_t max_seq = seqv[cand[an - 1]];
                double fallback = lut_lookup(&S.lut, an, max_seq);
                double smin = INFINITY;
                for (int k = 0; k < an; k++) {
                    int p = cand[k];
                    int64_t budget = I->tpot_slo_us * (S.ngen[p] + 1);
                    int64_t elapsed = t - S.tfirst[p];
                    double sl = (double)(budget - elapsed) - fallback;
                    if (sl < smin) smin = sl;
                }
                dck = 0; double tcur = 0.0;
                for (int k = 0; k < an; k++) {
                    int p = cand[k];
                    double ts = lut_lookup(&S.lut, dck + 1, seqv[p]);
                    if (ts <= smin && (dck == 0 || (double)(dck + 1) / ts > (double)dck / tcur)) {
                        dcb[dck++] = p; tcur = ts;
                    }
                }
                if (dck == 0) { memcpy(dcb, cand, (size_t)an * sizeof(int)); dck = an; }
            }
            int64_t mx = 0;
            for (int b = 0; b < dck; b++) if (seqv[dcb[b]] > mx) mx = seqv[dcb[b]];
            dc_bsz = dck; dc_max = mx;
            dc_dur = decode_gt(P, &S.frozen, &rng, dc_bsz, dc_max);
            dc_end = t + dc_dur;
            O->v_dec += an; O->b_dec += dck;
            if (an > O->max_active) O->max_active = an;
        }
    }

    /* metrics engine.py:274-284 -> metrics.py:72-144 */
    double* tps = malloc(nn * sizeof(double)); int ntps = 0;
    int64_t ww = 0;
    for (int p = 0; p < n; p++) {
        int64_t ttft = S.tfirst[p] - S.arr[p];
        int tm = ttft <= I->ttft_slo_us;
        double tpot = 0.0; int pm = 1; double tp = NAN;
        if (S.out[p] > 1) {
            int64_t span = S.tlast[p] - S.tfirst[p];
            tpot = idiv(span, S.out[p] - 1);
            pm = tpot <= (double)I->tpot_slo_us;
            tp = (double)(S.out[p] - 1) / ((double)span / 1e6);
            tps[ntps++] = tp;
        }
        O->ttft_met += tm; O->tpot_met += pm; O->e2e_met += (tm && pm);
        O->deadline_misses += S.miss[p];
        int64_t w = S.fsched[p] - S.arr[p];
        if (w > ww) ww = w;
        int64_t g = I->row_offset + p;
        if (B->flags & SLOSIM_F_ROWS) {
            const slosim_rows_t* R = &B->rows;
            if (R->ttft_us) R->ttft_us[g] = ttft;
            if (R->mean_tpot_us) R->mean_tpot_us[g] = tpot;
            if (R->decode_tps) R->decode_tps[g] = tp;
            if (R->met_flags) R->met_flags[g] = (uint8_t)(tm | (pm << 1) | ((tm && pm) << 2));
            if (R->deadline_misses) R->deadline_misses[g] = S.miss[p];
            if (R->t_prefill_finish) R->t_prefill_finish[g] = S.tpf[p];
            if (R->t_first_token) R->t_first_token[g] = S.tfirst[p];
            if (R->t_last_token) R->t_last_token[g] = S.tlast[p];
            if (R->first_sched_us) R->first_sched_us[g] = S.fsched[p];
        }
    }
    O->worst_queue_wait_us = ww;
    O->n_tps = ntps;
    if (ntps) {
        qsort(tps, (size_t)ntps, sizeof(double), cmp_dbl);
        /* nearest_rank metrics.py:87-92 */
        int64_t r50 = (int64_t)ceil(50 / 100.0 * (double)ntps);
        int64_t r90 = (int64_t)ceil(90 / 100.0 * (double)ntps);
        O->tps_p50 = tps[(r50 < 1 ? 1 : r50) - 1];
        O->tps_p90 = tps[(r90 < 1 ? 1 : r90) - 1];
    }
    O->digest = D;
    O->est_tokens = S.est_tok; O->est_busy_us = S.est_busy;
    O->status = finished == n ? SLOSIM_OK : -1;
    if (T.buf) {
        int64_t w[2] = {SLOSIM_EV_END, T.used + 2};
        if (T.used + 2 <= T.cap) memcpy(T.buf + T.used, w, 16);
        if (T.overflow) O->status |= 0x100;
    }
    if ((B->flags & SLOSIM_F_EXPORT_LUT) && B->lut_out_sums) {
        memcpy(B->lut_out_sums + ii * SLOSIM_MAX_BSZ_BUCKETS * SLOSIM_MAX_SEQ_BUCKETS, lsums, sizeof(lsums));
        memcpy(B->lut_out_counts + ii * SLOSIM_MAX_BSZ_BUCKETS * SLOSIM_MAX_SEQ_BUCKETS, lcounts, sizeof(lcounts));
    }
    free(tps); free(S.arr); free(S.done); free(S.ngen); free(S.miss); free(S.tpf); free(S.tfirst);
    free(S.tlast); free(S.fsched); free(queue); free(pf_pos); free(pf_take); free(pf_done); free(tr_t);
    free(tr_p); free(pend); free(act); free(dcb); free(seqv); free(cand); free(score);
}

/* -------------------------------------------------------- batch driver ---- */

typedef struct { const slosim_batch_t* B; int64_t next; pthread_mutex_t mu; } Pool;

static void* worker(void* arg) {
    Pool* pool = (Pool*)arg;
    for (;;) {
        pthread_mutex_lock(&pool->mu);
        int64_t i = pool->next++;
        pthread_mutex_unlock(&pool->mu);
        if (i >= pool->B->n_instances) break;
        run_instance(pool->B, i);
    }
    return NULL;
}

/* Runs every instance of a HOST batch; n_threads <= 1 runs inline. */
int oracle_run_batch(const slosim_batch_t* B, int n_threads) {
    if (n_threads <= 1) {
        for (int64_t i = 0; i < B->n_instances; i++) run_instance(B, i);
        return 0;
    }
    Pool pool = {B, 0, PTHREAD_MUTEX_INITIALIZER};
    pthread_t th[256];
    if (n_threads > 256) n_threads = 256;
    for (int k = 0; k < n_threads; k++) pthread_create(&th[k], NULL, worker, &pool);
    for (int k = 0; k < n_threads; k++) pthread_join(th[k], NULL);
    return 0;
}

/* ---------------------------------------------- snapshot entry points ---- */

static OLut mk_lut(int32_t nb, const int32_t* bb, int32_t ns, const int32_t* sb, const double* sums,
                   const int32_t* counts, double* s2, int32_t* c2) {
    for (int i = 0; i < nb; i++)
        for (int j = 0; j < ns; j++) { s2[CELL(i, j)] = sums[i * ns + j]; c2[CELL(i, j)] = counts[i * ns + j]; }
    return (OLut){nb, ns, bb, sb, s2, c2};
}

int oracle_lut_lookup(int32_t nb, const int32_t* bb, int32_t ns, const int32_t* sb, const double* sums,
                      const int32_t* counts, int64_t n, const int64_t* bsz, const int64_t* seq, double* out) {
    double s2[SLOSIM_MAX_BSZ_BUCKETS * SLOSIM_MAX_SEQ_BUCKETS];
    int32_t c2[SLOSIM_MAX_BSZ_BUCKETS * SLOSIM_MAX_SEQ_BUCKETS];
    OLut L = mk_lut(nb, bb, ns, sb, sums, counts, s2, c2);
    if (lut_empty(&L)) return SLOSIM_ECONFIG;
    for (int64_t k = 0; k < n; k++) out[k] = lut_lookup(&L, bsz[k], seq[k]);
    return 0;
}

int oracle_decode_formula(int32_t n_base, const int64_t* bx, const double* by, double gamma, int64_t n,
                          const int64_t* bsz, const int64_t* seq, double* out) {
    for (int64_t k = 0; k < n; k++)
        out[k] = interp_clamped(n_base, bx, by, seq[k]) * (1.0 + gamma * (double)(bsz[k] - 1));
    return 0;
}

int oracle_prefill_batch_us(int32_t n_curve, const int64_t* cx, const int64_t* cy, int32_t k,
                            const int64_t* done, const int64_t* take, int64_t* out) {
    slosim_profile_t* P = calloc(1, sizeof(slosim_profile_t));
    P->n_curve = n_curve;
    memcpy(P->curve_x, cx, (size_t)n_curve * 8); memcpy(P->curve_y, cy, (size_t)n_curve * 8);
    *out = prefill_gt(P, k, done, take);
    free(P);
    return 0;
}

/* select_decode_batch with f64 times (decode_sched.py:60-111), as in slosim_select_decode */
int oracle_select_decode(int32_t policy, int32_t n, const int64_t* seq_len, const int32_t* id_rank,
                         const int64_t* n_gen, const double* t_first, double t_now, int64_t tpot,
                         int32_t nb, const int32_t* bb, int32_t ns, const int32_t* sb,
                         const double* sums, const int32_t* counts, int32_t* out_batch, int32_t* n_batch,
                         int32_t* out_delayed, int32_t* n_delayed, double* out_admit, double* out_pred,
                         double* out_smin, int32_t* out_fb) {
    double s2[SLOSIM_MAX_BSZ_BUCKETS * SLOSIM_MAX_SEQ_BUCKETS];
    int32_t c2[SLOSIM_MAX_BSZ_BUCKETS * SLOSIM_MAX_SEQ_BUCKETS];
    OLut L = mk_lut(nb, bb, ns, sb, sums, counts, s2, c2);
    if (n < 1) return SLOSIM_EINVAL;
    int* ord = malloc((size_t)n * sizeof(int));
    for (int k = 0; k < n; k++) ord[k] = k;
    /* insertion sort by (seq, id_rank) */
    for (int a = 1; a < n; a++) {
        int x = ord[a], b = a - 1;
        while (b >= 0 && (seq_len[ord[b]] > seq_len[x] || (seq_len[ord[b]] == seq_len[x] && id_rank[ord[b]] > id_rank[x]))) {
            ord[b + 1] = ord[b]; b--;
        }
        ord[b + 1] = x;
    }
    int64_t max_seq = seq_len[ord[n - 1]];
    double fallback = lut_lookup(&L, n, max_seq);
    *n_delayed = 0; *out_fb = 0;
    if (policy == SLOSIM_DECODE_CONTINUOUS) {
        for (int k = 0; k < n; k++) out_batch[k] = ord[k];
        *n_batch = n; *out_pred = fallback; *out_smin = INFINITY;
        free(ord); return 0;
    }
    double smin = INFINITY;
    for (int k = 0; k < n; k++) {
        double sl = ((double)(tpot * (n_gen[k] + 1)) - (t_now - t_first[k])) - fallback;
        if (sl < smin) smin = sl;
    }
    int nbch = 0, nd = 0; double tcur = 0.0;
    for (int k = 0; k < n; k++) {
        int r = ord[k];
        double ts = lut_lookup(&L, nbch + 1, seq_len[r]);
        if (ts <= smin && (nbch == 0 || (double)(nbch + 1) / ts > (double)nbch / tcur)) {
            out_admit[nbch] = ts; out_batch[nbch++] = r; tcur = ts;
        } else out_delayed[nd++] = r;
    }
    *out_smin = smin;
    if (nbch == 0) {
        for (int k = 0; k < n; k++) out_batch[k] = ord[k];
        *n_batch = n; *n_delayed = 0; *out_pred = fallback; *out_fb = 1;
    } else { *n_batch = nbch; *n_delayed = nd; *out_pred = tcur; }
    free(ord);
    return 0;
}

/* PREFILL_POLICIES over one snapshot (prefill_sched.py:109-145) */
int oracle_select_prefill(int32_t policy, int32_t n, const int64_t* arrival, const int32_t* input_len,
                          const int64_t* remaining, const int32_t* id_rank, int64_t budget, int64_t t_now,
                          int64_t est_tok, int64_t est_busy, int64_t ttft, int32_t* out_index,
                          int64_t* out_take, int32_t* n_out, double* out_scores) {
    if (budget < 1) return SLOSIM_EINVAL;
    int* ord = malloc((size_t)(n > 0 ? n : 1) * sizeof(int));
    double* sc = malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
    for (int k = 0; k < n; k++) ord[k] = k;
#define FLESS(a, b) (arrival[a] != arrival[b] ? arrival[a] < arrival[b] : id_rank[a] < id_rank[b])
    for (int a = 1; a < n; a++) {
        int x = ord[a], b = a - 1;
        while (b >= 0 && FLESS(x, ord[b])) { ord[b + 1] = ord[b]; b--; }
        ord[b + 1] = x;
    }
    if (policy == SLOSIM_PREFILL_KAIROS_URGENCY) {
        int64_t cursor = t_now;
        for (int c = 0; c < n; c++) {
            int k = ord[c];
            cursor = (cursor > arrival[k] ? cursor : arrival[k]) + est_duration(est_tok, est_busy, remaining[k]);
            double u = idiv(ttft - (cursor - arrival[k]), ttft);
            sc[k] = u >= 0 ? u / (double)input_len[k] : u * (double)input_len[k];
            if (out_scores) out_scores[k] = sc[k];
        }
        for (int a = 1; a < n; a++) {
            int x = ord[a], b = a - 1;
            while (b >= 0 && (-sc[x] < -sc[ord[b]] || (-sc[x] == -sc[ord[b]] && FLESS(x, ord[b])))) { ord[b + 1] = ord[b]; b--; }
            ord[b + 1] = x;
        }
    } else if (policy == SLOSIM_PREFILL_SJF) {
        for (int a = 1; a < n; a++) {
            int x = ord[a], b = a - 1;
            while (b >= 0 && (remaining[x] < remaining[ord[b]] || (remaining[x] == remaining[ord[b]] && FLESS(x, ord[b])))) {
                ord[b + 1] = ord[b]; b--;
            }
            ord[b + 1] = x;
        }
    }
#undef FLESS
    int k = 0; int64_t left = budget;
    for (int c = 0; c < n; c++) {
        if (left == 0) break;
        int64_t take = remaining[ord[c]] < left ? remaining[ord[c]] : left;
        if (take <= 0) continue;
        out_index[k] = ord[c]; out_take[k] = take; k++; left -= take;
    }
    *n_out = k;
    free(ord); free(sc);
    return 0;
}

int oracle_predict_finish(int32_t n, const int64_t* arrival, const int64_t* remaining, int64_t t_now,
                          int64_t est_tok, int64_t est_busy, int64_t* out) {
    int64_t cursor = t_now;
    for (int k = 0; k < n; k++) {
        cursor = (cursor > arrival[k] ? cursor : arrival[k]) + est_duration(est_tok, est_busy, remaining[k]);
        out[k] = cursor;
    }
    return 0;
}

int oracle_estimate_duration(int64_t tok, int64_t busy, int64_t n, const int64_t* tokens, int64_t* out) {
    for (int64_t k = 0; k < n; k++) out[k] = est_duration(tok, busy, tokens[k]);
    return 0;
}

double oracle_idiv(int64_t p, int64_t q) { return idiv(p, q); }

/* synth_profile_from_anchors costmodel.py:271-309 (buckets preset in *P). */
int oracle_synth_profile(slosim_profile_t* P, int32_t na, const int64_t* ab, const int64_t* as,
                         const double* aus, double gamma, int64_t w) {
    int64_t bx[SLOSIM_MAX_BASE_POINTS]; double by[SLOSIM_MAX_BASE_POINTS]; int nbase = 0;
    for (int k = 0; k < na; k++) {
        if (ab[k] != 1) continue;
        if (nbase >= SLOSIM_MAX_BASE_POINTS) return SLOSIM_EINVAL;
        /* sorted((seq, float(us))) — insertion by (seq, us) */
        int b = nbase++;
        while (b > 0 && (bx[b - 1] > as[k] || (bx[b - 1] == as[k] && by[b - 1] > aus[k]))) {
            bx[b] = bx[b - 1]; by[b] = by[b - 1]; b--;
        }
        bx[b] = as[k]; by[b] = aus[k];
    }
    if (nbase == 0) return SLOSIM_EINVAL;
    for (int i = 0; i < SLOSIM_MAX_BSZ_BUCKETS * SLOSIM_MAX_SEQ_BUCKETS; i++) { P->lut_sums[i] = 0; P->lut_counts[i] = 0; }
    if (w == 0) return 0;
    for (int i = 0; i < P->nb; i++)
        for (int j = 0; j < P->ns; j++) {
            double f = interp_clamped(nbase, bx, by, P->seq_buckets[j]) * (1.0 + gamma * (double)(P->bsz_buckets[i] - 1));
            int64_t v = round_half_even(f);
            if (v < 1) v = 1;
            P->lut_sums[CELL(i, j)] = (double)(v * w);
            P->lut_counts[CELL(i, j)] = (int32_t)w;
        }
    for (int k = 0; k < na; k++) {
        int i = bucket_index(P->bsz_buckets, P->nb, ab[k]), j = bucket_index(P->seq_buckets, P->ns, as[k]);
        P->lut_sums[CELL(i, j)] = aus[k] * (double)w;
        P->lut_counts[CELL(i, j)] = (int32_t)w;
    }
    return 0;
}

uint64_t oracle_pcg_next(uint64_t* st4) {
    Pcg64 g = {(((unsigned __int128)st4[0]) << 64) | st4[1], (((unsigned __int128)st4[2]) << 64) | st4[3]};
    uint64_t r = pcg_next(&g);
    st4[0] = (uint64_t)(g.state >> 64); st4[1] = (uint64_t)g.state;
    return r;
}
