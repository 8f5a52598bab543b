/*
 * slosim_b200.h — C-ABI of the B200-native batched Kairos scheduling simulator.
 *
 * This is the drop-in boundary for the hot path of the reference `slosim`
 * package (/root/reference/pkg/src/slosim).  The reference is pure Python; the
 * entry points below replace, one-for-one, the reference interfaces cited on
 * each declaration.  Signatures use plain C types and caller-owned memory
 * only (no torch types).  All pointers named `d_*` are DEVICE pointers; the
 * `slosim_run_batch_host` entry point takes HOST pointers and does the copies
 * itself.  Every function returns a SLOSIM_* status code and never throws.
 *
 * Time is integer microseconds (int64) everywhere, as in domain.py:14-17.
 */
#ifndef SLOSIM_B200_H
#define SLOSIM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SLOSIM_ABI_VERSION 2

/* Status codes: mirror the CLI exit codes of cli.py:1-5 (0 ok, 2 invalid input,
 * 3 configuration error — ConfigurationError domain.py:32-33). */
#define SLOSIM_OK 0
#define SLOSIM_EINVAL 2
#define SLOSIM_ECONFIG 3
#define SLOSIM_ECUDA 4
#define SLOSIM_ENOMEM 5
#define SLOSIM_ERANGE 6  /* a generated value left the covered range (gen_longtail: token count > int32) */

/* Grid limits of the decode step LUT (costmodel.py:26-27 default 9 x 32). */
#define SLOSIM_MAX_BSZ_BUCKETS 16
#define SLOSIM_MAX_SEQ_BUCKETS 64
#define SLOSIM_MAX_CURVE_POINTS 16
#define SLOSIM_MAX_BASE_POINTS 16

/* Policy ids (prefill_sched.py:141-145, decode_sched.py:127-130). */
#define SLOSIM_PREFILL_FCFS 0
#define SLOSIM_PREFILL_SJF 1
#define SLOSIM_PREFILL_KAIROS_URGENCY 2
#define SLOSIM_DECODE_CONTINUOUS 0
#define SLOSIM_DECODE_KAIROS_SLACK 1

/* Event-trace record kinds (engine.py:41-47 EventKind + the Admit log line
 * engine.py:369).  Trace records are int64 words:
 *   ARRIVAL        : [0, t, pos]
 *   TRANSFER_DONE  : [1, t, pos]
 *   PREFILL_DONE   : [2, t, duration, k, (pos<<32 | take) x k]     (batch order)
 *   DECODE_DONE    : [3, t, duration, bsz, max_seq, pos x bsz]    (any order)
 *   ADMIT          : [4, t, pos, first_token_us]
 *   END            : [5, words_needed]                            (terminator)
 */
#define SLOSIM_EV_ARRIVAL 0
#define SLOSIM_EV_TRANSFER_DONE 1
#define SLOSIM_EV_PREFILL_DONE 2
#define SLOSIM_EV_DECODE_DONE 3
#define SLOSIM_EV_ADMIT 4
#define SLOSIM_EV_END 5

/* Cost profile: everything CostProfile (engine.py:54-101) resolves to.
 * `lut_sums/lut_counts` is the scheduler's initial DecodeStepLUT
 * (costmodel.py:61-227) in row-major [nb][ns]; a count of 0 is an unpopulated
 * cell.  `gt_*` is the engine ground truth (_GroundTruth, engine.py:135-192). */
typedef struct slosim_profile {
    int32_t nb, ns;
    int32_t bsz_buckets[SLOSIM_MAX_BSZ_BUCKETS];
    int32_t seq_buckets[SLOSIM_MAX_SEQ_BUCKETS];
    double lut_sums[SLOSIM_MAX_BSZ_BUCKETS * SLOSIM_MAX_SEQ_BUCKETS];
    int32_t lut_counts[SLOSIM_MAX_BSZ_BUCKETS * SLOSIM_MAX_SEQ_BUCKETS];
    /* PrefillThroughputEstimator seed (costmodel.py:237-241) */
    int64_t est_tokens, est_busy_us;
    /* ground-truth prefill curve incl. the (0,0) origin, sorted (engine.py:143-149) */
    int32_t n_curve;
    int32_t _pad0;
    int64_t curve_x[SLOSIM_MAX_CURVE_POINTS];
    int64_t curve_y[SLOSIM_MAX_CURVE_POINTS];
    /* ground-truth decode base curve: sorted bsz==1 anchors (engine.py:153-155) */
    int32_t n_base;
    int32_t gt_frozen; /* 1: ground truth decode = frozen file LUT (engine.py:141-142,186-187) */
    int64_t base_x[SLOSIM_MAX_BASE_POINTS];
    double base_y[SLOSIM_MAX_BASE_POINTS];
    double gamma;     /* batch_growth */
    double noise_eps; /* decode_noise_eps (engine.py:190-191) */
    double gt_sums[SLOSIM_MAX_BSZ_BUCKETS * SLOSIM_MAX_SEQ_BUCKETS];
    int32_t gt_counts[SLOSIM_MAX_BSZ_BUCKETS * SLOSIM_MAX_SEQ_BUCKETS];
} slosim_profile_t;

/* One simulated serving instance: one (trace, rate, SLO, policy pair) point —
 * a ClusterConfig (engine.py:104-132) applied to one workload. */
typedef struct slosim_instance {
    int64_t trace_offset;     /* first request of this instance's trace in the trace table */
    int32_t n_requests;
    int32_t profile_id;
    double rescale_factor;    /* >0: arrival = rint(base_arrival * factor) (workload.py:175-182); <=0: as is */
    int64_t ttft_slo_us, tpot_slo_us;
    int64_t kv_capacity_tokens;
    int64_t transfer_base_us;
    double transfer_per_token_us;
    int32_t chunk_budget;
    int8_t prefill_policy;
    int8_t decode_policy;
    int8_t _pad1[2];
    uint64_t rng_state_hi, rng_state_lo, rng_inc_hi, rng_inc_lo; /* numpy PCG64 state (engine.py:225) */
    int64_t row_offset;       /* per-request output rows start here (if rows requested) */
    int64_t trace_buf_offset; /* event-trace words start here (if tracing); -1 = not traced */
    int64_t trace_buf_words;  /* capacity of this instance's trace region */
} slosim_instance_t;

/* Trace table (SoA, device or host memory as the call states).  Within one trace
 * requests are sorted by (arrival_time, id) (workload.py:111, engine.py:206-208);
 * `id_rank` is the rank of the request id string inside its trace. */
typedef struct slosim_traces {
    const int64_t* arrival_us;
    const int32_t* input_len;
    const int32_t* output_len;
    const int32_t* prefix_hit_len;
    const int32_t* id_rank;
    int64_t n_total;
} slosim_traces_t;

/* Per-instance result: MetricsReport (metrics.py:95-106) reduced to counts, plus
 * the decision digest and the byte-model counters of SURVEY §8(d). */
typedef struct slosim_summary {
    int32_t status;           /* SLOSIM_OK; SLOSIM_ECONFIG (unrunnable config, engine.py:218-232);
                                 SLOSIM_EINVAL (malformed descriptor: n_requests > max_requests, profile_id
                                 out of range, trace range outside the trace table, bad policy id, ...);
                                 bit 8 set: trace buffer overflow */
    int32_t n;
    int32_t ttft_met, tpot_met, e2e_met, n_tps;
    double tps_p50, tps_p90;  /* NaN when no request has output_len >= 2 */
    int64_t worst_queue_wait_us;
    int64_t prefill_steps, decode_steps;
    uint64_t digest;
    int64_t v_dec, b_dec, v_pre; /* Σ|active| per decode step, Σ|batch|, Σ|queue| per prefill step */
    int64_t deadline_misses;
    int64_t t_end_us;
    int64_t est_tokens, est_busy_us; /* final estimator state */
    int32_t max_queue, max_active;
    int64_t sim_cycles;       /* SM clock cycles the instance occupied its warp (load-balance diagnostics) */
} slosim_summary_t;

/* Optional per-request rows (RequestMetrics metrics.py:14-23 + lifecycle times),
 * indexed by instance.row_offset + position-in-trace.  Any pointer may be NULL. */
typedef struct slosim_rows {
    int64_t* ttft_us;
    double* mean_tpot_us;
    double* decode_tps;       /* NaN = None */
    uint8_t* met_flags;       /* bit0 ttft, bit1 tpot, bit2 e2e */
    int32_t* deadline_misses;
    int64_t* t_prefill_finish;
    int64_t* t_first_token;
    int64_t* t_last_token;
    int64_t* first_sched_us;
} slosim_rows_t;

typedef struct slosim_batch {
    slosim_traces_t traces;
    const slosim_profile_t* profiles;
    int32_t n_profiles;
    int32_t flags;            /* SLOSIM_F_* */
    const slosim_instance_t* instances;
    int64_t n_instances;
    slosim_summary_t* summaries;
    slosim_rows_t rows;
    int64_t* trace_buf;       /* event-trace words (NULL = no tracing) */
    double* lut_out_sums;     /* optional final LUT per instance [n_instances][16*64] */
    int32_t* lut_out_counts;
    int64_t max_requests;     /* max n_requests over instances (sizes the per-warp workspace); <= 0: computed */
    const int64_t* order;     /* optional processing order (permutation of instance ids); NULL = identity.
                                 Entries outside [0, n_instances) are skipped. */
    int64_t rows_capacity;    /* length of each rows.* array (0 = unchecked) */
    int64_t trace_buf_capacity; /* words in trace_buf (0 = unchecked) */
} slosim_batch_t;

#define SLOSIM_F_ROWS 1          /* write per-request rows */
#define SLOSIM_F_EXPORT_LUT 2    /* export final LUT (Simulation.lut, engine.py:218) */
#define SLOSIM_F_ALWAYS_LUT 4    /* update the LUT even under continuous batching */

/* ---------------------------------------------------------------- engine ---
 * Replaces Simulation.run (engine.py:261-284) / run() (engine.py:416-420),
 * batched over instances (the qps x policy loop of cli.py:130-138).
 * All pointers in `batch` are DEVICE pointers; stream is a cudaStream_t.
 * Stream-ordered: the call enqueues work and returns.  Every instance descriptor
 * is validated on the device; a malformed one gets summary status SLOSIM_EINVAL
 * and touches no memory outside its own summary row.  Launches on one device
 * are serialised in stream order (a launch waits for the previous launch's
 * completion, whatever stream it used), so concurrent callers are safe. */
int slosim_run_batch(const slosim_batch_t* batch, void* stream);

/* Same, with HOST pointers: copies in, runs, copies out, synchronizes.
 * `elapsed_ms` (may be NULL) receives the device time of the kernels alone. */
int slosim_run_batch_host(const slosim_batch_t* host_batch, float* elapsed_ms);

/* Bytes of device workspace slosim_run_batch allocates for a batch. */
int64_t slosim_workspace_bytes(const slosim_batch_t* batch);

/* ------------------------------------------------------ cost models (A3-A6) */
/* Replaces synth_profile_from_anchors (costmodel.py:271-309): fills
 * lut_sums/lut_counts of *profile (host pointer) from decode anchors. */
int slosim_synth_profile(slosim_profile_t* profile, int32_t n_anchors,
                         const int64_t* anchor_bsz, const int64_t* anchor_seq,
                         const double* anchor_us, double batch_growth, int64_t prior_weight);

/* Replaces DecodeStepLUT.lookup (costmodel.py:157-187), batched: out[k] =
 * lookup(bsz[k], seq[k]) on the LUT given by buckets/sums/counts (host pointers). */
int slosim_lut_lookup(int32_t nb, const int32_t* bsz_buckets, int32_t ns, const int32_t* seq_buckets,
                      const double* sums, const int32_t* counts, int64_t n,
                      const int64_t* bsz, const int64_t* seq, double* out);

/* Replaces decode_step_formula (costmodel.py:50-58), batched (host pointers). */
int slosim_decode_formula(int32_t n_base, const int64_t* base_x, const double* base_y, double gamma,
                          int64_t n, const int64_t* bsz, const int64_t* seq, double* out);

/* Replaces PrefillThroughputEstimator.estimate_duration_us (costmodel.py:261-268). */
int slosim_estimate_duration(int64_t total_tokens, int64_t total_busy_us, int64_t n,
                             const int64_t* tokens, int64_t* out);

/* ------------------------------------------------- policy snapshots (A7-A12)
 * Test-level entry points over one snapshot (host pointers). */

/* Replaces predict_finish_times (prefill_sched.py:39-56): `order` must hold the
 * queue in FCFS order; out_finish[k] is the finish of queue entry k. */
int slosim_predict_finish(int32_t n, const int64_t* arrival, const int64_t* remaining,
                          int64_t t_now, int64_t est_tokens, int64_t est_busy, int64_t* out_finish);

/* Replaces PREFILL_POLICIES[p](queue, budget, t_now, est, slo) (prefill_sched.py:109-145).
 * Queue entries in any order; keys are (arrival, id_rank).  Writes the selected
 * entries (queue index, take) in batch order; *n_out receives the count. */
int slosim_select_prefill(int32_t policy, int32_t n, const int64_t* arrival, const int32_t* input_len,
                          const int64_t* remaining, const int32_t* id_rank, int64_t budget, int64_t t_now,
                          int64_t est_tokens, int64_t est_busy, int64_t ttft_slo_us,
                          int32_t* out_index, int64_t* out_take, int32_t* n_out, double* out_scores);

/* Replaces DECODE_POLICIES[p](active, t_now, slo, lut) (decode_sched.py:60-130).
 * t_now and t_first are f64 so the float-time decode loop of tests/oracles.py:33-68
 * is reproduced exactly.  Outputs: batch (active indices, admission order),
 * delayed (scan order), admission step times, predicted step time, s_min, fallback. */
int slosim_select_decode(int32_t policy, int32_t n, const int64_t* seq_len, const int32_t* id_rank,
                         const int64_t* n_gen, const double* t_first, double t_now, int64_t tpot_slo_us,
                         int32_t nb, const int32_t* bsz_buckets, int32_t ns, const int32_t* seq_buckets,
                         const double* sums, const int32_t* counts,
                         int32_t* out_batch, int32_t* n_batch, int32_t* out_delayed, int32_t* n_delayed,
                         double* out_admit_times, double* out_pred, double* out_smin, int32_t* out_fallback);

/* Replaces _GroundTruth.prefill_batch_us (engine.py:175-183). */
int slosim_prefill_batch_us(int32_t n_curve, const int64_t* curve_x, const int64_t* curve_y,
                            int32_t k, const int64_t* done_before, const int64_t* take, int64_t* out_us);

/* ----------------------------------------------------------- metrics (A18-A19)
 * Replaces request_metrics + aggregate (metrics.py:72-144) over explicit token
 * timestamps (CSR: ts_offsets[n+1]).  Times are f64 so both the int-µs engine and
 * float-time callers (tests/oracles.py:33-68) are reproduced exactly (integers
 * below 2^53 convert exactly, so int/int true division is matched). */
int slosim_request_metrics(int64_t n, const double* arrival, const int64_t* output_len,
                           const int64_t* ts_offsets, const double* ts, int64_t ttft_slo_us,
                           int64_t tpot_slo_us, double* ttft_us, double* mean_tpot, double* tps,
                           uint8_t* met_flags, int32_t* misses, double* agg /* [5]: att x3, p50, p90 */);

/* K6 pre-collective step: hist[cell[k]][e2e_met of instance k] += 1 over a device
 * summary array (int64 histogram, DEVICE pointers, stream-ordered).  The histogram is
 * then summed across GPUs with an integer all-reduce (bit-exact in any order). */
int slosim_histogram(int64_t n, const slosim_summary_t* d_summaries, const int32_t* d_cell, int32_t n_bins,
                     int64_t* d_hist, void* stream);

/* Replaces the final merge of a sharded sweep (the C-ABI form of
 * paper_2605_02329_b200.dist.exchange): over the caller's NCCL communicator
 * (`nccl_comm` is an ncclComm_t), sum-all-reduce the int64 histogram d_hist[n_hist]
 * in place and all-gather n_mine summary rows per rank from d_mine into d_all
 * (rank order, n_mine * world rows).  DEVICE pointers, stream-ordered; integer sums
 * make the result independent of the rank count.  NCCL (libnccl.so.2) is resolved
 * at run time; returns SLOSIM_ECUDA with slosim_last_error() if it is missing. */
int slosim_exchange(void* nccl_comm, const slosim_summary_t* d_mine, int64_t n_mine, slosim_summary_t* d_all,
                    int64_t* d_hist, int64_t n_hist, void* stream);

/* ------------------------------------------------ workload generation (§8(f)4)
 * LongTailSpec (workload.py:52-85): the fields of the reference dataclass, plus
 * where the trace goes in the output trace table. */
typedef struct slosim_longtail_spec {
    double qps;
    int64_t n_requests;
    double short_len_log_mean;
    double short_len_log_sigma;
    double p_long;
    int64_t long_len_min;
    int64_t long_len_max;
    double out_len_log_mean;
    double out_len_log_sigma;
    uint64_t seed;      /* default_rng(seed); 0 <= seed < 2^64 */
    int64_t offset;     /* first request's position in the output arrays */
} slosim_longtail_spec_t;

/* Replaces gen_longtail (workload.py:88-112), batched over specs: trace i is written
 * at [offset_i, offset_i + n_requests_i) of the output SoA, in (arrival, id) order,
 * with prefix_hit_len = 0 and id_rank = position (ids r{k:0w} sort by position).
 * The draws are numpy's (default_rng(seed): SeedSequence, PCG64, ziggurat
 * exponential/normal, Lemire integers; glibc exp/log1p), so the trace is identical
 * to the reference's.  d_status[i]: SLOSIM_OK, SLOSIM_EINVAL (spec fails
 * LongTailSpec's checks, tail range >= 2^32 - 1, or out of the table) or
 * SLOSIM_ERANGE.  DEVICE pointers, stream-ordered. */
int slosim_gen_longtail(const slosim_longtail_spec_t* d_specs, int64_t n_specs, int64_t* d_arrival_us,
                        int32_t* d_input_len, int32_t* d_output_len, int32_t* d_prefix_hit_len,
                        int32_t* d_id_rank, int64_t n_total, int32_t* d_status, void* stream);

/* Same with HOST pointers (copies in and out, synchronizes). */
int slosim_gen_longtail_host(const slosim_longtail_spec_t* specs, int64_t n_specs, int64_t* arrival_us,
                             int32_t* input_len, int32_t* output_len, int32_t* prefix_hit_len,
                             int32_t* id_rank, int64_t n_total, int32_t* status);

/* Test-level: n_per_seed draws of one Generator method for each default_rng(seed),
 * computed on the device (HOST pointers; out[i * n_per_seed + k], f64 results as
 * their bit patterns).  INTEGERS draws integers(p0, p1) (high exclusive, range below
 * 2^32 - 1); EXPONENTIAL uses scale p0; LOGNORMAL mean p0, sigma p1. */
#define SLOSIM_DRAW_RAW 0
#define SLOSIM_DRAW_RANDOM 1
#define SLOSIM_DRAW_STD_EXPONENTIAL 2
#define SLOSIM_DRAW_EXPONENTIAL 3
#define SLOSIM_DRAW_STD_NORMAL 4
#define SLOSIM_DRAW_LOGNORMAL 5
#define SLOSIM_DRAW_INTEGERS 6
int slosim_rng_draws(int32_t kind, const uint64_t* seeds, int64_t n_seeds, int64_t n_per_seed, double p0,
                     double p1, uint64_t* out, int32_t* status);

/* Test-level: the device restatement of libm exp (fn 0) / log1p (fn 1) that the
 * draws use, over x[n] (HOST pointers); ok[k] = 0 outside the restated domain. */
int slosim_libm(int32_t fn, int64_t n, const double* x, double* y, uint8_t* ok);

/* Library identity (ABI version, sm arch compiled for) and visible CUDA devices. */
int slosim_abi_version(void);
int slosim_device_count(void);
const char* slosim_build_info(void);

/* Text of the last CUDA error of this thread (valid after a SLOSIM_ECUDA return). */
const char* slosim_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* SLOSIM_B200_H */
