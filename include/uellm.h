/*
 * include/uellm.h -- C ABI of the B200-native UELLM batch scheduler (libuellm.so).
 *
 * UELLM (arXiv 2409.14961) Sec. 4.2: the batch scheduler receives "a list of requests after
 * profiling" and outputs "a list of batch" (Alg. 1).  This library
 * computes that step as a data-parallel GPU path on sm_100a:
 *
 *   uellm_profile_load      validate the profiled queries (input length, predicted output
 *                           length, SLO), convert SLO to integer microseconds, pack sort keys
 *   uellm_schedule_batches  sort by (SLO, predicted length) and segment the
 *                           sorted stream into batches (SEG-DP / Alg. 1 / FIFO / sort-only)
 *   uellm_batch_stats       per-batch padding, generated tokens (b x O), KV-cache peak
 *                           bytes (4*b*l*h*(s+n)), estimated latency and SLO violations
 *   uellm_schedule_pipelined  the three calls for host-resident queries, window groups
 *                           pipelined against the PCIe copies
 *
 * and the adjacent steps of SURVEY.md section 8(f):
 *   uellm_simulate          (f2) sequential execution of a schedule with arrivals: latency, SLO
 *                           violations, utilisation, throughput
 *   uellm_predict_lengths   (f4) profiler stand-ins + misprediction monitor that produce the
 *                           predicted output lengths
 *   uellm_helr_plan         (f3) HELR deployer: layer placement on a device chain (
 *                           S:341-400)
 *
 * Citations: P:NNN = /root/reference/PAPER.md line; S:NNN = SPEC.md line; Rk = reading k in
 * DESIGN.md.  The C ABI is plain: no exceptions, no C++ or torch types, no device allocation,
 * no global state except the pipelined call's reused streams / events.  All device work is stream-ordered on `stream` (a cudaStream_t passed as void*,
 * NULL = legacy default stream).
 *
 * Pointers: each pointer argument is marked [host], [device] or [host|device].  [host|device]
 * pointers are classified with cudaPointerGetAttributes: device/managed memory is used in
 * place; host memory (pinned or pageable) is staged through the workspace with
 * cudaMemcpyAsync on `stream`, and a call with a host OUTPUT synchronises `stream` before it
 * returns.  Ownership: the caller owns every buffer; the library never frees or retains them.
 *
 * Errors: every call returns a uellm_status.  Outputs are written only when the call returns
 * UELLM_OK.  Argument, configuration and launch errors are detected synchronously.
 * uellm_profile_load is the only call that always synchronises (it reads a 64-byte validation
 * record back from the device); schedule/stats with device outputs never synchronise.
 */
#ifndef UELLM_H_
#define UELLM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define UELLM_ABI_VERSION 3u

typedef int32_t uellm_status;
enum {
    UELLM_OK = 0,
    UELLM_ERR_ARG = 1,          /* NULL / misaligned pointer, workspace too small, n >= 2^32 - 1   */
    UELLM_ERR_CONTRACT = 2,     /* a query violates its invariants: input_len == 0,
                                   pred_out_len == 0, SLO not finite / <= 0, or slo_us outside
                                   [1, 2^32-1] ("contract error", S:98 typed rejection)     */
    UELLM_ERR_CONFIG = 3,       /* config invariant violated                       */
    UELLM_ERR_OVERFLOW = 4,     /* a KV-byte or cost bound could overflow 64 bits          */
    UELLM_ERR_CUDA = 5,         /* a CUDA runtime call or kernel launch failed                     */
    UELLM_ERR_UNSUPPORTED = 6,  /* valid, but outside this build's limits (e.g. max_batch > 4096)  */
    UELLM_ERR_STALE = 7         /* uellm_profile_reload: the new queries need other decisions than
                                   the profile holds (larger maxima, an SLO value outside the
                                   profile's set / other set size, new varying key bits): load
                                   them with uellm_profile_load                                  */
};

/* Segmentation of the sorted stream (uellm_config.mode). */
enum {
    UELLM_MODE_SEG_DP = 0,      /* exact min over contiguous segmentations of the (SLO, length)-
                                   sorted window of sum_batches est_us + lambda * violations, under
                                   b <= max_batch and the KV cap (R7, R8, R14) */
    UELLM_MODE_SLO_ODBS = 1,    /* Alg. 1 literal (readings R1-R5); SLO-DBS = w1 = 0,
                                   ODBS = w2 = 0                                            */
    UELLM_MODE_FIFO = 2,        /* default batching baseline: arrival order, chunks of W    */
    UELLM_MODE_SORT_ONLY = 3    /* sorted order, every query its own batch                          */
};

/* Profiled queries, caller SoA (input_len >= 1, predicted output length >= 1,
 * slo > 0 seconds).  Element k is the query with arrival index k. */
typedef struct {
    uint64_t n;                     /* number of queries, < 2^32 - 1                         */
    const uint32_t *input_len;      /* [host|device] n x Input_i (tokens)             */
    const uint32_t *pred_out_len;   /* [host|device] n x predicted Output_i (tokens)  */
    const float *slo_s;             /* [host|device] n x SLO_i in seconds            */
} uellm_queries;

/* Scheduler configuration.  Same meaning in every mode unless noted. */
typedef struct {
    uint32_t mode;                  /* UELLM_MODE_*                                                */
    uint32_t window;                /* queries per scheduling window (consecutive arrival chunks,
                                       R15); 0 = one window of all n.  No batch crosses a window. */
    uint32_t max_batch;             /* W >= 1, maximum batch size; <= 4096 in this build          */
    uint32_t split_on_slo_change;   /* 0|1: 1 = batches never mix SLO values (R15)                 */
    uint32_t kv_bytes_per_elem;     /* the "4" of 4*b*l*h*(s+n) (R13)                        */
    uint32_t n_layers;              /* l                                                    */
    uint32_t hidden;                /* h                                                    */
    uint32_t dp_tile;               /* SEG-DP tile length in queries, 0 = automatic; otherwise
                                       rounded up to a multiple of max_batch and >= 2*max_batch.
                                       A tuning knob: results are identical for every value.       */
    uint64_t kv_cap_bytes;          /* per-batch KV reserve T of P:366 (R6); 0 = no cap.  A batch
                                       of b >= 2 queries is admissible iff
                                       kv_bytes_per_elem*b*l*h*(s+O) <= kv_cap_bytes; a single
                                       query is always admissible (R10).                           */
    uint32_t t_batch_us;            /* service-time model est_us = t_batch + t_iter*O            */
    uint32_t t_iter_us;             /*      + t_tok*b*O + t_prefill*b*s   (R7; b batch size,       */
    uint32_t t_tok_us;              /*      s max input, O max predicted output)            */
    uint32_t t_prefill_us;
    uint64_t lambda_us;             /* SEG-DP penalty per query whose slo_us < est_us of its own
                                       batch (R8, R14)                                             */
    double w1, w2;                  /* Alg. 1 weights; w1, w2 >= 0, w1 + w2 > 0        */
    double l1, l2;                  /* Alg. 1 overheads L1, L2, >= 0                 */
    double threshold;               /* Alg. 1 Threshold, > 0                               */
    double eps;                     /* Alg. 1 line 20 dynamic-cap guard (R5), > 0                   */
    uint32_t eq2_additive;          /* 0|1: Alg. 1 T_o with Eq. 2's '+' instead of '-' (R2)        */
    uint32_t flags;                 /* bit 0: force the generic 64-bit SEG-DP kernels (testing; same
                                       results); other bits must be 0                               */
} uellm_config;

/* One batch (UELLM_MODE_*: batch t = order[batch_offsets[t] .. batch_offsets[t+1])). 80 bytes. */
typedef struct {
    uint32_t start;                 /* first scheduled position of the batch                       */
    uint32_t size;                  /* b                                                            */
    uint32_t max_in;                /* s = max Input_i, the padded input length             */
    uint32_t max_out;               /* O = max predicted Output_i                           */
    uint64_t gen_tokens;            /* b x O                                                */
    uint64_t pad_in;                /* sum (s - Input_i): input padding tokens       */
    uint64_t pad_out;               /* sum (O - Output_i): redundant generated tokens               */
    uint64_t kv_bytes;              /* kv_bytes_per_elem * b * l * h * (s + O)               */
    uint64_t est_us;                /* estimated service time (R7)                                  */
    uint64_t completion_us;         /* inclusive prefix of est_us over the window's batches
                                       (sequential execution, all queries present at t=0)  */
    uint32_t viol_alone;            /* members with slo_us < est_us                                 */
    uint32_t viol_seq;              /* members with slo_us < completion_us                          */
    uint32_t over_cap;              /* 1 if kv_cap_bytes != 0 and kv_bytes > kv_cap_bytes          */
    uint32_t window;                /* window index                                                 */
} uellm_batch_stat;

/* Totals over all batches. */
typedef struct {
    uint64_t n, batches, gen_tokens, pad_in, pad_out;
    uint64_t kv_bytes_max;
    uint64_t dp_cost;               /* sum_batches (est_us + lambda_us * viol_alone): the SEG-DP
                                       objective of this schedule                                  */
    uint64_t viol_alone, viol_seq, over_cap;
    uint64_t makespan_us;           /* sum of est_us                                        */
    double mean_latency_s;          /* sum over queries of completion_us(batch) / n * 1e-6          */
    double throughput_tok_s;        /* gen_tokens / (makespan_us * 1e-6)                            */
    uint64_t latency_sum_lo;        /* exact 128-bit sum over queries of completion_us(batch), the  */
    uint64_t latency_sum_hi;        /*   numerator of mean_latency_s (lets totals combine exactly) */
    uint64_t overflow;              /* bit i set iff the i-th u64 field above (n = bit 0 ...
                                       makespan_us = bit 10) did not fit 64 bits and saturated at
                                       2^64 - 1 (only dp_cost and makespan_us can: the load bounds
                                       one window, not the whole job); 0 normally                 */
} uellm_totals;                     /* 128 bytes: also the head of the a9 exchange record          */

/* Diagnostics of the last uellm_schedule_batches call on a profile (SEG-DP internals). */
typedef struct {
    uint64_t tiles;                 /* SEG-DP tiles                                                 */
    uint64_t tile_len;              /* tile length (queries)                                        */
    uint64_t fixups_unconverged;    /* tiles whose parallel fix-up did not converge in the tile     */
    uint64_t cascade_reruns;        /* sequential fix-up re-runs performed by the cascade           */
    uint64_t fixup_positions;       /* positions re-evaluated by fix-ups (parallel + cascade)      */
    uint64_t trace_unmerged;        /* traceback tiles whose walk did not coalesce in the tile      */
    uint64_t trace_rewalks;         /* full tile re-walks performed by the traceback cascade        */
    uint64_t sort_passes;           /* radix passes actually run (constant digits are skipped)      */
    uint64_t dp_cost;               /* SEG-DP: sum over windows of the optimal cost C[w1]; else 0   */
    uint64_t dp_candidate_evals;    /* SEG-DP: breakpoint candidates evaluated (all passes)         */
    uint64_t sched_launches;        /* kernels launched by the last uellm_schedule_batches          */
    uint64_t stats_launches;        /* kernels launched by the last uellm_batch_stats               */
    uint64_t sort_key_bits;         /* sort key width: bits(rank) + bits(max_out) when the distinct
                                       SLO values (<= 1024) were rank-compressed, else 64          */
    uint64_t dp_filled_positions;   /* SEG-DP: boundaries written by the periodic fill of uniform
                                       stretches (identical records; all passes)                   */
} uellm_diagnostics;

/* Optional per-stage timing.  Stage boundaries at which uellm_schedule_batches /
 * uellm_batch_stats record caller-supplied CUDA events on their stream: */
enum {
    UELLM_STAGE_SCHED_BEGIN = 0,    /* schedule entered                                  */
    UELLM_STAGE_SORT_END = 1,       /* radix sort done (a2/a3)                           */
    UELLM_STAGE_DECODE_END = 2,     /* scheduled-order records written (a4)              */
    UELLM_STAGE_DP_LOCAL_END = 3,   /* SEG-DP local tiles done (a6)                      */
    UELLM_STAGE_DP_FIX_END = 4,     /* SEG-DP fix-ups done                               */
    UELLM_STAGE_DP_CASCADE_END = 5, /* SEG-DP cascade done                               */
    UELLM_STAGE_TRACE_END = 6,      /* traceback / segmentation marks done (a7)          */
    UELLM_STAGE_SCHED_END = 7,      /* batch_offsets written                             */
    UELLM_STAGE_STATS_BEGIN = 8,
    UELLM_STAGE_STATS_END = 9,      /* per-batch stats + totals done (a8)                */
    UELLM_STAGE_COUNT = 10
};

/* Opaque POD view of a loaded profile: pointers into the workspace plus host-side metadata.
 * Valid while the workspace it was loaded into is alive and not reused by another load. */
typedef struct {
    uint64_t opaque[40];
} uellm_profile;

/* ABI version (UELLM_ABI_VERSION) and struct sizes, for bindings to check their layouts. [host] */
uint32_t uellm_abi_version(void);
uint64_t uellm_sizeof(int which);   /* 0 config, 1 batch_stat, 2 totals, 3 profile, 4 diagnostics,
                                       5 sim_totals, 6 predictor, 7 monitor_state,
                                       8 topology, 9 device_map */

/* Human-readable name of a status code.  [host]  Never NULL; static storage. */
const char *uellm_status_string(uellm_status s);

/* Device workspace bytes needed to load and schedule n queries with cfg (a pure function of
 * n, cfg->window, cfg->max_batch, cfg->dp_tile).  [host]  Returns 0 if cfg is NULL.
 * A profile is bound to the cfg it was loaded with: every later call on it must pass a cfg equal
 * in every field (compared through a hash of all fields), else UELLM_ERR_ARG. */
size_t uellm_workspace_bytes(uint64_t n, const uellm_config *cfg);

/* Validate and load n profiled queries (Sec. 4.1 output).
 *   q          [host] query SoA; its arrays are [host|device].  Device arrays are used in place
 *              and must stay unchanged until the last schedule/stats call on the profile.
 *   cfg        [host] configuration; checked here (UELLM_ERR_CONFIG).
 *   ws         [device] workspace of ws_bytes >= uellm_workspace_bytes(n, cfg), 256-B aligned.
 *   out        [host] receives the profile view.
 * Computes slo_us = rint(double(slo_s) * 1e6) (half-even, R12), rejects invalid queries with
 * UELLM_ERR_CONTRACT, and returns UELLM_ERR_OVERFLOW when
 * window * (E + lambda*W) >= 2^63 with E = t_batch + t_iter*max_out +
 * (t_tok*max_out + t_prefill*max_in)*W, or when kv_bytes_per_elem*l*h*W*(max_in+max_out)
 * does not fit 64 bits.  Synchronises `stream` once (64-byte validation record). */
uellm_status uellm_profile_load(const uellm_queries *q, const uellm_config *cfg, void *ws,
                                size_t ws_bytes, void *stream, uellm_profile *out);

/* Load the next n profiled queries into an existing profile WITHOUT a host synchronisation, so
 * that reload -> schedule -> stats can be enqueued (or captured in one CUDA graph) per step.
 *   p          [host] profile from uellm_profile_load with the same n and cfg; updated in place.
 *   q          [host] query SoA whose arrays are [device] (UELLM_ERR_ARG otherwise; same contract
 *              as uellm_profile_load: unchanged until the last call on the profile).
 * The validation of uellm_profile_load runs on the device and its verdict goes to the profile's
 * device status word (uellm_profile_status): UELLM_OK; UELLM_ERR_CONTRACT for an invalid query;
 * UELLM_ERR_STALE when the new queries exceed the decisions the profile was loaded with
 * (max_in or max_out larger; for a profile with the rank-compressed sort key -- at most 1024
 * distinct SLO values -- an SLO value outside the profile's distinct set; otherwise another number
 * of distinct SLO values or a distinct-set overflow, or key bits varying that were constant).
 * Every decision the later calls take from the profile stays valid for queries inside those
 * limits (the cost and KV overflow bounds, the 32-bit DP path and the packed sort payload only
 * need maxima not above the recorded ones; a subset of the SLO set keeps every rank; the radix
 * passes cover every digit that varied before).  For a rank-compressed profile the reload also
 * packs the sort keys and the first radix pass's histogram into the workspace (one pass over the
 * arrays), so the next uellm_schedule_batches calls skip that pass.  The schedule / stats of a
 * step whose status word is not UELLM_OK are undefined: read the word (asynchronously) before
 * using them. */
uellm_status uellm_profile_reload(uellm_profile *p, const uellm_queries *q, const uellm_config *cfg,
                                  void *stream);

/* Device address of the profile's status word (uint32_t, written by uellm_profile_reload). [host] */
uellm_status uellm_profile_status(const uellm_profile *p, uint32_t **device_word);

/* Sort and segment the loaded queries (Alg. 1 stages 1-3; SEG-DP, R14).
 *   p              [host] profile from uellm_profile_load (same cfg).
 *   order          [host|device] n x u32: caller index of the query at scheduled position k.
 *                  Windows ascending; inside a window (slo_us, pred_out_len, index) ascending
 *                  (R11, R9) except UELLM_MODE_FIFO (arrival order).
 *   batch_offsets  [host|device] capacity n+1 x u32: batch t is positions
 *                  [batch_offsets[t], batch_offsets[t+1]); batch_offsets[0] = 0,
 *                  batch_offsets[num_batches] = n.  Batches in scan order.
 *   num_batches    [host|device] 1 x u64.
 * SEG-DP ties: the smallest minimising breakpoint at every position (R9).  The device-side
 * results of the call also remain in the workspace for uellm_batch_stats. */
uellm_status uellm_schedule_batches(const uellm_profile *p, const uellm_config *cfg,
                                    uint32_t *order, uint32_t *batch_offsets,
                                    uint64_t *num_batches, void *stream);

/* Per-batch statistics of the schedule produced by the
 * last uellm_schedule_batches call on p.
 *   batch_offsets, num_batches  [host|device] that call's outputs.  Device pointers may hold
 *                  a caller-modified segmentation of the same order (a batch that crosses a
 *                  window boundary is counted with a linear scan and attributed to the window of
 *                  its first member).  Host pointers are accepted
 *                  only when that schedule call also returned its results to host memory; the
 *                  library then reads the workspace copy it staged them through.
 *   per_batch      [device] capacity num_batches x uellm_batch_stat, or NULL.
 *   totals         [host|device] 1 x uellm_totals.
 * Integer statistics are exact; mean_latency_s and throughput_tok_s are doubles computed from
 * exact 128-bit / 64-bit integer sums.  A job total that does not fit 64 bits (dp_cost or
 * makespan_us of a huge job) saturates and is flagged in totals->overflow; with a HOST totals
 * pointer the call then returns UELLM_ERR_OVERFLOW (the totals are still written). */
uellm_status uellm_batch_stats(const uellm_profile *p, const uellm_config *cfg,
                               const uint32_t *batch_offsets, const uint64_t *num_batches,
                               uellm_batch_stat *per_batch, uellm_totals *totals, void *stream);

/* Totals of a simulated execution (uellm_simulate, NEXT f2). */
typedef struct {
    uint64_t n, batches;
    uint64_t makespan_us;           /* end of the last batch; the timeline starts at 0             */
    uint64_t busy_us;               /* sum of est_us                                        */
    uint64_t idle_us;               /* makespan_us - busy_us: waits for arrivals            */
    uint64_t gen_tokens;            /* sum b x O                                            */
    uint64_t viol;                  /* queries with latency_us > slo_us                     */
    uint64_t latency_max_us;
    uint64_t latency_sum_lo, latency_sum_hi;   /* exact 128-bit sum of latencies (us)           */
    double mean_latency_s;          /* latency sum / n * 1e-6 ("Latency")                     */
    double slo_violation_rate;      /* viol / n                                      */
    double utilization;             /* busy_us / makespan_us                                */
    double throughput_tok_s;        /* gen_tokens / (makespan_us * 1e-6)                    */
    uint32_t status;                /* UELLM_OK, or UELLM_ERR_OVERFLOW if some batch end reached
                                       2^63 us (all other fields are then unspecified)            */
    uint32_t pad;
} uellm_sim_totals;

/* Sequential execution of a schedule on one replica with query arrivals (NEXT f2; PAPER.md
 * P:499 metrics, R19).  Batches run one after another in scan order
 * (windows ascending, then batch order) on one continuous timeline that starts at 0:
 *     start_t = max(end_{t-1}, max_{k in batch t} arrival_us[k])   ("a batch cannot start
 *               before the latest arrival among its members"), end_{-1} = 0,
 *     end_t   = start_t + est_us(t)                                 (service model R7),
 *     latency_k = end_{t(k)} - arrival_us[k], violation iff latency_k > slo_us[k].
 *   p, cfg         as for uellm_batch_stats; the schedule of the last uellm_schedule_batches.
 *   arrival_us     [host|device] n x u64, arrival time of caller query k in microseconds
 *                  (any order; values < 2^63).  Host arrays are staged through the workspace.
 *   order, batch_offsets, num_batches
 *                  [host|device] that schedule call's outputs (host pointers: only when that call
 *                  returned them to host memory; the workspace copies are read).
 *   batch_end_us   [device] capacity num_batches x u64 (end_t), or NULL.
 *   latency_us     [device] n x u64 in SCHEDULED order, or NULL: latency_us[k] is the latency
 *                  of caller query order[k] (coalesced; the caller maps it through `order`).
 *   totals         [host|device] 1 x uellm_sim_totals.
 * Integer results are exact; the doubles are formed once from exact integer sums.  Overflow of
 * the 2^63-us timeline is reported in totals->status (the call itself does not synchronise
 * unless totals is a host pointer). */
uellm_status uellm_simulate(const uellm_profile *p, const uellm_config *cfg, const uint64_t *arrival_us,
                            const uint32_t *order, const uint32_t *batch_offsets,
                            const uint64_t *num_batches, uint64_t *batch_end_us, uint64_t *latency_us,
                            uellm_sim_totals *totals, void *stream);

/* Profiler stand-ins (NEXT f4; R20).  The paper's
 * predictor is a fine-tuned ChatGLM3-6B that classifies output lengths into buckets (out of
 * scope); these stand-ins turn a true output length into the predicted one the scheduler
 * consumes. */
enum {
    UELLM_PREDICT_ORACLE = 0,       /* pred = true length                                          */
    UELLM_PREDICT_BUCKETED = 1,     /* pred = max(1, ceil(true / w)) * w                   */
    UELLM_PREDICT_NOISY = 2,        /* bucketed, moved one bucket up or down with probability
                                       error_rate (never below the first bucket, R20)       */
    UELLM_PREDICT_CONSTANT = 3      /* pred = constant_tokens                                      */
};
typedef struct {
    uint32_t variant;               /* UELLM_PREDICT_*                                             */
    uint32_t bucket_width;          /* w >= 1 (bucketed, noisy)                                    */
    uint32_t constant_tokens;       /* >= 1 (constant)                                             */
    uint32_t window;                /* monitor epoch in queries (R20); 0 = one epoch of all n      */
    double error_rate;              /* noisy: probability in [0, 1] (0.0049 mimics P:195's 99.51 %) */
    double gamma;                   /* monitor multiplier >= 1 (S:216 default 1.1)                 */
    double cap;                     /* monitor inflation cap >= 1 (S:216 default 2.0)              */
    uint64_t seed;                  /* noisy: counter-based draw splitmix64(seed ^ k * 0x9E3779B97F4A7C15)
                                       for caller index k; u = (z >> 11) * 2^-53, moved iff
                                       u < error_rate, up iff z is odd                             */
    uint32_t monitor;               /* 0|1: apply the misprediction monitor      */
    uint32_t pad;
} uellm_predictor;

/* Misprediction-monitor state, device-resident so that consecutive windows chain on the
 * stream without host round trips. */
typedef struct {
    uint64_t corrections;           /* observed under-predictions                          */
    double inflation_factor;        /* >= 1, multiplies every prediction                   */
    uint64_t scratch[2];            /* library scratch: zero before the first call, left zero      */
} uellm_monitor_state;

/* Predicted output lengths for n queries in windows of pc->window (R20): window w is predicted
 * with the inflation factor in force at its start,
 *     pred_k = min(ceil(base_k * factor), 2^32 - 1),   base_k from the variant above,
 * then its completions are observed (true length = actual): every under-prediction
 * (true_k > pred_k) increments corrections and sets factor <- min(factor * gamma, cap), one
 * observation at a time, before window w + 1 is predicted.
 *   true_out_len   [device] n x u32, true (generated) output length of caller query k.
 *   pc             [host] predictor; UELLM_ERR_CONFIG if a field is out of range.
 *   state          [device] 1 x uellm_monitor_state, read and updated on the stream; its
 *                  inflation_factor must be >= 1.
 *   pred_out_len   [device] n x u32 output (feeds uellm_queries.pred_out_len).
 *   window_factors [device] capacity nwin + 1 x f64 or NULL: factor used by each window, then
 *                  the final factor.
 *   ws, ws_bytes   [device] optional scratch (NULL, 0 = none).  With ws_bytes >=
 *                  uellm_predict_workspace_bytes(n, pc) > 0 the factor levels are evaluated for all
 *                  windows in one pass (4 launches); otherwise one launch per window.  Same results.
 * Never synchronises. */
size_t uellm_predict_workspace_bytes(uint64_t n, const uellm_predictor *pc);
uellm_status uellm_predict_lengths(uint64_t n, const uint32_t *true_out_len, const uellm_predictor *pc,
                                   uellm_monitor_state *state, uint32_t *pred_out_len,
                                   double *window_factors, void *ws, size_t ws_bytes, void *stream);

/* HELR deployer (NEXT f3; Sec. 4.3, Alg. 2, Eq. 4-6; SPEC
 * S:341-400; R21).  Places the model's layers on a chain of devices: the deploy-time
 * step that fixes the KV reserve T the scheduler's cap comes from. */
#define UELLM_HELR_MAX_DEVICES 20
typedef struct {
    uint32_t num_devices;           /* |D|, 1 .. UELLM_HELR_MAX_DEVICES                            */
    uint32_t num_layers;            /* Layer(M) >= 1                                               */
    uint64_t model_bytes;           /* M > 0; m = M / Layer(M) bytes per layer (Alg. 2 line 9)     */
    uint64_t kv_reserve_bytes;      /* T, memory reserved for the KV cache (Alg. 2 line 11)        */
    double p;                       /* >= 0, scales compute time (Eq. 5)                           */
    double a1, a2;                  /* >= 0 objective weights: a1 * latency + a2 * |S| / |D|;
                                       HE = (0, 1), LR = (10, 1)                            */
    const uint64_t *memory_bytes;   /* [host] |D| x Memory(d)                                      */
    const double *performance;      /* [host] |D| x Performance(d) > 0                             */
    const double *link_latency_s;   /* [host] |D| x |D| row-major Latency(E[i][j]), finite >= 0     */
} uellm_topology;

/* The chosen chain: device[t] is the t-th device visited, holding layers
 * [layer_begin[t], layer_begin[t] + layer_count[t]) (greedy fill in visit order). */
typedef struct {
    uint32_t count;                 /* devices on the chain                                        */
    uint32_t feasible;              /* 0: no subset can hold the model (Eq. 4); other fields 0     */
    uint32_t mask;                  /* the chosen subset S as a bit mask over device ids           */
    uint32_t pad;
    uint32_t device[32], layer_begin[32], layer_count[32];
    double objective;               /* a1 * latency_s + a2 * |S| / |D|                             */
    double latency_s;               /* chain latency: compute + link terms (Eq. 5)                 */
} uellm_device_map;

/* Device workspace for uellm_helr_plan with num_devices devices (0 if out of range).  [host] */
size_t uellm_helr_workspace_bytes(uint32_t num_devices);

/* HELR (Alg. 2) with readings R21: max_layers(d) = min(L, floor((Memory(d) - T) * L / M)) (0 when
 * Memory(d) <= T); layers filled greedily along the visit order; one bitmask DP over (visited
 * set, last device) dp[S][j] = min_i (dp[S\{j}][i] + Latency[i][j]) + p*x_j*m/Performance(j)
 * (smallest i on ties); subsets with sum max_layers < L skipped (Eq. 4); the answer minimises
 * (objective, latency, mask, last device) lexicographically.
 *   t    [host] topology + model; UELLM_ERR_CONFIG if out of range.
 *   ws   [device] workspace of ws_bytes >= uellm_helr_workspace_bytes(t->num_devices), 256-B aligned.
 *   out  [host|device] 1 x uellm_device_map (host: the call synchronises `stream`).
 * The host arrays are copied into the workspace on `stream` (pageable copies complete before the
 * call returns). */
uellm_status uellm_helr_plan(const uellm_topology *t, void *ws, size_t ws_bytes, uellm_device_map *out,
                             void *stream);

/* End-to-end scheduling of HOST-resident queries with the PCIe copies overlapped with the GPU
 * work.  Windows are independent (R15), so the job is cut into `groups` groups of whole windows
 * (0 = 12); group g+1's host->device copy and group g-1's device->host copy run on two internal
 * copy streams while group g is loaded, scheduled and summarised on `stream` -- the same
 * results as uellm_profile_load + uellm_schedule_batches + uellm_batch_stats on the whole job
 * (mean_latency_s is re-weighted from the groups' means: within 1e-12 relative).
 *   q                       [host] queries with HOST arrays (pinned for overlap; pageable works
 *                           but serialises the copies).
 *   ws                      [device] >= uellm_pipeline_workspace_bytes(n, cfg, groups), 256-B aligned.
 *   order, batch_offsets    [host] n and n+1 x u32 (pinned for overlap), as uellm_schedule_batches.
 *   num_batches, totals     [host].
 * Its three internal streams and the per-group events are created on the device's first call and
 * reused by every later call (held for the process lifetime; calls on one device serialise on
 * them); no device allocation.  Synchronises `stream` once per group (each group's load reads its
 * validation record) and at the end.  On an error the host outputs are unspecified. */
size_t uellm_pipeline_workspace_bytes(uint64_t n, const uellm_config *cfg, uint32_t groups);
uellm_status uellm_schedule_pipelined(const uellm_queries *q, const uellm_config *cfg, uint32_t groups, void *ws,
                                      size_t ws_bytes, uint32_t *order, uint32_t *batch_offsets,
                                      uint64_t *num_batches, uellm_totals *totals, void *stream);

/* Boundary bitmap of the last uellm_schedule_batches call on p (the a9 exchange format):
 * bit k of words (k = 0 .. n, word k / 32, bit k % 32) is set iff a batch starts at scheduled
 * position k, i.e. iff k is one of batch_offsets[0 .. num_batches] (bit n = the end).
 *   words  [device] capacity (n + 32) / 32 x u32; written stream-ordered, never synchronises. */
uellm_status uellm_boundary_bitmap(const uellm_profile *p, const uellm_config *cfg, uint32_t *words,
                                   void *stream);

/* a9 -- the one exchange step of the multi-GPU path (BASELINE.json north_star "one
 * NCCL allgather of batch boundaries and statistics").  Windows never share a batch (R15), so
 * rank r schedules the contiguous window block [q_r, q_{r+1}) of the job on its own GPU; each
 * rank then contributes ONE fixed-size record to an allgather:
 *     record = [ uellm_totals of the rank (128 B) | boundary bitmap of the rank's n_r + 1
 *                positions (bit k set iff a batch starts at local position k; bit n_r = end) ]
 * padded to uellm_exchange_bytes(n_max) with n_max the largest rank's query count.  From the
 * gathered records every rank rebuilds the whole job's batch_offsets and exact totals.
 * The collective itself is the caller's (torch.distributed / NCCL all_gather_into_tensor). */

/* Bytes of one rank's exchange record for ranks of at most n_max queries (multiple of 16). */
size_t uellm_exchange_bytes(uint64_t n_max);

/* Write this rank's record.  [stream-ordered, never synchronises]
 *   p, cfg     the rank's loaded profile; the schedule of its last uellm_schedule_batches call.
 *   totals     [device] the rank's uellm_totals (uellm_batch_stats output on the same stream).
 *   record     [device] uellm_exchange_bytes(n_max) bytes, 16-B aligned; n_max >= the rank's n. */
uellm_status uellm_exchange_pack(const uellm_profile *p, const uellm_config *cfg, const uellm_totals *totals,
                                 void *record, uint64_t n_max, void *stream);

/* Job totals from `count` partial uellm_totals (window groups, ranks) laid out `stride_bytes` apart
 * in device memory -- e.g. the heads of gathered exchange records (stride uellm_exchange_bytes).
 * Same combination as uellm_exchange_combine's totals.  parts [device]; out [host|device] (host:
 * the call synchronises `stream` and returns UELLM_ERR_OVERFLOW if out->overflow != 0). */
uellm_status uellm_totals_combine(const void *parts, uint32_t count, uint64_t stride_bytes, uellm_totals *out,
                                  void *ws, size_t ws_bytes, void *stream);

/* Workspace of uellm_exchange_combine for a job of n_total queries (device bytes). */
size_t uellm_exchange_workspace_bytes(uint64_t n_total, uint32_t world);

/* Rebuild the whole job from the gathered records (record r = rank r, contiguous).
 *   gathered        [device] world x uellm_exchange_bytes(n_max) bytes.
 *   query_begin     [host] world + 1 entries: rank r owns global positions
 *                   [query_begin[r], query_begin[r+1]); query_begin[world] = n_total < 2^32 - 1.
 *   ws              [device] >= uellm_exchange_workspace_bytes(n_total, world), 256-B aligned.
 *   batch_offsets   [device] capacity n_total + 1 x u32: the job's offsets (rank r's local
 *                   boundary k is global position query_begin[r] + k).
 *   num_batches     [device] 1 x u64.
 *   totals          [host|device] 1 x uellm_totals: sums of the ranks' integer totals (kv_bytes_max:
 *                   max), exact 128-bit latency numerator, doubles re-formed from the sums as
 *                   uellm_batch_stats forms them; overflow flags OR-ed plus any saturation here.
 * Host totals: the call synchronises `stream`.  Identical to a single-GPU run of the whole job
 * (tests/test_gpu_parity.py, tests/test_distributed_gloo.py). */
uellm_status uellm_exchange_combine(const void *gathered, uint32_t world, uint64_t n_max,
                                    const uint64_t *query_begin, void *ws, size_t ws_bytes,
                                    uint32_t *batch_offsets, uint64_t *num_batches, uellm_totals *totals,
                                    void *stream);

/* BGS, the paper's baseline deployer ("Greedy Scheduling Algorithm"):
 * devices in descending order of Memory(d) (ties: smaller id first) each take max_layers(d)
 * (as in uellm_helr_plan) until the layers are exhausted; that prefix is the chain.  latency_s and
 * objective use uellm_helr_plan's chain formula, so the two are directly comparable (HELR's
 * objective is never larger: BGS's chain is one of the chains it searches).  Same arguments and
 * workspace as uellm_helr_plan; feasible = 0 if all devices together cannot hold the model. */
uellm_status uellm_bgs_plan(const uellm_topology *t, void *ws, size_t ws_bytes, uellm_device_map *out,
                            void *stream);

/* Attach (n <= UELLM_STAGE_COUNT) caller-owned cudaEvent_t handles (void*, created with timing
 * enabled; NULL entries are skipped) to the profile; subsequent schedule/stats calls record
 * event k at stage boundary k on their stream.  n = 0 detaches.  [host] */
uellm_status uellm_set_stage_events(uellm_profile *p, void *const *events, uint32_t n);

/* Diagnostics of the last schedule call on p.  [host] out; synchronises `stream`. */
uellm_status uellm_get_diagnostics(const uellm_profile *p, uellm_diagnostics *out, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* UELLM_H_ */
