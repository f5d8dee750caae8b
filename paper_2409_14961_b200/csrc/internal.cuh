// internal.cuh -- shared declarations of the libuellm CUDA path (sm_100a).
// Product code only: nothing here is shared with oracle/ (the CPU oracle has its own types).
#pragma once
#include <cstddef>
#include <cstdint>
#include <initializer_list>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>        // header-only NVTX v3 (CUDA toolkit): host ranges for nsys / ncu

#include "../../include/uellm.h"

namespace uellm {

// NVTX range over a scope: every ABI entry point and the stages of uellm_schedule_batches show up
// by name on an nsys timeline (ncu --nvtx filters by them too).
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};

constexpr uint32_t kMaxBatchLimit = 4096;      // W limit of this build (UELLM_ERR_UNSUPPORTED)
// radix-sort CTA shape (tools/variant_run.sh on c4, sort ms: 2048 x 256: 2.51, 4096 x 512: 2.54,
// 2048 x 512: 2.64, 4096 x 256: 2.70, 8192 x 1024: 2.87, 1024 x 256: 3.10)
#ifndef UELLM_SORT_TILE
#define UELLM_SORT_TILE 2048
#endif
#ifndef UELLM_SORT_THREADS
#define UELLM_SORT_THREADS 256
#endif
constexpr uint32_t kSortTile = UELLM_SORT_TILE;         // keys per radix-sort CTA (256 threads x 8)
constexpr uint32_t kSortThreads = UELLM_SORT_THREADS;
constexpr uint32_t kSortItems = kSortTile / kSortThreads;
#ifndef UELLM_DP_WARPS
#define UELLM_DP_WARPS 8
#endif
constexpr uint32_t kDpWarpsPerCta = UELLM_DP_WARPS;
constexpr uint32_t kScanBlock = 1024;          // elements per CTA in the scan kernels
constexpr uint64_t kProfileMagic = 0x55454c4c4d763031ull;  // "UELLMv01"
constexpr uint32_t kSloSetSize = 4096;         // global hash set of distinct slo_us values
constexpr uint32_t kSloSetBits = 12;
constexpr uint32_t kSloRankMax = 1024;         // rank-compress the sort key up to this many values

static inline __host__ __device__ uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }
static inline __host__ __device__ uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

// a1 (R12): slo_us = rint(double(slo_s) * 1e6), round-half-to-even, valid iff in [1, 2^32-1].
// Used by the load (validation) and by the key packers -- one definition, bit-identical.
__device__ __forceinline__ uint32_t slo_to_us(float slo_s, bool &ok)
{
    const double x = (double)slo_s;
    if (!(x > 0.0) || !isfinite(x)) { ok = false; return 0; }
    const double r = rint(__dmul_rn(x, 1e6));      // one correctly rounded product
    if (r < 1.0 || r > 4294967295.0) { ok = false; return 0; }
    ok = true;
    return (uint32_t)r;
}
__device__ __forceinline__ uint32_t slo_hash(uint32_t v, uint32_t bits) { return (v * 0x9E3779B1u) >> (32 - bits); }

// --------------------------------------------------------------------------------------
// Device-side validation record written by the load kernel (read back once, 64 bytes).
struct LoadMeta {
    uint32_t bad;            // bit 0 input_len == 0, bit 1 out == 0, bit 2 SLO invalid
    uint32_t max_in, max_out, max_slo;
    unsigned long long key_or, key_and;
    uint32_t slo_distinct, slo_overflow;
    uint32_t status;         // uellm_profile_reload's verdict (device status word)
    uint32_t slo_missing;    // fused reload: an SLO value outside the profile's distinct set
    uint32_t pad[4];
};
static_assert(sizeof(LoadMeta) == 64, "LoadMeta is 64 bytes");
// reload: compare the fresh LoadMeta with the decisions recorded in the profile
struct ReloadRef {
    uint32_t max_in, max_out, slo_distinct, slo_overflow;
    unsigned long long key_or, key_and;
    uint32_t fused;          // k_reload_pack32 ran: the set test is "every SLO value in the profile's set"
};
cudaError_t launch_reload_check(LoadMeta *meta, ReloadRef ref, cudaStream_t st);

// Per-tile state of the SEG-DP and the traceback (one record per tile).
struct TileRec {
    uint32_t s, e;           // the tile decides boundaries (s, e]
    uint32_t conv;           // fix-up converged (tile 0 of a window: 1)
    uint32_t conv_pos;       // boundary at which the fix-up converged
    uint32_t fix_end;        // last boundary whose arg the fix-up wrote
    uint32_t valid;          // tile exists
    int64_t delta;           // C_fix - C_local on the converged region
    int64_t off_local;       // true C = Cx + off_local for boundaries > conv_pos   (cascade)
    int64_t off_fix;         // true C = CFx + off_fix for boundaries <= fix_end       (cascade)
    uint32_t exitA, exitB;   // traceback: exit of the walk from e / from the true entry
    uint32_t merged;
    uint32_t uni;            // local run: every record of the tile is the same (periodic fill)
    uint32_t fill_s, fill_P; // cascade: fix frame deferred to k_dp_fill, periodic with period fill_P
    int64_t fill_F;          //   from the reference boundaries (fill_s - fill_P, fill_s]: C += fill_F per period
    uint32_t remark;         // traceback: 1 + the true entry when the tile must be re-marked, else 0
    uint32_t refixed;        // k_dp_refix re-ran the fix-up from the predecessor's fix frame into the
    uint32_t rf_conv, rf_conv_pos, rf_fix_end;   //   side arrays; its results (the cascade may adopt them)
    int64_t rf_delta;
};

struct Diag {                // device counters, see uellm_diagnostics
    unsigned long long tiles, tile_len, fixups_unconverged, cascade_reruns, fixup_positions,
        trace_unmerged, trace_rewalks, sort_passes, dp_evals, sched_launches, stats_launches, sort_key_bits,
        dp_filled;
};

// Whole-job totals from partial totals (window groups of the pipelined call, ranks of the a9
// exchange): integer sums (kv_bytes_max: max) saturating at 2^64 - 1 with the overflow bit of the
// field (uellm_totals.overflow), exact 128-bit latency numerator; finish_totals re-forms the two
// doubles exactly as k_totals forms them.
__host__ __device__ inline void sat_add_u64(uint64_t &a, uint64_t b, uint64_t &of, int bit)
{
    const uint64_t s = a + b;
    if (s < a) { a = ~0ull; of |= 1ull << bit; } else a = s;
}
__host__ __device__ inline void combine_totals_into(uellm_totals &T, const uellm_totals &t)
{
    uint64_t *dst = &T.n;
    const uint64_t *src = &t.n;
    for (int f = 0; f < 11; ++f) {            // n .. makespan_us (struct order)
        if (f == 5) dst[f] = src[f] > dst[f] ? src[f] : dst[f];
        else sat_add_u64(dst[f], src[f], T.overflow, f);
    }
    const uint64_t lo = T.latency_sum_lo + t.latency_sum_lo;
    T.latency_sum_hi += t.latency_sum_hi + (lo < T.latency_sum_lo ? 1ull : 0ull);
    T.latency_sum_lo = lo;
    T.overflow |= t.overflow;
}
__host__ __device__ inline void finish_totals(uellm_totals &T)
{
    const double lat = (double)T.latency_sum_hi * 18446744073709551616.0 + (double)T.latency_sum_lo;
    T.mean_latency_s = T.n ? lat / (double)T.n * 1e-6 : 0.0;
    T.throughput_tok_s = T.makespan_us ? (double)T.gen_tokens / ((double)T.makespan_us * 1e-6) : 0.0;
}

// Exact 128-bit accumulator of sum(b * completion_us) for mean_latency_s.
struct StatAcc {
    unsigned long long gen, pad_in, pad_out, kv_max, dp_cost, viol_alone, viol_seq, over_cap,
        makespan, lat_lo, lat_hi, batches, overflow;
};

// Accumulators of uellm_simulate (exact 128-bit latency sum).
struct SimAcc {
    unsigned long long busy, gen, viol, lat_max, lat_lo, lat_hi, makespan, pad;
};

// --------------------------------------------------------------------------------------
// Workspace layout (byte offsets from the workspace base, 256-B aligned).
struct WsLayout {
    uint64_t n, nwin, window, W, tile_len, tpw, ntiles, sort_tpw, sort_tiles, nwords;
    uint64_t stage_in, stage_out, stage_slo;      // host-input staging
    uint64_t keys0, keys1, keys2;                 // packed keys (kept) + sort ping-pong;
    uint64_t vals0, vals1, vals2;                 // keys1/keys2 re-used as Cx/CFx, est/completion
    uint64_t rin, rout, rslo;                     // scheduled-order records
    uint64_t keysc;                               // rank-compressed u32 keys
    uint64_t slo_set, slo_ctab, slo_table;        // distinct-SLO hash set, compact (value, rank) hash, sorted values
    uint64_t order, offsets;                      // internal copies of the schedule
    uint64_t argx;                                // u16 per position
    uint64_t tiles;                               // TileRec[ntiles]
    uint64_t tmaps, twflag;                       // traceback exit maps (u16[ntiles][W]), window flags
    uint64_t tflags;                              // u32[ntiles + 2]: local-done flags + 2 work counters
    uint64_t bitmap, wscan, blocksum, blockagg;   // boundary bitmap + scan scratch
    uint64_t st_so, st_pin, st_pout;              // per-batch stats scratch (u64 each)
    uint64_t a1tiles;                             // Alg. 1 chain-walk tile exits (uint2)
    uint64_t hist;                                // u32[2][sort_tiles * 256] (passes alternate)
    uint64_t hist0;                               // u32[sort_tiles * 256]: first pass's counts (kept)
    uint64_t meta, diag, acc, nb, totals, wincost;
    uint64_t simacc, simtot;                      // uellm_simulate accumulators / host-totals staging
    uint64_t total;
};

// Host-side POD view stored inside uellm_profile (<= 320 bytes).
struct ProfileView {
    uint64_t magic;
    uint64_t n, window, nwin;
    uint8_t *ws;
    uint64_t ws_bytes;
    const uint32_t *d_in, *d_out;                 // caller device arrays or staging copies
    uint32_t max_in, max_out, max_slo, W;
    unsigned long long key_or, key_and;
    uint64_t cfg_hash;
    uint64_t diag_off, wincost_off;               // workspace offsets read by get_diagnostics
    uint64_t n_events;
    void *events[UELLM_STAGE_COUNT];              // caller cudaEvent_t handles (stage timing)
    uint32_t slo_distinct, slo_overflow;
    const float *d_slo;                           // caller device SLO array or its staging copy
    uint64_t meta_off;                            // workspace offset of the LoadMeta (status word)
    uint32_t keys_ready;                          // keysc + hist0 hold the current queries' keys (fused reload)
    uint32_t key_plan;                            // compressed-key eligibility: 1 | cbits << 8 | ob << 16 | rb << 24
    uint64_t pad[7];
};
static_assert(sizeof(ProfileView) <= sizeof(uellm_profile), "ProfileView fits uellm_profile");

WsLayout make_layout(uint64_t n, const uellm_config &cfg);

// Stream-ordered stores of small host values into device memory without a pageable copy (a
// pageable cudaMemcpyAsync synchronises the stream first).  zero_diag: the first pair's pointer is
// a Diag to clear before the stores.
struct U64Store {
    unsigned long long *dst;
    unsigned long long val;
};
cudaError_t launch_set_u64s(cudaStream_t st, std::initializer_list<U64Store> stores, bool zero_diag = false);
uint64_t choose_tile_len(uint64_t n, uint64_t window, uint32_t W, uint32_t dp_tile);
// the SEG-DP tile length of a throughput-bound job of n queries (the 16 W floor, no one-wave rule)
uint32_t tile_len_throughput(uint64_t n, uint32_t W);

// --------------------------------------------------------------------------------------
// Kernel launchers (each returns cudaGetLastError()).
cudaError_t launch_load(const uint32_t *in, const uint32_t *out, const float *slo, uint64_t n,
                        LoadMeta *meta, uint32_t *slo_set, cudaStream_t st);
// key64 = slo_us << 32 | out, val = arrival index (generic sort key; FIFO records)
cudaError_t launch_pack64(const uint32_t *out, const float *slo, uint64_t n, unsigned long long *keys,
                          uint32_t *vals, cudaStream_t st);
// decode arguments for the last radix pass (records written straight at the sorted position)
struct DecodeArgs {
    const uint32_t *in;        // caller input lengths (gathered by arrival index)
    const uint32_t *table;     // compressed keys: rank -> slo_us (kSloRankMax entries)
    int ob;                    // compressed keys: bits of max_out
    uint32_t nslo;             // compressed keys: ranks in use (table entries the decode stages)
    uint32_t packin;           // payload = (idx - window start) | (in - 1) << wb (no gather in the decode)
    int wb;
    uint32_t *rin, *rout, *rslo, *order;
};
// compressed path: rank table + compact (value, rank) hash of 2^cbits slots (ctab), then pack
// key32 = rank << ob | out with the digit-0 histogram
cudaError_t launch_slo_table(const uint32_t *slo_set, uint32_t *table, unsigned long long *ctab, int cbits,
                             cudaStream_t st);
// [w_first, w_first + nwin): the windows processed by this call (window groups keep a group's
// intermediate arrays resident in L2 across the passes)
cudaError_t launch_pack32_hist(const uint32_t *out, const float *slo, uint64_t n, uint64_t window, uint64_t w_first,
                               uint64_t nwin, const unsigned long long *ctab, int cbits, int ob, uint32_t *keys32,
                               uint32_t *vals, uint32_t *hist0, cudaStream_t st);
// uellm_profile_reload of a rank-compressed profile: validation (bad bits, maxima into meta) + key
// pack + digit-0 histogram in one pass over the caller arrays; an SLO value outside the profile's
// (value, rank) hash sets meta->slo_missing
cudaError_t launch_reload_pack32(const uint32_t *in, const uint32_t *out, const float *slo, uint64_t n,
                                 uint64_t window, const unsigned long long *ctab, int cbits, int ob, uint32_t *keys32,
                                 uint32_t *hist0, LoadMeta *meta, cudaStream_t st);
cudaError_t radix_sort_windows32(const uint32_t **keys_io, const uint32_t **vals_io, uint32_t *keys_a,
                                 uint32_t *vals_a, uint32_t *keys_b, uint32_t *vals_b, uint32_t *hist, uint32_t *hist2,
                                 uint64_t n,
                                 uint64_t window, uint64_t w_first, uint64_t nwin, uint32_t digit_mask, int *passes,
                                 cudaStream_t st, const uint32_t *hist0 = nullptr, const DecodeArgs *dec = nullptr,
                                 int *kernels = nullptr);
// windows per sort group: about kSortGroupQueries queries (env UELLM_SORT_GROUP_Q overrides, tuning)
uint64_t sort_group_windows(uint64_t window, uint64_t nwin);
cudaError_t launch_decode32(const uint32_t *keys, const uint32_t *vals, const uint32_t *in, uint64_t n,
                            const uint32_t *table, int ob, uint32_t *rin, uint32_t *rout, uint32_t *rslo,
                            uint32_t *order, cudaStream_t st);

// Segmented (per-window) stable LSD radix sort of (key, val) over the digits of
// `digit_mask` (bit d set = digit d of 8 bits varies).  *keys_io / *vals_io is the (read-only)
// input; passes alternate between buffers A and B and on return *keys_io / *vals_io point at
// the sorted result (the input itself when no digit varies).  *passes = passes run.
cudaError_t radix_sort_windows(const unsigned long long **keys_io, const uint32_t **vals_io,
                               unsigned long long *keys_a, uint32_t *vals_a,
                               unsigned long long *keys_b, uint32_t *vals_b, uint32_t *hist, uint32_t *hist2,
                               uint64_t n, uint64_t window, uint64_t w_first, uint64_t nwin, uint32_t digit_mask,
                               int *passes, cudaStream_t st, const struct DecodeArgs *dec = nullptr,
                               int *kernels = nullptr);

// Decode sorted keys into records: slo = key >> 32, out = key & 0xffffffff, idx = val.
cudaError_t launch_decode(const unsigned long long *keys, const uint32_t *vals, const uint32_t *in,
                          uint64_t n, uint32_t *rin, uint32_t *rout, uint32_t *rslo,
                          uint32_t *order, cudaStream_t st);

struct DPParams {
    const uint32_t *rin, *rout, *rslo;
    long long *Cx, *CFx;
    uint16_t *argx;
    long long *Crf;                              // k_dp_refix outputs (scratch free during the schedule)
    uint16_t *Arf;
    TileRec *tiles;
    uint32_t *tflags;                            // [ntiles] local-done flags, then the local / fix-up work counters
    Diag *diag;
    unsigned long long *wincost;
    uint32_t n, window, nwin, tile_len, tpw, W, cap_slots, split;
    uint32_t narrow;                             // 32-bit fast path valid (see k_segdp.cu)
    uint32_t many_runs;                          // more distinct SLO values than the compressed sort key holds
    unsigned long long cap_tok;                  // ~0ull = no cap
    unsigned long long t_batch, t_iter, t_tok, t_pre, lambda;
};
// ev[0..2]: events recorded after the local, fix-up and cascade kernels (NULL = none).
cudaError_t run_segdp(const DPParams &P, uint64_t ntiles, cudaStream_t st, void *const ev[3], int *launches);

// Traceback of SEG-DP args into the boundary bitmap (maps: u16[ntiles][W] scratch, wflag: u32[nwin]).
cudaError_t run_traceback(const DPParams &P, uint32_t *bitmap, uint64_t ntiles, uint16_t *maps, uint32_t *wflag,
                          cudaStream_t st, int *launches);

// Bitmaps of the other modes.
cudaError_t launch_mark_fifo(uint32_t *bitmap, uint64_t n, uint64_t window, uint32_t W, int sort_only,
                             cudaStream_t st);
struct Alg1Params {
    const uint32_t *rin, *rout, *rslo;
    uint32_t n, window, nwin, W, split;
    unsigned long long cap_tok;
    double w1, w2, l1, l2, threshold, eps;
    uint32_t eq2_additive;
};
cudaError_t launch_alg1(const Alg1Params &A, uint32_t *bitmap, uint16_t *next_delta, uint2 *tile_exits, Diag *diag,
                        cudaStream_t st);
uint64_t alg1_scratch_bytes(uint64_t window, uint64_t nwin, uint32_t W);

// Compaction of the boundary bitmap (n+1 bits) into batch_offsets, num_batches.
cudaError_t run_compact(const uint32_t *bitmap, uint64_t n, uint32_t *wscan, uint32_t *blocksum,
                        uint32_t *offsets, unsigned long long *num_batches, cudaStream_t st);

// a9: job bitmap + offsets + totals from the gathered exchange records (k_exchange.cu)
cudaError_t run_exchange_combine(const uint8_t *gathered, uint32_t world, uint64_t rec_bytes,
                                 const unsigned long long *d_qb, uint64_t n_total, uint32_t *bitmap, uint32_t *wscan,
                                 uint32_t *blocksum, uint32_t *offsets, unsigned long long *num_batches,
                                 uellm_totals *d_tot, cudaStream_t st);
cudaError_t launch_totals_combine(const uint8_t *parts, uint32_t count, uint64_t stride, uellm_totals *out,
                                  cudaStream_t st);
// bytes of one exchange record for ranks of <= n_max queries: totals + (n_max + 1)-bit bitmap
// + one spare word (the combine reads a word pair), 16-B multiple
inline uint64_t exchange_record_bytes(uint64_t n_max)
{
    return align_up(sizeof(uellm_totals) + 4 * ((n_max + 1 + 31) / 32 + 1), 16);
}

struct StatsParams {
    const uint32_t *rin, *rout, *rslo;
    const uint32_t *offsets;
    const unsigned long long *num_batches;
    uint64_t n_cap;                             // capacity bound of batches (n)
    uint32_t window, nwin;
    unsigned long long *est, *compl_;
    unsigned long long *so, *pin, *pout;        // per batch: s | O << 32, input / output padding
    uint32_t sorted;                            // members of a batch ascend in slo_us (all modes but FIFO)
    uint32_t *blocksum_u32;                     // scratch
    unsigned long long *blockagg;               // scratch
    uellm_batch_stat *per_batch;
    StatAcc *acc;
    uellm_totals *totals;
    uint64_t n;
    unsigned long long kv_unit;                 // kv_bytes_per_elem * l * h
    unsigned long long kv_cap;                  // 0 = none
    unsigned long long t_batch, t_iter, t_tok, t_pre, lambda;
};
cudaError_t run_stats(const StatsParams &S, cudaStream_t st);

struct SimParams {
    const uint32_t *rin, *rout, *rslo;          // scheduled-order records
    const uint32_t *order, *offsets;
    const unsigned long long *num_batches;
    const unsigned long long *arrival;          // caller index -> arrival time (us)
    unsigned long long *arr_s;                  // arrival in scheduled order (scratch)
    unsigned long long *est, *inc_a, *inc_b;    // per batch: est, CTA-local inclusive map
    unsigned long long *chunk_a, *chunk_b, *carry;   // per chunk of kScanBlock batches
    unsigned long long *batch_end, *latency;    // optional outputs (NULL = not requested)
    SimAcc *acc;
    uellm_sim_totals *totals;
    uint64_t n, n_cap;
    unsigned long long t_batch, t_iter, t_tok, t_pre;
};
cudaError_t run_simulate(const SimParams &S, cudaStream_t st, int *launches);

constexpr uint32_t kPredMaxLevels = 32;         // factor levels of the level path (chain v_0 .. v_K)
constexpr uint64_t kPredMaxWindows = 1ull << 20; // windows of the level path (histogram rows)
struct PredictParams {
    double *levels;                             // level path: [kPredMaxLevels] chain, NULL = window path
    uint32_t *nlevels;                          // K (last level index)
    unsigned long long *hist;                   // [nwin][kPredMaxLevels] under-predictions per level
    uint8_t *wlevel;                            // [nwin] level of each window
    const uint32_t *true_len;
    uint32_t *pred;
    uellm_monitor_state *state;
    double *factors;                            // per-window factors (nwin + 1) or NULL
    uint64_t nwin;
    uint32_t variant, bucket_width, constant_tokens, monitor;
    double error_rate, gamma, cap;
    unsigned long long err_thresh;              // ceil(error_rate * 2^53): u < e  <=>  (z >> 11) < err_thresh
    unsigned long long seed;
};
cudaError_t run_predict(const PredictParams &P, uint64_t n, uint64_t window, cudaStream_t st, int *launches);

constexpr uint32_t kHelrMaxDevices = 20;        // dp table 2^20 x 20 doubles = 168 MB
constexpr uint32_t kHelrParts = 296;            // CTAs of the feasible-minimum reduction
struct HelrParams {
    uint32_t D;
    unsigned long long L;
    double p, a1, a2, m;                        // m = M / L
    const uint32_t *cap;                        // [D] max_layers
    const unsigned long long *mem;              // [D] Memory(d) (BGS order)
    const double *perf;                         // [D]
    const double *lat;                          // [D*D]
    const unsigned long long *binom;            // [(kHelrMaxDevices+1)^2] C(n, k), device copy
    const unsigned long long *binom_host;       // same table on the host (launch sizing)
    unsigned long long *capsum;                 // [2^D]
    double *dp;                                 // [2^D * D]
    uint8_t *arg;                               // [2^D * D]
    double *part_obj, *part_lat;                // [kHelrParts]
    unsigned long long *part_sj;                // [kHelrParts] S << 32 | j
    uellm_device_map *out;
};
cudaError_t run_helr(const HelrParams &H, cudaStream_t st, int *launches);
cudaError_t run_bgs(const HelrParams &H, cudaStream_t st);

}  // namespace uellm
