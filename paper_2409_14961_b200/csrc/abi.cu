// abi.cu -- the C ABI of include/uellm.h: argument/config validation, workspace carving and
// stream-ordered orchestration of the kernels (host code only; no allocation, no globals).
#include <cstdlib>
#include <cmath>
#include <cstring>

#include "internal.cuh"

#ifndef UELLM_DP_PRUNE_EVERY
#define UELLM_DP_PRUNE_EVERY 1
#endif

using namespace uellm;

namespace uellm {

uint64_t sort_group_windows(uint64_t window, uint64_t nwin)
{
    // measured on c4 (tools/sweep_sort.sh): groups of 8 M / 4 M / 1 M queries cost 3.2 / 3.9 /
    // 7.6 ms against 2.5 ms for one group (launch tails outweigh the L2 reuse), so the default
    // is a single group of every window
    uint64_t q = ~0ull;
    if (const char *e = getenv("UELLM_SORT_GROUP_Q")) q = strtoull(e, nullptr, 10);
    uint64_t g = window ? q / window : 1;
    if (g < 1) g = 1;
    return g < nwin ? g : (nwin ? nwin : 1);
}

uint64_t choose_tile_len(uint64_t n, uint64_t window, uint32_t W, uint32_t dp_tile)
{
    uint64_t T;
    if (dp_tile) {
        T = align_up(dp_tile, W);
    } else {
        // ~4.6 tiles per resident DP warp (32 per SM): short tiles balance the data-dependent
        // per-tile work against the fix-ups (tools/sweep_tile.sh on c4, DP ms by tile length:
        // 3584: 7.10, 4608: 7.05, 5120: 7.36, 7168: 7.38, 8192: 7.79; fix-ups re-evaluate 7.4 %
        // of the positions at 4608).
        // The 16 W floor stays for small jobs too: one-wave tiles of 4 W .. 16 W were measured
        // slower on 6-7 M-query window groups (3.5-7 ms against 2.7 ms per group: more fix-ups
        // and cascade re-runs than the extra parallelism gains).
        // A job with fewer 16 W tiles than one wave of resident DP warps (148 SMs x 24) is bound by
        // its tiles' sequential walks, not by the total work: 8 W tiles there (measured: c3 1e6
        // queries 0.95 -> 0.69 ms, c5 1e7 3.42 -> 3.00 ms; 4 W: c5 3.90 ms, the fix-ups and cascade
        // grow faster than the walks shrink)  Throughput-bound callers (the pipelined host call,
        // whose window groups share the GPU) pass dp_tile = tile_len_throughput() instead.
        const uint64_t target_tiles = 148ull * 148;
        T = ceil_div(n ? n : 1, target_tiles);
        const uint64_t floor16 = 16ull * W;
        T = T < floor16 ? floor16 : T;
        // (at least one 16 W tile per SM: a job of a handful of tiles -- c2: 10 -- is bound by its
        // per-window cascade and launches instead, 0.75 vs 1.09 ms with 8 W tiles; and at most 1.5
        // waves of 8 W tiles: a 12.5 M-query c4-shaped job -- one rank of an 8-GPU run, 1.7 waves --
        // took 2.45 ms with 8 W tiles against 2.13 ms with 16 W, its fix-ups and cascade re-runs
        // outgrowing the shorter walks)
        const uint64_t t16 = ceil_div(n ? n : 1, floor16), t8 = ceil_div(n ? n : 1, 8ull * W);
        if (T == floor16 && t16 >= 148 && 2 * t8 <= 3ull * 148 * 24) T = 8ull * W;
        T = align_up(T, W);
    }
    if (T < 2ull * W) T = 2ull * W;
    if (T > window) T = align_up(window, W);   // one tile per window
    return T;
}

uint32_t tile_len_throughput(uint64_t n, uint32_t W)
{
    uint64_t T = ceil_div(n ? n : 1, 148ull * 148);
    if (T < 16ull * W) T = 16ull * W;
    return (uint32_t)align_up(T, W);
}

WsLayout make_layout(uint64_t n, const uellm_config &cfg)
{
    WsLayout L;
    std::memset(&L, 0, sizeof L);
    L.n = n;
    L.window = cfg.window ? (cfg.window < n ? cfg.window : n) : n;
    if (L.window == 0) L.window = 1;
    L.nwin = n ? ceil_div(n, L.window) : 0;
    L.W = cfg.max_batch ? cfg.max_batch : 1;
    L.tile_len = choose_tile_len(n, L.window, (uint32_t)L.W, cfg.dp_tile);
    L.tpw = ceil_div(L.window, L.tile_len);
    L.ntiles = L.tpw * L.nwin;
    L.sort_tpw = ceil_div(L.window, kSortTile);
    L.sort_tiles = L.sort_tpw * L.nwin;
    L.nwords = (n + 1 + 31) / 32;
    uint64_t off = 0;
    auto take = [&](uint64_t bytes) { uint64_t o = off; off = align_up(off + (bytes ? bytes : 1), 256); return o; };
    const uint64_t N = n ? n : 1;
    L.stage_in = take(4 * N); L.stage_out = take(4 * N); L.stage_slo = take(4 * N);
    L.keys0 = take(8 * N); L.keys1 = take(8 * N); L.keys2 = take(8 * N);
    L.vals0 = take(4 * N); L.vals1 = take(4 * N); L.vals2 = take(4 * N);
    L.rin = take(4 * N); L.rout = take(4 * N); L.rslo = take(4 * N);
    L.keysc = take(4 * N);
    L.slo_set = take(4 * kSloSetSize); L.slo_ctab = take(8 * kSloSetSize); L.slo_table = take(4 * kSloRankMax);
    L.order = take(4 * N); L.offsets = take(4 * (N + 1));
    L.argx = take(2 * N);
    L.tiles = take(sizeof(TileRec) * (L.ntiles ? L.ntiles : 1));
    L.tmaps = take(2 * L.W * (L.ntiles ? L.ntiles : 1));
    L.twflag = take(4 * (L.nwin ? L.nwin : 1));
    L.tflags = take(4 * (L.ntiles + 2));
    L.bitmap = take(4 * L.nwords); L.wscan = take(4 * L.nwords);
    const uint64_t nblk = ceil_div(L.nwords, kScanBlock) + ceil_div(N, kScanBlock) + 2;
    L.blocksum = take(4 * nblk);
    L.blockagg = take(8 * nblk);
    L.st_so = take(8 * N); L.st_pin = take(8 * N); L.st_pout = take(8 * N);
    L.a1tiles = take(alg1_scratch_bytes(L.window, L.nwin, (uint32_t)L.W));
    L.hist = take(2 * 4ull * 256 * (L.sort_tiles ? L.sort_tiles : 1));   // two histogram buffers (passes alternate)
    L.hist0 = take(4ull * 256 * (L.sort_tiles ? L.sort_tiles : 1));       // first pass's counts, kept
    L.meta = take(sizeof(LoadMeta)); L.diag = take(sizeof(Diag)); L.acc = take(sizeof(StatAcc));
    L.nb = take(8); L.totals = take(sizeof(uellm_totals));
    L.wincost = take(8 * (L.nwin ? L.nwin : 1));
    L.simacc = take(sizeof(SimAcc)); L.simtot = take(sizeof(uellm_sim_totals));
    L.total = off;
    return L;
}

struct HelrLayout {
    uint64_t cap, mem, perf, lat, binom, part_obj, part_lat, part_sj, out, capsum, dp, arg, total;
};

HelrLayout helr_layout(uint32_t D)
{
    HelrLayout H;
    uint64_t off = 0;
    auto take = [&](uint64_t bytes) { uint64_t o = off; off = align_up(off + (bytes ? bytes : 1), 256); return o; };
    const uint64_t NS = 1ull << D;
    H.cap = take(4 * kHelrMaxDevices);
    H.mem = take(8 * kHelrMaxDevices);
    H.perf = take(8 * kHelrMaxDevices);
    H.lat = take(8 * kHelrMaxDevices * kHelrMaxDevices);
    H.binom = take(8 * (kHelrMaxDevices + 1) * (kHelrMaxDevices + 1));
    H.part_obj = take(8 * kHelrParts); H.part_lat = take(8 * kHelrParts); H.part_sj = take(8 * kHelrParts);
    H.out = take(sizeof(uellm_device_map));
    H.capsum = take(8 * NS);
    H.dp = take(8 * NS * D);
    H.arg = take(NS * D);
    H.total = off;
    return H;
}

}  // namespace uellm

namespace {

template <class T>
T *at(uint8_t *ws, uint64_t off) { return reinterpret_cast<T *>(ws + off); }

bool is_device_ptr(const void *p)
{
    if (!p) return false;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) { cudaGetLastError(); return false; }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

uellm_status check_config(const uellm_config *c)
{
    if (c->mode > UELLM_MODE_SORT_ONLY) return UELLM_ERR_CONFIG;
    if (c->max_batch < 1) return UELLM_ERR_CONFIG;
    if (c->split_on_slo_change > 1 || c->eq2_additive > 1 || (c->flags & ~1u) != 0) return UELLM_ERR_CONFIG;
    if (c->mode == UELLM_MODE_SLO_ODBS) {
        if (!(c->w1 >= 0.0) || !(c->w2 >= 0.0) || !(c->w1 + c->w2 > 0.0)) return UELLM_ERR_CONFIG;
        if (!(c->threshold > 0.0) || !(c->eps > 0.0) || !(c->l1 >= 0.0) || !(c->l2 >= 0.0)) return UELLM_ERR_CONFIG;
    }
    if (c->kv_cap_bytes != 0 && (c->kv_bytes_per_elem == 0 || c->n_layers == 0 || c->hidden == 0))
        return UELLM_ERR_CONFIG;
    if (c->max_batch > kMaxBatchLimit) return UELLM_ERR_UNSUPPORTED;
    return UELLM_OK;
}

inline const ProfileView *view_of(const uellm_profile *p) { return reinterpret_cast<const ProfileView *>(p); }

// FNV-1a over every field of the config: a profile is bound to the exact cfg it was loaded with
// (the overflow bounds, the narrow DP path and the stats' sortedness are decided from it).
uint64_t layout_key(const uellm_config *c)
{
    uint64_t h = 0xcbf29ce484222325ull;
    auto mix = [&](uint64_t v) {
        for (int b = 0; b < 8; ++b) { h ^= (v >> (8 * b)) & 0xff; h *= 0x100000001b3ull; }
    };
    auto dbl = [](double d) { uint64_t u; std::memcpy(&u, &d, 8); return u; };
    mix(c->mode); mix(c->window); mix(c->max_batch); mix(c->split_on_slo_change);
    mix(c->kv_bytes_per_elem); mix(c->n_layers); mix(c->hidden); mix(c->dp_tile); mix(c->kv_cap_bytes);
    mix(c->t_batch_us); mix(c->t_iter_us); mix(c->t_tok_us); mix(c->t_prefill_us); mix(c->lambda_us);
    mix(dbl(c->w1)); mix(dbl(c->w2)); mix(dbl(c->l1)); mix(dbl(c->l2)); mix(dbl(c->threshold)); mix(dbl(c->eps));
    mix(c->eq2_additive); mix(c->flags);
    return h;
}

// Rank-compressed sort key plan of a loaded profile (independent of the mode): eligible when at most
// kSloRankMax distinct SLO values were collected and rank << bits(max_out) | out fits 32 bits.
struct KeyPlan {
    bool ok;
    int ob, rb, cbits;
};
KeyPlan key_plan(const ProfileView &v)
{
    KeyPlan k;
    k.ob = 0;
    while (k.ob < 32 && (v.max_out >> k.ob)) ++k.ob;                           // bits(max_out)
    k.rb = 0;
    while (v.slo_distinct > 1 && k.rb < 32 && ((v.slo_distinct - 1) >> k.rb)) ++k.rb;   // bits(distinct - 1)
    // compact hash: >= 8 slots per value (>= 4 at the 1024-value maximum: 4096 slots), so a lookup
    // almost never probes twice
    k.cbits = 6;
    while ((1u << k.cbits) < 8 * v.slo_distinct && k.cbits < (int)kSloSetBits) ++k.cbits;
    k.ok = !v.slo_overflow && v.slo_distinct >= 1 && v.slo_distinct <= kSloRankMax && k.rb + k.ob <= 32;
    return k;
}

inline void rec(const ProfileView &v, int k, cudaStream_t st)
{
    if ((uint64_t)k < v.n_events && v.events[k]) cudaEventRecord((cudaEvent_t)v.events[k], st);
}

#define CU(x)                                   \
    do {                                        \
        if ((x) != cudaSuccess) {               \
            cudaGetLastError();                 \
            return UELLM_ERR_CUDA;              \
        }                                       \
    } while (0)

}  // namespace

extern "C" {

uint32_t uellm_abi_version(void) { return UELLM_ABI_VERSION; }

uint64_t uellm_sizeof(int which)
{
    switch (which) {
    case 0: return sizeof(uellm_config);
    case 1: return sizeof(uellm_batch_stat);
    case 2: return sizeof(uellm_totals);
    case 3: return sizeof(uellm_profile);
    case 4: return sizeof(uellm_diagnostics);
    case 5: return sizeof(uellm_sim_totals);
    case 6: return sizeof(uellm_predictor);
    case 7: return sizeof(uellm_monitor_state);
    case 8: return sizeof(uellm_topology);
    case 9: return sizeof(uellm_device_map);
    default: return 0;
    }
}

const char *uellm_status_string(uellm_status s)
{
    switch (s) {
    case UELLM_OK: return "UELLM_OK";
    case UELLM_ERR_ARG: return "UELLM_ERR_ARG";
    case UELLM_ERR_CONTRACT: return "UELLM_ERR_CONTRACT";
    case UELLM_ERR_CONFIG: return "UELLM_ERR_CONFIG";
    case UELLM_ERR_OVERFLOW: return "UELLM_ERR_OVERFLOW";
    case UELLM_ERR_CUDA: return "UELLM_ERR_CUDA";
    case UELLM_ERR_UNSUPPORTED: return "UELLM_ERR_UNSUPPORTED";
    case UELLM_ERR_STALE: return "UELLM_ERR_STALE";
    default: return "UELLM_ERR_UNKNOWN";
    }
}

size_t uellm_workspace_bytes(uint64_t n, const uellm_config *cfg)
{
    if (!cfg) return 0;
    return (size_t)make_layout(n, *cfg).total;
}

uellm_status uellm_profile_load(const uellm_queries *q, const uellm_config *cfg, void *ws, size_t ws_bytes,
                                void *stream, uellm_profile *out)
{
    uellm::NvtxRange nvtx_("uellm_profile_load");
    if (!q || !cfg || !out) return UELLM_ERR_ARG;
    const uint64_t n = q->n;
    if (n >= 0xffffffffull) return UELLM_ERR_ARG;
    if (n > 0 && (!q->input_len || !q->pred_out_len || !q->slo_s)) return UELLM_ERR_ARG;
    uellm_status s = check_config(cfg);
    if (s != UELLM_OK) return s;
    const WsLayout L = make_layout(n, *cfg);
    if (!ws || (reinterpret_cast<uintptr_t>(ws) & 255) || ws_bytes < L.total) return UELLM_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    uint8_t *w = (uint8_t *)ws;

    ProfileView v;
    std::memset(&v, 0, sizeof v);
    v.magic = kProfileMagic;
    v.n = n; v.window = L.window; v.nwin = L.nwin; v.ws = w; v.ws_bytes = ws_bytes;
    v.W = cfg->max_batch;
    v.cfg_hash = layout_key(cfg);
    v.diag_off = L.diag;
    v.wincost_off = L.wincost;
    v.meta_off = L.meta;
    if (n == 0) {
        std::memcpy(out, &v, sizeof v);
        return UELLM_OK;
    }
    const uint32_t *din = q->input_len, *dout = q->pred_out_len;
    const float *dslo = q->slo_s;
    if (!is_device_ptr(din)) {
        CU(cudaMemcpyAsync(at<uint32_t>(w, L.stage_in), din, 4 * n, cudaMemcpyHostToDevice, st));
        din = at<uint32_t>(w, L.stage_in);
    }
    if (!is_device_ptr(dout)) {
        CU(cudaMemcpyAsync(at<uint32_t>(w, L.stage_out), dout, 4 * n, cudaMemcpyHostToDevice, st));
        dout = at<uint32_t>(w, L.stage_out);
    }
    if (!is_device_ptr(dslo)) {
        CU(cudaMemcpyAsync(at<float>(w, L.stage_slo), dslo, 4 * n, cudaMemcpyHostToDevice, st));
        dslo = at<float>(w, L.stage_slo);
    }
    LoadMeta *meta = at<LoadMeta>(w, L.meta);
    CU(cudaMemsetAsync(meta, 0, sizeof(LoadMeta), st));
    CU(cudaMemsetAsync(&meta->key_and, 0xff, sizeof(unsigned long long), st));
    CU(cudaMemsetAsync(at<uint32_t>(w, L.slo_set), 0, 4 * kSloSetSize, st));
    CU(launch_load(din, dout, dslo, n, meta, at<uint32_t>(w, L.slo_set), st));
    LoadMeta hm;
    CU(cudaMemcpyAsync(&hm, meta, sizeof hm, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    if (hm.bad) return UELLM_ERR_CONTRACT;
    // overflow bounds (checked once, with the true maxima)
    typedef unsigned __int128 u128;
    const u128 W = cfg->max_batch;
    const u128 E = (u128)cfg->t_batch_us + (u128)cfg->t_iter_us * hm.max_out +
                   ((u128)cfg->t_tok_us * hm.max_out + (u128)cfg->t_prefill_us * hm.max_in) * W;
    const u128 bound = (u128)L.window * (E + (u128)cfg->lambda_us * W);
    if (bound >= ((u128)1 << 63)) return UELLM_ERR_OVERFLOW;
    const u128 kv = (u128)cfg->kv_bytes_per_elem * cfg->n_layers * cfg->hidden * W * ((u128)hm.max_in + hm.max_out);
    if (kv >= ((u128)1 << 64)) return UELLM_ERR_OVERFLOW;
    v.d_in = din; v.d_out = dout; v.d_slo = dslo;
    v.max_in = hm.max_in; v.max_out = hm.max_out; v.max_slo = hm.max_slo;
    v.key_or = hm.key_or; v.key_and = hm.key_and;
    v.slo_distinct = hm.slo_distinct; v.slo_overflow = hm.slo_overflow;
    {
        // rank table + compact (value, rank) hash of the distinct SLO values, once per profile: the
        // compressed sort key of every later schedule (and the fused reload) uses it
        const KeyPlan kp = key_plan(v);
        if (kp.ok)
            CU(launch_slo_table(at<uint32_t>(w, L.slo_set), at<uint32_t>(w, L.slo_table),
                                at<unsigned long long>(w, L.slo_ctab), kp.cbits, st));
        v.key_plan = kp.ok ? 1u : 0u;
        v.keys_ready = 0;
    }
    std::memcpy(out, &v, sizeof v);
    return UELLM_OK;
}

uellm_status uellm_profile_reload(uellm_profile *p, const uellm_queries *q, const uellm_config *cfg, void *stream)
{
    uellm::NvtxRange nvtx_("uellm_profile_reload");
    if (!p || !q || !cfg) return UELLM_ERR_ARG;
    ProfileView v;
    std::memcpy(&v, p, sizeof v);
    if (v.magic != kProfileMagic || v.cfg_hash != layout_key(cfg) || q->n != v.n) return UELLM_ERR_ARG;
    const uint64_t n = v.n;
    if (n == 0) return UELLM_OK;
    if (!is_device_ptr(q->input_len) || !is_device_ptr(q->pred_out_len) || !is_device_ptr(q->slo_s))
        return UELLM_ERR_ARG;
    const WsLayout L = make_layout(n, *cfg);
    cudaStream_t st = (cudaStream_t)stream;
    uint8_t *w = v.ws;
    LoadMeta *meta = at<LoadMeta>(w, L.meta);
    CU(cudaMemsetAsync(meta, 0, sizeof(LoadMeta), st));
    ReloadRef ref;
    ref.max_in = v.max_in; ref.max_out = v.max_out; ref.slo_distinct = v.slo_distinct;
    ref.slo_overflow = v.slo_overflow; ref.key_or = v.key_or; ref.key_and = v.key_and;
    const KeyPlan kp = key_plan(v);
    ref.fused = kp.ok ? 1u : 0u;
    if (kp.ok) {
        // rank-compressed profile: validation + key pack + first-pass histogram in one kernel
        CU(launch_reload_pack32(q->input_len, q->pred_out_len, q->slo_s, n, L.window,
                                at<unsigned long long>(w, L.slo_ctab), kp.cbits, kp.ob, at<uint32_t>(w, L.keysc),
                                at<uint32_t>(w, L.hist0), meta, st));
    } else {
        CU(cudaMemsetAsync(&meta->key_and, 0xff, sizeof(unsigned long long), st));
        CU(cudaMemsetAsync(at<uint32_t>(w, L.slo_set), 0, 4 * kSloSetSize, st));
        CU(launch_load(q->input_len, q->pred_out_len, q->slo_s, n, meta, at<uint32_t>(w, L.slo_set), st));
    }
    CU(launch_reload_check(meta, ref, st));
    v.keys_ready = kp.ok ? 1u : 0u;
    v.d_in = q->input_len; v.d_out = q->pred_out_len; v.d_slo = q->slo_s;
    std::memcpy(p, &v, sizeof v);
    return UELLM_OK;
}

uellm_status uellm_profile_status(const uellm_profile *p, uint32_t **device_word)
{
    if (!p || !device_word) return UELLM_ERR_ARG;
    const ProfileView &v = *view_of(p);
    if (v.magic != kProfileMagic) return UELLM_ERR_ARG;
    *device_word = &reinterpret_cast<LoadMeta *>(v.ws + v.meta_off)->status;
    return UELLM_OK;
}

uellm_status uellm_schedule_batches(const uellm_profile *p, const uellm_config *cfg, uint32_t *order,
                                    uint32_t *batch_offsets, uint64_t *num_batches, void *stream)
{
    uellm::NvtxRange nvtx_("uellm_schedule_batches");
    if (!p || !cfg || !num_batches) return UELLM_ERR_ARG;
    const ProfileView &v = *view_of(p);
    if (v.magic != kProfileMagic || v.cfg_hash != layout_key(cfg)) return UELLM_ERR_ARG;
    uellm_status s = check_config(cfg);
    if (s != UELLM_OK) return s;
    const uint64_t n = v.n;
    if (n > 0 && (!order || !batch_offsets)) return UELLM_ERR_ARG;
    if (!batch_offsets) return UELLM_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    uint8_t *w = v.ws;
    const WsLayout L = make_layout(n, *cfg);
    if (L.total > v.ws_bytes) return UELLM_ERR_ARG;
    const bool dev_order = n == 0 || is_device_ptr(order);
    const bool dev_offs = is_device_ptr(batch_offsets);
    const bool dev_nb = is_device_ptr(num_batches);
    uint32_t *d_order = dev_order ? order : at<uint32_t>(w, L.order);
    uint32_t *d_offs = dev_offs ? batch_offsets : at<uint32_t>(w, L.offsets);
    unsigned long long *d_nb = dev_nb ? (unsigned long long *)num_batches : at<unsigned long long>(w, L.nb);
    Diag *diag = at<Diag>(w, L.diag);
    {
        Diag hd;
        std::memset(&hd, 0, sizeof hd);
        hd.tiles = cfg->mode == UELLM_MODE_SEG_DP ? L.ntiles : 0;
        hd.tile_len = L.tile_len;
        CU(launch_set_u64s(st, {{reinterpret_cast<unsigned long long *>(diag), 0ull}}, true));
        CU(launch_set_u64s(st, {{&diag->tiles, hd.tiles}, {&diag->tile_len, hd.tile_len}}));
        CU(cudaMemsetAsync(at<unsigned long long>(w, L.wincost), 0, 8 * (L.nwin ? L.nwin : 1), st));
    }
    rec(v, UELLM_STAGE_SCHED_BEGIN, st);
    int launches = 4;     // small-store kernels: diag clear, tile sizes, sort record, launch count
    if (n == 0) {
        if (dev_offs) { CU(cudaMemsetAsync(batch_offsets, 0, 4, st)); }
        else batch_offsets[0] = 0;
        if (dev_nb) { CU(cudaMemsetAsync(num_batches, 0, 8, st)); }
        else *num_batches = 0;
        if (!dev_offs || !dev_nb) CU(cudaStreamSynchronize(st));
        return UELLM_OK;
    }
    // a3: sort (every mode except FIFO) + a4: records in scheduled order
    uint32_t *rin = at<uint32_t>(w, L.rin), *rout = at<uint32_t>(w, L.rout), *rslo = at<uint32_t>(w, L.rslo);
    int passes = 0, sk = 0;
    const KeyPlan kp = key_plan(v);
    const int ob = kp.ob, rb = kp.rb;
    const bool compressed = cfg->mode != UELLM_MODE_FIFO && kp.ok;
    DecodeArgs D;
    D.in = v.d_in; D.table = at<uint32_t>(w, L.slo_table); D.ob = ob;
    D.nslo = v.slo_distinct < kSloRankMax ? v.slo_distinct : kSloRankMax;
    D.packin = 0; D.wb = 0;
    D.rin = rin; D.rout = rout; D.rslo = rslo; D.order = d_order;
    if (compressed) {
        // keys rank << ob | out (rank table built at load) packed straight from the caller arrays
        // together with the digit-0 histogram -- by the fused reload already (keys_ready), else
        // here; the last pass writes the records (fused decode)
        uint32_t *kc = at<uint32_t>(w, L.keysc);
        uint32_t *vals0 = at<uint32_t>(w, L.vals0);
        const int cbits = kp.cbits;
        // window-local index and input length packed into the payload when they fit 32 bits
        int wbits = 0, ibits = 0;
        while (wbits < 32 && ((L.window - 1) >> wbits)) ++wbits;
        while (ibits < 32 && ((uint64_t)(v.max_in - 1) >> ibits)) ++ibits;
        if (wbits + ibits <= 32 && wbits < 32) { D.packin = 1; D.wb = wbits; }
        uint32_t mask = 0;
        for (int d = 0; d < 4; ++d) if (8 * d < rb + ob) mask |= 1u << d;
        // window groups: every pass of a group runs before the next group starts, so the group's
        // keys / payloads stay in L2 between passes
        const uint64_t gw = mask ? sort_group_windows(L.window, L.nwin) : L.nwin;
        const uint32_t *k32 = kc;
        for (uint64_t w0 = 0; w0 < L.nwin; w0 += gw) {
            const uint64_t wn = L.nwin - w0 < gw ? L.nwin - w0 : gw;
            if (!v.keys_ready) {
                CU(launch_pack32_hist(v.d_out, v.d_slo, n, L.window, w0, wn, at<unsigned long long>(w, L.slo_ctab),
                                      cbits, ob, kc, vals0, at<uint32_t>(w, L.hist0), st));
                launches += 1;
            }
            k32 = kc;
            const uint32_t *vals = nullptr;            // identity payload (arrival index = position)
            CU(radix_sort_windows32(&k32, &vals, (uint32_t *)at<unsigned long long>(w, L.keys1), at<uint32_t>(w, L.vals1),
                                    (uint32_t *)at<unsigned long long>(w, L.keys2), at<uint32_t>(w, L.vals2),
                                    at<uint32_t>(w, L.hist), at<uint32_t>(w, L.hist) + 256 * L.sort_tiles, n,
                                    L.window, w0, wn, mask, &passes, st,
                                    (mask & 1u) ? at<uint32_t>(w, L.hist0) : nullptr, &D, &sk));
            launches += sk;                            // scan + scatter per pass, histogram kernels
            if (passes == 0) {
                CU(launch_decode32(k32, vals, v.d_in, n, at<uint32_t>(w, L.slo_table), ob, rin, rout, rslo, d_order, st));
                launches += 1;                         // (mask == 0: one group covers every window)
            }
        }
        (void)vals0;
        rec(v, UELLM_STAGE_SORT_END, st);
    } else {
        unsigned long long *k0 = at<unsigned long long>(w, L.keys0);
        uint32_t *v0 = at<uint32_t>(w, L.vals0);
        CU(launch_pack64(v.d_out, v.d_slo, n, k0, v0, st));
        launches += 1;
        const unsigned long long *keys = k0;
        const uint32_t *vals = v0;
        if (cfg->mode != UELLM_MODE_FIFO) {
            const unsigned long long vary = v.key_or ^ v.key_and;
            uint32_t mask = 0;
            for (int d = 0; d < 8; ++d) if ((vary >> (8 * d)) & 0xffull) mask |= 1u << d;
            const uint64_t gw = sort_group_windows(L.window, L.nwin);
            for (uint64_t w0 = 0; w0 < L.nwin; w0 += gw) {
                const uint64_t wn = L.nwin - w0 < gw ? L.nwin - w0 : gw;
                keys = k0;
                vals = v0;
                CU(radix_sort_windows(&keys, &vals, at<unsigned long long>(w, L.keys1), at<uint32_t>(w, L.vals1),
                                      at<unsigned long long>(w, L.keys2), at<uint32_t>(w, L.vals2),
                                      at<uint32_t>(w, L.hist), at<uint32_t>(w, L.hist) + 256 * L.sort_tiles, n,
                                    L.window, w0, wn, mask, &passes, st, &D, &sk));
                launches += sk;
                if (passes == 0) break;
            }
        }
        rec(v, UELLM_STAGE_SORT_END, st);
        if (passes == 0) {
            CU(launch_decode(keys, vals, v.d_in, n, rin, rout, rslo, d_order, st));
            launches += 1;
        }
    }
    rec(v, UELLM_STAGE_DECODE_END, st);
    {
        unsigned long long sp[2] = {(unsigned long long)passes, compressed ? (unsigned long long)(rb + ob) : 64ull};
        CU(launch_set_u64s(st, {{&diag->sort_passes, sp[0]}, {&diag->sort_key_bits, sp[1]}}));
    }
    // a6/a7: segmentation -> boundary bitmap
    uint32_t *bm = at<uint32_t>(w, L.bitmap);
    CU(cudaMemsetAsync(bm, 0, 4 * L.nwords, st));
    const unsigned long long unit =
        (unsigned long long)cfg->kv_bytes_per_elem * cfg->n_layers * cfg->hidden;
    const unsigned long long cap_tok = cfg->kv_cap_bytes ? cfg->kv_cap_bytes / unit : ~0ull;
    if (cfg->mode == UELLM_MODE_SEG_DP) {
        DPParams P;
        std::memset(&P, 0, sizeof P);
        P.rin = rin; P.rout = rout; P.rslo = rslo;
        P.Cx = at<long long>(w, L.keys1); P.CFx = at<long long>(w, L.keys2);
        P.argx = at<uint16_t>(w, L.argx);
        P.Crf = at<long long>(w, L.st_so);             // the stats' scratch is free during the schedule
        P.Arf = at<uint16_t>(w, L.st_pin);
        P.tiles = at<TileRec>(w, L.tiles);
        P.tflags = at<uint32_t>(w, L.tflags);
        P.diag = diag;
        P.wincost = at<unsigned long long>(w, L.wincost);
        P.n = (uint32_t)n; P.window = (uint32_t)L.window; P.nwin = (uint32_t)L.nwin;
        P.tile_len = (uint32_t)L.tile_len; P.tpw = (uint32_t)L.tpw; P.W = cfg->max_batch;
        P.split = cfg->split_on_slo_change;
        P.cap_tok = cap_tok;
        P.t_batch = cfg->t_batch_us; P.t_iter = cfg->t_iter_us; P.t_tok = cfg->t_tok_us;
        P.t_pre = cfg->t_prefill_us; P.lambda = cfg->lambda_us;
        {
            typedef unsigned __int128 u128;
            const u128 E = (u128)cfg->t_batch_us + (u128)cfg->t_iter_us * v.max_out +
                           ((u128)cfg->t_tok_us * v.max_out + (u128)cfg->t_prefill_us * v.max_in) * cfg->max_batch;
            P.narrow = (v.max_in < 65536u && v.max_out < 65536u && E < ((u128)1 << 32) && !(cfg->flags & 1u)) ? 1u : 0u;
            P.many_runs = (v.slo_overflow || v.slo_distinct > kSloRankMax) ? 1u : 0u;
        }
        // candidate slots per warp: the blocked path holds at most W + 1 candidates after a prune
        // (b = 0 .. W at the block end) + 32 new ones (+ 32 more when a block only folds); the
        // generic path at most W + 1 and reads one slot ahead
        P.cap_slots = (uint32_t)align_up(cfg->max_batch + (P.narrow ? 33 + (UELLM_DP_PRUNE_EVERY > 1 ? 32 : 0) : 33), 32);
        // narrow path: the idle lanes of the fast block's u16 max table read up to 1984 bytes below it
        // (inside the warp's slot array, k_segdp.cu)
        if (P.narrow && P.cap_slots < 128) P.cap_slots = 128;
        void *ev[3] = {nullptr, nullptr, nullptr};
        for (int k = 0; k < 3; ++k)
            if ((uint64_t)(UELLM_STAGE_DP_LOCAL_END + k) < v.n_events) ev[k] = v.events[UELLM_STAGE_DP_LOCAL_END + k];
        int dl = 0;
        CU(run_segdp(P, L.ntiles, st, ev, &dl));
        launches += dl;
        int tl = 0;
        CU(run_traceback(P, bm, L.ntiles, at<uint16_t>(w, L.tmaps), at<uint32_t>(w, L.twflag), st, &tl));
        launches += tl;
    } else if (cfg->mode == UELLM_MODE_SLO_ODBS) {
        Alg1Params A;
        std::memset(&A, 0, sizeof A);
        A.rin = rin; A.rout = rout; A.rslo = rslo;
        A.n = (uint32_t)n; A.window = (uint32_t)L.window; A.nwin = (uint32_t)L.nwin; A.W = cfg->max_batch;
        A.split = cfg->split_on_slo_change; A.cap_tok = cap_tok;
        A.w1 = cfg->w1; A.w2 = cfg->w2; A.l1 = cfg->l1; A.l2 = cfg->l2; A.threshold = cfg->threshold;
        A.eps = cfg->eps; A.eq2_additive = cfg->eq2_additive;
        rec(v, UELLM_STAGE_DP_LOCAL_END, st); rec(v, UELLM_STAGE_DP_FIX_END, st); rec(v, UELLM_STAGE_DP_CASCADE_END, st);
        CU(launch_alg1(A, bm, at<uint16_t>(w, L.argx), at<uint2>(w, L.a1tiles), diag, st));
        launches += 4;
    } else {
        rec(v, UELLM_STAGE_DP_LOCAL_END, st); rec(v, UELLM_STAGE_DP_FIX_END, st); rec(v, UELLM_STAGE_DP_CASCADE_END, st);
        CU(launch_mark_fifo(bm, n, L.window, cfg->max_batch, cfg->mode == UELLM_MODE_SORT_ONLY, st));
        launches += 1;
    }
    rec(v, UELLM_STAGE_TRACE_END, st);
    // a7: compaction -> batch_offsets, num_batches (also kept in the workspace for stats)
    CU(run_compact(bm, n, at<uint32_t>(w, L.wscan), at<uint32_t>(w, L.blocksum), d_offs, d_nb, st));
    launches += 3;
    rec(v, UELLM_STAGE_SCHED_END, st);
    {
        unsigned long long lc = (unsigned long long)launches;
        CU(launch_set_u64s(st, {{&diag->sched_launches, lc}}));
    }
    if (!dev_order || !dev_offs || !dev_nb) {
        uint64_t m = 0;
        CU(cudaMemcpyAsync(&m, d_nb, 8, cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        if (!dev_nb) *num_batches = m;
        if (!dev_offs) CU(cudaMemcpyAsync(batch_offsets, d_offs, 4 * (m + 1), cudaMemcpyDeviceToHost, st));
        if (!dev_order) CU(cudaMemcpyAsync(order, d_order, 4 * n, cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
    }
    CU(cudaGetLastError());
    return UELLM_OK;
}

uellm_status uellm_batch_stats(const uellm_profile *p, const uellm_config *cfg, const uint32_t *batch_offsets,
                               const uint64_t *num_batches, uellm_batch_stat *per_batch, uellm_totals *totals,
                               void *stream)
{
    uellm::NvtxRange nvtx_("uellm_batch_stats");
    if (!p || !cfg || !totals || !batch_offsets || !num_batches) return UELLM_ERR_ARG;
    const ProfileView &v = *view_of(p);
    if (v.magic != kProfileMagic || v.cfg_hash != layout_key(cfg)) return UELLM_ERR_ARG;
    uellm_status s = check_config(cfg);
    if (s != UELLM_OK) return s;
    if (per_batch && !is_device_ptr(per_batch)) return UELLM_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    uint8_t *w = v.ws;
    const uint64_t n = v.n;
    const WsLayout L = make_layout(n, *cfg);
    const bool dev_tot = is_device_ptr(totals);
    const uint32_t *d_offs = is_device_ptr(batch_offsets) ? batch_offsets : at<uint32_t>(w, L.offsets);
    const unsigned long long *d_nb = is_device_ptr(num_batches) ? (const unsigned long long *)num_batches
                                                                : at<unsigned long long>(w, L.nb);
    if (n == 0) d_nb = at<unsigned long long>(w, L.nb);
    if (n == 0) CU(cudaMemsetAsync(at<unsigned long long>(w, L.nb), 0, 8, st));
    uellm_totals *d_tot = dev_tot ? totals : at<uellm_totals>(w, L.totals);
    StatsParams S;
    std::memset(&S, 0, sizeof S);
    S.rin = at<uint32_t>(w, L.rin); S.rout = at<uint32_t>(w, L.rout); S.rslo = at<uint32_t>(w, L.rslo);
    S.offsets = d_offs; S.num_batches = d_nb; S.n_cap = n; S.window = (uint32_t)L.window; S.nwin = (uint32_t)L.nwin;
    S.est = at<unsigned long long>(w, L.keys1); S.compl_ = at<unsigned long long>(w, L.keys2);
    S.blocksum_u32 = at<uint32_t>(w, L.blocksum); S.blockagg = at<unsigned long long>(w, L.blockagg);
    S.so = at<unsigned long long>(w, L.st_so); S.pin = at<unsigned long long>(w, L.st_pin);
    S.pout = at<unsigned long long>(w, L.st_pout);
    S.sorted = cfg->mode != UELLM_MODE_FIFO;
    S.per_batch = per_batch; S.acc = at<StatAcc>(w, L.acc); S.totals = d_tot; S.n = n;
    S.kv_unit = (unsigned long long)cfg->kv_bytes_per_elem * cfg->n_layers * cfg->hidden;
    S.kv_cap = cfg->kv_cap_bytes;
    S.t_batch = cfg->t_batch_us; S.t_iter = cfg->t_iter_us; S.t_tok = cfg->t_tok_us; S.t_pre = cfg->t_prefill_us;
    S.lambda = cfg->lambda_us;
    rec(v, UELLM_STAGE_STATS_BEGIN, st);
    CU(run_stats(S, st));
    rec(v, UELLM_STAGE_STATS_END, st);
    {
        unsigned long long lc = n ? 7ull : 2ull;       // + this small-store kernel
        CU(launch_set_u64s(st, {{&at<Diag>(w, L.diag)->stats_launches, lc}}));
    }
    if (!dev_tot) {
        CU(cudaMemcpyAsync(totals, d_tot, sizeof(uellm_totals), cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        if (totals->overflow) return UELLM_ERR_OVERFLOW;
    }
    return UELLM_OK;
}

uellm_status uellm_simulate(const uellm_profile *p, const uellm_config *cfg, const uint64_t *arrival_us,
                            const uint32_t *order, const uint32_t *batch_offsets, const uint64_t *num_batches,
                            uint64_t *batch_end_us, uint64_t *latency_us, uellm_sim_totals *totals, void *stream)
{
    uellm::NvtxRange nvtx_("uellm_simulate");
    if (!p || !cfg || !totals || !batch_offsets || !num_batches) return UELLM_ERR_ARG;
    const ProfileView &v = *view_of(p);
    if (v.magic != kProfileMagic || v.cfg_hash != layout_key(cfg)) return UELLM_ERR_ARG;
    uellm_status s = check_config(cfg);
    if (s != UELLM_OK) return s;
    const uint64_t n = v.n;
    if (n > 0 && (!arrival_us || !order)) return UELLM_ERR_ARG;
    if ((batch_end_us && !is_device_ptr(batch_end_us)) || (latency_us && !is_device_ptr(latency_us)))
        return UELLM_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    uint8_t *w = v.ws;
    const WsLayout L = make_layout(n, *cfg);
    if (L.total > v.ws_bytes) return UELLM_ERR_ARG;
    const bool dev_tot = is_device_ptr(totals);
    SimParams S;
    std::memset(&S, 0, sizeof S);
    if (n > 0) {
        const unsigned long long *arr = (const unsigned long long *)arrival_us;
        if (!is_device_ptr(arrival_us)) {
            // host arrivals: staged through keys2 (free scratch once the schedule is done)
            CU(cudaMemcpyAsync(at<unsigned long long>(w, L.keys2), arrival_us, 8 * n, cudaMemcpyHostToDevice, st));
            arr = at<unsigned long long>(w, L.keys2);
        }
        S.arrival = arr;
        S.order = is_device_ptr(order) ? order : at<uint32_t>(w, L.order);
        S.offsets = is_device_ptr(batch_offsets) ? batch_offsets : at<uint32_t>(w, L.offsets);
        S.num_batches = is_device_ptr(num_batches) ? (const unsigned long long *)num_batches
                                                   : at<unsigned long long>(w, L.nb);
    } else {
        S.num_batches = at<unsigned long long>(w, L.nb);
        CU(cudaMemsetAsync(at<unsigned long long>(w, L.nb), 0, 8, st));
    }
    S.rin = at<uint32_t>(w, L.rin); S.rout = at<uint32_t>(w, L.rout); S.rslo = at<uint32_t>(w, L.rslo);
    S.est = at<unsigned long long>(w, L.st_so);
    S.inc_a = at<unsigned long long>(w, L.st_pin);
    S.inc_b = at<unsigned long long>(w, L.st_pout);
    const uint64_t nch = ceil_div(n ? n : 1, kScanBlock);
    S.chunk_a = at<unsigned long long>(w, L.keys1);
    S.chunk_b = S.chunk_a + nch;
    S.carry = S.chunk_b + nch;
    S.arr_s = at<unsigned long long>(w, L.keys0);       // keys0: sort scratch, free after the schedule
    S.batch_end = (unsigned long long *)batch_end_us;
    S.latency = (unsigned long long *)latency_us;
    S.acc = at<SimAcc>(w, L.simacc);
    S.totals = dev_tot ? totals : at<uellm_sim_totals>(w, L.simtot);
    S.n = n; S.n_cap = n;
    S.t_batch = cfg->t_batch_us; S.t_iter = cfg->t_iter_us; S.t_tok = cfg->t_tok_us; S.t_pre = cfg->t_prefill_us;
    CU(run_simulate(S, st, nullptr));
    if (!dev_tot) {
        CU(cudaMemcpyAsync(totals, S.totals, sizeof(uellm_sim_totals), cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
    }
    return UELLM_OK;
}

// level-path scratch (0 = the level path does not apply: too many windows or factor levels)
static uint64_t predict_ws_bytes(uint64_t n, const uellm_predictor *pc, uint64_t *nwin_out)
{
    const uint64_t window = pc->window ? (pc->window < n ? pc->window : n) : (n ? n : 1);
    const uint64_t nwin = n ? ceil_div(n, window) : 0;
    if (nwin_out) *nwin_out = nwin;
    if (n == 0 || nwin > kPredMaxWindows) return 0;
    if (pc->monitor) {
        // the chain from factor 1 is the longest from any factor >= 1 (fl(v*gamma) is monotone)
        double v = 1.0;
        uint32_t K = 0;
        for (;;) {
            const double h = v * pc->gamma;
            const double nv = h < pc->cap ? h : pc->cap;
            if (nv == v) break;
            v = nv;
            if (++K >= kPredMaxLevels - 1) return 0;
        }
    }
    return align_up(8 * kPredMaxLevels, 256) + 256 + align_up(8ull * kPredMaxLevels * nwin, 256) + align_up(nwin, 256);
}

size_t uellm_predict_workspace_bytes(uint64_t n, const uellm_predictor *pc)
{
    if (!pc) return 0;
    return (size_t)predict_ws_bytes(n, pc, nullptr);
}

uellm_status uellm_predict_lengths(uint64_t n, const uint32_t *true_out_len, const uellm_predictor *pc,
                                   uellm_monitor_state *state, uint32_t *pred_out_len, double *window_factors,
                                   void *ws, size_t ws_bytes, void *stream)
{
    uellm::NvtxRange nvtx_("uellm_predict_lengths");
    if (!pc || !state || !is_device_ptr(state)) return UELLM_ERR_ARG;
    if (n >= 0xffffffffull) return UELLM_ERR_ARG;
    if (n > 0 && (!true_out_len || !pred_out_len || !is_device_ptr(true_out_len) || !is_device_ptr(pred_out_len)))
        return UELLM_ERR_ARG;
    if (window_factors && !is_device_ptr(window_factors)) return UELLM_ERR_ARG;
    if (pc->variant > UELLM_PREDICT_CONSTANT || pc->monitor > 1) return UELLM_ERR_CONFIG;
    if ((pc->variant == UELLM_PREDICT_BUCKETED || pc->variant == UELLM_PREDICT_NOISY) && pc->bucket_width < 1)
        return UELLM_ERR_CONFIG;
    if (pc->variant == UELLM_PREDICT_CONSTANT && pc->constant_tokens < 1) return UELLM_ERR_CONFIG;
    if (!(pc->error_rate >= 0.0 && pc->error_rate <= 1.0)) return UELLM_ERR_CONFIG;
    if (pc->monitor && !(pc->gamma >= 1.0 && pc->cap >= 1.0 && pc->gamma < 1e308 && pc->cap < 1e308))
        return UELLM_ERR_CONFIG;
    const uint64_t window = pc->window ? (pc->window < n ? pc->window : n) : (n ? n : 1);
    PredictParams P;
    std::memset(&P, 0, sizeof P);
    P.true_len = true_out_len; P.pred = pred_out_len; P.state = state; P.factors = window_factors;
    P.nwin = n ? ceil_div(n, window) : 0;
    P.variant = pc->variant; P.bucket_width = pc->bucket_width; P.constant_tokens = pc->constant_tokens;
    P.monitor = pc->monitor; P.error_rate = pc->error_rate; P.gamma = pc->gamma; P.cap = pc->cap;
    // the noisy draw u = (z >> 11) * 2^-53 is exact, so u < e  <=>  (z >> 11) < ceil(e * 2^53)
    // (e * 2^53 is exact; 0 <= e <= 1 checked above): one integer compare instead of FP64 work
    P.err_thresh = (unsigned long long)std::ceil(pc->error_rate * 9007199254740992.0);
    P.seed = pc->seed;
    uint64_t nwin_l = 0;
    const uint64_t need = predict_ws_bytes(n, pc, &nwin_l);
    if (ws && need && ws_bytes >= need && is_device_ptr(ws) && !(reinterpret_cast<uintptr_t>(ws) & 255)) {
        uint8_t *b = (uint8_t *)ws;
        P.levels = (double *)b;
        P.nlevels = (uint32_t *)(b + align_up(8 * kPredMaxLevels, 256));
        P.hist = (unsigned long long *)(b + align_up(8 * kPredMaxLevels, 256) + 256);
        P.wlevel = b + align_up(8 * kPredMaxLevels, 256) + 256 + align_up(8ull * kPredMaxLevels * nwin_l, 256);
    }
    CU(run_predict(P, n, window, (cudaStream_t)stream, nullptr));
    return UELLM_OK;
}

uellm_status uellm_boundary_bitmap(const uellm_profile *p, const uellm_config *cfg, uint32_t *words, void *stream)
{
    uellm::NvtxRange nvtx_("uellm_boundary_bitmap");
    if (!p || !cfg || !words) return UELLM_ERR_ARG;
    const ProfileView &v = *view_of(p);
    if (v.magic != kProfileMagic || v.cfg_hash != layout_key(cfg)) return UELLM_ERR_ARG;
    if (!is_device_ptr(words)) return UELLM_ERR_ARG;
    const WsLayout L = make_layout(v.n, *cfg);
    if (v.n == 0) {
        CU(cudaMemsetAsync(words, 0, 4, (cudaStream_t)stream));   // n = 0: the single boundary 0 (= n)
        CU(cudaMemsetAsync(words, 1, 1, (cudaStream_t)stream));
        return UELLM_OK;
    }
    CU(cudaMemcpyAsync(words, v.ws + L.bitmap, 4 * L.nwords, cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
    return UELLM_OK;
}

size_t uellm_exchange_bytes(uint64_t n_max) { return (size_t)exchange_record_bytes(n_max); }

uellm_status uellm_exchange_pack(const uellm_profile *p, const uellm_config *cfg, const uellm_totals *totals,
                                 void *record, uint64_t n_max, void *stream)
{
    if (!p || !cfg || !totals || !record) return UELLM_ERR_ARG;
    const ProfileView &v = *view_of(p);
    if (v.magic != kProfileMagic || v.cfg_hash != layout_key(cfg)) return UELLM_ERR_ARG;
    if (v.n > n_max || !is_device_ptr(record) || !is_device_ptr(totals) ||
        (reinterpret_cast<uintptr_t>(record) & 15))
        return UELLM_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    const uint64_t rb = exchange_record_bytes(n_max);
    uint8_t *r = (uint8_t *)record;
    const uint64_t bm_bytes = 4 * ((v.n + 1 + 31) / 32);
    CU(cudaMemcpyAsync(r, totals, sizeof(uellm_totals), cudaMemcpyDeviceToDevice, st));
    if (v.n == 0) {
        CU(cudaMemsetAsync(r + sizeof(uellm_totals), 0, rb - sizeof(uellm_totals), st));
        CU(cudaMemsetAsync(r + sizeof(uellm_totals), 1, 1, st));           // the single boundary 0 (= n)
        return UELLM_OK;
    }
    const WsLayout L = make_layout(v.n, *cfg);
    CU(cudaMemcpyAsync(r + sizeof(uellm_totals), v.ws + L.bitmap, bm_bytes, cudaMemcpyDeviceToDevice, st));
    const uint64_t used = sizeof(uellm_totals) + bm_bytes;
    if (rb > used) CU(cudaMemsetAsync(r + used, 0, rb - used, st));      // padding (initialised)
    return UELLM_OK;
}

namespace {
struct XcLayout { uint64_t qb, bitmap, wscan, blocksum, totals, total; };
XcLayout xc_layout(uint64_t n_total, uint32_t world)
{
    XcLayout X;
    uint64_t off = 0;
    auto take = [&](uint64_t bytes) { uint64_t o = off; off = align_up(off + (bytes ? bytes : 1), 256); return o; };
    const uint64_t nwords = (n_total + 1 + 31) / 32;
    X.qb = take(8ull * ((uint64_t)world + 1));
    X.bitmap = take(4 * nwords);
    X.wscan = take(4 * nwords);
    X.blocksum = take(4 * (ceil_div(nwords, kScanBlock) + 2));
    X.totals = take(sizeof(uellm_totals));
    X.total = off;
    return X;
}
}  // namespace

uellm_status uellm_totals_combine(const void *parts, uint32_t count, uint64_t stride_bytes, uellm_totals *out,
                                  void *ws, size_t ws_bytes, void *stream)
{
    uellm::NvtxRange nvtx_("uellm_totals_combine");
    if (!parts || count < 1 || stride_bytes < sizeof(uellm_totals) || (stride_bytes & 7) || !out) return UELLM_ERR_ARG;
    if (!is_device_ptr(parts)) return UELLM_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    const bool dev_out = is_device_ptr(out);
    if (!dev_out && (!ws || ws_bytes < sizeof(uellm_totals) || !is_device_ptr(ws))) return UELLM_ERR_ARG;
    uellm_totals *d_out = dev_out ? out : (uellm_totals *)ws;
    CU(launch_totals_combine((const uint8_t *)parts, count, stride_bytes, d_out, st));
    if (!dev_out) {
        CU(cudaMemcpyAsync(out, d_out, sizeof(uellm_totals), cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        if (out->overflow) return UELLM_ERR_OVERFLOW;
    }
    return UELLM_OK;
}

size_t uellm_exchange_workspace_bytes(uint64_t n_total, uint32_t world)
{
    if (world < 1) return 0;
    return (size_t)xc_layout(n_total, world).total;
}

uellm_status uellm_exchange_combine(const void *gathered, uint32_t world, uint64_t n_max, const uint64_t *query_begin,
                                    void *ws, size_t ws_bytes, uint32_t *batch_offsets, uint64_t *num_batches,
                                    uellm_totals *totals, void *stream)
{
    uellm::NvtxRange nvtx_("uellm_exchange_combine");
    if (!gathered || world < 1 || !query_begin || !batch_offsets || !num_batches || !totals) return UELLM_ERR_ARG;
    if (query_begin[0] != 0) return UELLM_ERR_ARG;
    for (uint32_t r = 0; r < world; ++r)
        if (query_begin[r + 1] < query_begin[r] || query_begin[r + 1] - query_begin[r] > n_max) return UELLM_ERR_ARG;
    const uint64_t n_total = query_begin[world];
    if (n_total >= 0xffffffffull) return UELLM_ERR_ARG;
    const XcLayout X = xc_layout(n_total, world);
    if (!ws || (reinterpret_cast<uintptr_t>(ws) & 255) || ws_bytes < X.total) return UELLM_ERR_ARG;
    if (!is_device_ptr(gathered) || !is_device_ptr(batch_offsets) || !is_device_ptr(num_batches)) return UELLM_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    uint8_t *w = (uint8_t *)ws;
    const bool dev_tot = is_device_ptr(totals);
    uellm_totals *d_tot = dev_tot ? totals : at<uellm_totals>(w, X.totals);
    // query_begin goes down as kernel parameters (a pageable host->device copy would synchronise
    // the stream first, and cannot be captured in a CUDA graph)
    unsigned long long *dqb = at<unsigned long long>(w, X.qb);
    for (uint32_t r0 = 0; r0 <= world; r0 += 4) {
        const uint32_t c = world + 1 - r0 < 4 ? world + 1 - r0 : 4;
        CU(launch_set_u64s(st, {{dqb + r0, query_begin[r0]},
                                {dqb + r0 + (c > 1 ? 1 : 0), query_begin[r0 + (c > 1 ? 1 : 0)]},
                                {dqb + r0 + (c > 2 ? 2 : 0), query_begin[r0 + (c > 2 ? 2 : 0)]},
                                {dqb + r0 + (c > 3 ? 3 : 0), query_begin[r0 + (c > 3 ? 3 : 0)]}}));
    }
    CU(run_exchange_combine((const uint8_t *)gathered, world, exchange_record_bytes(n_max),
                            at<unsigned long long>(w, X.qb), n_total, at<uint32_t>(w, X.bitmap),
                            at<uint32_t>(w, X.wscan), at<uint32_t>(w, X.blocksum), batch_offsets,
                            (unsigned long long *)num_batches, d_tot, st));
    if (!dev_tot) {
        CU(cudaMemcpyAsync(totals, d_tot, sizeof(uellm_totals), cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        if (totals->overflow) return UELLM_ERR_OVERFLOW;
    }
    return UELLM_OK;
}

size_t uellm_helr_workspace_bytes(uint32_t num_devices)
{
    if (num_devices < 1 || num_devices > kHelrMaxDevices) return 0;
    return (size_t)helr_layout(num_devices).total;
}

static uellm_status deploy_plan(const uellm_topology *t, void *ws, size_t ws_bytes, uellm_device_map *out, void *stream,
                                bool bgs)
{
    if (!t || !out) return UELLM_ERR_ARG;
    const uint32_t D = t->num_devices;
    if (D < 1 || D > kHelrMaxDevices || t->num_layers < 1 || t->model_bytes == 0) return UELLM_ERR_CONFIG;
    if (!t->memory_bytes || !t->performance || !t->link_latency_s) return UELLM_ERR_ARG;
    if (!(t->p >= 0.0) || !(t->a1 >= 0.0) || !(t->a2 >= 0.0) || !(t->p < 1e308) || !(t->a1 < 1e308) || !(t->a2 < 1e308))
        return UELLM_ERR_CONFIG;
    for (uint32_t d = 0; d < D; ++d)
        if (!(t->performance[d] > 0.0) || !(t->performance[d] < 1e308)) return UELLM_ERR_CONFIG;
    for (uint32_t e = 0; e < D * D; ++e)
        if (!(t->link_latency_s[e] >= 0.0) || !(t->link_latency_s[e] < 1e308)) return UELLM_ERR_CONFIG;
    const HelrLayout Lh = helr_layout(D);
    if (!ws || (reinterpret_cast<uintptr_t>(ws) & 255) || ws_bytes < Lh.total) return UELLM_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    uint8_t *w = (uint8_t *)ws;
    // host-side tables: caps (exact integer floor((mem - T) * L / M)), binomials
    uint32_t cap[kHelrMaxDevices];
    for (uint32_t d = 0; d < D; ++d) {
        const uint64_t mem = t->memory_bytes[d];
        if (mem <= t->kv_reserve_bytes) { cap[d] = 0; continue; }
        const unsigned __int128 q = (unsigned __int128)(mem - t->kv_reserve_bytes) * t->num_layers / t->model_bytes;
        cap[d] = q >= t->num_layers ? t->num_layers : (uint32_t)q;
    }
    static_assert(kHelrMaxDevices <= 20, "binomial table size");
    unsigned long long binom[(kHelrMaxDevices + 1) * (kHelrMaxDevices + 1)];
    for (uint32_t a = 0; a <= kHelrMaxDevices; ++a)
        for (uint32_t b = 0; b <= kHelrMaxDevices; ++b)
            binom[a * (kHelrMaxDevices + 1) + b] =
                b > a ? 0ull : (b == 0 || b == a) ? 1ull
                      : binom[(a - 1) * (kHelrMaxDevices + 1) + b - 1] + binom[(a - 1) * (kHelrMaxDevices + 1) + b];
    CU(cudaMemcpyAsync(at<uint32_t>(w, Lh.cap), cap, 4 * D, cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(at<unsigned long long>(w, Lh.mem), t->memory_bytes, 8 * D, cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(at<double>(w, Lh.perf), t->performance, 8 * D, cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(at<double>(w, Lh.lat), t->link_latency_s, 8 * D * D, cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(at<unsigned long long>(w, Lh.binom), binom, sizeof binom, cudaMemcpyHostToDevice, st));
    const bool dev_out = is_device_ptr(out);
    HelrParams H;
    std::memset(&H, 0, sizeof H);
    H.D = D; H.L = t->num_layers; H.p = t->p; H.a1 = t->a1; H.a2 = t->a2;
    H.m = (double)t->model_bytes / (double)t->num_layers;
    H.cap = at<uint32_t>(w, Lh.cap); H.mem = at<unsigned long long>(w, Lh.mem); H.perf = at<double>(w, Lh.perf); H.lat = at<double>(w, Lh.lat);
    H.binom = at<unsigned long long>(w, Lh.binom); H.binom_host = binom;
    H.capsum = at<unsigned long long>(w, Lh.capsum); H.dp = at<double>(w, Lh.dp); H.arg = at<uint8_t>(w, Lh.arg);
    H.part_obj = at<double>(w, Lh.part_obj); H.part_lat = at<double>(w, Lh.part_lat);
    H.part_sj = at<unsigned long long>(w, Lh.part_sj);
    H.out = dev_out ? out : at<uellm_device_map>(w, Lh.out);
    if (bgs) CU(run_bgs(H, st));
    else CU(run_helr(H, st, nullptr));
    if (!dev_out) {
        CU(cudaMemcpyAsync(out, H.out, sizeof(uellm_device_map), cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
    }
    // (pageable host->device copies return once the source has been staged, so the stack tables
    // above may go out of scope without a synchronisation)
    return UELLM_OK;
}

uellm_status uellm_helr_plan(const uellm_topology *t, void *ws, size_t ws_bytes, uellm_device_map *out, void *stream)
{
    uellm::NvtxRange nvtx_("uellm_helr_plan");
    return deploy_plan(t, ws, ws_bytes, out, stream, false);
}

uellm_status uellm_bgs_plan(const uellm_topology *t, void *ws, size_t ws_bytes, uellm_device_map *out, void *stream)
{
    uellm::NvtxRange nvtx_("uellm_bgs_plan");
    return deploy_plan(t, ws, ws_bytes, out, stream, true);
}

uellm_status uellm_set_stage_events(uellm_profile *p, void *const *events, uint32_t n)
{
    if (!p || n > UELLM_STAGE_COUNT || (n && !events)) return UELLM_ERR_ARG;
    ProfileView &v = *reinterpret_cast<ProfileView *>(p);
    if (v.magic != kProfileMagic) return UELLM_ERR_ARG;
    for (uint32_t k = 0; k < UELLM_STAGE_COUNT; ++k) v.events[k] = k < n ? events[k] : nullptr;
    v.n_events = n;
    return UELLM_OK;
}

uellm_status uellm_get_diagnostics(const uellm_profile *p, uellm_diagnostics *out, void *stream)
{
    uellm::NvtxRange nvtx_("uellm_get_diagnostics");
    if (!p || !out) return UELLM_ERR_ARG;
    const ProfileView &v = *view_of(p);
    if (v.magic != kProfileMagic) return UELLM_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    Diag hd;
    CU(cudaMemcpyAsync(&hd, v.ws + v.diag_off, sizeof hd, cudaMemcpyDeviceToHost, st));
    uint64_t nwin = v.nwin;
    uint64_t cost = 0;
    if (nwin) {
        uint64_t *wc = new uint64_t[nwin];
        if (cudaMemcpyAsync(wc, v.ws + v.wincost_off, 8 * nwin, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess) {
            delete[] wc;
            cudaGetLastError();
            return UELLM_ERR_CUDA;
        }
        for (uint64_t i = 0; i < nwin; ++i) cost += wc[i];
        delete[] wc;
    } else {
        CU(cudaStreamSynchronize(st));
    }
    out->tiles = hd.tiles; out->tile_len = hd.tile_len; out->fixups_unconverged = hd.fixups_unconverged;
    out->cascade_reruns = hd.cascade_reruns; out->fixup_positions = hd.fixup_positions;
    out->trace_unmerged = hd.trace_unmerged; out->trace_rewalks = hd.trace_rewalks;
    out->sort_passes = hd.sort_passes; out->dp_cost = cost;
    out->dp_candidate_evals = hd.dp_evals; out->sched_launches = hd.sched_launches;
    out->stats_launches = hd.stats_launches; out->sort_key_bits = hd.sort_key_bits;
    out->dp_filled_positions = hd.dp_filled;
    return UELLM_OK;
}

}  // extern "C"
