// k_sort.cu -- a3: stable LSD radix sort of (key, arrival index), segmented by scheduling
// window (P:228 / P:256 "sort by SLO in ascending order", with the predicted length as
// secondary key, R11).  8-bit digits; digits constant over all keys are skipped.
//
// Two key layouts (chosen on the host after load):
//   u64  key = slo_us << 32 | out                           (any input)
//   u32  key = rank(slo_us) << bits(max_out) | out           (few distinct SLO values: the rank
//        of slo_us among the distinct values preserves the order exactly; 2 passes for c3/c4)
//
// Per pass (reduce-then-scan):
//   k_sort_up    per 2048-key tile (tiles never cross a window): digit histogram, warp-
//                aggregated with match.any (skewed class-valued SLO digits would otherwise
//                serialise on a few shared-memory bins).  Only for the first pass without a
//                fused histogram: every scatter counts the next pass's digit per destination tile.
//   k_sort_scan  per window: exclusive offsets of (tile, digit) in window-major order.
//   k_sort_down  per tile: stable rank of every key (match.any peers + per-warp running
//                counts), then scatter.  Stability: tile order, warp order, iteration order,
//                lane order all follow input order.
#include <type_traits>

#include "internal.cuh"

namespace uellm {

__device__ __forceinline__ uint32_t lanemask_lt()
{
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ void tile_range(uint64_t t, uint64_t n, uint64_t window, uint64_t tpw,
                                           uint64_t &start, uint64_t &end)
{
    uint64_t w = t / tpw, k = t % tpw;
    uint64_t w0 = w * window, wend = min(w0 + window, n);
    start = w0 + k * kSortTile;
    end = min(start + kSortTile, wend);
    if (start > end) start = end;
}

template <class K>
__global__ void __launch_bounds__(kSortThreads) k_sort_up(const K *__restrict__ kin, uint32_t *__restrict__ hist,
                                                          uint64_t n, uint64_t window, uint64_t tpw, int shift,
                                                          uint64_t t0)
{
    // per-warp digit counts by plain shared REDs (same-digit lanes serialise in the shared pipe,
    // no match.any), summed per digit at the end
    __shared__ uint32_t hw[kSortThreads / 32][256];
    const int tid = threadIdx.x;
#pragma unroll
    for (int w = 0; w < kSortThreads / 32; ++w) hw[w][tid] = 0;
    __syncthreads();
    uint32_t *const myh = hw[tid >> 5];
    uint64_t start, end;
    const uint64_t tile = t0 + blockIdx.x;
    tile_range(tile, n, window, tpw, start, end);
    const uint32_t cnt = (uint32_t)(end - start);
    if (sizeof(K) == 4 && cnt == (uint32_t)kSortTile && (((uintptr_t)(kin + start)) & 15u) == 0) {
        // full tile of u32 keys: two 16-byte loads per thread
        const uint4 *src = reinterpret_cast<const uint4 *>(kin + start);
        const uint4 a = __ldg(src + tid), b = __ldg(src + kSortThreads + tid);
        const uint32_t v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
        for (int u = 0; u < 8; ++u) atomicAdd(myh + ((v[u] >> shift) & 0xffu), 1u);
    } else {
#pragma unroll 4
        for (uint32_t i = 0; i < kSortItems; ++i) {
            const uint64_t p = start + (uint64_t)i * kSortThreads + tid;
            if (p < end) atomicAdd(myh + ((uint32_t)(kin[p] >> shift) & 0xffu), 1u);
        }
    }
    __syncthreads();
    uint32_t c = 0;
#pragma unroll
    for (int w = 0; w < kSortThreads / 32; ++w) c += hw[w][tid];
    hist[tile * 256 + tid] = c;
}

// 1024 threads per window: thread (g, d) owns digit d of the g-th quarter of the window's tiles.
// Column loads are issued 8 at a time (independent), so the pass is bandwidth- not latency-bound.
constexpr int kScanGroups = 4;
// src: the per-tile counts (src == hist: in place; the first pass reads the kept hist0 counts)
__global__ void __launch_bounds__(256 * kScanGroups) k_sort_scan(const uint32_t *src, uint32_t *hist, uint64_t n,
                                                                 uint64_t window, uint64_t tpw, uint64_t w_first)
{
    __shared__ uint32_t gs[kScanGroups][256];
    __shared__ uint32_t s[256];
    const uint64_t w = w_first + blockIdx.x;
    const int d = threadIdx.x & 255, g = threadIdx.x >> 8;
    const uint64_t w0 = w * window;
    const uint64_t L = min(window, n - w0);
    const uint32_t ntl = (uint32_t)ceil_div(L, kSortTile);
    const uint32_t per = (ntl + kScanGroups - 1) / kScanGroups;
    const uint32_t k0 = min(ntl, g * per), k1 = min(ntl, k0 + per);
    const uint32_t *scol = src + (w * tpw) * 256 + d;
    uint32_t *col = hist + (w * tpw) * 256 + d;
    uint32_t sum = 0;
    uint32_t k = k0;
    for (; k + 8 <= k1; k += 8) {
        uint32_t v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = scol[(uint64_t)(k + u) * 256];
#pragma unroll
        for (int u = 0; u < 8; ++u) sum += v[u];
    }
    for (; k < k1; ++k) sum += scol[(uint64_t)k * 256];
    gs[g][d] = sum;
    __syncthreads();
    if (g == 0) {
        uint32_t tot = 0;
#pragma unroll
        for (int q = 0; q < kScanGroups; ++q) tot += gs[q][d];
        s[d] = tot;
    }
    __syncthreads();
    for (int off = 1; off < 256; off <<= 1) {   // Hillis-Steele inclusive scan over digits
        uint32_t v = 0;
        if (g == 0 && d >= off) v = s[d - off];
        __syncthreads();
        if (g == 0) s[d] += v;
        __syncthreads();
    }
    uint32_t run = (uint32_t)w0 + (d ? s[d - 1] : 0u);
    for (int q = 0; q < g; ++q) run += gs[q][d];
    for (k = k0; k + 8 <= k1; k += 8) {
        uint32_t v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = scol[(uint64_t)(k + u) * 256];
#pragma unroll
        for (int u = 0; u < 8; ++u) { col[(uint64_t)(k + u) * 256] = run; run += v[u]; }
    }
    for (; k < k1; ++k) { const uint32_t v = scol[(uint64_t)k * 256]; col[(uint64_t)k * 256] = run; run += v; }
}

#ifndef UELLM_SORT_PIPE
#define UELLM_SORT_PIPE 1
#endif
// scatter rank phase: ballot multisplit instead of match.any -- kept for the one-tile u64 kernel
// (c5 sort 0.876 -> 0.831 ms), not for the pipelined u32 kernel (c4 sort 1.44 -> 1.64 ms)
#ifndef UELLM_SORT_RANK_BALLOT
#define UELLM_SORT_RANK_BALLOT 0
#endif
#ifndef UELLM_SORT_RANK_BALLOT64
#define UELLM_SORT_RANK_BALLOT64 1
#endif
#ifndef UELLM_SORT_NEXT32
#define UELLM_SORT_NEXT32 0          // u32 keys: k_sort_up counts the next pass's digits
#endif
#ifndef UELLM_SORT_NEXT
#define UELLM_SORT_NEXT 1            // the scatter counts the next pass's digits (no k_sort_up)
#endif
#ifndef UELLM_SORT_DOWN_MINB
#define UELLM_SORT_DOWN_MINB 5
#endif

// ---- TMA bulk copies (cp.async.bulk) into shared memory, completion on an mbarrier -------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    asm volatile("{\n\t.reg .pred P1;\n"
                 "WAIT_%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
                 "@!P1 bra WAIT_%=;\n}" :: "r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// Scatter pass of one digit.  Per 2048-key tile (tiles never cross a window): stable rank of
// every key (match.any peers + per-warp running counts), per-digit exclusive offsets, the tile
// staged in shared memory in (digit, rank) order, then every digit bucket written as one
// contiguous run.  Stability: tile order x warp order x iteration order x lane order = input order.
// PIPE: persistent CTAs; tile i+1's keys, payloads and histogram row are brought into shared
// memory by TMA bulk copies (cp.async.bulk, mbarrier completion) while tile i is ranked and
// written -- the load latency no longer sits between the CTA's phases.
// NEXT: also count the next pass's digit (shift_next) per destination tile into hist_next (the
// next pass then needs no histogram kernel of its own); a warp's (tile, digit) pairs are
// aggregated with match.any first.
// DECODE (last pass): a4 fused -- records written straight at the scheduled position.
#ifndef UELLM_SORT_PIPE_MINB
#define UELLM_SORT_PIPE_MINB 4
#endif
template <class K, bool DECODE, bool NEXT, bool PIPE>
__global__ void __launch_bounds__(kSortThreads, PIPE ? UELLM_SORT_PIPE_MINB : UELLM_SORT_DOWN_MINB)
k_sort_down(const K *__restrict__ kin, const uint32_t *__restrict__ vin, K *__restrict__ kout,
            uint32_t *__restrict__ vout, const uint32_t *__restrict__ hist, uint64_t n, uint64_t window,
            uint64_t tpw, int shift, DecodeArgs D, uint64_t t0, uint64_t ntiles, uint32_t *__restrict__ hist_next,
            int shift_next)
{
    constexpr int kWarps = kSortThreads / 32;
    constexpr int kPerWarpIters = kSortTile / kWarps / 32;
    constexpr uint32_t kStageBytes = kSortTile * (sizeof(K) + 4) + 1024;   // keys, payloads, hist row
    __shared__ uint32_t whist[kWarps][256];
    __shared__ uint32_t dofs[256], wsum[kWarps];
    __shared__ uint32_t tbase_s[PIPE ? 1 : 256];
    __shared__ uint32_t stab[DECODE && sizeof(K) == 4 ? kSloRankMax : 1];
    __shared__ __align__(8) uint64_t mbar[2];
    // dynamic smem: PIPE: 2 stages {keys, payloads, hist row}; a stage's keys / payloads are in
    // registers after the first phase, so its buffer doubles as the (digit, rank) staging area.
    // !PIPE: the staging area only.
    extern __shared__ __align__(16) unsigned char dyn[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    unsigned char *stg = dyn;
    // payload source of the tile: vin, or (first pass, packin) the caller's input lengths
    const bool vsrc = vin != nullptr || D.packin;
    const uint32_t *vptr = vin ? vin : D.in;
    auto issue = [&](uint64_t tile, int s) {                  // one thread: stage s <- tile
        uint64_t st_, en_;
        tile_range(tile, n, window, tpw, st_, en_);
        const uint32_t cnt = (uint32_t)(en_ - st_);
        const uint32_t bk = (cnt * (uint32_t)sizeof(K)) & ~15u, bv = vsrc ? (cnt * 4u) & ~15u : 0u;
        unsigned char *b = stg + s * kStageBytes;
        mbar_expect_tx(&mbar[s], bk + bv + 1024u);
        bulk_g2s(b + kSortTile * (sizeof(K) + 4), hist + tile * 256, 1024u, &mbar[s]);
        if (bk) bulk_g2s(b, kin + st_, bk, &mbar[s]);
        if (bv) bulk_g2s(b + kSortTile * sizeof(K), vptr + st_, bv, &mbar[s]);
    };
    if (DECODE && sizeof(K) == 4)
        for (uint32_t i = tid; i < D.nslo; i += kSortThreads) stab[i] = D.table[i];
    if (PIPE) {
        if (tid == 0) {
            mbar_init(&mbar[0], 1);
            mbar_init(&mbar[1], 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            if (blockIdx.x < ntiles) issue(t0 + blockIdx.x, 0);
        }
        __syncthreads();
    }
    const uint32_t lt = lanemask_lt();
    for (uint32_t it = 0;; ++it) {
        const uint64_t tl = (uint64_t)blockIdx.x + (PIPE ? (uint64_t)it * gridDim.x : 0ull);
        if (tl >= ntiles || (!PIPE && it > 0)) break;
        const uint64_t tile = t0 + tl;
        const int s = (int)(it & 1u);
        if (PIPE && tid == 0 && tl + gridDim.x < ntiles) issue(tile + gridDim.x, s ^ 1);   // stage s^1: read last round
        uint64_t start, end;
        tile_range(tile, n, window, tpw, start, end);
        const uint32_t cnt = (uint32_t)(end - start);
        const uint64_t wt0 = (tile / tpw) * tpw;                 // first tile of this window
        const uint64_t wp0 = (tile / tpw) * window;              // first position of this window
        K *sk = reinterpret_cast<K *>(stg + (PIPE ? s * kStageBytes : 0));
        uint32_t *sv = reinterpret_cast<uint32_t *>(stg + (PIPE ? s * kStageBytes : 0) + kSortTile * sizeof(K));
        const K *bkp = reinterpret_cast<const K *>(stg + s * kStageBytes);
        const uint32_t *bvp = reinterpret_cast<const uint32_t *>(stg + s * kStageBytes + kSortTile * sizeof(K));
        const uint32_t *tbase = PIPE ? reinterpret_cast<const uint32_t *>(stg + s * kStageBytes + kSortTile * (sizeof(K) + 4))
                                     : tbase_s;
        for (int i = tid; i < kWarps * 256; i += kSortThreads) (&whist[0][0])[i] = 0;
        if (!PIPE) {
            if (start >= end) return;
            if (tid < 256) tbase_s[tid] = hist[tile * 256 + tid];
        } else {
            mbar_wait(&mbar[s], (it >> 1) & 1u);
            // the bulk copies moved whole 16-byte granules: the last few keys / payloads directly
            K *bk_w = const_cast<K *>(bkp);
            uint32_t *bv_w = const_cast<uint32_t *>(bvp);
            const uint32_t ck = ((cnt * (uint32_t)sizeof(K)) & ~15u) / (uint32_t)sizeof(K);
            const uint32_t cv = vsrc ? ((cnt * 4u) & ~15u) / 4u : cnt;
            for (uint32_t i = ck + tid; i < cnt; i += kSortThreads) bk_w[i] = kin[start + i];
            for (uint32_t i = cv + tid; i < cnt; i += kSortThreads) bv_w[i] = vptr[start + i];
        }
        __syncthreads();

        K kr[kPerWarpIters];
        uint32_t vr[kPerWarpIters], rank[kPerWarpIters];
        const uint32_t base = (uint32_t)warp * (kPerWarpIters * 32);   // offset in the tile
        // FULL (every tile but a window's last): no per-key bounds tests
        const bool full = cnt == (uint32_t)kSortTile;
        auto load_rank = [&](auto full_tag) {
            constexpr bool FULL = decltype(full_tag)::value;
#pragma unroll
            for (int r = 0; r < kPerWarpIters; ++r) {
                const uint32_t o = base + r * 32 + lane;
                const bool valid = FULL || o < cnt;
                const uint64_t p = start + o;
                uint32_t v = 0;
                if (PIPE) {
                    kr[r] = valid ? bkp[o] : (K)0;
                    if (valid) v = vsrc ? bvp[o] : (uint32_t)p;
                } else {
                    kr[r] = valid ? kin[p] : (K)0;
                    if (valid) v = vin ? vin[p] : D.packin ? __ldg(D.in + p) : (uint32_t)p;
                }
                // first pass with packin: window-local index and input length (no gather at decode)
                if (!vin && D.packin) v = (uint32_t)(p - wp0) | ((v - 1u) << D.wb);
                vr[r] = v;
            }
#pragma unroll
            for (int r = 0; r < kPerWarpIters; ++r) {
                const bool valid = FULL || base + r * 32 + lane < cnt;
                const uint32_t act = FULL ? 0xffffffffu : __ballot_sync(0xffffffffu, valid);
                const uint32_t d = (uint32_t)(kr[r] >> shift) & 0xffu;
                uint32_t peers = 0;
                if (sizeof(K) == 8 ? UELLM_SORT_RANK_BALLOT64 : UELLM_SORT_RANK_BALLOT) {
                    // peers by a ballot per digit bit (multisplit): eight short-latency votes in
                    // place of one match.any whose result the rank chain waits for
                    peers = act;
#pragma unroll
                    for (int bb = 0; bb < 8; ++bb) {
                        const bool bit = (d >> bb) & 1u;
                        const uint32_t bal = __ballot_sync(0xffffffffu, bit);
                        peers &= bit ? bal : ~bal;
                    }
                    if (valid) rank[r] = whist[warp][d] + __popc(peers & lt);
                } else if (valid) {
                    peers = __match_any_sync(act, d);
                    rank[r] = whist[warp][d] + __popc(peers & lt);
                }
                __syncwarp();
                if (valid && lane == __ffs(peers) - 1) whist[warp][d] += __popc(peers);
                __syncwarp();
            }
        };
        if (full) load_rank(std::true_type{}); else load_rank(std::false_type{});
        __syncthreads();
        {   // per digit (thread tid): the 8 warps' counts -> each warp's first staging slot of the
            // digit, and dofs[d] = global position of staging slot 0 of digit d's run
            static_assert(kSortThreads == 256, "one thread per digit");
            uint32_t c[kWarps];
            uint32_t run = 0;
#pragma unroll
            for (int wv = 0; wv < kWarps; ++wv) { c[wv] = whist[wv][tid]; run += c[wv]; }
            uint32_t v = run;               // inclusive scan of the digit totals: shuffles + warp sums
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
                if (lane >= o) v += y;
            }
            if (lane == 31) wsum[warp] = v;
            __syncthreads();
            uint32_t add = 0;
            for (int q = 0; q < warp; ++q) add += wsum[q];
            const uint32_t excl = v + add - run;
            uint32_t acc = excl;
#pragma unroll
            for (int wv = 0; wv < kWarps; ++wv) { whist[wv][tid] = acc; acc += c[wv]; }
            dofs[tid] = tbase[tid] - excl;  // (mod 2^32)
            __syncthreads();
        }
        // stage the tile in shared memory in (digit, rank) order (PIPE: over the stage buffer, whose
        // reads all precede the __syncthreads of the scan above)
#pragma unroll
        for (int r = 0; r < kPerWarpIters; ++r) {
            if (full || base + r * 32 + lane < cnt) {
                const uint32_t d = (uint32_t)(kr[r] >> shift) & 0xffu;
                const uint32_t loc = whist[warp][d] + rank[r];
                sk[loc] = kr[r];
                sv[loc] = vr[r];
            }
        }
        __syncthreads();
        // every digit bucket as one contiguous run: consecutive threads store consecutive addresses
        const uint32_t wt0_32 = (uint32_t)wt0, wp0_32 = (uint32_t)wp0;
        // one key's record stores (payload idx from the staging area)
        auto store = [&](K key, uint32_t pos, uint32_t i) {
            const uint32_t idx = sv[i];
            if (DECODE) {
                if (sizeof(K) == 8) {
                    D.rslo[pos] = (uint32_t)((unsigned long long)key >> 32);
                    D.rout[pos] = (uint32_t)key;
                } else {
                    const uint32_t k32 = (uint32_t)key;
                    D.rslo[pos] = stab[D.ob >= 32 ? 0u : k32 >> D.ob];
                    D.rout[pos] = D.ob >= 32 ? k32 : (k32 & ((1u << D.ob) - 1));
                }
                if (D.packin) {
                    D.order[pos] = wp0_32 + (idx & ((1u << D.wb) - 1u));
                    D.rin[pos] = (idx >> D.wb) + 1u;
                } else {
                    D.order[pos] = idx;
                    D.rin[pos] = __ldg(D.in + idx);
                }
            } else {
                kout[pos] = key;
                vout[pos] = idx;
            }
        };
        auto next_slot = [&](K key, uint32_t pos) -> uint32_t {
            return (wt0_32 + ((pos - wp0_32) / (uint32_t)kSortTile)) * 256u + ((uint32_t)(key >> shift_next) & 0xffu);
        };
        auto write_out = [&](auto full_tag) {
            constexpr bool FULL = decltype(full_tag)::value;
#pragma unroll(FULL ? kSortItems : 4)
            for (uint32_t r = 0; r < kSortItems; ++r) {                  // whole warps iterate together
                const uint32_t i = r * kSortThreads + tid;
                if (!FULL && r * kSortThreads + (uint32_t)(tid - lane) >= cnt) break;
                const bool valid = FULL || i < cnt;
                K key = 0;
                uint32_t pos = 0;
                if (valid) {
                    key = sk[i];
                    pos = dofs[(uint32_t)(key >> shift) & 0xffu] + i;
                }
                if (NEXT) {
                    const uint32_t act = FULL ? 0xffffffffu : __ballot_sync(0xffffffffu, valid);
                    if (valid) {
                        const uint32_t slot = next_slot(key, pos);
                        const uint32_t peers = __match_any_sync(act, slot);
                        if (lane == (uint32_t)(__ffs(peers) - 1)) atomicAdd(hist_next + slot, (uint32_t)__popc(peers));
                    }
                }
                if (valid) store(key, pos, i);
            }
        };
        if (full) write_out(std::true_type{}); else write_out(std::false_type{});
        // staging and stage s are free for the next round; the generic-proxy accesses of this round
        // are ordered before the next round's bulk copies (async proxy) into the same buffer
        if (PIPE) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
    }
}

// launches one scatter pass (pipelined persistent kernel when the TMA copies are 16-byte aligned)
template <class K, bool DECODE, bool NEXT>
static cudaError_t launch_down(bool pipe, const K *kin, const uint32_t *vin, K *kout, uint32_t *vout,
                               const uint32_t *hist, uint64_t n, uint64_t window, uint64_t tpw, int shift,
                               const DecodeArgs &D, uint64_t t0, uint64_t tiles, uint32_t *hist_next, int shift_next,
                               cudaStream_t st)
{
    const size_t stage = kSortTile * (sizeof(K) + sizeof(uint32_t));
    if (!pipe) {
        cudaFuncSetAttribute(k_sort_down<K, DECODE, NEXT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)stage);
        k_sort_down<K, DECODE, NEXT, false><<<(unsigned)tiles, kSortThreads, stage, st>>>(
            kin, vin, kout, vout, hist, n, window, tpw, shift, D, t0, tiles, hist_next, shift_next);
        return cudaGetLastError();
    }
    const size_t smem = 2 * (stage + 1024);
    cudaError_t e = cudaFuncSetAttribute(k_sort_down<K, DECODE, NEXT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, nsm = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_sort_down<K, DECODE, NEXT, true>, kSortThreads, smem);
    if (per < 1) per = 1;
    const uint64_t grid = tiles < (uint64_t)nsm * per ? tiles : (uint64_t)nsm * per;
    k_sort_down<K, DECODE, NEXT, true><<<(unsigned)grid, kSortThreads, smem, st>>>(
        kin, vin, kout, vout, hist, n, window, tpw, shift, D, t0, tiles, hist_next, shift_next);
    return cudaGetLastError();
}

template <class K>
static cudaError_t radix_sort_impl(const K **keys_io, const uint32_t **vals_io, K *keys_a, uint32_t *vals_a,
                                   K *keys_b, uint32_t *vals_b, uint32_t *hist, uint32_t *hist2, uint64_t n,
                                   uint64_t window, uint64_t w_first, uint64_t nwin, uint32_t digit_mask, int *passes,
                                   cudaStream_t st, const uint32_t *hist0, const DecodeArgs *dec, int *kernels)
{
    *passes = 0;
    int nk = 0;                                // kernels launched (scan, scatter, histogram)
    if (n == 0) return cudaSuccess;
    const uint64_t tpw = ceil_div(window, kSortTile);
    const uint64_t tiles = tpw * nwin, t0 = tpw * w_first;
    const K *kin = *keys_io;
    const uint32_t *vin = *vals_io;
    const DecodeArgs D0 = dec ? *dec : DecodeArgs{};
    uint32_t *hcur = hist, *hnext = hist2;
    // the first pass's per-tile counts: given (hist0, kept: the scan writes the offsets into hcur),
    // else counted here; later passes: counted by the previous scatter into hcur
    const uint32_t *hsrc = hist0;
    bool ready = hist0 != nullptr;
    for (int d = 0; d < (int)sizeof(K); ++d) {
        if (!(digit_mask >> d & 1u)) continue;
        int dn = -1;                           // the next pass's digit
        for (int q = d + 1; q < (int)sizeof(K); ++q) if (digit_mask >> q & 1u) { dn = q; break; }
        // u32 keys: the next pass's per-tile counts by a separate shared-RED histogram kernel over
        // this pass's output (c4 sort 1.47 -> 1.43 ms: the scatter's next-digit match.any was a
        // quarter of its stall samples); u64 keys (six passes) keep the fused count (c5 0.88 vs 0.90 ms)
        const bool fuse_next = (sizeof(K) == 8 ? UELLM_SORT_NEXT : UELLM_SORT_NEXT32) && dn >= 0;
        K *kout = (*passes & 1) ? keys_b : keys_a;
        uint32_t *vout = (*passes & 1) ? vals_b : vals_a;
        if (!ready) {
            k_sort_up<K><<<(unsigned)tiles, kSortThreads, 0, st>>>(kin, hcur, n, window, tpw, 8 * d, t0);
            hsrc = hcur;
            ++nk;
        }
        k_sort_scan<<<(unsigned)nwin, 256 * kScanGroups, 0, st>>>(hsrc ? hsrc : hcur, hcur, n, window, tpw, w_first);
        nk += 2;                               // scan + scatter
        hsrc = nullptr;
        // TMA bulk copies need 16-byte aligned tile starts: every tile of a window starts at a
        // multiple of kSortTile, so window starts (and the base pointers) must be aligned
        const bool vals_ok = vin ? ((uintptr_t)vin & 15u) == 0 : (!D0.packin || ((uintptr_t)D0.in & 15u) == 0);
        // (u64 keys: 83 KB per pipelined CTA leaves 2 CTAs per SM -- measured slower than the
        // one-tile kernel on c5, 0.94 vs 0.73 ms)
        const bool pipe = UELLM_SORT_PIPE && sizeof(K) == 4 && ((uintptr_t)kin & 15u) == 0 && vals_ok &&
                          (nwin + w_first == 1 || (window * sizeof(K)) % 16 == 0) && (window * 4) % 16 == 0;
        cudaError_t e;
        if (fuse_next) {
            if ((e = cudaMemsetAsync(hnext + t0 * 256, 0, tiles * 256 * sizeof(uint32_t), st))) return e;
            e = launch_down<K, false, true>(pipe, kin, vin, kout, vout, hcur, n, window, tpw, 8 * d, D0, t0, tiles,
                                            hnext, 8 * dn, st);
        } else if (dn >= 0 || !dec) {
            e = launch_down<K, false, false>(pipe, kin, vin, kout, vout, hcur, n, window, tpw, 8 * d, D0, t0, tiles,
                                             nullptr, 0, st);
        } else {
            e = launch_down<K, true, false>(pipe, kin, vin, kout, vout, hcur, n, window, tpw, 8 * d, D0, t0, tiles,
                                            nullptr, 0, st);
        }
        if (e != cudaSuccess) return e;
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        kin = kout;
        vin = vout;
        ++*passes;
        uint32_t *tmp = hcur; hcur = hnext; hnext = tmp;
        ready = fuse_next;
    }
    *keys_io = kin;
    *vals_io = vin;
    if (kernels) *kernels = nk;
    return cudaSuccess;
}

cudaError_t radix_sort_windows(const unsigned long long **keys_io, const uint32_t **vals_io,
                               unsigned long long *keys_a, uint32_t *vals_a,
                               unsigned long long *keys_b, uint32_t *vals_b, uint32_t *hist, uint32_t *hist2,
                               uint64_t n, uint64_t window, uint64_t w_first, uint64_t nwin, uint32_t digit_mask,
                               int *passes, cudaStream_t st, const DecodeArgs *dec, int *kernels)
{
    return radix_sort_impl<unsigned long long>(keys_io, vals_io, keys_a, vals_a, keys_b, vals_b, hist, hist2, n,
                                               window, w_first, nwin, digit_mask, passes, st, nullptr, dec, kernels);
}

cudaError_t radix_sort_windows32(const uint32_t **keys_io, const uint32_t **vals_io, uint32_t *keys_a,
                                 uint32_t *vals_a, uint32_t *keys_b, uint32_t *vals_b, uint32_t *hist, uint32_t *hist2,
                                 uint64_t n, uint64_t window, uint64_t w_first, uint64_t nwin, uint32_t digit_mask,
                                 int *passes, cudaStream_t st, const uint32_t *hist0, const DecodeArgs *dec,
                                 int *kernels)
{
    return radix_sort_impl<uint32_t>(keys_io, vals_io, keys_a, vals_a, keys_b, vals_b, hist, hist2, n, window,
                                     w_first, nwin, digit_mask, passes, st, hist0, dec, kernels);
}

// a2 (compressed key) fused with the digit-0 histogram of the first radix pass:
// key32 = rank(slo_us) << ob | out per 2048-query tile, payload = arrival index (implicit).
// The rank comes from the compact (value, rank) hash of k_slo_table (2^cbits slots).
__global__ void __launch_bounds__(kSortThreads) k_pack32_hist(const uint32_t *__restrict__ out,
                                                              const float *__restrict__ slo, uint64_t n,
                                                              uint64_t window, uint64_t tpw,
                                                              const unsigned long long *__restrict__ ctab, int cbits,
                                                              int ob, uint32_t *__restrict__ keys32,
                                                              uint32_t *__restrict__ hist, uint64_t t0)
{
    extern __shared__ unsigned long long sct[];
    __shared__ uint32_t h[256];
    const int tid = threadIdx.x;
    const uint32_t C = 1u << cbits;
    for (uint32_t i = tid; i < C; i += kSortThreads) sct[i] = ctab[i];
    if (tid < 256) h[tid] = 0;
    __syncthreads();
    uint64_t start, end;
    const uint64_t tile = t0 + blockIdx.x;
    tile_range(tile, n, window, tpw, start, end);
    // all loads first (independent, in flight together), then probe / pack / count
    float fr[kSortItems];
    uint32_t orr[kSortItems];
#pragma unroll
    for (uint32_t i = 0; i < kSortItems; ++i) {
        const uint64_t p = start + (uint64_t)i * kSortThreads + tid;
        fr[i] = p < end ? __ldg(slo + p) : 0.0f;
        orr[i] = p < end ? __ldg(out + p) : 0u;
    }
#pragma unroll
    for (uint32_t i = 0; i < kSortItems; ++i) {
        const uint64_t p = start + (uint64_t)i * kSortThreads + tid;
        const bool valid = p < end;
        const uint32_t act = __ballot_sync(0xffffffffu, valid);
        if (valid) {
            bool ok;
            const uint32_t su = slo_to_us(fr[i], ok);
            uint32_t hh = slo_hash(su, (uint32_t)cbits);
            unsigned long long e = sct[hh];
            while ((uint32_t)(e >> 32) != su) { hh = (hh + 1) & (C - 1); e = sct[hh]; }
            const uint32_t key = ((uint32_t)e << ob) | orr[i];
            keys32[p] = key;                       // payload = arrival index p: implicit (NULL vals)
            const uint32_t d = key & 0xffu;
            const uint32_t peers = __match_any_sync(act, d);
            if ((threadIdx.x & 31) == (uint32_t)(__ffs(peers) - 1)) atomicAdd(&h[d], __popc(peers));
        }
    }
    __syncthreads();
    if (tid < 256) hist[tile * 256 + tid] = h[tid];
}

cudaError_t launch_pack32_hist(const uint32_t *out, const float *slo, uint64_t n, uint64_t window, uint64_t w_first,
                               uint64_t nwin, const unsigned long long *ctab, int cbits, int ob, uint32_t *keys32,
                               uint32_t *vals, uint32_t *hist0, cudaStream_t st)
{
    (void)vals;
    if (n == 0) return cudaSuccess;
    const uint64_t tpw = ceil_div(window, kSortTile);
    k_pack32_hist<<<(unsigned)(tpw * nwin), kSortThreads, sizeof(unsigned long long) << cbits, st>>>(
        out, slo, n, window, tpw, ctab, cbits, ob, keys32, hist0, tpw * w_first);
    return cudaGetLastError();
}

// uellm_profile_reload of a rank-compressed profile: a1 (validation, maxima) + a2 (key pack) + the
// digit-0 histogram of the first radix pass in ONE pass over the caller arrays (the separate load and
// pack kernels read out / slo twice).  The key's rank comes from the profile's compact (value, rank)
// hash (k_slo_table ran at uellm_profile_load); a value outside the profile's distinct set has no
// rank and sets meta->slo_missing (-> UELLM_ERR_STALE: the compressed key was decided for that set).
// Persistent CTAs walk the sort tiles; VEC (16-byte aligned tiles): thread t owns elements
// 4t..4t+3 and 1024+4t..1024+4t+3 of a tile (16-byte loads and key stores), and the next tile's
// loads are issued before the current one is processed.  Validation bits and maxima are reduced per
// warp in registers and merged with one atomic each at the end.
#ifndef UELLM_RELOAD_FCACHE
#define UELLM_RELOAD_FCACHE 1
#endif
#ifndef UELLM_RELOAD_PERSIST
#define UELLM_RELOAD_PERSIST 1      // persistent CTAs with the next tile's loads in flight (else one tile per CTA)
#endif
template <bool VEC>
__global__ void __launch_bounds__(kSortThreads, UELLM_RELOAD_PERSIST ? 4 : 6) k_reload_pack32(const uint32_t *__restrict__ in,
                                                                const uint32_t *__restrict__ out,
                                                                const float *__restrict__ slo, uint64_t n,
                                                                uint64_t window, uint64_t tpw, uint64_t ntiles,
                                                                const unsigned long long *__restrict__ ctab,
                                                                int cbits, int ob, uint32_t *__restrict__ keys32,
                                                                uint32_t *__restrict__ hist, LoadMeta *meta)
{
    static_assert(kSortTile == 2048 && kSortThreads == 256, "VEC layout: 2 x 4 elements per thread");
    extern __shared__ unsigned long long sct[];
    // per-warp digit counts (no match.any: a lane's count is one shared RED, same-address lanes of a
    // warp serialise in the shared-memory pipe instead of costing issue slots), summed per tile
    __shared__ uint32_t hw[kSortThreads / 32][256];
    const int tid = threadIdx.x;
    const uint32_t lane = tid & 31;
    const uint32_t C = 1u << cbits;
    for (uint32_t i = tid; i < C; i += kSortThreads) sct[i] = ctab[i];
    uint32_t *const myh = hw[tid >> 5];
    uint32_t mx_in = 0, mx_out = 0, mn_in = 0xffffffffu, mn_out = 0xffffffffu, missing = 0;
    bool okall = true;
    // per-CTA cache float bits -> rank of the SLO values already validated and ranked (class-valued
    // SLOs hit it almost always: no double conversion, no rank-hash probe); one 64-bit entry per
    // slot, written whole, so a reader sees an old or a new entry, never a mix
    __shared__ unsigned long long fcache[64];
    if (UELLM_RELOAD_FCACHE && tid < 64) fcache[tid] = 0ull;
    // element e (0..7) of this thread inside the tile
    auto off = [&](int e) -> uint32_t {
        return VEC ? (uint32_t)((e >> 2) * 1024 + 4 * tid + (e & 3)) : (uint32_t)(e * kSortThreads + tid);
    };
    uint32_t na[kSortItems], no[kSortItems];
    float nf[kSortItems];
    auto fetch = [&](uint64_t tile) {
        uint64_t st_, en_;
        tile_range(tile, n, window, tpw, st_, en_);
        const uint32_t cnt = (uint32_t)(en_ - st_);
        if (VEC) {
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const uint32_t o0 = r * 1024 + 4 * tid;
                if (o0 + 4 <= cnt) {
                    const uint4 a = __ldg(reinterpret_cast<const uint4 *>(in + st_ + o0));
                    const uint4 o = __ldg(reinterpret_cast<const uint4 *>(out + st_ + o0));
                    const float4 f = __ldg(reinterpret_cast<const float4 *>(slo + st_ + o0));
                    na[4 * r] = a.x; na[4 * r + 1] = a.y; na[4 * r + 2] = a.z; na[4 * r + 3] = a.w;
                    no[4 * r] = o.x; no[4 * r + 1] = o.y; no[4 * r + 2] = o.z; no[4 * r + 3] = o.w;
                    nf[4 * r] = f.x; nf[4 * r + 1] = f.y; nf[4 * r + 2] = f.z; nf[4 * r + 3] = f.w;
                } else {
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const bool v = o0 + c < cnt;
                        na[4 * r + c] = v ? __ldg(in + st_ + o0 + c) : 1u;
                        no[4 * r + c] = v ? __ldg(out + st_ + o0 + c) : 1u;
                        nf[4 * r + c] = v ? __ldg(slo + st_ + o0 + c) : 1.0f;
                    }
                }
            }
        } else {
#pragma unroll
            for (int e = 0; e < kSortItems; ++e) {
                const uint32_t o = off(e);
                const bool v = o < cnt;
                na[e] = v ? __ldg(in + st_ + o) : 1u;
                no[e] = v ? __ldg(out + st_ + o) : 1u;
                nf[e] = v ? __ldg(slo + st_ + o) : 1.0f;
            }
        }
    };
    if ((uint64_t)blockIdx.x < ntiles) fetch(blockIdx.x);
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        uint32_t ca[kSortItems], co[kSortItems];
        float cf[kSortItems];
#pragma unroll
        for (int e = 0; e < kSortItems; ++e) { ca[e] = na[e]; co[e] = no[e]; cf[e] = nf[e]; }
        if (UELLM_RELOAD_PERSIST && tile + gridDim.x < ntiles) fetch(tile + gridDim.x);   // next tile in flight
#pragma unroll
        for (int w = 0; w < kSortThreads / 32; ++w) hw[w][tid] = 0;
        __syncthreads();                                  // (also orders the hash staging)
        uint64_t start, end;
        tile_range(tile, n, window, tpw, start, end);
        const uint32_t cnt = (uint32_t)(end - start);
        const bool full = cnt == kSortTile;
        uint32_t key[kSortItems];
#pragma unroll
        for (int e = 0; e < kSortItems; ++e) {
            const bool valid = full || off(e) < cnt;
            key[e] = 0;
            if (!valid) continue;
            const uint32_t a = ca[e], o = co[e];
            // validation by minima (a zero length is the minimum 0) and one flag: no per-key branches
            mn_in = min(mn_in, a);
            mn_out = min(mn_out, o);
            mx_in = max(mx_in, a);
            mx_out = max(mx_out, o);
            uint32_t rank;
            const uint32_t fb = __float_as_uint(cf[e]);
            const unsigned long long ce = UELLM_RELOAD_FCACHE ? fcache[(fb * 0x9E3779B1u) >> 26] : 0ull;
            if (UELLM_RELOAD_FCACHE && fb != 0u && (uint32_t)(ce >> 32) == fb) {
                rank = (uint32_t)ce;                       // this float was validated and ranked before
            } else {
                bool ok;
                const uint32_t su = slo_to_us(cf[e], ok);
                okall &= ok;
                uint32_t hh = slo_hash(su, (uint32_t)cbits);
                unsigned long long en = sct[hh];
                // (>= 8 slots per value up to 4096 slots: the first probe almost always decides; an
                // absent value ends at an empty slot)
                if ((uint32_t)(en >> 32) != su) {
                    while (en != 0ull && (uint32_t)(en >> 32) != su) { hh = (hh + 1) & (C - 1); en = sct[hh]; }
                    missing |= en == 0ull ? 1u : 0u;
                }
                rank = (uint32_t)en;
                if (UELLM_RELOAD_FCACHE && ok && en != 0ull)
                    fcache[(fb * 0x9E3779B1u) >> 26] = ((unsigned long long)fb << 32) | rank;
            }
            key[e] = (rank << ob) | o;
            atomicAdd(myh + (key[e] & 0xffu), 1u);
        }
        if (VEC) {
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const uint32_t o0 = r * 1024 + 4 * tid;
                if (o0 + 4 <= cnt)
                    *reinterpret_cast<uint4 *>(keys32 + start + o0) =
                        make_uint4(key[4 * r], key[4 * r + 1], key[4 * r + 2], key[4 * r + 3]);
                else
#pragma unroll
                    for (int c = 0; c < 4; ++c) if (o0 + c < cnt) keys32[start + o0 + c] = key[4 * r + c];
            }
        } else {
#pragma unroll
            for (int e = 0; e < kSortItems; ++e) if (off(e) < cnt) keys32[start + off(e)] = key[e];
        }
        __syncthreads();
        {
            uint32_t c = 0;
#pragma unroll
            for (int w = 0; w < kSortThreads / 32; ++w) c += hw[w][tid];
            hist[tile * 256 + tid] = c;
        }
        __syncthreads();                                  // hw is cleared for the next tile
    }
    uint32_t bad = (mn_in == 0u ? 1u : 0u) | (mn_out == 0u ? 2u : 0u) | (okall ? 0u : 4u);
    for (int d = 16; d; d >>= 1) {
        bad |= __shfl_xor_sync(0xffffffffu, bad, d);
        missing |= __shfl_xor_sync(0xffffffffu, missing, d);
        mx_in = max(mx_in, __shfl_xor_sync(0xffffffffu, mx_in, d));
        mx_out = max(mx_out, __shfl_xor_sync(0xffffffffu, mx_out, d));
    }
    if (lane == 0) {
        if (bad) atomicOr(&meta->bad, bad);
        if (missing) atomicOr(&meta->slo_missing, 1u);
        if (mx_in > *(volatile uint32_t *)&meta->max_in) atomicMax(&meta->max_in, mx_in);
        if (mx_out > *(volatile uint32_t *)&meta->max_out) atomicMax(&meta->max_out, mx_out);
    }
}

cudaError_t launch_reload_pack32(const uint32_t *in, const uint32_t *out, const float *slo, uint64_t n,
                                 uint64_t window, const unsigned long long *ctab, int cbits, int ob, uint32_t *keys32,
                                 uint32_t *hist0, LoadMeta *meta, cudaStream_t st)
{
    if (n == 0) return cudaSuccess;
    const uint64_t tpw = ceil_div(window, kSortTile);
    const uint64_t nwin = ceil_div(n, window);
    const uint64_t tiles = tpw * nwin;
    const size_t smem = sizeof(unsigned long long) << cbits;
    // 16-byte tiles: every tile starts at a multiple of kSortTile inside its window
    const bool vec = ((((uintptr_t)in | (uintptr_t)out | (uintptr_t)slo | (uintptr_t)keys32) & 15u) == 0) &&
                     (nwin == 1 || window % 4 == 0);
    int dev = 0, nsm = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (vec) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_reload_pack32<true>, kSortThreads, smem);
    else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_reload_pack32<false>, kSortThreads, smem);
    if (per < 1) per = 1;
    // persistent: one resident wave; otherwise one tile per CTA
    const uint64_t cap = UELLM_RELOAD_PERSIST ? (uint64_t)nsm * per : tiles;
    const unsigned grid = (unsigned)(tiles < cap ? tiles : cap);
    if (vec)
        k_reload_pack32<true><<<grid, kSortThreads, smem, st>>>(in, out, slo, n, window, tpw, tiles, ctab, cbits, ob,
                                                                keys32, hist0, meta);
    else
        k_reload_pack32<false><<<grid, kSortThreads, smem, st>>>(in, out, slo, n, window, tpw, tiles, ctab, cbits, ob,
                                                                 keys32, hist0, meta);
    return cudaGetLastError();
}

}  // namespace uellm
