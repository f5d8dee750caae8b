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
//   k_sort_up    per 4096-key tile (tiles never cross a window): digit histogram, warp-
//                aggregated with match.any (skewed class-valued SLO digits would otherwise
//                serialise on a few shared-memory bins).
//   k_sort_scan  per window: exclusive offsets of (tile, digit) in window-major order.
//   k_sort_down  per tile: stable rank of every key (match.any peers + per-warp running
//                counts), then scatter.  Stability: tile order, warp order, iteration order,
//                lane order all follow input order.
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
    __shared__ uint32_t h[256];
    const int tid = threadIdx.x;
    if (tid < 256) h[tid] = 0;
    __syncthreads();
    uint64_t start, end;
    const uint64_t tile = t0 + blockIdx.x;
    tile_range(tile, n, window, tpw, start, end);
#pragma unroll 4
    for (uint32_t i = 0; i < kSortItems; ++i) {
        uint64_t p = start + (uint64_t)i * kSortThreads + tid;
        bool valid = p < end;
        uint32_t act = __ballot_sync(0xffffffffu, valid);
        if (valid) {
            uint32_t d = (uint32_t)(kin[p] >> shift) & 0xffu;
            uint32_t peers = __match_any_sync(act, d);
            if ((threadIdx.x & 31) == (uint32_t)(__ffs(peers) - 1)) atomicAdd(&h[d], __popc(peers));
        }
    }
    __syncthreads();
    if (tid < 256) hist[tile * 256 + tid] = h[tid];
}

// 1024 threads per window: thread (g, d) owns digit d of the g-th quarter of the window's tiles.
// Column loads are issued 8 at a time (independent), so the pass is bandwidth- not latency-bound.
constexpr int kScanGroups = 4;
__global__ void __launch_bounds__(256 * kScanGroups) k_sort_scan(uint32_t *__restrict__ hist, uint64_t n,
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
    uint32_t *col = hist + (w * tpw) * 256 + d;
    uint32_t sum = 0;
    uint32_t k = k0;
    for (; k + 8 <= k1; k += 8) {
        uint32_t v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = col[(uint64_t)(k + u) * 256];
#pragma unroll
        for (int u = 0; u < 8; ++u) sum += v[u];
    }
    for (; k < k1; ++k) sum += col[(uint64_t)k * 256];
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
        for (int u = 0; u < 8; ++u) v[u] = col[(uint64_t)(k + u) * 256];
#pragma unroll
        for (int u = 0; u < 8; ++u) { col[(uint64_t)(k + u) * 256] = run; run += v[u]; }
    }
    for (; k < k1; ++k) { const uint32_t v = col[(uint64_t)k * 256]; col[(uint64_t)k * 256] = run; run += v; }
}

#ifndef UELLM_SORT_DOWN_MINB
#define UELLM_SORT_DOWN_MINB 5
#endif
template <class K, bool DECODE>
__global__ void __launch_bounds__(kSortThreads, UELLM_SORT_DOWN_MINB) k_sort_down(const K *__restrict__ kin, const uint32_t *__restrict__ vin,
                                                            K *__restrict__ kout, uint32_t *__restrict__ vout,
                                                            const uint32_t *__restrict__ hist, uint64_t n,
                                                            uint64_t window, uint64_t tpw, int shift, DecodeArgs D,
                                                            uint64_t t0)
{
    constexpr int kWarps = kSortThreads / 32;
    constexpr int kPerWarpIters = kSortTile / kWarps / 32;     // 16
    __shared__ uint32_t whist[kWarps][256];
    __shared__ uint32_t tbase[256], dstart[256];
    __shared__ uint32_t stab[DECODE && sizeof(K) == 4 ? kSloRankMax : 1];
    extern __shared__ __align__(16) unsigned char dyn[];      // staging: K[kSortTile] + u32[kSortTile]
    uint64_t start, end;
    const uint64_t tile = t0 + blockIdx.x;
    tile_range(tile, n, window, tpw, start, end);
    if (start >= end) return;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < kWarps * 256; i += kSortThreads) (&whist[0][0])[i] = 0;
    if (tid < 256) tbase[tid] = hist[tile * 256 + tid];
    if (DECODE && sizeof(K) == 4)
        for (int i = tid; i < (int)kSloRankMax; i += kSortThreads) stab[i] = D.table[i];
    __syncthreads();

    K kr[kPerWarpIters];
    uint32_t vr[kPerWarpIters], rank[kPerWarpIters];
    const uint64_t base = start + (uint64_t)warp * (kPerWarpIters * 32);
#pragma unroll
    for (int r = 0; r < kPerWarpIters; ++r) {
        uint64_t p = base + r * 32 + lane;
        bool valid = p < end;
        kr[r] = valid ? kin[p] : (K)0;
        vr[r] = valid ? (vin ? vin[p] : (uint32_t)p) : 0u;     // vin == NULL: identity payload
    }
    const uint32_t lt = lanemask_lt();
#pragma unroll
    for (int r = 0; r < kPerWarpIters; ++r) {
        uint64_t p = base + r * 32 + lane;
        bool valid = p < end;
        uint32_t act = __ballot_sync(0xffffffffu, valid);
        uint32_t d = (uint32_t)(kr[r] >> shift) & 0xffu;
        uint32_t peers = 0;
        if (valid) {
            peers = __match_any_sync(act, d);
            rank[r] = whist[warp][d] + __popc(peers & lt);
        }
        __syncwarp();
        if (valid && lane == __ffs(peers) - 1) whist[warp][d] += __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    if (tid < 256) {   // exclusive scan over warps, per digit; dstart = tile total of the digit
        uint32_t run = 0;
#pragma unroll
        for (int wv = 0; wv < kWarps; ++wv) {
            uint32_t c = whist[wv][tid];
            whist[wv][tid] = run;
            run += c;
        }
        dstart[tid] = run;
    }
    __syncthreads();
    for (int off = 1; off < 256; off <<= 1) {   // inclusive scan of the digit totals
        uint32_t v = (tid < 256 && tid >= off) ? dstart[tid - off] : 0u;
        __syncthreads();
        if (tid < 256) dstart[tid] += v;
        __syncthreads();
    }
    // stage the tile in shared memory in (digit, rank) order, then write every digit bucket as
    // one contiguous run: consecutive threads store consecutive addresses
    K *sk = reinterpret_cast<K *>(dyn);
    uint32_t *sv = reinterpret_cast<uint32_t *>(dyn + kSortTile * sizeof(K));
#pragma unroll
    for (int r = 0; r < kPerWarpIters; ++r) {
        uint64_t p = base + r * 32 + lane;
        if (p < end) {
            const uint32_t d = (uint32_t)(kr[r] >> shift) & 0xffu;
            const uint32_t loc = (d ? dstart[d - 1] : 0u) + whist[warp][d] + rank[r];
            sk[loc] = kr[r];
            sv[loc] = vr[r];
        }
    }
    __syncthreads();
    const uint32_t cnt = (uint32_t)(end - start);
    for (uint32_t i = tid; i < cnt; i += kSortThreads) {
        const K key = sk[i];
        const uint32_t d = (uint32_t)(key >> shift) & 0xffu;
        const uint32_t pos = tbase[d] + i - (d ? dstart[d - 1] : 0u);
        const uint32_t idx = sv[i];
        if (DECODE) {           // a4 fused: records at the final scheduled position
            if (sizeof(K) == 8) {
                D.rslo[pos] = (uint32_t)((unsigned long long)key >> 32);
                D.rout[pos] = (uint32_t)key;
            } else {
                const uint32_t k32 = (uint32_t)key;
                D.rslo[pos] = stab[D.ob >= 32 ? 0u : k32 >> D.ob];
                D.rout[pos] = D.ob >= 32 ? k32 : (k32 & ((1u << D.ob) - 1));
            }
            D.order[pos] = idx;
            D.rin[pos] = __ldg(D.in + idx);
        } else {
            kout[pos] = key;
            vout[pos] = idx;
        }
    }
}

template <class K>
static cudaError_t radix_sort_impl(const K **keys_io, const uint32_t **vals_io, K *keys_a, uint32_t *vals_a,
                                   K *keys_b, uint32_t *vals_b, uint32_t *hist, uint64_t n, uint64_t window,
                                   uint64_t w_first, uint64_t nwin, uint32_t digit_mask, int *passes,
                                   cudaStream_t st, bool hist0_ready, const DecodeArgs *dec)
{
    *passes = 0;
    if (n == 0) return cudaSuccess;
    const uint64_t tpw = ceil_div(window, kSortTile);
    const uint64_t tiles = tpw * nwin, t0 = tpw * w_first;
    const K *kin = *keys_io;
    const uint32_t *vin = *vals_io;
    int last = -1;
    for (int d = 0; d < (int)sizeof(K); ++d) if (digit_mask >> d & 1u) last = d;
    const DecodeArgs D0 = dec ? *dec : DecodeArgs{};
    for (int d = 0; d < (int)sizeof(K); ++d) {
        if (!(digit_mask >> d & 1u)) continue;
        K *kout = (*passes & 1) ? keys_b : keys_a;
        uint32_t *vout = (*passes & 1) ? vals_b : vals_a;
        if (!(hist0_ready && *passes == 0))
            k_sort_up<K><<<(unsigned)tiles, kSortThreads, 0, st>>>(kin, hist, n, window, tpw, 8 * d, t0);
        k_sort_scan<<<(unsigned)nwin, 256 * kScanGroups, 0, st>>>(hist, n, window, tpw, w_first);
        const size_t stage = kSortTile * (sizeof(K) + sizeof(uint32_t));
        if (dec && d == last) {
            cudaFuncSetAttribute(k_sort_down<K, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)stage);
            k_sort_down<K, true><<<(unsigned)tiles, kSortThreads, stage, st>>>(kin, vin, kout, vout, hist, n, window,
                                                                              tpw, 8 * d, D0, t0);
        } else {
            cudaFuncSetAttribute(k_sort_down<K, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)stage);
            k_sort_down<K, false><<<(unsigned)tiles, kSortThreads, stage, st>>>(kin, vin, kout, vout, hist, n, window,
                                                                               tpw, 8 * d, D0, t0);
        }
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        kin = kout;
        vin = vout;
        ++*passes;
    }
    *keys_io = kin;
    *vals_io = vin;
    return cudaSuccess;
}

cudaError_t radix_sort_windows(const unsigned long long **keys_io, const uint32_t **vals_io,
                               unsigned long long *keys_a, uint32_t *vals_a,
                               unsigned long long *keys_b, uint32_t *vals_b, uint32_t *hist,
                               uint64_t n, uint64_t window, uint64_t w_first, uint64_t nwin, uint32_t digit_mask,
                               int *passes, cudaStream_t st, const DecodeArgs *dec)
{
    return radix_sort_impl<unsigned long long>(keys_io, vals_io, keys_a, vals_a, keys_b, vals_b, hist, n, window,
                                               w_first, nwin, digit_mask, passes, st, false, dec);
}

cudaError_t radix_sort_windows32(const uint32_t **keys_io, const uint32_t **vals_io, uint32_t *keys_a,
                                 uint32_t *vals_a, uint32_t *keys_b, uint32_t *vals_b, uint32_t *hist, uint64_t n,
                                 uint64_t window, uint64_t w_first, uint64_t nwin, uint32_t digit_mask, int *passes,
                                 cudaStream_t st, bool hist0_ready, const DecodeArgs *dec)
{
    return radix_sort_impl<uint32_t>(keys_io, vals_io, keys_a, vals_a, keys_b, vals_b, hist, n, window, w_first,
                                     nwin, digit_mask, passes, st, hist0_ready, dec);
}

// a2 (compressed key) fused with the digit-0 histogram of the first radix pass:
// key32 = rank(slo_us) << ob | out per 4096-query tile, payload = arrival index.
__global__ void __launch_bounds__(kSortThreads) k_pack32_hist(const uint32_t *__restrict__ out,
                                                              const float *__restrict__ slo, uint64_t n,
                                                              uint64_t window, uint64_t tpw,
                                                              const uint32_t *__restrict__ slo_set,
                                                              const uint32_t *__restrict__ rank_of_slot, int ob,
                                                              uint32_t *__restrict__ keys32, uint32_t *__restrict__ vals,
                                                              uint32_t *__restrict__ hist, uint64_t t0)
{
    __shared__ uint32_t sset[kSloSetSize], srank[kSloSetSize];
    __shared__ uint32_t h[256];
    const int tid = threadIdx.x;
    for (uint32_t i = tid; i < kSloSetSize; i += kSortThreads) { sset[i] = slo_set[i]; srank[i] = rank_of_slot[i]; }
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
            uint32_t hh = slo_hash(su, kSloSetBits);
            while (sset[hh] != su) hh = (hh + 1) & (kSloSetSize - 1);
            const uint32_t key = (srank[hh] << ob) | orr[i];
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
                               uint64_t nwin, const uint32_t *slo_set, const uint32_t *rank_of_slot, int ob,
                               uint32_t *keys32, uint32_t *vals, uint32_t *hist0, cudaStream_t st)
{
    if (n == 0) return cudaSuccess;
    const uint64_t tpw = ceil_div(window, kSortTile);
    k_pack32_hist<<<(unsigned)(tpw * nwin), kSortThreads, 0, st>>>(out, slo, n, window, tpw, slo_set, rank_of_slot,
                                                                  ob, keys32, vals, hist0, tpw * w_first);
    return cudaGetLastError();
}

}  // namespace uellm
