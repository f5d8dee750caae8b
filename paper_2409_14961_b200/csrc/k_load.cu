// k_load.cu -- a1/a2: validate profiled queries, SLO seconds -> integer us, key packing;
// SLO rank compression; decode of sorted keys into scheduled-order records; boundary marks of
// FIFO / sort-only.
//
// a1: reject input_len == 0, pred_out_len == 0, non-finite or <= 0 SLO and
//     slo_us outside [1, 2^32-1]; slo_us = rint(double(slo_s) * 1e6), half-even
//     (R12; the paper's SLOs are seconds).
// a2: key = slo_us << 32 | pred_out_len, payload = arrival index.  Ascending key order is
//     (SLO, predicted length) order (P:228 + R11); a stable sort keeps arrival order on ties
//     (R9).  Digits that are constant across all keys are skipped by the sort (OR/AND masks).
//     The load also collects the set of distinct slo_us values (per-CTA shared-memory hash set,
//     merged into a 4096-slot global set); with at most kSloRankMax distinct values the sort key
//     becomes rank(slo_us) << bits(max_out) | out in 32 bits -- the rank among the distinct
//     values preserves the key order exactly.
#include "internal.cuh"

namespace uellm {

__global__ void __launch_bounds__(256) k_load(const uint32_t *__restrict__ in, const uint32_t *__restrict__ out,
                                              const float *__restrict__ slo, uint64_t n,
                                              LoadMeta *meta, uint32_t *__restrict__ slo_set)
{
    constexpr uint32_t kCtaSlots = 2048, kCtaBits = 11, kCtaMax = kSloRankMax;
    __shared__ uint32_t cset[kCtaSlots];
    __shared__ uint32_t ccount, cover;
    for (uint32_t i = threadIdx.x; i < kCtaSlots; i += blockDim.x) cset[i] = 0;
    if (threadIdx.x == 0) { ccount = 0; cover = meta->slo_overflow; }
    __syncthreads();
    uint32_t bad = 0, mx_in = 0, mx_out = 0, mx_slo = 0;
    unsigned long long kor = 0, kand = ~0ull;
    // distinct-SLO collection, warp-synchronous and race-free: the warp's SLO values are grouped
    // with match.any and only one lane per distinct value touches the CTA set (atomicCAS only:
    // present -> old == su); stops once the CTA saw more than kCtaMax values (cover).
    const uint32_t lane = threadIdx.x & 31;
    constexpr int kLaneCache = 8;
    uint32_t cache[kLaneCache];
#pragma unroll
    for (int c = 0; c < kLaneCache; ++c) cache[c] = 0u;       // 0 is never a member (su >= 1)
    auto consume = [&](uint32_t a, uint32_t o, float sf, bool valid, bool cv) {
        bool ok = true;
        const uint32_t su = valid ? slo_to_us(sf, ok) : 0u;
        if (valid) {
            if (a == 0) bad |= 1u;
            if (o == 0) bad |= 2u;
            if (!ok) bad |= 4u;
            const unsigned long long key = ((unsigned long long)su << 32) | o;
            mx_in = max(mx_in, a); mx_out = max(mx_out, o); mx_slo = max(mx_slo, su);
            kor |= key; kand &= key;
        }
        if (cv) return;                                        // warp-uniform
        // per-lane cache of the last 8 values this lane already put through the CTA set: class-
        // valued SLOs hit it almost always, and a warp with no new value skips the match + CAS
        bool known = false;
#pragma unroll
        for (int c = 0; c < kLaneCache; ++c) known |= (cache[c] == su);
        const bool need = valid && su != 0u && !known;
        if (!__any_sync(0xffffffffu, need)) return;            // warp-uniform
        if (need) {
#pragma unroll
            for (int c = kLaneCache - 1; c > 0; --c) cache[c] = cache[c - 1];
            cache[0] = su;
        }
        const uint32_t k = need ? su : 0u;
        const uint32_t peers = __match_any_sync(0xffffffffu, k);
        if (k == 0u || lane != (uint32_t)(__ffs(peers) - 1)) return;
        uint32_t h = slo_hash(su, kCtaBits);
        for (uint32_t probe = 0; probe < kCtaSlots; ++probe) {
            const uint32_t old = atomicCAS(&cset[h], 0u, su);
            if (old == 0u) {
                if (atomicAdd(&ccount, 1u) + 1 > kCtaMax) atomicExch(&cover, 1u);
                break;
            }
            if (old == su) break;
            h = (h + 1) & (kCtaSlots - 1);
        }
    };
    auto cover_now = [&]() -> bool {                           // one shared atomic read per warp
        uint32_t c = 0;
        if (lane == 0) c = atomicOr(&cover, 0u);
        return __shfl_sync(0xffffffffu, c, 0) != 0u;
    };
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t head = 0;                          // elements handled by the vector loop
    if ((((uintptr_t)in | (uintptr_t)out | (uintptr_t)slo) & 15u) == 0) {
        const uint64_t n4 = n / 4;
        const uint4 *in4 = reinterpret_cast<const uint4 *>(in), *out4 = reinterpret_cast<const uint4 *>(out);
        const float4 *slo4 = reinterpret_cast<const float4 *>(slo);
        // the next iteration's three 16-byte loads are issued before this one is consumed (twice
        // the bytes in flight per warp: the consume loop is long enough to hide them)
        uint4 na = make_uint4(0, 0, 0, 0), no = make_uint4(0, 0, 0, 0);
        float4 nf = make_float4(0.f, 0.f, 0.f, 0.f);
        auto fetch = [&](uint64_t g) {
            if (g < n4) { na = __ldg(in4 + g); no = __ldg(out4 + g); nf = __ldg(slo4 + g); }
        };
        fetch(tid);
        for (uint64_t g0 = tid - lane; g0 < n4; g0 += stride) {    // whole warps iterate together
            const uint64_t g = g0 + lane;
            const bool v = g < n4;
            const uint4 a = na, o = no;
            const float4 f = nf;
            fetch(g + stride);
            const bool cv = cover_now();
            consume(a.x, o.x, f.x, v, cv);
            consume(a.y, o.y, f.y, v, cv);
            consume(a.z, o.z, f.z, v, cv);
            consume(a.w, o.w, f.w, v, cv);
        }
        head = n4 * 4;
    }
    for (uint64_t k0 = head + tid - lane; k0 < n; k0 += stride) {
        const uint64_t k = k0 + lane;
        const bool v = k < n;
        consume(v ? __ldg(in + k) : 0u, v ? __ldg(out + k) : 0u, v ? __ldg(slo + k) : 0.f, v, cover_now());
    }
    // warp reductions, one atomic per warp
    for (int d = 16; d; d >>= 1) {
        bad |= __shfl_xor_sync(0xffffffffu, bad, d);
        mx_in = max(mx_in, __shfl_xor_sync(0xffffffffu, mx_in, d));
        mx_out = max(mx_out, __shfl_xor_sync(0xffffffffu, mx_out, d));
        mx_slo = max(mx_slo, __shfl_xor_sync(0xffffffffu, mx_slo, d));
        kor |= __shfl_xor_sync(0xffffffffu, kor, d);
        kand &= __shfl_xor_sync(0xffffffffu, kand, d);
    }
    if ((threadIdx.x & 31) == 0) {
        if (bad) atomicOr(&meta->bad, bad);
        atomicMax(&meta->max_in, mx_in);
        atomicMax(&meta->max_out, mx_out);
        atomicMax(&meta->max_slo, mx_slo);
        atomicOr(&meta->key_or, kor);
        atomicAnd(&meta->key_and, kand);
    }
    __syncthreads();
    // merge the CTA's distinct SLO values into the global set
    if (*(volatile uint32_t *)&cover) {
        if (threadIdx.x == 0) atomicExch(&meta->slo_overflow, 1u);
        return;
    }
    for (uint32_t i = threadIdx.x; i < kCtaSlots; i += blockDim.x) {
        const uint32_t su = cset[i];
        if (!su) continue;
        uint32_t h = slo_hash(su, kSloSetBits);
        for (uint32_t probe = 0; probe < kSloSetSize; ++probe) {
            // a plain read first: after the first CTAs, every class value is already in the set, and
            // thousands of CTAs CAS-ing the same few slots serialised the kernel's tail
            const uint32_t cur = *(volatile uint32_t *)&slo_set[h];
            if (cur == su) break;
            if (cur != 0u) { h = (h + 1) & (kSloSetSize - 1); continue; }
            if (*(volatile uint32_t *)&meta->slo_distinct > kSloRankMax) { atomicExch(&meta->slo_overflow, 1u); break; }
            const uint32_t old = atomicCAS(&slo_set[h], 0u, su);
            if (old == 0u) { atomicAdd(&meta->slo_distinct, 1u); break; }
            if (old == su) break;
            h = (h + 1) & (kSloSetSize - 1);
        }
    }
}

// uellm_profile_reload: the verdict on the freshly loaded queries against the profile's decisions
// (every decision of the schedule / stats calls is monotone in these limits, see uellm.h)
__global__ void k_reload_check(LoadMeta *meta, ReloadRef ref)
{
    const LoadMeta m = *meta;
    uint32_t st = UELLM_OK;
    if (m.bad) st = UELLM_ERR_CONTRACT;
    else if (ref.fused) {
        // rank-compressed profile (k_reload_pack32): the keys were packed with the profile's rank
        // table, valid when every SLO value is in the profile's set and the maxima are not above it
        if (m.max_in > ref.max_in || m.max_out > ref.max_out || m.slo_missing) st = UELLM_ERR_STALE;
    } else if (m.max_in > ref.max_in || m.max_out > ref.max_out || m.slo_distinct != ref.slo_distinct ||
               m.slo_overflow != ref.slo_overflow || (m.key_or & ~ref.key_or) != 0ull ||
               (~m.key_and & ref.key_and) != 0ull)
        st = UELLM_ERR_STALE;
    meta->status = st;
}

cudaError_t launch_reload_check(LoadMeta *meta, ReloadRef ref, cudaStream_t st)
{
    k_reload_check<<<1, 1, 0, st>>>(meta, ref);
    return cudaGetLastError();
}

cudaError_t launch_load(const uint32_t *in, const uint32_t *out, const float *slo, uint64_t n,
                        LoadMeta *meta, uint32_t *slo_set, cudaStream_t st)
{
    if (n == 0) return cudaSuccess;
#ifndef UELLM_LOAD_CTAS_PER_SM
#define UELLM_LOAD_CTAS_PER_SM 16
#endif
    uint64_t blocks = ceil_div(n, 256ull * 8);      // ~8 queries per thread
    if (blocks > 148ull * UELLM_LOAD_CTAS_PER_SM) blocks = 148ull * UELLM_LOAD_CTAS_PER_SM;
    if (blocks < 1) blocks = 1;
    k_load<<<(unsigned)blocks, 256, 0, st>>>(in, out, slo, n, meta, slo_set);
    return cudaGetLastError();
}

// a2 (generic key): key64 = slo_us << 32 | out, payload = arrival index (inputs validated by load)
__global__ void __launch_bounds__(256) k_pack64(const uint32_t *__restrict__ out, const float *__restrict__ slo,
                                                uint64_t n, unsigned long long *__restrict__ keys,
                                                uint32_t *__restrict__ vals)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) {
        bool ok;
        const uint32_t su = slo_to_us(__ldg(slo + k), ok);
        keys[k] = ((unsigned long long)su << 32) | __ldg(out + k);
        vals[k] = (uint32_t)k;
    }
}

cudaError_t launch_pack64(const uint32_t *out, const float *slo, uint64_t n, unsigned long long *keys,
                          uint32_t *vals, cudaStream_t st)
{
    if (n == 0) return cudaSuccess;
    uint64_t blocks = ceil_div(n, 256ull * 4);
    if (blocks > 148ull * 16) blocks = 148ull * 16;
    k_pack64<<<(unsigned)blocks, 256, 0, st>>>(out, slo, n, keys, vals);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------
// Rank table of the distinct SLO values (one CTA): table[r] = r-th smallest value, and a compact
// open-addressing hash ctab (2^cbits slots >= 2 x the distinct values) of (value << 32 | rank) for
// the key packer -- a few hundred bytes to stage per CTA instead of the 4096-slot set.
__global__ void __launch_bounds__(1024) k_slo_table(const uint32_t *__restrict__ slo_set, uint32_t *__restrict__ table,
                                                    unsigned long long *__restrict__ ctab, int cbits)
{
    __shared__ uint32_t vals[kSloRankMax];
    __shared__ uint32_t cnt;
    const uint32_t C = 1u << cbits;
    if (threadIdx.x == 0) cnt = 0;
    for (uint32_t h = threadIdx.x; h < C; h += blockDim.x) ctab[h] = 0ull;
    __syncthreads();
    for (uint32_t h = threadIdx.x; h < kSloSetSize; h += blockDim.x) {
        const uint32_t v = slo_set[h];
        if (v) { const uint32_t k = atomicAdd(&cnt, 1u); if (k < kSloRankMax) vals[k] = v; }
    }
    __syncthreads();
    const uint32_t K = min(cnt, kSloRankMax);
    for (uint32_t r = K + threadIdx.x; r < kSloRankMax; r += blockDim.x) table[r] = 0;   // unused ranks
    for (uint32_t f = threadIdx.x; f < K; f += blockDim.x) {
        const uint32_t v = vals[f];
        uint32_t r = 0;
        for (uint32_t g = 0; g < K; ++g) r += vals[g] < v;
        table[r] = v;
        const unsigned long long e = ((unsigned long long)v << 32) | r;
        uint32_t h = slo_hash(v, (uint32_t)cbits);
        while (atomicCAS(ctab + h, 0ull, e) != 0ull) h = (h + 1) & (C - 1);    // values are distinct
    }
}

cudaError_t launch_slo_table(const uint32_t *slo_set, uint32_t *table, unsigned long long *ctab, int cbits,
                             cudaStream_t st)
{
    k_slo_table<<<1, 1024, 0, st>>>(slo_set, table, ctab, cbits);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------
// Decode: sorted (key, idx) -> records in scheduled order + order[] (caller indices).
__global__ void __launch_bounds__(256) k_decode(const unsigned long long *__restrict__ keys,
                                                const uint32_t *__restrict__ vals,
                                                const uint32_t *__restrict__ in, uint64_t n,
                                                uint32_t *__restrict__ rin, uint32_t *__restrict__ rout,
                                                uint32_t *__restrict__ rslo, uint32_t *__restrict__ order)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += stride) {
        unsigned long long key = keys[p];
        uint32_t idx = vals[p];
        rslo[p] = (uint32_t)(key >> 32);
        rout[p] = (uint32_t)key;
        rin[p] = __ldg(in + idx);
        order[p] = idx;
    }
}

__global__ void __launch_bounds__(256) k_decode32(const uint32_t *__restrict__ keys, const uint32_t *__restrict__ vals,
                                                  const uint32_t *__restrict__ in, uint64_t n,
                                                  const uint32_t *__restrict__ table, int ob,
                                                  uint32_t *__restrict__ rin, uint32_t *__restrict__ rout,
                                                  uint32_t *__restrict__ rslo, uint32_t *__restrict__ order)
{
    __shared__ uint32_t st[kSloRankMax];
    for (uint32_t i = threadIdx.x; i < kSloRankMax; i += blockDim.x) st[i] = table[i];
    __syncthreads();
    const uint32_t mask = ob >= 32 ? 0xffffffffu : ((1u << ob) - 1);
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += stride) {
        const uint32_t key = keys[p];
        const uint32_t idx = vals ? vals[p] : (uint32_t)p;
        rslo[p] = st[ob >= 32 ? 0 : key >> ob];
        rout[p] = key & mask;
        rin[p] = __ldg(in + idx);
        order[p] = idx;
    }
}

cudaError_t launch_decode(const unsigned long long *keys, const uint32_t *vals, const uint32_t *in,
                          uint64_t n, uint32_t *rin, uint32_t *rout, uint32_t *rslo,
                          uint32_t *order, cudaStream_t st)
{
    if (n == 0) return cudaSuccess;
    uint64_t blocks = ceil_div(n, 256ull * 4);
    if (blocks > 148ull * 32) blocks = 148ull * 32;
    k_decode<<<(unsigned)blocks, 256, 0, st>>>(keys, vals, in, n, rin, rout, rslo, order);
    return cudaGetLastError();
}

cudaError_t launch_decode32(const uint32_t *keys, const uint32_t *vals, const uint32_t *in, uint64_t n,
                            const uint32_t *table, int ob, uint32_t *rin, uint32_t *rout, uint32_t *rslo,
                            uint32_t *order, cudaStream_t st)
{
    if (n == 0) return cudaSuccess;
    uint64_t blocks = ceil_div(n, 256ull * 4);
    if (blocks > 148ull * 32) blocks = 148ull * 32;
    k_decode32<<<(unsigned)blocks, 256, 0, st>>>(keys, vals, in, n, table, ob, rin, rout, rslo, order);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------
// FIFO: batches are consecutive chunks of W inside each window, in arrival
// order.  Sort-only: every position is a boundary.  Bit b of the bitmap = "a batch starts at
// position b" (bit n = end).  One thread per 32-bit word, no atomics.
__global__ void k_mark_fifo(uint32_t *bitmap, uint64_t n, uint64_t window, uint32_t W, int sort_only)
{
    const uint64_t nwords = (n + 1 + 31) / 32;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nwords; w += stride) {
        uint32_t bits = 0;
        for (int b = 0; b < 32; ++b) {
            uint64_t p = w * 32 + b;
            if (p > n) break;
            bool set = (p == n) || sort_only || ((p % window) % W == 0);
            if (set) bits |= 1u << b;
        }
        bitmap[w] = bits;
    }
}

cudaError_t launch_mark_fifo(uint32_t *bitmap, uint64_t n, uint64_t window, uint32_t W, int sort_only,
                             cudaStream_t st)
{
    uint64_t nwords = (n + 1 + 31) / 32;
    uint64_t blocks = ceil_div(nwords, 256);
    if (blocks > 148ull * 16) blocks = 148ull * 16;
    if (blocks < 1) blocks = 1;
    k_mark_fifo<<<(unsigned)blocks, 256, 0, st>>>(bitmap, n, window, W, sort_only);
    return cudaGetLastError();
}

}  // namespace uellm

namespace uellm {

struct U64Stores4 {
    unsigned long long *dst[4];
    unsigned long long val[4];
    int n, zero_diag;
};

__global__ void k_set_u64s(U64Stores4 S)
{
    if (S.zero_diag) {
        unsigned long long *d = S.dst[0];
        for (unsigned i = threadIdx.x; i < sizeof(Diag) / 8; i += blockDim.x) d[i] = 0ull;
        return;
    }
    if ((int)threadIdx.x < S.n) *S.dst[threadIdx.x] = S.val[threadIdx.x];
}

cudaError_t launch_set_u64s(cudaStream_t st, std::initializer_list<U64Store> stores, bool zero_diag)
{
    U64Stores4 S = {};
    for (const U64Store &u : stores) {
        if (S.n == 4) return cudaErrorInvalidValue;
        S.dst[S.n] = u.dst;
        S.val[S.n] = u.val;
        ++S.n;
    }
    S.zero_diag = zero_diag ? 1 : 0;
    k_set_u64s<<<1, 32, 0, st>>>(S);
    return cudaGetLastError();
}

}  // namespace uellm
