// k_stats.cu -- a8: per-batch statistics of a schedule.
//   size b, s = max input (padded length), O = max predicted output, b x O generated
//   tokens, input / output padding, KV peak bytes 4*b*l*h*(s+O), est_us (R7),
//   completion_us = inclusive prefix of est_us over each window's batches,
//   viol_alone = #{slo_us < est_us}, viol_seq = #{slo_us < completion_us}, over_cap.
// Totals are exact integer sums (sum b*completion in 128 bits); the two reported doubles are
// formed once at the end.
//
//   k_stats_est    warp per batch: b, s, O -> est_us
//   k_seg_scan_*   segmented inclusive scan of est_us by window (chunk scan, chunk carries,
//                  carry-in), giving completion_us
//   k_stats_final  warp per batch: all fields, per-batch record, block-aggregated totals
//   k_totals       one thread: uellm_totals
#include "internal.cuh"

namespace uellm {

#ifndef UELLM_GROUP_LANES
#define UELLM_GROUP_LANES 8
#endif
constexpr uint32_t kStatsGroup = UELLM_GROUP_LANES;   // lanes per batch in the member-streaming loops

__device__ __forceinline__ uint32_t warp_max(uint32_t v)
{
    return __reduce_max_sync(0xffffffffu, v);
}
__device__ __forceinline__ uint32_t warp_sum(uint32_t v) { return __reduce_add_sync(0xffffffffu, v); }
__device__ __forceinline__ unsigned long long warp_sum64(unsigned long long v)
{
#pragma unroll
    for (int d = 16; d; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    return v;
}

struct BatchCore {
    uint32_t a, z, b, s, O;
    unsigned long long sin, sout, est;
};

__device__ __forceinline__ BatchCore batch_core(const StatsParams &S, uint64_t t)
{
    const uint32_t lane = threadIdx.x & 31;
    BatchCore c;
    c.a = S.offsets[t];
    c.z = S.offsets[t + 1];
    c.b = c.z - c.a;
    uint32_t s = 0, O = 0;
    unsigned long long si = 0, so = 0;
    for (uint32_t k = c.a + lane; k < c.z; k += 32) {
        const uint32_t vi = __ldg(S.rin + k), vo = __ldg(S.rout + k);
        s = max(s, vi); O = max(O, vo);
        si += vi; so += vo;
    }
    c.s = warp_max(s);
    c.O = warp_max(O);
    c.sin = warp_sum64(si);
    c.sout = warp_sum64(so);
    c.est = S.t_batch + S.t_iter * c.O + S.t_tok * (unsigned long long)c.b * c.O +
            S.t_pre * (unsigned long long)c.b * c.s;
    return c;
}

template <uint32_t G>
__device__ __forceinline__ void stats_est_body(const StatsParams &S, uint64_t m)
{
    // G lanes per batch: the group streams the batch's contiguous members with consecutive lanes
    // on consecutive positions (one 32-byte sector per load instruction and group), then reduces
    // across the group with shuffles
    const uint32_t lane = threadIdx.x & 31, sub = lane % G;
    const uint64_t ng = (uint64_t)gridDim.x * (blockDim.x / G);
    for (uint64_t t0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) / G; t0 < ceil_div(m, 32 / G) * (32 / G);
         t0 += ng) {
        const bool act = t0 < m;
        const uint64_t t = act ? t0 : m - 1;
        const uint32_t a = S.offsets[t], z = S.offsets[t + 1];
        uint32_t s = 0, O = 0;
        unsigned long long si64 = 0, so64 = 0;
        // four member loads per array in flight per lane (the batch's loads are independent; a
        // rolled loop waited for each before issuing the next)
        uint32_t k = a + sub;
        for (; k + 3 * G < z; k += 4 * G) {
            uint32_t vi[4], vo[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) { vi[u] = __ldg(S.rin + k + u * G); vo[u] = __ldg(S.rout + k + u * G); }
#pragma unroll
            for (int u = 0; u < 4; ++u) { s = max(s, vi[u]); O = max(O, vo[u]); si64 += vi[u]; so64 += vo[u]; }
        }
        for (; k < z; k += G) {
            const uint32_t vi = __ldg(S.rin + k), vo = __ldg(S.rout + k);
            s = max(s, vi); O = max(O, vo);
            si64 += vi; so64 += vo;
        }
#pragma unroll
        for (int d = G / 2; d; d >>= 1) {
            s = max(s, __shfl_xor_sync(0xffffffffu, s, d));
            O = max(O, __shfl_xor_sync(0xffffffffu, O, d));
            si64 += __shfl_xor_sync(0xffffffffu, si64, d);
            so64 += __shfl_xor_sync(0xffffffffu, so64, d);
        }
        if (act && sub == 0) {
            const unsigned long long b = z - a;
            S.est[t] = S.t_batch + S.t_iter * O + S.t_tok * b * O + S.t_pre * b * s;
            S.so[t] = (unsigned long long)s | ((unsigned long long)O << 32);
            S.pin[t] = b * s - si64;
            S.pout[t] = b * O - so64;
        }
    }
}

__global__ void __launch_bounds__(256) k_stats_est(StatsParams S)
{
    // lanes per batch from the mean batch size (uniform over the grid): 8 for SEG-DP-sized batches
    // (c4: 38 queries), 2 or 1 for the many small batches of Alg. 1 / sort-only schedules
    const uint64_t m = *S.num_batches;
    if (m == 0) return;
    const uint64_t mean = S.n / m;
    if (mean >= 24) stats_est_body<kStatsGroup>(S, m);
    else if (mean >= 6) stats_est_body<2>(S, m);
    else stats_est_body<1>(S, m);
}

// both violation counts of a batch: the two binary searches run in lockstep so their
// dependent loads overlap
__device__ __forceinline__ void count_below2(const StatsParams &S, uint32_t a, uint32_t z, unsigned long long x1,
                                             unsigned long long x2, uint32_t &c1, uint32_t &c2)
{
    // members ascend in slo_us only inside one window (a caller-modified segmentation may cross a
    // window boundary: then the plain count)
    if (S.sorted && a / S.window == (z - 1) / S.window) {
        uint32_t lo1 = a, hi1 = z, lo2 = a, hi2 = z;
        while (lo1 < hi1 || lo2 < hi2) {
            const uint32_t m1 = lo1 + (hi1 - lo1) / 2, m2 = lo2 + (hi2 - lo2) / 2;
            const bool g1 = lo1 < hi1, g2 = lo2 < hi2;
            const unsigned long long v1 = g1 ? __ldg(S.rslo + m1) : 0, v2 = g2 ? __ldg(S.rslo + m2) : 0;
            if (g1) { if (v1 < x1) lo1 = m1 + 1; else hi1 = m1; }
            if (g2) { if (v2 < x2) lo2 = m2 + 1; else hi2 = m2; }
        }
        c1 = lo1 - a;
        c2 = lo2 - a;
        return;
    }
    c1 = c2 = 0;
    for (uint32_t k = a; k < z; ++k) {
        const unsigned long long v = __ldg(S.rslo + k);
        c1 += v < x1;
        c2 += v < x2;
    }
}

// ---- segmented inclusive scan of est by window (head flag = first batch of a window) ----
__device__ __forceinline__ bool head_flag(const StatsParams &S, uint64_t t)
{
    return t == 0 || (S.offsets[t] / S.window) != (S.offsets[t - 1] / S.window);
}

// block-wide segmented inclusive scan of (v, f); returns inclusive value, aggregate in *agg/*aggf
__device__ unsigned long long block_seg_scan(unsigned long long v, uint32_t f, unsigned long long *agg,
                                             uint32_t *aggf)
{
    __shared__ unsigned long long sv[kScanBlock / 32];
    __shared__ uint32_t sf[kScanBlock / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        unsigned long long ov = __shfl_up_sync(0xffffffffu, v, d);
        uint32_t of = __shfl_up_sync(0xffffffffu, f, d);
        if (lane >= d) { if (!f) v += ov; f |= of; }
    }
    if (lane == 31) { sv[warp] = v; sf[warp] = f; }
    __syncthreads();
    if (warp == 0) {
        unsigned long long wv = lane < kScanBlock / 32 ? sv[lane] : 0;
        uint32_t wf = lane < kScanBlock / 32 ? sf[lane] : 0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            unsigned long long ov = __shfl_up_sync(0xffffffffu, wv, d);
            uint32_t of = __shfl_up_sync(0xffffffffu, wf, d);
            if (lane >= d) { if (!wf) wv += ov; wf |= of; }
        }
        if (lane < kScanBlock / 32) { sv[lane] = wv; sf[lane] = wf; }
    }
    __syncthreads();
    if (warp > 0 && !f) v += sv[warp - 1];   // f here = "a head in my warp prefix up to me"
    *agg = sv[kScanBlock / 32 - 1];
    *aggf = sf[kScanBlock / 32 - 1];
    __syncthreads();
    return v;
}

__global__ void __launch_bounds__(kScanBlock) k_seg_scan_local(StatsParams S)
{
    const uint64_t m = *S.num_batches;
    const uint64_t nchunks = ceil_div(m, kScanBlock);
    for (uint64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
        const uint64_t t = c * kScanBlock + threadIdx.x;
        const bool v = t < m;
        unsigned long long x = v ? S.est[t] : 0;
        uint32_t f = v ? head_flag(S, t) : 0;
        unsigned long long agg;
        uint32_t aggf;
        unsigned long long inc = block_seg_scan(x, f, &agg, &aggf);
        if (v) S.compl_[t] = inc;
        if (threadIdx.x == 0) { S.blockagg[c] = agg; S.blocksum_u32[c] = aggf; }
    }
}

// carry-in of every chunk: segmented exclusive scan of the chunk aggregates (one CTA)
__global__ void __launch_bounds__(kScanBlock) k_seg_scan_chunks(StatsParams S)
{
    const uint64_t m = *S.num_batches;
    const uint64_t nchunks = ceil_div(m, kScanBlock);
    const uint64_t per = ceil_div(nchunks, kScanBlock);
    const uint64_t a = threadIdx.x * per, z = min(a + per, nchunks);
    unsigned long long v = 0;
    uint32_t f = 0;
    for (uint64_t c = a; c < z; ++c) {             // thread-local segmented reduce
        if (S.blocksum_u32[c]) { v = S.blockagg[c]; f = 1; } else v += S.blockagg[c];
    }
    unsigned long long agg;
    uint32_t aggf;
    // exclusive = inclusive of the previous thread: shift by one via shared memory
    unsigned long long inc = block_seg_scan(v, f, &agg, &aggf);
    __shared__ unsigned long long incs[kScanBlock];
    incs[threadIdx.x] = inc;
    __syncthreads();
    unsigned long long carry = threadIdx.x ? incs[threadIdx.x - 1] : 0;
    for (uint64_t c = a; c < z; ++c) {
        const unsigned long long ag = S.blockagg[c];
        const uint32_t fl = S.blocksum_u32[c];
        S.blockagg[c] = carry;                     // carry into chunk c
        carry = fl ? ag : carry + ag;
    }
}

__global__ void __launch_bounds__(kScanBlock) k_seg_scan_apply(StatsParams S)
{
    __shared__ uint32_t seen_head;
    const uint64_t m = *S.num_batches;
    const uint64_t nchunks = ceil_div(m, kScanBlock);
    for (uint64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
        const uint64_t t = c * kScanBlock + threadIdx.x;
        const bool v = t < m;
        // carry applies to elements before the chunk's first head
        uint32_t f = v ? head_flag(S, t) : 0;
        const uint32_t bal = __ballot_sync(0xffffffffu, f);
        if (threadIdx.x == 0) seen_head = 0xffffffffu;
        __syncthreads();
        if (bal && (threadIdx.x & 31) == 0) atomicMin(&seen_head, (threadIdx.x & ~31u) + (__ffs(bal) - 1));
        __syncthreads();
        if (v && threadIdx.x < seen_head) S.compl_[t] += S.blockagg[c];
        __syncthreads();
    }
}

static_assert(sizeof(uellm_batch_stat) % 16 == 0, "record copied as uint4");
// ---- all fields + totals ----
__global__ void __launch_bounds__(256) k_stats_final(StatsParams S)
{
    // thread per batch: reads the pass-1 record, two binary searches for the violation counts
    __shared__ unsigned long long red[8][13];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t m = *S.num_batches;
    const uint64_t nt = (uint64_t)gridDim.x * blockDim.x;
    unsigned long long a_gen = 0, a_pin = 0, a_pout = 0, a_kv = 0, a_obj = 0, a_v1 = 0, a_v2 = 0, a_oc = 0,
                       a_mk = 0, a_llo = 0, a_lhi = 0, a_nb = 0;
    // dp_cost and makespan are the only sums the load's per-window bound does not cover: carry a
    // sticky overflow flag per field (bit 6 dp_cost, bit 10 makespan_us, as in uellm_totals)
    unsigned long long of = 0;
    // block-uniform loop: the 80-byte records go through shared memory and leave as coalesced
    // 16-byte stores (a record per thread would be ten 8-byte stores at an 80-byte lane stride)
    __shared__ __align__(16) uellm_batch_stat rec[256];
    const bool vec = ((uintptr_t)S.per_batch & 15) == 0;
    for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < m; base += nt) {
        const uint64_t t = base + threadIdx.x;
        if (t < m) {
            const uint32_t a = S.offsets[t], z = S.offsets[t + 1], b = z - a;
            const unsigned long long so = S.so[t], est = S.est[t], compl_us = S.compl_[t];
            const uint32_t s = (uint32_t)so, O = (uint32_t)(so >> 32);
            const unsigned long long pin = S.pin[t], pout = S.pout[t];
            uint32_t v1, v2;
            count_below2(S, a, z, est, compl_us, v1, v2);
            const unsigned long long kv = S.kv_unit * (unsigned long long)b * ((unsigned long long)s + O);
            const uint32_t oc = (S.kv_cap != 0 && kv > S.kv_cap) ? 1u : 0u;
            const unsigned long long gen = (unsigned long long)b * O;
            if (S.per_batch) {
                uellm_batch_stat &r = rec[threadIdx.x];
                r.start = a; r.size = b; r.max_in = s; r.max_out = O;
                r.gen_tokens = gen; r.pad_in = pin; r.pad_out = pout; r.kv_bytes = kv;
                r.est_us = est; r.completion_us = compl_us;
                r.viol_alone = v1; r.viol_seq = v2; r.over_cap = oc; r.window = a / S.window;
            }
            a_gen += gen; a_pin += pin; a_pout += pout; a_kv = max(a_kv, kv);
            const unsigned long long obj = est + S.lambda * v1;     // <= E + lambda*W (load bound)
            a_obj += obj; a_v1 += v1; a_v2 += v2; a_oc += oc; a_mk += est; a_nb += 1;
            of |= (a_obj < obj ? (1ull << 6) : 0ull) | (a_mk < est ? (1ull << 10) : 0ull);
            const unsigned long long lo = (unsigned long long)b * compl_us;
            const unsigned long long hi = __umul64hi((unsigned long long)b, compl_us);
            a_llo += lo; a_lhi += hi + (a_llo < lo ? 1ull : 0ull);
        }
        if (S.per_batch) {
            __syncthreads();
            const uint32_t cnt = (uint32_t)min((uint64_t)blockDim.x, m - base);
            if (vec) {
                const uint4 *src = reinterpret_cast<const uint4 *>(rec);
                uint4 *dst = reinterpret_cast<uint4 *>(S.per_batch + base);
                for (uint32_t i = threadIdx.x; i < cnt * (uint32_t)(sizeof(uellm_batch_stat) / 16); i += blockDim.x)
                    dst[i] = src[i];
            } else {
                const unsigned long long *src = reinterpret_cast<const unsigned long long *>(rec);
                unsigned long long *dst = reinterpret_cast<unsigned long long *>(S.per_batch + base);
                for (uint32_t i = threadIdx.x; i < cnt * (uint32_t)(sizeof(uellm_batch_stat) / 8); i += blockDim.x)
                    dst[i] = src[i];
            }
            __syncthreads();
        }
    }
    // warp reduction (128-bit carry for the latency sum)
#pragma unroll
    for (int d = 16; d; d >>= 1) {
        a_gen += __shfl_xor_sync(0xffffffffu, a_gen, d); a_pin += __shfl_xor_sync(0xffffffffu, a_pin, d);
        a_pout += __shfl_xor_sync(0xffffffffu, a_pout, d); a_kv = max(a_kv, __shfl_xor_sync(0xffffffffu, a_kv, d));
        {
            const unsigned long long o2 = __shfl_xor_sync(0xffffffffu, a_obj, d);
            const unsigned long long m2 = __shfl_xor_sync(0xffffffffu, a_mk, d);
            of |= __shfl_xor_sync(0xffffffffu, of, d);
            a_obj += o2; a_mk += m2;
            of |= (a_obj < o2 ? (1ull << 6) : 0ull) | (a_mk < m2 ? (1ull << 10) : 0ull);
        }
        a_v1 += __shfl_xor_sync(0xffffffffu, a_v1, d);
        a_v2 += __shfl_xor_sync(0xffffffffu, a_v2, d); a_oc += __shfl_xor_sync(0xffffffffu, a_oc, d);
        a_nb += __shfl_xor_sync(0xffffffffu, a_nb, d);
        const unsigned long long lo2 = __shfl_xor_sync(0xffffffffu, a_llo, d), hi2 = __shfl_xor_sync(0xffffffffu, a_lhi, d);
        const unsigned long long lo = a_llo + lo2;
        a_lhi += hi2 + (lo < a_llo ? 1ull : 0ull);
        a_llo = lo;
    }
    if (lane == 0) {
        unsigned long long *r = red[warp];
        r[0] = a_gen; r[1] = a_pin; r[2] = a_pout; r[3] = a_kv; r[4] = a_obj; r[5] = a_v1;
        r[6] = a_v2; r[7] = a_oc; r[8] = a_mk; r[9] = a_llo; r[10] = a_lhi; r[11] = a_nb; r[12] = of;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long s[13] = {};
        const int nwarps = blockDim.x >> 5;
        for (int w = 0; w < nwarps; ++w) {
            for (int f = 0; f < 13; ++f) {
                if (f == 3) s[3] = max(s[3], red[w][3]);
                else if (f == 9) { unsigned long long lo = red[w][9]; s[9] += lo; if (s[9] < lo) s[10] += 1; }
                else if (f == 12) s[12] |= red[w][12];
                else {
                    const unsigned long long x = red[w][f];
                    s[f] += x;
                    if (f == 4 && s[4] < x) s[12] |= 1ull << 6;
                    if (f == 8 && s[8] < x) s[12] |= 1ull << 10;
                }
            }
        }
        StatAcc *A = S.acc;
        if (s[11] == 0) return;
        atomicAdd(&A->gen, s[0]); atomicAdd(&A->pad_in, s[1]); atomicAdd(&A->pad_out, s[2]);
        atomicMax(&A->kv_max, s[3]); atomicAdd(&A->viol_alone, s[5]);
        atomicAdd(&A->viol_seq, s[6]); atomicAdd(&A->over_cap, s[7]);
        {
            const unsigned long long o4 = atomicAdd(&A->dp_cost, s[4]);
            const unsigned long long o8 = atomicAdd(&A->makespan, s[8]);
            if (o4 + s[4] < o4) s[12] |= 1ull << 6;
            if (o8 + s[8] < o8) s[12] |= 1ull << 10;
            if (s[12]) atomicOr(&A->overflow, s[12]);
        }
        const unsigned long long old = atomicAdd(&A->lat_lo, s[9]);
        atomicAdd(&A->lat_hi, s[10] + (old + s[9] < old ? 1ull : 0ull));
        atomicAdd(&A->batches, s[11]);
    }
}

__global__ void k_totals(StatsParams S)
{
    const StatAcc &A = *S.acc;
    uellm_totals T;
    T.n = S.n;
    T.batches = *S.num_batches;
    T.gen_tokens = A.gen; T.pad_in = A.pad_in; T.pad_out = A.pad_out; T.kv_bytes_max = A.kv_max;
    T.dp_cost = A.dp_cost; T.viol_alone = A.viol_alone; T.viol_seq = A.viol_seq; T.over_cap = A.over_cap;
    T.makespan_us = A.makespan;
    T.overflow = A.overflow;
    if (T.overflow & (1ull << 6)) T.dp_cost = ~0ull;          // saturate (flagged)
    if (T.overflow & (1ull << 10)) T.makespan_us = ~0ull;
    T.latency_sum_lo = A.lat_lo;
    T.latency_sum_hi = A.lat_hi;
    finish_totals(T);
    *S.totals = T;
}

cudaError_t run_stats(const StatsParams &S, cudaStream_t st)
{
    cudaError_t e;
    if ((e = cudaMemsetAsync(S.acc, 0, sizeof(StatAcc), st))) return e;
    if (S.n > 0) {
        const unsigned wblocks = 148 * 8;
        uint64_t sb = ceil_div(S.n_cap, kScanBlock);
        const unsigned sblocks = (unsigned)(sb < 296 ? sb : 296);
        k_stats_est<<<wblocks, 256, 0, st>>>(S);
        k_seg_scan_local<<<sblocks, kScanBlock, 0, st>>>(S);
        k_seg_scan_chunks<<<1, kScanBlock, 0, st>>>(S);
        k_seg_scan_apply<<<sblocks, kScanBlock, 0, st>>>(S);
        k_stats_final<<<wblocks, 256, 0, st>>>(S);
    }
    k_totals<<<1, 1, 0, st>>>(S);
    return cudaGetLastError();
}

}  // namespace uellm
