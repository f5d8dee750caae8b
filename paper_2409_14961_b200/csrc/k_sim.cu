// k_sim.cu -- NEXT f2: sequential execution of a schedule on one replica with query arrivals
// (PAPER.md P:499 metrics; R19).
//
//   start_t = max(end_{t-1}, A_t)   A_t = latest arrival among batch t's members
//   end_t   = start_t + est_t       est_t = t_batch + t_iter*O + t_tok*b*O + t_prefill*b*s (R7)
//   latency_k = end_{t(k)} - arrival_k,  violation iff latency_k > slo_us_k
//
// The recurrence end_t = max(end_{t-1} + est_t, A_t + est_t) is the max-plus affine map
// f_t(x) = max(x + a_t, b_t) with a_t = est_t, b_t = A_t + est_t applied to end_{t-1}.  Maps of
// this form compose associatively,
//     (g o f)(x) = max(x + f.a + g.a, max(f.b + g.a, g.b)),
// so every end_t is an inclusive scan of maps applied to end_{-1} = 0, i.e. the b component of
// the prefix composition (b >= a holds for every map and is preserved by composition).  Times
// saturate at 2^63 (sat(x + y) and max commute with min(., 2^63) on non-negative values, so the
// saturated scan equals min(true value, 2^63) exactly); ends are nondecreasing in t, so the
// timeline overflowed iff the last end reached 2^63.
//
//   k_sim_gather   position-linear: arrival in scheduled order, arr_s[k] = arrival[order[k]]
//                  (the random gather stays inside the window the resident CTAs work on, so it
//                  is served from L2; everything after it streams coalesced)
//   k_sim_batches  chunks of kScanBlock batches per CTA: groups of 8 lanes stream each batch's
//                  members (s, O, A_t, est_t), then thread = batch for the CTA-wide inclusive
//                  scan of the maps; chunk aggregates
//   k_sim_chunks   one CTA: exclusive scan of the chunk aggregates -> end value entering chunk
//   k_sim_members  8 lanes per batch: end_t, member latencies (scheduled order, written straight
//                  to the caller's buffer when requested) / violations, block-aggregated totals
//                  (exact 128-bit latency sum)
//   k_sim_totals   one thread: uellm_sim_totals
#include "internal.cuh"

namespace uellm {

namespace {

constexpr unsigned long long kTimeCap = 1ull << 63;

struct MaxPlus {
    unsigned long long a, b;       // f(x) = max(x + a, b)
};

__device__ __forceinline__ unsigned long long sat_add(unsigned long long x, unsigned long long y)
{
    // x, y <= 2^63: x + y can only wrap when one of them is already at the cap
    return (x >= kTimeCap || y >= kTimeCap || x + y >= kTimeCap) ? kTimeCap : x + y;
}

// f first, then g
__device__ __forceinline__ MaxPlus compose(MaxPlus f, MaxPlus g)
{
    MaxPlus r;
    r.a = sat_add(f.a, g.a);
    r.b = max(sat_add(f.b, g.a), g.b);
    return r;
}

// CTA-wide inclusive scan of maps (identity = (0, 0): every map has b >= a >= 0)
__device__ MaxPlus block_scan_maps(MaxPlus v, MaxPlus *agg)
{
    __shared__ unsigned long long sa[kScanBlock / 32], sb[kScanBlock / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int nw = kScanBlock / 32;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        MaxPlus o;
        o.a = __shfl_up_sync(0xffffffffu, v.a, d);
        o.b = __shfl_up_sync(0xffffffffu, v.b, d);
        if (lane >= d) v = compose(o, v);
    }
    if (lane == 31) { sa[warp] = v.a; sb[warp] = v.b; }
    __syncthreads();
    if (warp == 0) {
        MaxPlus w;
        w.a = lane < nw ? sa[lane] : 0ull;
        w.b = lane < nw ? sb[lane] : 0ull;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            MaxPlus o;
            o.a = __shfl_up_sync(0xffffffffu, w.a, d);
            o.b = __shfl_up_sync(0xffffffffu, w.b, d);
            if (lane >= d) w = compose(o, w);
        }
        if (lane < nw) { sa[lane] = w.a; sb[lane] = w.b; }
    }
    __syncthreads();
    if (warp > 0) {
        MaxPlus p;
        p.a = sa[warp - 1];
        p.b = sb[warp - 1];
        v = compose(p, v);
    }
    agg->a = sa[nw - 1];
    agg->b = sb[nw - 1];
    __syncthreads();
    return v;
}

__device__ __forceinline__ unsigned long long warp_sum64(unsigned long long v)
{
#pragma unroll
    for (int d = 16; d; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    return v;
}

}  // namespace

__global__ void __launch_bounds__(256) k_sim_gather(SimParams S)
{
    const uint64_t nt = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < S.n; k += nt)
        S.arr_s[k] = __ldg(S.arrival + __ldg(S.order + k));
}

#ifndef UELLM_GROUP_LANES
#define UELLM_GROUP_LANES 8
#endif
constexpr uint32_t kSimGroup = UELLM_GROUP_LANES;   // lanes per batch in the member-streaming loops

__global__ void __launch_bounds__(kScanBlock) k_sim_batches(SimParams S)
{
    // phase 1: groups of kSimGroup lanes stream each batch's members (consecutive lanes on
    // consecutive positions); phase 2: thread = batch, CTA-wide scan of the maps
    __shared__ unsigned long long s_est[kScanBlock], s_A[kScanBlock];
    const uint64_t m = *S.num_batches;
    const uint64_t nch = ceil_div(m, kScanBlock);
    const uint32_t sub = threadIdx.x % kSimGroup;
    unsigned long long busy = 0, gen = 0;
    for (uint64_t c = blockIdx.x; c < nch; c += gridDim.x) {
        for (uint32_t loc = threadIdx.x / kSimGroup; loc < kScanBlock; loc += blockDim.x / kSimGroup) {
            const uint64_t t = c * kScanBlock + loc;
            const bool act = t < m;
            uint32_t s = 0, O = 0, a = 0, z = 0;
            unsigned long long A = 0;
            if (act) {
                a = S.offsets[t];
                z = S.offsets[t + 1];
                for (uint32_t k = a + sub; k < z; k += kSimGroup) {
                    s = max(s, __ldg(S.rin + k));
                    O = max(O, __ldg(S.rout + k));
                    A = max(A, __ldg(S.arr_s + k));
                }
            }
#pragma unroll
            for (int d = kSimGroup / 2; d; d >>= 1) {
                s = max(s, __shfl_xor_sync(0xffffffffu, s, d));
                O = max(O, __shfl_xor_sync(0xffffffffu, O, d));
                A = max(A, __shfl_xor_sync(0xffffffffu, A, d));
            }
            if (act && sub == 0) {
                const unsigned long long b = z - a;
                const unsigned long long est = S.t_batch + S.t_iter * O + S.t_tok * b * O + S.t_pre * b * s;
                S.est[t] = est;
                s_est[loc] = est;
                s_A[loc] = A;
                busy += est;
                gen += b * O;
            }
        }
        __syncthreads();
        const uint64_t t = c * kScanBlock + threadIdx.x;
        MaxPlus f = {0ull, 0ull};
        if (t < m) {
            f.a = s_est[threadIdx.x];
            f.b = sat_add(s_A[threadIdx.x], f.a);
        }
        MaxPlus agg;
        const MaxPlus inc = block_scan_maps(f, &agg);        // ends with a barrier: smem reusable
        if (t < m) { S.inc_a[t] = inc.a; S.inc_b[t] = inc.b; }
        if (threadIdx.x == 0) { S.chunk_a[c] = agg.a; S.chunk_b[c] = agg.b; }
    }
    busy = warp_sum64(busy);
    gen = warp_sum64(gen);
    if ((threadIdx.x & 31) == 0 && (busy | gen)) {
        atomicAdd(&S.acc->busy, busy);
        atomicAdd(&S.acc->gen, gen);
    }
}

// end value entering every chunk: exclusive scan of the chunk maps applied to end_{-1} = 0
__global__ void __launch_bounds__(kScanBlock) k_sim_chunks(SimParams S)
{
    const uint64_t m = *S.num_batches;
    const uint64_t nch = ceil_div(m, kScanBlock);
    const uint64_t per = ceil_div(nch, kScanBlock);
    const uint64_t a = threadIdx.x * per, z = min(a + per, nch);
    MaxPlus f = {0ull, 0ull};
    for (uint64_t c = a; c < z; ++c) {
        MaxPlus g;
        g.a = S.chunk_a[c];
        g.b = S.chunk_b[c];
        f = compose(f, g);
    }
    MaxPlus agg;
    const MaxPlus inc = block_scan_maps(f, &agg);
    __shared__ unsigned long long ia[kScanBlock], ib[kScanBlock];
    ia[threadIdx.x] = inc.a;
    ib[threadIdx.x] = inc.b;
    __syncthreads();
    MaxPlus carry = {0ull, 0ull};
    if (threadIdx.x) { carry.a = ia[threadIdx.x - 1]; carry.b = ib[threadIdx.x - 1]; }
    for (uint64_t c = a; c < z; ++c) {
        MaxPlus g;
        g.a = S.chunk_a[c];
        g.b = S.chunk_b[c];
        S.carry[c] = carry.b;          // end_{t-1} for the chunk's first batch
        carry = compose(carry, g);
    }
}

__global__ void __launch_bounds__(256) k_sim_members(SimParams S)
{
    __shared__ unsigned long long red[8][5];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, sub = lane % kSimGroup;
    const uint64_t m = *S.num_batches;
    const uint64_t ng = (uint64_t)gridDim.x * (blockDim.x / kSimGroup);
    const uint64_t mpad = ceil_div(m, 32 / kSimGroup) * (32 / kSimGroup);   // whole warps iterate together
    unsigned long long viol = 0, lmax = 0, llo = 0, lhi = 0, any = 0;
    for (uint64_t t = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) / kSimGroup; t < mpad; t += ng) {
        if (t >= m) continue;
        const unsigned long long e_in = S.carry[t / kScanBlock];
        const unsigned long long end = max(sat_add(e_in, S.inc_a[t]), S.inc_b[t]);
        if (sub == 0) {
            if (S.batch_end) S.batch_end[t] = end;
            if (t == m - 1) S.acc->makespan = end;
        }
        const uint32_t a = S.offsets[t], z = S.offsets[t + 1];
        for (uint32_t k = a + sub; k < z; k += kSimGroup) {
            const unsigned long long arr = __ldg(S.arr_s + k);
            const unsigned long long lat = end > arr ? end - arr : 0ull;
            viol += lat > (unsigned long long)__ldg(S.rslo + k);
            lmax = max(lmax, lat);
            llo += lat;
            lhi += llo < lat ? 1ull : 0ull;
            if (S.latency) S.latency[k] = lat;
        }
        any = 1;
    }
#pragma unroll
    for (int d = 16; d; d >>= 1) {
        viol += __shfl_xor_sync(0xffffffffu, viol, d);
        lmax = max(lmax, __shfl_xor_sync(0xffffffffu, lmax, d));
        any |= __shfl_xor_sync(0xffffffffu, any, d);
        const unsigned long long lo2 = __shfl_xor_sync(0xffffffffu, llo, d), hi2 = __shfl_xor_sync(0xffffffffu, lhi, d);
        const unsigned long long lo = llo + lo2;
        lhi += hi2 + (lo < llo ? 1ull : 0ull);
        llo = lo;
    }
    if (lane == 0) {
        red[warp][0] = viol; red[warp][1] = lmax; red[warp][2] = llo; red[warp][3] = lhi; red[warp][4] = any;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long v = 0, mx = 0, lo = 0, hi = 0, an = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            v += red[w][0];
            mx = max(mx, red[w][1]);
            lo += red[w][2];
            hi += red[w][3] + (lo < red[w][2] ? 1ull : 0ull);
            an |= red[w][4];
        }
        if (!an) return;
        SimAcc *A = S.acc;
        atomicAdd(&A->viol, v);
        atomicMax(&A->lat_max, mx);
        const unsigned long long old = atomicAdd(&A->lat_lo, lo);
        atomicAdd(&A->lat_hi, hi + (old + lo < old ? 1ull : 0ull));
    }
}

__global__ void k_sim_totals(SimParams S)
{
    const SimAcc &A = *S.acc;
    uellm_sim_totals T;
    T.n = S.n;
    T.batches = S.n ? *S.num_batches : 0ull;
    T.makespan_us = A.makespan;
    T.busy_us = A.busy;
    T.idle_us = A.makespan - A.busy;
    T.gen_tokens = A.gen;
    T.viol = A.viol;
    T.latency_max_us = A.lat_max;
    T.latency_sum_lo = A.lat_lo;
    T.latency_sum_hi = A.lat_hi;
    const double lat = (double)A.lat_hi * 18446744073709551616.0 + (double)A.lat_lo;
    T.mean_latency_s = S.n ? lat / (double)S.n * 1e-6 : 0.0;
    T.slo_violation_rate = S.n ? (double)A.viol / (double)S.n : 0.0;
    T.utilization = A.makespan ? (double)A.busy / (double)A.makespan : 0.0;
    T.throughput_tok_s = A.makespan ? (double)A.gen / ((double)A.makespan * 1e-6) : 0.0;
    T.status = A.makespan >= kTimeCap ? (uint32_t)UELLM_ERR_OVERFLOW : (uint32_t)UELLM_OK;
    T.pad = 0;
    *S.totals = T;
}

cudaError_t run_simulate(const SimParams &S, cudaStream_t st, int *launches)
{
    cudaError_t e;
    if ((e = cudaMemsetAsync(S.acc, 0, sizeof(SimAcc), st))) return e;
    int l = 1;
    if (S.n > 0) {
        const uint64_t nch = ceil_div(S.n_cap, kScanBlock);
        const unsigned cblocks = (unsigned)(nch < 296 ? nch : 296);
        const uint64_t pb = ceil_div(S.n, 256);
        const unsigned pblocks = (unsigned)(pb < 148 * 16 ? pb : 148 * 16);
        k_sim_gather<<<pblocks, 256, 0, st>>>(S);
        k_sim_batches<<<cblocks, kScanBlock, 0, st>>>(S);
        k_sim_chunks<<<1, kScanBlock, 0, st>>>(S);
        k_sim_members<<<148 * 8, 256, 0, st>>>(S);
        l += 4;
    }
    k_sim_totals<<<1, 1, 0, st>>>(S);
    if (launches) *launches = l;
    return cudaGetLastError();
}

}  // namespace uellm
