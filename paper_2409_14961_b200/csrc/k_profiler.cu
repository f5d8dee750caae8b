// k_profiler.cu -- NEXT f4: profiler stand-ins and the misprediction monitor (PAPER.md P:73,
// P:195; R20).  The step before the scheduling path: predicted output
// lengths for a stream of queries, one monitor epoch per window.
//
//   variant oracle      pred = true length
//           bucketed(w) pred = max(1, ceil(true / w)) * w
//           noisy(e, w) the bucketed value moved one bucket up or down with probability e
//                       (counter-based draw per caller index; never below the first bucket)
//           constant(v) pred = v
//   then pred = min(ceil(pred * factor), 2^32 - 1) ("multiplied by the inflation factor
//   and rounded up").  Monitor: every under-prediction (true > pred) counts one
//   correction and factor <- min(factor * gamma, cap).
//
// Two schedules of the same computation:
//  * level path (a workspace is given, <= kPredMaxLevels factor levels, <= kPredMaxWindows
//    windows): the factor only ever moves along the chain v_0 = factor, v_{i+1} = min(v_i*gamma,
//    cap) (one step per correction), so every window's under-prediction count is computed for
//    EVERY level at once (k_pred_count, one position-linear pass over all windows), a single
//    thread walks the windows through the chain (k_pred_chain: level l_{w+1} = min(l_w + c_w(l_w),
//    K)), and k_pred_write writes each window's predictions with its level's factor -- 4 launches
//    in total instead of one per window;
//  * window path: k_predict_window, one launch per window: predictions with the factor in
//    force, under-prediction count reduced per CTA; the last CTA to finish (threadfence +
//    arrival counter) applies the monitor update and publishes the next window's factor.
#include "internal.cuh"

namespace uellm {

namespace {

// counter-based draw (splitmix64 finaliser of seed ^ index * golden gamma)
__device__ __forceinline__ unsigned long long mix64(unsigned long long seed, unsigned long long index)
{
    unsigned long long z = seed ^ (index * 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// the variant's prediction before the inflation factor (R20)
__device__ __forceinline__ unsigned long long base_of(const PredictParams &P, unsigned long long index, uint32_t t)
{
    if (P.variant == UELLM_PREDICT_ORACLE) return t;
    if (P.variant == UELLM_PREDICT_CONSTANT) return P.constant_tokens;
    const uint32_t w = P.bucket_width;
    const uint32_t q = t / w;                                 // ceil(t / w) in 32-bit arithmetic
    unsigned long long k = q + (q * w != t ? 1u : 0u);
    k = k < 1 ? 1 : k;
    if (P.variant == UELLM_PREDICT_NOISY) {
        const unsigned long long z = mix64(P.seed, index);
        const double u = (double)(z >> 11) * 0x1.0p-53;
        if (u < P.error_rate) {
            if (z & 1ull) k += 1;
            else if (k > 1) k -= 1;
        }
    }
    return k * (unsigned long long)w;
}

// "multiplied by monitor.inflation_factor and rounded up", saturating (R20)
__device__ __forceinline__ uint32_t inflate(unsigned long long base, double factor)
{
    const double x = ceil(__dmul_rn((double)base, factor));
    return x >= 4294967295.0 ? 4294967295u : (uint32_t)x;
}

__device__ __forceinline__ uint32_t predict_one(const PredictParams &P, unsigned long long index, uint32_t t,
                                                double factor)
{
    return inflate(base_of(P, index, t), factor);
}

}  // namespace

__global__ void __launch_bounds__(256) k_predict_window(PredictParams P, uint64_t a, uint64_t z, uint64_t w)
{
    __shared__ unsigned long long red[8];
    __shared__ bool last;
    uellm_monitor_state *M = P.state;
    unsigned long long *cnt = reinterpret_cast<unsigned long long *>(M->scratch);   // [0] under, [1] CTAs done
    const double f = M->inflation_factor;       // read before this CTA's arrival below
    unsigned long long under = 0;
    const uint64_t nt = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = a + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < z; k += nt) {
        const uint32_t t = __ldg(P.true_len + k);
        const uint32_t p = predict_one(P, k, t, f);
        P.pred[k] = p;
        under += t > p;
    }
#pragma unroll
    for (int d = 16; d; d >>= 1) under += __shfl_xor_sync(0xffffffffu, under, d);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = under;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long c = 0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) c += red[i];
        if (c) atomicAdd(&cnt[0], c);
        __threadfence();
        last = atomicAdd(&cnt[1], 1ull) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last || threadIdx.x != 0) return;
    __threadfence();
    const unsigned long long k = atomicAdd(&cnt[0], 0ull);   // every CTA's count is in
    double g = f;
    if (P.monitor) {
        for (unsigned long long i = 0; i < k; ++i) {     // S:216, one observation at a time
            const double h = __dmul_rn(g, P.gamma);
            const double n2 = h < P.cap ? h : P.cap;
            if (n2 == g) break;                          // fixpoint (cap reached or gamma == 1)
            g = n2;
        }
        M->corrections += k;
        M->inflation_factor = g;
    }
    if (P.factors) {
        P.factors[w] = f;
        if (w + 1 == P.nwin) P.factors[w + 1] = g;
    }
    cnt[0] = 0;
    cnt[1] = 0;
}

// ---- level path
__global__ void k_pred_levels(PredictParams P)
{
    if (threadIdx.x != 0) return;
    double v = P.state->inflation_factor;
    uint32_t K = 0;
    P.levels[0] = v;
    if (P.monitor) {
        while (K < kPredMaxLevels - 1) {
            const double h = __dmul_rn(v, P.gamma);
            const double nv = h < P.cap ? h : P.cap;
            if (nv == v) break;                 // fixpoint: cap reached (or gamma == 1)
            v = nv;
            P.levels[++K] = v;
        }
    }
    *P.nlevels = K;
}

__global__ void __launch_bounds__(256) k_pred_count(PredictParams P, uint64_t n, uint64_t window)
{
    __shared__ double V[kPredMaxLevels];
    const uint32_t K = *P.nlevels;
    if (threadIdx.x <= K) V[threadIdx.x] = P.levels[threadIdx.x];
    __syncthreads();
    const uint64_t nt = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t n_pad = ceil_div(n, 32) * 32;             // whole warps stay in the loop
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n_pad; k += nt) {
        uint32_t under = 0;
        uint32_t w = 0xffffffffu;
        if (k < n) {
            const uint32_t t = __ldg(P.true_len + k);
            w = (uint32_t)k / (uint32_t)window;             // 32-bit: n < 2^32 (a 64-bit divide is ~10x)
            const unsigned long long base = base_of(P, k, t);
            // every level factor is >= 1, so inflate(base, v) >= base: only a base below the true
            // length can be an under-prediction at some level (the noisy variant's downward moves,
            // a small constant) -- the common case needs no double arithmetic
            if (base < t)
                for (uint32_t i = 0; i <= K; ++i) under |= (uint32_t)(t > inflate(base, V[i])) << i;
        }
        const uint32_t grp = __match_any_sync(0xffffffffu, w);
        const uint32_t lane = threadIdx.x & 31;
        const bool leader = (__ffs(grp) - 1) == (int)lane;
        for (uint32_t i = 0; i <= K; ++i) {
            const uint32_t b = __ballot_sync(0xffffffffu, (under >> i) & 1u) & grp;
            if (leader && b && w != 0xffffffffu)
                atomicAdd(P.hist + (uint64_t)w * kPredMaxLevels + i, (unsigned long long)__popc(b));
        }
    }
}

__global__ void k_pred_chain(PredictParams P, uint64_t nwin)
{
    if (threadIdx.x != 0) return;
    const uint32_t K = *P.nlevels;
    uint32_t l = 0;
    unsigned long long corr = 0;
    for (uint64_t w = 0; w < nwin; ++w) {
        P.wlevel[w] = (uint8_t)l;
        if (P.factors) P.factors[w] = P.levels[l];
        const unsigned long long c = P.hist[w * kPredMaxLevels + l];
        corr += c;
        const unsigned long long nl = (unsigned long long)l + c;
        l = nl < K ? (uint32_t)nl : K;
    }
    if (P.factors) P.factors[nwin] = P.levels[l];
    if (P.monitor) {
        P.state->corrections += corr;
        P.state->inflation_factor = P.levels[l];
    }
}

__global__ void __launch_bounds__(256) k_pred_write(PredictParams P, uint64_t n, uint64_t window)
{
    const uint64_t nt = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += nt) {
        const uint32_t t = __ldg(P.true_len + k);
        P.pred[k] = predict_one(P, k, t, P.levels[P.wlevel[(uint32_t)k / (uint32_t)window]]);
    }
}

__global__ void k_predict_empty(PredictParams P)
{
    if (P.factors) P.factors[0] = P.state->inflation_factor;
}

cudaError_t run_predict(const PredictParams &P, uint64_t n, uint64_t window, cudaStream_t st, int *launches)
{
    int l = 0;
    if (n == 0) {
        k_predict_empty<<<1, 1, 0, st>>>(P);
        l = 1;
    } else if (P.levels) {
        const uint64_t nwin = ceil_div(n, window);
        cudaError_t e;
        if ((e = cudaMemsetAsync(P.hist, 0, 8 * kPredMaxLevels * nwin, st))) return e;
        k_pred_levels<<<1, 32, 0, st>>>(P);
        const uint64_t nb = ceil_div(n, 256 * 4);
        const unsigned blocks = (unsigned)(nb < 148 * 8 ? nb : 148 * 8);
        k_pred_count<<<blocks, 256, 0, st>>>(P, n, window);
        k_pred_chain<<<1, 32, 0, st>>>(P, nwin);
        k_pred_write<<<blocks, 256, 0, st>>>(P, n, window);
        l = 4;
    } else {
        for (uint64_t w = 0, a = 0; a < n; a += window, ++w) {
            const uint64_t z = a + window < n ? a + window : n;
            // (measured: 2 CTAs per SM, to shorten the same-address atomic tail, is slower --
            // 1.65 vs 1.03 ms per 10^8 -- the window is too small to hide latency with fewer CTAs)
            const uint64_t nb = ceil_div(z - a, 256 * 4);
            const unsigned blocks = (unsigned)(nb < 148 * 8 ? nb : 148 * 8);
            k_predict_window<<<blocks, 256, 0, st>>>(P, a, z, w);
            ++l;
        }
    }
    if (launches) *launches = l;
    return cudaGetLastError();
}

}  // namespace uellm
