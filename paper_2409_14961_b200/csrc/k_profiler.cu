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

// the variant's prediction before the inflation factor (R20); VAR >= 0 fixes the
// variant at compile time (the level-path kernels are instantiated per variant), -1 reads P.variant
template <int VAR = -1>
__device__ __forceinline__ unsigned long long base_of(const PredictParams &P, unsigned long long index, uint32_t t)
{
    const uint32_t var = VAR >= 0 ? (uint32_t)VAR : P.variant;
    if (var == UELLM_PREDICT_ORACLE) return t;
    if (var == UELLM_PREDICT_CONSTANT) return P.constant_tokens;
    const uint32_t w = P.bucket_width;
    // ceil(t / w) in 32-bit arithmetic (power-of-two widths by a shift: the 16-token buckets)
    const uint32_t q = (w & (w - 1)) == 0 ? t >> (__ffs(w) - 1) : t / w;
    unsigned long long k = q + (q * w != t ? 1u : 0u);
    k = k < 1 ? 1 : k;
    if (var == UELLM_PREDICT_NOISY) {
        const unsigned long long z = mix64(P.seed, index);
        if ((z >> 11) < P.err_thresh) {                     // u = (z >> 11) * 2^-53 < error_rate
            if (z & 1ull) k += 1;
            else if (k > 1) k -= 1;
        }
    }
    return k * (unsigned long long)w;
}

// "multiplied by monitor.inflation_factor and rounded up", saturating (R20)
__device__ __forceinline__ uint32_t inflate(unsigned long long base, double factor)
{
    const double b = base <= 0xffffffffull ? (double)(uint32_t)base : (double)base;   // (exact either way)
    const double x = ceil(__dmul_rn(b, factor));
    return x >= 4294967295.0 ? 4294967295u : (uint32_t)x;
}

template <int VAR = -1>
__device__ __forceinline__ uint32_t predict_one(const PredictParams &P, unsigned long long index, uint32_t t,
                                                double factor)
{
    return inflate(base_of<VAR>(P, index, t), factor);
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

// Per query, the levels at which it is under-predicted form a PREFIX of the chain (the factors
// ascend and ceil(RN(base * v)) is monotone in v), and a base >= the true length is never under-
// predicted (every factor >= 1): the common warp has no work beyond the draw.  Four consecutive
// queries per thread (one 16-byte load when aligned); window indices from one division.
template <int VAR>
__global__ void __launch_bounds__(256) k_pred_count(PredictParams P, uint64_t n, uint64_t window)
{
    __shared__ double V[kPredMaxLevels];
    const uint32_t K = *P.nlevels;
    if (threadIdx.x <= K) V[threadIdx.x] = P.levels[threadIdx.x];
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nq = ceil_div(n, 4);
    const uint64_t nt = (uint64_t)gridDim.x * blockDim.x;
    const bool vec = ((uintptr_t)P.true_len & 15u) == 0;
    for (uint64_t g0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x - lane; g0 < nq; g0 += nt) {
        const uint64_t g = g0 + lane;
        const uint64_t k0 = 4 * g;
        uint32_t t[4] = {0, 0, 0, 0};
        if (g < nq) {
            if (vec && k0 + 4 <= n) {
                const uint4 v = __ldg(reinterpret_cast<const uint4 *>(P.true_len) + g);
                t[0] = v.x; t[1] = v.y; t[2] = v.z; t[3] = v.w;
            } else {
                for (int i = 0; i < 4; ++i) t[i] = k0 + i < n ? __ldg(P.true_len + k0 + i) : 0u;
            }
        }
        unsigned long long base[4];
        bool any = false;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            base[i] = k0 + i < n ? base_of<VAR>(P, k0 + i, t[i]) : ~0ull;
            any |= base[i] < t[i];
        }
        if (!__any_sync(0xffffffffu, any)) continue;            // warp-uniform: nothing under-predicted
        const uint32_t w0 = g < nq ? (uint32_t)k0 / (uint32_t)window : 0u;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            uint32_t c = 0;                                     // levels under-predicted: 0 .. K+1
            if (base[i] < t[i])
                while (c <= K && t[i] > inflate(base[i], V[c])) ++c;
            const uint32_t w = (k0 + i) < n ? w0 + ((uint32_t)(k0 + i) >= (w0 + 1) * (uint32_t)window ? 1u : 0u)
                                            : 0xffffffffu;
            if (c && w != 0xffffffffu)
                for (uint32_t l = 0; l < c; ++l) atomicAdd(P.hist + (uint64_t)w * kPredMaxLevels + l, 1ull);
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

template <int VAR>
__global__ void __launch_bounds__(256) k_pred_write(PredictParams P, uint64_t n, uint64_t window)
{
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nq = ceil_div(n, 4);
    const uint64_t nt = (uint64_t)gridDim.x * blockDim.x;
    const bool vec = (((uintptr_t)P.true_len | (uintptr_t)P.pred) & 15u) == 0;
    for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < nq; g += nt) {
        const uint64_t k0 = 4 * g;
        uint32_t t[4] = {0, 0, 0, 0}, p[4];
        const bool full = vec && k0 + 4 <= n;
        if (full) {
            const uint4 v = __ldg(reinterpret_cast<const uint4 *>(P.true_len) + g);
            t[0] = v.x; t[1] = v.y; t[2] = v.z; t[3] = v.w;
        } else {
            for (int i = 0; i < 4; ++i) t[i] = k0 + i < n ? __ldg(P.true_len + k0 + i) : 0u;
        }
        const uint32_t w0 = (uint32_t)k0 / (uint32_t)window;
        const double f0 = P.levels[P.wlevel[w0]];
        const uint32_t wend = (w0 + 1) * (uint32_t)window;      // first query of the next window
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const double f = (k0 + i >= n || (uint32_t)(k0 + i) < wend) ? f0 : P.levels[P.wlevel[w0 + 1]];
            p[i] = predict_one<VAR>(P, k0 + i, t[i], f);
        }
        if (full) {
            reinterpret_cast<uint4 *>(P.pred)[g] = make_uint4(p[0], p[1], p[2], p[3]);
        } else {
            for (int i = 0; i < 4; ++i) if (k0 + i < n) P.pred[k0 + i] = p[i];
        }
    }
    (void)lane;
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
        const uint64_t nb = ceil_div(n, 256 * 4 * 4);
        const unsigned blocks = (unsigned)(nb < 148 * 8 ? nb : 148 * 8);
        switch (P.variant) {
        case UELLM_PREDICT_ORACLE: k_pred_count<UELLM_PREDICT_ORACLE><<<blocks, 256, 0, st>>>(P, n, window); break;
        case UELLM_PREDICT_BUCKETED: k_pred_count<UELLM_PREDICT_BUCKETED><<<blocks, 256, 0, st>>>(P, n, window); break;
        case UELLM_PREDICT_NOISY: k_pred_count<UELLM_PREDICT_NOISY><<<blocks, 256, 0, st>>>(P, n, window); break;
        default: k_pred_count<UELLM_PREDICT_CONSTANT><<<blocks, 256, 0, st>>>(P, n, window); break;
        }
        k_pred_chain<<<1, 32, 0, st>>>(P, nwin);
        switch (P.variant) {
        case UELLM_PREDICT_ORACLE: k_pred_write<UELLM_PREDICT_ORACLE><<<blocks, 256, 0, st>>>(P, n, window); break;
        case UELLM_PREDICT_BUCKETED: k_pred_write<UELLM_PREDICT_BUCKETED><<<blocks, 256, 0, st>>>(P, n, window); break;
        case UELLM_PREDICT_NOISY: k_pred_write<UELLM_PREDICT_NOISY><<<blocks, 256, 0, st>>>(P, n, window); break;
        default: k_pred_write<UELLM_PREDICT_CONSTANT><<<blocks, 256, 0, st>>>(P, n, window); break;
        }
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
