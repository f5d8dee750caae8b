// k_load.cu -- a1/a2: validate profiled queries, SLO seconds -> integer us, key packing;
// decode of sorted keys into scheduled-order records; boundary marks of FIFO / sort-only.
//
// a1: reject input_len == 0, pred_out_len == 0, non-finite or <= 0 SLO and
//     slo_us outside [1, 2^32-1]; slo_us = rint(double(slo_s) * 1e6), half-even
//     (R12; the paper's SLOs are seconds).
// a2: key = slo_us << 32 | pred_out_len, payload = arrival index.  Ascending key order is
//     (SLO, predicted length) order (P:228 + R11); a stable sort keeps arrival order on ties
//     (R9).  Digits that are constant across all keys are skipped by the sort (OR/AND masks).
#include "internal.cuh"

namespace uellm {

__global__ void __launch_bounds__(256) k_load(const uint32_t *__restrict__ in,
                                              const uint32_t *__restrict__ out,
                                              const float *__restrict__ slo, uint64_t n,
                                              unsigned long long *__restrict__ keys,
                                              uint32_t *__restrict__ vals, LoadMeta *meta)
{
    uint32_t bad = 0, mx_in = 0, mx_out = 0, mx_slo = 0;
    unsigned long long kor = 0, kand = ~0ull;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) {
        uint32_t a = __ldg(in + k), o = __ldg(out + k);
        float sf = __ldg(slo + k);
        double x = (double)sf;
        uint32_t su = 0;
        if (a == 0) bad |= 1u;
        if (o == 0) bad |= 2u;
        if (!(x > 0.0) || !isfinite(x)) {
            bad |= 4u;
        } else {
            double r = rint(__dmul_rn(x, 1e6));      // one correctly rounded product, half-even
            if (r < 1.0 || r > 4294967295.0) bad |= 4u; else su = (uint32_t)r;
        }
        unsigned long long key = ((unsigned long long)su << 32) | o;
        keys[k] = key;
        vals[k] = (uint32_t)k;
        mx_in = max(mx_in, a); mx_out = max(mx_out, o); mx_slo = max(mx_slo, su);
        kor |= key; kand &= key;
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
}

cudaError_t launch_load(const uint32_t *in, const uint32_t *out, const float *slo, uint64_t n,
                        unsigned long long *keys, uint32_t *vals, LoadMeta *meta, cudaStream_t st)
{
    if (n == 0) return cudaSuccess;
    uint64_t blocks = ceil_div(n, 256ull * 8);      // ~8 queries per thread
    if (blocks > 148ull * 16) blocks = 148ull * 16;
    if (blocks < 1) blocks = 1;
    k_load<<<(unsigned)blocks, 256, 0, st>>>(in, out, slo, n, keys, vals, meta);
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
