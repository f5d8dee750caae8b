// k_exchange.cu -- a9: the multi-GPU exchange record and its combination (
// BASELINE.json north_star: "one NCCL allgather of batch boundaries and statistics").
//
// Windows are independent (R15: no batch crosses a window), so rank r schedules the contiguous
// window block [q_r, q_{r+1}) of the job alone.  Its exchange record is
//     [ uellm_totals (128 B) | boundary bitmap of local positions 0 .. n_r (u32 words) ]
// and after ONE allgather of the fixed-size records every rank rebuilds, on its GPU,
//   * the job's boundary bitmap: global position p < n belongs to the rank r with
//     q_r <= p < q_{r+1}; its bit is bit p - q_r of rank r's bitmap (bit n = the end);
//   * batch_offsets / num_batches by the same compaction as uellm_schedule_batches;
//   * the job totals: integer sums (kv max), exact 128-bit latency numerator.
#include "internal.cuh"

namespace uellm {

__global__ void k_xc_totals(const uint8_t *__restrict__ g, uint32_t world, uint64_t rec_bytes, uellm_totals *out)
{
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    uellm_totals T;
    uint64_t *t = &T.n;
    for (uint32_t k = 0; k < sizeof(uellm_totals) / 8; ++k) t[k] = 0;
    for (uint32_t r = 0; r < world; ++r)
        combine_totals_into(T, *reinterpret_cast<const uellm_totals *>(g + (uint64_t)r * rec_bytes));
    finish_totals(T);
    *out = T;
}

// One thread per global bitmap word.  The 32 positions of a word usually belong to one rank
// (rank ranges are whole windows): then the word is one funnel shift of two source words.
__global__ void __launch_bounds__(256) k_xc_bitmap(const uint8_t *__restrict__ g, uint32_t world, uint64_t rec_bytes,
                                                   const unsigned long long *__restrict__ qb, uint64_t n_total,
                                                   uint32_t *__restrict__ bm, uint64_t nwords)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nwords; w += stride) {
        const uint64_t p0 = 32 * w;
        const uint64_t end = min(p0 + 32, n_total + 1);
        uint32_t out = 0;
        uint64_t p = p0;
        while (p < end) {
            if (p == n_total) { out |= 1u << (uint32_t)(p - p0); break; }
            // owner: the largest r with q_r <= p (then q_{r+1} > p: ranks with empty ranges are
            // passed over because their q_r equals the next rank's)
            uint32_t lo = 0, hi = world - 1;
            while (lo < hi) {
                const uint32_t mid = (lo + hi + 1) / 2;
                if (qb[mid] <= p) lo = mid; else hi = mid - 1;
            }
            const uint32_t r = lo;
            const uint64_t local = p - qb[r];
            const uint64_t stop = min(end, (uint64_t)qb[r + 1]);
            const uint32_t cnt = (uint32_t)(stop - p);                    // 1 .. 32
            const uint32_t *words = reinterpret_cast<const uint32_t *>(g + (uint64_t)r * rec_bytes + sizeof(uellm_totals));
            const uint64_t wi = local >> 5;
            const uint32_t v = __funnelshift_r(words[wi], words[wi + 1], (uint32_t)(local & 31));
            const uint32_t mask = cnt >= 32 ? 0xffffffffu : ((1u << cnt) - 1u);
            out |= (v & mask) << (uint32_t)(p - p0);
            p = stop;
        }
        bm[w] = out;
    }
}

cudaError_t launch_totals_combine(const uint8_t *parts, uint32_t count, uint64_t stride, uellm_totals *out,
                                  cudaStream_t st)
{
    k_xc_totals<<<1, 32, 0, st>>>(parts, count, stride, out);
    return cudaGetLastError();
}

cudaError_t run_exchange_combine(const uint8_t *gathered, uint32_t world, uint64_t rec_bytes,
                                 const unsigned long long *d_qb, uint64_t n_total, uint32_t *bitmap, uint32_t *wscan,
                                 uint32_t *blocksum, uint32_t *offsets, unsigned long long *num_batches,
                                 uellm_totals *d_tot, cudaStream_t st)
{
    k_xc_totals<<<1, 32, 0, st>>>(gathered, world, rec_bytes, d_tot);
    const uint64_t nwords = (n_total + 1 + 31) / 32;
    uint64_t nb = ceil_div(nwords, 256);
    if (nb > 148ull * 8) nb = 148ull * 8;
    k_xc_bitmap<<<(unsigned)nb, 256, 0, st>>>(gathered, world, rec_bytes, d_qb, n_total, bitmap, nwords);
    cudaError_t e = cudaGetLastError();
    if (e) return e;
    return run_compact(bitmap, n_total, wscan, blocksum, offsets, num_batches, st);
}

}  // namespace uellm
