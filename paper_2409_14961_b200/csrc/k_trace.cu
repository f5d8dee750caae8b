// k_trace.cu -- a7: traceback of the SEG-DP argmins into a boundary bitmap, compaction of the
// bitmap into batch_offsets (P:245 / P:286-290: "ready list" of batches in scan order), and the
// Alg. 1 (SLO-ODBS) segmentation.
//
// Bit b of the bitmap = "a batch starts at scheduled position b"; bit n closes the last batch.
// Traceback: the path from a window end w1 is w1 -> arg[w1] -> ... -> w0.  Tile-parallel:
//   T1  every tile walks from its own last boundary e (assumed on the path), marks its nodes
//       and records where the walk leaves the tile (exitA);
//   T2  every tile re-walks from the true entry candidate (the next tile's exitA) until the
//       walk meets a marked node (paths coalesce) and clears the nodes that are not on it;
//   T3  per window, tiles whose entry turned out different are re-walked in full (rare).
#include "internal.cuh"

namespace uellm {

__device__ __forceinline__ void bm_set(uint32_t *bm, uint32_t b) { atomicOr(bm + (b >> 5), 1u << (b & 31)); }
__device__ __forceinline__ bool bm_test(uint32_t *bm, uint32_t b) { return (__ldcg(bm + (b >> 5)) >> (b & 31)) & 1u; }
// clear bits [a, z] (inclusive); no-op if a > z
__device__ void bm_clear(uint32_t *bm, uint32_t a, uint32_t z)
{
    if (a > z) return;
    const uint32_t wa = a >> 5, wz = z >> 5;
    for (uint32_t w = wa; w <= wz; ++w) {
        const uint32_t lo = (w == wa) ? (a & 31) : 0;
        const uint32_t hi = (w == wz) ? (z & 31) : 31;
        const uint32_t m = (hi == 31 ? 0xffffffffu : ((1u << (hi + 1)) - 1)) & ~((1u << lo) - 1);
        atomicAnd(bm + w, ~m);
    }
}

__device__ __forceinline__ uint32_t arg_of(const uint16_t *argx, uint32_t j) { return j - (uint32_t)argx[j - 1]; }

__global__ void k_trace_a(const uint16_t *__restrict__ argx, TileRec *tiles, uint64_t ntiles, uint32_t *bm)
{
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ntiles) return;
    const TileRec r = tiles[t];
    if (!r.valid) return;
    uint32_t j = r.e, i;
    bm_set(bm, j);
    for (;;) {
        i = arg_of(argx, j);
        if (i <= r.s) break;
        bm_set(bm, i);
        j = i;
    }
    tiles[t].exitA = i;
}

// Walk A with the tile's args staged in shared memory (one CTA per tile): the pointer chase
// then costs a shared-memory latency per hop instead of a DRAM one.
__global__ void __launch_bounds__(1024) k_trace_a_smem(const uint16_t *__restrict__ argx, TileRec *tiles, uint32_t *bm)
{
    extern __shared__ uint16_t sa[];
    const uint64_t t = blockIdx.x;
    const TileRec r = tiles[t];
    if (!r.valid) return;
    const uint32_t len = r.e - r.s;              // sa[k] = delta of boundary s+1+k
    for (uint32_t k = threadIdx.x; k < len; k += blockDim.x) sa[k] = argx[r.s + k];
    __syncthreads();
    if (threadIdx.x != 0) return;
    uint32_t j = r.e, i;
    bm_set(bm, j);
    for (;;) {
        i = j - (uint32_t)sa[j - 1 - r.s];
        if (i <= r.s) break;
        bm_set(bm, i);
        j = i;
    }
    tiles[t].exitA = i;
}

// Walk A, one warp per tile (kTraceWarps tiles per CTA): the warp stages the tile's args in shared
// memory (16-byte loads when aligned), lane 0 walks them and sets the path's bits in a shared copy
// of the tile's bitmap words, and the warp ORs the words into the global bitmap -- neither the walk's
// hops nor its bit sets wait on global memory (the thread walk's hops each waited for a DRAM read).
constexpr uint32_t kTraceWarps = 4;
__host__ __device__ constexpr uint32_t trace_warp_smem(uint32_t tile_len)
{
    return ((tile_len * 2 + 15) & ~15u) + (((tile_len / 32 + 3) * 4 + 15) & ~15u);   // 16-byte aligned per warp
}
__global__ void __launch_bounds__(32 * kTraceWarps) k_trace_a_warp(const uint16_t *__restrict__ argx, TileRec *tiles,
                                                                   uint64_t ntiles, uint32_t *bm, uint32_t tile_len)
{
    extern __shared__ __align__(16) unsigned char tsm[];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t t = (uint64_t)blockIdx.x * kTraceWarps + warp;
    if (t >= ntiles) return;
    const TileRec r = tiles[t];
    if (!r.valid) return;
    unsigned char *base = tsm + (size_t)warp * trace_warp_smem(tile_len);
    uint16_t *sa = reinterpret_cast<uint16_t *>(base);
    uint32_t *sw = reinterpret_cast<uint32_t *>(base + ((tile_len * 2 + 15) & ~15u));
    const uint32_t len = r.e - r.s;                               // sa[k] = delta of boundary s+1+k
    if ((r.s & 7u) == 0 && (len & 7u) == 0) {
        const uint4 *src = reinterpret_cast<const uint4 *>(argx + r.s);
        uint4 *dst = reinterpret_cast<uint4 *>(sa);
        for (uint32_t k = lane; k < len / 8; k += 32) dst[k] = __ldg(src + k);
    } else {
        for (uint32_t k = lane; k < len; k += 32) sa[k] = argx[r.s + k];
    }
    // bitmap words w0 .. w1 cover the positions (s, e] the walk marks
    const uint32_t w0 = (r.s + 1) >> 5, w1 = r.e >> 5, nw = w1 - w0 + 1;
    for (uint32_t k = lane; k < nw; k += 32) sw[k] = 0u;
    __syncwarp();
    if (lane == 0) {
        uint32_t j = r.e, i;
        sw[(j >> 5) - w0] |= 1u << (j & 31);
        for (;;) {
            i = j - (uint32_t)sa[j - 1 - r.s];
            if (i <= r.s) break;
            sw[(i >> 5) - w0] |= 1u << (i & 31);
            j = i;
        }
        tiles[t].exitA = i;
    }
    __syncwarp();
    for (uint32_t k = lane; k < nw; k += 32) {
        const uint32_t v = sw[k];
        if (v) atomicOr(bm + w0 + k, v);
    }
}

__global__ void k_trace_b(const uint16_t *__restrict__ argx, TileRec *tiles, uint64_t ntiles, uint64_t tpw,
                          uint32_t *bm, Diag *diag, uint32_t *wflag)
{
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ntiles) return;
    const TileRec r = tiles[t];
    if (!r.valid) return;
    const bool last = ((t + 1) % tpw == 0) || !tiles[t + 1].valid;
    uint32_t exitB = r.exitA, merged = 1;
    if (!last) {
        const uint32_t q = tiles[t + 1].exitA;      // entry into this tile if tile t+1 is right
        if (q != r.e) {
            bm_clear(bm, q + 1, r.e);
            uint32_t j = q;
            for (;;) {
                if (bm_test(bm, j)) break;              // met the A-walk: identical below
                bm_set(bm, j);
                const uint32_t i = arg_of(argx, j);
                bm_clear(bm, max(i, r.s) + 1, j - 1);
                if (i <= r.s) { exitB = i; merged = (i == r.exitA); break; }
                j = i;
            }
            if (!merged) { atomicAdd(&diag->trace_unmerged, 1ull); wflag[t / tpw] = 1u; }
        }
    }
    tiles[t].exitB = exitB;
    tiles[t].merged = merged;
}

// Walk B, one warp per tile (as walk A): the tile's args and its bitmap words are staged in shared
// memory, lane 0 walks, clears and marks there, and the warp writes back only the changed bits of
// each word (atomicOr / atomicAnd: a neighbouring tile's walk owns the other bits of a shared word).
__device__ __forceinline__ void sbm_clear(uint32_t *sw, uint32_t w0, uint32_t a, uint32_t z)
{
    if (a > z) return;
    const uint32_t wa = a >> 5, wz = z >> 5;
    for (uint32_t w = wa; w <= wz; ++w) {
        const uint32_t lo = (w == wa) ? (a & 31) : 0;
        const uint32_t hi = (w == wz) ? (z & 31) : 31;
        const uint32_t m = (hi == 31 ? 0xffffffffu : ((1u << (hi + 1)) - 1)) & ~((1u << lo) - 1);
        sw[w - w0] &= ~m;
    }
}
__global__ void __launch_bounds__(32 * kTraceWarps) k_trace_b_warp(const uint16_t *__restrict__ argx, TileRec *tiles,
                                                                   uint64_t ntiles, uint64_t tpw, uint32_t *bm,
                                                                   Diag *diag, uint32_t *wflag, uint32_t tile_len)
{
    extern __shared__ __align__(16) unsigned char tsm[];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t t = (uint64_t)blockIdx.x * kTraceWarps + warp;
    if (t >= ntiles) return;
    const TileRec r = tiles[t];
    if (!r.valid) return;
    const bool last = ((t + 1) % tpw == 0) || !tiles[t + 1].valid;
    uint32_t exitB = r.exitA, merged = 1;
    const uint32_t q = last ? r.e : tiles[t + 1].exitA;          // entry into this tile if tile t+1 is right
    if (!last && q != r.e) {
        unsigned char *base = tsm + (size_t)warp * trace_warp_smem(tile_len);
        uint16_t *sa = reinterpret_cast<uint16_t *>(base);
        uint32_t *sw = reinterpret_cast<uint32_t *>(base + ((tile_len * 2 + 15) & ~15u));
        const uint32_t len = r.e - r.s;
        if ((r.s & 7u) == 0 && (len & 7u) == 0) {
            const uint4 *src = reinterpret_cast<const uint4 *>(argx + r.s);
            uint4 *dst = reinterpret_cast<uint4 *>(sa);
            for (uint32_t k = lane; k < len / 8; k += 32) dst[k] = __ldg(src + k);
        } else {
            for (uint32_t k = lane; k < len; k += 32) sa[k] = argx[r.s + k];
        }
        const uint32_t w0 = (r.s + 1) >> 5, w1 = r.e >> 5, nw = w1 - w0 + 1;
        for (uint32_t k = lane; k < nw; k += 32) sw[k] = __ldcg(bm + w0 + k);
        __syncwarp();
        uint32_t orig[9];                                          // lane's words before the walk (nw <= 258)
#pragma unroll
        for (int u = 0; u < 9; ++u) orig[u] = (lane + 32u * u < nw) ? sw[lane + 32u * u] : 0u;
        __syncwarp();
        if (lane == 0) {
            sbm_clear(sw, w0, q + 1, r.e);
            uint32_t j = q;
            for (;;) {
                if ((sw[(j >> 5) - w0] >> (j & 31)) & 1u) break;       // met the A-walk: identical below
                sw[(j >> 5) - w0] |= 1u << (j & 31);
                const uint32_t i = j - (uint32_t)sa[j - 1 - r.s];
                sbm_clear(sw, w0, max(i, r.s) + 1, j - 1);
                if (i <= r.s) { exitB = i; merged = (i == r.exitA); break; }
                j = i;
            }
            if (!merged) { atomicAdd(&diag->trace_unmerged, 1ull); wflag[t / tpw] = 1u; }
        }
        __syncwarp();
#pragma unroll
        for (int u = 0; u < 9; ++u) {
            const uint32_t k = lane + 32u * u;
            if (k < nw) {
                const uint32_t nv = sw[k], ov = orig[u];
                if (nv & ~ov) atomicOr(bm + w0 + k, nv & ~ov);
                if (ov & ~nv) atomicAnd(bm + w0 + k, ~(ov & ~nv));
            }
        }
        exitB = __shfl_sync(0xffffffffu, exitB, 0);
        merged = __shfl_sync(0xffffffffu, merged, 0);
    }
    if (lane == 0) {
        tiles[t].exitB = exitB;
        tiles[t].merged = merged;
    }
}

// Tile args staged in shared memory (up to kTraceStage positions; longer tiles read global memory).
constexpr uint32_t kTraceStage = 16384;
struct TileArgs {
    const uint16_t *g, *sm;
    uint32_t s;
    __device__ __forceinline__ uint32_t arg(uint32_t j) const
    {
        const uint32_t k = j - 1 - s;
        return j - (uint32_t)(sm && k < kTraceStage ? sm[k] : g[j - 1]);
    }
};
__device__ __forceinline__ TileArgs stage_args(const uint16_t *argx, const TileRec &r, uint16_t *sa)
{
    const uint32_t len = r.e - r.s;
    for (uint32_t k = threadIdx.x; k < len && k < kTraceStage; k += blockDim.x) sa[k] = argx[r.s + k];
    __syncthreads();
    return TileArgs{argx, sa, r.s};
}

// T2b (windows with an unmerged B-walk only): exit maps.  For every possible entry q into tile t
// -- q in [e - W + 1, e], where the walk from the next tile lands -- the first node <= s of the
// walk from q, stored as s - exit (< W).  One CTA per tile, one thread per entry.
__global__ void __launch_bounds__(256) k_trace_maps(const uint16_t *__restrict__ argx, const TileRec *tiles,
                                                    uint64_t ntiles, uint64_t tpw, const uint32_t *wflag, uint32_t W,
                                                    uint16_t *maps)
{
    extern __shared__ uint16_t sa[];
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        if (!wflag[t / tpw]) continue;
        const TileRec r = tiles[t];
        if (!r.valid) continue;
        const TileArgs A = stage_args(argx, r, sa);
        for (uint32_t qo = threadIdx.x; qo < W; qo += blockDim.x) {
            uint32_t j = r.e - qo, i = j;                // entry e - qo (a node <= s exits at once)
            while (i > r.s) { j = i; i = A.arg(j); }
            maps[t * W + qo] = (uint16_t)(r.s - i);
        }
        __syncthreads();
    }
}

// T3: one warp per window.  Counts the valid tiles (a prefix) and checks 32 tiles at a time whether
// every B-walk merged (exitB == exitA for tiles 1 .. K-1) -- then every tile's entry was right and
// nothing needs re-walking.  Otherwise lane 0 follows the true path through the tiles from the
// window end: a tile entered where its B-walk started keeps its marks and exit; any other tile
// takes its exit from the exit map and is queued for re-marking (k_trace_remark, in parallel).
__global__ void k_trace_c(const uint16_t *__restrict__ maps, TileRec *tiles, uint64_t tpw, uint64_t nwin,
                          uint64_t window, uint32_t W, uint32_t *bm, Diag *diag)
{
    const uint64_t w = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    if (w >= nwin) return;
    const uint64_t t0 = w * tpw;
    uint32_t K = 0;
    bool allm = true;
    for (uint32_t k0 = 0; k0 < tpw; k0 += 32) {
        const uint32_t k = k0 + lane;
        const bool v = k < tpw && tiles[t0 + k].valid;
        const uint32_t bv = __ballot_sync(0xffffffffu, v);
        K += __popc(bv);
        const bool bad = v && k >= 1 && tiles[t0 + k].exitB != tiles[t0 + k].exitA;
        if (__any_sync(0xffffffffu, bad)) allm = false;
        if (bv != 0xffffffffu) break;
    }
    if (K == 0 || lane != 0) return;
    bm_set(bm, (uint32_t)(w * window));                 // every window starts a batch
    if (allm) return;
    uint32_t exit_true = tiles[t0 + K - 1].exitB;
    uint32_t rewalks = 0;
    for (int k = (int)K - 2; k >= 0; --k) {
        const TileRec &r = tiles[t0 + k];
        if (exit_true == tiles[t0 + k + 1].exitA) {
            exit_true = r.exitB;
            continue;
        }
        ++rewalks;
        tiles[t0 + k].remark = exit_true + 1u;
        exit_true = r.s - (uint32_t)maps[(t0 + k) * W + (r.e - exit_true)];
        tiles[t0 + k].exitB = exit_true;
    }
    if (rewalks) atomicAdd(&diag->trace_rewalks, (unsigned long long)rewalks);
}

// k_trace_c with the walk's data staged (one 32-thread CTA per window, W <= kTraceCStageW): for 32
// tiles at a time the warp brings their exit maps (W u16 each, 16-byte loads) and the record fields
// the walk reads into shared memory, then lane 0 follows the true path through them -- one
// shared-memory hop per tile instead of a dependent global load (windows of one long uniform
// stretch re-walk every tile: c5's identical-key segment).
constexpr uint32_t kTraceCStageW = 384;
__device__ __forceinline__ uint32_t tr_smem(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void tr_mbar_init(uint64_t *bar)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(tr_smem(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void tr_mbar_wait(uint64_t *bar, uint32_t parity)
{
    asm volatile("{\n\t.reg .pred P1;\n"
                 "TRW_%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
                 "@!P1 bra TRW_%=;\n}" :: "r"(tr_smem(bar)), "r"(parity) : "memory");
}
// one TMA bulk copy global -> shared of `bytes` (a multiple of 16) completing on `bar`
__device__ __forceinline__ void tr_bulk(void *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(tr_smem(bar)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(tr_smem(dst)), "l"(src), "r"(bytes), "r"(tr_smem(bar)) : "memory");
}

// The maps of the chunk's (up to) 32 consecutive tiles are one contiguous range: one TMA bulk copy
// per chunk, double buffered (the next chunk's copy and record loads are in flight while lane 0
// walks the current one).  W % 8 == 0 (16-byte rows).
__global__ void __launch_bounds__(32) k_trace_c_staged(const uint16_t *__restrict__ maps, TileRec *tiles, uint64_t tpw,
                                                       uint64_t nwin, uint64_t window, uint32_t W, uint32_t *bm,
                                                       Diag *diag)
{
    extern __shared__ __align__(16) uint16_t smap[];             // [2][32][W]
    __shared__ uint32_t fs[2][32], fe[2][32], fa[2][33], fb[2][32];
    __shared__ __align__(8) uint64_t bar[2];
    const uint64_t w = blockIdx.x;
    const uint32_t lane = threadIdx.x;
    if (w >= nwin) return;
    const uint64_t t0 = w * tpw;
    uint32_t K = 0;
    bool allm = true;
    for (uint32_t k0 = 0; k0 < tpw; k0 += 32) {
        const uint32_t k = k0 + lane;
        const bool v = k < tpw && tiles[t0 + k].valid;
        const uint32_t bv = __ballot_sync(0xffffffffu, v);
        K += __popc(bv);
        const bool bad = v && k >= 1 && tiles[t0 + k].exitB != tiles[t0 + k].exitA;
        if (__any_sync(0xffffffffu, bad)) allm = false;
        if (bv != 0xffffffffu) break;
    }
    if (K == 0) return;
    if (lane == 0) bm_set(bm, (uint32_t)(w * window));          // every window starts a batch
    if (allm) return;
    if (lane == 0) { tr_mbar_init(&bar[0]); tr_mbar_init(&bar[1]); }
    __syncwarp();
    uint32_t exit_true = tiles[t0 + K - 1].exitB;                 // (uniform across the warp)
    uint32_t rewalks = 0;
    // chunk c covers tiles [k_lo, k_hi] with k_hi = K - 2 - 32 c
    uint32_t rs = 0, re = 0, ra = 0, rb = 0, rtop = 0;             // the next chunk's record fields
    auto issue = [&](int k_hi, int b) {
        const int k_lo = k_hi - 31 > 0 ? k_hi - 31 : 0;
        const int rows = k_hi - k_lo + 1;
        if (lane == 0)
            tr_bulk(smap + (size_t)b * 32 * W, maps + (t0 + (uint64_t)k_lo) * W, (uint32_t)rows * W * 2u, &bar[b]);
        if ((int)lane < rows) {
            const TileRec &r = tiles[t0 + k_lo + lane];
            rs = r.s; re = r.e; ra = r.exitA; rb = r.exitB;
        }
        if (lane == 0) rtop = tiles[t0 + k_hi + 1].exitA;
    };
    issue((int)K - 2, 0);
    uint32_t use[2] = {0u, 0u};
    int b = 0;
    for (int k_hi = (int)K - 2; k_hi >= 0; k_hi -= 32, b ^= 1) {
        const int k_lo = k_hi - 31 > 0 ? k_hi - 31 : 0;
        const int rows = k_hi - k_lo + 1;
        if ((int)lane < rows) { fs[b][lane] = rs; fe[b][lane] = re; fa[b][lane] = ra; fb[b][lane] = rb; }
        if (lane == 0) fa[b][rows] = rtop;
        if (k_hi - 32 >= 0) issue(k_hi - 32, b ^ 1);            // buffer b^1 was consumed last round
        tr_mbar_wait(&bar[b], use[b] & 1u);
        ++use[b];
        __syncwarp();
        if (lane == 0) {
            const uint16_t *sm = smap + (size_t)b * 32 * W;
            for (int k = k_hi; k >= k_lo; --k) {
                const int q = k - k_lo;
                if (exit_true == fa[b][q + 1]) { exit_true = fb[b][q]; continue; }
                ++rewalks;
                tiles[t0 + k].remark = exit_true + 1u;
                exit_true = fs[b][q] - (uint32_t)sm[(uint32_t)q * W + (fe[b][q] - exit_true)];
                tiles[t0 + k].exitB = exit_true;
            }
        }
        exit_true = __shfl_sync(0xffffffffu, exit_true, 0);
        // this buffer's generic reads precede the next bulk copy into it (async proxy)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
    }
    if (lane == 0 && rewalks) atomicAdd(&diag->trace_rewalks, (unsigned long long)rewalks);
}

// T4: tiles entered elsewhere than their B-walk assumed are re-marked from the true entry (one CTA
// per tile, the walk over the staged args).
__global__ void __launch_bounds__(128) k_trace_remark(const uint16_t *__restrict__ argx, const TileRec *tiles,
                                                      uint64_t ntiles, uint64_t tpw, const uint32_t *wflag,
                                                      uint32_t *bm)
{
    extern __shared__ uint16_t sa[];
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        if (!wflag[t / tpw]) continue;
        const TileRec r = tiles[t];
        if (!r.valid || !r.remark) continue;
        const TileArgs A = stage_args(argx, r, sa);
        if (threadIdx.x == 0) {
            bm_clear(bm, r.s + 1, r.e);
            uint32_t j = r.remark - 1u;
            for (;;) {
                bm_set(bm, j);
                const uint32_t i = A.arg(j);
                if (i <= r.s) break;
                j = i;
            }
        }
        __syncthreads();
    }
}

cudaError_t run_traceback(const DPParams &P, uint32_t *bitmap, uint64_t ntiles, uint16_t *maps, uint32_t *wflag,
                          cudaStream_t st, int *launches)
{
    *launches = 0;
    if (P.n == 0) return cudaSuccess;
    const unsigned tb = 128;
    const size_t stage = (size_t)(P.tile_len < kTraceStage ? P.tile_len : kTraceStage) * sizeof(uint16_t);
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const unsigned grid = (unsigned)(ntiles < (uint64_t)nsm * 8 ? ntiles : (uint64_t)nsm * 8);
    cudaError_t e = cudaMemsetAsync(wflag, 0, 4 * P.nwin, st);
    if (e != cudaSuccess) return e;
// walk A: thread per tile through L1/L2, or one CTA of kTraceAThreads per tile with the tile's
// args staged in shared memory.  Measured (traceback ms, thread / CTA of 128 / CTA of 256):
// c4 (21,800 tiles): 0.321 / 0.329 / 0.333 -- every walk runs at once and hides its own latency;
// c5 (2,450 tiles of 4096): 0.772 / 0.390 / 0.392 -- too few walks in flight, each hop an L2
// round trip.  So the thread walk only for jobs with many tiles.
#ifndef UELLM_TRACE_A
#define UELLM_TRACE_A 128
#endif
#ifndef UELLM_TRACE_C_STAGED
#define UELLM_TRACE_C_STAGED 1
#endif
#ifndef UELLM_TRACE_A_WARP
#define UELLM_TRACE_A_WARP 1
#endif
#ifndef UELLM_TRACE_B_WARP
#define UELLM_TRACE_B_WARP 1
#endif
    const bool stage_walk = UELLM_TRACE_A && ntiles < (uint64_t)nsm * 64 &&
                            P.tile_len * sizeof(uint16_t) <= 160 * 1024;
    if (UELLM_TRACE_A_WARP && P.tile_len <= 8192) {
        const size_t sm = (size_t)kTraceWarps * trace_warp_smem(P.tile_len);
        if (sm > 48 * 1024) {
            e = cudaFuncSetAttribute(k_trace_a_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            if (e != cudaSuccess) return e;
        }
        k_trace_a_warp<<<(unsigned)ceil_div(ntiles, kTraceWarps), 32 * kTraceWarps, sm, st>>>(P.argx, P.tiles, ntiles,
                                                                                            bitmap, P.tile_len);
    } else if (stage_walk) {
        e = cudaFuncSetAttribute(k_trace_a_smem, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(P.tile_len * sizeof(uint16_t)));
        if (e != cudaSuccess) return e;
        k_trace_a_smem<<<(unsigned)ntiles, UELLM_TRACE_A, P.tile_len * sizeof(uint16_t), st>>>(P.argx, P.tiles, bitmap);
    } else {
        k_trace_a<<<(unsigned)ceil_div(ntiles, tb), tb, 0, st>>>(P.argx, P.tiles, ntiles, bitmap);
    }
    if (UELLM_TRACE_B_WARP && P.tile_len <= 8192) {
        const size_t sm = (size_t)kTraceWarps * trace_warp_smem(P.tile_len);
        if (sm > 48 * 1024) {
            e = cudaFuncSetAttribute(k_trace_b_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            if (e != cudaSuccess) return e;
        }
        k_trace_b_warp<<<(unsigned)ceil_div(ntiles, kTraceWarps), 32 * kTraceWarps, sm, st>>>(
            P.argx, P.tiles, ntiles, P.tpw, bitmap, P.diag, wflag, P.tile_len);
    } else {
        k_trace_b<<<(unsigned)ceil_div(ntiles, tb), tb, 0, st>>>(P.argx, P.tiles, ntiles, P.tpw, bitmap, P.diag, wflag);
    }
    k_trace_maps<<<grid, 256, stage, st>>>(P.argx, P.tiles, ntiles, P.tpw, wflag, P.W, maps);
    if (UELLM_TRACE_C_STAGED && P.W <= kTraceCStageW && (P.W & 7u) == 0) {
        const size_t sm = (size_t)2 * 32 * P.W * sizeof(uint16_t);
        if (sm > 48 * 1024) {
            e = cudaFuncSetAttribute(k_trace_c_staged, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            if (e != cudaSuccess) return e;
        }
        k_trace_c_staged<<<(unsigned)P.nwin, 32, sm, st>>>(maps, P.tiles, P.tpw, P.nwin, P.window, P.W, bitmap, P.diag);
    } else {
        k_trace_c<<<(unsigned)ceil_div(P.nwin * 32, 128), 128, 0, st>>>(maps, P.tiles, P.tpw, P.nwin, P.window, P.W,
                                                                       bitmap, P.diag);
    }
    k_trace_remark<<<grid, 128, stage, st>>>(P.argx, P.tiles, ntiles, P.tpw, wflag, bitmap);
    *launches = 5;
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------
// Alg. 1 SLO-ODBS with readings R1-R6/R10/R12 -- parallel form.
//
// A flush always leaves an empty batch (line 14-19 seeds the next batch with q exactly as an
// admission into an empty batch would; the line-20 dynamic-cap flush and the SLO-split flush
// clear the state), so the batch that starts at position x evolves independently of how x was
// reached: next(x), the start of the following batch, is a function of x alone (<= W steps).
//   k_alg1_next   one thread per position: simulate Alg. 1 from a fresh batch at x -> next(x)
//   k_a1_*        mark the chain w0 -> next(w0) -> ... by binary lifting (below).
// Doubles with explicit round-to-nearest intrinsics (no FMA contraction): every decision is
// bit-identical to the CPU oracle's sequential scan.
// Line-20 flush test without the division (exact): with den = max(CM, eps) > 0 and finite,
// q = RN(threshold / den) and k = bsize + 1 <= W, "bsize >= cap" is "q < k".  The sign of
// fma(-k, den, threshold) is the sign of threshold - k*den exactly, so q >= k when it is >= 0;
// when the same test against km (the double below k) is < 0, q <= km < k.  Only a quotient in
// [km, k) -- where rounding decides -- takes the division.
__device__ __forceinline__ bool a1_cap_flush(double threshold, double den, uint32_t bsize, uint32_t W)
{
    if (bsize >= W) return true;                               // cap <= W
    const double k = (double)(bsize + 1);
    if (__fma_rn(-k, den, threshold) >= 0.0) return false;
    const double km = __longlong_as_double(__double_as_longlong(k) - 1);
    if (__fma_rn(-km, den, threshold) < 0.0) return true;
    return !(__ddiv_rn(threshold, den) >= k);
}

// SPLIT: split_on_slo_change; UNIT: w1 == l1 == l2 == 1 (x * 1.0 == x exactly, so those four
// multiplications are skipped without changing a bit).  O (the batch's max predicted length) is
// kept as an integer beside its double copy (outputs are u32, exact in a double).
template <bool SPLIT, bool UNIT>
__global__ void __launch_bounds__(256) k_alg1_next(Alg1Params A, uint16_t *__restrict__ nd)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const bool thr_finite = isfinite(A.threshold);
    for (uint64_t xx = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; xx < A.n; xx += stride) {
        const uint32_t x = (uint32_t)xx;
        const uint32_t w1 = (uint32_t)min(((uint64_t)(x / A.window) + 1) * A.window, (uint64_t)A.n);
        uint32_t bsize = 0, MI = 0, Oi = 0;
        double L_CM = 0.0, O_CM = 0.0, CM = 0.0, nb1 = 1.0;
        uint32_t p = x, next = w1;
        // the slo division is cached (exactly): slo_s only changes with the SLO value (sorted runs)
        uint32_t last_su = A.rslo[x];
        double slo = __ddiv_rn((double)last_su, 1e6);
        for (; p < w1; ++p) {
            const uint32_t su = A.rslo[p];
            if (SPLIT && bsize > 0 && su != last_su) { next = p; break; }
            if (su != last_su) { slo = __ddiv_rn((double)su, 1e6); last_su = su; }
            const uint32_t outp = A.rout[p];
            const double len = (double)outp;
            const uint32_t inx = A.rin[p];
            double T_l = __dmul_rn(__dadd_rn(slo, L_CM), nb1);
            if (!UNIT) T_l = __dmul_rn(T_l, A.l1);
            double T_o = A.eq2_additive ? __dadd_rn(len, O_CM) : __dsub_rn(len, O_CM);
            T_o = __dmul_rn(T_o, nb1);
            if (!UNIT) T_o = __dmul_rn(T_o, A.l2);
            const double Total = __dadd_rn(UNIT ? T_l : __dmul_rn(A.w1, T_l), __dmul_rn(A.w2, T_o));
            bool admit = (bsize == 0);
            if (!admit && Total <= A.threshold) {
                const uint64_t s = max(inx, MI);
                const uint64_t O = max(outp, Oi);
                admit = (uint64_t)(bsize + 1) * (s + O) <= A.cap_tok;
            }
            if (!admit) { next = p; break; }                  // q seeds the next batch
            const double cmq = __dadd_rn(UNIT ? len : __dmul_rn(A.w1, len), __dmul_rn(A.w2, slo));
            bsize += 1;
            nb1 = __dadd_rn(nb1, 1.0);                         // = bsize + 1, exact
            if (slo > L_CM) L_CM = slo;
            if (outp > Oi) { Oi = outp; O_CM = len; }
            if (cmq > CM) CM = cmq;
            if (inx > MI) MI = inx;
            const double den = CM > A.eps ? CM : A.eps;
            bool flush;
            if (thr_finite && den > 0.0 && isfinite(den)) {
                flush = a1_cap_flush(A.threshold, den, bsize, A.W);
            } else {                                           // the literal form
                const double capd = floor(__ddiv_rn(A.threshold, den));
                const uint64_t cap = capd < 1.0 ? 1 : (capd > (double)A.W ? (uint64_t)A.W : (uint64_t)capd);
                flush = bsize >= cap;
            }
            if (flush) { next = p + 1; break; }                // line 20: flush after q
        }
        nd[x] = (uint16_t)(next - x);                          // in [1, W]
    }
}

// Chain marking w0 -> next(w0) -> ... without a serial walk.  Greedy chains started at
// different positions phase-lock on the dynamic cap and rarely re-merge, so the walk is split
// by binary lifting instead, per sub-tile of T positions (T a power of two >= W):
//   k_a1_lift         lift tables L[k][x] = next^(2^k)(x) inside the sub-tile (EXIT once it
//                     leaves), then for each possible entry x < W the exit offset into the next
//                     sub-tile;
//   k_a1_entries      per window, sub-tile entries in order (one table lookup per sub-tile);
//   k_a1_mark         with the entries known, walk each sub-tile's part of the chain from its
//                     entry (one thread per sub-tile).
constexpr uint16_t kExit = 0xffff;

#ifndef UELLM_A1_LIFT_THREADS
#define UELLM_A1_LIFT_THREADS 256
#endif
__global__ void __launch_bounds__(UELLM_A1_LIFT_THREADS) k_a1_lift(Alg1Params A, const uint16_t *__restrict__ nd, uint32_t T, uint32_t K,
                                                 uint64_t spw, uint16_t *__restrict__ exit_first,
                                                 const uint32_t *__restrict__ entries, uint32_t *bm)
{
    extern __shared__ uint16_t sl[];            // K levels x T, then E0[T] (exit offset of the last hop)
    uint16_t *E0 = sl + (size_t)K * T;
    const uint64_t t = blockIdx.x, w = t / spw, kk = t % spw;
    const uint64_t w0 = w * A.window, w1 = min(w0 + A.window, (uint64_t)A.n);
    const uint64_t s = w0 + kk * T;
    if (s >= w1) return;
    const uint32_t len = (uint32_t)min((uint64_t)T, w1 - s);
    for (uint32_t x = threadIdx.x; x < len; x += blockDim.x) {
        const uint32_t nx = x + nd[s + x];
        sl[x] = nx < len ? (uint16_t)nx : kExit;
        E0[x] = nx < len ? 0 : (uint16_t)(nx - len);
    }
    __syncthreads();
    for (uint32_t lv = 1; lv < K; ++lv) {
        for (uint32_t x = threadIdx.x; x < len; x += blockDim.x) {
            const uint16_t a = sl[(lv - 1) * T + x];
            sl[lv * T + x] = a == kExit ? kExit : sl[(lv - 1) * T + a];
        }
        __syncthreads();
    }
    auto climb = [&](uint32_t x, uint32_t &depth, uint32_t &ex) {     // hops until the exit
        uint32_t y = x, h = 0;
        for (int lv = (int)K - 1; lv >= 0; --lv) {
            const uint16_t a = sl[lv * T + y];
            if (a != kExit) { y = a; h += 1u << lv; }
        }
        depth = h + 1;
        ex = E0[y];
    };
    const uint32_t Wf = min(A.W, len);
    for (uint32_t x = threadIdx.x; x < Wf; x += blockDim.x) {
        uint32_t d, ex;
        climb(x, d, ex);
        exit_first[t * A.W + x] = (uint16_t)ex;
    }

}

// One warp per window: the exit rows of the next CH sub-tiles (contiguous in exit_first) are
// staged in shared memory by the whole warp, then lane 0 follows the chain through them with
// shared-memory lookups only -- one global-memory latency per CH sub-tiles instead of per sub-tile.
constexpr uint32_t kA1EntWarps = 4, kA1EntElems = 4096;          // u16 staged per warp
__global__ void __launch_bounds__(kA1EntWarps * 32) k_a1_entries(Alg1Params A, uint32_t T, uint64_t spw,
                                                                 const uint16_t *__restrict__ exit_first,
                                                                 uint32_t *entries)
{
    __shared__ __align__(16) uint16_t buf[kA1EntWarps][kA1EntElems];
    const uint32_t lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
    const uint64_t w = (uint64_t)blockIdx.x * kA1EntWarps + wi;
    if (w >= A.nwin) return;
    const uint64_t w0 = w * A.window, w1 = min(w0 + A.window, (uint64_t)A.n);
    const uint64_t nsub = ceil_div(w1 - w0, (uint64_t)T);
    const uint32_t CH = max(1u, kA1EntElems / A.W);
    uint16_t *b = buf[wi];
    // chunk k0: sub-tiles [k0, k0 + c), their exit rows at src, m staged u16
    auto chunk = [&](uint64_t k0, uint32_t &c, const uint16_t *&src, uint32_t &m) {
        c = (uint32_t)min((uint64_t)CH, nsub - k0);
        src = exit_first + (w * spw + k0) * A.W;
        // only a window's last sub-tile can be shorter than W (its exit row holds len entries)
        const uint64_t last_len = min((uint64_t)T, w1 - (w0 + (k0 + c - 1) * T));
        m = (uint32_t)min((uint64_t)(c - 1) * A.W + min((uint64_t)A.W, last_len),
                          (uint64_t)kA1EntElems);              // W > kA1EntElems: first part only
    };
    constexpr uint32_t kV = kA1EntElems / 8 / 32;
    const bool vec = A.W % 8 == 0;                             // rows 16-byte aligned: uint4 loads
    uint4 r[kV];                                               // next chunk, in flight during the walk
    auto issue = [&](const uint16_t *src, uint32_t m) {
        const uint4 *s4 = reinterpret_cast<const uint4 *>(src);
#pragma unroll
        for (uint32_t u = 0; u < kV; ++u)
            if (lane + 32 * u < (m >> 3)) r[u] = s4[lane + 32 * u];
    };
    uint64_t e = w0;
    if (vec && nsub > 0) {
        uint32_t c0, m0;
        const uint16_t *s0;
        chunk(0, c0, s0, m0);
        issue(s0, m0);
    }
    for (uint64_t k0 = 0; k0 < nsub; k0 += CH) {
        uint32_t c, m;
        const uint16_t *src;
        chunk(k0, c, src, m);
        if (vec) {
            const uint32_t m8 = m >> 3;
            uint4 *b4 = reinterpret_cast<uint4 *>(b);
#pragma unroll
            for (uint32_t u = 0; u < kV; ++u)
                if (lane + 32 * u < m8) b4[lane + 32 * u] = r[u];
            for (uint32_t i = 8 * m8 + lane; i < m; i += 32) b[i] = src[i];
            if (k0 + CH < nsub) {
                uint32_t c1, m1;
                const uint16_t *s1;
                chunk(k0 + CH, c1, s1, m1);
                issue(s1, m1);
            }
        } else {
            for (uint32_t i = lane; i < m; i += 32) b[i] = src[i];
        }
        __syncwarp();
        if (lane == 0) {
            for (uint32_t j = 0; j < c; ++j) {
                const uint64_t s = w0 + (k0 + j) * T;
                entries[w * spw + k0 + j] = (uint32_t)e;
                const uint64_t len = min((uint64_t)T, w1 - s), off = e - s;
                const uint64_t idx = (uint64_t)j * A.W + off;
                e = s + len + (idx < m ? b[idx] : src[idx]);
            }
        }
        e = __shfl_sync(0xffffffffu, e, 0);
        __syncwarp();
    }
}

// With every sub-tile's entry known (k_a1_entries), marking its part of the chain is a plain walk
// e -> next(e) -> ... inside the sub-tile (same marks as climbing the lift tables).  One warp per
// sub-tile: the warp stages next_delta of the sub-tile in shared memory with 16-byte loads, lane 0
// walks it there and sets the bits in a shared-memory copy of the sub-tile's bitmap words, which
// the warp then ORs into the global bitmap (neighbouring sub-tiles may share a boundary word).
#ifndef UELLM_A1_SUB
#define UELLM_A1_SUB 1024
#endif
// staged deltas per warp: one minimum-size sub-tile plus the word-alignment slack (larger T,
// i.e. W > UELLM_A1_SUB, walks global memory)
constexpr uint32_t kA1MarkWarps = 8, kA1MarkElems = UELLM_A1_SUB + 32, kA1MarkWords = kA1MarkElems / 32;
constexpr uint32_t kA1MarkVec = (kA1MarkElems / 8 + 31) / 32;      // uint4 loads per lane
__global__ void __launch_bounds__(kA1MarkWarps * 32) k_a1_mark(Alg1Params A, const uint16_t *__restrict__ nd,
                                                               uint32_t T, uint64_t spw,
                                                               const uint32_t *__restrict__ entries, uint32_t *bm)
{
    __shared__ __align__(16) uint16_t snd[kA1MarkWarps][kA1MarkElems];
    __shared__ uint32_t sbits[kA1MarkWarps][kA1MarkWords];
    const uint32_t lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
    const uint64_t t = (uint64_t)blockIdx.x * kA1MarkWarps + wi;
    if (t >= spw * A.nwin) return;
    const uint64_t w = t / spw, kk = t % spw;
    const uint64_t w0 = w * A.window, w1 = min(w0 + A.window, (uint64_t)A.n);
    const uint64_t s = w0 + kk * T;
    if (s >= w1) return;
    const uint64_t z = min(s + (uint64_t)T, w1);
    const uint64_t bb = s & ~31ull;                       // staging and bitmap base (word aligned)
    const uint64_t nwords = (z - 1 - bb) / 32 + 1;
    if (nwords > kA1MarkWords) {                          // T > UELLM_A1_SUB (large W): walk global memory
        if (lane == 0) {
            for (uint64_t x = entries[t]; x < z; x += nd[x]) bm_set(bm, (uint32_t)x);
            if (z == A.n) bm_set(bm, A.n);
        }
        return;
    }
    const uint32_t L = (uint32_t)(z - bb);                // <= kA1MarkElems
    uint16_t *b = snd[wi];
    uint32_t *sw = sbits[wi];
    {
        const uint32_t L8 = L >> 3;
        const uint4 *s4 = reinterpret_cast<const uint4 *>(nd + bb);
        uint4 *b4 = reinterpret_cast<uint4 *>(b);
        uint4 r[kA1MarkVec];
#pragma unroll
        for (uint32_t u = 0; u < kA1MarkVec; ++u)
            if (lane + 32 * u < L8) r[u] = s4[lane + 32 * u];
#pragma unroll
        for (uint32_t u = 0; u < kA1MarkVec; ++u)
            if (lane + 32 * u < L8) b4[lane + 32 * u] = r[u];
        for (uint32_t i = 8 * L8 + lane; i < L; i += 32) b[i] = nd[bb + i];
        for (uint32_t i = lane; i < nwords; i += 32) sw[i] = 0;
    }
    __syncwarp();
    if (lane == 0) {
        // offsets are monotone along the chain, so each bitmap word is visited in one run:
        // accumulate it in a register and store it once (no shared-memory read-modify-write)
        uint32_t o = (uint32_t)(entries[t] - bb), cw = o >> 5, acc = 0;
        while (o < L) {
            const uint32_t wd = o >> 5;
            if (wd != cw) { sw[cw] = acc; acc = 0; cw = wd; }
            acc |= 1u << (o & 31);
            o += b[o];
        }
        if (acc) sw[cw] = acc;
        if (z == A.n) bm_set(bm, A.n);
    }
    __syncwarp();
    for (uint32_t i = lane; i < nwords; i += 32)
        if (sw[i]) atomicOr(bm + (bb >> 5) + i, sw[i]);
}

static uint32_t a1_sub(uint32_t W)
{
    uint32_t T = UELLM_A1_SUB;
    while (T < W) T <<= 1;
    return T;
}

cudaError_t launch_alg1(const Alg1Params &A, uint32_t *bitmap, uint16_t *next_delta, uint2 *tile_exits, Diag *diag,
                        cudaStream_t st)
{
    (void)diag;
    if (A.n == 0) return cudaSuccess;
    uint64_t blocks = ceil_div(A.n, 256);
    if (blocks > 148ull * 64) blocks = 148ull * 64;
    const bool unit = A.w1 == 1.0 && A.l1 == 1.0 && A.l2 == 1.0;
    if (A.split) {
        if (unit) k_alg1_next<true, true><<<(unsigned)blocks, 256, 0, st>>>(A, next_delta);
        else k_alg1_next<true, false><<<(unsigned)blocks, 256, 0, st>>>(A, next_delta);
    } else {
        if (unit) k_alg1_next<false, true><<<(unsigned)blocks, 256, 0, st>>>(A, next_delta);
        else k_alg1_next<false, false><<<(unsigned)blocks, 256, 0, st>>>(A, next_delta);
    }
    const uint32_t T = a1_sub(A.W);
    uint32_t K = 0;
    while ((1u << K) < T) ++K;
    const uint64_t spw = ceil_div(A.window, T), nt = spw * A.nwin;
    // scratch inside the Alg. 1 tile area: entries (u32 per sub-tile), exit_first (u16 x W per sub-tile)
    uint32_t *entries = reinterpret_cast<uint32_t *>(tile_exits);
    uint16_t *exit_first = reinterpret_cast<uint16_t *>(entries + ((nt + 1 + 3) & ~3ull));   // 16-byte aligned rows
    const size_t smem = ((size_t)K + 1) * T * sizeof(uint16_t);
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(k_a1_lift, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem))) return e;
    k_a1_lift<<<(unsigned)nt, UELLM_A1_LIFT_THREADS, smem, st>>>(A, next_delta, T, K, spw, exit_first, entries, bitmap);
    k_a1_entries<<<(unsigned)ceil_div(A.nwin, kA1EntWarps), kA1EntWarps * 32, 0, st>>>(A, T, spw, exit_first, entries);
    k_a1_mark<<<(unsigned)ceil_div(nt, kA1MarkWarps), kA1MarkWarps * 32, 0, st>>>(A, next_delta, T, spw, entries, bitmap);
    return cudaGetLastError();
}

// bytes of Alg. 1 scratch: per sub-tile an entry (u32) and W exit offsets (u16)
uint64_t alg1_scratch_bytes(uint64_t window, uint64_t nwin, uint32_t W)
{
    const uint64_t nt = ceil_div(window, a1_sub(W)) * nwin;
    return 4 * (nt + 1) + 2ull * W * nt + 16;
}


// ---------------------------------------------------------------------------------------
// Compaction: batch_offsets = ascending positions of the set bits; num_batches = count - 1.
template <int NT>
__device__ uint32_t block_excl_scan(uint32_t v, uint32_t *total)
{
    __shared__ uint32_t wsum[NT / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t s = lane < NT / 32 ? wsum[lane] : 0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, s, d);
            if (lane >= d) s += y;
        }
        if (lane < NT / 32) wsum[lane] = s;
    }
    __syncthreads();
    const uint32_t before = warp ? wsum[warp - 1] : 0;
    *total = wsum[NT / 32 - 1];
    __syncthreads();
    return before + x - v;
}

__global__ void __launch_bounds__(kScanBlock) k_compact_count(const uint32_t *bm, uint64_t nwords, uint32_t *wscan,
                                                              uint32_t *blocksum)
{
    const uint64_t w = (uint64_t)blockIdx.x * kScanBlock + threadIdx.x;
    const uint32_t c = w < nwords ? __popc(bm[w]) : 0;
    uint32_t tot;
    const uint32_t ex = block_excl_scan<kScanBlock>(c, &tot);
    if (w < nwords) wscan[w] = ex;
    if (threadIdx.x == 0) blocksum[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kScanBlock) k_compact_blocks(uint32_t *blocksum, uint64_t nblocks,
                                                               unsigned long long *num_batches)
{
    const uint64_t per = ceil_div(nblocks, kScanBlock);
    const uint64_t a = threadIdx.x * per, z = min(a + per, nblocks);
    uint32_t s = 0;
    for (uint64_t b = a; b < z; ++b) s += blocksum[b];
    uint32_t tot;
    uint32_t run = block_excl_scan<kScanBlock>(s, &tot);
    for (uint64_t b = a; b < z; ++b) { uint32_t v = blocksum[b]; blocksum[b] = run; run += v; }
    if (threadIdx.x == 0) *num_batches = (unsigned long long)tot - 1ull;
}

__global__ void __launch_bounds__(256) k_compact_write(const uint32_t *bm, uint64_t nwords, const uint32_t *wscan,
                                                       const uint32_t *blocksum, uint32_t *offsets)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nwords; w += stride) {
        uint32_t bits = bm[w];
        if (!bits) continue;
        uint32_t pos = blocksum[w / kScanBlock] + wscan[w];
        while (bits) {
            const int b = __ffs(bits) - 1;
            bits &= bits - 1;
            offsets[pos++] = (uint32_t)(w * 32 + b);
        }
    }
}

cudaError_t run_compact(const uint32_t *bitmap, uint64_t n, uint32_t *wscan, uint32_t *blocksum,
                        uint32_t *offsets, unsigned long long *num_batches, cudaStream_t st)
{
    const uint64_t nwords = (n + 1 + 31) / 32;
    const uint64_t nblocks = ceil_div(nwords, kScanBlock);
    k_compact_count<<<(unsigned)nblocks, kScanBlock, 0, st>>>(bitmap, nwords, wscan, blocksum);
    k_compact_blocks<<<1, kScanBlock, 0, st>>>(blocksum, nblocks, num_batches);
    uint64_t wb = ceil_div(nwords, 256);
    if (wb > 148ull * 16) wb = 148ull * 16;
    k_compact_write<<<(unsigned)wb, 256, 0, st>>>(bitmap, nwords, wscan, blocksum, offsets);
    return cudaGetLastError();
}

}  // namespace uellm
