// k_segdp.cu -- a6 SEG-DP: exact segmentation of each (SLO, length)-sorted window into batches.
//
//   C[w0] = 0,  C[j] = min_{i in [j-W, j), feasible} C[i] + est(i,j) + lambda * viol(i,j)
//   est(i,j)  = t_batch + t_iter*MO + b*(t_tok*MO + t_prefill*MI)          (R7)
//   viol(i,j) = #{k in [i,j): slo_us[k] < est(i,j)}                         (R8)
//   feasible  = b == 1  or  b*(MI+MO) <= cap_tok, cap_tok = floor(kv_cap / (kvpe*l*h))
//               (P:60 KV peak, P:366 reserve; equivalent to the byte form)    (R10)
//   arg[j]    = the smallest minimising i                                      (R9)
//
// GPU design:
//  * one warp per tile of T positions (T a multiple of W, tiles never cross windows); lanes
//    evaluate the live breakpoint candidates of the tile's current position in parallel and
//    reduce (cost, i) with three redux.sync.min;
//  * exact dominance pruning D1 against the next live candidate:
//      i dead once C[i'] - C[i] < (i' - i) * (t_tok*MO(i',j) + t_prefill*MI(i',j)),
//    plus the monotone deaths (b > W, KV cap, SLO split) which always form a prefix;
//  * tile k > 0 first runs "locally" (as if a batch started at its first position); a fix-up
//    pass re-runs its head from tile k-1's tail until the fixed values differ from the local
//    ones by one constant over W consecutive boundaries -- from there on every later value is
//    local + constant and every argmin is identical (the recurrence reads only the last W
//    values).  A per-window cascade re-runs the (rare) tiles whose predecessor did not
//    converge, so the result is exact for every input; see DESIGN.md for the argument.
#include "internal.cuh"

namespace uellm {

struct WarpSlots {
    long long *cC;
    uint32_t *ci, *mo, *mi;
};

__device__ __forceinline__ WarpSlots slots_for(char *base, uint32_t cap, int w)
{
    char *p = base + (size_t)w * cap * 20;
    WarpSlots S;
    S.cC = (long long *)p;
    S.ci = (uint32_t *)(p + (size_t)cap * 8);
    S.mo = (uint32_t *)(p + (size_t)cap * 12);
    S.mi = (uint32_t *)(p + (size_t)cap * 16);
    return S;
}

__device__ __forceinline__ uint32_t lane_lt()
{
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// #{k in [i, j) : rslo[k] < est} on an ascending run rslo[i..j), slo_x = rslo[j-1].
__device__ __noinline__ uint32_t viol_count_slow(const uint32_t *__restrict__ rslo, uint32_t i, uint32_t j,
                                                 unsigned long long est, uint32_t slo_x)
{
    if ((unsigned long long)slo_x < est) return j - i;
    if ((unsigned long long)__ldg(rslo + i) >= est) return 0;
    uint32_t lo = i + 1, hi = j - 1;      // rslo[i] < est <= rslo[j-1]
    while (lo < hi) {
        uint32_t mid = lo + (hi - lo) / 2;
        if ((unsigned long long)__ldg(rslo + mid) < est) lo = mid + 1; else hi = mid;
    }
    return lo - i;
}

struct DpResult {
    int conv;
    uint32_t conv_pos, fix_end;
    long long delta;
    uint64_t positions;
    uint64_t evals;
};

// Runs the DP for boundaries j = s+1 .. e on one warp.
//   FIX = false: local run (candidate set {s}, C[s] = 0), writes Cx.
//   FIX = true : fix-up run; candidates are boundaries [s-W+1, s] with C taken from src (the
//                frame of tile k-1, src[i-1] = C at boundary i); writes CFx; compares with the
//                local values Cx of this tile and stops once converged and j >= stop_min.
// Boundary j's value/arg is stored at index j-1 (Cx/CFx/argx).
template <bool FIX>
__device__ DpResult dp_warp(const DPParams &P, const WarpSlots &S, uint32_t s, uint32_t e,
                            const long long *__restrict__ src, uint32_t stop_min)
{
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t lt = lane_lt();
    const uint32_t W = P.W;
    DpResult R;
    R.conv = 0; R.conv_pos = e; R.fix_end = e; R.delta = 0; R.positions = 0; R.evals = 0;
    uint32_t L;
    uint32_t run_start;
    uint32_t prev_slo;
    long long Cprev;
    long long d_run = 0;
    uint32_t run = 0;

    if (!FIX) {
        if (lane == 0) { S.ci[0] = s; S.cC[0] = 0; S.mo[0] = 0; S.mi[0] = 0; }
        L = 1;
        run_start = s;
        prev_slo = (s < P.n) ? __ldg(P.rslo + s) : 0;
        Cprev = 0;
    } else {
        // candidates: boundaries i = s-W+1+q, q in [0, W); MO/MI over [i, s) by suffix max
        const uint32_t i0 = s - W + 1;
        uint32_t cmo = 0, cmi = 0;
        uint32_t rs = i0;
        for (uint32_t r = 0; r * 32 < W; ++r) {
            uint32_t off = r * 32 + lane + 1;            // position p = s - off
            bool valid = off <= W - 1;                    // p >= i0
            uint32_t p = s - off;
            uint32_t vo = valid ? __ldg(P.rout + p) : 0, vi = valid ? __ldg(P.rin + p) : 0;
            uint32_t vs = valid ? __ldg(P.rslo + p) : 0;
            uint32_t vsp = (valid && p > i0) ? __ldg(P.rslo + p - 1) : vs;
            if (valid && p > i0 && vs != vsp) rs = max(rs, p);
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                uint32_t to = __shfl_up_sync(0xffffffffu, vo, d), ti = __shfl_up_sync(0xffffffffu, vi, d);
                if ((int)lane >= d) { vo = max(vo, to); vi = max(vi, ti); }
            }
            vo = max(vo, cmo); vi = max(vi, cmi);
            if (valid) {
                uint32_t q = p - i0;
                S.ci[q] = p; S.mo[q] = vo; S.mi[q] = vi; S.cC[q] = src[p - 1];
            }
            cmo = __shfl_sync(0xffffffffu, vo, 31);
            cmi = __shfl_sync(0xffffffffu, vi, 31);
        }
        if (lane == 0) { S.ci[W - 1] = s; S.mo[W - 1] = 0; S.mi[W - 1] = 0; S.cC[W - 1] = src[s - 1]; }
        L = W;
        run_start = __reduce_max_sync(0xffffffffu, rs);
        prev_slo = __ldg(P.rslo + s - 1);
        Cprev = src[s - 1];
        d_run = Cprev;          // local C at boundary s is 0
        run = 1;
    }
    __syncwarp();

    // element cache: lane l holds position cbase + l; output buffer aligned with it
    uint32_t cbase = s, c_in = 0, c_out = 0, c_slo = 0;
    long long c_cl = 0, o_C = 0;
    uint32_t o_A = 0;
    auto refill = [&](uint32_t base) {
        uint32_t p = base + lane;
        bool v = p < e;
        c_in = v ? __ldg(P.rin + p) : 0;
        c_out = v ? __ldg(P.rout + p) : 0;
        c_slo = v ? __ldg(P.rslo + p) : 0;
        if (FIX) c_cl = v ? P.Cx[p] : 0;
    };
    auto flush = [&](uint32_t upto) {            // positions [cbase, upto)
        uint32_t p = cbase + lane;
        if (p < upto) {
            (FIX ? P.CFx : P.Cx)[p] = o_C;
            P.argx[p] = (uint16_t)o_A;
        }
    };
    refill(cbase);

    uint32_t j = s + 1;
    for (; j <= e; ++j) {
        const uint32_t x = j - 1;
        if (x - cbase >= 32) { flush(x); cbase = x; refill(cbase); }
        const uint32_t in_x = __shfl_sync(0xffffffffu, c_in, x - cbase);
        const uint32_t out_x = __shfl_sync(0xffffffffu, c_out, x - cbase);
        const uint32_t slo_x = __shfl_sync(0xffffffffu, c_slo, x - cbase);
        if (slo_x != prev_slo) { run_start = x; prev_slo = slo_x; }
        if (j >= s + 2) {
            if (lane == 0) { S.ci[L] = x; S.cC[L] = Cprev; S.mo[L] = 0; S.mi[L] = 0; }
            ++L;
            __syncwarp();
        }
        unsigned long long lb = ~0ull;
        uint32_t lbi = 0xffffffffu;
        uint32_t wr = 0;
        R.evals += L;
        const uint32_t nr = (L + 31) >> 5;
        for (uint32_t r = 0; r < nr; ++r) {
            const uint32_t k = r * 32 + lane;
            const bool valid = k < L;
            uint32_t ci = 0, mo = 0, mi = 0;
            long long cC = 0;
            if (valid) { ci = S.ci[k]; cC = S.cC[k]; mo = S.mo[k]; mi = S.mi[k]; }
            mo = max(mo, out_x);
            mi = max(mi, in_x);
            const uint32_t b = j - ci;
            const unsigned long long Sk = P.t_tok * mo + P.t_pre * mi;
            bool dead = !valid || b > W ||
                        (b > 1 && (unsigned long long)b * ((unsigned long long)mo + mi) > P.cap_tok) ||
                        (P.split && ci < run_start);
            // next live slot (k+1) for the dominance test
            long long nC = __shfl_down_sync(0xffffffffu, cC, 1);
            uint32_t ni = __shfl_down_sync(0xffffffffu, ci, 1);
            unsigned long long nS = __shfl_down_sync(0xffffffffu, Sk, 1);
            const bool has_next = k + 1 < L;
            if (lane == 31 && has_next) {
                ni = S.ci[k + 1];
                nC = S.cC[k + 1];
                nS = P.t_tok * max(S.mo[k + 1], out_x) + P.t_pre * max(S.mi[k + 1], in_x);
            }
            bool keep = false;
            if (!dead) {
                unsigned long long est = P.t_batch + P.t_iter * mo + (unsigned long long)b * Sk;
                unsigned long long pen = 0;
                if (P.lambda) {
                    uint32_t v;
                    if (ci >= run_start) v = ((unsigned long long)slo_x < est) ? b : 0;
                    else v = viol_count_slow(P.rslo, ci, j, est, slo_x);
                    pen = P.lambda * v;
                }
                unsigned long long tot = (unsigned long long)cC + est + pen;
                if (tot < lb) { lb = tot; lbi = ci; }
                const bool dominated = has_next && (nC - cC < (long long)((unsigned long long)(ni - ci) * nS));
                keep = !dominated;
            }
            __syncwarp();
            const uint32_t bal = __ballot_sync(0xffffffffu, keep);
            if (keep) {
                const uint32_t pos = wr + __popc(bal & lt);
                S.ci[pos] = ci; S.cC[pos] = cC; S.mo[pos] = mo; S.mi[pos] = mi;
            }
            wr += __popc(bal);
            __syncwarp();
        }
        L = wr;
        // warp argmin of (total, i), smallest i on ties: hi word, lo word, index
        const uint32_t hi = (uint32_t)(lb >> 32);
        const uint32_t mhi = __reduce_min_sync(0xffffffffu, hi);
        const uint32_t lo = (hi == mhi) ? (uint32_t)lb : 0xffffffffu;
        const uint32_t mlo = __reduce_min_sync(0xffffffffu, lo);
        const uint32_t ii = (hi == mhi && (uint32_t)lb == mlo) ? lbi : 0xffffffffu;
        const uint32_t barg = __reduce_min_sync(0xffffffffu, ii);
        const long long best = (long long)(((unsigned long long)mhi << 32) | mlo);
        Cprev = best;
        if (lane == x - cbase) { o_C = best; o_A = j - barg; }
        ++R.positions;
        if (FIX) {
            const long long cl = __shfl_sync(0xffffffffu, c_cl, x - cbase);
            const long long dj = best - cl;
            if (dj == d_run) ++run; else { d_run = dj; run = 1; }
            if (run >= W && j >= stop_min) {
                R.conv = 1; R.conv_pos = j; R.fix_end = j; R.delta = d_run;
                ++j;
                break;
            }
        }
    }
    flush(j - 1);                          // positions [cbase, last x + 1)
    return R;
}

// -------------------------------------------------------------------------------------
__device__ __forceinline__ void tile_bounds(const DPParams &P, uint64_t t, uint32_t &s, uint32_t &e,
                                            uint32_t &k, uint32_t &w, bool &valid)
{
    w = (uint32_t)(t / P.tpw);
    k = (uint32_t)(t % P.tpw);
    uint64_t w0 = (uint64_t)w * P.window, w1 = min(w0 + P.window, (uint64_t)P.n);
    uint64_t ss = w0 + (uint64_t)k * P.tile_len;
    valid = w < P.nwin && ss < w1;
    s = (uint32_t)ss;
    e = (uint32_t)min(ss + P.tile_len, w1);
}

__global__ void k_dp_local(DPParams P, uint64_t ntiles)
{
    extern __shared__ __align__(16) char smem[];
    const uint64_t t = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (t >= ntiles) return;
    uint32_t s, e, k, w; bool valid;
    tile_bounds(P, t, s, e, k, w, valid);
    const uint32_t lane = threadIdx.x & 31;
    if (!valid) {
        if (lane == 0) { TileRec r = {}; r.valid = 0; P.tiles[t] = r; }
        return;
    }
    WarpSlots S = slots_for(smem, P.cap_slots, threadIdx.x >> 5);
    DpResult R = dp_warp<false>(P, S, s, e, nullptr, 0);
    if (lane == 0) {
        atomicAdd(&P.diag->dp_evals, (unsigned long long)R.evals);
        TileRec r = {};
        r.s = s; r.e = e; r.valid = 1;
        r.conv = (k == 0); r.conv_pos = s; r.fix_end = s;
        P.tiles[t] = r;
    }
}

__global__ void k_dp_fix(DPParams P, uint64_t ntiles)
{
    extern __shared__ __align__(16) char smem[];
    const uint64_t t = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (t >= ntiles) return;
    uint32_t s, e, k, w; bool valid;
    tile_bounds(P, t, s, e, k, w, valid);
    if (!valid || k == 0) return;
    const uint32_t lane = threadIdx.x & 31;
    WarpSlots S = slots_for(smem, P.cap_slots, threadIdx.x >> 5);
    DpResult R = dp_warp<true>(P, S, s, e, P.Cx, 0);
    if (lane == 0) {
        TileRec &r = P.tiles[t];
        r.conv = R.conv; r.conv_pos = R.conv_pos; r.fix_end = R.fix_end; r.delta = R.delta;
        atomicAdd(&P.diag->fixup_positions, (unsigned long long)R.positions);
        atomicAdd(&P.diag->dp_evals, (unsigned long long)R.evals);
        if (!R.conv) atomicAdd(&P.diag->fixups_unconverged, 1ull);
    }
}

// One warp per window: resolve tiles whose predecessor did not converge, compute the frame
// offsets of every tile and the window's optimal cost C[w1].
__global__ void k_dp_cascade(DPParams P)
{
    extern __shared__ __align__(16) char smem[];
    const uint32_t w = blockIdx.x;
    const uint32_t lane = threadIdx.x & 31;
    WarpSlots S = slots_for(smem, P.cap_slots, 0);
    const uint64_t t0 = (uint64_t)w * P.tpw;
    uint32_t K = 0;
    while (K < P.tpw && P.tiles[t0 + K].valid) ++K;
    if (K == 0) return;
    // tile 0 is exact in its local frame
    long long tail_off = 0;          // offset of the frame holding tile (k-1)'s tail values
    bool tail_local = true;          // tail in Cx (local frame) vs CFx (fix-up frame)
    if (lane == 0) { P.tiles[t0].off_local = 0; P.tiles[t0].off_fix = 0; }
    for (uint32_t k = 1; k < K; ++k) {
        TileRec r = P.tiles[t0 + k];
        if (!tail_local) {
            DpResult R = dp_warp<true>(P, S, r.s, r.e, P.CFx, r.fix_end);
            r.conv = R.conv; r.conv_pos = R.conv_pos; r.fix_end = R.fix_end; r.delta = R.delta;
            if (lane == 0) {
                atomicAdd(&P.diag->cascade_reruns, 1ull);
                atomicAdd(&P.diag->fixup_positions, (unsigned long long)R.positions);
                atomicAdd(&P.diag->dp_evals, (unsigned long long)R.evals);
            }
        }
        r.off_fix = tail_off;
        if (r.conv) { r.off_local = tail_off + r.delta; tail_off = r.off_local; tail_local = true; }
        else { r.off_local = 0; tail_local = false; }
        if (lane == 0) P.tiles[t0 + k] = r;
        __syncwarp();
    }
    if (lane == 0) {
        const TileRec &r = P.tiles[t0 + K - 1];
        long long c;
        if (K == 1) c = P.Cx[r.e - 1];
        else c = r.conv ? P.Cx[r.e - 1] + r.off_local : P.CFx[r.e - 1] + r.off_fix;
        P.wincost[w] = (unsigned long long)c;
    }
}

static uint32_t warps_per_cta(uint32_t cap_slots)
{
    uint32_t per = cap_slots * 20;
    uint32_t wpc = kDpWarpsPerCta;
    while (wpc > 1 && wpc * per > 200 * 1024) --wpc;
    return wpc;
}

cudaError_t run_segdp(const DPParams &P, uint64_t ntiles, cudaStream_t st, void *const ev[3], int *launches)
{
    *launches = 0;
    if (P.n == 0 || ntiles == 0) return cudaSuccess;
    const uint32_t wpc = warps_per_cta(P.cap_slots);
    const size_t smem = (size_t)wpc * P.cap_slots * 20;
    const size_t smem1 = (size_t)P.cap_slots * 20;
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(k_dp_local, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem))) return e;
    if ((e = cudaFuncSetAttribute(k_dp_fix, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem))) return e;
    if ((e = cudaFuncSetAttribute(k_dp_cascade, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1))) return e;
    const unsigned blocks = (unsigned)ceil_div(ntiles, wpc);
    k_dp_local<<<blocks, wpc * 32, smem, st>>>(P, ntiles);
    ++*launches;
    if (ev[0]) cudaEventRecord((cudaEvent_t)ev[0], st);
    if (P.tpw > 1) { k_dp_fix<<<blocks, wpc * 32, smem, st>>>(P, ntiles); ++*launches; }
    if (ev[1]) cudaEventRecord((cudaEvent_t)ev[1], st);
    k_dp_cascade<<<P.nwin, 32, smem1, st>>>(P);
    ++*launches;
    if (ev[2]) cudaEventRecord((cudaEvent_t)ev[2], st);
    return cudaGetLastError();
}

}  // namespace uellm
