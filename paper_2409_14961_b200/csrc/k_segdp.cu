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
//  * one warp per tile of T positions (T a multiple of W, tiles never cross windows);
//  * fast path (dp_warp_blocked, 32-bit cost arithmetic): blocks of 32 boundaries, lane =
//    boundary for the candidates born before the block, lane = candidate for the ones born
//    inside it (argmin by three redux.sync.min per boundary); generic path (dp_warp, 64-bit):
//    lane = candidate, one boundary at a time;
//  * exact dominance pruning D1 against the next live candidate:
//      i dead once C[i'] - C[i] < (i' - i) * (t_tok*MO(i',j) + t_prefill*MI(i',j)),
//    plus the monotone deaths (b > W, KV cap, SLO split) which always form a prefix;
//  * tile k > 0 first runs "locally" (as if a batch started at its first position); a fix-up
//    pass re-runs its head from tile k-1's tail until the fixed values differ from the local
//    ones by one constant over W consecutive boundaries -- from there on every later value is
//    local + constant and every argmin is identical (the recurrence reads only the last W
//    values).  A per-window cascade re-runs the (rare) tiles whose predecessor did not
//    converge, so the result is exact for every input; see DESIGN.md for the argument.
#include <type_traits>

#include "internal.cuh"

namespace uellm {

#ifndef UELLM_EXT_UNROLL
#define UELLM_EXT_UNROLL 4
#endif
constexpr int kExtUnroll = UELLM_EXT_UNROLL;   // unroll of the fast block's external-candidate loop

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t *p)
{
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// relaxed (gpu scope) poll: unlike ld.acquire it does not invalidate the SM's L1 on every
// iteration (CCTL.IVALL), which would evict the records other warps on the SM are streaming; the
// acquire is a single fence once the flag is seen
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t *p)
{
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(uint32_t *p, uint32_t v)
{
    asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}

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
    uint64_t filled;            // boundaries written by the periodic fill of a uniform stretch
    uint32_t uni;               // local run: every record of the tile equals its first one
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
    R.conv = 0; R.conv_pos = e; R.fix_end = e; R.delta = 0; R.positions = 0; R.evals = 0; R.filled = 0;
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
                S.ci[q] = p; S.mo[q] = vo; S.mi[q] = vi; S.cC[q] = __ldcg(src + p - 1);
            }
            cmo = __shfl_sync(0xffffffffu, vo, 31);
            cmi = __shfl_sync(0xffffffffu, vi, 31);
        }
        if (lane == 0) { S.ci[W - 1] = s; S.mo[W - 1] = 0; S.mi[W - 1] = 0; S.cC[W - 1] = __ldcg(src + s - 1); }
        L = W;
        run_start = __reduce_max_sync(0xffffffffu, rs);
        prev_slo = __ldg(P.rslo + s - 1);
        Cprev = __ldcg(src + s - 1);
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
// Fast path ("narrow"): valid when max_in, max_out < 2^16 and
//   E = t_batch + t_iter*max_out + W*(t_tok*max_out + t_prefill*max_in) < 2^32,
// so est, S = t_tok*MO + t_prefill*MI, b*S and b*(MI+MO) all fit 32 bits (checked on the host).
// A candidate slot is 16 bytes, one LDS.128: C (i64) and (i | MO << 32 | MI << 48).
struct NarrowSlots {
    longlong2 *sl;              // .x = C, .y = i | mo << 32 | mi << 48
    uint32_t *tri;              // per-block triangular max table M[q][k], q < k < 32 (496 words)
    uint2 *hl;                  // per-block lower-hull subset of the lean external candidates
    uint32_t *ss;               // many-run variants: the block's SLO range staged for the violation counts
};

// #{k in [i, j) : slo[k] < est} on an ascending run staged in shared memory (ss[k - base]).
__device__ __forceinline__ uint32_t viol_count_sm(const uint32_t *ss, uint32_t base, uint32_t i, uint32_t j,
                                                  unsigned long long est, uint32_t slo_x)
{
    if ((unsigned long long)slo_x < est) return j - i;
    if ((unsigned long long)ss[i - base] >= est) return 0;
    uint32_t lo = i + 1, hi = j - 1;      // slo[i] < est <= slo[j-1]
    while (lo < hi) {
        const uint32_t mid = lo + (hi - lo) / 2;
        if ((unsigned long long)ss[mid - base] < est) lo = mid + 1; else hi = mid;
    }
    return lo - i;
}
// Capacity of the hull subset (larger subsets fall back to the whole list).
constexpr uint32_t kHullCap = 64;
#ifndef UELLM_HULL_MIN
#define UELLM_HULL_MIN 12
#endif
constexpr uint32_t kHullMin = UELLM_HULL_MIN;
#ifndef UELLM_DP_PREFETCH
#define UELLM_DP_PREFETCH 1
#endif
#ifndef UELLM_DP_VFREE
#define UELLM_DP_VFREE 1
#endif
#ifndef UELLM_DP_PRUNE_EVERY
#define UELLM_DP_PRUNE_EVERY 1
#endif
#ifndef UELLM_DP_REFIX
#define UELLM_DP_REFIX 1
#endif   // shorter lean ranges are evaluated whole
// fast blocks: the intra-block maxima as a u16 table of input-length window maxima indexed by batch
// length (3 instructions per row to build instead of 5) and the block-end maxima by a shuffle scan
#ifndef UELLM_DP_TRI16
#define UELLM_DP_TRI16 1
#endif
// fast blocks: merged MI groups and the predecessor test in the hull subset (see the chord filter).
// Off: c4 evaluations 34.7 -> 31.8 per query, but the filter's extra work costs more (DP 5.76 -> 5.94 ms)
#ifndef UELLM_DP_HULL2
#define UELLM_DP_HULL2 0
#endif
// fast blocks: the unrolled intra loop stops at checkpoints once no later intra candidate can win
#ifndef UELLM_DP_EXIT
#define UELLM_DP_EXIT 1
#endif
#ifndef UELLM_DP_EXIT_MASK
#define UELLM_DP_EXIT_MASK 0x2AA40000u    // q = 18, 21, 23, 25, 27, 29 (0x11111000u: 12, 16, 20, 24, 28)
#endif
// many-run variants: stage the slow block's SLO range in shared memory for the violation counts
#ifndef UELLM_DP_SLO_STAGE
#define UELLM_DP_SLO_STAGE 1
#endif
// block prefix maxima as one packed u16x2 scan; RSV_SKIP: the run-start scan only when needed
#ifndef UELLM_DP_PACKSCAN
#define UELLM_DP_PACKSCAN 1
#endif
#ifndef UELLM_DP_RSV_SKIP
#define UELLM_DP_RSV_SKIP 0
#endif
// offset of row q of the triangular table (row q holds k = q+1 .. 31)
__host__ __device__ constexpr uint32_t tri_off(int q) { return (uint32_t)(q * 31 - q * (q - 1) / 2); }

__device__ __forceinline__ unsigned long long pack_slot(uint32_t i, uint32_t mo, uint32_t mi)
{
    return (unsigned long long)i | ((unsigned long long)mo << 32) | ((unsigned long long)mi << 48);
}

struct SlotWriter {            // writes a candidate slot with its derived cost terms
    uint32_t t_b, t_it, t_tok, t_pre;
    __device__ __forceinline__ void put(const NarrowSlots &S, uint32_t pos, long long C, uint32_t i, uint32_t mo,
                                        uint32_t mi) const
    {
        S.sl[pos] = make_longlong2(C, (long long)pack_slot(i, mo, mi));
    }
};

// -------------------------------------------------------------------------------------
// Periodic fill of a uniform stretch (exact, step 8).  Inside a run of
// identical records (in, out, slo) the cost of a batch [i, j) depends on j - i only, so the
// recurrence is shift-equivariant: if C[i] = C[i-P] + F for the W boundaries i = j0-W+1 .. j0
// and the elements [j0-W-P+1, j) are identical, then by induction C[j] = C[j-P] + F and
// arg[j] = arg[j-P] + P for every later j up to the end of the stretch (each boundary's W
// candidates and their costs map one to one onto those of j-P, the tie rule is shift-invariant).
// Identical keys never converge in a fix-up (the optimal batch period, e.g. 42 under a KV cap,
// is not a divisor of the tile stride), so without this the cascade re-ran such windows
// sequentially (BJ configs[4], c5).  P is the last batch length (j0 - arg[j0]); any P for which
// the check passes is valid.  Returns the last boundary written (j0 if the check failed).
// Reference args for boundaries at or below s come from the source frame's argx when the
// caller vouches for them (cascade), else from a direct scan of the boundary's W candidates.
// (inlined: out of line, the caller's NarrowSlots would live in local memory -- c4 DP 5.81 -> 7.98 ms)
template <bool FIX>
__device__ __forceinline__ uint32_t periodic_fill(const DPParams &P, const NarrowSlots &S, uint32_t s, uint32_t e,
                                               const long long *__restrict__ src, bool src_args_ok, uint32_t j0,
                                               uint32_t kin, uint32_t kout, uint32_t kslo, bool known_uniform)
{
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t W = P.W;
    const uint32_t lowb = FIX ? s + 1 - 2 * W : s;          // lowest boundary readable through fval
    long long *const outC = FIX ? P.CFx : P.Cx;
    const uint32_t *__restrict__ rin = P.rin;
    const uint32_t *__restrict__ rout = P.rout;
    const uint32_t *__restrict__ rslo = P.rslo;
    // C at boundary b in this run's frame (as in dp_warp_blocked)
    auto fval = [&](uint32_t b) -> long long {
        if (b > s) return __ldcg(outC + b - 1);
        if (FIX) return __ldcg(src + b - 1);
        return 0ll;
    };
    const uint32_t Pp = (uint32_t)__ldcg(reinterpret_cast<const unsigned short *>(P.argx) + j0 - 1);
    if (Pp < 1 || Pp > W || j0 < lowb + W + Pp - 1) return j0;
    const uint32_t lo1 = j0 + 1 - W - Pp;                // boundaries / elements from lo1 on are read
    // elements [lo1, j0) identical to the key (known_uniform: the caller knows [lo1, e) is)
    bool ok = true;
    if (!known_uniform) {
        for (uint32_t q = lo1 + lane; q < j0; q += 32)
            ok &= (__ldg(rin + q) == kin) & (__ldg(rout + q) == kout) & (__ldg(rslo + q) == kslo);
        if (!__all_sync(0xffffffffu, ok)) return j0;
    }
    // C[i] - C[i-P] == F on the W boundaries i = j0-W+1 .. j0
    const long long F = fval(j0) - fval(j0 - Pp);
    for (uint32_t i = j0 + 1 - W + lane; i <= j0; i += 32) ok &= (fval(i) - fval(i - Pp)) == F;
    if (!__all_sync(0xffffffffu, ok)) return j0;
    // reference boundaries r = j0-P+1 .. j0 (slot r - (j0-P) - 1): C and the distance r - arg[r]
    const uint32_t rb = j0 - Pp;
    const unsigned long long cap = P.cap_tok;
    const unsigned long long T_ = P.t_tok * kout + P.t_pre * kin;
    const unsigned long long A_ = P.t_batch + P.t_iter * kout;
    for (uint32_t q = lane; q < Pp; q += 32) {
        const uint32_t r = rb + 1 + q;
        uint32_t dist = 0;
        if (r > s || src_args_ok) dist = (uint32_t)__ldcg(reinterpret_cast<const unsigned short *>(P.argx) + r - 1);
        S.sl[q] = make_longlong2(fval(r), (long long)dist);
    }
    __syncwarp();
    if (!(rb + 1 > s || src_args_ok)) {
        // boundaries r <= s with untrusted args: scan the W candidates i = r-W .. r-1 (ascending,
        // strict '<': the smallest minimising i, R9); the batch [i, r) lies in the stretch
        for (uint32_t r = rb + 1; r <= min(j0, s); ++r) {
            unsigned long long best_hi = ~0ull;
            uint32_t bi = 0xffffffffu;
            for (uint32_t c = lane; c < W; c += 32) {
                const uint32_t b = W - c, i = r - b;          // c ascending -> i ascending
                const bool feas = b == 1 || (unsigned long long)b * ((unsigned long long)kin + kout) <= cap;
                const unsigned long long est = A_ + (unsigned long long)b * T_;
                const unsigned long long pen = ((unsigned long long)kslo < est) ? P.lambda * b : 0ull;
                const unsigned long long tot = (unsigned long long)(fval(i) + (long long)est) + pen;
                if (feas && tot < best_hi) { best_hi = tot; bi = i; }
            }
            const uint32_t h = (uint32_t)(best_hi >> 32);
            const uint32_t mh = __reduce_min_sync(0xffffffffu, h);
            const uint32_t lo = (h == mh) ? (uint32_t)best_hi : 0xffffffffu;
            const uint32_t ml = __reduce_min_sync(0xffffffffu, lo);
            const uint32_t ii = (h == mh && (uint32_t)best_hi == ml) ? bi : 0xffffffffu;
            const uint32_t arg = __reduce_min_sync(0xffffffffu, ii);
            if (lane == 0) S.sl[r - rb - 1].y = (long long)(r - arg);
        }
        __syncwarp();
    }
    // fill j = j0+1 .. while the element j-1 is identical to the key (and j <= e)
    uint32_t j1 = j0;
    for (uint32_t jb = j0; jb < e; jb += 32) {
        const uint32_t j = jb + lane + 1;
        const bool in_t = j <= e;
        const bool uni = in_t && (known_uniform || (__ldg(rin + j - 1) == kin && __ldg(rout + j - 1) == kout &&
                                                    __ldg(rslo + j - 1) == kslo));
        const uint32_t bad = __ballot_sync(0xffffffffu, !uni);
        const uint32_t lim = bad ? jb + (uint32_t)__ffs(bad) - 1 : jb + 32;   // boundaries <= lim
        if (j <= lim) {
            const uint32_t k = (j - j0 + Pp - 1) / Pp;   // j - k*P in (j0-P, j0]
            const longlong2 rv = S.sl[j - k * Pp - rb - 1];
            outC[j - 1] = rv.x + (long long)k * F;
            P.argx[j - 1] = (uint16_t)rv.y;
        }
        j1 = lim;
        if (bad) break;
    }
    __syncwarp();
    return min(j1, e);
}

// -------------------------------------------------------------------------------------
// Blocked fast path (narrow arithmetic).  Positions are processed in blocks of 32 boundaries
// (lane l <-> boundary j0+l+1, element j0+l):
//  1. external candidates (C known before the block, i <= j0): every lane evaluates every live
//     candidate for its own boundary; candidate data is a shared-memory broadcast and the
//     maxima over [i, j) are max(candidate maxima, block prefix maxima) -- no per-step list
//     maintenance;
//  2. intra-block candidates (i in (j0, j)): boundary j0+k+1 for k = 0..31 in order; lane q
//     holds the candidate born at boundary j0+q+1 and folds one element per step; the argmin
//     combines the lane's intra total with the external minimum of boundary k (ties -> the
//     smaller i, which is always the external one);
//  3. once per block the list is extended by the 32 new candidates and pruned at the block-end
//     state (dead prefix + D1), which is valid for every later boundary.
// LAMK: 0 = no SLO penalty, 1 = lambda < 2^32 (32x32 -> 64-bit product), 2 = 64-bit lambda.
template <bool FIX, int LAMK, bool SPLIT, bool VFREE = false>
__device__ DpResult dp_warp_blocked(const DPParams &P, const NarrowSlots &S, uint32_t s, uint32_t e,
                                    const long long *__restrict__ src, uint32_t stop_min, bool src_args_ok,
                                    bool entry_uni)
{
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t lt = lane_lt();
    uint32_t W = P.W;
    uint32_t cap32 = (uint32_t)min(P.cap_tok, 0xffffffffull);
    uint32_t t_b = (uint32_t)P.t_batch, t_it = (uint32_t)P.t_iter, t_tok = (uint32_t)P.t_tok,
             t_pre = (uint32_t)P.t_pre;
    uint32_t lam32 = (uint32_t)P.lambda;
    // keep the cost constants in registers (the compiler would otherwise re-load them from the
    // constant bank inside the candidate loops, one issue slot each)
    asm volatile("" : "+r"(W), "+r"(cap32), "+r"(t_b), "+r"(t_it), "+r"(t_tok), "+r"(t_pre), "+r"(lam32));
    // a single query always satisfies the cap test when the cap exceeds any one query's tokens,
    // so the b > 1 guard can be dropped (2 * 0xffff: narrow-path lengths are < 2^16)
    const bool single_ok = cap32 >= 2u * 0xffffu;
    constexpr bool LAM = LAMK != 0;
    constexpr bool split = SPLIT;
    const unsigned long long lam = P.lambda;
    auto penalty = [&](uint32_t v) -> unsigned long long {
        return LAMK == 1 ? (unsigned long long)lam32 * v : lam * v;
    };
    const SlotWriter SW{t_b, t_it, t_tok, t_pre};
    const uint32_t *__restrict__ rin = P.rin;
    const uint32_t *__restrict__ rout = P.rout;
    const uint32_t *__restrict__ rslo = P.rslo;
    DpResult R;
    R.conv = 0; R.conv_pos = e; R.fix_end = e; R.delta = 0; R.positions = 0; R.evals = 0; R.filled = 0; R.uni = 0;
    if (FIX && entry_uni) {
        // this tile and its predecessor hold one identical record: if the entry state is already
        // periodic the whole tile is a periodic fill (no candidate list at all)
        const uint32_t j1 = periodic_fill<FIX>(P, S, s, e, src, src_args_ok, s, __ldg(P.rin + s), __ldg(P.rout + s),
                                               __ldg(P.rslo + s), true);
        if (j1 >= e) { R.positions = R.filled = e - s; return R; }
    }
    uint32_t L, run_start, prev_slo;
    long long d_run = 0;
    uint32_t run = 0;
    long long *const outC = FIX ? P.CFx : P.Cx;
    // C at boundary b in this run's frame: this run's own output above s; at or below s the source
    // frame (fix-up) or the local start C[s] = 0 (local run).  Boundary b is stored at index b-1.
    auto fval = [&](uint32_t b) -> long long {
        if (b > s) return __ldcg(outC + b - 1);
        if (FIX) return __ldcg(src + b - 1);
        return 0ll;
    };
    // The W candidates i = jb-W+1 .. jb (maxima over elements [i, jb) by suffix max, C from the
    // frame) -- the fix-up's initial list, and the list after a periodic fill.  Returns the run
    // start (largest SLO change position in [jb-W+1, jb)).
    auto init_window = [&](uint32_t jb) -> uint32_t {
        const uint32_t i0 = jb - W + 1;
        uint32_t cmo = 0, cmi = 0, rs = i0;
        for (uint32_t r = 0; r * 32 < W; ++r) {
            const uint32_t off = r * 32 + lane + 1;
            const bool valid = off <= W - 1;
            const uint32_t p = jb - off;
            uint32_t vo = valid ? __ldg(rout + p) : 0, vi = valid ? __ldg(rin + p) : 0;
            const uint32_t vs = valid ? __ldg(rslo + p) : 0;
            const uint32_t vsp = (valid && p > i0) ? __ldg(rslo + p - 1) : vs;
            if (valid && p > i0 && vs != vsp) rs = max(rs, p);
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t to = __shfl_up_sync(0xffffffffu, vo, d), ti = __shfl_up_sync(0xffffffffu, vi, d);
                if ((int)lane >= d) { vo = max(vo, to); vi = max(vi, ti); }
            }
            vo = max(vo, cmo); vi = max(vi, cmi);
            if (valid) SW.put(S, p - i0, fval(p), p, vo, vi);
            cmo = __shfl_sync(0xffffffffu, vo, 31);
            cmi = __shfl_sync(0xffffffffu, vi, 31);
        }
        if (lane == 0) SW.put(S, W - 1, fval(jb), jb, 0, 0);
        return __reduce_max_sync(0xffffffffu, rs);
    };
    if (!FIX) {
        if (lane == 0) SW.put(S, 0, 0, s, 0, 0);
        L = 1;
        run_start = s;
        prev_slo = __ldg(rslo + s);
    } else {
        run_start = init_window(s);
        L = W;
        prev_slo = __ldg(rslo + s - 1);
        d_run = __ldcg(src + s - 1);  // local C at boundary s is 0
        run = 1;
    }
    __syncwarp();
    // Prune slots [0, Lt) at the state of boundary jend: slots below Lold first fold the block
    // maxima (bmo, bmi).  Drops the dead prefix (b > W, KV cap, SLO split) and every candidate
    // dominated (D1) by its successor; survivors are compacted in order.
    // onerun: every candidate and every element up to jend lie in one SLO run of value slo_run
    // (enables the penalty-aware D1, see dominated_by)
    auto prune = [&](uint32_t Lt, uint32_t Lold, uint32_t bmo, uint32_t bmi, uint32_t jend, bool onerun,
                     uint32_t slo_run) {
        uint32_t wr = 0;
        for (uint32_t r = 0; r * 32 < Lt; ++r) {
            const uint32_t k = r * 32 + lane;
            const bool valid = k < Lt;
            longlong2 sv = make_longlong2(0, 0);
            if (valid) sv = S.sl[k];
            const long long cC = sv.x;
            const unsigned long long cp = (unsigned long long)sv.y;
            const uint32_t ci = (uint32_t)cp;
            uint32_t mo = (uint32_t)(cp >> 32) & 0xffffu, mi = (uint32_t)(cp >> 48);
            if (k < Lold) { mo = max(mo, bmo); mi = max(mi, bmi); }
            const uint32_t b = jend - ci;
            const bool dead = !valid | (b > W) | ((b > 1) & (b * (mo + mi) > cap32)) | (split & (ci < run_start));
            // D1 against the successors at list distance 1 and 32 (any later candidate is a valid
            // dominator: strict dominance is transitive and a later candidate outlives an earlier
            // one, so dropping i needs no dominator to be kept).  (n_i - i) * S < W * S <= E < 2^32.
            // Penalty-aware D1 (exact): when the later candidate i' already violates at this state
            // inside one SLO run (slo_run < est(i', jend)), every member of [i, i') violates under
            // est(i', j) <= est(i, j) for every later j -- est only grows and the members' SLOs are
            // slo_run -- so viol(i, j) >= viol(i', j) + (i' - i) and the dominance slope gains
            // lambda per position: i is dead once C[i'] - C[i] < (i' - i) * (S(i', j) + lambda).
            auto dominated_by = [&](uint32_t k2) -> bool {
                const longlong2 nv = S.sl[k2];
                const unsigned long long np = (unsigned long long)nv.y;
                uint32_t nmo = (uint32_t)(np >> 32) & 0xffffu, nmi = (uint32_t)(np >> 48);
                if (k2 < Lold) { nmo = max(nmo, bmo); nmi = max(nmi, bmi); }
                const uint32_t nS = t_tok * nmo + t_pre * nmi;
                const uint32_t gap = (uint32_t)np - ci;
                long long rhs = (long long)(unsigned long long)(gap * nS);
                if (LAM && onerun) {
                    const uint32_t nest = t_b + t_it * nmo + (jend - (uint32_t)np) * nS;
                    if (slo_run < nest) rhs += (long long)penalty(gap);
                }
                return nv.x - cC < rhs;
            };
            bool dominated = false;
            if (!dead) {
// successors tested besides the next one (tools/variant_run.sh on c4, DP ms: {8, 32}: 6.74,
// {32}: 6.57, {16}: 6.59, {64}: 6.67, {8}: 6.69, {}: 6.82, {4, 16}: 6.84, {16, 64}: 6.68; with the
// hull subset of the fast block the list length matters less: {}: 5.93, {32}: 6.06, {64}: 6.10,
// {8}: 6.38)
#ifndef UELLM_D1_D2
#define UELLM_D1_D2 0
#endif
#ifndef UELLM_D1_D3
#define UELLM_D1_D3 0
#endif
                if (k + 1 < Lt) dominated = dominated_by(k + 1);
                if (UELLM_D1_D2 && !dominated && k + UELLM_D1_D2 < Lt) dominated = dominated_by(k + UELLM_D1_D2);
                if (UELLM_D1_D3 && !dominated && k + UELLM_D1_D3 < Lt) dominated = dominated_by(k + UELLM_D1_D3);
            }
            const bool keep = !dead && !dominated;
            __syncwarp();
            const uint32_t bal = __ballot_sync(0xffffffffu, keep);
            if (keep) {
                const uint32_t pos = wr + __popc(bal & lt);
                SW.put(S, pos, cC, ci, mo, mi);
            }
            wr += __popc(bal);
            __syncwarp();
        }
        L = wr;
    };
    if (FIX) prune(L, L, 0, 0, s, false, 0u);   // the W fix-up candidates, pruned before the first block

    uint32_t evals = 0;
    uint32_t nblk = 0;
    bool stop = false;
    uint32_t done = s;
    uint64_t filled = 0;
    // local runs: the tile's first record is the uniform key; blocks equal to it may start a fill
    uint32_t next_try = s + W + 1;                           // earliest block of a fill attempt
    uint32_t kin = 0, kout = 0, kslo = 0;
    bool tile_uni = !FIX;
    if (!FIX) { kin = __ldg(rin + s); kout = __ldg(rout + s); kslo = prev_slo; }
    // records of the next block, loaded one block ahead (the block's own loads were the largest
    // single source of long-scoreboard stalls)
    uint32_t pf_j0 = s, pf_in = 0, pf_out = 0, pf_slo = 0;
    auto prefetch = [&](uint32_t jb) {
        const uint32_t p = jb + lane;
        const bool v = p < e;
        pf_j0 = jb;
        pf_in = v ? __ldg(rin + p) : 0u;
        pf_out = v ? __ldg(rout + p) : 0u;
        pf_slo = v ? __ldg(rslo + p) : 0u;
    };
    prefetch(s);
    for (uint32_t j0 = s; j0 < e && !stop; j0 += 32) {
        const uint32_t B = min(32u, e - j0);
        const bool vl = lane < B;
        const uint32_t x = j0 + lane, jl = x + 1;
        if (!UELLM_DP_PREFETCH || pf_j0 != j0) prefetch(j0);   // (after a periodic fill moved j0)
        const uint32_t in_l = pf_in, out_l = pf_out, slo_l = pf_slo;
        if (UELLM_DP_PREFETCH && j0 + 32 < e) prefetch(j0 + 32);
        if (!FIX && tile_uni) {
            tile_uni = __all_sync(0xffffffffu, !vl || (in_l == kin && out_l == kout && slo_l == kslo));
            if (tile_uni && B == 32 && j0 >= next_try) {
                const uint32_t j1 = periodic_fill<FIX>(P, S, s, e, src, src_args_ok, j0, kin, kout, kslo, false);
                next_try = j0 + 96;                            // (a failed check is retried later)
                if (j1 > j0) {
                    filled += j1 - j0;
                    done = j1;
                    if (j1 >= e) break;
                    // continue the DP at boundary j1 with its W candidates (the fill passed them)
                    run_start = init_window(j1);
                    L = W;
                    prev_slo = kslo;
                    __syncwarp();
                    prune(L, L, 0, 0, j1, false, 0u);
                    if (FIX) { run = 0; d_run = 0; }           // convergence counts restart
                    next_try = j1 + 96;
                    j0 = j1 - 32;                              // (the loop adds 32)
                    continue;
                }
            }
        }
        long long cl_l = 0;
        if (FIX) cl_l = vl ? P.Cx[x] : 0;
        // block prefix maxima of the elements j0..j0+lane and run starts
        uint32_t sprev = __shfl_up_sync(0xffffffffu, slo_l, 1);
        if (lane == 0) sprev = prev_slo;
        uint32_t rsv = (vl && slo_l != sprev) ? x : 0u;
#if UELLM_DP_PACKSCAN
        // (out, in) as one u16x2 word (narrow path: both < 2^16; idle lanes hold 0): one shuffle and
        // one paired max per step; the run-start scan only when a run starts in the block
        uint32_t pk = (out_l << 16) | in_l;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t a = __shfl_up_sync(0xffffffffu, pk, d);
            if ((int)lane >= d) pk = __vmaxu2(pk, a);
        }
        if (!UELLM_DP_RSV_SKIP || __any_sync(0xffffffffu, rsv != 0u)) {
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t c = __shfl_up_sync(0xffffffffu, rsv, d);
                if ((int)lane >= d) rsv = max(rsv, c);
            }
        }
        const uint32_t pmo = pk >> 16, pmi = pk & 0xffffu;
#else
        uint32_t pmo = out_l, pmi = in_l;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t a = __shfl_up_sync(0xffffffffu, pmo, d), b = __shfl_up_sync(0xffffffffu, pmi, d);
            const uint32_t c = __shfl_up_sync(0xffffffffu, rsv, d);
            if ((int)lane >= d) { pmo = max(pmo, a); pmi = max(pmi, b); rsv = max(rsv, c); }
        }
#endif
        const uint32_t rs_l = max(run_start, rsv);
        const uint32_t rs_last = __shfl_sync(0xffffffffu, rs_l, B - 1);
        // An interval [i, j) lies inside one SLO run iff i >= run start of element j-1; only then
        // is viol a single comparison.  Crossing intervals exist in this block only if the oldest
        // external candidate starts before the last run start (external), or a run starts inside
        // the block (intra); those rare blocks take the binary-search variant.
        const bool one_run_ext = (uint32_t)S.sl[0].y >= rs_last;     // every candidate and element in one run
        const bool one_run_intra = rs_last <= j0;                   // every element of the block in one run
        const bool ext_slow = LAM && !split && !one_run_ext;
        const bool intra_slow = LAM && !split && !one_run_intra;
        // ---- 1. external candidates
        unsigned long long lb = ~0ull;
        uint32_t lbi = 0xffffffffu;
        // candidates oldest -> newest; strict '<' keeps the smallest minimising i (R9)
        evals += L * B;
        // In one SLO run the elements ascend in predicted length (sort key), so the max output of
        // any interval ending at the lane's element is that element's own: MO = pmo for every
        // candidate and the lane-constant parts of est are computed once.
        const uint32_t A_l = t_b + t_it * pmo, T_l = t_tok * pmo;
        // violation count of [ci, jl) for the binary-search (several-run) case: from the staged SLO
        // range when this block staged it (many-run variants), else from global memory
        bool staged = false;
        uint32_t ss_base = 0;
        auto vcount = [&](uint32_t ci, unsigned long long est) -> uint32_t {
            return (VFREE && staged) ? viol_count_sm(S.ss, ss_base, ci, jl, est, slo_l)
                                     : viol_count_slow(rslo, ci, jl, est, slo_l);
        };
        auto ext_pass = [&](auto slow_tag, auto single_tag, auto onerun_tag, uint32_t c0, uint32_t c1) {
            constexpr bool SLOW = decltype(slow_tag)::value;
            constexpr bool SINGLE_OK = decltype(single_tag)::value;
            constexpr bool ONERUN = decltype(onerun_tag)::value;
#pragma unroll 2
            for (uint32_t c = c0; c < c1; ++c) {
                const longlong2 sv = S.sl[c];
                const unsigned long long cp = (unsigned long long)sv.y;
                const uint32_t ci = (uint32_t)cp;
                const long long cC = sv.x;
                const uint32_t b = jl - ci;
                const uint32_t mo = ONERUN ? pmo : max((uint32_t)(cp >> 32) & 0xffffu, pmo);
                const uint32_t mi = max((uint32_t)(cp >> 48), pmi);
                const uint32_t est = ONERUN ? A_l + b * (T_l + t_pre * mi)
                                            : t_b + t_it * mo + b * (t_tok * mo + t_pre * mi);
                const bool dead = !vl | (b > W) | ((SINGLE_OK | (b > 1)) & (b * (mo + mi) > cap32)) |
                                  (!ONERUN & split & (ci < rs_l));
                unsigned long long tot = (unsigned long long)cC + est;
                if (LAM) {
                    uint32_t v;
                    if (SLOW) v = (ci >= rs_l) ? ((slo_l < est) ? b : 0u)
                                               : (dead ? 0u : vcount(ci, est));
                    else v = (slo_l < est) ? b : 0u;
                    tot += penalty(v);
                }
                if (!dead && tot < lb) { lb = tot; lbi = ci; }
            }
        };
        // In one SLO run the only deaths are the monotone ones (b > W, KV cap): a candidate alive
        // at the block-end state (b and maxima largest) is alive for every boundary of the block,
        // and the candidates dead there form a prefix of the list.  Only that prefix (Pd slots)
        // needs the feasibility test; the rest take the lean loop.
        auto ext_lean = [&](uint32_t c0, uint32_t c1) {
#pragma unroll 4
            for (uint32_t c = c0; c < c1; ++c) {
                const longlong2 sv = S.sl[c];
                const uint32_t ci = (uint32_t)sv.y;
                const uint32_t b = jl - ci;
                const uint32_t mi = max((uint32_t)((unsigned long long)sv.y >> 48), pmi);
                const uint32_t est = A_l + b * (T_l + t_pre * mi);
                unsigned long long tot = (unsigned long long)sv.x + est;
                if (LAM) tot += penalty((slo_l < est) ? b : 0u);
                if (tot < lb) { lb = tot; lbi = ci; }
            }
        };
        using T1 = std::true_type;
        using F0 = std::false_type;
        // ---- 2. intra-block candidates.  Lane = boundary again: the candidate born at boundary
        //      j0+q+1 (final once lane q has seen every older candidate) is broadcast and every
        //      later lane k evaluates it with the maxima of elements q+1..k, one shared load from a
        //      triangular table M[q][k] of packed (out << 16 | in) maxima built backwards
        //      (M[q][k] = max(M[q+1][k], element q+1)).  Candidates arrive in ascending i, so the
        //      strict '<' keeps the smallest minimising i.
        uint32_t *M = S.tri + 1;                   // S.tri[0] is padding (read by idle lanes)
        const uint32_t pk_l = vl ? ((out_l << 16) | in_l) : 0u;
        // the packed (out << 16 | in) triangular table M[q][k] (k > q): maxima of elements q+1..k
        auto build_tri = [&]() {
            uint32_t m = pk_l;
#pragma unroll
            for (int q = 30; q >= 0; --q) {
                const uint32_t el = __shfl_sync(0xffffffffu, pk_l, q + 1);
                if ((int)lane > q) { m = __vmaxu2(m, el); M[tri_off(q) + lane - q - 1] = m; }
            }
            __syncwarp();
        };
        // block-end maxima of this lane's own candidate (elements lane+1 .. B-1), reused below
        uint32_t mend;
        if (UELLM_DP_TRI16) {
            uint32_t sfx = pk_l;                   // suffix max over lanes lane..31 (lanes >= B hold 0)
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) sfx = __vmaxu2(sfx, __shfl_down_sync(0xffffffffu, sfx, d));
            mend = __shfl_down_sync(0xffffffffu, sfx, 1);
            if (lane + 1 >= B) mend = 0u;
        } else {
            build_tri();
            mend = (lane + 1 < B) ? M[tri_off(lane) + B - 2 - lane] : 0u;
        }
        // Pd = candidates dead at the block end (a prefix); V = candidates that violate the SLO at
        // the block's last boundary (also a prefix in one run: est shrinks with i).  In one run all
        // lanes share the SLO and est grows with the boundary, so candidates >= V violate for no lane.
        uint32_t Pd = 0, V = 0;
        if (one_run_ext) {
            const uint32_t jend = j0 + B;
            const uint32_t bmo = __shfl_sync(0xffffffffu, pmo, B - 1), bmi = __shfl_sync(0xffffffffu, pmi, B - 1);
            const uint32_t slo_run = __shfl_sync(0xffffffffu, slo_l, B - 1);
            const uint32_t A_e = t_b + t_it * bmo, T_e = t_tok * bmo;
            for (uint32_t r = 0; r * 32 < L; ++r) {
                const uint32_t k = r * 32 + lane;
                bool d = false, v = false;
                if (k < L) {
                    const unsigned long long cp = (unsigned long long)S.sl[k].y;
                    const uint32_t ci = (uint32_t)cp, b = jend - ci;
                    const uint32_t mo = max((uint32_t)(cp >> 32) & 0xffffu, bmo), mi = max((uint32_t)(cp >> 48), bmi);
                    d = (b > W) | ((b > 1) & (b * (mo + mi) > cap32));
                    v = LAM && (d || slo_run < A_e + b * (T_e + t_pre * mi));
                }
                const uint32_t bd = __ballot_sync(0xffffffffu, d), bv = __ballot_sync(0xffffffffu, v);
                Pd += __popc(bd);
                V += __popc(bv);
                if (bd != 0xffffffffu && bv != 0xffffffffu) break;   // both are prefixes
            }
        }
        const uint32_t Vs = max(Pd, V);
        // ---- fast block (one SLO run): candidates from Vs on and all intra candidates violate for
        //      no lane, so their costs are C + est with C >= base = C of candidate Vs.  C is
        //      non-decreasing in the boundary (a batch's cost only grows with its members), so when
        //      every such cost lies within 2^32 of base they are compared as 32-bit offsets (one
        //      add, one compare, two selects per candidate); the older candidates [0, Vs) are
        //      evaluated in 64 bits first and merged (they win ties: smaller i).
        bool fast = false;
        long long base = 0;
        if (one_run_ext && one_run_intra && Vs < L) {
            const longlong2 sP = S.sl[Vs];
            base = sP.x;
            const long long cmax = S.sl[L - 1].x;
            const uint32_t bP = jl - (uint32_t)sP.y;
            const uint32_t eP = A_l + bP * (T_l + t_pre * max((uint32_t)((unsigned long long)sP.y >> 48), pmi));
            // eP bounds est of every lean external and every intra candidate of this lane (largest
            // b and maxima); intra C values are bounded by the lane-(B-2) external minimum
            const unsigned long long span = (unsigned long long)(cmax - base) + 2ull * eP;
            const bool ok = !vl || span < 0xfffffff0ull;
            fast = __all_sync(0xffffffffu, ok);
        }
        // u16 table of input-length maxima by batch length d = k - q (fast blocks, TRI16): row d at
        // T16 + 32 d holds max(in[k-d+1 .. k]) for lane k >= d; entry (q, lane) is T16l[-32 q] with
        // T16l = T16 + 33 lane (an immediate offset per step).  Lanes k < d read stale words at most
        // 31 rows below the table, inside the warp's slot array (cap_slots >= 128): masked.
        unsigned short *const T16 = reinterpret_cast<unsigned short *>(S.tri) - 32;
        if (fast && UELLM_DP_TRI16) {
            uint32_t m = vl ? in_l : 0u;
#pragma unroll
            for (int d = 1; d < 32; ++d) {
                T16[d * 32 + lane] = (unsigned short)m;
                m = max(m, __shfl_up_sync(0xffffffffu, in_l, d));
            }
            __syncwarp();
        } else if (UELLM_DP_TRI16) {
            build_tri();
        }
        const unsigned short *const T16l = T16 + 33 * lane;
        if (fast) {
            if (Pd) { if (single_ok) ext_pass(F0{}, T1{}, T1{}, 0, Pd); else ext_pass(F0{}, F0{}, T1{}, 0, Pd); }
            if (Vs > Pd) ext_lean(Pd, Vs);             // may violate: 64-bit with the penalty
            const uint32_t base_lo = (uint32_t)base;
            uint32_t r32 = 0xffffffffu, ri = 0xffffffffu;
            // Lower-hull subset of the lean candidates [Vs, L) (exact).  Inside one SLO run every
            // candidate of a group with one stored MI (the maxima up to the block start) has the
            // same MI = max(mi, pmi) and MO = pmo at every boundary of the block, so its cost is
            // (C_i - i*K) + const with one slope K per (group, lane): the minimum over the group is
            // attained on the lower convex hull of its points (i, C_i).  A candidate k lying on or
            // above the chord of two other members a < k < c is never the SMALLEST minimiser (if it
            // minimised, equality would make a minimise too), so dropping every such k keeps the
            // minimum and the smallest minimising i (R9); the chord of the list neighbours
            // removes almost all non-vertices in one pass.  C offsets from base fit 32 bits
            // (checked above) and |dC| * di < 2^45.
            uint32_t H = 0xffffffffu;
            if (L - Vs >= kHullMin) {
                H = 0;
                // HULL2: (i) candidates whose stored MI is at most the block's first element's prefix
                // maximum pmi0 have MI = pmi_l at every lane: one group (key max(mi, pmi0));
                // (ii) a candidate whose list predecessor (same group, lean) is strictly cheaper at the
                // block's largest slope Kmax = t_tok*bmo + t_pre*max(g, bmi) is strictly worse for every
                // lane (K_l <= Kmax and cost_a - cost_k = C_a - C_k + (k - a) K_l): dropped for this
                // block.  The smallest minimiser of any lane is a hull vertex not beaten by its
                // predecessor, so it survives both tests.
                const uint32_t pmi0 = UELLM_DP_HULL2 ? __shfl_sync(0xffffffffu, pmi, 0) : 0u;
                const uint32_t hbmo = __shfl_sync(0xffffffffu, pmo, B - 1), hbmi = __shfl_sync(0xffffffffu, pmi, B - 1);
                for (uint32_t r0 = Vs; r0 < L; r0 += 32) {
                    const uint32_t k = r0 + lane;
                    bool keep = false;
                    uint2 ent = make_uint2(0u, 0u);
                    if (k < L) {
                        const longlong2 sv = S.sl[k];
                        const uint32_t ck = (uint32_t)sv.x - base_lo, ik = (uint32_t)sv.y;
                        const uint32_t mk = (uint32_t)((unsigned long long)sv.y >> 48);
                        const uint32_t gk = max(mk, pmi0);
                        keep = true;
                        if (k > Vs) {
                            const longlong2 sa = S.sl[k - 1];
                            const uint32_t ga = max((uint32_t)((unsigned long long)sa.y >> 48), pmi0);
                            const long long ca = (long long)((uint32_t)sa.x - base_lo);
                            const uint32_t ia = (uint32_t)sa.y;
                            if (UELLM_DP_HULL2 && ga == gk) {
                                const unsigned long long Kmax = (unsigned long long)t_tok * hbmo +
                                                                (unsigned long long)t_pre * max(gk, hbmi);
                                if ((long long)ck - ca > (long long)((unsigned long long)(ik - ia) * Kmax)) keep = false;
                            }
                            if (keep && k + 1 < L) {
                                const longlong2 sc = S.sl[k + 1];
                                if (ga == gk && max((uint32_t)((unsigned long long)sc.y >> 48), pmi0) == gk) {
                                    const long long cc = (long long)((uint32_t)sc.x - base_lo);
                                    const uint32_t ic = (uint32_t)sc.y;
                                    keep = ((long long)ck - ca) * (long long)(ic - ia) < (cc - ca) * (long long)(ik - ia);
                                }
                            }
                        }
                        ent = make_uint2(ck, (j0 - ik) | (mk << 16));
                    }
                    const uint32_t bal = __ballot_sync(0xffffffffu, keep);
                    const uint32_t pos = H + __popc(bal & lt);
                    if (keep && pos < kHullCap) S.hl[pos] = ent;
                    H += __popc(bal);
                }
                __syncwarp();
                if (H > kHullCap) H = 0xffffffffu;
            }
            if (H != 0xffffffffu) {
                const uint32_t lp1 = lane + 1;           // b = jl - i = lane + 1 + (j0 - i)
                uint32_t rd = 0;
                evals -= (L - Vs - H) * B;           // evaluations actually run
#pragma unroll (kExtUnroll)
                for (uint32_t c = 0; c < H; ++c) {
                    const uint2 he = S.hl[c];
                    const uint32_t b = lp1 + (he.y & 0xffffu);
                    const uint32_t mi = max(he.y >> 16, pmi);
                    const uint32_t tot = he.x + A_l + b * (T_l + t_pre * mi);
                    if (tot < r32) { r32 = tot; rd = he.y; }
                }
                if (r32 != 0xffffffffu) ri = j0 - (rd & 0xffffu);
            } else {
#pragma unroll (kExtUnroll)
                for (uint32_t c = Vs; c < L; ++c) {
                    const longlong2 sv = S.sl[c];
                    const uint32_t ci = (uint32_t)sv.y;
                    const uint32_t b = jl - ci;
                    const uint32_t mi = max((uint32_t)((unsigned long long)sv.y >> 48), pmi);
                    const uint32_t tot = ((uint32_t)sv.x - base_lo) + A_l + b * (T_l + t_pre * mi);
                    if (tot < r32) { r32 = tot; ri = ci; }
                }
            }
            // the older candidates (win ties) were evaluated in 64 bits: lb >= C(jl) >= base
            if (lb <= (unsigned long long)base + r32) { r32 = (uint32_t)(lb - (unsigned long long)base); ri = lbi; }
            // intra candidates in 32-bit offsets: dead prefix q < Qd checked, the rest lean
            bool dend = false;
            if (lane + 1 < B) {
                const uint32_t be = B - 1 - lane, mo_e = mend >> 16, mi_e = mend & 0xffffu;
                dend = (be > W) | ((be > 1) & (be * (mo_e + mi_e) > cap32));
            }
            const uint32_t Qd = __popc(__ballot_sync(0xffffffffu, dend));
            int off = (int)lane - 1;                 // M[tri_off(q) + lane - q - 1], M[-1] is padding
            for (uint32_t q = 0; q < Qd; ++q) {
                const uint32_t Cq = __shfl_sync(0xffffffffu, r32, q);
                const uint32_t b = lane - q;
                const uint32_t mi = UELLM_DP_TRI16 ? (uint32_t)T16l[-32 * (int)q] : M[off] & 0xffffu;
                off += 30 - (int)q;
                const uint32_t tot = Cq + A_l + b * (T_l + t_pre * mi);
                const bool dead = (lane <= q) | (b > W) | ((single_ok | (b > 1)) & (b * (pmo + mi) > cap32));
                if (!dead && tot < r32) { r32 = tot; ri = j0 + 1 + q; }
            }
            if (Qd == 0 && B == 32) {
                // the common case, fully unrolled: q is a compile-time constant, so the table
                // entry of (q, lane) is M[lane + tri_off(q) - q - 1] -- an immediate offset from
                // the lane's base, no address arithmetic per step
                const uint32_t *Ml = M + (int)lane;
                const uint32_t j0p1 = j0 + 1;
                // lower bound of any intra candidate q' >= q for this lane: C[q'] >= C[q] (C is
                // non-decreasing in the boundary), b >= 1 and the maxima include the lane's element
                const uint32_t LB_l = A_l + T_l + t_pre * in_l;
                // EXIT == 2: C also grows by at least t_tok*out[e] + t_pre*in[e] per element e
                // between two boundaries (adding e to the last batch raises its est by at least that
                // much and never lowers its violations), so C[q'] >= C[q] + (q' - q) * dblk with dblk
                // the block's smallest such increment, and the bound of lane k over q' in [q, k)
                // becomes C[q] + LB_k + (k - q - 1) * dblk.  (A 32-bit wrap of a bound only lowers
                // it: the test stays conservative.)
                const uint32_t dblk = UELLM_DP_EXIT == 2 ? __reduce_min_sync(0xffffffffu, t_tok * out_l + t_pre * in_l) : 0u;
#pragma unroll
                for (int q = 0; q < 31; ++q) {
                    const uint32_t Cq = __shfl_sync(0xffffffffu, r32, q);
                    // checkpoints q = 18, 21, 23, 25, 27, 29: the cheapest set under the exit-step
                    // distribution of a sequential C model on c3 data (mean first exact exit 21.5)
                    if (UELLM_DP_EXIT && ((UELLM_DP_EXIT_MASK >> q) & 1u)) {
                        // every later lane already at or below that bound: no later intra candidate
                        // can win (ties keep the smaller, current i)
                        const uint32_t bnd = Cq + LB_l + (UELLM_DP_EXIT == 2 ? (lane - (uint32_t)q - 1u) * dblk : 0u);
                        if (__all_sync(0xffffffffu, lane <= (uint32_t)q || r32 <= bnd)) {
                            // (diagnostics: the pairs (q', k) with q' >= q were not evaluated)
                            evals -= (uint32_t)((31 - q) * (32 - q) / 2);
                            break;
                        }
                    }
                    const uint32_t b = lane - (uint32_t)q;
                    const uint32_t mi = UELLM_DP_TRI16 ? (uint32_t)T16l[-32 * q] : Ml[(int)tri_off(q) - q - 1] & 0xffffu;
                    const uint32_t tot = Cq + A_l + b * (T_l + t_pre * mi);
                    if (lane > (uint32_t)q && tot < r32) { r32 = tot; ri = j0p1 + (uint32_t)q; }
                }
            } else {
#pragma unroll 4
                for (uint32_t q = Qd; q + 1 < B; ++q) {
                    const uint32_t Cq = __shfl_sync(0xffffffffu, r32, q);
                    const uint32_t b = lane - q;
                    const uint32_t mi = UELLM_DP_TRI16 ? (uint32_t)T16l[-32 * (int)q] : M[off] & 0xffffu;
                    off += 30 - (int)q;
                    const uint32_t tot = Cq + A_l + b * (T_l + t_pre * mi);
                    if (lane > q && tot < r32) { r32 = tot; ri = j0 + 1 + q; }
                }
            }
            lb = (unsigned long long)base + r32;
            lbi = ri;
        } else {
            // Violation-free block (only computed here, off the fast block's path): records ascend in
            // slo_us inside a window, so the smallest SLO of any interval this block evaluates is that
            // of the oldest live candidate i0, and est is largest for [i0, block end); when even that
            // SLO is not below that est, nothing violates for any lane and the one-comparison
            // violation test (0 here) replaces the binary-search count.
            bool vfree = false;
            if (VFREE && (ext_slow || intra_slow)) {
                const unsigned long long cp0 = (unsigned long long)S.sl[0].y;
                const uint32_t i0 = (uint32_t)cp0;
                const uint32_t bmo_ = __shfl_sync(0xffffffffu, pmo, B - 1), bmi_ = __shfl_sync(0xffffffffu, pmi, B - 1);
                const unsigned long long mo = max((uint32_t)(cp0 >> 32) & 0xffffu, bmo_);
                const unsigned long long mi = max((uint32_t)(cp0 >> 48), bmi_);
                const unsigned long long emax = (unsigned long long)t_b + (unsigned long long)t_it * mo +
                                                (unsigned long long)(j0 + B - i0) *
                                                    ((unsigned long long)t_tok * mo + (unsigned long long)t_pre * mi);
                vfree = (unsigned long long)__ldg(rslo + i0) >= emax;
            }
            if (VFREE && S.ss && !vfree && (ext_slow || intra_slow)) {
                // stage slo[oldest candidate .. block end) (b <= W after the last prune: <= W + 32)
                const uint32_t lo = (uint32_t)S.sl[0].y, len = j0 + B - lo;
                if (len <= (P.W + 64u + 31u & ~31u)) {
                    for (uint32_t k = lane; k < len; k += 32) S.ss[k] = __ldg(rslo + lo + k);
                    __syncwarp();
                    staged = true;
                    ss_base = lo;
                }
            }
            if (ext_slow && !vfree) {
                if (single_ok) ext_pass(T1{}, T1{}, F0{}, 0, L); else ext_pass(T1{}, F0{}, F0{}, 0, L);
            } else if (one_run_ext) {
                if (single_ok) ext_pass(F0{}, T1{}, T1{}, 0, Pd); else ext_pass(F0{}, F0{}, T1{}, 0, Pd);
                ext_lean(Pd, L);
            } else {
                if (single_ok) ext_pass(F0{}, T1{}, F0{}, 0, L); else ext_pass(F0{}, F0{}, F0{}, 0, L);
            }
            // steps q in [q0, q1); the table offset of (q, lane) advances by 30 - q per step
            auto intra_pass = [&](auto slow_tag, auto single_tag, auto onerun_tag, auto check_tag, uint32_t q0,
                                  uint32_t q1) {
                constexpr bool SLOW = decltype(slow_tag)::value;
                constexpr bool SINGLE_OK = decltype(single_tag)::value;
                constexpr bool ONERUN = decltype(onerun_tag)::value;
                constexpr bool CHECK = decltype(check_tag)::value;
                uint32_t off = tri_off((int)q0) + lane - q0 - 1;
    #pragma unroll 2
                for (uint32_t q = q0; q < q1; ++q) {
                    const long long Cq = (long long)__shfl_sync(0xffffffffu, lb, q);
                    const bool act = lane > q;
                    const uint32_t b = lane - q;                     // boundary jl minus candidate j0+1+q
                    const uint32_t m = act ? M[off] : 0u;
                    off += 30 - q;
                    const uint32_t mo = ONERUN ? pmo : m >> 16, mi = m & 0xffffu;
                    const uint32_t ci = j0 + 1 + q;
                    const uint32_t est = ONERUN ? A_l + b * (T_l + t_pre * mi)
                                                : t_b + t_it * mo + b * (t_tok * mo + t_pre * mi);
                    unsigned long long tot = (unsigned long long)Cq + est;
                    if (!CHECK) {                                    // alive at the block end: alive here
                        if (LAM) tot += penalty((slo_l < est) ? b : 0u);
                        if (act && tot < lb) { lb = tot; lbi = ci; }
                        continue;
                    }
                    const bool dead = !act | (b > W) | ((SINGLE_OK | (b > 1)) & (b * (mo + mi) > cap32)) |
                                      (!ONERUN & split & (ci < rs_l));
                    if (LAM) {
                        uint32_t v;
                        if (SLOW) v = (ci >= rs_l) ? ((slo_l < est) ? b : 0u)
                                                   : (dead ? 0u : vcount(ci, est));
                        else v = (slo_l < est) ? b : 0u;
                        tot += penalty(v);
                    }
                    if (!dead && tot < lb) { lb = tot; lbi = ci; }
                }
            };
            const uint32_t QB = B - 1;                   // intra candidates q = 0 .. B-2
            if (intra_slow && !vfree) {
                if (single_ok) intra_pass(T1{}, T1{}, F0{}, T1{}, 0, QB); else intra_pass(T1{}, F0{}, F0{}, T1{}, 0, QB);
            } else if (one_run_intra) {
                // deaths inside one run are monotone (b > W, KV cap): candidates dead at the block end
                // form a prefix q < Qd; the rest need no feasibility test
                bool dend = false;
                if (lane + 1 < B) {
                    const uint32_t be = B - 1 - lane, mo_e = mend >> 16, mi_e = mend & 0xffffu;
                    dend = (be > W) | ((be > 1) & (be * (mo_e + mi_e) > cap32));
                }
                const uint32_t Qd = __popc(__ballot_sync(0xffffffffu, dend));
                if (Qd) {
                    if (single_ok) intra_pass(F0{}, T1{}, T1{}, T1{}, 0, Qd); else intra_pass(F0{}, F0{}, T1{}, T1{}, 0, Qd);
                }
                intra_pass(F0{}, F0{}, T1{}, F0{}, Qd, QB);
            } else {
                if (single_ok) intra_pass(F0{}, T1{}, F0{}, T1{}, 0, QB); else intra_pass(F0{}, F0{}, F0{}, T1{}, 0, QB);
            }
        }
        const long long o_C = (long long)lb;
        const long long iC = o_C;
        const uint32_t o_A = jl - lbi;
        uint32_t kdone = B;
        if (FIX) {
            // convergence: first boundary ending a run of W equal differences C_fix - C_local
            const long long dk = o_C - cl_l;
            long long dprev = __shfl_up_sync(0xffffffffu, dk, 1);
            if (lane == 0) dprev = d_run;
            const uint32_t brk = __ballot_sync(0xffffffffu, vl && dk != dprev);
            const uint32_t upto = brk & (lane == 31 ? 0xffffffffu : ((2u << lane) - 1));
            const uint32_t runk = upto ? lane - (31 - __clz(upto)) + 1 : run + lane + 1;
            const uint32_t cv = __ballot_sync(0xffffffffu, vl && runk >= W && jl >= stop_min);
            if (cv) {
                const uint32_t c = __ffs(cv) - 1;
                R.conv = 1; R.conv_pos = j0 + c + 1; R.fix_end = R.conv_pos;
                R.delta = __shfl_sync(0xffffffffu, dk, c);
                stop = true;
                kdone = c + 1;
            } else {
                d_run = __shfl_sync(0xffffffffu, dk, B - 1);
                run = __shfl_sync(0xffffffffu, runk, B - 1);
            }
        }
        // outputs of this block
        if (lane < kdone) {
            (FIX ? P.CFx : P.Cx)[x] = o_C;
            P.argx[x] = (uint16_t)o_A;
        }
        done = j0 + kdone;
        if (stop) break;
        // maxima of the block's own candidates over [i, block end): elements q+1 .. B-1
        const uint32_t imo = mend >> 16, imi = mend & 0xffffu;
        // ---- 3. extend the list by the block's candidates and prune at the block-end state
        const uint32_t jend = j0 + B;
        const uint32_t bmo = __shfl_sync(0xffffffffu, pmo, B - 1), bmi = __shfl_sync(0xffffffffu, pmi, B - 1);
        run_start = __shfl_sync(0xffffffffu, rs_l, B - 1);
        prev_slo = __shfl_sync(0xffffffffu, slo_l, B - 1);
        if (vl) SW.put(S, L + lane, iC, j0 + 1 + lane, imo, imi);
        evals += B * (B - 1) / 2;
        __syncwarp();
        // Pruning is optional (any subset of what D1 allows is exact); folding the block maxima into
        // the older slots is not.  With UELLM_DP_PRUNE_EVERY = 2 every other block only folds and
        // appends (the list then holds at most W + 1 + 2 * 32 candidates, see cap_slots).
        if (UELLM_DP_PRUNE_EVERY == 1 || (++nblk % UELLM_DP_PRUNE_EVERY) == 0 || L + 2 * B > P.cap_slots) {
            prune(L + B, L, bmo, bmi, jend, one_run_ext && one_run_intra, prev_slo);
        } else {
            for (uint32_t k = lane; k < L; k += 32) {
                const unsigned long long cp = (unsigned long long)S.sl[k].y;
                const uint32_t mo = max((uint32_t)(cp >> 32) & 0xffffu, bmo), mi = max((uint32_t)(cp >> 48), bmi);
                S.sl[k].y = (long long)pack_slot((uint32_t)cp, mo, mi);
            }
            L += B;
            __syncwarp();
        }
    }
    R.positions = done - s;
    R.evals = evals;
    R.filled = filled;
    R.uni = tile_uni && done >= e ? 1u : 0u;
    if (!R.conv) { R.conv_pos = e; R.fix_end = e; }
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

// shared memory per warp: narrow = 16 B slots + the 496-word triangular max table; wide = 20 B slots
constexpr uint32_t kRmqBytes = 500 * 4;            // 1 pad word + 496 + 3, keeps 16-byte alignment
// many-run variants (7, 8): the SLO values of a slow block's candidate range [oldest candidate,
// block end) -- at most W + 32 positions -- staged per warp, so each violation count is a binary
// search in shared memory instead of up to 9 dependent global loads (c5's anti-sorted segment)
static __host__ __device__ __forceinline__ uint32_t slo_stage_cap(const DPParams &P)
{
    return (P.narrow && P.many_runs && P.W <= 480u && UELLM_DP_SLO_STAGE) ? ((P.W + 64u + 31u) & ~31u) : 0u;
}
static __host__ __device__ __forceinline__ uint32_t warp_smem_bytes(const DPParams &P)
{
    return P.narrow ? P.cap_slots * 16 + kRmqBytes + kHullCap * 8 + slo_stage_cap(P) * 4 : P.cap_slots * 20;
}

// Variant V of the SEG-DP kernels, fixed on the host (one instantiation per kernel keeps the code
// the SMs fetch small: with every variant behind a runtime switch the kernel was 60 K SASS
// instructions and 10 % of the warp samples were "no instruction"):
//   V = 0: generic 64-bit path;  V = 1 + LK + 3 * SPLIT: narrow blocked path (LK: lambda kind).
template <bool FIX, int V>
__device__ DpResult dp_run(const DPParams &P, char *smem, int warp, uint32_t s, uint32_t e,
                           const long long *src, uint32_t stop_min, bool src_args_ok, bool entry_uni = false)
{
    if constexpr (V == 0) {
        DpResult R = dp_warp<FIX>(P, slots_for(smem, P.cap_slots, warp), s, e, src, stop_min);
        R.filled = 0; R.uni = 0;
        return R;
    } else {
        // V = 1 + LK + 3 * SPLIT (1 .. 6); V = 6 + LK (7, 8): lambda > 0, no split, many SLO runs
        constexpr int LK = V >= 7 ? V - 6 : (V - 1) % 3;
        constexpr bool SPLIT = V >= 7 ? false : (V - 1) / 3 != 0;
        constexpr bool VF = V >= 7;
        char *p = smem + (size_t)warp * warp_smem_bytes(P);
        NarrowSlots S;
        S.sl = (longlong2 *)p;
        S.tri = (uint32_t *)(p + (size_t)P.cap_slots * 16);
        S.hl = (uint2 *)(p + (size_t)P.cap_slots * 16 + kRmqBytes);
        S.ss = (VF && slo_stage_cap(P)) ? (uint32_t *)(p + (size_t)P.cap_slots * 16 + kRmqBytes + kHullCap * 8) : nullptr;
        return dp_warp_blocked<FIX, LK, SPLIT, VF>(P, S, s, e, src, stop_min, src_args_ok, entry_uni);
    }
}

// Variants 7 / 8 add the violation-free block test for inputs with many SLO runs (more distinct
// SLO values than the rank-compressed sort key takes, e.g. BJ c5's anti-sorted segment): there
// most blocks span several runs and would count violations by binary search.  A separate
// instantiation, because the extra code in the same kernel cost the one-run fast block of c4
// 0.11 ms (register allocation / instruction footprint), while c5 gains 0.39 ms.
static int dp_variant(const DPParams &P)
{
    if (!P.narrow) return 0;
    const int lk = P.lambda == 0 ? 0 : (P.lambda < (1ull << 32) ? 1 : 2);
    if (lk && !P.split && P.many_runs && UELLM_DP_VFREE) return 6 + lk;
    return 1 + lk + 3 * (P.split ? 1 : 0);
}

// Tile t (> first of its window) and its predecessor each hold one repeated record and the two
// records agree: [s_{t-1}, e_t) is one uniform stretch (enables the fix-up's entry fill).
__device__ __forceinline__ bool entry_uniform(const DPParams &P, uint64_t t, uint32_t s)
{
    const TileRec &a = P.tiles[t], &b = P.tiles[t - 1];
    return a.uni && b.uni && __ldg(P.rin + s - 1) == __ldg(P.rin + s) && __ldg(P.rout + s - 1) == __ldg(P.rout + s) &&
           __ldg(P.rslo + s - 1) == __ldg(P.rslo + s);
}

// Local run and fix-up fused in one persistent kernel.  Warps first claim local runs in tile
// order from one counter; a finished local run is published (flag[t], release).  Once the local
// runs are all claimed, warps claim fix-ups in tile order from a second counter; the fix-up of
// tile t waits (acquire) for tile t-1's flag and runs from t-1's local values.  Every claimed
// local run belongs to a running warp that sets its flag before claiming anything else, so the
// waits always end; the fix-ups fill the SMs as the local runs drain instead of a second,
// tail-bound launch.
#ifndef UELLM_DP_MINB
#define UELLM_DP_MINB 3     // 78 registers, no spills, 24 warps per SM (DP 6.53 vs 6.57 ms at 4)
#endif
template <int V>
__global__ void __launch_bounds__(kDpWarpsPerCta * 32, UELLM_DP_MINB) k_dp_tiles(DPParams P, uint64_t ntiles)
{
    extern __shared__ __align__(16) char smem[];
    const uint32_t lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    uint32_t *counter = P.tflags + ntiles;          // [0] local runs, [1] fix-ups
    unsigned long long evals = 0;
    for (;;) {
        uint32_t t = 0;
        if (lane == 0) t = atomicAdd(counter, 1u);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= ntiles) break;
        uint32_t s, e, k, w; bool valid;
        tile_bounds(P, t, s, e, k, w, valid);
        if (!valid) {
            if (lane == 0) { TileRec r = {}; r.valid = 0; P.tiles[t] = r; }
            __syncwarp();
            __threadfence();
            if (lane == 0) st_release(P.tflags + t, 1u);
            continue;
        }
        DpResult R = dp_run<false, V>(P, smem, warp, s, e, nullptr, 0, false);
        evals += R.evals;
        if (lane == 0 && R.filled) atomicAdd(&P.diag->dp_filled, (unsigned long long)R.filled);
        if (lane == 0) {
            TileRec r = {};
            r.s = s; r.e = e; r.valid = 1;
            r.conv = (k == 0); r.conv_pos = s; r.fix_end = s;
            r.uni = R.uni;
            P.tiles[t] = r;
        }
        __syncwarp();
        __threadfence();
        if (lane == 0) st_release(P.tflags + t, 1u);
    }
    for (;;) {
        uint32_t t = 0;
        if (lane == 0) t = atomicAdd(counter + 1, 1u);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= ntiles) break;
        uint32_t s, e, k, w; bool valid;
        tile_bounds(P, t, s, e, k, w, valid);
        if (!valid || k == 0) continue;
        if (lane == 0) {
            while (ld_relaxed(P.tflags + t - 1) == 0u) __nanosleep(128);
            while (ld_relaxed(P.tflags + t) == 0u) __nanosleep(128);
            asm volatile("fence.acq_rel.gpu;" ::: "memory");     // acquire: pairs with st.release
        }
        __syncwarp();
        __threadfence();
        const bool eu = entry_uniform(P, t, s);
        DpResult F = dp_run<true, V>(P, smem, warp, s, e, P.Cx, 0, false, eu);
        evals += F.evals;
        if (lane == 0 && F.filled) atomicAdd(&P.diag->dp_filled, (unsigned long long)F.filled);
        if (lane == 0) {
            TileRec &r = P.tiles[t];
            r.conv = F.conv; r.conv_pos = F.conv_pos; r.fix_end = F.fix_end; r.delta = F.delta;
            atomicAdd(&P.diag->fixup_positions, (unsigned long long)F.positions);
            if (!F.conv) atomicAdd(&P.diag->fixups_unconverged, 1ull);
        }
    }
    if (lane == 0 && evals) atomicAdd(&P.diag->dp_evals, evals);
}

// Periodic reference of the fix frame CFx at boundary s (the start of a tile inside a uniform
// stretch whose predecessor starts at s_prev): Pp = s - arg[s] (the last batch) when
// C[i] - C[i-Pp] = F on the W boundaries (s-W, s] and every boundary read lies in (s_prev, s]
// (the predecessor's fix frame, true args); 0 if the check fails.  Warp-collective.
__device__ uint32_t periodic_ref(const DPParams &P, uint32_t s, uint32_t s_prev, long long &F)
{
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t W = P.W;
    const uint32_t Pp = (uint32_t)__ldcg(reinterpret_cast<const unsigned short *>(P.argx) + s - 1);
    if (Pp < 1 || Pp > W || s < s_prev + W + Pp) return 0;
    F = __ldcg(P.CFx + s - 1) - __ldcg(P.CFx + s - Pp - 1);
    bool ok = true;
    for (uint32_t i = s + 1 - W + lane; i <= s; i += 32)
        ok &= (__ldcg(P.CFx + i - 1) - __ldcg(P.CFx + i - Pp - 1)) == F;
    return __all_sync(0xffffffffu, ok) ? Pp : 0u;
}

// Writes boundaries j in (a, b] of the fix frame from the periodic reference (ref_s - Pp, ref_s]:
// j - m*Pp lands in the reference for m = ceil((j - ref_s) / Pp).
__device__ __forceinline__ void fill_from_ref(const DPParams &P, uint32_t a, uint32_t b, uint32_t ref_s, uint32_t Pp,
                                              long long F, uint32_t tid, uint32_t nthr)
{
    for (uint32_t j = a + 1 + tid; j <= b; j += nthr) {
        const uint32_t m = (j - ref_s + Pp - 1) / Pp;
        const uint32_t src = j - m * Pp;
        P.CFx[j - 1] = __ldcg(P.CFx + src - 1) + (long long)m * F;
        P.argx[j - 1] = __ldcg(reinterpret_cast<const unsigned short *>(P.argx) + src - 1);
    }
}

// The tiles the cascade deferred (fill_P != 0), written in parallel: one CTA per tile.
__global__ void __launch_bounds__(256) k_dp_fill(DPParams P, uint64_t ntiles)
{
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const TileRec &r = P.tiles[t];
        if (!r.valid || r.fill_P == 0) continue;
        fill_from_ref(P, r.s, r.e, r.fill_s, r.fill_P, r.fill_F, threadIdx.x, blockDim.x);
        if (threadIdx.x == 0) atomicAdd(&P.diag->dp_filled, (unsigned long long)(r.e - r.s));
    }
}

// One warp per window: resolve tiles whose predecessor did not converge, compute the frame
// offsets of every tile and the window's optimal cost C[w1].
// Second fix-up round, in parallel (speculative).  A tile whose predecessor's fix-up did not
// converge has a fix-up computed from the wrong (local) frame; the cascade would re-run it from the
// predecessor's fix frame, one tile after another.  Here every such tile whose pre-predecessor
// converged in round 1 is re-run from the predecessor's round-1 fix frame in parallel, into side
// arrays (round 1's values stay intact).  The cascade adopts a re-run (copies it in) only when it
// did not touch the predecessor itself -- then the frame the re-run read is the one the cascade
// would read.  Eligibility reads round-1 states only, and an eligible tile's predecessor is never
// eligible, so no re-run reads what another writes.  Uniform stretches stay with the cascade.
template <int V>
__global__ void __launch_bounds__(kDpWarpsPerCta * 32, UELLM_DP_MINB) k_dp_refix(DPParams P, uint64_t ntiles)
{
    extern __shared__ __align__(16) char smem[];
    const uint32_t lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t t = (uint64_t)blockIdx.x * (blockDim.x >> 5) + warp; t < ntiles; t += nw) {
        uint32_t s, e, k, w; bool valid;
        tile_bounds(P, t, s, e, k, w, valid);
        if (!valid || k < 2) continue;
        const TileRec &a = P.tiles[t - 2], &b = P.tiles[t - 1];
        if (b.conv || !a.conv || !b.valid) continue;
        if (entry_uniform(P, t, s)) continue;                  // uniform stretches: the cascade's deferral
        TileRec r = P.tiles[t];
        DPParams Q = P;                   // outputs to the side arrays: round 1's values stay intact
        Q.CFx = P.Crf;
        Q.argx = P.Arf;
        DpResult R = dp_run<true, V>(Q, smem, warp, r.s, r.e, P.CFx, r.fix_end, true, false);
        if (lane == 0) {
            TileRec &q = P.tiles[t];
            q.rf_conv = R.conv; q.rf_conv_pos = R.conv_pos; q.rf_fix_end = max(R.fix_end, r.fix_end);
            q.rf_delta = R.delta;
            q.refixed = 1;
            atomicAdd(&P.diag->fixup_positions, (unsigned long long)R.positions);
            atomicAdd(&P.diag->dp_evals, (unsigned long long)R.evals);
            if (R.filled) atomicAdd(&P.diag->dp_filled, (unsigned long long)R.filled);
        }
        __syncwarp();
    }
}

#ifndef UELLM_CASCADE_STAGE
#define UELLM_CASCADE_STAGE 1
#endif
template <int V>
__global__ void k_dp_cascade(DPParams P)
{
    extern __shared__ __align__(16) char smem[];
    __shared__ TileRec srec[32];
    const uint32_t w = blockIdx.x;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t t0 = (uint64_t)w * P.tpw;
    // valid tiles form a prefix of the window's tpw slots: count them 32 at a time, and check
    // whether every fix-up converged (the common case: then the frame offsets are a prefix sum
    // of the deltas, computed warp-parallel instead of walking the tiles one by one)
    uint32_t K = 0;
    for (uint32_t k0 = 0; k0 < P.tpw; k0 += 32) {
        const uint32_t k = k0 + lane;
        const bool v = k < P.tpw && P.tiles[t0 + k].valid;
        const uint32_t bv = __ballot_sync(0xffffffffu, v);
        K += __popc(bv);
        if (bv != 0xffffffffu) break;
    }
    if (K == 0) return;
    // every fix-up converged except possibly the window's LAST tile's (it has no successor to meet:
    // its fix-up runs to the window end in the exact frame of its predecessor) -- the common case
    bool allconv = true;
    for (uint32_t k0 = 0; k0 + 1 < K; k0 += 32) {
        const uint32_t k = k0 + lane;
        const bool nc = k >= 1 && k + 1 < K && !P.tiles[t0 + k].conv;
        if (__any_sync(0xffffffffu, nc)) { allconv = false; break; }
    }
    if (allconv) {
        long long carry = 0;                                    // off_local of the previous tile
        for (uint32_t k0 = 0; k0 < K; k0 += 32) {
            const uint32_t k = k0 + lane;
            const long long d = (k >= 1 && k < K) ? P.tiles[t0 + k].delta : 0ll;
            long long inc = d;                                  // inclusive warp scan of deltas
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const long long y = __shfl_up_sync(0xffffffffu, inc, o);
                if ((int)lane >= o) inc += y;
            }
            if (k < K) {
                // (an unconverged last tile has delta 0: off_fix = its predecessor's off_local)
                const bool lc = k == 0 || P.tiles[t0 + k].conv;
                P.tiles[t0 + k].off_fix = k ? carry + inc - d : 0ll;
                P.tiles[t0 + k].off_local = (k && lc) ? carry + inc : 0ll;
            }
            carry += __shfl_sync(0xffffffffu, inc, 31);
        }
        __syncwarp();
        if (lane == 0) {
            const TileRec &r = P.tiles[t0 + K - 1];
            long long c;
            if (K == 1) c = P.Cx[r.e - 1];
            else c = r.conv ? P.Cx[r.e - 1] + r.off_local : P.CFx[r.e - 1] + r.off_fix;
            P.wincost[w] = (unsigned long long)c;
        }
        return;
    }
    // tile 0 is exact in its local frame
    long long tail_off = 0;          // offset of the frame holding tile (k-1)'s tail values
    bool tail_local = true;          // tail in Cx (local frame) vs CFx (fix-up frame)
    // Deferred periodic fill of uniform stretches (DESIGN.md "SEG-DP" step 8): once tile k-1's
    // fix frame is periodic at the start of tile k (C[i] = C[i-Pp] + F on the W boundaries up to
    // s_k, uniform elements behind them), every later boundary of the same uniform stretch is
    // C[j] = C[j - m*Pp] + m*F, arg[j] = arg[j - m*Pp] + m*Pp (periodic_fill's induction), so the
    // tiles of the stretch only record that reference here and k_dp_fill writes them in
    // parallel afterwards; a re-run that leaves the stretch first gets its predecessor's tail.
    uint32_t ref_s = 0, ref_P = 0;   // active reference: boundaries (ref_s - ref_P, ref_s] of CFx
    long long ref_F = 0;
    if (lane == 0) { P.tiles[t0].off_local = 0; P.tiles[t0].off_fix = 0; }
    uint32_t eu_mask = 0;            // entry_uniform of tiles (k & ~31) + lane, 32 at a time
    bool prev_touched = false;       // the cascade changed tile k-1's fix frame (re-run / adopted / deferred)
    for (uint32_t k = 1; k < K; ++k) {
        bool touched = false;
        if (k == 1 || (k & 31u) == 0) {
            const uint32_t kk = (k & ~31u) + lane;
            bool e = false;
            if (kk >= 1 && kk < K) {
                uint32_t ts, te, tk, tw; bool tv;
                tile_bounds(P, t0 + kk, ts, te, tk, tw, tv);
                e = tv && entry_uniform(P, t0 + kk, ts);
                // the chunk's records, one per lane: the walk below reads tile k's record from shared
                // memory instead of a dependent global load per tile (only the walk writes them, tile
                // k at step k, so the staged copy of a later tile is current when the walk reaches it)
                if (UELLM_CASCADE_STAGE) srec[lane] = P.tiles[t0 + kk];
            }
            eu_mask = __ballot_sync(0xffffffffu, e);
            __syncwarp();
        }
        const bool eu = (eu_mask >> (k & 31u)) & 1u;
        if (V != 0 && !tail_local && eu && ref_P != 0) {
            // further tiles of the deferred stretch: only the record fields change (no reads), and
            // every tile of the run of entry-uniform tiles from k to the end of this 32-tile chunk
            // takes the same fields -- one lane per tile
            const uint32_t sh = k & 31u;
            const uint32_t run = (uint32_t)__ffs(~(eu_mask >> sh)) - 1u;     // set bits from bit sh
            uint32_t cnt = (run == 0xffffffffu || sh + run > 32u) ? 32u - sh : run;
            if (k + cnt > K) cnt = K - k;
            if (lane < cnt) {
                uint32_t ts, te, tk, tw; bool tv;
                tile_bounds(P, t0 + k + lane, ts, te, tk, tw, tv);
                TileRec &q = P.tiles[t0 + k + lane];
                q.fill_s = ref_s; q.fill_P = ref_P; q.fill_F = ref_F;
                q.conv = 0; q.fix_end = te; q.off_fix = tail_off; q.off_local = 0;
            }
            __syncwarp();
            prev_touched = true;
            k += cnt - 1;                                // (the loop adds 1)
            continue;
        }
        TileRec r = UELLM_CASCADE_STAGE ? srec[k & 31u] : P.tiles[t0 + k];
        r.fill_s = 0; r.fill_P = 0; r.fill_F = 0;
        if (!tail_local) {
            bool deferred = false;
            if (V != 0 && eu) {
                if (ref_P == 0) {
                    ref_P = periodic_ref(P, r.s, P.tiles[t0 + k - 1].s, ref_F);
                    ref_s = r.s;
                }
                deferred = ref_P != 0;
            } else if (ref_P) {
                // leaving the stretch: materialise the last 2W boundaries of the deferred predecessor
                const TileRec &q = P.tiles[t0 + k - 1];
                fill_from_ref(P, max(q.s, q.e > 2 * P.W ? q.e - 2 * P.W : 0u), q.e, ref_s, ref_P, ref_F, lane, 32);
                __syncwarp();
                __threadfence_block();
                ref_P = 0; ref_s = 0;
            }
            if (deferred) {
                r.fill_s = ref_s; r.fill_P = ref_P; r.fill_F = ref_F;
                r.conv = 0; r.fix_end = r.e;
                touched = true;
            } else if (r.refixed && !prev_touched) {
                // k_dp_refix already re-ran it from the predecessor's round-1 fix frame, which the
                // cascade left untouched: adopt the side arrays' values and results
                for (uint32_t j = r.s + 1 + lane; j <= r.rf_fix_end; j += 32) {
                    P.CFx[j - 1] = __ldcg(P.Crf + j - 1);
                    P.argx[j - 1] = __ldcg(reinterpret_cast<const unsigned short *>(P.Arf) + j - 1);
                }
                __syncwarp();
                r.conv = r.rf_conv; r.conv_pos = r.rf_conv_pos; r.fix_end = max(r.rf_fix_end, r.fix_end);
                r.delta = r.rf_delta;
                touched = true;
            } else {
                DpResult R = dp_run<true, V>(P, smem, 0, r.s, r.e, P.CFx, r.fix_end, true, eu);
                r.conv = R.conv; r.conv_pos = R.conv_pos; r.fix_end = max(R.fix_end, r.fix_end); r.delta = R.delta;
                touched = true;
                if (lane == 0) {
                    atomicAdd(&P.diag->cascade_reruns, 1ull);
                    atomicAdd(&P.diag->fixup_positions, (unsigned long long)R.positions);
                    atomicAdd(&P.diag->dp_evals, (unsigned long long)R.evals);
                    if (R.filled) atomicAdd(&P.diag->dp_filled, (unsigned long long)R.filled);
                }
            }
        } else {
            ref_P = 0; ref_s = 0;
        }
        r.off_fix = tail_off;
        if (r.conv) { r.off_local = tail_off + r.delta; tail_off = r.off_local; tail_local = true; }
        else { r.off_local = 0; tail_local = false; }
        if (lane == 0) P.tiles[t0 + k] = r;
        __syncwarp();
        prev_touched = touched;
    }
    if (ref_P) {            // the window ends inside a deferred stretch: its last value is needed now
        const TileRec &q = P.tiles[t0 + K - 1];
        fill_from_ref(P, q.e - 1, q.e, ref_s, ref_P, ref_F, lane, 32);
        __syncwarp();
        __threadfence_block();
    }
    if (lane == 0) {
        const TileRec &r = P.tiles[t0 + K - 1];
        long long c;
        if (K == 1) c = P.Cx[r.e - 1];
        else c = r.conv ? P.Cx[r.e - 1] + r.off_local : P.CFx[r.e - 1] + r.off_fix;
        P.wincost[w] = (unsigned long long)c;
    }
}

static uint32_t warps_per_cta(uint32_t per)
{
    uint32_t wpc = kDpWarpsPerCta;
    while (wpc > 1 && wpc * per > 200 * 1024) --wpc;
    return wpc;
}

template <int V>
static cudaError_t launch_segdp(const DPParams &P, uint64_t ntiles, cudaStream_t st, void *const ev[3], int *launches)
{
    const uint32_t per = warp_smem_bytes(P);
    const uint32_t wpc = warps_per_cta(per);
    const size_t smem = (size_t)wpc * per;
    const size_t smem1 = (size_t)per;
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(k_dp_tiles<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem))) return e;
    if ((e = cudaFuncSetAttribute(k_dp_cascade<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1))) return e;
    int dev = 0, nsm = 0, per_sm = 0;
    if ((e = cudaGetDevice(&dev))) return e;
    if ((e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev))) return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dp_tiles<V>, (int)(wpc * 32), smem))) return e;
    if (per_sm < 1) per_sm = 1;
    const uint64_t want = ceil_div(ntiles, wpc);
    const uint64_t cap = (uint64_t)nsm * (uint64_t)per_sm;
    const unsigned blocks = (unsigned)(want < cap ? want : cap);
    if ((e = cudaMemsetAsync(P.tflags, 0, 4 * (ntiles + 2), st))) return e;
    k_dp_tiles<V><<<blocks, wpc * 32, smem, st>>>(P, ntiles);
    ++*launches;
    if (ev[0]) cudaEventRecord((cudaEvent_t)ev[0], st);
    if (UELLM_DP_REFIX && V != 0) {
        if ((e = cudaFuncSetAttribute(k_dp_refix<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem))) return e;
        k_dp_refix<V><<<blocks, wpc * 32, smem, st>>>(P, ntiles);
        ++*launches;
    }
    if (ev[1]) cudaEventRecord((cudaEvent_t)ev[1], st);
    k_dp_cascade<V><<<P.nwin, 32, smem1, st>>>(P);
    ++*launches;
    if (V != 0) {           // deferred uniform tiles (none: every CTA exits after reading the records)
        k_dp_fill<<<(unsigned)(ntiles < (uint64_t)nsm * 8 ? ntiles : (uint64_t)nsm * 8), 256, 0, st>>>(P, ntiles);
        ++*launches;
    }
    if (ev[2]) cudaEventRecord((cudaEvent_t)ev[2], st);
    return cudaGetLastError();
}

cudaError_t run_segdp(const DPParams &P, uint64_t ntiles, cudaStream_t st, void *const ev[3], int *launches)
{
    *launches = 0;
    if (P.n == 0 || ntiles == 0) return cudaSuccess;
    switch (dp_variant(P)) {
    case 0: return launch_segdp<0>(P, ntiles, st, ev, launches);
    case 1: return launch_segdp<1>(P, ntiles, st, ev, launches);
    case 2: return launch_segdp<2>(P, ntiles, st, ev, launches);
    case 3: return launch_segdp<3>(P, ntiles, st, ev, launches);
    case 4: return launch_segdp<4>(P, ntiles, st, ev, launches);
    case 5: return launch_segdp<5>(P, ntiles, st, ev, launches);
    case 6: return launch_segdp<6>(P, ntiles, st, ev, launches);
    case 7: return launch_segdp<7>(P, ntiles, st, ev, launches);
    default: return launch_segdp<8>(P, ntiles, st, ev, launches);
    }
}

}  // namespace uellm
