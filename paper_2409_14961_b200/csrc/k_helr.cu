// k_helr.cu -- NEXT f3: the HELR deployer (Sec. 4.3, Alg. 2, Eq. 4-6
// P:305-324; R21) as a level-synchronous bitmask DP on the GPU.
//
// With the greedy layer fill along the chain, the layers device j takes when it is appended
// after the visited set P depend only on P (x_j = min(max(0, L - sum_{d in P} cap_d), cap_j)),
// so one Held-Karp table dp[S][j] (visited set S, last device j) serves every subset of Alg. 2's
// outer loop at once:
//     dp[{j}][j] = cost(j, min(L, cap_j))
//     dp[S][j]   = min_{i in S\{j}} (dp[S\{j}][i] + Latency[i][j]) + cost(j, x_j)
// cost(j, x) = ((p * x) * m) / Performance(j), m = M / L; every operation is an explicitly
// rounded double op in the oracle's order (no contraction), so values are bit-identical.
//
//   k_helr_caps     thread per mask: capsum[S] = sum of cap over S
//   k_helr_level    one launch per popcount k: thread per (k-subset rank, member j); the subset
//                   is unranked in the combinatorial number system, the member is the q-th set bit
//   k_helr_reduce   CTA-wise lexicographic min of (a1*dp + a2*|S|/|D|, dp, S, j) over feasible S
//   k_helr_final    one CTA: min of the CTA minima, chain decode through the back-pointers,
//                   greedy layer ranges -> uellm_device_map
#include "internal.cuh"

namespace uellm {

namespace {

struct Key {
    double obj, lat;
    uint32_t S, j;
};

__device__ __forceinline__ bool key_less(const Key &a, const Key &b)
{
    if (a.obj != b.obj) return a.obj < b.obj;
    if (a.lat != b.lat) return a.lat < b.lat;
    if (a.S != b.S) return a.S < b.S;
    return a.j < b.j;
}

__device__ __forceinline__ double cost_of(const HelrParams &H, uint32_t j, uint32_t x)
{
    return __ddiv_rn(__dmul_rn(__dmul_rn(H.p, (double)x), H.m), H.perf[j]);
}

__device__ __forceinline__ uint32_t layers_after(const HelrParams &H, uint32_t P, uint32_t j)
{
    const unsigned long long cs = H.capsum[P];
    const unsigned long long rem = cs >= H.L ? 0ull : H.L - cs;
    return rem < H.cap[j] ? (uint32_t)rem : H.cap[j];
}

}  // namespace

__global__ void k_helr_caps(HelrParams H)
{
    const uint64_t NS = 1ull << H.D;
    for (uint64_t S = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; S < NS; S += (uint64_t)gridDim.x * blockDim.x) {
        unsigned long long c = 0;
        for (uint32_t d = 0; d < H.D; ++d)
            if ((S >> d) & 1ull) c += H.cap[d];
        H.capsum[S] = c;
    }
}

__global__ void __launch_bounds__(256) k_helr_level(HelrParams H, uint32_t k, unsigned long long count)
{
    __shared__ double lat[kHelrMaxDevices * kHelrMaxDevices];
    const uint32_t D = H.D;
    for (uint32_t e = threadIdx.x; e < D * D; e += blockDim.x) lat[e] = H.lat[e];
    __syncthreads();
    const unsigned long long total = count * k;
    for (unsigned long long g = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; g < total;
         g += (unsigned long long)gridDim.x * blockDim.x) {
        // unrank: the (g / k)-th k-subset in colex order
        unsigned long long r = g / k;
        const uint32_t q = (uint32_t)(g % k);
        uint32_t S = 0, kk = k;
        for (int pos = (int)D - 1; pos >= 0 && kk > 0; --pos) {
            const unsigned long long c = H.binom[pos * (kHelrMaxDevices + 1) + kk];
            if (r >= c) { S |= 1u << pos; r -= c; --kk; }
        }
        // member j = q-th set bit of S (ascending)
        uint32_t t = S;
        for (uint32_t i = 0; i < q; ++i) t &= t - 1;
        const uint32_t j = __ffs(t) - 1;
        const uint32_t P = S & ~(1u << j);
        const double cj = cost_of(H, j, layers_after(H, P, j));
        double best;
        uint32_t bi = 0xffu;
        if (P == 0) {
            best = cj;
        } else {
            best = __longlong_as_double(0x7ff0000000000000ll);   // +inf
            for (uint32_t m = P; m; m &= m - 1) {                 // i ascending: smallest wins ties
                const uint32_t i = __ffs(m) - 1;
                const double v = __dadd_rn(__dadd_rn(H.dp[(uint64_t)P * D + i], lat[i * D + j]), cj);
                if (v < best) { best = v; bi = i; }
            }
        }
        H.dp[(uint64_t)S * D + j] = best;
        H.arg[(uint64_t)S * D + j] = (uint8_t)bi;
    }
}

__global__ void __launch_bounds__(256) k_helr_reduce(HelrParams H)
{
    __shared__ Key sk[256];
    const uint32_t D = H.D;
    const unsigned long long total = (1ull << D) * D;
    Key best;
    best.obj = best.lat = __longlong_as_double(0x7ff0000000000000ll);
    best.S = 0xffffffffu;
    best.j = 0xffffffffu;
    for (unsigned long long g = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; g < total;
         g += (unsigned long long)gridDim.x * blockDim.x) {
        const uint32_t S = (uint32_t)(g / D), j = (uint32_t)(g % D);
        if (S == 0 || !((S >> j) & 1u) || H.capsum[S] < H.L) continue;     // Eq. 4
        Key c;
        c.lat = H.dp[g];
        const double size = __ddiv_rn((double)__popc(S), (double)D);
        c.obj = __dadd_rn(__dmul_rn(H.a1, c.lat), __dmul_rn(H.a2, size));
        c.S = S;
        c.j = j;
        if (key_less(c, best)) best = c;
    }
    sk[threadIdx.x] = best;
    __syncthreads();
    for (int s = 128; s; s >>= 1) {
        if ((int)threadIdx.x < s && key_less(sk[threadIdx.x + s], sk[threadIdx.x])) sk[threadIdx.x] = sk[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        H.part_obj[blockIdx.x] = sk[0].obj;
        H.part_lat[blockIdx.x] = sk[0].lat;
        H.part_sj[blockIdx.x] = ((unsigned long long)sk[0].S << 32) | sk[0].j;
    }
}

__global__ void __launch_bounds__(256) k_helr_final(HelrParams H, uint32_t nparts)
{
    __shared__ Key sk[256];
    Key best;
    best.obj = best.lat = __longlong_as_double(0x7ff0000000000000ll);
    best.S = 0xffffffffu;
    best.j = 0xffffffffu;
    for (uint32_t b = threadIdx.x; b < nparts; b += blockDim.x) {
        Key c;
        c.obj = H.part_obj[b];
        c.lat = H.part_lat[b];
        c.S = (uint32_t)(H.part_sj[b] >> 32);
        c.j = (uint32_t)H.part_sj[b];
        if (key_less(c, best)) best = c;
    }
    sk[threadIdx.x] = best;
    __syncthreads();
    for (int s = 128; s; s >>= 1) {
        if ((int)threadIdx.x < s && key_less(sk[threadIdx.x + s], sk[threadIdx.x])) sk[threadIdx.x] = sk[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x != 0) return;
    best = sk[0];
    uellm_device_map M;
    for (int t = 0; t < 32; ++t) { M.device[t] = 0; M.layer_begin[t] = 0; M.layer_count[t] = 0; }
    M.count = 0; M.feasible = 0; M.mask = 0; M.pad = 0; M.objective = 0.0; M.latency_s = 0.0;
    if (best.S != 0xffffffffu) {
        const uint32_t D = H.D;
        uint32_t chain[kHelrMaxDevices], k = 0, S = best.S, j = best.j;
        while (S) {
            chain[k++] = j;
            const uint32_t i = H.arg[(uint64_t)S * D + j];
            S &= ~(1u << j);
            j = i;
        }
        unsigned long long used = 0;
        for (uint32_t t = 0; t < k; ++t) {                  // visit order = reverse of the walk
            const uint32_t d = chain[k - 1 - t];
            const unsigned long long rem = used >= H.L ? 0ull : H.L - used;
            const uint32_t x = rem < H.cap[d] ? (uint32_t)rem : H.cap[d];
            M.device[t] = d;
            M.layer_begin[t] = (uint32_t)(used < H.L ? used : H.L);
            M.layer_count[t] = x;
            used += H.cap[d];
        }
        M.count = k; M.feasible = 1; M.mask = best.S;
        M.objective = best.obj; M.latency_s = best.lat;
    }
    *H.out = M;
}

// BGS, the paper's baseline deployer: devices by descending memory (ties:
// smaller id), each takes max_layers until the layers are exhausted.  One thread: |D| <= 20.
__global__ void k_bgs(HelrParams H)
{
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const uint32_t D = H.D;
    uint32_t ord[kHelrMaxDevices];
    for (uint32_t d = 0; d < D; ++d) ord[d] = d;
    for (uint32_t a = 1; a < D; ++a) {
        const uint32_t x = ord[a];
        uint32_t b = a;
        while (b > 0 && H.mem[ord[b - 1]] < H.mem[x]) { ord[b] = ord[b - 1]; --b; }
        ord[b] = x;
    }
    uellm_device_map M;
    for (int t = 0; t < 32; ++t) { M.device[t] = 0; M.layer_begin[t] = 0; M.layer_count[t] = 0; }
    M.count = 0; M.feasible = 0; M.mask = 0; M.pad = 0; M.objective = 0.0; M.latency_s = 0.0;
    unsigned long long used = 0;
    uint32_t k = 0, mask = 0;
    double l = 0.0;
    while (used < H.L && k < D) {
        const uint32_t d = ord[k];
        const uint32_t cap = H.cap[d];
        const unsigned long long rem = H.L - used;
        const uint32_t x = rem < cap ? (uint32_t)rem : cap;
        const double c = cost_of(H, d, x);
        l = k == 0 ? c : __dadd_rn(__dadd_rn(l, H.lat[ord[k - 1] * D + d]), c);
        M.device[k] = d; M.layer_begin[k] = (uint32_t)used; M.layer_count[k] = x;
        used += cap;
        mask |= 1u << d;
        ++k;
    }
    if (used >= H.L) {
        M.count = k; M.feasible = 1; M.mask = mask; M.latency_s = l;
        M.objective = __dadd_rn(__dmul_rn(H.a1, l), __dmul_rn(H.a2, __ddiv_rn((double)k, (double)D)));
    } else {
        for (int t = 0; t < 32; ++t) { M.device[t] = 0; M.layer_begin[t] = 0; M.layer_count[t] = 0; }
    }
    *H.out = M;
}

cudaError_t run_bgs(const HelrParams &H, cudaStream_t st)
{
    k_bgs<<<1, 32, 0, st>>>(H);
    return cudaGetLastError();
}

cudaError_t run_helr(const HelrParams &H, cudaStream_t st, int *launches)
{
    const uint64_t NS = 1ull << H.D;
    int l = 0;
    const uint64_t cb = ceil_div(NS, 256);
    k_helr_caps<<<(unsigned)(cb < 148 * 8 ? cb : 148 * 8), 256, 0, st>>>(H);
    ++l;
    for (uint32_t k = 1; k <= H.D; ++k) {
        const unsigned long long cnt = H.binom_host[H.D * (kHelrMaxDevices + 1) + k];
        const uint64_t nb = ceil_div(cnt * k, 256);
        k_helr_level<<<(unsigned)(nb < 148 * 16 ? nb : 148 * 16), 256, 0, st>>>(H, k, cnt);
        ++l;
    }
    k_helr_reduce<<<kHelrParts, 256, 0, st>>>(H);
    k_helr_final<<<1, 256, 0, st>>>(H, kHelrParts);
    l += 2;
    if (launches) *launches = l;
    return cudaGetLastError();
}

}  // namespace uellm
