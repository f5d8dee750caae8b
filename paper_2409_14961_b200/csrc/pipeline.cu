// pipeline.cu -- end-to-end scheduling of HOST-resident queries with the PCIe copies overlapped
// with the GPU work (uellm_schedule_pipelined).  Windows are independent (R15, O1), so the job
// is cut into groups of whole windows; group g's host->device copy runs on a copy stream while
// group g-1 is loaded / scheduled / summarised on the caller's stream, and group g-1's results
// go back on a second copy stream.  Host code (stream/event orchestration) plus one tiny kernel.
//
//   H stream : H2D(g+1) into input staging slot (g+1)%2   [waits: compute of g-1 done]
//   C stream : load(g) (sync: host decisions need its maxima) -> schedule(g) -> stats(g)
//              -> rebase order/offsets to global indices      [waits: H2D(g), D2H(g-2) done]
//   D stream : D2H(g) of order, offsets, totals                [waits: compute of g done]
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "internal.cuh"

namespace uellm {

__global__ void k_add_base(uint32_t *a, uint64_t n, uint32_t base)
{
    const uint64_t nt = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += nt) a[k] += base;
}

static cudaError_t add_base(uint32_t *a, uint64_t n, uint32_t base, cudaStream_t st)
{
    if (n == 0 || base == 0) return cudaSuccess;
    const uint64_t nb = ceil_div(n, 256 * 4);
    k_add_base<<<(unsigned)(nb < 148 * 8 ? nb : 148 * 8), 256, 0, st>>>(a, n, base);
    return cudaGetLastError();
}

constexpr uint64_t kPipeMaxGroups = 64;

struct PipeLayout {
    uint64_t group_q;                 // queries of the largest group (whole windows)
    uint64_t groups;
    uint64_t wl, nwin, tail;          // group g = windows [start[g], start[g+1])
    uint64_t start[kPipeMaxGroups + 1];
    uint64_t ws[2], ws_bytes;         // scheduling workspaces of the two compute lanes
    uint64_t in[3], out[3], slo[3];   // input staging slots (g % 3)
    uint64_t order[3], offs[3];       // output staging slots (g % 3)
    uint64_t tot, nb;                 // per-group totals / num_batches (device)
    uint64_t tail_groups;             // the tapered last groups
    uint64_t total;
};
#ifndef UELLM_PIPE_TAIL_AUTO
#define UELLM_PIPE_TAIL_AUTO 1        // tail groups: automatic (one-wave) DP tiles
#endif

static PipeLayout pipe_layout(uint64_t n, const uellm_config &cfg, uint32_t groups)
{
    PipeLayout P;
    std::memset(&P, 0, sizeof P);
    const uint64_t wl = cfg.window ? (cfg.window < n ? cfg.window : n) : n;
    const uint64_t nwin = n ? ceil_div(n, wl ? wl : 1) : 0;
    uint64_t G = groups ? groups : 12;
    if (G > kPipeMaxGroups) G = kPipeMaxGroups;
    if (G > nwin) G = nwin ? nwin : 1;
    // The pipeline is bound by the host->device copies; once the last copy lands, the groups still
    // computing (two compute lanes) and the last device->host copy are exposed.  So the last groups
    // taper -- about 1/2, 1/4, 1/8 of an even share (at least one window each) -- and the rest
    // split evenly: little GPU work is left when the copies end.
    P.wl = wl; P.nwin = nwin;
    const uint64_t share = G ? nwin / G : 0;
    uint64_t K = G > 1 ? (G - 1 < 3 ? G - 1 : 3) : 0;
    uint64_t tsz[3] = {0, 0, 0}, tail = 0;
    for (uint64_t k = 0; k < K; ++k) {
        tsz[k] = share >> (k + 1);
        if (tsz[k] < 1) tsz[k] = 1;
        tail += tsz[k];
    }
    if (tail + (G - K) > nwin) { K = 0; tail = 0; }   // too few windows to taper
    P.tail = tail;
    const uint64_t body = nwin - tail, nb = G - K;
    uint64_t w = 0;
    for (uint64_t g = 0; g < nb; ++g) {
        P.start[g] = w;
        w += body / nb + (g < body % nb ? 1 : 0);
    }
    for (uint64_t k = 0; k < K; ++k) {
        P.start[nb + k] = w;
        w += tsz[k];
    }
    P.start[G] = nwin;
    uint64_t maxw = 0;
    for (uint64_t g = 0; g < G; ++g) maxw = P.start[g + 1] - P.start[g] > maxw ? P.start[g + 1] - P.start[g] : maxw;
    P.group_q = n ? maxw * wl : 0;
    if (P.group_q > n) P.group_q = n;
    P.groups = n ? G : 0;
    uint64_t off = 0;
    auto take = [&](uint64_t bytes) { uint64_t o = off; off = align_up(off + (bytes ? bytes : 1), 256); return o; };
    uellm_config c = cfg;
    c.window = (uint32_t)wl;
    // the body groups share the GPU (throughput-bound): no one-wave short tiles; the tapered tail
    // groups are exposed after the last copy (latency-bound): the automatic tile choice
    const bool auto_tile = !c.dp_tile;
    if (auto_tile) c.dp_tile = tile_len_throughput(P.group_q, c.max_batch ? c.max_batch : 1);
    P.ws_bytes = make_layout(P.group_q, c).total;
    if (auto_tile && UELLM_PIPE_TAIL_AUTO) {
        uellm_config ct = c;
        ct.dp_tile = 0;
        for (uint64_t g = G - K; g < G; ++g) {
            const uint64_t q = (P.start[g + 1] - P.start[g]) * wl;
            const uint64_t b = make_layout(q < n ? q : n, ct).total;
            if (b > P.ws_bytes) P.ws_bytes = b;
        }
    }
    P.tail_groups = K;
    P.ws[0] = take(P.ws_bytes);
    P.ws[1] = take(P.ws_bytes);
    const uint64_t q = P.group_q ? P.group_q : 1;
    for (int s = 0; s < 3; ++s) { P.in[s] = take(4 * q); P.out[s] = take(4 * q); P.slo[s] = take(4 * q); }
    for (int s = 0; s < 3; ++s) { P.order[s] = take(4 * q); P.offs[s] = take(4 * (q + 1)); }
    P.tot = take(sizeof(uellm_totals) * (P.groups ? P.groups : 1));
    P.nb = take(8 * (P.groups ? P.groups : 1));
    P.total = off;
    return P;
}

// first window of group g (g = groups gives nwin)
static uint64_t gwin(const PipeLayout &P, uint64_t g)
{
    if (P.groups <= 1) return g ? P.nwin : 0;
    return g >= P.groups ? P.nwin : P.start[g];
}

}  // namespace uellm

using namespace uellm;

namespace {
// Streams and events of uellm_schedule_pipelined, created on a device's first call and reused by
// every later call on it (held for the process lifetime): the per-call creation and destruction of
// 3 streams and 3 x groups events is gone from the call.  Calls on one device serialise on its
// pool's mutex (they share the copy streams).
struct PipePool {
    std::mutex mu;
    bool ready = false;
    cudaStream_t H = nullptr, D = nullptr, C2 = nullptr;
    cudaEvent_t start = nullptr;
    cudaEvent_t ev[3][kPipeMaxGroups] = {};     // h2d, done, d2h per group
    bool timing = false;
    cudaError_t init(bool with_timing)
    {
        if (ready && timing == with_timing) return cudaSuccess;
        cudaError_t e;
        if (!ready) {
            if ((e = cudaStreamCreateWithFlags(&H, cudaStreamNonBlocking))) return e;
            if ((e = cudaStreamCreateWithFlags(&D, cudaStreamNonBlocking))) return e;
            if ((e = cudaStreamCreateWithFlags(&C2, cudaStreamNonBlocking))) return e;
        } else {
                for (auto &row : ev) for (auto &x : row) cudaEventDestroy(x);
        }
        const unsigned fl = with_timing ? cudaEventDefault : cudaEventDisableTiming;
        if ((e = cudaEventCreateWithFlags(&start, fl))) return e;
        for (auto &row : ev)
            for (auto &x : row) if ((e = cudaEventCreateWithFlags(&x, fl))) return e;
        timing = with_timing;
        ready = true;
        return cudaSuccess;
    }
};
constexpr int kPoolDevices = 64;
PipePool g_pools[kPoolDevices];
}  // namespace

extern "C" {

size_t uellm_pipeline_workspace_bytes(uint64_t n, const uellm_config *cfg, uint32_t groups)
{
    if (!cfg) return 0;
    return (size_t)pipe_layout(n, *cfg, groups).total;
}

uellm_status uellm_schedule_pipelined(const uellm_queries *q, const uellm_config *cfg, uint32_t groups, void *ws,
                                      size_t ws_bytes, uint32_t *order, uint32_t *batch_offsets,
                                      uint64_t *num_batches, uellm_totals *totals, void *stream)
{
    uellm::NvtxRange nvtx_("uellm_schedule_pipelined");
    if (!q || !cfg || !order || !batch_offsets || !num_batches || !totals) return UELLM_ERR_ARG;
    const uint64_t n = q->n;
    if (n >= 0xffffffffull) return UELLM_ERR_ARG;
    if (n > 0 && (!q->input_len || !q->pred_out_len || !q->slo_s)) return UELLM_ERR_ARG;
    const PipeLayout PL = pipe_layout(n, *cfg, groups);
    if (!ws || (reinterpret_cast<uintptr_t>(ws) & 255) || ws_bytes < PL.total) return UELLM_ERR_ARG;
    uint8_t *w = (uint8_t *)ws;
    cudaStream_t C = (cudaStream_t)stream;
    if (n == 0) {
        // the single-call path handles the empty job (no copies to overlap)
        uellm_profile p;
        uellm_status s = uellm_profile_load(q, cfg, w + PL.ws[0], PL.ws_bytes, stream, &p);
        if (s != UELLM_OK) return s;
        if ((s = uellm_schedule_batches(&p, cfg, order, batch_offsets, num_batches, stream)) != UELLM_OK) return s;
        return uellm_batch_stats(&p, cfg, batch_offsets, num_batches, nullptr, totals, stream);
    }
    const uint64_t G = PL.groups;
    uellm_config gcfg = *cfg;
    gcfg.window = (uint32_t)(cfg->window ? (cfg->window < n ? cfg->window : n) : n);
    uellm_config tcfg = gcfg;                                  // the tapered tail groups' config
    if (!gcfg.dp_tile) gcfg.dp_tile = tile_len_throughput(PL.group_q, gcfg.max_batch ? gcfg.max_batch : 1);
    if (!UELLM_PIPE_TAIL_AUTO || cfg->dp_tile) tcfg = gcfg;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kPoolDevices) return UELLM_ERR_CUDA;
    PipePool &pool = g_pools[dev];
    std::lock_guard<std::mutex> pool_lock(pool.mu);
    cudaStream_t H = nullptr, D = nullptr, C2 = nullptr;
    cudaEvent_t *h2d = pool.ev[0], *done = pool.ev[1], *d2h = pool.ev[2];
    std::vector<uint64_t> m(G, 0);
    std::vector<uellm_totals> tot_host(G);
    uellm_status status = UELLM_OK;
    auto qa = [&](uint64_t g) { const uint64_t q = gwin(PL, g) * PL.wl; return q < n ? q : n; };
    auto qz = [&](uint64_t g) { return qa(g + 1); };
#define PCU(x)                                   \
    do {                                         \
        if ((x) != cudaSuccess) {                \
            cudaGetLastError();                  \
            return UELLM_ERR_CUDA;               \
        }                                        \
    } while (0)
    // UELLM_PIPE_TRACE=1: host-side timestamps per group on stderr (diagnosis only)
    const bool trace = getenv("UELLM_PIPE_TRACE") != nullptr;
    const auto t_start = std::chrono::steady_clock::now();
    auto ms = [&]() {
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
    };
  auto body = [&]() -> uellm_status {
    PCU(pool.init(trace));
    H = pool.H; D = pool.D; C2 = pool.C2;
    cudaStream_t CS[2] = {C, C2};       // compute lanes: group g runs on lane g % 2
    cudaEvent_t start = pool.start;
    {
        // everything already queued on the caller's stream happens before our copies
        cudaEventRecord(start, C);
        cudaStreamWaitEvent(H, start, 0);
        cudaStreamWaitEvent(D, start, 0);
        cudaStreamWaitEvent(C2, start, 0);
    }
    auto enqueue_h2d = [&](uint64_t g) -> cudaError_t {
        const int s = (int)(g % 3);
        if (g >= 3) cudaStreamWaitEvent(H, done[g - 3], 0);    // staging slot free again
        const uint64_t a = qa(g), len = qz(g) - a;
        cudaError_t e;
        if ((e = cudaMemcpyAsync(w + PL.in[s], q->input_len + a, 4 * len, cudaMemcpyHostToDevice, H))) return e;
        if ((e = cudaMemcpyAsync(w + PL.out[s], q->pred_out_len + a, 4 * len, cudaMemcpyHostToDevice, H))) return e;
        if ((e = cudaMemcpyAsync(w + PL.slo[s], q->slo_s + a, 4 * len, cudaMemcpyHostToDevice, H))) return e;
        return cudaEventRecord(h2d[g], H);
    };
    // D2H of group g's offsets needs m[g] (read after the host has synchronised past schedule(g))
    auto enqueue_d2h = [&](uint64_t g, uint64_t moff) -> cudaError_t {
        const int s = (int)(g % 3);
        const uint64_t a = qa(g), len = qz(g) - a;
        cudaStreamWaitEvent(D, done[g], 0);
        cudaError_t e;
        if ((e = cudaMemcpyAsync(order + a, w + PL.order[s], 4 * len, cudaMemcpyDeviceToHost, D))) return e;
        // offsets[0 .. m_g) of the group (its closing offset is the next group's first, or n)
        if ((e = cudaMemcpyAsync(batch_offsets + moff, w + PL.offs[s], 4 * m[g], cudaMemcpyDeviceToHost, D))) return e;
        return cudaEventRecord(d2h[g], D);
    };
    PCU(enqueue_h2d(0));
    {
        // Two compute lanes: group g loads / schedules / summarises on lane g % 2 with its own
        // workspace, so one group's latency-bound tail (the DP's last tiles, the traceback)
        // overlaps the next group's sort.  Group g's load synchronises its lane, i.e. group g-2 is
        // complete: its batch count is read and its results go back on the D stream then.
        uint64_t moff = 0;
        auto flush_group = [&](uint64_t gd, cudaStream_t lane) -> cudaError_t {
            cudaError_t e;
            if ((e = cudaMemcpyAsync(&m[gd], (uint64_t *)(w + PL.nb) + gd, 8, cudaMemcpyDeviceToHost, lane))) return e;
            if ((e = cudaStreamSynchronize(lane))) return e;
            if ((e = enqueue_d2h(gd, moff))) return e;
            moff += m[gd];
            return cudaSuccess;
        };
        for (uint64_t g = 0; g < G; ++g) {
            const int s = (int)(g & 1), o = (int)(g % 3);
            cudaStream_t L = CS[s];
            const uint64_t a = qa(g), len = qz(g) - a;
            if (g == 0 && G > 1) PCU(enqueue_h2d(1));
            if (g + 2 < G) PCU(enqueue_h2d(g + 2));           // copies run up to two groups ahead
            PCU(cudaStreamWaitEvent(L, h2d[g], 0));
            const int si = (int)(g % 3);
            uellm_queries gq_ = {len, (const uint32_t *)(w + PL.in[si]), (const uint32_t *)(w + PL.out[si]),
                                 (const float *)(w + PL.slo[si])};
            uellm_profile prof;
            const double t0 = ms();
            const uellm_config &ccfg = g >= G - PL.tail_groups ? tcfg : gcfg;
            uellm_status st = uellm_profile_load(&gq_, &ccfg, w + PL.ws[s], PL.ws_bytes, L, &prof);
            if (st != UELLM_OK) return st;
            const double t1 = ms();
            if (g >= 2) PCU(flush_group(g - 2, L));
            if (g >= 3) PCU(cudaStreamWaitEvent(L, d2h[g - 3], 0));     // output slot g % 3 free again
            uint32_t *d_order = (uint32_t *)(w + PL.order[o]);
            uint32_t *d_offs = (uint32_t *)(w + PL.offs[o]);
            uint64_t *d_nb = (uint64_t *)(w + PL.nb) + g;
            uellm_totals *d_tot = (uellm_totals *)(w + PL.tot) + g;
            if ((st = uellm_schedule_batches(&prof, &ccfg, d_order, d_offs, d_nb, L)) != UELLM_OK) return st;
            const double t2 = ms();
            if ((st = uellm_batch_stats(&prof, &ccfg, d_offs, d_nb, nullptr, d_tot, L)) != UELLM_OK) return st;
            if (trace)
                fprintf(stderr, "[pipe] g=%llu load_in %.3f load_out %.3f sched_out %.3f stats_out %.3f ms\n",
                        (unsigned long long)g, t0, t1, t2, ms());
            PCU(add_base(d_order, len, (uint32_t)a, L));       // group-local -> caller indices
            PCU(add_base(d_offs, len + 1, (uint32_t)a, L));    // (only [0, m_g] are copied)
            PCU(cudaEventRecord(done[g], L));
        }
        for (uint64_t gd = G >= 2 ? G - 2 : 0; gd < G; ++gd) PCU(flush_group(gd, CS[gd & 1]));
        PCU(cudaStreamSynchronize(CS[0]));
        PCU(cudaStreamSynchronize(CS[1]));
        PCU(cudaMemcpy(tot_host.data(), w + PL.tot, sizeof(uellm_totals) * G, cudaMemcpyDeviceToHost));
        PCU(cudaStreamSynchronize(D));
        if (trace) {
            fprintf(stderr, "[pipe] end %.3f ms (%llu groups)\n", ms(), (unsigned long long)G);
            for (uint64_t g = 0; g < G; ++g) {
                float a = 0, b = 0, c = 0;
                cudaEventElapsedTime(&a, start, h2d[g]);
                cudaEventElapsedTime(&b, start, done[g]);
                cudaEventElapsedTime(&c, start, d2h[g]);
                fprintf(stderr, "[pipe]   g=%llu q=%llu  h2d_done %.3f  compute_done %.3f  d2h_done %.3f ms\n",
                        (unsigned long long)g, (unsigned long long)(qz(g) - qa(g)), a, b, c);
            }
        }
        batch_offsets[moff] = (uint32_t)n;
        *num_batches = moff;
        // whole-job totals from the per-group integer totals (exact); the latency mean is
        // re-weighted by the group sizes, the throughput recomputed from the integer sums
        uellm_totals T;
        std::memset(&T, 0, sizeof T);
        for (uint64_t g = 0; g < G; ++g) combine_totals_into(T, tot_host[g]);
        finish_totals(T);
        *totals = T;
        if (T.overflow) return UELLM_ERR_OVERFLOW;
    }
    return UELLM_OK;
  };
    status = body();
    if (status != UELLM_OK) { cudaStreamSynchronize(C); }
    // (the pool's streams stay; an error leaves no copy of this call in flight on them)
    if (H) cudaStreamSynchronize(H);
    if (D) cudaStreamSynchronize(D);
    if (C2) cudaStreamSynchronize(C2);
#undef PCU
    return status;
}

}  // extern "C"
