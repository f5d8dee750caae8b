/*
 * oracle/uellm_oracle.c -- plain, slow, obviously-correct CPU oracle for the UELLM
 * batch-scheduler hot path (arXiv 2409.14961, "UELLM", Sec. 4.2 + Alg. 1).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2409_14961_b200/) never includes, links or calls it, and this file includes
 * nothing from the product path: the two share no code, headers, tables or constants.
 *
 * Citations: "P:NNN" = line NNN of /root/reference/PAPER.md, "S:NNN" = line of SPEC.md,
 * "Rk" = reading k of DESIGN.md (paper silent / ambiguous / garbled).
 *
 * What it computes (one function per hot-path step, in the paper's order):
 *   orc_slo_us          O2   SLO seconds -> integer microseconds (R12)
 *   orc_kv_bytes        A1   KV-cache peak bytes 4*b*l*h*(s+n)
 *   orc_schedule        O1   windows of the arrival stream (R15)
 *                       O3   sort ascending by SLO (then predicted length, R11)
 *                       O4   SEG-DP: exact min over contiguous segmentations of
 *                            sum_batches est_us + lambda * violations (R7, R8, R14)
 *                       O5   Alg. 1 SLO-ODBS, literal (R1-R5)
 *                       O6   FIFO baseline
 *   orc_stats           O7   per-batch padding / tokens / KV / latency stats
 *   orc_simulate        O8   sequential execution of a schedule with arrivals
 *                            (NEXT f2; latency, SLO violations, utilisation,
 *                            throughput)
 *   orc_predict         O9   profiler stand-ins: oracle / bucketed / noisy /      P:195
 *                            constant predicted output length (NEXT f4)
 *   orc_monitor_observe O10  misprediction monitor, gamma-inflation (NEXT f4)
 *   orc_profile_stream  O11  predict + observe, one monitor epoch per window      R20
 *   orc_helr            O12  HELR deployer: subsets x bitmask DP over device      P:301-384,
 *                            visit orders (HE: a1 = 0, LR: a1:a2 = 10:1) (f3)
 *   orc_bgs             O13  BGS baseline deployer: greedy by memory (f3)
 *
 * Parity pins (tests/test_oracle_*.py, -m "not gpu"): brute-force enumeration of all
 * 2^(n-1) segmentations (n <= 12), closed forms (identical queries), special cases
 * (W = 1, zero overhead), SPEC worked examples, invariants.
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fPIC -shared -pthread (see __graft_entry__.build).
 * -ffp-contract=off: Alg. 1's double expressions are evaluated as written, no FMA.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <pthread.h>

/* ---- status codes (own copy; deliberately not shared with include/uellm.h) ---- */
enum { ORC_OK = 0, ORC_ERR_ARG = 1, ORC_ERR_CONTRACT = 2, ORC_ERR_CONFIG = 3,
       ORC_ERR_OVERFLOW = 4 };
/* ---- segmentation modes ---- */
enum { ORC_MODE_SEG_DP = 0, ORC_MODE_SLO_ODBS = 1, ORC_MODE_FIFO = 2, ORC_MODE_SORT_ONLY = 3 };

typedef struct {
    uint32_t mode;                 /* ORC_MODE_*                                         */
    uint32_t window;               /* queries per scheduling window, 0 = all (R15)       */
    uint32_t max_batch;            /* W >= 1                                             */
    uint32_t split_on_slo_change;  /* 1: batches never mix SLO values (R15)              */
    uint32_t kv_bytes_per_elem;    /* the "4" of P:60 (R13)                              */
    uint32_t n_layers;             /* l of P:60                                          */
    uint32_t hidden;               /* h of P:60                                          */
    uint32_t pad0;
    uint64_t kv_cap_bytes;         /* per-batch KV reserve, T of P:366 (R6); 0 = none    */
    uint32_t t_batch_us, t_iter_us, t_tok_us, t_prefill_us;   /* service model (R7)      */
    uint64_t lambda_us;            /* penalty per violating query (R8, R14)              */
    double   w1, w2, l1, l2, threshold, eps;                   /* Alg. 1     */
    uint32_t eq2_additive;         /* R2: 1 -> Eq. 2 '+' form instead of Alg. 1 '-'      */
    uint32_t pad1;
} orc_config;

typedef struct {
    uint32_t start, size, max_in, max_out;
    uint64_t gen_tokens, pad_in, pad_out, kv_bytes, est_us, completion_us;
    uint32_t viol_alone, viol_seq, over_cap, window;
} orc_batch_stat;

typedef struct {
    uint64_t n, batches, gen_tokens, pad_in, pad_out, kv_bytes_max, dp_cost,
             viol_alone, viol_seq, over_cap, makespan_us;
    double   mean_latency_s, throughput_tok_s;
} orc_totals;

/* ======================================================================== */
/* O2  SLO seconds -> microseconds.  P:463 gives SLOs in seconds ("1 second to 350
 * seconds"); R12: one integer representation after load: slo_us = rint(slo_s * 1e6)
 * computed in double, round-half-to-even, required to lie in [1, 2^32 - 1].            */
int orc_slo_us(float slo_s, uint32_t *slo_us)
{
    double x = (double)slo_s;
    if (!(x > 0.0) || !isfinite(x)) return ORC_ERR_CONTRACT;
    double us = x * 1e6;                                        /* one correctly rounded product */
    double r = nearbyint(us);                                   /* default mode: half-to-even   */
    if (r < 1.0 || r > 4294967295.0) return ORC_ERR_CONTRACT;
    *slo_us = (uint32_t)r;
    return ORC_OK;
}

/* A1  KV-cache peak bytes: "4 x blh(s + n)"; the 4 is kv_bytes_per_elem (R13).
 * Exact, overflow detected.                                                    */
int orc_kv_bytes(uint32_t kvpe, uint64_t b, uint32_t l, uint32_t h, uint64_t s, uint64_t n,
                 uint64_t *out)
{
    uint64_t t = kvpe, sn;
    if (__builtin_add_overflow(s, n, &sn)) return ORC_ERR_OVERFLOW;
    if (__builtin_mul_overflow(t, b, &t)) return ORC_ERR_OVERFLOW;
    if (__builtin_mul_overflow(t, (uint64_t)l, &t)) return ORC_ERR_OVERFLOW;
    if (__builtin_mul_overflow(t, (uint64_t)h, &t)) return ORC_ERR_OVERFLOW;
    if (__builtin_mul_overflow(t, sn, &t)) return ORC_ERR_OVERFLOW;
    *out = t;
    return ORC_OK;
}

/* R7  estimated service time of one batch (integer microseconds):
 *   est = t_batch + t_iter*O + t_tok*b*O + t_prefill*b*s
 * b = batch size, s = max input (inputs padded to it), O = max predicted output
 * (all members generate O tokens, "b x O").                                     */
static int est_us(const orc_config *c, uint64_t b, uint64_t s, uint64_t O, uint64_t *out)
{
    uint64_t a, t, e;
    if (__builtin_mul_overflow((uint64_t)c->t_iter_us, O, &a)) return ORC_ERR_OVERFLOW;
    if (__builtin_add_overflow((uint64_t)c->t_batch_us, a, &e)) return ORC_ERR_OVERFLOW;
    if (__builtin_mul_overflow((uint64_t)c->t_tok_us, b, &t)) return ORC_ERR_OVERFLOW;
    if (__builtin_mul_overflow(t, O, &t)) return ORC_ERR_OVERFLOW;
    if (__builtin_add_overflow(e, t, &e)) return ORC_ERR_OVERFLOW;
    if (__builtin_mul_overflow((uint64_t)c->t_prefill_us, b, &t)) return ORC_ERR_OVERFLOW;
    if (__builtin_mul_overflow(t, s, &t)) return ORC_ERR_OVERFLOW;
    if (__builtin_add_overflow(e, t, &e)) return ORC_ERR_OVERFLOW;
    *out = e;
    return ORC_OK;
}

/* per-batch memory constraint (A1 with the KV reserve of P:366 as cap, R6, R10):
 * a single query is always admissible; a larger batch needs kv_bytes <= cap.          */
static int batch_feasible(const orc_config *c, uint64_t b, uint64_t s, uint64_t O, int *ok)
{
    uint64_t kv;
    if (b <= 1 || c->kv_cap_bytes == 0) { *ok = 1; return ORC_OK; }
    int st = orc_kv_bytes(c->kv_bytes_per_elem, b, c->n_layers, c->hidden, s, O, &kv);
    if (st == ORC_ERR_OVERFLOW) { *ok = 0; return ORC_OK; }   /* > any u64 cap */
    *ok = (kv <= c->kv_cap_bytes);
    return ORC_OK;
}

/* ======================================================================== */
/* O3  sort.  P:228 "sorted in ascending order according to their SLO"; R11 adds the
 * predicted output length as secondary key; R9 breaks remaining ties by arrival index.
 * (slo_us, out, idx) is a total order, so qsort yields the unique stable order.        */
typedef struct { uint32_t slo_us, out, in, idx; } orc_q;

static int cmp_q(const void *pa, const void *pb)
{
    const orc_q *a = (const orc_q *)pa, *b = (const orc_q *)pb;
    if (a->slo_us != b->slo_us) return a->slo_us < b->slo_us ? -1 : 1;
    if (a->out != b->out) return a->out < b->out ? -1 : 1;
    if (a->idx != b->idx) return a->idx < b->idx ? -1 : 1;
    return 0;
}

/* number of members k in [i, j) with slo_us[k] < e.  The window is sorted ascending by
 * slo_us (O3), so this is lower_bound(slo[i..j), e) - i (plain binary search).         */
static uint64_t count_below(const orc_q *q, uint64_t i, uint64_t j, uint64_t e)
{
    uint64_t lo = i, hi = j;                 /* first k in [i,j) with slo >= e */
    while (lo < hi) {
        uint64_t mid = lo + (hi - lo) / 2;
        if ((uint64_t)q[mid].slo_us < e) lo = mid + 1; else hi = mid;
    }
    return lo - i;
}

/* O4  SEG-DP over one sorted window q[0..L).
 *   C[0] = 0;  C[j] = min_{i in [max(0,j-W), j), feasible(i,j), same-SLO if split}
 *                     C[i] + est_us(i,j) + lambda * viol(i,j)
 *   viol(i,j) = #{k in [i,j) : slo_us[k] < est_us(i,j)}   (R8: standalone violations)
 *   arg[j] = the SMALLEST minimising i (R9).  Every candidate is evaluated (no pruning).
 * Writes batch starts (ascending, window-local) to starts[], returns count in *nb.     */
static int seg_dp_window(const orc_config *c, const orc_q *q, uint64_t L,
                         uint64_t *starts, uint64_t *nb, uint64_t *cost)
{
    uint64_t W = c->max_batch;
    uint64_t *C = (uint64_t *)malloc((L + 1) * sizeof(uint64_t));
    uint64_t *arg = (uint64_t *)malloc((L + 1) * sizeof(uint64_t));
    if (!C || !arg) { free(C); free(arg); return ORC_ERR_ARG; }
    int st = ORC_OK;
    C[0] = 0;
    for (uint64_t j = 1; j <= L && st == ORC_OK; ++j) {
        uint64_t lo = (j > W) ? j - W : 0;
        uint64_t best = UINT64_MAX, barg = j;   /* i = j-1 (singleton) is always feasible */
        uint64_t MI = 0, MO = 0;                 /* maxima over [i, j), built as i descends */
        for (uint64_t i = j; i-- > lo; ) {
            if (q[i].in > MI) MI = q[i].in;
            if (q[i].out > MO) MO = q[i].out;
            if (c->split_on_slo_change && q[i].slo_us != q[j - 1].slo_us) continue;
            uint64_t b = j - i;
            int ok;
            batch_feasible(c, b, MI, MO, &ok);
            if (!ok) continue;
            uint64_t e, tot, pen;
            if ((st = est_us(c, b, MI, MO, &e)) != ORC_OK) break;
            uint64_t v = count_below(q, i, j, e);
            if (__builtin_mul_overflow(c->lambda_us, v, &pen)) { st = ORC_ERR_OVERFLOW; break; }
            if (__builtin_add_overflow(C[i], e, &tot) || __builtin_add_overflow(tot, pen, &tot)) {
                st = ORC_ERR_OVERFLOW; break;
            }
            if (tot <= best) { best = tot; barg = i; }   /* descending i: '<=' keeps the smallest */
        }
        C[j] = best;
        arg[j] = barg;
    }
    if (st == ORC_OK) {
        /* traceback from the window end; batch starts come out in descending order */
        uint64_t k = 0;
        for (uint64_t j = L; j > 0; j = arg[j]) starts[k++] = arg[j];
        for (uint64_t a = 0, b = k; a + 1 < b; ++a, --b) { uint64_t t = starts[a]; starts[a] = starts[b - 1]; starts[b - 1] = t; }
        *nb = k;
        *cost = C[L];
    }
    free(C); free(arg);
    return st;
}

/* O5  Alg. 1, SLO-ODBS, literal, with the readings of DESIGN.md:
 *   R1 incremental T_l / T_o of Alg. 1 lines 6-7, not Eq. 1's sum;
 *   R2 '-' in T_o unless eq2_additive ('+', Eq. 2);
 *   R3 Total = w1*T_l + w2*T_o <= Threshold;
 *   R4 CM = max(CM, w1*length + w2*SLO) as printed;
 *   R5 line 20: cap = clamp(floor(threshold / max(CM, eps)), 1, W) after every
 *      iteration; the batch is flushed once |batch_c| >= cap;
 *   R6/R10 a non-empty batch additionally admits q only if the KV bytes stay <= cap;
 *   R12 SLO in seconds as slo_us / 1e6.
 * SLO-DBS = w1 = 0, ODBS = w2 = 0.  Doubles, fixed expression trees, no FMA.   */
static int slo_odbs_window(const orc_config *c, const orc_q *q, uint64_t L,
                           uint64_t *starts, uint64_t *nb)
{
    uint64_t k = 0, bsize = 0;          /* |batch_c| */
    double L_CM = 0.0, O_CM = 0.0, CM = 0.0;
    uint64_t MI = 0;                     /* current max input, for the KV constraint */
    for (uint64_t x = 0; x < L; ++x) {
        double slo = (double)q[x].slo_us / 1e6;
        double len = (double)q[x].out;
        if (c->split_on_slo_change && bsize > 0 && q[x].slo_us != q[x - 1].slo_us) {
            bsize = 0; L_CM = 0.0; O_CM = 0.0; CM = 0.0; MI = 0;   /* flush */
        }
        double nb1 = (double)(bsize + 1);
        double T_l = ((slo + L_CM) * nb1) * c->l1;                          /* Alg.1 l.6 */
        double T_o = (c->eq2_additive ? (len + O_CM) : (len - O_CM));
        T_o = (T_o * nb1) * c->l2;                                          /* Alg.1 l.7 */
        double p1 = c->w1 * T_l;
        double p2 = c->w2 * T_o;
        double Total = p1 + p2;                                             /* Alg.1 l.8 */
        int admit = (bsize == 0);
        if (!admit && Total <= c->threshold) {
            uint64_t s = q[x].in > MI ? q[x].in : MI;
            uint64_t O = (uint64_t)(len > O_CM ? len : O_CM);
            int ok; batch_feasible(c, bsize + 1, s, O, &ok);
            admit = ok;
        }
        double cmq = c->w1 * len;
        double cm2 = c->w2 * slo;
        cmq = cmq + cm2;
        if (admit) {                                                        /* l.10-13 */
            if (bsize == 0) starts[k++] = x;
            bsize += 1;
            if (slo > L_CM) L_CM = slo;
            if (len > O_CM) O_CM = len;
            if (cmq > CM) CM = cmq;
            if (q[x].in > MI) MI = q[x].in;
        } else {                                                            /* l.14-19 */
            starts[k++] = x;
            bsize = 1; L_CM = slo; O_CM = len; CM = cmq; MI = q[x].in;
        }
        /* l.20: "Dynamically adjust batch_size according to the value of CM" (R5) */
        double den = CM > c->eps ? CM : c->eps;
        double capd = floor(c->threshold / den);
        uint64_t cap = capd < 1.0 ? 1 : (capd > (double)c->max_batch ? c->max_batch : (uint64_t)capd);
        if (bsize >= cap) { bsize = 0; L_CM = 0.0; O_CM = 0.0; CM = 0.0; MI = 0; }
    }
    *nb = k;
    return ORC_OK;
}

/* ======================================================================== */
typedef struct {
    const orc_config *cfg;
    uint64_t n, wlen, nwin;
    const uint32_t *in, *out;
    const uint32_t *slo_us;
    uint64_t *wstarts;      /* per window: batch starts (global sorted positions), capacity n */
    uint64_t *wcount;       /* per window: number of batches                               */
    uint64_t *wcost;        /* per window: DP cost                                           */
    uint32_t *order;
    int *wstatus;
    uint64_t next;          /* next window to take (protected by mu) */
    pthread_mutex_t mu;
} orc_job;

static void run_window(orc_job *J, uint64_t w)
{
    const orc_config *c = J->cfg;
    uint64_t w0 = w * J->wlen, w1 = w0 + J->wlen < J->n ? w0 + J->wlen : J->n, L = w1 - w0;
    orc_q *q = (orc_q *)malloc((L ? L : 1) * sizeof(orc_q));
    uint64_t *st = J->wstarts + w0;
    if (!q) { J->wstatus[w] = ORC_ERR_ARG; return; }
    for (uint64_t k = 0; k < L; ++k) {
        q[k].slo_us = J->slo_us[w0 + k]; q[k].out = J->out[w0 + k];
        q[k].in = J->in[w0 + k]; q[k].idx = (uint32_t)k;
    }
    uint64_t nb = 0, cost = 0;
    int s = ORC_OK;
    if (c->mode == ORC_MODE_FIFO) {
        /* O6: caller (arrival) order, consecutive chunks of max_batch */
        for (uint64_t k = 0; k < L; ++k) J->order[w0 + k] = (uint32_t)(w0 + k);
        for (uint64_t k = 0; k < L; k += c->max_batch) st[nb++] = k;
    } else {
        qsort(q, L, sizeof(orc_q), cmp_q);
        for (uint64_t k = 0; k < L; ++k) J->order[w0 + k] = (uint32_t)(w0 + q[k].idx);
        if (c->mode == ORC_MODE_SORT_ONLY) {
            for (uint64_t k = 0; k < L; ++k) st[nb++] = k;
        } else if (c->mode == ORC_MODE_SEG_DP) {
            s = seg_dp_window(c, q, L, st, &nb, &cost);
        } else {
            s = slo_odbs_window(c, q, L, st, &nb);
        }
    }
    for (uint64_t k = 0; k < nb; ++k) st[k] += w0;
    J->wcount[w] = nb;
    J->wcost[w] = cost;
    J->wstatus[w] = s;
    free(q);
}

static void *worker(void *p)
{
    orc_job *J = (orc_job *)p;
    for (;;) {
        pthread_mutex_lock(&J->mu);
        uint64_t w = J->next++;
        pthread_mutex_unlock(&J->mu);
        if (w >= J->nwin) break;
        run_window(J, w);
    }
    return NULL;
}

static int check_config(const orc_config *c)
{
    if (c->mode > ORC_MODE_SORT_ONLY) return ORC_ERR_CONFIG;
    if (c->max_batch < 1) return ORC_ERR_CONFIG;
    if (c->split_on_slo_change > 1) return ORC_ERR_CONFIG;
    if (c->mode == ORC_MODE_SLO_ODBS) {
        /* w1, w2 >= 0, w1 + w2 > 0, threshold > 0 */
        if (!(c->w1 >= 0.0) || !(c->w2 >= 0.0) || !(c->w1 + c->w2 > 0.0)) return ORC_ERR_CONFIG;
        if (!(c->threshold > 0.0) || !(c->eps > 0.0)) return ORC_ERR_CONFIG;
        if (!(c->l1 >= 0.0) || !(c->l2 >= 0.0)) return ORC_ERR_CONFIG;
    }
    if (c->kv_cap_bytes != 0 && (c->kv_bytes_per_elem == 0 || c->n_layers == 0 || c->hidden == 0))
        return ORC_ERR_CONFIG;
    return ORC_OK;
}

/* O1-O6: schedule n queries (caller SoA).  Outputs:
 *   order[k]      caller index at scheduled position k (windows ascending)
 *   offsets[0..m] batch t = order[offsets[t] .. offsets[t+1]); offsets[m] = n
 *   *m            number of batches;  *dp_cost  sum over windows of the DP optimum
 *                 (0 unless mode == SEG_DP)
 * nthreads >= 1: windows are independent and distributed over a thread pool.            */
int orc_schedule(uint64_t n, const uint32_t *in, const uint32_t *out, const float *slo_s,
                 const orc_config *cfg, uint32_t *order, uint32_t *offsets, uint64_t *m,
                 uint64_t *dp_cost, int nthreads)
{
    if (!cfg || !m || !dp_cost) return ORC_ERR_ARG;
    if (n > 0 && (!in || !out || !slo_s || !order || !offsets)) return ORC_ERR_ARG;
    if (n >= 4294967295ull) return ORC_ERR_ARG;
    int s = check_config(cfg);
    if (s != ORC_OK) return s;
    if (n == 0) { *m = 0; *dp_cost = 0; if (offsets) offsets[0] = 0; return ORC_OK; }
    /* O2: validate every query before any output is written */
    uint32_t *slo_us = (uint32_t *)malloc(n * sizeof(uint32_t));
    if (!slo_us) return ORC_ERR_ARG;
    for (uint64_t k = 0; k < n; ++k) {
        if (in[k] < 1 || out[k] < 1 || orc_slo_us(slo_s[k], &slo_us[k]) != ORC_OK) {
            free(slo_us); return ORC_ERR_CONTRACT;
        }
    }
    orc_job J;
    memset(&J, 0, sizeof J);
    J.cfg = cfg; J.n = n; J.in = in; J.out = out; J.slo_us = slo_us; J.order = order;
    J.wlen = cfg->window ? cfg->window : n;
    J.nwin = (n + J.wlen - 1) / J.wlen;
    J.wstarts = (uint64_t *)malloc(n * sizeof(uint64_t));
    J.wcount = (uint64_t *)calloc(J.nwin, sizeof(uint64_t));
    J.wcost = (uint64_t *)calloc(J.nwin, sizeof(uint64_t));
    J.wstatus = (int *)calloc(J.nwin, sizeof(int));
    pthread_mutex_init(&J.mu, NULL);
    if (!J.wstarts || !J.wcount || !J.wcost || !J.wstatus) { s = ORC_ERR_ARG; goto done; }
    if (nthreads < 1) nthreads = 1;
    if ((uint64_t)nthreads > J.nwin) nthreads = (int)J.nwin;
    if (nthreads == 1) {
        worker(&J);
    } else {
        pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * nthreads);
        for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, worker, &J);
        for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
        free(th);
    }
    uint64_t k = 0, cost = 0;
    for (uint64_t w = 0; w < J.nwin; ++w) {
        if (J.wstatus[w] != ORC_OK) { s = J.wstatus[w]; goto done; }
        if (__builtin_add_overflow(cost, J.wcost[w], &cost)) { s = ORC_ERR_OVERFLOW; goto done; }
        uint64_t w0 = w * J.wlen;
        for (uint64_t t = 0; t < J.wcount[w]; ++t) offsets[k++] = (uint32_t)J.wstarts[w0 + t];
    }
    offsets[k] = (uint32_t)n;
    *m = k;
    *dp_cost = cost;
done:
    pthread_mutex_destroy(&J.mu);
    free(J.wstarts); free(J.wcount); free(J.wcost); free(J.wstatus); free(slo_us);
    return s;
}

/* O7  per-batch statistics of a schedule (any mode), following P:60 / P:210 and
 * S:138-156 / S:449-452:
 *   size b, max_in s, max_out O, gen_tokens = b*O ("b x O"),
 *   pad_in = sum(s - in_k) (inputs padded to the max), pad_out = sum(O - out_k),
 *   kv_bytes = 4*b*l*h*(s+O), est_us (R7),
 *   completion_us = inclusive prefix of est_us over the window's batches (sequential
 *                   execution, all queries present at t = 0),
 *   viol_alone = #{slo_us < est_us}, viol_seq = #{slo_us < completion_us},
 *   over_cap = kv_bytes > cap (cap != 0).
 * Totals: sums, kv_bytes_max, dp_cost = sum(est + lambda*viol_alone) (the SEG-DP
 * objective evaluated on this schedule), makespan = sum est,
 * mean_latency_s = sum_k completion(batch(k)) / n * 1e-6,
 * throughput_tok_s = sum gen / (makespan * 1e-6).                                       */
int orc_stats(uint64_t n, const uint32_t *in, const uint32_t *out, const float *slo_s,
              const orc_config *cfg, const uint32_t *order, const uint32_t *offsets,
              uint64_t m, orc_batch_stat *per_batch, orc_totals *tot)
{
    if (!cfg || !tot) return ORC_ERR_ARG;
    memset(tot, 0, sizeof *tot);
    tot->n = n;
    tot->batches = m;
    if (n == 0) return ORC_OK;
    uint64_t wlen = cfg->window ? cfg->window : n;
    uint64_t clock = 0, cur_win = UINT64_MAX;
    unsigned __int128 lat_sum = 0;          /* exact; converted to double once at the end */
    for (uint64_t t = 0; t < m; ++t) {
        uint64_t a = offsets[t], z = offsets[t + 1];
        if (z <= a || z > n) return ORC_ERR_ARG;
        uint64_t win = a / wlen;
        if ((z - 1) / wlen != win) return ORC_ERR_ARG;     /* batches never cross windows */
        if (win != cur_win) { cur_win = win; clock = 0; }
        uint64_t b = z - a, s = 0, O = 0, sin = 0, sout = 0;
        for (uint64_t k = a; k < z; ++k) {
            uint32_t x = order[k];
            if (in[x] > s) s = in[x];
            if (out[x] > O) O = out[x];
            sin += in[x]; sout += out[x];
        }
        uint64_t kv, e, v1 = 0, v2 = 0;
        if (orc_kv_bytes(cfg->kv_bytes_per_elem, b, cfg->n_layers, cfg->hidden, s, O, &kv) != ORC_OK)
            return ORC_ERR_OVERFLOW;
        if (est_us(cfg, b, s, O, &e) != ORC_OK) return ORC_ERR_OVERFLOW;
        if (__builtin_add_overflow(clock, e, &clock)) return ORC_ERR_OVERFLOW;
        for (uint64_t k = a; k < z; ++k) {
            uint32_t su;
            if (orc_slo_us(slo_s[order[k]], &su) != ORC_OK) return ORC_ERR_CONTRACT;
            if (su < e) v1++;
            if (su < clock) v2++;
        }
        uint32_t oc = (cfg->kv_cap_bytes != 0 && kv > cfg->kv_cap_bytes);
        if (per_batch) {
            orc_batch_stat *p = &per_batch[t];
            p->start = (uint32_t)a; p->size = (uint32_t)b; p->max_in = (uint32_t)s; p->max_out = (uint32_t)O;
            p->gen_tokens = b * O; p->pad_in = b * s - sin; p->pad_out = b * O - sout;
            p->kv_bytes = kv; p->est_us = e; p->completion_us = clock;
            p->viol_alone = (uint32_t)v1; p->viol_seq = (uint32_t)v2; p->over_cap = oc;
            p->window = (uint32_t)win;
        }
        tot->gen_tokens += b * O;
        tot->pad_in += b * s - sin;
        tot->pad_out += b * O - sout;
        if (kv > tot->kv_bytes_max) tot->kv_bytes_max = kv;
        uint64_t pen, obj;
        if (__builtin_mul_overflow(cfg->lambda_us, v1, &pen) || __builtin_add_overflow(e, pen, &obj)
            || __builtin_add_overflow(tot->dp_cost, obj, &tot->dp_cost)) return ORC_ERR_OVERFLOW;
        tot->viol_alone += v1;
        tot->viol_seq += v2;
        tot->over_cap += oc;
        tot->makespan_us += e;
        lat_sum += (unsigned __int128)b * clock;
    }
    tot->mean_latency_s = (double)lat_sum / (double)n * 1e-6;
    tot->throughput_tok_s = tot->makespan_us ? (double)tot->gen_tokens / ((double)tot->makespan_us * 1e-6) : 0.0;
    return ORC_OK;
}


/* ======================================================================== */
/* O8  sequential-execution simulator with arrivals (NEXT f2; R19).
 * P:499 names the paper's metrics (latency = "time taken for the system to respond", SLO
 * violation, GPU utilisation, throughput); S:445-457 fixes the execution model:
 *   - batches execute sequentially on one replica, in scan order (windows ascending,
 *     P:245), the service time of batch t is est_us(t) (R7);
 *   - "a batch cannot start before the latest arrival among its members":
 *         start_t = max(end_{t-1}, max_{k in t} arrival_k),   end_{-1} = 0,
 *         end_t   = start_t + est_us(t);
 *   - latency_k = end_{t(k)} - arrival_k; a violation is latency_k > slo_us_k
 *     ("latency > slo");
 *   - makespan = end of the last batch (the timeline starts at 0), busy = sum est,
 *     idle = makespan - busy (S:471 work conservation), utilisation = busy / makespan,
 *     throughput = sum b*O / makespan.
 * One continuous timeline over all windows of the call.  Integers are exact; a batch end at
 * or beyond 2^63 us is an overflow error (the limit include/uellm.h states); the four doubles
 * are formed once at the end.                                                              */
typedef struct {
    uint64_t n, batches, makespan_us, busy_us, idle_us, gen_tokens, viol, latency_max_us;
    uint64_t latency_sum_lo, latency_sum_hi;      /* exact 128-bit sum of latencies (us) */
    double   mean_latency_s, slo_violation_rate, utilization, throughput_tok_s;
} orc_sim_totals;

/* batch_end_us[t] = end_t; latency_us[k] = latency of query order[k] (scheduled position k). */
int orc_simulate(uint64_t n, const uint32_t *in, const uint32_t *out, const float *slo_s,
                 const orc_config *cfg, const uint32_t *order, const uint32_t *offsets,
                 uint64_t m, const uint64_t *arrival_us, uint64_t *batch_end_us,
                 uint64_t *latency_us, orc_sim_totals *tot)
{
    if (!cfg || !tot) return ORC_ERR_ARG;
    if (n > 0 && (!in || !out || !slo_s || !order || !offsets || !arrival_us)) return ORC_ERR_ARG;
    memset(tot, 0, sizeof *tot);
    tot->n = n;
    tot->batches = m;
    if (n == 0) return ORC_OK;
    uint64_t end = 0;                       /* end_{t-1}; the server is free from time 0 */
    unsigned __int128 lat_sum = 0;
    for (uint64_t t = 0; t < m; ++t) {
        uint64_t a = offsets[t], z = offsets[t + 1];
        if (z <= a || z > n) return ORC_ERR_ARG;
        uint64_t b = z - a, s = 0, O = 0, last_arrival = 0, e;
        for (uint64_t k = a; k < z; ++k) {
            uint32_t x = order[k];
            if (in[x] > s) s = in[x];
            if (out[x] > O) O = out[x];
            if (arrival_us[x] > last_arrival) last_arrival = arrival_us[x];
        }
        if (est_us(cfg, b, s, O, &e) != ORC_OK) return ORC_ERR_OVERFLOW;
        uint64_t start = end > last_arrival ? end : last_arrival;
        tot->idle_us += start - end;
        if (__builtin_add_overflow(start, e, &end) || end >= (1ull << 63)) return ORC_ERR_OVERFLOW;
        if (batch_end_us) batch_end_us[t] = end;
        tot->busy_us += e;
        tot->gen_tokens += b * O;
        for (uint64_t k = a; k < z; ++k) {
            uint32_t x = order[k], su;
            if (orc_slo_us(slo_s[x], &su) != ORC_OK) return ORC_ERR_CONTRACT;
            uint64_t lat = end - arrival_us[x];
            if (latency_us) latency_us[k] = lat;                           /* scheduled position */
            if (lat > su) tot->viol++;
            if (lat > tot->latency_max_us) tot->latency_max_us = lat;
            lat_sum += lat;
        }
    }
    tot->makespan_us = end;
    tot->latency_sum_lo = (uint64_t)lat_sum;
    tot->latency_sum_hi = (uint64_t)(lat_sum >> 64);
    tot->mean_latency_s = (double)lat_sum / (double)n * 1e-6;
    tot->slo_violation_rate = (double)tot->viol / (double)n;
    tot->utilization = end ? (double)tot->busy_us / (double)end : 0.0;
    tot->throughput_tok_s = end ? (double)tot->gen_tokens / ((double)end * 1e-6) : 0.0;
    return ORC_OK;
}

/* ======================================================================== */
/* O9-O11  profiler stand-ins and the misprediction monitor (NEXT f4; R20).
 * the resource profiler "categorize[s] the output lengths" of requests into buckets (a
 * fine-tuned ChatGLM3-6B, out of scope); a backend monitor "detect[s] erroneous
 * predictions and adjust[s] the allocated memory size".  SPEC S:200-207 / S:211-218 fix the
 * stand-ins used here:
 *   oracle      pred = true length
 *   bucketed(w) pred = true length rounded up to the bucket ceiling (R20: at least one bucket)
 *   noisy(e, w) the bucketed value displaced by +-1 bucket with probability e (seeded,
 *               reproducible; R20: never below the first bucket)
 *   constant(v) pred = v
 * then "multiplied by monitor.inflation_factor and rounded up"; R20 saturates at
 * 2^32 - 1.  The monitor: on actual > predicted, corrections += 1 and
 * factor <- min(factor * gamma, cap).
 * Random draws: a counter-based generator (splitmix64 finaliser of seed ^ (index * golden
 * gamma)); u = (z >> 11) * 2^-53, displaced iff u < e, direction + iff z is odd.  The CUDA path
 * implements the same generator independently (③: same counter-based generator on each side). */
typedef struct {
    uint32_t variant;          /* 0 oracle, 1 bucketed, 2 noisy, 3 constant */
    uint32_t bucket_width;     /* >= 1 for bucketed / noisy */
    uint32_t constant_tokens;  /* >= 1 for constant */
    uint32_t window;           /* monitor epoch in queries (0 = all) */
    double   error_rate;       /* [0, 1] */
    double   gamma;            /* >= 1 */
    double   cap;              /* >= 1 */
    uint64_t seed;
    uint32_t monitor;          /* 0|1 */
    uint32_t pad;
} orc_predictor;

static uint64_t orc_mix64(uint64_t seed, uint64_t index)
{
    uint64_t z = seed ^ (index * 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static int check_predictor(const orc_predictor *p)
{
    if (p->variant > 3) return ORC_ERR_CONFIG;
    if ((p->variant == 1 || p->variant == 2) && p->bucket_width < 1) return ORC_ERR_CONFIG;
    if (p->variant == 3 && p->constant_tokens < 1) return ORC_ERR_CONFIG;
    if (!(p->error_rate >= 0.0 && p->error_rate <= 1.0)) return ORC_ERR_CONFIG;
    if (p->monitor > 1) return ORC_ERR_CONFIG;
    if (p->monitor && !(p->gamma >= 1.0 && p->cap >= 1.0 && isfinite(p->gamma) && isfinite(p->cap)))
        return ORC_ERR_CONFIG;
    return ORC_OK;
}

/* O9: prediction for query `index` (global caller index) with inflation `factor` */
static uint32_t predict_one(const orc_predictor *p, uint64_t index, uint32_t true_len, double factor)
{
    uint64_t base;
    if (p->variant == 0) {
        base = true_len;
    } else if (p->variant == 3) {
        base = p->constant_tokens;
    } else {
        uint64_t w = p->bucket_width;
        uint64_t k = (true_len + w - 1) / w;          /* bucket of the true length (ceiling) */
        if (k < 1) k = 1;
        if (p->variant == 2) {
            uint64_t z = orc_mix64(p->seed, index);
            double u = (double)(z >> 11) * 0x1.0p-53;
            if (u < p->error_rate) {
                if (z & 1) k += 1;
                else if (k > 1) k -= 1;
            }
        }
        base = k * w;
    }
    double x = ceil((double)base * factor);           /* "multiplied ... and rounded up" */
    return x >= 4294967295.0 ? 4294967295u : (uint32_t)x;
}

int orc_predict(uint64_t n, uint64_t index0, const uint32_t *true_len, const orc_predictor *p,
                double factor, uint32_t *pred)
{
    if (!p || (n && (!true_len || !pred))) return ORC_ERR_ARG;
    int s = check_predictor(p);
    if (s != ORC_OK) return s;
    if (!(factor >= 1.0) || !isfinite(factor)) return ORC_ERR_CONFIG;
    for (uint64_t k = 0; k < n; ++k) pred[k] = predict_one(p, index0 + k, true_len[k], factor);
    return ORC_OK;
}

/* O10: S:211-218, one observation at a time, in order */
int orc_monitor_observe(uint64_t n, const uint32_t *pred, const uint32_t *actual, double gamma,
                        double cap, uint64_t *corrections, double *factor)
{
    if (!corrections || !factor || (n && (!pred || !actual))) return ORC_ERR_ARG;
    for (uint64_t k = 0; k < n; ++k) {
        if (actual[k] > pred[k]) {
            *corrections += 1;
            double f = *factor * gamma;
            *factor = f < cap ? f : cap;
        }
    }
    return ORC_OK;
}

/* O11 (R20): the profiler and the monitor over a stream cut into windows (the scheduling
 * windows, R15).  Window w is predicted with the factor in force when it starts; its
 * completions are then observed (true length = actual) before window w + 1 is predicted.
 * factors[w] = factor used for window w (nwin entries), factors[nwin] = final factor. */
int orc_profile_stream(uint64_t n, const uint32_t *true_len, const orc_predictor *p, double factor0,
                       uint32_t *pred, double *factors, uint64_t *corrections)
{
    if (!p || !corrections || (n && (!true_len || !pred || !factors))) return ORC_ERR_ARG;
    int s = check_predictor(p);
    if (s != ORC_OK) return s;
    uint64_t wl = p->window ? p->window : (n ? n : 1);
    double f = factor0;
    uint64_t w = 0;
    *corrections = 0;
    for (uint64_t a = 0; a < n; a += wl, ++w) {
        uint64_t z = a + wl < n ? a + wl : n;
        factors[w] = f;
        s = orc_predict(z - a, a, true_len + a, p, f, pred + a);
        if (s != ORC_OK) return s;
        if (p->monitor) orc_monitor_observe(z - a, pred + a, true_len + a, p->gamma, p->cap, corrections, &f);
    }
    if (factors) factors[w] = f;
    return ORC_OK;
}

/* ======================================================================== */
/* O12  HELR deployer (NEXT f3; R21).  PAPER.md Sec. 4.3, Alg. 2,
 * Eq. 4-6, with SPEC's readings of the garbled passages:
 *   m = M / Layer(M) bytes per layer (Alg. 2 line 9);
 *   max_layers(d) = min(L, floor((Memory(d) - T) / m)), 0 when Memory(d) <= T (Alg. 2 line 12,
 *                   S:354), computed exactly as floor((Memory(d) - T) * L / M);
 *   compute_cost(d, x) = p * x * m / Performance(d) (Eq. 5 term), evaluated as
 *                   ((p * x) * m) / perf in doubles;
 *   layers along a chain are filled greedily in visit order: after the visited set S the
 *   remaining layers are max(0, L - sum_{d in S} max_layers(d)) and the next device j takes
 *   min(remaining, max_layers(j));
 *   dp[{j}][j] = compute_cost(j, min(L, max_layers(j)));
 *   dp[S][j]   = min over i in S\{j} of (dp[S\{j}][i] + Latency(E[i][j])) + compute_cost(j, x_j)
 *                (Eq. 5 as a Hamiltonian-path DP over (visited set, last device));
 *   a subset is feasible iff sum max_layers >= L (Eq. 4 with the sign of Alg. 2 line 5 fixed,
 *   S:393); its objective is a1 * min_j dp[S][j] + a2 * |S| / |D|;
 *   the answer minimises (objective, chain latency, subset mask, last device) lexicographically;
 *   inside the DP the smallest predecessor i wins ties.  HE = (a1 = 0), LR = (a1 : a2 = 10 : 1)
 *   (P:337).  Device map: the chain decoded through the back-pointers, each device with its
 *   greedy layer range (devices that receive 0 layers stay on the chain with an empty range). */
typedef struct {
    uint32_t num_devices, num_layers;
    uint64_t model_bytes, kv_reserve_bytes;
    double p, a1, a2;
} orc_helr_cfg;

typedef struct {
    uint32_t count;                       /* devices on the chosen chain, in visit order */
    uint32_t feasible;                    /* 0: no subset covers the model (Eq. 4)     */
    uint32_t mask, pad;
    uint32_t device[32], layer_begin[32], layer_count[32];
    double objective, latency_s;
} orc_device_map;

static uint32_t helr_max_layers(const orc_helr_cfg *c, uint64_t mem)
{
    if (mem <= c->kv_reserve_bytes) return 0;
    unsigned __int128 q = (unsigned __int128)(mem - c->kv_reserve_bytes) * c->num_layers / c->model_bytes;
    return q >= c->num_layers ? c->num_layers : (uint32_t)q;
}

static double helr_cost(const orc_helr_cfg *c, double m, double perf, uint32_t x)
{
    return ((c->p * (double)x) * m) / perf;
}

int orc_helr(const orc_helr_cfg *c, const uint64_t *memory, const double *perf, const double *lat,
             orc_device_map *out)
{
    if (!c || !memory || !perf || !lat || !out) return ORC_ERR_ARG;
    const uint32_t D = c->num_devices, L = c->num_layers;
    if (D < 1 || D > 20 || L < 1 || c->model_bytes == 0) return ORC_ERR_CONFIG;
    if (!(c->p >= 0.0) || !(c->a1 >= 0.0) || !(c->a2 >= 0.0)) return ORC_ERR_CONFIG;
    for (uint32_t d = 0; d < D; ++d) if (!(perf[d] > 0.0)) return ORC_ERR_CONFIG;
    memset(out, 0, sizeof *out);
    const double m = (double)c->model_bytes / (double)L;
    uint32_t cap[32];
    for (uint32_t d = 0; d < D; ++d) cap[d] = helr_max_layers(c, memory[d]);
    const uint64_t NS = 1ull << D;
    double *dp = (double *)malloc(sizeof(double) * NS * D);
    uint8_t *arg = (uint8_t *)malloc(NS * D);
    uint64_t *capsum = (uint64_t *)malloc(sizeof(uint64_t) * NS);
    if (!dp || !arg || !capsum) { free(dp); free(arg); free(capsum); return ORC_ERR_ARG; }
    capsum[0] = 0;
    for (uint64_t S = 1; S < NS; ++S) {
        uint32_t low = (uint32_t)__builtin_ctzll(S);
        capsum[S] = capsum[S & (S - 1)] + cap[low];
    }
    for (uint64_t S = 1; S < NS; ++S) {                 /* numeric order: S \ {j} < S */
        for (uint32_t j = 0; j < D; ++j) {
            double *cell = &dp[S * D + j];
            arg[S * D + j] = 0xff;
            if (!((S >> j) & 1)) { *cell = INFINITY; continue; }
            uint64_t P = S & ~(1ull << j);
            uint64_t rem = capsum[P] >= L ? 0 : L - capsum[P];
            uint32_t x = rem < cap[j] ? (uint32_t)rem : cap[j];
            double cj = helr_cost(c, m, perf[j], x);
            if (P == 0) { *cell = cj; continue; }
            double best = INFINITY;
            uint32_t bi = 0xff;
            for (uint32_t i = 0; i < D; ++i) {
                if (!((P >> i) & 1)) continue;
                double v = (dp[P * D + i] + lat[i * D + j]) + cj;
                if (v < best) { best = v; bi = i; }
            }
            *cell = best;
            arg[S * D + j] = (uint8_t)bi;
        }
    }
    /* Alg. 2 lines 3-20: best subset / chain by (objective, latency, mask, last device) */
    int found = 0;
    double bobj = 0, blat = 0;
    uint64_t bS = 0;
    uint32_t bj = 0;
    for (uint64_t S = 1; S < NS; ++S) {
        if (capsum[S] < L) continue;                    /* Eq. 4 */
        double size = (double)__builtin_popcountll(S) / (double)D;
        for (uint32_t j = 0; j < D; ++j) {
            if (!((S >> j) & 1)) continue;
            double l = dp[S * D + j];
            double obj = c->a1 * l + c->a2 * size;
            if (!found || obj < bobj || (obj == bobj && l < blat)) {
                found = 1; bobj = obj; blat = l; bS = S; bj = j;
            }
        }
    }
    if (found) {
        uint32_t chain[32], k = 0;
        uint64_t S = bS;
        uint32_t j = bj;
        while (S) {
            chain[k++] = j;
            uint32_t i = arg[S * D + j];
            S &= ~(1ull << j);
            j = i;
        }
        uint64_t used = 0;
        for (uint32_t t = 0; t < k; ++t) {            /* visit order = reverse of the walk */
            uint32_t d = chain[k - 1 - t];
            uint64_t rem = used >= L ? 0 : L - used;
            uint32_t x = rem < cap[d] ? (uint32_t)rem : cap[d];
            out->device[t] = d; out->layer_begin[t] = (uint32_t)(used < L ? used : L); out->layer_count[t] = x;
            used += x;
        }
        out->count = k; out->feasible = 1; out->mask = (uint32_t)bS;
        out->objective = bobj; out->latency_s = blat;
    }
    free(dp); free(arg); free(capsum);
    return ORC_OK;
}

/* O13  BGS, the paper's baseline deployer ("Greedy Scheduling Algorithm (BGS)"), as SPEC
 * S:385-393 reads it: devices in descending order of memory (ties: smaller id first), each takes
 * max_layers(d) until the layers are exhausted; that prefix is the chain.  Its latency and
 * objective are evaluated with O12's chain formula (same operation order) for comparison. */
int orc_bgs(const orc_helr_cfg *c, const uint64_t *memory, const double *perf, const double *lat,
            orc_device_map *out)
{
    if (!c || !memory || !perf || !lat || !out) return ORC_ERR_ARG;
    const uint32_t D = c->num_devices, L = c->num_layers;
    if (D < 1 || D > 20 || L < 1 || c->model_bytes == 0) return ORC_ERR_CONFIG;
    if (!(c->p >= 0.0) || !(c->a1 >= 0.0) || !(c->a2 >= 0.0)) return ORC_ERR_CONFIG;
    for (uint32_t d = 0; d < D; ++d) if (!(perf[d] > 0.0)) return ORC_ERR_CONFIG;
    memset(out, 0, sizeof *out);
    uint32_t ord[32];
    for (uint32_t d = 0; d < D; ++d) ord[d] = d;
    for (uint32_t a = 1; a < D; ++a) {                  /* insertion sort: memory desc, id asc */
        uint32_t x = ord[a], b = a;
        while (b > 0 && memory[ord[b - 1]] < memory[x]) { ord[b] = ord[b - 1]; --b; }
        ord[b] = x;
    }
    const double m = (double)c->model_bytes / (double)L;
    uint64_t used = 0;
    uint32_t k = 0, mask = 0;
    double l = 0.0;
    while (used < L && k < D) {
        uint32_t d = ord[k];
        uint32_t cap = helr_max_layers(c, memory[d]);
        uint64_t rem = L - used;
        uint32_t x = rem < cap ? (uint32_t)rem : cap;
        double cst = helr_cost(c, m, perf[d], x);
        l = k == 0 ? cst : (l + lat[ord[k - 1] * D + d]) + cst;
        out->device[k] = d; out->layer_begin[k] = (uint32_t)used; out->layer_count[k] = x;
        used += cap;
        mask |= 1u << d;
        ++k;
    }
    if (used < L) { memset(out, 0, sizeof *out); return ORC_OK; }   /* infeasible */
    out->count = k; out->feasible = 1; out->mask = mask;
    out->latency_s = l;
    out->objective = c->a1 * l + c->a2 * ((double)k / (double)D);
    return ORC_OK;
}

/* ABI self-description for the Python side (sizes checked by tests). */
uint64_t orc_sizeof_config(void) { return sizeof(orc_config); }
uint64_t orc_sizeof_batch_stat(void) { return sizeof(orc_batch_stat); }
uint64_t orc_sizeof_totals(void) { return sizeof(orc_totals); }
uint64_t orc_sizeof_sim_totals(void) { return sizeof(orc_sim_totals); }
uint64_t orc_sizeof_predictor(void) { return sizeof(orc_predictor); }
uint64_t orc_sizeof_device_map(void) { return sizeof(orc_device_map); }
