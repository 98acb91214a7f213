/*
 * rtgpu_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference schedulability analysis
 * (reference: pkg/src/gpusched/{suspension,gpu,analysis}.py) used as the
 * parity checker for the CUDA engine and as the `cpu_baseline` leg of
 * bench.py.  Nothing in the product path links or calls this file.
 *
 * Exactness.  The reference computes in exact rationals (fractions.Fraction).
 * For one SM allocation every quantity of the analysis is a rational whose
 * denominator divides Q = 2 * A * lcm(GN_i) input ticks (A = common
 * denominator of the interleave ratios; GN_i physical SMs per GPU task):
 * Lemma 4 (gpu.py:25) is the only place that divides, and everything after
 * it (gaps, chain workloads, fixed points, sums, min/max, comparisons) is
 * additive.  So the oracle scales every input by Q and computes in 128-bit
 * integers, checking every operation for overflow (overflow -> status
 * RTGPU_RANGE, never a silently wrong answer).  Results are (num, Q) pairs.
 *
 * Faithfulness.  Default mode restates the reference loop for loop:
 * lexicographic allocation enumeration (gpu.py:43,69), per-allocation
 * evaluation stopping at the first failing task (analysis.py:280), the
 * literal greedy chain walk (suspension.py:77) and the literal fixed-point
 * iteration from the base (suspension.py:123).  The reference's memo
 * (analysis.py:127) only caches values and is omitted.
 *
 * Baselines.  analysis.py:319/355 call SuspTask, task_response and
 * ExecBounds without importing them (NameError at run time in the
 * reference).  The oracle restates their evident intent -- the code as
 * written with the missing imports present -- and tests pin it against
 * the reference run with those three names injected (tests/golden).
 */
#include <setjmp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/rtgpu.h"
#include "rtgpu_oracle.h"

typedef __int128 i128;

#define MAXT RTGPU_MAX_TASKS
#define MAXM RTGPU_MAX_M
#define MAXP (2 * RTGPU_MAX_M - 2)
#define MAXG (RTGPU_MAX_M - 1)

enum { ERR_RANGE = 1, ERR_INVALID = 2, ERR_BUDGET = 3 };

typedef struct {
    jmp_buf jb;
    int64_t evals;
    int64_t budget;
} octx;

static i128 ck_add(octx *c, i128 a, i128 b) {
    i128 r;
    if (__builtin_add_overflow(a, b, &r)) longjmp(c->jb, ERR_RANGE);
    return r;
}
static i128 ck_sub(octx *c, i128 a, i128 b) {
    i128 r;
    if (__builtin_sub_overflow(a, b, &r)) longjmp(c->jb, ERR_RANGE);
    return r;
}
static i128 ck_mul(octx *c, i128 a, i128 b) {
    i128 r;
    if (__builtin_mul_overflow(a, b, &r)) longjmp(c->jb, ERR_RANGE);
    return r;
}
static i128 gcd128(i128 a, i128 b) {
    if (a < 0) a = -a;
    if (b < 0) b = -b;
    while (b) {
        i128 t = a % b;
        a = b;
        b = t;
    }
    return a;
}

/* ---------------------------------------------------------------- input */

typedef struct {
    int m, p, g;
    int64_t D, T, prio;
    int64_t seg_off;
    const int64_t *cl_lo, *cl_hi, *ml_lo, *ml_hi, *gw_lo, *gw_hi, *gl, *an;
} otask;

typedef struct {
    int n, gn, mm;
    int64_t A;
    otask t[MAXT];
} oset;

/* int64 copy of compact (int32) segment areas */
static __thread int64_t seg64[MAXT * (2 * MAXM + 2 * MAXP + 4 * MAXG)];

static int parse_set(const int64_t *b, oset *s) {
    const int compact = b[7] == 1 || b[7] == 2; /* 2: int32 task records too */
    int64_t used64 = 0;
    s->n = (int)b[0];
    s->gn = (int)b[1];
    s->mm = (int)b[2];
    s->A = b[3];
    if (s->n < 0 || s->n > MAXT || s->A < 1 || (s->mm != 0 && s->mm != 1)) return -1;
    for (int i = 0; i < s->n; i++) {
        otask *t = &s->t[i];
        t->m = (int)rtgpu_rec_word(b, i, 0);
        t->p = (int)rtgpu_rec_word(b, i, 1);
        t->g = t->m - 1;
        t->D = rtgpu_rec_word(b, i, 2);
        t->T = rtgpu_rec_word(b, i, 3);
        t->prio = rtgpu_rec_word(b, i, 4);
        t->seg_off = rtgpu_rec_word(b, i, 5);
        if (t->m < 1 || t->m > MAXM || t->p < 0 || t->p > MAXP) return -1;
        const int64_t *q = b + t->seg_off;
        if (compact) {
            const int32_t *q32 = (const int32_t *)b + t->seg_off;
            const int words = 2 * t->m + 2 * t->p + 4 * t->g;
            for (int j = 0; j < words; j++) seg64[used64 + j] = q32[j];
            q = seg64 + used64;
            used64 += words;
        }
        t->cl_lo = q;
        t->cl_hi = q + t->m;
        t->ml_lo = q + 2 * t->m;
        t->ml_hi = t->ml_lo + t->p;
        t->gw_lo = t->ml_hi + t->p;
        t->gw_hi = t->gw_lo + t->g;
        t->gl = t->gw_hi + t->g;
        t->an = t->gl + t->g;
    }
    return 0;
}

/* ------------------------------------------------- per-allocation view */

/* Everything of one task scaled to units of 1/Q input ticks. */
typedef struct {
    i128 D, T;
    i128 clu[MAXM], cll[MAXM], mlu[MAXP], mll[MAXP], grl[MAXG], gru[MAXG];
    i128 sum_clu, sum_cll, sum_mlu, sum_mll, sum_grl, sum_gru;
    int vs; /* virtual SMs, 0 for pure-CPU */
} sview;

typedef struct {
    const oset *s;
    i128 Q;
    sview v[MAXT];
} aview;

/* gpu.py:25 gpu_response_bounds, scaled: lo = gw_lo/vs,
 * hi = (gw_hi*alpha - gl)/vs + gl, vs = 2*GN, alpha = an/A. */
static void build_view(octx *c, const oset *s, const int *gn, aview *av) {
    i128 L = 1;
    int any_gpu = 0;
    for (int i = 0; i < s->n; i++) {
        if (s->t[i].g > 0) {
            any_gpu = 1;
            i128 g = gn[i];
            L = ck_mul(c, L / gcd128(L, g), g);
        }
    }
    i128 Q = any_gpu ? ck_mul(c, ck_mul(c, L, 2), s->A) : 1;
    av->s = s;
    av->Q = Q;
    for (int i = 0; i < s->n; i++) {
        const otask *t = &s->t[i];
        sview *v = &av->v[i];
        v->D = ck_mul(c, t->D, Q);
        v->T = ck_mul(c, t->T, Q);
        v->sum_clu = v->sum_cll = v->sum_mlu = v->sum_mll = 0;
        v->sum_grl = v->sum_gru = 0;
        for (int j = 0; j < t->m; j++) {
            v->clu[j] = ck_mul(c, t->cl_hi[j], Q);
            v->cll[j] = ck_mul(c, t->cl_lo[j], Q);
            v->sum_clu = ck_add(c, v->sum_clu, v->clu[j]);
            v->sum_cll = ck_add(c, v->sum_cll, v->cll[j]);
        }
        for (int j = 0; j < t->p; j++) {
            v->mlu[j] = ck_mul(c, t->ml_hi[j], Q);
            v->mll[j] = ck_mul(c, t->ml_lo[j], Q);
            v->sum_mlu = ck_add(c, v->sum_mlu, v->mlu[j]);
            v->sum_mll = ck_add(c, v->sum_mll, v->mll[j]);
        }
        v->vs = t->g > 0 ? 2 * gn[i] : 0;
        for (int j = 0; j < t->g; j++) {
            i128 vs = v->vs;
            i128 per_lo = Q / vs;                      /* exact: vs | Q */
            i128 per_hi = Q / ck_mul(c, vs, s->A);     /* exact: vs*A | Q */
            v->grl[j] = ck_mul(c, t->gw_lo[j], per_lo);
            i128 infl = ck_sub(c, ck_mul(c, t->gw_hi[j], t->an[j]),
                               ck_mul(c, t->gl[j], s->A));
            v->gru[j] = ck_add(c, ck_mul(c, infl, per_hi), ck_mul(c, t->gl[j], Q));
            v->sum_grl = ck_add(c, v->sum_grl, v->grl[j]);
            v->sum_gru = ck_add(c, v->sum_gru, v->gru[j]);
        }
    }
}

/* ------------------------------------------------------------ gaps */

/* analysis.py:89 cpu_inter_arrival.  Returns 1 on InfeasibleGapError. */
static int cpu_gap(octx *c, const aview *av, int i, int64_t j, i128 *out) {
    const otask *t = &av->s->t[i];
    const sview *v = &av->v[i];
    int m = t->m;
    int64_t jp = j % m;
    if (jp != m - 1) {
        if (av->s->mm == RTGPU_TWO_COPY)
            *out = ck_add(c, ck_add(c, v->mll[2 * jp], v->grl[jp]), v->mll[2 * jp + 1]);
        else
            *out = ck_add(c, v->mll[jp], v->grl[jp]);
        return 0;
    }
    if (j == m - 1) {
        *out = ck_sub(c, v->T, v->D);
        return 0;
    }
    i128 wrap = ck_sub(c, ck_sub(c, ck_sub(c, v->T, v->sum_clu), v->sum_mll), v->sum_grl);
    if (wrap < 0) return 1;
    *out = wrap;
    return 0;
}

/* analysis.py:57 mem_inter_arrival. */
static int mem_gap(octx *c, const aview *av, int i, int64_t j, i128 *out) {
    const otask *t = &av->s->t[i];
    const sview *v = &av->v[i];
    int p = t->p, m = t->m;
    int64_t jp = j % p;
    if (av->s->mm == RTGPU_TWO_COPY) {
        if (jp != p - 1) {
            *out = (jp % 2 == 0) ? v->grl[jp / 2] : v->cll[(jp + 1) / 2];
            return 0;
        }
        if (j == p - 1) {
            i128 x = ck_add(c, ck_add(c, ck_sub(c, v->T, v->D), v->cll[m - 1]), v->cll[0]);
            if (x < 0) return 1;
            *out = x;
            return 0;
        }
    } else {
        if (jp != p - 1) {
            *out = ck_add(c, v->grl[jp], v->cll[jp + 1]);
            return 0;
        }
        if (j == p - 1) {
            i128 x = ck_add(c, ck_add(c, ck_add(c, ck_sub(c, v->T, v->D), v->grl[m - 2]),
                                      v->cll[m - 1]), v->cll[0]);
            if (x < 0) return 1;
            *out = x;
            return 0;
        }
    }
    i128 inner = 0;
    for (int q = 1; q < m - 1; q++) inner = ck_add(c, inner, v->cll[q]);
    i128 wrap = ck_sub(c, ck_sub(c, ck_sub(c, v->T, v->sum_mlu), inner), v->sum_grl);
    if (wrap < 0) return 1;
    *out = wrap;
    return 0;
}

/* suspension.py:65 inter_arrival for a SuspTask given by arrays. */
typedef struct {
    int m;
    i128 D, T;
    i128 eh[MAXM], el[MAXM], sh[MAXG], sl[MAXG];
    i128 sum_eh, sum_sh, sum_sl;
} susp;

static i128 susp_gap(octx *c, const susp *t, int64_t j) {
    int m = t->m;
    int64_t jp = j % m;
    if (jp != m - 1) return t->sl[jp];
    if (j == m - 1) return ck_sub(c, t->T, t->D);
    return ck_sub(c, ck_sub(c, t->T, t->sum_eh), t->sum_sl);
}

/* ----------------------------------------------------- chain workload */

enum { K_CPU = 0, K_MEM = 1 };

/* suspension.py:77 chain_workload, literal greedy walk.  Returns 1 on an
 * InfeasibleGapError raised by a gap evaluation. */
static int chain_rtgpu(octx *c, const aview *av, int i, int kind, int64_t h,
                       i128 horizon, i128 *out) {
    const otask *t = &av->s->t[i];
    const sview *v = &av->v[i];
    int p = kind == K_CPU ? t->m : t->p;
    const i128 *ex = kind == K_CPU ? v->clu : v->mlu;
    if (p == 0 || horizon <= 0) {
        *out = 0;
        return 0;
    }
    i128 cum = 0, work = 0;
    int64_t j = h;
    int64_t guard = 0;
    for (;;) {
        i128 seg = ex[j % p], g;
        int e = kind == K_CPU ? cpu_gap(c, av, i, j, &g) : mem_gap(c, av, i, j, &g);
        if (e) return 1;
        i128 step = ck_add(c, seg, g);
        if (ck_add(c, cum, step) <= horizon) {
            cum = ck_add(c, cum, step);
            work = ck_add(c, work, seg);
            j++;
            /* more than two periods of zero-length steps: the chain is
             * all zero and the reference loop never returns */
            if (step != 0) guard = 0;
            else if (++guard > 2 * (int64_t)p + 2) longjmp(c->jb, ERR_INVALID);
        } else {
            i128 tail = ck_sub(c, horizon, cum);
            if (seg < tail) tail = seg;
            *out = ck_add(c, work, tail > 0 ? tail : 0);
            return 0;
        }
    }
}

static i128 chain_susp(octx *c, const susp *t, int64_t h, i128 horizon) {
    int p = t->m;
    if (p == 0 || horizon <= 0) return 0;
    i128 cum = 0, work = 0;
    int64_t j = h, guard = 0;
    for (;;) {
        i128 seg = t->eh[j % p];
        i128 g = susp_gap(c, t, j);
        i128 step = ck_add(c, seg, g);
        if (ck_add(c, cum, step) <= horizon) {
            cum = ck_add(c, cum, step);
            work = ck_add(c, work, seg);
            j++;
            if (step != 0) guard = 0;
            else if (++guard > 2 * (int64_t)p + 2) longjmp(c->jb, ERR_INVALID);
        } else {
            i128 tail = ck_sub(c, horizon, cum);
            if (seg < tail) tail = seg;
            return ck_add(c, work, tail > 0 ? tail : 0);
        }
    }
}

/* analysis.py:131 _max_workload (memo omitted). */
static int max_workload_rtgpu(octx *c, const aview *av, int i, int kind, i128 horizon,
                              i128 *out) {
    const otask *t = &av->s->t[i];
    int ns = kind == K_MEM ? t->p : t->m;
    if (ns == 0 || horizon <= 0) {
        *out = 0;
        return 0;
    }
    i128 best = 0;
    for (int h = 0; h < ns; h++) {
        i128 w;
        if (chain_rtgpu(c, av, i, kind, h, horizon, &w)) return 1;
        if (h == 0 || w > best) best = w;
    }
    *out = best;
    return 0;
}

/* suspension.py:116 max_workload. */
static i128 max_workload_susp(octx *c, const susp *t, i128 horizon) {
    if (horizon <= 0) return 0;
    i128 best = 0;
    for (int h = 0; h < t->m; h++) {
        i128 w = chain_susp(c, t, h, horizon);
        if (h == 0 || w > best) best = w;
    }
    return best;
}

/* ------------------------------------------------------ fixed points */

#define NONE128 ((i128)-1)

/* Interference of a higher-priority set at horizon r. */
typedef struct {
    const aview *av;
    int kind;
    int hp[MAXT];
    int nhp;
} rtgpu_intf;

static int intf_rtgpu(octx *c, const rtgpu_intf *f, i128 r, i128 *out) {
    i128 acc = 0;
    for (int q = 0; q < f->nhp; q++) {
        i128 w;
        if (max_workload_rtgpu(c, f->av, f->hp[q], f->kind, r, &w)) return 1;
        acc = ck_add(c, acc, w);
    }
    *out = acc;
    return 0;
}

/* suspension.py:123 fixed_point; gap errors (InfeasibleGapError) make the
 * caller's result None, as in analysis.py:165-172. */
static i128 fixed_point_rtgpu(octx *c, i128 base, const rtgpu_intf *f, i128 bound) {
    if (base > bound) return NONE128;
    i128 r = base;
    for (;;) {
        i128 I;
        if (intf_rtgpu(c, f, r, &I)) return NONE128;
        i128 nxt = ck_add(c, base, I);
        if (nxt == r) return r;
        if (nxt > bound) return NONE128;
        r = nxt;
    }
}

typedef struct {
    const susp *t[MAXT];
    int nhp;
} susp_intf;

static i128 fixed_point_susp(octx *c, i128 base, const susp_intf *f, i128 bound) {
    if (base > bound) return NONE128;
    i128 r = base;
    for (;;) {
        i128 I = 0;
        for (int q = 0; q < f->nhp; q++) I = ck_add(c, I, max_workload_susp(c, f->t[q], r));
        i128 nxt = ck_add(c, base, I);
        if (nxt == r) return r;
        if (nxt > bound) return NONE128;
        r = nxt;
    }
}

/* ---------------------------------------------------- RTGPU evaluate */

typedef struct {
    int present;
    i128 e2e;
    i128 cpu_r[MAXM];
    i128 mem_r[MAXP];
} trep;

/* analysis.py:156 mem_response */
static i128 mem_response(octx *c, const aview *av, int k, int j) {
    const oset *s = av->s;
    rtgpu_intf f;
    f.av = av;
    f.kind = K_MEM;
    f.nhp = 0;
    i128 blocking = 0;
    for (int i = 0; i < s->n; i++) {
        if (s->t[i].prio < s->t[k].prio && s->t[i].p > 0) f.hp[f.nhp++] = i;
        if (s->t[i].prio > s->t[k].prio)
            for (int q = 0; q < s->t[i].p; q++)
                if (av->v[i].mlu[q] > blocking) blocking = av->v[i].mlu[q];
    }
    i128 base = ck_add(c, av->v[k].mlu[j], blocking);
    return fixed_point_rtgpu(c, base, &f, av->v[k].D);
}

static void hp_all(const aview *av, int k, int kind, rtgpu_intf *f) {
    f->av = av;
    f->kind = kind;
    f->nhp = 0;
    for (int i = 0; i < av->s->n; i++)
        if (av->s->t[i].prio < av->s->t[k].prio) f->hp[f->nhp++] = i;
}

/* analysis.py:175 cpu_response */
static i128 cpu_response(octx *c, const aview *av, int k, int j) {
    rtgpu_intf f;
    hp_all(av, k, K_CPU, &f);
    return fixed_point_rtgpu(c, av->v[k].clu[j], &f, av->v[k].D);
}

/* analysis.py:191 end_to_end */
static i128 end_to_end(octx *c, const aview *av, int k, const trep *r) {
    const otask *t = &av->s->t[k];
    const sview *v = &av->v[k];
    for (int j = 0; j < t->p; j++)
        if (r->mem_r[j] == NONE128) return NONE128;
    i128 mr = 0;
    for (int j = 0; j < t->p; j++) mr = ck_add(c, mr, r->mem_r[j]);
    i128 r1 = NONE128;
    int all = 1;
    i128 cs = 0;
    for (int j = 0; j < t->m; j++) {
        if (r->cpu_r[j] == NONE128) all = 0;
        else cs = ck_add(c, cs, r->cpu_r[j]);
    }
    if (all) {
        i128 cand = ck_add(c, ck_add(c, v->sum_gru, mr), cs);
        if (cand <= v->D) r1 = cand;
    }
    rtgpu_intf f;
    hp_all(av, k, K_CPU, &f);
    i128 r2 = fixed_point_rtgpu(c, ck_add(c, ck_add(c, v->sum_gru, mr), v->sum_clu), &f, v->D);
    if (r1 == NONE128) return r2;
    if (r2 == NONE128) return r1;
    return r1 < r2 ? r1 : r2;
}

/* analysis.py:280 evaluate (RTGPU).  Returns 1 if all tasks pass. */
static int eval_rtgpu(octx *c, const aview *av, trep *rep) {
    const oset *s = av->s;
    for (int k = 0; k < s->n; k++) rep[k].present = 0;
    for (int k = 0; k < s->n; k++) {
        if (c->budget > 0 && c->evals >= c->budget) longjmp(c->jb, ERR_BUDGET);
        c->evals++;
        const otask *t = &s->t[k];
        for (int j = 0; j < t->p; j++) rep[k].mem_r[j] = mem_response(c, av, k, j);
        for (int j = 0; j < t->m; j++) rep[k].cpu_r[j] = cpu_response(c, av, k, j);
        rep[k].e2e = end_to_end(c, av, k, &rep[k]);
        rep[k].present = 1;
        if (rep[k].e2e == NONE128 || rep[k].e2e > av->v[k].D) return 0;
    }
    return 1;
}

/* ------------------------------------------------------- baselines */

/* suspension.py:35 SuspTask.__post_init__ validation. */
static int susp_valid(const susp *t) {
    if (t->m < 1) return 0;
    if (!(0 < t->D && t->D <= t->T)) return 0;
    for (int j = 0; j < t->m; j++)
        if (!(0 <= t->el[j] && t->el[j] <= t->eh[j])) return 0;
    for (int j = 0; j < t->m - 1; j++)
        if (!(0 <= t->sl[j] && t->sl[j] <= t->sh[j])) return 0;
    return t->sum_eh + t->sum_sl <= t->T;
}

static void susp_sums(octx *c, susp *t) {
    t->sum_eh = t->sum_sh = t->sum_sl = 0;
    for (int j = 0; j < t->m; j++) t->sum_eh = ck_add(c, t->sum_eh, t->eh[j]);
    for (int j = 0; j < t->m - 1; j++) {
        t->sum_sh = ck_add(c, t->sum_sh, t->sh[j]);
        t->sum_sl = ck_add(c, t->sum_sl, t->sl[j]);
    }
}

/* suspension.py:155 task_response */
static i128 task_response(octx *c, const susp *k, const susp_intf *f, i128 blocking) {
    i128 r1 = k->sum_sh;
    for (int j = 0; j < k->m; j++) {
        i128 seg = fixed_point_susp(c, ck_add(c, k->eh[j], blocking), f, k->D);
        if (seg == NONE128) {
            r1 = NONE128;
            break;
        }
        r1 = ck_add(c, r1, seg);
    }
    if (r1 != NONE128 && r1 > k->D) r1 = NONE128;
    i128 base = ck_add(c, ck_add(c, k->sum_sh, k->sum_eh), blocking);
    i128 r2 = fixed_point_susp(c, base, f, k->D);
    if (r1 == NONE128) return r2;
    if (r2 == NONE128) return r1;
    return r1 < r2 ? r1 : r2;
}

/* analysis.py:303 _suspension_bounds / analysis.py:360 busy-wait mapping */
static void map_susp(octx *c, const aview *av, int i, int method, susp *o) {
    const otask *t = &av->s->t[i];
    const sview *v = &av->v[i];
    o->D = v->D;
    o->T = v->T;
    if (method == RTGPU_METHOD_SELFSUSP) {
        o->m = t->m;
        for (int j = 0; j < t->m; j++) {
            o->eh[j] = v->clu[j];
            o->el[j] = v->cll[j];
        }
        for (int j = 0; j < t->m - 1; j++) {
            if (av->s->mm == RTGPU_TWO_COPY) {
                o->sl[j] = ck_add(c, ck_add(c, v->mll[2 * j], v->grl[j]), v->mll[2 * j + 1]);
                o->sh[j] = ck_add(c, ck_add(c, v->mlu[2 * j], v->gru[j]), v->mlu[2 * j + 1]);
            } else {
                o->sl[j] = ck_add(c, v->mll[j], v->grl[j]);
                o->sh[j] = ck_add(c, v->mlu[j], v->gru[j]);
            }
        }
    } else {
        o->m = 1;
        o->el[0] = ck_add(c, ck_add(c, v->sum_cll, v->sum_mll), v->sum_grl);
        o->eh[0] = ck_add(c, ck_add(c, v->sum_clu, v->sum_mlu), v->sum_gru);
    }
    susp_sums(c, o);
}

static int eval_baseline(octx *c, const aview *av, int method, trep *rep) {
    const oset *s = av->s;
    static __thread susp mapped[MAXT];
    for (int k = 0; k < s->n; k++) rep[k].present = 0;
    for (int i = 0; i < s->n; i++) {
        map_susp(c, av, i, method, &mapped[i]);
        if (!susp_valid(&mapped[i])) return 0; /* ValueError -> (False, {}) */
    }
    for (int k = 0; k < s->n; k++) {
        if (c->budget > 0 && c->evals >= c->budget) longjmp(c->jb, ERR_BUDGET);
        c->evals++;
        susp_intf f;
        f.nhp = 0;
        i128 blocking = 0;
        for (int i = 0; i < s->n; i++) {
            if (s->t[i].prio < s->t[k].prio) f.t[f.nhp++] = &mapped[i];
            if (method == RTGPU_METHOD_SELFSUSP && s->t[i].prio > s->t[k].prio)
                for (int q = 0; q < mapped[i].m - 1; q++)
                    if (mapped[i].sh[q] > blocking) blocking = mapped[i].sh[q];
        }
        rep[k].e2e = task_response(c, &mapped[k], &f, blocking);
        rep[k].present = 1;
        if (rep[k].e2e == NONE128 || rep[k].e2e > av->v[k].D) return 0;
    }
    return 1;
}

/* ------------------------------------------------------ grid search */

/* analysis.py:239 _min_feasible_gn, exact: sum_j[(gw_hi*a/A - gl)/(2gn) + gl]
 * + sum ml_hi + sum cl_hi <= D.  Raises (INVALID) like gpu.py:36 when the
 * overhead exceeds the inflated work. */
static int min_feasible_gn(octx *c, const oset *s, int i) {
    const otask *t = &s->t[i];
    i128 infl = 0, fixed = 0;
    for (int gn = 1; gn <= s->gn; gn++) {
        if (gn == 1) {
            for (int j = 0; j < t->g; j++) {
                i128 w = ck_mul(c, t->gw_hi[j], t->an[j]);
                i128 o = ck_mul(c, t->gl[j], s->A);
                if (o > w) longjmp(c->jb, ERR_INVALID);
                infl = ck_add(c, infl, ck_sub(c, w, o));
                fixed = ck_add(c, fixed, t->gl[j]);
            }
            for (int j = 0; j < t->p; j++) fixed = ck_add(c, fixed, t->ml_hi[j]);
            for (int j = 0; j < t->m; j++) fixed = ck_add(c, fixed, t->cl_hi[j]);
        }
        /* infl/(2*A*gn) + fixed <= D  <=>  infl + 2*A*gn*(fixed - D) <= 0 */
        i128 lhs = ck_add(c, infl, ck_mul(c, ck_mul(c, 2 * (i128)gn, s->A),
                                          ck_sub(c, fixed, t->D)));
        if (lhs <= 0) return gn;
    }
    return 0;
}

static void write_report(const oset *s, const aview *av, const trep *rep, int method,
                         const int *gn, int has_alloc, int64_t *blob_detail,
                         int32_t *vsm, int64_t *e2e_num, int64_t *den, int *range_err) {
    for (int k = 0; k < s->n; k++) {
        const otask *t = &s->t[k];
        vsm[k] = (has_alloc && t->g > 0) ? 2 * gn[k] : 0;
        if (!rep || !rep[k].present) {
            e2e_num[k] = RTGPU_ABSENT;
            den[k] = 1;
            if (blob_detail) {
                int64_t *d = blob_detail + t->seg_off;
                for (int j = 0; j < 2 * t->m + 2 * t->p + 4 * t->g; j++) d[j] = RTGPU_ABSENT;
            }
            continue;
        }
        /* reduce all values of the task by a common gcd with Q */
        const sview *v = &av->v[k];
        i128 g = av->Q;
        g = gcd128(g, rep[k].e2e == NONE128 ? 0 : rep[k].e2e);
        if (blob_detail) {
            for (int j = 0; j < t->g; j++) g = gcd128(gcd128(g, v->grl[j]), v->gru[j]);
            if (method == RTGPU_METHOD_RTGPU) {
                for (int j = 0; j < t->m; j++)
                    if (rep[k].cpu_r[j] != NONE128) g = gcd128(g, rep[k].cpu_r[j]);
                for (int j = 0; j < t->p; j++)
                    if (rep[k].mem_r[j] != NONE128) g = gcd128(g, rep[k].mem_r[j]);
            }
        }
        if (g == 0) g = 1;
        i128 q = av->Q / g;
        const i128 lim = (i128)INT64_MAX;
#define OUTV(x) ((x) == NONE128 ? (int64_t)RTGPU_NONE : ((x) / g > lim ? (*range_err = 1, 0) : (int64_t)((x) / g)))
        if (q > lim) *range_err = 1;
        den[k] = (int64_t)q;
        e2e_num[k] = OUTV(rep[k].e2e);
        if (blob_detail) {
            int64_t *d = blob_detail + t->seg_off;
            int64_t *cl = d, *clh = d + t->m, *ml = d + 2 * t->m, *mlh = ml + t->p;
            int64_t *gl = mlh + t->p, *gh = gl + t->g, *x1 = gh + t->g, *x2 = x1 + t->g;
            for (int j = 0; j < t->m; j++) {
                cl[j] = method == RTGPU_METHOD_RTGPU ? OUTV(rep[k].cpu_r[j]) : RTGPU_ABSENT;
                clh[j] = RTGPU_ABSENT;
            }
            for (int j = 0; j < t->p; j++) {
                ml[j] = method == RTGPU_METHOD_RTGPU ? OUTV(rep[k].mem_r[j]) : RTGPU_ABSENT;
                mlh[j] = RTGPU_ABSENT;
            }
            for (int j = 0; j < t->g; j++) {
                gl[j] = OUTV(v->grl[j]);
                gh[j] = OUTV(v->gru[j]);
                x1[j] = x2[j] = RTGPU_ABSENT;
            }
        }
#undef OUTV
    }
}

/* Greedy restatement (flags & ORACLE_GREEDY): each GPU task in priority
 * order takes the smallest count at which the faithful per-allocation
 * evaluation (eval_rtgpu: literal walks and literal iteration) passes it,
 * given the counts already chosen; later tasks sit at their minimum (they do
 * not influence earlier tasks).  DESIGN.md section 3 shows this equals the
 * reference's lexicographic grid search for regular task sets; tests check
 * it against the full enumeration above on small sets and use it as the
 * checker where the enumeration cannot finish (148 SMs). */
static int greedy_rtgpu(octx *c, const oset *s, const int *mins, int *gn, aview *av, trep *rep) {
    for (int k = 0; k < s->n; k++) gn[k] = s->t[k].g > 0 ? mins[k] : 0;
    int64_t used = 0;
    for (int k = 0; k < s->n; k++) {
        const otask *t = &s->t[k];
        if (t->g == 0) {
            build_view(c, s, gn, av);
            eval_rtgpu(c, av, rep);
            if (!rep[k].present || rep[k].e2e == NONE128) return 0;
            continue;
        }
        int64_t after = 0;
        for (int i = k + 1; i < s->n; i++)
            if (s->t[i].g > 0) after += mins[i];
        int64_t gmax = s->gn - used - after;
        int found = 0;
        for (int g = mins[k]; g <= gmax && !found; g++) {
            gn[k] = g;
            build_view(c, s, gn, av);
            eval_rtgpu(c, av, rep);
            /* task k passes iff the evaluation got past it */
            if (rep[k].present && rep[k].e2e != NONE128 && rep[k].e2e <= av->v[k].D) found = g;
        }
        if (!found) return 0;
        gn[k] = found;
        used += found;
    }
    return 1;
}

#define ORACLE_GREEDY 0x100u
#define ORACLE_PREFIX 0x200u

/* Prefix-pruned enumeration (flags & ORACLE_PREFIX): the reference's
 * lexicographic grid search (analysis.py:250 over gpu.py:43 _compositions),
 * skipping only subtrees whose prefix already fails.  It rests on nothing
 * but the prefix property visible in analysis.py:156-217 -- task k's bounds
 * read the counts of higher-priority tasks only (interference from hp(k);
 * the blocking term is lower-priority copy lengths, independent of the
 * allocation) -- and NOT on the monotonicity / dominance argument the
 * engine's greedy descent and ORACLE_GREEDY use.  Same first schedulable
 * allocation as the full enumeration; the budget (task evaluations) makes
 * undecidable sets RTGPU_UNDECIDED.  Returns 1 schedulable (gn holds the
 * allocation), 0 unschedulable. */
static int prefix_rtgpu(octx *c, const oset *s, const int *mins, const int *ids, int nid, int *gn, aview *av,
                        trep *rep) {
    int x[MAXT];
    for (int k = 0; k < s->n; k++) gn[k] = s->t[k].g > 0 ? mins[k] : 0;
    if (nid == 0) {
        build_view(c, s, gn, av);
        return eval_rtgpu(c, av, rep);
    }
    int q = 0;
    x[0] = mins[ids[0]] - 1;
    for (;;) {
        /* next count of GPU task q within its range, else backtrack */
        int64_t used = 0, after = 0;
        for (int a = 0; a < q; a++) used += x[a];
        for (int a = q + 1; a < nid; a++) after += mins[ids[a]];
        if (x[q] + 1 > s->gn - used - after) {
            gn[ids[q]] = mins[ids[q]];
            if (--q < 0) return 0;
            continue;
        }
        x[q]++;
        gn[ids[q]] = x[q];
        build_view(c, s, gn, av);
        int ok = eval_rtgpu(c, av, rep);
        if (ok) return 1;
        /* first failing task; tasks before GPU task q + 1 depend on x[0..q] only */
        int f = 0;
        while (f < s->n && rep[f].present && rep[f].e2e != NONE128 && rep[f].e2e <= av->v[f].D) f++;
        const int next_pos = q + 1 < nid ? ids[q + 1] : s->n;
        if (f < next_pos) continue; /* this prefix fails for every completion */
        q++;
        x[q] = mins[ids[q]] - 1;
    }
}

int oracle_analyze_set(const int64_t *blob, int method, unsigned flags, int64_t budget,
                       int32_t *status, int64_t *evals, int32_t *vsm, int64_t *e2e_num,
                       int64_t *den, int64_t *blob_detail) {
    static __thread oset s;
    static __thread aview av;
    static __thread trep rep[MAXT];
    static __thread trep last[MAXT];
    static __thread aview last_av;
    octx c;
    c.evals = 0;
    c.budget = budget;
    int gn[MAXT], mins[MAXT];
    int range_err = 0;
    (void)flags;
    if (parse_set(blob, &s)) {
        *status = RTGPU_INVALID;
        *evals = 0;
        return 0;
    }
    for (int k = 0; k < s.n; k++) {
        vsm[k] = 0;
        e2e_num[k] = RTGPU_ABSENT;
        den[k] = 1;
    }
    int rc = setjmp(c.jb);
    if (rc) {
        *status = rc == ERR_RANGE ? RTGPU_RANGE : rc == ERR_BUDGET ? RTGPU_UNDECIDED : RTGPU_INVALID;
        *evals = c.evals;
        for (int k = 0; k < s.n; k++) {
            vsm[k] = 0;
            e2e_num[k] = RTGPU_ABSENT;
            den[k] = 1;
        }
        return 0;
    }
    /* analysis.py:250 _grid_search */
    int ids[MAXT], nid = 0;
    for (int k = 0; k < s.n; k++) {
        const otask *t = &s.t[k];
        if (t->g > 0) {
            int g = min_feasible_gn(&c, &s, k);
            if (!g) goto unsched_empty;
            mins[k] = g;
            ids[nid++] = k;
        } else {
            i128 iso = 0;
            for (int j = 0; j < t->p; j++) iso += t->ml_hi[j];
            for (int j = 0; j < t->m; j++) iso += t->cl_hi[j];
            if (iso > t->D) goto unsched_empty;
            mins[k] = 0;
        }
    }
    if ((flags & ORACLE_GREEDY) && method == RTGPU_METHOD_RTGPU) {
        int64_t need = 0;
        for (int q = 0; q < nid; q++) need += mins[ids[q]];
        if (need > s.gn) goto unsched_empty;
        int ok = greedy_rtgpu(&c, &s, mins, gn, &av, rep);
        *status = ok ? RTGPU_SCHEDULABLE : RTGPU_UNSCHEDULABLE;
        *evals = c.evals;
        if (!ok) {
            /* the reference reports the lexicographically last allocation */
            int first = -1;
            int64_t others = 0;
            for (int q = 0; q < nid; q++) {
                if (first < 0) first = ids[q];
                else others += mins[ids[q]];
            }
            for (int k = 0; k < s.n; k++)
                gn[k] = s.t[k].g > 0 ? (k == first ? (int)(s.gn - others) : mins[k]) : 0;
        }
        build_view(&c, &s, gn, &av);
        eval_rtgpu(&c, &av, rep);
        write_report(&s, &av, rep, method, gn, ok, blob_detail, vsm, e2e_num, den, &range_err);
        if (range_err) *status = RTGPU_RANGE;
        return 0;
    }
    if ((flags & ORACLE_PREFIX) && method == RTGPU_METHOD_RTGPU) {
        int64_t need = 0;
        for (int q = 0; q < nid; q++) need += mins[ids[q]];
        if (need > s.gn) goto unsched_empty;
        int ok = prefix_rtgpu(&c, &s, mins, ids, nid, gn, &av, rep);
        *status = ok ? RTGPU_SCHEDULABLE : RTGPU_UNSCHEDULABLE;
        *evals = c.evals;
        if (!ok) {
            /* the reference reports the lexicographically last allocation */
            int first = -1;
            int64_t others = 0;
            for (int q = 0; q < nid; q++) {
                if (first < 0) first = ids[q];
                else others += mins[ids[q]];
            }
            for (int k = 0; k < s.n; k++)
                gn[k] = s.t[k].g > 0 ? (k == first ? (int)(s.gn - others) : mins[k]) : 0;
            build_view(&c, &s, gn, &av);
            eval_rtgpu(&c, &av, rep);
        }
        write_report(&s, &av, rep, method, gn, ok, blob_detail, vsm, e2e_num, den, &range_err);
        if (range_err) *status = RTGPU_RANGE;
        return 0;
    }
    {
        /* gpu.py:43 _compositions in lexicographic order */
        int x[MAXT];
        int64_t need = 0;
        for (int q = 0; q < nid; q++) need += mins[ids[q]];
        if (need > s.gn) goto unsched_empty;
        for (int q = 0; q < nid; q++) x[q] = mins[ids[q]];
        int have_last = 0;
        for (;;) {
            for (int k = 0; k < s.n; k++) gn[k] = 0;
            for (int q = 0; q < nid; q++) gn[ids[q]] = x[q];
            build_view(&c, &s, gn, &av);
            int ok = method == RTGPU_METHOD_RTGPU ? eval_rtgpu(&c, &av, rep)
                                                  : eval_baseline(&c, &av, method, rep);
            if (ok) {
                *status = RTGPU_SCHEDULABLE;
                *evals = c.evals;
                write_report(&s, &av, rep, method, gn, 1, blob_detail, vsm, e2e_num, den,
                             &range_err);
                if (range_err) *status = RTGPU_RANGE;
                return 0;
            }
            memcpy(last, rep, sizeof(trep) * s.n);
            last_av = av;
            have_last = 1;
            /* next composition */
            int q;
            for (q = nid - 1; q >= 0; q--) {
                int64_t used = 0, after = 0;
                for (int a = 0; a < q; a++) used += x[a];
                for (int a = q + 1; a < nid; a++) after += mins[ids[a]];
                if (x[q] + 1 <= s.gn - used - after) {
                    x[q]++;
                    for (int a = q + 1; a < nid; a++) x[a] = mins[ids[a]];
                    break;
                }
            }
            if (q < 0) break;
        }
        *status = RTGPU_UNSCHEDULABLE;
        *evals = c.evals;
        if (have_last) {
            int zero[MAXT] = {0};
            write_report(&s, &last_av, last, method, zero, 0, blob_detail, vsm, e2e_num, den,
                         &range_err);
            if (range_err) *status = RTGPU_RANGE;
        }
        return 0;
    }
unsched_empty:
    *status = RTGPU_UNSCHEDULABLE;
    *evals = c.evals;
    write_report(&s, NULL, NULL, method, gn, 0, blob_detail, vsm, e2e_num, den, &range_err);
    return 0;
}

/* ------------------------------------------------------ batch driver */

#include <pthread.h>

typedef struct {
    const int64_t *blobs, *set_off, *task_base;
    int64_t n_sets;
    int method;
    unsigned flags;
    int64_t budget;
    int32_t *status;
    int64_t *evals;
    int32_t *vsm;
    int64_t *e2e_num, *den, *detail;
    int64_t next;
    pthread_mutex_t mu;
} batch_job;

static void *batch_worker(void *arg) {
    batch_job *b = (batch_job *)arg;
    for (;;) {
        pthread_mutex_lock(&b->mu);
        int64_t s0 = b->next;
        b->next += 8;
        pthread_mutex_unlock(&b->mu);
        if (s0 >= b->n_sets) break;
        int64_t s1 = s0 + 8 < b->n_sets ? s0 + 8 : b->n_sets;
        for (int64_t s = s0; s < s1; s++) {
            int64_t tb = b->task_base[s];
            oracle_analyze_set(b->blobs + b->set_off[s], b->method, b->flags, b->budget,
                               b->status + s, b->evals + s, b->vsm + tb, b->e2e_num + tb,
                               b->den + tb, b->detail ? b->detail + b->set_off[s] : NULL);
        }
    }
    return NULL;
}

int oracle_analyze_batch(const int64_t *blobs, const int64_t *set_off, const int64_t *task_base,
                         int64_t n_sets, int method, unsigned flags, int64_t budget,
                         int n_threads, int32_t *status, int64_t *evals, int32_t *vsm,
                         int64_t *e2e_num, int64_t *den, int64_t *detail) {
    batch_job b = {blobs, set_off, task_base, n_sets, method, flags, budget, status, evals,
                   vsm, e2e_num, den, detail, 0, PTHREAD_MUTEX_INITIALIZER};
    if (n_threads < 1) n_threads = 1;
    if (n_threads > 256) n_threads = 256;
    pthread_t th[256];
    for (int i = 0; i < n_threads; i++) pthread_create(&th[i], NULL, batch_worker, &b);
    for (int i = 0; i < n_threads; i++) pthread_join(th[i], NULL);
    return 0;
}
