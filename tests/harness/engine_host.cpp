/*
 * TEST HARNESS ONLY -- never loaded by the package.
 *
 * Runs engine_core.cuh (the exact code the sm_100a kernels run) with the
 * sequential SeqTeam emulation of a warp, so the CPU-only test suite can
 * check the engine's algorithm (greedy search, closed-form walks,
 * accelerated fixed points, range escalation) against the oracle without a
 * GPU.  The product path is the CUDA build in paper_2101_10463_b200/csrc.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <vector>

#include "../../paper_2101_10463_b200/csrc/engine_core.cuh"
#include "../../paper_2101_10463_b200/csrc/lattice.cuh"

#ifdef RT_COUNTERS
namespace rtgpu {
long long g_cnt_interf[2], g_cnt_lfp[2], g_cnt_eval, g_cnt_views, g_cnt_rounds;
long long g_cnt_flfp[8], g_cnt_fit[8], g_cnt_frounds, g_cnt_passes;
}
extern "C" void host_counters(long long *out, int reset) {
    using namespace rtgpu;
    long long v[] = {g_cnt_interf[0], g_cnt_interf[1], g_cnt_lfp[0], g_cnt_lfp[1], g_cnt_eval, g_cnt_rounds,
                     g_cnt_flfp[0], g_cnt_flfp[1], g_cnt_fit[0], g_cnt_fit[1], g_cnt_frounds, g_cnt_passes,
                     g_cnt_flfp[4], g_cnt_flfp[5], g_cnt_flfp[6], g_cnt_flfp[7],
                     g_cnt_fit[4], g_cnt_fit[5], g_cnt_fit[6], g_cnt_fit[7], g_cnt_flfp[2], g_cnt_flfp[3]};
    for (int i = 0; i < 22; i++) out[i] = v[i];
    if (reset) {
        g_cnt_interf[0] = g_cnt_interf[1] = g_cnt_lfp[0] = g_cnt_lfp[1] = g_cnt_eval = g_cnt_rounds = 0;
        for (int i = 0; i < 8; i++) g_cnt_flfp[i] = g_cnt_fit[i] = 0;
        g_cnt_frounds = g_cnt_passes = 0;
    }
}
#endif

using namespace rtgpu;

namespace {

template <class V>
int run_one(const Dims &d, const i64 *blob, int method, unsigned flags, i64 budget, OutPtrs<V> o, i64 *evals) {
    Layout<V> L;
    L.init(d);
    std::vector<unsigned char> slab((size_t)L.bytes + 64);
    unsigned char *base = (unsigned char *)(((uintptr_t)slab.data() + 15) & ~(uintptr_t)15);
    SetCtx<V> c;
    c.blob = blob;
    c.hbase = base;
    c.o_tr = 0;
    c.o_vc = L.off_views_c;
    c.o_vm = L.off_views_m;
    c.o_scr = L.off_scr;
    c.L = L;
    c.maxn = d.maxn;
    c.MC = d.MC;
    c.MP = d.MP;
    set_groups(c);
    c.budget = budget > 0 ? budget : 0;
    c.method = method;
    SeqTeam tm;
    int st = analyze_set(tm, c, flags, o);
    *evals = c.evals;
    return st;
}

}  // namespace

extern "C" int host_analyze_batch(const int64_t *blobs, const int64_t *set_off,
                                  const int64_t *task_base, int64_t n_sets, int method, unsigned flags,
                                  int64_t budget, int first_stage, int32_t *status,
                                  int64_t *evals, int32_t *vsm, int64_t *e2e, int64_t *den,
                                  int64_t *detail, int32_t *stage_used) {
    Dims d;
    d.maxn = 1;
    d.MC = 1;
    d.MP = 0;
    for (int64_t s = 0; s < n_sets; s++) {
        const int64_t *h = blobs + set_off[s];
        if (h[0] > d.maxn) d.maxn = (int)h[0];
        if (h[5] > d.MC) d.MC = (int)h[5];
        if (h[6] > d.MP) d.MP = (int)h[6];
    }
    for (int64_t s = 0; s < n_sets; s++) {
        const i64 *blob = (const i64 *)blobs + set_off[s];
        int64_t tb = task_base[s];
        int st = ST_ESCALATE;
        int stage = first_stage;
        if (flags == 0 && method == RTGPU_METHOD_RTGPU && first_stage == 0) {
            /* the kernels' front stage: verdict fast path */
            Layout<double> L;
            L.init(d);
            std::vector<unsigned char> slab((size_t)L.bytes + 64);
            unsigned char *base = (unsigned char *)(((uintptr_t)slab.data() + 15) & ~(uintptr_t)15);
            SetCtx<double> c;
            c.blob = blob;
            c.hbase = base;
            c.o_tr = 0;
            c.o_vc = L.off_views_c;
            c.o_vm = L.off_views_m;
            c.o_scr = L.off_scr;
            c.L = L;
            c.maxn = d.maxn;
            c.MC = d.MC;
            c.MP = d.MP;
            set_groups(c);
            c.budget = budget > 0 ? budget : 0;
            c.method = method;
            SeqTeam tm;
            st = fast_verdict(tm, c, vsm + tb);
            if (st == ST_ESCALATE_RANGE) st = ST_ESCALATE;
            evals[s] = c.evals;
            if (st != ST_ESCALATE) {
                status[s] = st;
                if (stage_used) stage_used[s] = -1;
                continue;
            }
        }
        for (; stage < 3 && st == ST_ESCALATE; stage++) {
            i64 ev = 0;
            if (stage == 0) {
                OutPtrs<double> o{vsm + tb, (i64 *)e2e + tb, (i64 *)den + tb,
                                  detail ? (i64 *)detail + set_off[s] : nullptr};
                st = run_one<double>(d, blob, method, flags, budget, o, &ev);
            } else if (stage == 1) {
                OutPtrs<i64> o{vsm + tb, (i64 *)e2e + tb, (i64 *)den + tb,
                               detail ? (i64 *)detail + set_off[s] : nullptr};
                st = run_one<i64>(d, blob, method, flags, budget, o, &ev);
            } else {
                OutPtrs<i128> o{vsm + tb, (i64 *)e2e + tb, (i64 *)den + tb,
                                detail ? (i64 *)detail + set_off[s] : nullptr};
                st = run_one<i128>(d, blob, method, flags, budget, o, &ev);
            }
            evals[s] = ev;
        }
        if (st == ST_ESCALATE) st = RTGPU_RANGE;
        status[s] = st;
        if (stage_used) stage_used[s] = stage - 1;
    }
    return 0;
}

extern "C" int host_query(const int64_t *blobs, const int64_t *set_off, int64_t n_sets,
                          const rtgpu_query *qs, int64_t nq, int32_t *status, int64_t *num,
                          int64_t *den) {
    Dims d;
    d.maxn = 1;
    d.MC = 1;
    d.MP = 0;
    for (int64_t s = 0; s < n_sets; s++) {
        const int64_t *h = blobs + set_off[s];
        if (h[0] > d.maxn) d.maxn = (int)h[0];
        if (h[5] > d.MC) d.MC = (int)h[5];
        if (h[6] > d.MP) d.MP = (int)h[6];
    }
    for (int64_t qi = 0; qi < nq; qi++) {
        const rtgpu_query &q = qs[qi];
        int st = ST_ESCALATE;
        for (int stage = 0; stage < 3 && st == ST_ESCALATE; stage++) {
            auto go = [&](auto tag) {
                typedef decltype(tag) V;
                Layout<V> L;
                L.init(d);
                std::vector<unsigned char> slab((size_t)L.bytes + 64);
                unsigned char *base = (unsigned char *)(((uintptr_t)slab.data() + 15) & ~(uintptr_t)15);
                SetCtx<V> c;
                c.blob = (const i64 *)blobs + set_off[q.set];
                c.hbase = base;
                c.o_tr = 0;
                c.o_vc = L.off_views_c;
                c.o_vm = L.off_views_m;
                c.o_scr = L.off_scr;
                c.L = L;
                c.maxn = d.maxn;
                c.MC = d.MC;
                c.MP = d.MP;
                set_groups(c);
                c.budget = 0;
                c.method = 0;
                SeqTeam tm;
                i64 n = RTGPU_NONE, dd = 1;
                int r = run_query(tm, c, q.kind, q.task, q.index, q.horizon, q.blocking, &n, &dd);
                num[qi] = n;
                den[qi] = dd;
                return r;
            };
            if (stage == 0) st = go(0.0);
            else if (stage == 1) st = go((i64)0);
            else st = go((i128)0);
        }
        if (st == ST_ESCALATE) st = RTGPU_RANGE;
        status[qi] = st;
    }
    return 0;
}

/* The lattice path (lattice.cuh) alone: status ST_ESCALATE (99) where it
 * hands the set on. */
extern "C" int host_lattice_batch(const int64_t *blobs, const int64_t *set_off, const int64_t *task_base,
                                  int64_t n_sets, int bounds, int32_t *status, int64_t *evals, int32_t *vsm,
                                  int64_t *e2e, int64_t *den) {
    Dims d;
    d.maxn = 1;
    d.MC = 1;
    d.MP = 0;
    for (int64_t s = 0; s < n_sets; s++) {
        const int64_t *h = blobs + set_off[s];
        if (h[0] > d.maxn) d.maxn = (int)h[0];
        if (h[5] > d.MC) d.MC = (int)h[5];
        if (h[6] > d.MP) d.MP = (int)h[6];
    }
    LCtx c;
    c.Lh.init(d);
    std::vector<unsigned char> slab((size_t)c.Lh.bytes + 64);
    c.hbase = (unsigned char *)(((uintptr_t)slab.data() + 15) & ~(uintptr_t)15);
    c.base = 0;
    LSt st;
    c.sth = &st;
    for (int64_t s = 0; s < n_sets; s++) {
        c.blob = (const i64 *)blobs + set_off[s];
        LSeq tm;
        const int64_t tb = task_base[s];
        i64 ev = 0;
        status[s] = lattice_set(tm, c, bounds != 0, vsm + tb, bounds ? (i64 *)e2e + tb : nullptr,
                                bounds ? (i64 *)den + tb : nullptr, ev);
        evals[s] = ev;
    }
    return 0;
}
