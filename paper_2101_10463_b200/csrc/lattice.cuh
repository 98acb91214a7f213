/*
 * lattice.cuh -- the RTGPU verdict / end-to-end-bounds path for task sets on
 * any number of SMs, in exact integer-valued FP64 without a common scale.
 *
 * Why a second path.  fast_verdict (engine_core.cuh) scales every value of a
 * set by one factor 2*A*lcm(1..gtop) so that all GR terms (gpu.py:25, the
 * only division in the analysis) become integers.  On 148 SMs lcm(1..gtop)
 * leaves every exact range, and the general path's per-task scale
 * lcm(2*lcm(g_1..g_{k-1}), 2*A*g_k) does too after a few tasks (int64 and
 * int128 stages, rebuilt views on every count change).  This path needs no
 * lcm at all.  Two facts:
 *
 *  1. The least fixed point of r = b + I(r) (suspension.py:123) lies on the
 *     lattice b + Z (in input ticks).  I(r) = sum_i max_h W_i^h(r) is
 *     continuous, non-decreasing, piecewise linear with integer slopes: a
 *     walk (suspension.py:77) that ends inside a segment grows with slope 1.
 *     At the least fixed point r* every left slope is 0 (slope >= 1 just
 *     left of r* would make r* - eps a pre-fixed point), so every walk ends
 *     in a gap or on a segment boundary and W_i(r*) is a sum of whole
 *     segments' upper bounds -- integers.  Hence r* = b + N*, N* integer.
 *  2. Within one hp task i every position of its chains is a multiple of
 *     1/(2 g_i) (GR lo = GW lo / (2 g_i), gpu.py:38; segments and CPU/copy
 *     gaps are integers).  A walk compares the window H with such positions
 *     and divides by the cycle length, so it depends on H only through
 *     floor(2 g_i H) and whether 2 g_i H is an integer.
 *
 * So views are built once per task at its own scale s_i = 2 g_i (1 for a
 * CPU-only task) and never rescaled; a fixed point iterates over the integer
 * offset N with H = b + N, and each lane forms its task's window as the
 * integer floor(s_i H) plus 0.5 when s_i H is not an integer (the walk's
 * comparisons and floor divisions against integers then behave exactly as
 * with the true fraction, and a tail ending in the fraction comes back
 * marked by the .5).  Convergence is decided exactly: every task's maximum
 * is a whole multiple of s_i (an integer in ticks) and their sum equals N.
 * The next offset is a lower bound of N*:
 *     max(N + 1, ceil(I(r) + sum_i rho_i - eps)),
 * rho_i the remaining slope-1 length of task i's maximising walk: for
 * d >= 0, I_i(r + d) >= I_i(r) + min(d, rho_i), so no fixed point lies
 * below f(r) + sum_i rho_i (engine_core.cuh's lfp jumps by the largest
 * rho_i only).  I(r) is summed as exact integer quotients plus FP64
 * fractions: a rounding error can only cost an extra iteration, never a
 * wrong fixed point.  Bases have denominator d = 2 A g_k (R2 with GR up of
 * task k, analysis.py:214) or 1 (memory and CPU segment responses); results
 * are exact rationals over d.
 *
 * Same search as fast_verdict (greedy descent over counts, verdict shortcut,
 * warm starts) and, for RTGPU_F_BOUNDS, a report pass
 * exactly as analysis.py:280-298.  Anything else (irregular sets, inverted
 * kernels, int64 blobs, ranges beyond 2^51) returns ST_ESCALATE for the
 * general stages.
 *
 * Layout and teams (B200): a team of W warps (1, 2 or 4, chosen per batch
 * from the slab size so ~32 warps stay resident per SM) analyses one set
 * out of one shared-memory slab: struct-of-arrays task records and, per
 * task and resource, a chain view P[0..PM] | EP[0..PM] | F1 | 1/C at the
 * task's scale (segment j's length is EP[j+1] - EP[j]).  Lanes take
 * (task, start segment) pairs: 2^lg lanes per hp task, lg chosen per fixed
 * point so the rounds cover the hp tasks once per warp, each lane walking
 * every 2^lg-th start segment; the team's warps split the rounds and
 * combine their sums through the slab (one named barrier per team).  Only
 * the fixed point is an out-of-line call, with a small by-value argument,
 * so no set context lives on the stack.
 */
#pragma once
#include "engine_core.cuh"

namespace rtgpu {

/* a fixed point's base: bi + bf / d with 0 <= bf < d */
struct LBase {
    i64 bi, bf, d;
};

RT_HD bool lb_le(const LBase &a, const LBase &b) {
    if (a.bi != b.bi) return a.bi < b.bi;
    return (i128)a.bf * b.d <= (i128)b.bf * a.d;
}

/* b + N > D (N integer-valued) */
RT_HD bool lb_over(const LBase &b, double N, i64 D) {
    const double v = (double)b.bi + N;
    return b.bf > 0 ? v >= (double)D : v > (double)D;
}

/* ------------------------------------------------------------ slab */

/* Byte offsets inside one team's slab (16-byte aligned regions). */
struct LSlab {
    int maxn, MC, MP, SC, SM;
    int o_D, o_sClu, o_sInfl, o_sGL, o_B; /* i64 [maxn] */
    int o_T, o_sMlu, o_Mx;                 /* i64 [maxn]: period, sum of copy bounds, longest copy */
    int o_invT;                            /* double [maxn]: 1 / period */
    int o_prio;                            /* i64 [maxn]: priority (record word 4) */
    int o_s, o_invs;                       /* double [maxn]: scale s_i, 1 / s_i */
    int o_seg, o_gmin, o_g, o_info, o_hpn; /* int32 [maxn] */
    int o_vc, o_vm;                        /* double [maxn][SC], [maxn][SM] */
    int o_bases, o_ord, o_red;             /* i64 [32], int [32], double [20]: [4 w + 0..3] partials of warp w, [16] set index */
    int bytes;
    RT_HD void init(const Dims &d) {
        maxn = d.maxn;
        MC = d.MC;
        MP = d.MP;
        SC = 2 * MC + 4;
        SM = MP > 0 ? 2 * MP + 4 : 0;
        int o = 0;
        auto take = [&](int n) {
            const int r = o;
            o += (n + 15) & ~15;
            return r;
        };
        o_D = take(8 * maxn);
        o_sClu = take(8 * maxn);
        o_sInfl = take(8 * maxn);
        o_sGL = take(8 * maxn);
        o_B = take(8 * maxn);
        o_T = take(8 * maxn);
        o_sMlu = take(8 * maxn);
        o_Mx = take(8 * maxn);
        o_invT = take(8 * maxn);
        o_prio = take(8 * maxn);
        o_s = take(8 * maxn);
        o_invs = take(8 * maxn);
        o_seg = take(4 * maxn);
        o_gmin = take(4 * maxn);
        o_g = take(4 * maxn);
        o_info = take(4 * maxn);
        o_hpn = take(4 * maxn);
        o_vc = take(8 * SC * maxn);
        o_vm = take(8 * SM * maxn);
        o_bases = take(8 * 32);
        o_ord = take(4 * 32);
        o_red = take(8 * 20);
        bytes = o;
    }
};

/* info word: m | p << 8 | isgpu << 16 | flags << 20 */
RT_HD int li_m(int w) { return w & 0xff; }
RT_HD int li_p(int w) { return (w >> 8) & 0xff; }
RT_HD int li_gpu(int w) { return (w >> 16) & 1; }
RT_HD int li_flags(int w) { return w >> 20; }

/* Typed access to a team's slab: on the device addressed from the dynamic
 * shared-memory symbol (LDS/STS), in the host harness from a heap buffer. */
/* On the device one copy of the slab geometry per CTA sits at the start of
 * dynamic shared memory (LSLAB_HDR bytes, before the teams' slabs): read
 * from there at every use, the offsets never occupy registers across the
 * out-of-line fixed points (they were a third of the kernel's stack frame). */
#define LSLAB_HDR 128
static_assert(sizeof(LSlab) <= LSLAB_HDR, "slab header");
#ifdef __CUDACC__
__device__ __forceinline__ const LSlab &lslab_dev() { return *(const LSlab *)rt_dyn_smem; }
#endif

/* The warp-uniform state of one set's allocation search (lattice_set): one
 * per warp in shared memory on the device, after the slab header. */
struct LSt {
    LBase mw, cw, lbm;
    double mwN, cwN, mg;
    i64 used, rest_min, evals, mr_ub, sum_mr, bsum, sum_cr;
    int k, st, glo, ghi, g, lo, hi, phase, cand, fail, rmax_exact, pass;
};
#define LST_BYTES ((int)((sizeof(LSt) + 15) & ~(size_t)15))

struct LCtx {
    unsigned char *hbase; /* host harness only */
    int base;             /* byte offset of the slab */
    int sto;              /* byte offset of the warp's LSt (device) */
    LSt *sth;             /* the LSt (host harness) */
    LSlab Lh;             /* host harness only */
    const i64 *blob;
    int n, GN, mm;
    i64 A;
    RT_HD const LSlab &L() const {
#ifdef __CUDA_ARCH__
        return lslab_dev();
#else
        return Lh;
#endif
    }
    RT_HD unsigned char *sb() const {
#ifdef __CUDA_ARCH__
        return rt_dyn_smem + base;
#else
        return hbase + base;
#endif
    }
    RT_HD LSt *stp() const {
#ifdef __CUDA_ARCH__
        return (LSt *)(rt_dyn_smem + sto);
#else
        return sth;
#endif
    }
    RT_HD i64 *D() const { return (i64 *)(sb() + L().o_D); }
    RT_HD i64 *sClu() const { return (i64 *)(sb() + L().o_sClu); }
    RT_HD i64 *sInfl() const { return (i64 *)(sb() + L().o_sInfl); }
    RT_HD i64 *sGL() const { return (i64 *)(sb() + L().o_sGL); }
    RT_HD i64 *B() const { return (i64 *)(sb() + L().o_B); }
    RT_HD i64 *T() const { return (i64 *)(sb() + L().o_T); }
    RT_HD i64 *sMlu() const { return (i64 *)(sb() + L().o_sMlu); }
    RT_HD i64 *Mx() const { return (i64 *)(sb() + L().o_Mx); }
    RT_HD double *invT() const { return (double *)(sb() + L().o_invT); }
    RT_HD i64 *prio() const { return (i64 *)(sb() + L().o_prio); }
    RT_HD double *S() const { return (double *)(sb() + L().o_s); }
    RT_HD double *IS() const { return (double *)(sb() + L().o_invs); }
    RT_HD int *seg() const { return (int *)(sb() + L().o_seg); }
    RT_HD int *gmin() const { return (int *)(sb() + L().o_gmin); }
    RT_HD int *g() const { return (int *)(sb() + L().o_g); }
    RT_HD int *info() const { return (int *)(sb() + L().o_info); }
    RT_HD int *hpn() const { return (int *)(sb() + L().o_hpn); }
    RT_HD double *VC() const { return (double *)(sb() + L().o_vc); }
    RT_HD double *VM() const { return (double *)(sb() + L().o_vm); }
    RT_HD i64 *bases() const { return (i64 *)(sb() + L().o_bases); }
    RT_HD int *ord() const { return (int *)(sb() + L().o_ord); }
    RT_HD Seg32 segs(int i) const { return Seg32{(const int32_t *)blob + seg()[i]}; }
};

/* What a lane remembers of its walks between the iterations of one fixed
 * point (same task, same start segments; the window only grows): the best
 * walk ending inside a segment (m1, its remaining length r1), the best one
 * ending in a gap (m0), and how far the window may grow with every walk
 * exactly predictable (v: the least remaining length / gap).  Scale units. */
struct LCache {
    double m1, r1, m0, v, H;
};

/* ------------------------------------------------------------ teams */

#ifdef __CUDACC__
/* W warps on one set; bar = the team's named barrier (W > 1). */
template <int W> struct LTeam {
    int lane, warp, bar;
    __device__ __forceinline__ void sync() const {
        if (W == 1) __syncwarp();
        else asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(W * 32) : "memory");
    }
    __device__ __forceinline__ bool leader() const { return lane == 0 && warp == 0; }
    __device__ __forceinline__ int width() const { return W; }
    typedef LCache Cache; /* the lane's own */
    __device__ __forceinline__ void cache_reset(Cache &c) const { c.H = -1; }
    __device__ __forceinline__ Cache &cache_ptr(Cache &c) const { return c; }
    template <class F> __device__ __forceinline__ void pfor(int n, F f) const {
        #pragma unroll 1
        for (int i = warp * 32 + lane; i < n; i += 32 * W) f(i);
        sync();
    }
};
#endif

/* sequential emulation of a one-warp team (test harness) */
struct LSeq {
    RT_HD void sync() const {}
    RT_HD bool leader() const { return true; }
    RT_HD int width() const { return 1; }
    struct Cache {
        LCache c[32]; /* one per emulated lane */
    };
    RT_HD void cache_reset(Cache &c) const {
        for (int i = 0; i < 32; i++) c.c[i].H = -1;
    }
    RT_HD LCache *cache_ptr(Cache &c) const { return c.c; }
    template <class F> RT_HD void pfor(int n, F f) const {
        for (int i = 0; i < n; i++) f(i);
    }
};

/* ------------------------------------------------------------ chain walk */

/* W_i^h(H) of suspension.py:77 over a regular chain view at the task's
 * scale: P[0..p] (P[p] = cycle length C), EP[0..p], F1, 1/C; rho = the
 * remaining slope-1 length when the window ends inside a segment, else
 * gap = the distance from the window's end to the next segment start (the
 * window can grow by that much with W unchanged).  First (partial) job, or
 * a floor-division jump over whole cycles and the last one; then the last
 * segment start <= the window end by a galloping binary search (half =
 * power of two >= PM / 2). */
RT_HD double walk_lat(const double *v, int PM, int half, int p, int h, double H, double &rho, double &gap) {
    rho = 0;
    gap = 0;
    if (H <= 0) return 0;
    const double *P = v, *EP = v + PM + 1;
    const double lim = H + P[h];
    const double F1 = v[2 * PM + 2], C = P[p], EPp = EP[p], EPh = EP[h];
    /* both cases computed, one selected (no divergence between lanes) */
    const bool first = F1 > lim;
    double r;
    const double kq = Num<double>::divmod_inv(first ? 0.0 : lim - F1, C, v[2 * PM + 3], r);
    const double Hs = first ? lim : r;
    const double w0 = first ? -EPh : fma(kq, EPp, EPp - EPh);
    const double nxt = first ? F1 : C; /* after the last segment: job 2, or the next cycle */
    int x = first ? h : 0;
    #pragma unroll
    for (int st = 16; st > 0; st >>= 1) { /* half <= 16 (PM <= 32) */
        const int y = x + st;
        if (st <= half && y <= p - 1 && P[y] <= Hs) x = y;
    }
    const double tail = Hs - P[x];
    const double e0 = EP[x], e1 = EP[x + 1];
    const double ex = e1 - e0;
    if (ex > tail) {
        rho = ex - tail;
        return w0 + e0 + tail;
    }
    gap = (x < p - 1 ? P[x + 1] : nxt) - Hs;
    return w0 + e1;
}

/* per-iteration accumulators of the interference rounds */
struct LatAcc {
    double q;    /* sum of floor(W_i) in ticks (exact integers) */
    double f;    /* the fractional parts of the W_i plus every task's slope-1
                  * length of a maximising walk (ticks, FP64): the jump */
    bool nonint; /* some W_i is not an integer number of ticks */
};

/* the per-task bookkeeping: m = the task's maximum at scale s */
RT_HD void lat_group(double m, double s, double invs, double phv, LatAcc &a) {
    const double mi = floor(m);
    double q = floor(mi * invs);
    double r = fma(-q, s, mi);
    if (r < 0) {
        q -= 1.0;
        r += s;
    } else if (r >= s) {
        q += 1.0;
        r -= s;
    }
    const bool mh = m != mi;
    a.q += q;
    a.nonint = a.nonint || r != 0 || mh;
    a.f += (r + (mh ? phv : 0.0)) * invs;
}

/* What a fixed point iterates over (the hp chains of one resource) and
 * where they are: everything lfp_lat reads, by value. */
struct LChains {
    unsigned char *hbase; /* host harness only */
    int base, o_s, o_invs, o_info, o_red, vbase;
    int k;   /* hp tasks are [0, k) */
    int res; /* K_CPU / K_MEM */
    int lg;  /* log2 lanes per task */
    int PM, half, stride;
    RT_HD unsigned char *sb() const {
#ifdef __CUDA_ARCH__
        return rt_dyn_smem + base;
#else
        return hbase + base;
#endif
    }
};

/* lanes per task: the largest power of two with k * G <= 32 * W (one round
 * per warp), at most the power of two covering the chain's segments */
RT_HD int lat_lg(int k, int PM, int W) {
    int G = 1, lg = 0;
    while (G < PM && 2 * G * k <= 32 * W) {
        G <<= 1;
        lg++;
    }
    return lg;
}

/* What an out-of-line fixed point is handed (a few words, no set context):
 * where the slab is, the batch dims, the task and the resource; the chain
 * geometry is rebuilt from them inside. */
struct LKey {
    unsigned char *hbase; /* host harness only */
    int base, maxn, MC, MP, task, res;
};

RT_HD LKey lat_key(const LCtx &c, int k, int res) {
    LKey q;
    q.hbase = c.hbase;
    q.base = c.base;
    q.maxn = c.L().maxn;
    q.MC = c.L().MC;
    q.MP = c.L().MP;
    q.task = k;
    q.res = res;
    return q;
}

RT_HD LChains lat_chains(const LCtx &c, int k, int res, int W) {
    LChains ch;
    ch.hbase = c.hbase;
    ch.base = c.base;
    ch.o_s = c.L().o_s;
    ch.o_invs = c.L().o_invs;
    ch.o_info = c.L().o_info;
    ch.o_red = c.L().o_red;
    ch.k = c.hpn()[k];
    ch.res = res;
    ch.PM = res == K_CPU ? c.L().MC : c.L().MP;
    ch.stride = res == K_CPU ? c.L().SC : c.L().SM;
    ch.vbase = res == K_CPU ? c.L().o_vc : c.L().o_vm;
    ch.lg = lat_lg(ch.k, ch.PM, W);
    int hf = 1;
    while (2 * hf < ch.PM) hf <<= 1;
    ch.half = ch.PM > 1 ? hf : 0;
    return ch;
}

/* One slot's contribution for task i = i0 + slot / G: the maximum over its
 * start segments h = slot % G, + G, ... and the slope-1 length (ticks) of a
 * maximising walk (largest among ties); s / invs / phv are the task's. */
RT_HD void lat_slot(const LChains &ch, double bN, i64 bf, i64 d, double invd, int i0, int slot, double &bw,
                    double &br, double &s, double &invs, double &phv, LCache *cc) {
    const int G = 1 << ch.lg;
    const int i = i0 + (slot >> ch.lg), h0 = slot & (G - 1);
    bw = 0;
    br = 0;
    s = 1;
    invs = 1;
    phv = 0;
    if (i >= ch.k) return;
    unsigned char *sb = ch.sb();
    s = ((const double *)(sb + ch.o_s))[i];
    invs = ((const double *)(sb + ch.o_invs))[i];
    double Hi = bN * s, hf = 0;
    if (bf) {
        /* floor(bf * s / d) and whether it is exact (bf * s < 2^53) */
        const double x = (double)bf * s, dd = (double)d;
        double u = floor(x * invd);
        double rem = fma(-u, dd, x);
        if (rem < 0) {
            u -= 1.0;
            rem += dd;
        } else if (rem >= dd) {
            u += 1.0;
            rem -= dd;
        }
        Hi += u;
        if (rem > 0) {
            hf = 0.5;
            phv = rem * invd;
        }
    }
    const int info = ((const int *)(sb + ch.o_info))[i];
    const int p = ch.res == K_CPU ? li_m(info) : li_p(info);
    const double *v = (const double *)(sb + ch.vbase) + (size_t)i * ch.stride;
    const double H = Hi + hf;
    const double NONE = -1e300;
    if (cc && cc->H >= 0 && H - cc->H <= cc->v) {
        /* every walk predictable: the ones inside a segment grew by the
         * window's growth, the ones in a gap did not move (a walk that just
         * reached a boundary keeps its exact value; its slope-1 length is
         * under-reported as 0, which only shortens the jump) */
        const double dl = H - cc->H;
        cc->m1 += dl;
        cc->r1 -= dl;
        cc->v -= dl;
        cc->H = H;
        if (cc->m1 >= cc->m0) {
            bw = cc->m1;
            br = cc->r1;
        } else {
            bw = cc->m0;
        }
    } else {
        double m1 = NONE, r1 = 0, m0 = 0, vmin = 1e300;
        auto take = [&](double w, double r, double gp) {
            if (r > 0) {
                if (w > m1 || (w == m1 && r > r1)) {
                    m1 = w;
                    r1 = r;
                }
                vmin = tmin(vmin, r);
            } else {
                m0 = tmax(m0, w);
                vmin = tmin(vmin, gp);
            }
        };
        #pragma unroll 1
        for (int h = h0; h < p; h += G) {
            RT_COUNT(g_cnt_frounds);
            double r, gp;
            const double w = walk_lat(v, ch.PM, ch.half, p, h, H, r, gp);
            take(w, r, gp);
        }
        if (m1 >= m0) {
            bw = m1;
            br = r1;
        } else {
            bw = m0;
        }
        if (cc) {
            cc->m1 = m1;
            cc->r1 = r1;
            cc->m0 = m0;
            cc->v = vmin;
            cc->H = H;
        }
    }
    br = br > 0 ? (br + hf - phv) * invs : 0.0;
}

/* The interference sums at H = bN + bf / d over the hp tasks. */
#ifdef __CUDACC__
template <int W>
__device__ __forceinline__ LatAcc lat_interf(const LTeam<W> &tm, const LChains &ch, double bN, i64 bf, i64 d,
                                             double invd, LCache &cache, bool jump = true) {
    LatAcc a = {0.0, 0.0, false};
    const int per = 32 >> ch.lg, G = 1 << ch.lg;
    const int R = (ch.k + per - 1) / per;
#ifdef RTGPU_LAT_NOCACHE
    LCache *cc = nullptr;
    (void)cache;
#else
    LCache *cc = R <= W ? &cache : nullptr; /* one round per warp: the lane's walks are the same every iteration */
#endif
    #pragma unroll 1
    for (int r = tm.warp; r < R; r += W) {
        double bw, br, s, invs, phv;
        lat_slot(ch, bN, bf, d, invd, r * per, tm.lane, bw, br, s, invs, phv, cc);
        for (int off = 1; off < G; off <<= 1) {
            const double ow = shfl_x(bw, off), orr = shfl_x(br, off);
            if (ow > bw || (ow == bw && orr > br)) {
                bw = ow;
                br = orr;
            }
        }
        lat_group(bw, s, invs, phv, a); /* every lane of the group holds its task's sums */
        if (jump) a.f += br;
    }
    /* butterfly sums over the groups: identical on every lane (IEEE
     * addition commutes), so the team takes one decision */
    for (int off = G; off < 32; off <<= 1) {
        a.q += shfl_x(a.q, off);
        a.f += shfl_x(a.f, off);
    }
    a.nonint = __any_sync(0xffffffffu, a.nonint);
    if (W > 1) {
        double *red = (double *)(ch.sb() + ch.o_red);
        tm.sync(); /* the previous iteration's partials have been read */
        if (tm.lane == 0) {
            red[4 * tm.warp + 0] = a.q;
            red[4 * tm.warp + 1] = a.f;
            red[4 * tm.warp + 3] = a.nonint ? 1.0 : 0.0;
        }
        tm.sync();
        a.q = a.f = 0;
        a.nonint = false;
        #pragma unroll
        for (int w = 0; w < W; w++) { /* the same order in every warp */
            a.q += red[4 * w];
            a.f += red[4 * w + 1];
            a.nonint = a.nonint || red[4 * w + 3] != 0;
        }
    }
    return a;
}
#endif

RT_HD LatAcc lat_interf(const LSeq &, const LChains &ch, double bN, i64 bf, i64 d, double invd, LCache *cache,
                        bool jump = true) {
    LatAcc a = {0.0, 0.0, false};
    const int per = 32 >> ch.lg, G = 1 << ch.lg;
#ifdef RTGPU_LAT_NOCACHE
    const bool one = false;
#else
    const bool one = ch.k <= per; /* one round: the emulated lanes keep their caches */
#endif
    for (int i0 = 0; i0 < ch.k; i0 += per)
        for (int g0 = 0; g0 < 32; g0 += G) {
            double m = 0, rm = 0, s = 1, invs = 1, phv = 0;
            for (int x = 0; x < G; x++) {
                double bw, br;
                lat_slot(ch, bN, bf, d, invd, i0, g0 + x, bw, br, s, invs, phv, one ? cache + g0 + x : nullptr);
                if (x == 0 || bw > m || (bw == m && br > rm)) {
                    m = bw;
                    rm = br;
                }
            }
            lat_group(m, s, invs, phv, a);
            if (jump) a.f += rm;
        }
    return a;
}

/* 1 / d to within 2^-46 relative (d < 2^40): a float estimate and one Newton
 * step -- lat_slot's floor correction absorbs any error below one unit */
RT_HD double lat_rcp(i64 d) {
#ifdef __CUDA_ARCH__
    float y0;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y0) : "f"((float)d));
    const double y = (double)y0;
    return y * fma(-(double)d, y, 2.0);
#else
    return 1.0 / (double)d;
#endif
}

/* Least fixed point of r = b + I(r) as the offset N* = r* - b, iterated from
 * N (a lower bound of N*).  -1 = None (suspension.py:123: beyond D),
 * -2 = iteration cap. */
template <class TM>
RT_HD double lfp_lat_body(const TM &tm, const LKey key, const LBase b, double N, i64 D, int mode) {
    LCtx c;
    c.hbase = key.hbase;
    c.base = key.base;
#ifndef __CUDA_ARCH__
    c.Lh.init(Dims{key.maxn, key.MC, key.MP});
#endif
    const LChains ch = lat_chains(c, key.task, key.res, tm.width());
    RT_COUNT(g_cnt_flfp[4 + ch.res + 2 * (mode ? 1 : 0)]);
    if (lb_over(b, N, D)) return -1.0;
    const double invd = b.bf ? lat_rcp(b.d) : 0.0;
    typename TM::Cache cache;
    tm.cache_reset(cache);
    if (mode == 1) {
        /* Is b + N a pre-fixed point?  f(r) <= r with r = b + N puts the lfp
         * at or below r (and then, f being monotone, at or below f(r)):
         * return floor(I(r)), the offset of f(r) rounded down to the
         * lattice, or -1 when not verified.  I(r) = q + F, F the exact sum
         * of the fractional parts (FP64 a.f within 1e-9 of it). */
        RT_COUNT(g_cnt_fit[6 + ch.res]);
        const LatAcc a = lat_interf(tm, ch, (double)b.bi + N, b.bf, b.d, invd, tm.cache_ptr(cache), false);
        const double ub = floor(a.q + a.f + 1e-6);
        return (a.q + a.f + 1e-6 <= N) ? ub : -1.0;
    }
    if (mode == 2) {
        /* an upper bound of I(b + N) (one evaluation, FP64 error < 1e-6) */
        RT_COUNT(g_cnt_fit[6 + ch.res]);
        const LatAcc a = lat_interf(tm, ch, (double)b.bi + N, b.bf, b.d, invd, tm.cache_ptr(cache), false);
        return a.q + a.f + 1e-6;
    }
    #pragma unroll 1
    for (int it = 0; it < ITER_CAP; it++) {
        RT_COUNT(g_cnt_fit[4 + ch.res]);
        const LatAcc a = lat_interf(tm, ch, (double)b.bi + N, b.bf, b.d, invd, tm.cache_ptr(cache));
        if (!a.nonint && a.q <= N) return N; /* f(r) <= r with r <= lfp: r is the lfp */
        double Nn = a.q + ceil(a.f - 1e-6);
        if (Nn < N + 1.0) Nn = N + 1.0;
        if (lb_over(b, Nn, D)) return -1.0;
        N = Nn;
    }
    return -2.0;
}

/* out of line (the report pass and its chains call it from several sites) */
template <class TM>
RT_NI double lfp_lat(const TM &tm, const LKey key, const LBase b, double N, i64 D, int mode = 0) {
    return lfp_lat_body(tm, key, b, N, D, mode);
}

/* ------------------------------------------------------------ per-set steps */

/* Load task i (one lane): record, sums, flags and the minimum count of
 * analysis.py:239 _min_feasible_gn in closed form.  Returns the range bound
 * D + T + every sum; B[i] receives the task's longest copy.  Tasks the
 * lattice path does not take are flagged TF_UNSUP / TF_IRREG / TF_INV. */
RT_HD i64 lat_load(const LCtx &c, int i) {
    const RecP r = rec_at(c.blob, i);
    const int m = (int)r[0], p = (int)r[1];
    const i64 D = r[2], T = r[3];
    c.prio()[i] = r[4];
    const int want_p = m < 2 ? 0 : (c.mm == RTGPU_TWO_COPY ? 2 * m - 2 : m - 1);
    const bool isgpu = m > 1;
    int flags = 0;
    c.D()[i] = D;
    c.g()[i] = 0;
    c.gmin()[i] = 0;
    c.B()[i] = 0;
    if (m < 1 || m > c.L().MC || p != want_p || p > c.L().MP || T <= 0 || D <= 0 || D > T || T >= ((i64)1 << 56) ||
        c.A >= (1 << 16) || r[5] < 0 || r[5] > (1 << 30)) {
        c.info()[i] = (m & 0xff) | (p & 0xff) << 8 | TF_UNSUP << 20;
        return 0;
    }
    c.seg()[i] = (int)r[5];
    const Seg32 sg{(const int32_t *)c.blob + r[5]};
    const int g = m - 1;
    i64 clu = 0, cll = 0, mlu = 0, mll = 0, gwl = 0, infl = 0, gls = 0, inner = 0, mx = 0, ih = 0, acc = 0;
    #pragma unroll 1
    for (int j = 0; j < m; j++) {
        const i64 lo = sg[j], hi = sg[m + j];
        acc |= lo | hi;
        clu += hi;
        cll += lo;
        if (j >= 1 && j <= m - 2) inner += lo;
    }
    #pragma unroll 1
    for (int j = 0; j < p; j++) {
        const i64 lo = sg[2 * m + j], h = sg[2 * m + p + j];
        acc |= lo | h;
        mll += lo;
        mlu += h;
        mx = tmax(mx, h);
    }
    #pragma unroll 1
    for (int j = 0; j < g; j++) {
        const i64 lo = sg[2 * m + 2 * p + j], hi = sg[2 * m + 2 * p + g + j];
        const i64 gl = sg[2 * m + 2 * p + 2 * g + j], an = sg[2 * m + 2 * p + 3 * g + j];
        acc |= lo | hi | gl | an;
        const i64 w = hi * an, o = gl * c.A; /* < 2^47 */
        if (o > w) flags |= TF_INV;
        infl += w - o;
        ih += w;
        gls += gl;
        gwl += lo;
    }
    if (acc < 0) {
        c.info()[i] = m | p << 8 | TF_UNSUP << 20;
        return 0;
    }
    c.sClu()[i] = clu;
    c.sInfl()[i] = infl;
    c.sGL()[i] = gls;
    c.B()[i] = mx;
    c.T()[i] = T;
    c.invT()[i] = 1.0 / (double)T;
    c.sMlu()[i] = mlu;
    c.Mx()[i] = mx;
    int gm = 0;
    if (isgpu) {
        const i64 X = D - gls - mlu - clu;
        if (c.GN >= 1) {
            if (X > 0) {
                if (X > ((i64)1 << 60) / (2 * c.A)) gm = 1; /* infl / (2 A X) < 1 */
                else {
                    const i64 den = 2 * c.A * X;
                    const i64 q = (infl + den - 1) / den;
                    gm = q < 1 ? 1 : (q > c.GN ? 0 : (int)q);
                }
            } else if (X == 0 && infl == 0) {
                gm = 1;
            }
        }
        if (gm == 0) flags |= TF_ISOFAIL;
        if (gm > 0) {
            /* regular: no wrap-around gap negative at any count >= gm */
            const i64 need = (gwl + 2 * gm - 1) / (2 * gm);
            if (T - clu - mll < need) flags |= TF_IRREG;
            if (T - mlu - inner < need) flags |= TF_IRREG;
        }
    } else {
        if (clu > D) flags |= TF_ISOFAIL;
        if (T - clu < 0) flags |= TF_IRREG;
    }
    c.gmin()[i] = gm;
    c.info()[i] = m | p << 8 | (isgpu ? 1 : 0) << 16 | flags << 20;
    return D + T + clu + cll + mlu + mll + gwl + gls + ih / c.A + 1;
}

/* Chain views of task i at its scale s = 2 g_i (1 without kernels).
 * Regular chains (every wrap-around gap >= 0): C = T s for CPU chains and
 * two-copy memory chains, T s - GW lo of the last kernel for one-copy
 * memory chains; gaps of analysis.py:89 cpu_inter_arrival and :57
 * mem_inter_arrival.  `lane` = -1: sequential build (host harness);
 * otherwise lane j of a warp holds segment j and P / EP are warp scans. */
RT_HD void lat_build_chain(double *v, int PM, int q, int lane, double e_j, double gap_j, double C, double first) {
#ifdef __CUDA_ARCH__
    if (lane >= 0) {
        double s1 = e_j + gap_j, s2 = e_j;
        #pragma unroll 1
        for (int off = 1; off < q; off <<= 1) {
            const double a1 = __shfl_up_sync(0xffffffffu, s1, off), a2 = __shfl_up_sync(0xffffffffu, s2, off);
            if (lane >= off) {
                s1 += a1;
                s2 += a2;
            }
        }
        if (lane < q) {
            v[lane] = s1 - e_j - gap_j;
            v[PM + 1 + lane] = s2 - e_j;
            if (lane == q - 1) {
                v[q] = C;
                v[PM + 1 + q] = s2;
                v[2 * PM + 2] = s1 + first;
                v[2 * PM + 3] = 1.0 / C;
            }
        }
        return;
    }
#endif
    (void)v, (void)PM, (void)q, (void)lane, (void)e_j, (void)gap_j, (void)C, (void)first;
}

RT_HD void lat_view_lane(const LCtx &c, int i, int lane) {
    const RecP r = rec_at(c.blob, i);
    const int info = c.info()[i];
    const int m = li_m(info), p = li_p(info);
    const i64 T = r[3], D = r[2];
    const double ds = li_gpu(info) ? 2.0 * (double)c.g()[i] : 1.0;
    const Seg32 sg = c.segs(i);
    const Seg32 cl_lo = sg, cl_hi = sg + m, ml_lo = sg + 2 * m, ml_hi = ml_lo + p, gw_lo = ml_hi + p;
    const bool two = c.mm == RTGPU_TWO_COPY;
    auto cpu_seg = [&](int j, double &e, double &gap) {
        e = (double)cl_hi[j] * ds;
        gap = j < m - 1 ? (double)(two ? ml_lo[2 * j] + ml_lo[2 * j + 1] : ml_lo[j]) * ds + (double)gw_lo[j] : 0.0;
    };
    auto mem_seg = [&](int j, double &e, double &gap) {
        e = (double)ml_hi[j] * ds;
        gap = 0;
        if (j < p - 1) {
            if (two) gap = (j % 2 == 0) ? (double)gw_lo[j / 2] : (double)cl_lo[(j + 1) / 2] * ds;
            else gap = (double)gw_lo[j] + (double)cl_lo[j + 1] * ds;
        }
    };
    const double Cc = (double)T * ds, Fc = (double)(T - D) * ds;
    double Cm = 0, Fm = 0;
    if (p > 0) {
        Cm = (double)T * ds - (two ? 0.0 : (double)gw_lo[m - 2]);
        Fm = (double)(T - D + cl_lo[m - 1] + cl_lo[0]) * ds + (two ? 0.0 : (double)gw_lo[m - 2]);
    }
    double *vc = c.VC() + (size_t)i * c.L().SC;
    double *vm = c.VM() + (size_t)i * c.L().SM;
    if (lane >= 0) {
        double e = 0, gap = 0;
        if (lane < m) cpu_seg(lane, e, gap);
        lat_build_chain(vc, c.L().MC, m, lane, e, gap, Cc, Fc);
        if (p > 0) {
            e = gap = 0;
            if (lane < p) mem_seg(lane, e, gap);
            lat_build_chain(vm, c.L().MP, p, lane, e, gap, Cm, Fm);
        }
        return;
    }
    /* sequential (host harness) */
    auto seq = [&](double *v, int PM, int q, bool cpu, double C, double first) {
        double P = 0, EP = 0;
        for (int j = 0; j < q; j++) {
            double e, gap;
            if (cpu) cpu_seg(j, e, gap);
            else mem_seg(j, e, gap);
            v[j] = P;
            v[PM + 1 + j] = EP;
            P += e + gap;
            EP += e;
        }
        v[q] = C;
        v[PM + 1 + q] = EP;
        v[2 * PM + 2] = P + first;
        v[2 * PM + 3] = 1.0 / C;
    };
    seq(vc, c.L().MC, m, true, Cc, Fc);
    if (p > 0) seq(vm, c.L().MP, p, false, Cm, Fm);
}

#ifdef __CUDACC__
/* views of task i by warp 0 of the team (the others wait at the barrier) */
template <int W> __device__ __forceinline__ void lat_view(const LTeam<W> &tm, const LCtx &c, int i) {
    if (tm.warp == 0) {
        lat_view_lane(c, i, tm.lane);
        if (tm.lane == 0) {
            const double s = li_gpu(c.info()[i]) ? 2.0 * (double)c.g()[i] : 1.0;
            c.S()[i] = s;
            c.IS()[i] = 1.0 / s;
        }
        __syncwarp();
    }
    tm.sync();
}
#endif
RT_HD void lat_view(const LSeq &, const LCtx &c, int i) {
    lat_view_lane(c, i, -1);
    const double s = li_gpu(c.info()[i]) ? 2.0 * (double)c.g()[i] : 1.0;
    c.S()[i] = s;
    c.IS()[i] = 1.0 / s;
}

/* Sum of the fixed points of the integer bases c.bases()[0..cnt) (one
 * resource), ascending with warm starts lfp(b') - b' >= lfp(b) - b; the
 * first None makes every larger base None.  Returns the sum, -1 (some None)
 * or -2 (iteration cap). */
template <class TM>
RT_HD i64 lat_chain_sum(const TM &tm, const LCtx &c, const LKey &key, int cnt, i64 D) {
    i64 *bases = c.bases();
    int *ord = c.ord();
    tm.pfor(cnt, [&](int j) {
        int rk = 0;
        #pragma unroll 1
        for (int x = 0; x < cnt; x++) rk += (bases[x] < bases[j] || (bases[x] == bases[j] && x < j)) ? 1 : 0;
        ord[rk] = j;
    });
    double N = 0;
    i64 sum = 0;
    #pragma unroll 1
    for (int st = 0; st < cnt; st++) {
        const i64 b = bases[ord[st]];
        const double r = lfp_lat(tm, key, LBase{b, 0, 1}, N, D);
        if (r < 0) {
            sum = r == -2.0 ? -2 : -1;
            break;
        }
        sum += b + (i64)r;
        N = r;
    }
    tm.sync(); /* bases / ord are rewritten by the next chain */
    return sum;
}

/* max and sum of ml[j] + B over the p copies of a task: one load per lane
 * and two butterflies on a team (p <= 30), a loop in the host harness */
#ifdef __CUDACC__
template <int W>
__device__ __forceinline__ void lat_copy_sums(const LTeam<W> &tm, Seg32 ml, int p, i64 B, i64 &mx, i64 &sm) {
    const i64 v = tm.lane < p ? (i64)ml[tm.lane] + B : 0;
    mx = v;
    sm = v;
    #pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        mx = tmax(mx, shfl_x(mx, off));
        sm += shfl_x(sm, off);
    }
}
#endif
RT_HD void lat_copy_sums(const LSeq &, Seg32 ml, int p, i64 B, i64 &mx, i64 &sm) {
    mx = 0;
    sm = 0;
    for (int j = 0; j < p; j++) {
        mx = tmax(mx, (i64)ml[j] + B);
        sm += ml[j] + B;
    }
}

/* A cheap upper bound of the interference sum_{i in hp(k)} max_h W_i^h(H)
 * of one resource (ticks), from the views alone: a window of length H meets
 * at most floor(H / C) + 2 jobs of a regular chain (the first, partial one
 * and those starting every C after it), each contributing at most its
 * segments' total EP[p] -- one division per hp task instead of its walks.
 * Exact integer floor (the divmod correction); FP64 sum of the quotients
 * EP / s within 1e-9, which the callers' 1e-6 margins absorb. */
RT_HD double lat_cycle_term(const LCtx &c, int i, int res, double H) {
    const int info = c.info()[i];
    const int p = res == K_CPU ? li_m(info) : li_p(info);
    if (p <= 0) return 0.0;
    const int PM = res == K_CPU ? c.L().MC : c.L().MP;
    const double *v = (res == K_CPU ? c.VC() + (size_t)i * c.L().SC : c.VM() + (size_t)i * c.L().SM);
    const double s = c.S()[i], C = v[p], EPp = v[PM + 1 + p];
    double r;
    const double q = Num<double>::divmod_inv(H * s, C, v[2 * PM + 3], r);
    return (q + 2.0) * EPp * c.IS()[i];
}
#ifdef __CUDACC__
template <int W>
__device__ __forceinline__ double lat_cycle_bound(const LTeam<W> &tm, const LCtx &c, int k, int res, double H) {
    double u = 0.0;
    const int nh = c.hpn()[k];
    for (int i = tm.lane; i < nh; i += 32) u += lat_cycle_term(c, i, res, H);
    #pragma unroll
    for (int off = 16; off > 0; off >>= 1) u += shfl_x(u, off);
    return u;
}
#endif
RT_HD double lat_cycle_bound(const LSeq &, const LCtx &c, int k, int res, double H) {
    double u = 0.0;
    const int nh = c.hpn()[k];
    for (int i = 0; i < nh; i++) u += lat_cycle_term(c, i, res, H);
    return u;
}

/* GR up of task i at count g (gpu.py:25 summed over its kernels) as
 * bi + bf / d, d = 2 A g */
RT_HD LBase lat_grup(const LCtx &c, int i, int g) {
    LBase r;
    if (!li_gpu(c.info()[i])) {
        r.bi = 0;
        r.bf = 0;
        r.d = 1;
        return r;
    }
    r.d = 2 * c.A * (i64)g;
    const i64 infl = c.sInfl()[i];
    i64 q, rem;
#ifdef RTGPU_LAT_FPQ /* off: more spills than the division costs (r2u: -2.5%) */
    if (infl >= 0 && infl < ((i64)1 << 53)) {
#else
    if (false) {
#endif
        /* FP64 quotient (both operands exact) and one correction step: no
         * 64-bit integer division on the search's path */
        q = (i64)floor((double)infl / (double)r.d);
        rem = infl - q * r.d;
        if (rem < 0) {
            q--;
            rem += r.d;
        } else if (rem >= r.d) {
            q++;
            rem -= r.d;
        }
    } else {
        q = infl / r.d;
        rem = infl % r.d;
    }
    r.bi = c.sGL()[i] + q;
    r.bf = rem;
    return r;
}

/* Report pass over the allocation in g[] (analysis.py:280-298 evaluate:
 * every memory / CPU segment response, end_to_end): each task's e2e bound
 * as a numerator over den = 2 A g (1 without kernels).  Views of tasks
 * [0, have_views) are current.  Returns 0 or ST_ESCALATE. */
template <class TM>
RT_HD int lat_report(const TM &tm, const LCtx &c, int have_views, bool stop_at_fail, i64 *e2e, i64 *den) {
    const int n = c.n;
    int k = 0;
    #pragma unroll 1
    for (; k < n; k++) {
        if (k > 0 && k > have_views) lat_view(tm, c, k - 1);
        const int info = c.info()[k];
        const int m = li_m(info), p = li_p(info);
        const i64 D = c.D()[k];
        const Seg32 sg = c.segs(k);
        const Seg32 cl_hi = sg + m, ml_hi = sg + 2 * m + p;
        const LBase gr = lat_grup(c, k, c.g()[k]);
        i64 sum_mr = 0;
        i64 *bases = c.bases();
        if (p > 0) { /* analysis.py:156, every copy */
            const i64 B = c.B()[k];
            tm.pfor(p, [&](int j) { bases[j] = ml_hi[j] + B; });
            sum_mr = lat_chain_sum(tm, c, lat_key(c, k, K_MEM), p, D);
            if (sum_mr == -2) return ST_ESCALATE;
        }
        tm.pfor(m, [&](int j) { bases[j] = cl_hi[j]; });
        const LKey chc = lat_key(c, k, K_CPU);
        const i64 sum_cr = lat_chain_sum(tm, c, chc, m, D); /* analysis.py:175 */
        if (sum_cr == -2) return ST_ESCALATE;
        /* end_to_end (analysis.py:191): None if some MR is None; R1 if every
         * CR exists and the sum fits D; R2 the whole-task recurrence */
        i64 e_int = -1;
        if (sum_mr >= 0) {
            if (sum_cr >= 0) {
                const i64 r1 = gr.bi + sum_mr + sum_cr;
                if (!lb_over(LBase{r1, gr.bf, gr.d}, 0.0, D)) e_int = r1;
            }
            const LBase b2 = {gr.bi + sum_mr + c.sClu()[k], gr.bf, gr.d};
            const double r2 = lfp_lat(tm, chc, b2, 0.0, D);
            if (r2 == -2.0) return ST_ESCALATE;
            if (r2 >= 0) {
                const i64 v = b2.bi + (i64)r2;
                if (e_int < 0 || v < e_int) e_int = v;
            }
        }
        i64 num = RTGPU_NONE;
        if (e_int >= 0) {
            const i128 w = (i128)e_int * gr.d + gr.bf;
            if (w > (i128)((i64)1 << 62)) return ST_ESCALATE;
            num = (i64)w;
        }
        if (tm.leader()) {
            e2e[k] = num;
            den[k] = gr.d;
        }
        if (e_int < 0 && stop_at_fail) {
            k++;
            break;
        }
    }
    #pragma unroll 1
    for (; k < n; k++)
        if (tm.leader()) {
            e2e[k] = RTGPU_ABSENT;
            den[k] = 1;
        }
    tm.sync();
    return 0;
}

/* Per-task code of lattice_set's setup scan: ST_ESCALATE (unsupported,
 * irregular, inverted kernel, priorities out of order), the unschedulable
 * verdict of an isolated failure (RTGPU_UNSCHEDULABLE is 0), or
 * LAT_GO (-1): nothing decided. */
enum { LAT_GO = -1 };
RT_HD int lat_task_code(const LCtx &c, int k) {
    const int fl = li_flags(c.info()[k]);
    if (fl & (TF_UNSUP | TF_IRREG | TF_INV)) return ST_ESCALATE;
    if (fl & TF_ISOFAIL) return RTGPU_UNSCHEDULABLE; /* empty report */
    if (k > 0 && c.prio()[k] < c.prio()[k - 1]) return ST_ESCALATE;
    return LAT_GO;
}
#ifdef __CUDACC__
template <int W>
__device__ __forceinline__ int lat_setup_scan(const LTeam<W> &tm, const LCtx &c, int n, int GN, i64 &need,
                                              i64 &vb_max, int &gtop) {
    i64 nd = 0, vb = 0;
    #pragma unroll 1
    for (int base = 0; base < n; base += 32) {
        const int k = base + tm.lane;
        int ck = LAT_GO;
        if (k < n) {
            ck = lat_task_code(c, k);
            if (li_gpu(c.info()[k])) nd += c.gmin()[k];
            vb = tmax(vb, *(const i64 *)(c.VC() + (size_t)k * c.L().SC));
        }
        const unsigned bad = __ballot_sync(0xffffffffu, ck != LAT_GO);
        if (bad) return __shfl_sync(0xffffffffu, ck, __ffs(bad) - 1);
    }
    #pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        nd += shfl_x(nd, off);
        vb = tmax(vb, shfl_x(vb, off));
    }
    need = nd;
    vb_max = vb;
    if (need > GN) return RTGPU_UNSCHEDULABLE; /* no allocation at all: empty report */
    int gt = 1;
    for (int k = tm.lane; k < n; k += 32)
        if (li_gpu(c.info()[k])) gt = tmax(gt, (int)tmin((i64)GN, (i64)c.gmin()[k] + (GN - need)));
    #pragma unroll
    for (int off = 16; off > 0; off >>= 1) gt = tmax(gt, __shfl_xor_sync(0xffffffffu, gt, off));
    gtop = gt;
    return LAT_GO;
}
#endif
RT_HD int lat_setup_scan(const LSeq &, const LCtx &c, int n, int GN, i64 &need, i64 &vb_max, int &gtop) {
    need = 0;
    vb_max = 0;
    for (int k = 0; k < n; k++) {
        const int ck = lat_task_code(c, k);
        if (ck != LAT_GO) return ck;
        if (li_gpu(c.info()[k])) need += c.gmin()[k];
        vb_max = tmax(vb_max, *(const i64 *)(c.VC() + (size_t)k * c.L().SC));
    }
    if (need > GN) return RTGPU_UNSCHEDULABLE;
    gtop = 1;
    for (int k = 0; k < n; k++)
        if (li_gpu(c.info()[k])) gtop = tmax(gtop, (int)tmin((i64)GN, (i64)c.gmin()[k] + (GN - need)));
    return LAT_GO;
}

/* The whole RTGPU analysis of one compact blob: status, allocation (vsm),
 * the number of task evaluations, and with `bounds` the report's end-to-end
 * bounds (e2e / den, else unused). */
template <class TM>
RT_HD int lattice_set(const TM &tm, LCtx &c, bool bounds, int32_t *vsm, i64 *e2e, i64 *den, i64 &evals) {
    const i64 *h = c.blob;
    const int n = (int)h[0], GN = (int)h[1];
    const i64 A = h[3];
    c.n = n;
    c.GN = GN;
    c.mm = (int)h[2];
    c.A = A;
    evals = 0;
    if ((h[7] != 1 && h[7] != 2) || n < 1 || n > c.L().maxn || A < 1 || (c.mm != 0 && c.mm != 1) || GN < 1 || GN > (1 << 20))
        return ST_ESCALATE;
    /* loads; each task's range bound parks in its (not yet built) CPU view */
    tm.pfor(n, [&](int i) {
        *(i64 *)(c.VC() + (size_t)i * c.L().SC) = lat_load(c, i);
        vsm[i] = 0;
        if (bounds) {
            e2e[i] = RTGPU_ABSENT;
            den[i] = 1;
        }
    });
    const int *info = c.info();
    i64 need = 0, vb_max = 0;
    int gtop = 1;
    {
        /* reference order: the first task whose minimum-count search raises
         * or fails decides; then the minimum counts' sum, the range bound
         * and gtop -- lane-parallel, one ballot per 32 tasks */
        const int code = lat_setup_scan(tm, c, n, GN, need, vb_max, gtop);
        if (code != LAT_GO) return code;
    }
    /* hp(k) = [0, first index of k's priority); blocking term of
     * analysis.py:162 = longest copy of a lower-priority task (B[] holds each
     * task's longest copy until the barrier) */
    i64 *bases = c.bases();
    tm.pfor(n, [&](int k) {
        const i64 pk = c.prio()[k];
        int first = k;
        while (first > 0 && c.prio()[first - 1] == pk) first--;
        c.hpn()[k] = first;
        i64 b = 0;
        #pragma unroll 1
        for (int i = k + 1; i < n; i++)
            if (c.prio()[i] > pk) b = tmax(b, c.B()[i]);
        *(i64 *)(c.VC() + (size_t)k * c.L().SC) = b;
    });
    tm.pfor(n, [&](int k) { c.B()[k] = *(const i64 *)(c.VC() + (size_t)k * c.L().SC); });
    bool allq = false;
#ifndef RTGPU_LAT_NOALLQUICK
    /* ---- every task at its minimum count at once (two-copy sets whose
     * tasks all have kernels).  The quick pass's cycle bounds do not depend
     * on the hp tasks' counts there: a CPU chain's cycle is C = T s and its
     * segments total sClu s, a two-copy memory chain's C = T s and sMlu s,
     * so task i's bound (floor(H s / C) + 2) EP / s is (floor(H / T_i) + 2)
     * sClu_i (CPU) or sMlu_i (memory), exact integers.  Each task's test is
     * then independent of the others' views: lanes test all tasks in
     * parallel, and if every one passes at g_min, the all-minimum allocation
     * -- the first one Algorithm 2 enumerates (analysis.py:250) -- is
     * schedulable: that is the reference's answer, with no view built. */
    if (c.mm == RTGPU_TWO_COPY) {
        /* floor(a / b), 0 <= a, b < 2^52, from 1 / b: estimate + exact corrections */
        auto fdiv = [](i64 a, i64 b, double inv) -> i64 {
            if ((a | b) >= ((i64)1 << 52)) return a / b; /* beyond the exact FP64 estimate */
            i64 q = (i64)((double)a * inv);
            if (q * b > a) q--;
            else if ((q + 1) * b <= a) q++;
            return q;
        };
        int *gk = c.g();
        tm.pfor(n, [&](int k) {
            const int inf = info[k];
            int ok = 0;
            if (li_gpu(inf) && li_p(inf) > 0) {
                const int p = li_p(inf), nh = c.hpn()[k];
                const i64 D = c.D()[k];
                i64 iu = 0;
                #pragma unroll 1
                for (int i = 0; i < nh && iu <= D; i++) iu += (fdiv(D, c.T()[i], c.invT()[i]) + 2) * c.sClu()[i];
                const LBase gr = lat_grup(c, k, c.gmin()[k]);
                const i64 B = c.B()[k];
                const i64 bmax = c.Mx()[k] + B, bsum = c.sMlu()[k] + (i64)p * B;
                const i64 M = D - iu - c.sClu()[k] - gr.bi - (gr.bf > 0 ? 1 : 0) - bsum;
                if (M >= 0) {
                    i64 rs = M / p;
                    if (rs > D - bmax) rs = D - bmax;
                    if (rs >= 0) {
                        const i64 H = bmax + rs;
                        i64 um = 0;
                        #pragma unroll 1
                        for (int i = 0; i < nh && um <= rs; i++) um += (fdiv(H, c.T()[i], c.invT()[i]) + 2) * c.sMlu()[i];
                        ok = um <= rs;
                    }
                }
            }
            gk[k] = ok ? c.gmin()[k] : -1;
        });
        bool all = true;
        #pragma unroll 1
        for (int k = 0; k < n; k++) all = all && gk[k] > 0;
        if (all) {
            RT_COUNT(g_cnt_eval);
            if (!bounds) {
                evals = n;
                tm.pfor(n, [&](int i) { vsm[i] = 2 * gk[i]; });
                return RTGPU_SCHEDULABLE;
            }
            allq = true; /* counts in g[]: the search is skipped, the report (one call site) follows */
        } else {
            tm.pfor(n, [&](int k) { gk[k] = 0; });
        }
    }
#endif
    /* the search and the report run on FP64 views: every value at any scale
     * s_i <= 2 gtop below 2^51 (room for the half-tick marker), the window
     * fraction bf * s_i below 2^52 (the all-minimum pass above is integer
     * arithmetic and takes any range the loads accept) */
    if ((i128)vb_max * range_factor(n, c.L().MC, c.L().MP) * (2 * gtop) >= ((i128)1 << 51) ||
        (i128)4 * A * gtop * gtop >= ((i128)1 << 52)) {
        if (allq) tm.pfor(n, [&](int k) { c.g()[k] = 0; });
        return ST_ESCALATE;
    }
    (void)bases;
    /* The search state is warp-uniform and lives in the warp's LSt in shared
     * memory (every lane stores the same value): across the out-of-line fixed
     * points it is reloaded from there instead of being spilled per lane to
     * a stack frame that does not fit L1 (the r2w profile: 60% of the
     * control code's stall samples waited on local loads missing to L2).
     * Per-task values are re-read from the slab's task records at use. */
    LSt &S = *c.stp();
    S.used = 0;
    S.rest_min = need;
    /* warm starts: the last converged memory / CPU fixed point (base, N);
     * valid for any later task (hp(k) only grows) at a base >= its base */
    S.mw = LBase{-1, 0, 1};
    S.cw = LBase{-1, 0, 1};
    S.mwN = 0;
    S.cwN = 0;
    S.mg = -1.0; /* the last task's memory offset (or its verified bound): the next guess */
    S.st = RTGPU_SCHEDULABLE;
    S.evals = allq ? n : 0;
    #pragma unroll 1
    for (S.k = allq ? c.n : 0; S.k < c.n; S.k++) {
        if (S.k > 0) lat_view(tm, c, S.k - 1); /* counts of tasks before k are final */
        {
            const int k = S.k;
            const int inf = c.info()[k];
            const bool gpu = li_gpu(inf);
            S.glo = S.ghi = 0;
            if (gpu) {
                const int gm = c.gmin()[k];
                S.rest_min -= gm;
                const i64 gmax = c.GN - S.used - S.rest_min;
                if (gmax < gm) {
                    S.st = RTGPU_UNSCHEDULABLE;
                    break;
                }
                S.glo = gm;
                S.ghi = (int)gmax;
            }
        }
        /* ---- g-independent: the longest copy's response bounds every MR.
         * First a guess verified in one evaluation: the previous task's
         * offset grown by half, accepted when b + N is a pre-fixed point
         * (then lfp <= f(b + N) <= D: every MR exists and MR_j <= the bound
         * minus (bmax - b_j)); consecutive tasks' memory fixed points differ
         * by ~14% (hp(k) grows by one task), so the guess usually holds and
         * saves the iterations from 0.  The exact fixed point is computed
         * only if R2 fails with the looser bound. */
#ifndef RTGPU_LAT_NOQUICK
        /* ---- quick pass at the minimum count (sufficient, one CPU and one
         * memory evaluation): I_cpu(D) bounds the CPU interference of any
         * window <= D, so R2 passes at glo as soon as
         *   GR_bi + [GR_bf > 0] + sum MR + sClu + I_cpu(D) <= D
         * (a pre-fixed point at b + floor offset <= D, analysis.py:214).
         * That leaves room M for sum MR <= p r + bsum, r the longest copy's
         * offset bound; r* = floor((M - bsum) / p) is verified as a memory
         * pre-fixed point (then every MR exists and MR_j <= b_j + r*,
         * analysis.py:156).  Otherwise the exact search below. */
        if (li_gpu(c.info()[S.k]) && li_p(c.info()[S.k]) > 0) {
            const int k = S.k, inf = c.info()[k], m = li_m(inf), p = li_p(inf);
            i64 bmax = 0, bsum = 0;
            lat_copy_sums(tm, c.segs(k) + 2 * m + p, p, c.B()[k], bmax, bsum);
            S.bsum = bsum;
            S.lbm = LBase{bmax, 0, 1};
#ifndef RTGPU_LAT_NOCYCLE
            /* the CPU interference at D first from the cycle bound (no walks);
             * the exact I_cpu(D) only if that leaves too little room */
            double iu = lat_cycle_bound(tm, c, S.k, K_CPU, (double)c.D()[S.k]) + 1e-6;
            bool iu_exact = false;
#else
            double iu = lfp_lat(tm, lat_key(c, S.k, K_CPU), LBase{0, 0, 1}, (double)c.D()[S.k], c.D()[S.k], 2);
            bool iu_exact = true;
#endif
            double r = -1.0;
            #pragma unroll 1
            for (;;) {
                const int kk = S.k;
                const LBase gr = lat_grup(c, kk, S.glo);
                const double M = (double)c.D()[kk] - iu - (double)c.sClu()[kk] - (double)gr.bi -
                                 (gr.bf > 0 ? 1.0 : 0.0) - (double)S.bsum;
                /* (any smaller offset bound leaves R2 passing: at most the deadline) */
                const double rs = tmin(floor(M / (double)li_p(c.info()[kk])), (double)(c.D()[kk] - S.lbm.bi));
                if (rs >= 0) {
#ifndef RTGPU_LAT_NOCYCLE
                    /* the memory pre-fixed point from the cycle bound, then by one evaluation */
                    if (lat_cycle_bound(tm, c, S.k, K_MEM, (double)S.lbm.bi + rs) + 1e-6 <= rs) {
                        RT_COUNT(g_cnt_flfp[3]);
                        r = rs;
                        break;
                    }
#endif
                    r = lfp_lat(tm, lat_key(c, S.k, K_MEM), S.lbm, rs, c.D()[S.k], 1);
                    if (r >= 0) break;
                }
                if (iu_exact) break;
                iu = lfp_lat(tm, lat_key(c, S.k, K_CPU), LBase{0, 0, 1}, (double)c.D()[S.k], c.D()[S.k], 2);
                iu_exact = true;
            }
            {
                if (r >= 0) {
                    RT_COUNT(g_cnt_flfp[2]);
                    S.mg = r;
                    S.evals++;
                    if (tm.leader()) c.g()[S.k] = S.glo;
                    tm.sync();
                    S.used += S.glo;
                    continue;
                }
            }
        }
#endif
        S.mr_ub = 0;
        S.sum_mr = -1;
        S.bsum = 0;
        S.lbm = LBase{0, 0, 1};
        S.rmax_exact = 1;
        if (li_p(c.info()[S.k]) > 0) {
            {
                const int k = S.k, inf = c.info()[k], m = li_m(inf), p = li_p(inf);
                i64 bmax = 0, bsum = 0;
                lat_copy_sums(tm, c.segs(k) + 2 * m + p, p, c.B()[k], bmax, bsum);
                S.bsum = bsum;
                S.lbm = LBase{bmax, 0, 1};
            }
            double r = -1.0;
#ifndef RTGPU_LAT_NOGUESS
            if (S.mg >= 1.0) { /* (after a task without memory interference there is nothing to grow) */
#else
            if (false) {
#endif
#ifndef RTGPU_LAT_GUESS_F
#define RTGPU_LAT_GUESS_F 1.5
#endif
#ifndef RTGPU_LAT_GUESS_MODE
#define RTGPU_LAT_GUESS_MODE 0
#endif
#if RTGPU_LAT_GUESS_MODE == 1
                /* the interference grows with the hp count: k / (k - 1) */
                const int nh = c.hpn()[S.k], ph = S.k > 0 ? c.hpn()[S.k - 1] : 0;
                const double Ng = ceil(RTGPU_LAT_GUESS_F * S.mg * (double)nh / (double)(ph > 0 ? ph : 1)) + 1.0;
#else
                const double Ng = ceil(RTGPU_LAT_GUESS_F * S.mg) + 1.0;
#endif
                const i64 D = c.D()[S.k];
                if (!lb_over(S.lbm, Ng, D)) r = lfp_lat(tm, lat_key(c, S.k, K_MEM), S.lbm, Ng, D, 1);
                S.rmax_exact = r < 0;
            }
            if (r < 0) {
                RT_COUNT(g_cnt_flfp[0]);
                const LBase lbm = S.lbm;
                r = lfp_lat(tm, lat_key(c, S.k, K_MEM), lbm, (S.mw.bi >= 0 && lb_le(S.mw, lbm)) ? S.mwN : 0.0,
                            c.D()[S.k]);
                if (r == -2.0) return ST_ESCALATE;
                if (r < 0) {
                    S.st = RTGPU_UNSCHEDULABLE; /* the longest copy's MR is None at every count */
                    break;
                }
                S.mw = S.lbm;
                S.mwN = r;
            }
            S.mg = r;
            S.mr_ub = (i64)li_p(c.info()[S.k]) * (i64)r + S.bsum;
        } else {
            S.sum_mr = 0;
        }
        S.sum_cr = -3; /* not computed yet; -1: some CR is None */
        /* task k passes at count g?  1 / 0, -1 = escalate */
        auto passes = [&](int g) -> int {
            RT_COUNT(g_cnt_passes);
            /* R2 (analysis.py:214) with the upper bound on sum MR (passing is
             * then exact), then with the exact sum: one CPU fixed-point site */
            #pragma unroll 1
            for (S.pass = 0; S.pass < 2; S.pass++) {
                i64 smr = 0;
                if (S.pass == 0) {
                    smr = li_p(c.info()[S.k]) > 0 ? S.mr_ub : 0;
                } else {
                    const int p = li_p(c.info()[S.k]);
                    if (p == 0) break;
                    if (!S.rmax_exact) {
                        /* the verified guess was too loose for R2: the exact
                         * fixed point of the longest copy, then R2 again */
                        RT_COUNT(g_cnt_flfp[1]);
                        const double r = lfp_lat(tm, lat_key(c, S.k, K_MEM), S.lbm, 0.0, c.D()[S.k]);
                        if (r < 0) return -1; /* cannot be None below a verified bound */
                        S.rmax_exact = 1;
                        S.mw = S.lbm;
                        S.mwN = r;
                        S.mg = r;
                        const i64 ub = (i64)li_p(c.info()[S.k]) * (i64)r + S.bsum;
                        if (ub < S.mr_ub) {
                            S.mr_ub = ub;
                            S.pass = -1; /* retry R2 with the exact bound */
                            continue;
                        }
                    }
                    if (S.sum_mr < 0) {
                        {
                            const int k = S.k, inf = c.info()[k], m = li_m(inf), pp = li_p(inf);
                            const Seg32 ml_hi = c.segs(k) + 2 * m + pp;
                            const i64 B = c.B()[k];
                            tm.pfor(pp, [&](int j) { c.bases()[j] = ml_hi[j] + B; });
                        }
                        RT_COUNT(g_cnt_flfp[2]);
                        S.sum_mr = lat_chain_sum(tm, c, lat_key(c, S.k, K_MEM), li_p(c.info()[S.k]), c.D()[S.k]);
                        if (S.sum_mr < 0) return -1; /* -2, or None (impossible: the longest copy's is not) */
                    }
                    if (S.sum_mr == S.mr_ub) break;
                    smr = S.sum_mr;
                }
                const LBase gr = lat_grup(c, S.k, g);
                const i64 D = c.D()[S.k];
                const LBase b = {gr.bi + smr + c.sClu()[S.k], gr.bf, gr.d};
                /* R2 passes iff lfp <= D; a pre-fixed point at the deadline
                 * itself (f(D) <= D) proves it in one evaluation -- the
                 * common case with slack; otherwise the fixed point */
                const double nd = (double)(D - b.bi - (b.bf > 0 ? 1 : 0));
#ifndef RTGPU_LAT_NODCHECK
                if (nd >= 0 && lfp_lat(tm, lat_key(c, S.k, K_CPU), b, nd, D, 1) >= 0) return 1;
#else
                (void)nd;
#endif
                {
                    const i64 D2 = c.D()[S.k];
                    const LBase gr2 = lat_grup(c, S.k, g);
                    const LBase b2 = {gr2.bi + smr + c.sClu()[S.k], gr2.bf, gr2.d};
                    RT_COUNT(g_cnt_lfp[1]);
                    const double r = lfp_lat(tm, lat_key(c, S.k, K_CPU), b2, (S.cw.bi >= 0 && lb_le(S.cw, b2)) ? S.cwN : 0.0, D2);
                    if (r == -2.0) return -1;
                    if (r >= 0) {
                        S.cw = b2;
                        S.cwN = r;
                        return 1;
                    }
                }
            }
            /* R1 = GR up + sum MR + sum CR (analysis.py:207); CRs do not depend on g */
            if (S.sum_cr == -3) {
                {
                    const int k = S.k, inf = c.info()[k], m = li_m(inf);
                    const Seg32 cl_hi = c.segs(k) + m;
                    tm.pfor(m, [&](int j) { c.bases()[j] = cl_hi[j]; });
                }
                RT_COUNT(g_cnt_flfp[3]);
                S.sum_cr = lat_chain_sum(tm, c, lat_key(c, S.k, K_CPU), li_m(c.info()[S.k]), c.D()[S.k]);
                if (S.sum_cr == -2) return -1;
            }
            if (S.sum_cr < 0) return 0;
            const LBase gr = lat_grup(c, S.k, g);
            return lb_over(LBase{gr.bi + S.sum_mr + S.sum_cr, gr.bf, gr.d}, 0.0, c.D()[S.k]) ? 0 : 1;
        };
        S.evals++;
        /* smallest passing count: glo, else ghi, else bisection (own-count
         * monotone); one call site keeps one inlined copy of `passes` */
        {
            const bool gpu = li_gpu(c.info()[S.k]);
            S.g = 0;
            S.lo = S.glo;
            S.hi = S.ghi;
            /* the largest count first (fast path: engine_core.cuh) */
            S.phase = gpu ? 1 : 3;
            S.cand = gpu ? S.ghi : 0;
            S.fail = 0;
        }
        #pragma unroll 1
        for (;;) {
            const int o = passes(S.cand);
            if (o < 0) return ST_ESCALATE;
            const int phase = S.phase;
            if (phase == 3) {
                S.fail = !o;
                break;
            }
            if (phase == 1) {
                if (!o) {
                    S.fail = 1;
                    break;
                }
                if (S.glo >= S.ghi) {
                    S.g = S.ghi;
                    break;
                }
                S.phase = 0;
                S.cand = S.glo;
                continue;
            }
            if (phase == 0) {
                if (o) {
                    S.g = S.glo;
                    break;
                }
                S.phase = 2;
            } else if (o) {
                S.hi = S.cand;
            } else {
                S.lo = S.cand;
            }
            const int lo = S.lo, hi = S.hi;
            if (hi - lo <= 1) {
                S.g = hi;
                break;
            }
            S.cand = lo + (hi - lo) / 2;
        }
        if (S.fail) {
            S.st = RTGPU_UNSCHEDULABLE;
            break;
        }
        if (!li_gpu(c.info()[S.k])) continue;
        if (tm.leader()) c.g()[S.k] = S.g;
        tm.sync();
        S.used += S.g;
    }
    const int st = S.st;
    evals = S.evals;
    if (st == RTGPU_SCHEDULABLE) tm.pfor(n, [&](int i) { vsm[i] = li_gpu(c.info()[i]) ? 2 * c.g()[i] : 0; });
    if (!bounds) return st;
    int have = allq ? 0 : n - 1;
    if (st == RTGPU_UNSCHEDULABLE) {
        /* the reference reports the last allocation it tried: the
         * lexicographically largest (first GPU task takes the rest) */
        int first = -1;
        i64 others = 0;
        #pragma unroll 1
        for (int k = 0; k < n; k++)
            if (li_gpu(info[k])) {
                if (first < 0) first = k;
                else others += c.gmin()[k];
            }
        tm.sync();
        if (tm.leader())
            #pragma unroll 1
            for (int k = 0; k < n; k++)
                c.g()[k] = li_gpu(info[k]) ? (k == first ? (int)(GN - others) : c.gmin()[k]) : 0;
        tm.sync();
        have = 0;
    }
    const int r = lat_report(tm, c, have, st == RTGPU_UNSCHEDULABLE, e2e, den);
    return r ? r : st;
}

}  // namespace rtgpu
