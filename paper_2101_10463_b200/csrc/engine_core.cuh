/*
 * engine_core.cuh -- the RTGPU analysis of one packed task set, written once
 * for a cooperating "team": a 32-lane warp on sm_100a (WarpTeam, the
 * product) or a sequential emulation of the same lanes (SeqTeam, used only by
 * the test harness in tests/ to check the logic on a CPU-only box).
 *
 * What is computed: exactly gpusched.analysis.analyze(ts, RTGPU) -- verdict,
 * the lexicographically first schedulable SM allocation of Algorithm 2
 * (reference analysis.py:250 _grid_search over gpu.py:69
 * feasible_allocations) and, on request, the report bounds.
 *
 * How (DESIGN.md section 3 has the proofs):
 *  - Exact arithmetic.  For a given prefix of the allocation every value is a
 *    rational with denominator dividing Q = 2*lcm(GN_i)*[A*GN_k]; the warp
 *    scales inputs by Q and computes in V = double (integer-valued, exact
 *    below 2^52), int64 or int128.  A set whose range does not fit V is
 *    escalated to the next V by the host driver, never approximated.
 *  - Chain workload W_i^h(t) (suspension.py:77) in O(p): prefix sums of
 *    segment+gap over one job, a floor-division jump over whole periods
 *    (one steady period is exactly the cycle length C), and the final
 *    partial period.  Lanes own (task i, start segment h) pairs; max over h
 *    and sum over hp(k) are warp shuffles.
 *  - Fixed points (suspension.py:123) iterate from below with two exact
 *    accelerations that cannot skip the least fixed point: warm starts from
 *    the fixed point of a smaller base, and a slope-1 jump (a maximising
 *    walk still inside a segment keeps the interference growing at slope 1,
 *    so no fixed point lies within its remaining length).
 *  - Allocation search.  Task k's verdict depends only on the SM counts of
 *    tasks before it in priority order (prefix property) and is monotone in
 *    its own count (Lemma 4 bound shrinks with GN_k).  When no gap can go
 *    negative ("regular" sets -- every validated set), interference is also
 *    monotone in the hp counts, so the first schedulable allocation in
 *    lexicographic order is the greedy one: each task takes the smallest
 *    passing count, found by bisection.  Irregular sets run an exact
 *    depth-first search with prefix pruning under an evaluation budget.
 */
#pragma once
#include <stdint.h>
#include <string.h>

#include "../../include/rtgpu.h"

#ifdef __CUDACC__
#define RT_HD __host__ __device__ inline
/* out-of-line: one copy of each big routine keeps the kernel inside the
 * instruction cache (the fully inlined kernel was ~680 KB of SASS) */
#define RT_NI __host__ __device__ __noinline__
#else
#define RT_HD inline
#define RT_NI inline
#endif

namespace rtgpu {

typedef long long i64;
typedef __int128 i128;

enum { K_CPU = 0, K_MEM = 1 };

/* internal status: range exceeded for this arithmetic -> escalate */
enum { ST_ESCALATE = 99 };

static const int ITER_CAP = 1 << 22; /* safety net per fixed point */

/* ------------------------------------------------------------ arithmetic */

template <class V> struct Num;

template <> struct Num<double> {
    typedef i64 Qt;
    static RT_HD i64 limit() { return (i64)1 << 52; }
    /* x * q as an exact double: both factors are exact (< 2^53) and the
     * stage's range check keeps every product below 2^52, so one DMUL
     * replaces a 64-bit integer multiply and its conversion */
    static RT_HD double sc(i64 x, i64 q) { return (double)x * (double)q; }
    static RT_HD double of(i64 x) { return (double)x; }
    static RT_HD double floordiv(double a, double b) {
        double q = floor(a / b);
        if (q * b > a) q -= 1.0;
        else if ((q + 1.0) * b <= a) q += 1.0;
        return q;
    }
    static RT_HD double make_inv(double C) { return C > 0 ? 1.0 / C : 0.0; }
    /* floor(a / b) from a precomputed inv ~ 1/b: estimate, then exact
     * corrections (products are exact integers below 2^53) */
    static RT_HD double floordiv_inv(double a, double b, double inv) {
        double q = floor(a * inv);
        while (q * b > a) q -= 1.0;
        while ((q + 1.0) * b <= a) q += 1.0;
        return q;
    }
    /* q = floor(a / b) and r = a - q b (a >= 0, b > 0, integers < 2^52):
     * the fma remainder is exact, one correction covers the estimate's error */
    static RT_HD double divmod_inv(double a, double b, double inv, double &r) {
        double q = floor(a * inv);
        r = fma(-q, b, a);
        if (r < 0) {
            q -= 1.0;
            r += b;
        } else if (r >= b) {
            q += 1.0;
            r -= b;
        }
        if (r < 0 || r >= b) { /* never for |a| < 2^52; kept for safety */
            q = floordiv(a, b);
            r = a - q * b;
        }
        return q;
    }
    static RT_HD i128 wide(double v) { return (i128)(i64)v; }
};

template <> struct Num<i64> {
    typedef i64 Qt;
    static RT_HD i64 limit() { return (i64)1 << 62; }
    static RT_HD i64 sc(i64 x, i64 q) { return x * q; }
    static RT_HD i64 of(i64 x) { return x; }
    static RT_HD i64 floordiv(i64 a, i64 b) { return a / b; }
    static RT_HD i64 make_inv(i64 C) {
        double inv = C > 0 ? 1.0 / (double)C : 0.0;
        i64 bits;
        memcpy(&bits, &inv, 8);
        return bits;
    }
    static RT_HD i64 divmod_inv(i64 a, i64 b, i64 inv_bits, i64 &r) {
        i64 q = floordiv_inv(a, b, inv_bits);
        r = a - q * b;
        return q;
    }
    static RT_HD i64 floordiv_inv(i64 a, i64 b, i64 inv_bits) {
        double inv;
        memcpy(&inv, &inv_bits, 8);
        i64 q = (i64)((double)a * inv);
        if (q < 0) q = 0;
        while (q > 0 && q * b > a) q--;
        while ((q + 1) * b <= a) q++;
        return q;
    }
    static RT_HD i128 wide(i64 v) { return (i128)v; }
};

template <> struct Num<i128> {
    typedef i128 Qt;
    static RT_HD i128 limit() { return (i128)1 << 125; }
    static RT_HD i128 sc(i64 x, i128 q) { return (i128)x * q; }
    static RT_HD i128 of(i64 x) { return (i128)x; }
    static RT_HD i128 floordiv(i128 a, i128 b) { return a / b; }
    static RT_HD i128 make_inv(i128) { return 0; }
    static RT_HD i128 floordiv_inv(i128 a, i128 b, i128) { return a / b; }
    static RT_HD i128 divmod_inv(i128 a, i128 b, i128, i128 &r) {
        i128 q = a / b;
        r = a - q * b;
        return q;
    }
    static RT_HD i128 wide(i128 v) { return v; }
};

template <class T> RT_HD T tmax(T a, T b) { return a > b ? a : b; }
template <class T> RT_HD T tmin(T a, T b) { return a < b ? a : b; }

template <class T> RT_HD T gcdq(T a, T b) {
    if (a < 0) a = -a;
    if (b < 0) b = -b;
    if (a <= (T)0x7fffffff && b <= (T)0x7fffffff) { /* native 32-bit remainder */
        unsigned x = (unsigned)a, y = (unsigned)b;
        while (y != 0) {
            unsigned t = x % y;
            x = y;
            y = t;
        }
        return (T)x;
    }
    while (b != 0) {
        T t = a % b;
        a = b;
        b = t;
    }
    return a;
}

/* lcm with overflow detection against lim; returns 0 on overflow */
template <class T> RT_HD T lcm_lim(T a, T b, T lim) {
    T g = gcdq(a, b);
    T a1 = a / g;
    if (a1 > lim / b) return 0;
    return a1 * b;
}

/* lcm(1..n) for n <= 42 (lcm(1..43) exceeds int64): the fast path's
 * scale factor, a constant per GN instead of GN - 1 gcd loops per set */
#define RT_LCM_TABLE                                                                                      \
    {1LL, 1LL, 2LL, 6LL, 12LL, 60LL, 60LL, 420LL, 840LL, 2520LL, 2520LL, 27720LL, 27720LL, 360360LL,            \
     360360LL, 360360LL, 720720LL, 12252240LL, 12252240LL, 232792560LL, 232792560LL, 232792560LL,           \
     232792560LL, 5354228880LL, 5354228880LL, 26771144400LL, 26771144400LL, 80313433200LL,                  \
     80313433200LL, 2329089562800LL, 2329089562800LL, 72201776446800LL, 144403552893600LL,                  \
     144403552893600LL, 144403552893600LL, 144403552893600LL, 144403552893600LL, 5342931457063200LL,        \
     5342931457063200LL, 5342931457063200LL, 5342931457063200LL, 219060189739591200LL,                      \
     219060189739591200LL}
#ifdef __CUDACC__
static __constant__ i64 rt_lcm_dev[43] = RT_LCM_TABLE;
#endif
static const i64 rt_lcm_host[43] = RT_LCM_TABLE;
RT_HD i64 lcm_upto(int n) {
    if (n < 0 || n > 42) return 0;
#ifdef __CUDA_ARCH__
    return rt_lcm_dev[n];
#else
    return rt_lcm_host[n];
#endif
}

/* ------------------------------------------------------------ segment access */

/* A task's segment area in either blob format: int64 words (header word 7
 * = 0) or int32 (header word 7 = 1, the compact form the generator writes;
 * halves the bytes a batch moves over PCIe and HBM). */
/* a task record of either form (header word 7 == 2: packed 4-word
 * records, include/rtgpu.h); fields numbered as in the 8-word record */
struct RecP {
    const i64 *w;
    bool packed;
    RT_HD i64 operator[](int f) const {
        if (!packed) return w[f];
        switch (f) {
        case 0: return w[2] & 0xff;
        case 1: return (w[2] >> 8) & 0xff;
        case 2: return w[0];
        case 3: return w[1];
        case 4: return (i64)(int32_t)(uint32_t)((unsigned long long)w[3] & 0xffffffffull);
        case 5: return w[3] >> 32;
        case 6: return w[2] >> 16;
        default: return 0;
        }
    }
};
RT_HD RecP rec_at(const i64 *blob, int i) {
    RecP r;
    r.packed = blob[7] == 2;
    r.w = blob + RTGPU_HDR_WORDS + (r.packed ? RTGPU_TASK_WORDS / 2 : RTGPU_TASK_WORDS) * i;
    return r;
}

struct SegPtr {
    const void *p;
    int w; /* 0: int64, 1: int32 */
    RT_HD i64 operator[](int j) const {
        return w ? (i64)((const int32_t *)p)[j] : ((const i64 *)p)[j];
    }
    RT_HD SegPtr operator+(int j) const {
        SegPtr r;
        r.p = w ? (const void *)((const int32_t *)p + j) : (const void *)((const i64 *)p + j);
        r.w = w;
        return r;
    }
};

/* The compact (int32) segment area with the width known at compile time:
 * the verdict fast path runs only on compact blobs, so its reads are plain
 * 32-bit loads with no per-access width select. */
#if defined(__CUDA_ARCH__) && defined(RTGPU_BLOB_EVICT_FIRST)
/* batch words are read once per set: an L2 evict-first hint keeps the stream
 * of them from evicting the warps' (dirty) local-memory lines, whose
 * write-backs otherwise double the kernel's DRAM traffic */
__device__ __forceinline__ int32_t ld_batch32(const int32_t *a) {
    int32_t v;
    asm("{\n\t.reg .b64 pol;\n\tcreatepolicy.fractional.L2::evict_first.b64 pol, 1.0;\n\t"
        "ld.global.L2::cache_hint.b32 %0, [%1], pol;\n\t}"
        : "=r"(v)
        : "l"(__cvta_generic_to_global(a)));
    return v;
}
#endif

struct Seg32 {
    const int32_t *p;
#if defined(__CUDA_ARCH__) && defined(RTGPU_BLOB_EVICT_FIRST)
    __device__ i64 operator[](int j) const { return ld_batch32(p + j); }
#else
    RT_HD i64 operator[](int j) const { return p[j]; }
#endif
    RT_HD Seg32 operator+(int j) const { return Seg32{p + j}; }
};

/* ------------------------------------------------------------ per-task data */

struct TaskRec {
    i64 D, T, prio, seg;
    i64 sClu, sCll, sMlu, sMll, sGWlo, sInfl, sGL, innerCll, maxMlu, B;
    double invT; /* 1 / T (fast path: the all-minimum pass's floor(H / T)) */
    int m, p, gmin, g;
    int isgpu, flags, idx, pad;
};

enum { TF_INV = 1, TF_ISOFAIL = 2, TF_IRREG = 4, TF_UNSUP = 8 };

/* Sizes of the per-warp shared-memory slab for a batch whose sets have at
 * most maxn tasks, MC CPU and MP memory segments per task. */
struct Dims {
    int maxn, MC, MP;
};

/* Range factor: every intermediate of an evaluation is a sum of at most
 * max(n + 2, p + m + 1, 2p + 3) terms each bounded by the per-set
 * max(D + T + sum of segments): interference sums (n), R1 = GR + sum MR +
 * sum CR (p + m + 1), the verdict shortcut's MR upper bound and R2 base
 * (2p + 3); walks and views stay below 2 max(D + T + sums). */
RT_HD int range_factor(int n, int MC, int MP) {
    int f = n + 4;
    if (MP + MC + 4 > f) f = MP + MC + 4;
    if (2 * MP + 4 > f) f = 2 * MP + 4;
    return f;
}

template <class V> struct Layout {
    int SC, SM;        /* view stride (in V) per task for CPU / memory chains */
    int off_views_c;   /* byte offsets inside the slab */
    int off_views_m;
    int off_scr;
    int scr_n;         /* scratch V entries */
    int bytes;
    RT_HD void init(const Dims &d) {
        SC = 3 * d.MC + 5;
        SM = d.MP > 0 ? 3 * d.MP + 5 : 0;
        int o = (int)sizeof(TaskRec) * d.maxn;
        o = (o + 15) & ~15;
        off_views_c = o;
        o += (int)sizeof(V) * SC * d.maxn;
        off_views_m = o;
        o += (int)sizeof(V) * SM * d.maxn;
        off_scr = o;
        scr_n = 2 * (d.MP + d.MC + 2) + d.MP + 3 * d.MC;
        scr_n += (int)((32 * sizeof(int) + sizeof(V) - 1) / sizeof(V)); /* lfp_many order */
        o += (int)sizeof(V) * scr_n;
        bytes = (o + 15) & ~15;
    }
};

/* view word WN: negative gaps of the chain (analysis.py:57, :89) */
enum {
    WN_WRAP = 1,          /* the steady-state wrap-around gap (checked: InfeasibleGapError) */
    WN_FIRST_CHECKED = 2, /* the first job's deadline-side gap of a memory chain (checked) */
    WN_FIRST_OPEN = 4     /* the first job's CPU gap T - D < 0 (used as is) */
};

/* view offsets inside one task's chain view */
struct VOff {
    int e, P, EP, F1, WN, INV;
    RT_HD VOff(int p_max)
        : e(0), P(p_max), EP(2 * p_max + 1), F1(3 * p_max + 2), WN(3 * p_max + 3), INV(3 * p_max + 4) {}
};

/* ------------------------------------------------------------ set context */

template <class V> struct SetCtx {
    typedef typename Num<V>::Qt Qt;
    const i64 *blob; /* global: this set's blob */
    /* Shared-memory slab of the warp, as byte offsets from the dynamic
     * shared-memory base: pointers are rebuilt from the extern __shared__
     * symbol inside every routine, so the compiler always knows they are
     * shared (LDS/STS, not generic LD/ST) -- also across out-of-line calls. */
    unsigned char *hbase; /* host harness only */
    int o_tr, o_vc, o_vm, o_scr;
    RT_HD unsigned char *sbase() const;
    int segw; /* header word 7: 0 int64 segment areas, 1 int32 */
    RT_HD SegPtr segs(i64 seg_off) const {
        SegPtr r;
        r.w = segw;
        r.p = segw ? (const void *)((const int32_t *)blob + seg_off) : (const void *)(blob + seg_off);
        return r;
    }
    RT_HD TaskRec *TR() const { return (TaskRec *)(sbase() + o_tr); }
    RT_HD V *VC() const { return (V *)(sbase() + o_vc); }
    RT_HD V *VM() const { return (V *)(sbase() + o_vm); }
    RT_HD V *SCR() const { return (V *)(sbase() + o_scr); }
    Layout<V> L;
    int n, GN, mm;
    i64 A;
    int maxn, MC, MP, GC, GM; /* batch maxima, lane group sizes */
    int lgC, lgM, halfC, halfM; /* log2 group sizes; binary-search first steps */
    int single_seg;     /* busy-waiting baseline: one CPU segment per task */
    int method;         /* RTGPU_METHOD_* */
    i64 Vb;             /* range bound in input ticks */
    Qt qlim;            /* largest admissible scale: limit / Vb */
    /* current views: tasks [0, vn) at scale vq */
    int vn;
    Qt vq;
    int esc;            /* range exceeded -> escalate */
    int stuck;          /* fixed point iteration cap hit */
    i64 evals, budget;
    int budget_hit;
    Qt fixed_q; /* 2*A*lcm(1..GN) when it fits the stage: one scale for the whole search */
};

#ifdef __CUDACC__
extern __shared__ __align__(16) unsigned char rt_dyn_smem[];
#endif
template <class V> RT_HD unsigned char *SetCtx<V>::sbase() const {
#ifdef __CUDA_ARCH__
    return rt_dyn_smem;
#else
    return hbase;
#endif
}

/* lane-group sizes (2^lg lanes per hp task) and binary-search first steps */
template <class V> RT_HD void set_groups(SetCtx<V> &c) {
    int g = 1, lg = 0;
    while (g < c.MC) g <<= 1, lg++;
    c.GC = g;
    c.lgC = lg;
    c.halfC = g >> 1;
    g = 1;
    lg = 0;
    while (g < (c.MP > 0 ? c.MP : 1)) g <<= 1, lg++;
    c.GM = g;
    c.lgM = lg;
    c.halfM = g >> 1;
}

/* ------------------------------------------------------------ teams */

template <class V> struct WRE { V w, rho; };

#ifdef __CUDACC__
template <class V> __device__ __forceinline__ V shfl_x(V v, int off) {
    return __shfl_xor_sync(0xffffffffu, v, off);
}
template <> __device__ __forceinline__ i128 shfl_x<i128>(i128 v, int off) {
    unsigned long long lo = (unsigned long long)v, hi = (unsigned long long)(v >> 64);
    lo = __shfl_xor_sync(0xffffffffu, lo, off);
    hi = __shfl_xor_sync(0xffffffffu, hi, off);
    return (i128)(((unsigned __int128)hi << 64) | lo);
}

struct WarpTeam {
    int lane;
    __device__ __forceinline__ void sync() const { __syncwarp(); }
    __device__ __forceinline__ bool leader() const { return lane == 0; }
    template <class F> __device__ __forceinline__ void pfor(int n, F f) const {
        /* one copy of the body: these loops are setup code (n <= 64) */
#pragma unroll 1
        for (int i = lane; i < n; i += 32) f(i);
        __syncwarp();
    }
    __device__ __forceinline__ bool any(bool b) const { return __any_sync(0xffffffffu, b); }
    /* Interference rounds: slot = lane; f(slot, w, rho, err) gives the walk
     * of one (task, start segment) pair.  Per round only the max over the
     * 2^lg lanes of a task is shuffled; each lane accumulates its group's
     * max and, if it is a maximiser, its rho.  acc_finish sums the groups
     * and takes the rho max once for all rounds. */
    template <class V> struct Acc {
        V sum, rho;
        bool err;
    };
    template <class V> __device__ __forceinline__ void acc_init(Acc<V> &a) const {
        a.sum = 0;
        a.rho = 0;
        a.err = false;
    }
    template <class V, class F>
    __device__ __forceinline__ void group_max_round(int lg, F f, Acc<V> &a) const {
        V w = 0, rho = 0;
        bool e = false;
        f(lane, w, rho, e);
        V m = w;
        for (int off = 1; off < (1 << lg); off <<= 1) {
            V o = shfl_x(m, off);
            if (o > m) m = o;
        }
        a.sum += m;
        if (w == m && rho > a.rho) a.rho = rho;
        a.err = a.err || e;
    }
    /* the group sum and the error vote only; acc_rho gives the slope-1
     * length when the iteration continues (not on the converging one) */
    template <class V>
    __device__ __forceinline__ void acc_sum(int lg, const Acc<V> &a, V &wsum, bool &err) const {
        V s = a.sum;
        for (int off = 1 << lg; off < 32; off <<= 1) s += shfl_x(s, off);
        wsum = s;
        err = __any_sync(0xffffffffu, a.err);
    }
    template <class V> __device__ __forceinline__ V acc_rho(const Acc<V> &a) const {
        V r = a.rho;
        for (int off = 1; off < 32; off <<= 1) {
            V o = shfl_x(r, off);
            if (o > r) r = o;
        }
        return r;
    }
    template <class V>
    __device__ __forceinline__ void acc_finish(int lg, Acc<V> &a, V &wsum, V &rhomax, bool &err) const {
        V s = a.sum;
        for (int off = 1 << lg; off < 32; off <<= 1) s += shfl_x(s, off);
        V r = a.rho;
        for (int off = 1; off < 32; off <<= 1) {
            V o = shfl_x(r, off);
            if (o > r) r = o;
        }
        wsum = s;
        rhomax = r;
        err = __any_sync(0xffffffffu, a.err);
    }
};
#endif

/* Sequential emulation of the warp (test harness only). */
struct SeqTeam {
    RT_HD void sync() const {}
    RT_HD bool leader() const { return true; }
    template <class F> RT_HD void pfor(int n, F f) const {
        for (int i = 0; i < n; i++) f(i);
    }
    RT_HD bool any(bool b) const { return b; }
    template <class V> struct Acc {
        V sum, rho;
        bool err;
    };
    template <class V> RT_HD void acc_init(Acc<V> &a) const {
        a.sum = 0;
        a.rho = 0;
        a.err = false;
    }
    template <class V, class F> RT_HD void group_max_round(int lg, F f, Acc<V> &a) const {
        const int G = 1 << lg;
        for (int g0 = 0; g0 < 32; g0 += G) {
            V w[32], r[32];
            V m = 0;
            for (int s = g0; s < g0 + G; s++) {
                bool es = false;
                w[s - g0] = 0;
                r[s - g0] = 0;
                f(s, w[s - g0], r[s - g0], es);
                a.err = a.err || es;
                if (s == g0 || w[s - g0] > m) m = w[s - g0];
            }
            a.sum += m;
            for (int s = 0; s < G; s++)
                if (w[s] == m && r[s] > a.rho) a.rho = r[s];
        }
    }
    template <class V> RT_HD void acc_sum(int, const Acc<V> &a, V &wsum, bool &err) const {
        wsum = a.sum;
        err = a.err;
    }
    template <class V> RT_HD V acc_rho(const Acc<V> &a) const { return a.rho; }
    template <class V> RT_HD void acc_finish(int, Acc<V> &a, V &wsum, V &rhomax, bool &err) const {
        wsum = a.sum;
        rhomax = a.rho;
        err = a.err;
    }
};

/* ------------------------------------------------------------ views */

/* Build the CPU and (if any) memory chain views of task i at scale q.
 * Gap definitions: analysis.py:89 cpu_inter_arrival, analysis.py:57
 * mem_inter_arrival; GR lo from gpu.py:25 gpu_response_bounds. */
template <class V> RT_HD SegPtr seg_area(const SetCtx<V> &c, i64 off, SegPtr *) { return c.segs(off); }
template <class V> RT_HD Seg32 seg_area(const SetCtx<V> &c, i64 off, Seg32 *) {
    return Seg32{(const int32_t *)c.blob + off};
}

template <class V, class SA = SegPtr>
RT_NI void build_view(SetCtx<V> &c, int i, typename Num<V>::Qt q) {
    typedef Num<V> N;
    const TaskRec &t = c.TR()[i];
    const SA sg = seg_area(c, t.seg, (SA *)nullptr);
    const int m = t.m, p = t.p, g = m - 1;
    const SA cl_lo = sg, cl_hi = sg + m, ml_lo = sg + 2 * m, ml_hi = ml_lo + p;
    const SA gw_lo = ml_hi + p;
    typename Num<V>::Qt perlo = t.isgpu ? q / (2 * (typename Num<V>::Qt)t.g) : q;
    if (c.single_seg) {
        /* busy-waiting baseline (analysis.py:360): one execution segment of
         * length sum(CL up) + sum(ML up) + sum(GR up), no suspension */
        VOff o(c.MC);
        V *v = c.VC() + (size_t)i * c.L.SC;
        V gru = 0;
        if (t.isgpu) {
            typename Num<V>::Qt per = q / ((typename Num<V>::Qt)2 * (typename Num<V>::Qt)c.A * t.g);
            gru = (V)t.sInfl * (V)per + Num<V>::sc(t.sGL, q);
        }
        V e = N::sc(t.sClu + t.sMlu, q) + gru;
        v[o.e] = e;
        v[o.P] = 0;
        v[o.EP] = 0;
        v[o.EP + 1] = e;
        v[o.F1] = e + N::sc(t.T - t.D, q);
        V wrap = N::sc(t.T, q) - e;
        v[o.WN] = wrap < 0 ? (V)1 : (V)0;
        v[o.P + 1] = e + (wrap < 0 ? (V)0 : wrap);
        v[o.INV] = Num<V>::make_inv(v[o.P + 1]);
        return;
    }
    if (m == 0) return; /* no segments: no chain (walks need p >= 1) */
    /* CPU chain */
    {
        VOff o(c.MC);
        V *v = c.VC() + (size_t)i * c.L.SC;
        V P = 0, EP = 0;
        #pragma unroll 1
        for (int j = 0; j < m; j++) {
            V e = N::sc(cl_hi[j], q);
            v[o.e + j] = e;
            v[o.P + j] = P;
            v[o.EP + j] = EP;
            EP += e;
            if (j < m - 1) {
                V gap;
                if (c.mm == RTGPU_TWO_COPY)
                    gap = N::sc(ml_lo[2 * j] + ml_lo[2 * j + 1], q) + (V)gw_lo[j] * (V)perlo;
                else
                    gap = N::sc(ml_lo[j], q) + (V)gw_lo[j] * (V)perlo;
                P += e + gap;
            }
        }
        V elast = v[o.e + m - 1];
        v[o.EP + m] = EP;
        v[o.F1] = P + elast + N::sc(t.T - t.D, q);
        V wrap = N::sc(t.T - t.sClu - t.sMll, q) - (t.isgpu ? (V)t.sGWlo * (V)perlo : (V)0);
        v[o.WN] = (wrap < 0 ? (V)WN_WRAP : (V)0) + (t.D > t.T ? (V)WN_FIRST_OPEN : (V)0);
        v[o.P + m] = P + elast + (wrap < 0 ? (V)0 : wrap);
        v[o.INV] = Num<V>::make_inv(v[o.P + m]);
        (void)g;
    }
    /* memory chain */
    if (p > 0) {
        VOff o(c.MP);
        V *v = c.VM() + (size_t)i * c.L.SM;
        V P = 0, EP = 0;
        #pragma unroll 1
        for (int j = 0; j < p; j++) {
            V e = N::sc(ml_hi[j], q);
            v[o.e + j] = e;
            v[o.P + j] = P;
            v[o.EP + j] = EP;
            EP += e;
            if (j < p - 1) {
                V gap;
                if (c.mm == RTGPU_TWO_COPY)
                    gap = (j % 2 == 0) ? (V)gw_lo[j / 2] * (V)perlo : N::sc(cl_lo[(j + 1) / 2], q);
                else
                    gap = (V)gw_lo[j] * (V)perlo + N::sc(cl_lo[j + 1], q);
                P += e + gap;
            }
        }
        V elast = v[o.e + p - 1];
        v[o.EP + p] = EP;
        V first = N::sc(t.T - t.D + cl_lo[m - 1] + cl_lo[0], q);
        if (c.mm == RTGPU_ONE_COPY) first += (V)gw_lo[m - 2] * (V)perlo;
        v[o.F1] = P + elast + first;
        V wrap = N::sc(t.T - t.sMlu - t.innerCll, q) - (V)t.sGWlo * (V)perlo;
        v[o.WN] = (wrap < 0 ? (V)WN_WRAP : (V)0) + (first < 0 ? (V)WN_FIRST_CHECKED : (V)0);
        v[o.P + p] = P + elast + (wrap < 0 ? (V)0 : wrap);
        v[o.INV] = Num<V>::make_inv(v[o.P + p]);
    }
}

#ifdef __CUDA_ARCH__
/* build_view for the verdict fast path (compact blobs, RTGPU chains), with
 * the segments spread over the lanes: lane j holds segment j's length and
 * the gap after it, and the prefix sums P (segment + gap) and EP (segment)
 * are two warp scans -- instead of one lane walking the chain while 31
 * wait.  Integer-valued doubles below 2^52: the sums are exact in any
 * order, so the view is identical to build_view's. */
template <class V>
__device__ __forceinline__ void build_view_warp_body(SetCtx<V> &c, int i, i64 q, int lane) {
    typedef Num<V> N;
    const TaskRec &t = c.TR()[i];
    const Seg32 sg{(const int32_t *)c.blob + t.seg};
    const int m = t.m, p = t.p;
    const Seg32 cl_lo = sg, cl_hi = sg + m, ml_lo = sg + 2 * m, ml_hi = ml_lo + p;
    const Seg32 gw_lo = ml_hi + p;
    const i64 perlo = t.isgpu ? q / (2 * (i64)t.g) : q;
    const V vper = (V)perlo;
    const bool two = c.mm == RTGPU_TWO_COPY;
    /* CPU chain */
    {
        VOff o(c.MC);
        V *v = c.VC() + (size_t)i * c.L.SC;
        V e = 0, gap = 0;
        if (lane < m) {
            e = N::sc(cl_hi[lane], q);
            if (lane < m - 1)
                gap = (two ? N::sc(ml_lo[2 * lane] + ml_lo[2 * lane + 1], q) : N::sc(ml_lo[lane], q)) +
                      (V)gw_lo[lane] * vper;
        }
        V s1 = e + gap, s2 = e;
        #pragma unroll 1
        for (int off = 1; off < m; off <<= 1) {
            const V a1 = __shfl_up_sync(0xffffffffu, s1, off), a2 = __shfl_up_sync(0xffffffffu, s2, off);
            if (lane >= off) {
                s1 += a1;
                s2 += a2;
            }
        }
        if (lane < m) {
            const V P = s1 - e - gap, EP = s2 - e;
            v[o.e + lane] = e;
            v[o.P + lane] = P;
            v[o.EP + lane] = EP;
            if (lane == m - 1) {
                v[o.EP + m] = s2;
                v[o.F1] = P + e + N::sc(t.T - t.D, q);
                const V wrap = N::sc(t.T - t.sClu - t.sMll, q) - (t.isgpu ? (V)t.sGWlo * vper : (V)0);
                v[o.WN] = wrap < 0 ? (V)1 : (V)0;
                v[o.P + m] = P + e + (wrap < 0 ? (V)0 : wrap);
                v[o.INV] = N::make_inv(v[o.P + m]);
            }
        }
    }
    /* memory chain */
    if (p > 0) {
        VOff o(c.MP);
        V *v = c.VM() + (size_t)i * c.L.SM;
        V e = 0, gap = 0;
        if (lane < p) {
            e = N::sc(ml_hi[lane], q);
            if (lane < p - 1) {
                if (two)
                    gap = (lane % 2 == 0) ? (V)gw_lo[lane / 2] * vper : N::sc(cl_lo[(lane + 1) / 2], q);
                else
                    gap = (V)gw_lo[lane] * vper + N::sc(cl_lo[lane + 1], q);
            }
        }
        V s1 = e + gap, s2 = e;
        #pragma unroll 1
        for (int off = 1; off < p; off <<= 1) {
            const V a1 = __shfl_up_sync(0xffffffffu, s1, off), a2 = __shfl_up_sync(0xffffffffu, s2, off);
            if (lane >= off) {
                s1 += a1;
                s2 += a2;
            }
        }
        if (lane < p) {
            const V P = s1 - e - gap, EP = s2 - e;
            v[o.e + lane] = e;
            v[o.P + lane] = P;
            v[o.EP + lane] = EP;
            if (lane == p - 1) {
                v[o.EP + p] = s2;
                V first = N::sc(t.T - t.D + cl_lo[m - 1] + cl_lo[0], q);
                if (!two) first += (V)gw_lo[m - 2] * vper;
                v[o.F1] = P + e + first;
                const V wrap = N::sc(t.T - t.sMlu - t.innerCll, q) - (V)t.sGWlo * vper;
                v[o.WN] = wrap < 0 ? (V)1 : (V)0;
                v[o.P + p] = P + e + (wrap < 0 ? (V)0 : wrap);
                v[o.INV] = N::make_inv(v[o.P + p]);
            }
        }
    }
    __syncwarp();
}

/* The out-of-line entry of build_view_warp_body: the set context is rebuilt
 * from scalars, so the caller's SetCtx never has its address taken and stays
 * in registers (a SetCtx passed by reference to an out-of-line routine lives
 * in the stack frame, whose dirty lines were the fast kernel's DRAM write
 * traffic). */
template <class V>
__device__ __noinline__ void build_view_warp_s(const i64 *blob, int o_tr, int o_vc, int o_vm, int SC, int SM,
                                              int MC, int MP, int mm, int i, i64 q, int lane) {
    SetCtx<V> c;
    c.blob = blob;
    c.hbase = nullptr;
    c.o_tr = o_tr;
    c.o_vc = o_vc;
    c.o_vm = o_vm;
    c.L.SC = SC;
    c.L.SM = SM;
    c.MC = MC;
    c.MP = MP;
    c.mm = mm;
    c.segw = 1;
    build_view_warp_body(c, i, q, lane);
}
#endif

/* Views of tasks [0, k) at scale q (reused when already current). */
template <class V, class TM>
RT_HD void ensure_views(const TM &tm, SetCtx<V> &c, int k, typename Num<V>::Qt q) {
    if (c.vq == q && c.vn >= k) return;
    int from = (c.vq == q) ? c.vn : 0;
    tm.pfor(k - from, [&](int x) { build_view(c, from + x, q); });
    c.vq = q;
    c.vn = k;
}

/* ------------------------------------------------------------ chain walk */

/* W_i^h(H) of suspension.py:77 chain_workload over the view, in O(p).
 * rho = remaining slope-1 length (the walk ends inside a segment), err =
 * an InfeasibleGapError the reference would raise (walk reaches the first
 * negative wrap-around gap). */
template <class V>
RT_HD V walk(const V *v, int PM, int half, int p, int h, V H, V &rho, bool &err) {
    VOff o(PM);
    rho = 0;
    if (H <= 0) return 0;
    const V *e = v + o.e, *P = v + o.P, *EP = v + o.EP;
    V base = P[h];
    V lim = H + base;
    V F1 = v[o.F1];
    const int fl = (int)v[o.WN];
    bool in_first = F1 > lim;
    if (fl & (WN_FIRST_CHECKED | WN_FIRST_OPEN)) {
        /* a negative gap after the first job (D > T): the walk evaluates it
         * once it reaches the job's last segment -- the memory chain's is
         * checked (InfeasibleGapError), the CPU chain's used as is, so the
         * walk leaves the first job only if it got there */
        const bool reach_last = P[p - 1] <= lim;
        if ((fl & WN_FIRST_CHECKED) && reach_last) {
            err = true;
            return 0;
        }
        if (!reach_last) in_first = true;
    }
    if (in_first) {
        /* stops inside the first (partial) job: the last x in [h, p-1] with
         * P[x] <= lim (P is non-decreasing; P[h] = base <= lim) */
        int x = h;
#pragma unroll 5
        for (int st = half; st > 0; st >>= 1) {
            int y = x + st;
            if (y <= p - 1 && P[y] <= lim) x = y;
        }
        V tail = lim - P[x];
        V ex = e[x];
        if (ex > tail) {
            rho = ex - tail;
            return EP[x] - EP[h] + tail;
        }
        return EP[x] - EP[h] + ex;
    }
    V w = EP[p] - EP[h];
    V H2 = lim - F1; /* H minus the first job's span */
    int x = 0;
    V Hs;
    if (fl & WN_WRAP) {
        /* negative wrap: the walk raises iff it reaches index 2p-1 */
        if (P[p - 1] <= H2) {
            err = true;
            return 0;
        }
#pragma unroll 5
        for (int st = half; st > 0; st >>= 1) {
            int y = x + st;
            if (y <= p - 2 && P[y] <= H2) x = y;
        }
        Hs = H2;
    } else {
        V C = P[p];
        if (C <= 0) {
            /* all-zero period: the reference loops forever */
            err = true;
            return 0;
        }
        V k = Num<V>::divmod_inv(H2, C, v[o.INV], Hs);
        w += k * EP[p];
#pragma unroll 5
        for (int st = half; st > 0; st >>= 1) {
            int y = x + st;
            if (y <= p - 1 && P[y] <= Hs) x = y;
        }
    }
    V tail = Hs - P[x];
    if (e[x] > tail) {
        rho = e[x] - tail;
        return w + EP[x] + tail;
    }
    return w + EP[x] + e[x];
}

/* Sum over hp(k) of max over start segments of W (analysis.py:131
 * _max_workload summed as in mem_response / cpu_response). */
#ifdef RT_COUNTERS
extern long long g_cnt_interf[2], g_cnt_lfp[2], g_cnt_eval, g_cnt_views, g_cnt_rounds;
extern long long g_cnt_flfp[8], g_cnt_fit[8], g_cnt_frounds, g_cnt_passes;
#define RT_COUNT(x) (x)++
#else
#define RT_COUNT(x)
#endif

/* What the interference loop reads, copied out of the set context so the
 * hot loop keeps it in registers (no aliasing with shared-memory writes). */
template <class V> struct IView {
    const TaskRec *tr;
    const V *views;
    int k, kind, lg, PM, half, stride, p1;
    i64 prio_k;
};

template <class V>
RT_HD IView<V> make_iview(const SetCtx<V> &c, int k, int kind) {
    IView<V> v;
    v.tr = c.TR();
    v.k = k;
    v.kind = kind;
    v.lg = kind == K_CPU ? c.lgC : c.lgM;
    v.PM = kind == K_CPU ? c.MC : c.MP;
    v.half = kind == K_CPU ? c.halfC : c.halfM;
    v.stride = kind == K_CPU ? c.L.SC : c.L.SM;
    v.views = kind == K_CPU ? c.VC() : c.VM();
    v.p1 = c.single_seg;
    v.prio_k = c.TR()[k].prio;
    return v;
}

template <class V, class TM>
RT_HD V interference(const TM &tm, const IView<V> &iv, V H, V &rho, bool &err) {
    RT_COUNT(g_cnt_interf[iv.kind]);
    rho = 0;
    err = false;
    if (H <= 0 || iv.k == 0) return 0;
    typename TM::template Acc<V> acc;
    tm.acc_init(acc);
    const int lg = iv.lg;
    for (int i0 = 0; i0 < iv.k; i0 += (32 >> lg)) {
        RT_COUNT(g_cnt_rounds);
        tm.group_max_round(lg, [&](int slot, V &w, V &r, bool &es) {
            int i = i0 + (slot >> lg), h = slot & ((1 << lg) - 1);
            if (i < iv.k) {
                const TaskRec &ti = iv.tr[i];
                int p = iv.kind == K_CPU ? (iv.p1 ? 1 : ti.m) : ti.p;
                if (h < p && ti.prio < iv.prio_k)
                    w = walk(iv.views + (size_t)i * iv.stride, iv.PM, iv.half, p, h, H, r, es);
            }
        }, acc);
    }
    V total;
    tm.acc_finish(lg, acc, total, rho, err);
    return total;
}

/* Least fixed point of r = base + I(r) searched from `start` (base <= start
 * <= lfp).  Returns -1 for the reference's None (suspension.py:123: iterate
 * beyond the bound, or an InfeasibleGapError inside the interference). */
template <class V, class TM>
RT_NI V lfp(const TM &tm, SetCtx<V> &c, int k, int kind, V base, V start, V bound) {
    RT_COUNT(g_cnt_lfp[kind]);
    /* a warm start is a lower bound of the lfp: beyond the bound, the
     * reference's iteration from `base` would pass it too (None) */
    if (base > bound || start > bound) return (V)-1;
    const IView<V> iv = make_iview(c, k, kind);
    V r = start;
    for (int it = 0; it < ITER_CAP; it++) {
        V rho;
        bool err;
        V I = interference(tm, iv, r, rho, err);
        if (err) return (V)-1;
        V nxt = base + I;
        if (nxt <= r) return r; /* nxt == r in exact arithmetic */
        nxt += rho; /* slope-1 jump: nxt + rho <= lfp, so exceeding the
                     * bound here means lfp > bound (reference: None) */
        if (nxt > bound) return (V)-1;
        r = nxt;
    }
    c.stuck = 1;
    return (V)-1;
}

/* Fixed points for several bases sharing one interference function, with
 * warm starts: lfp(b') >= lfp(b) + (b' - b) for b' >= b, and None(b) implies
 * None(b') (both monotone).  Results in out[] (-1 = None). */
template <class V, class TM>
RT_NI void lfp_many(const TM &tm, SetCtx<V> &c, int k, int kind, const V *bases, V *out, int cnt,
                    V bound, bool stop_on_none, bool &any_none) {
    /* Ascending order of the bases via lane-parallel ranks (ties by index).
     * lfp(b) - b is non-decreasing in b, so the best warm start for a base
     * is its predecessor's fixed point plus the base difference, and a None
     * predecessor makes every later base None. */
    any_none = false;
    int *ord = (int *)(c.SCR() + c.L.scr_n) - 32;
    tm.pfor(cnt, [&](int j) {
        int r = 0;
        for (int q = 0; q < cnt; q++) r += (bases[q] < bases[j] || (bases[q] == bases[j] && q < j)) ? 1 : 0;
        ord[r] = j;
    });
    V prev_b = 0, prev_r = 0;
    bool prev_none = false;
    for (int step = 0; step < cnt; step++) {
        const int j = ord[step];
        const V b = bases[j];
        V r;
        if (prev_none) {
            r = (V)-1;
        } else {
            V start = step ? tmax(b, prev_r + (b - prev_b)) : b;
            r = lfp(tm, c, k, kind, b, start, bound);
        }
        tm.sync();
        if (tm.leader()) out[j] = r;
        tm.sync();
        if (r < 0) {
            any_none = true;
            prev_none = true;
            if (stop_on_none) {
                for (int q = step + 1; q < cnt; q++)
                    if (tm.leader()) out[ord[q]] = (V)-1;
                tm.sync();
                return;
            }
        }
        prev_b = b;
        prev_r = r;
    }
}

/* ------------------------------------------------------------ task evaluation */

template <class V> struct TaskEval {
    /* results at scale q (numerators), -1 = None */
    typename Num<V>::Qt q;
    V e2e, r1, r2;
    bool pass;
};

/* Scale for evaluating task k at count g given the prefix lcm. */
template <class V>
RT_HD typename Num<V>::Qt task_scale(SetCtx<V> &c, int k, int g, typename Num<V>::Qt lcm_pre) {
    typedef typename Num<V>::Qt Qt;
    if (c.fixed_q) return c.fixed_q; /* multiple of every 2*A*g: views never rescale */
    Qt q = lcm_lim<Qt>(lcm_pre, (Qt)1, c.qlim);
    q = (q == 0 || q > c.qlim / 2) ? 0 : q * 2;
    if (q != 0 && c.TR()[k].isgpu) q = lcm_lim<Qt>(q, (Qt)2 * (Qt)c.A * (Qt)g, c.qlim);
    if (q == 0) c.esc = 1;
    return q;
}

/* GR^j up (gpu.py:25) summed over task k's kernels, at scale q:
 * sum_j[(gw_hi*an - gl*A)/(2*A*g) + gl] = sInfl*(q/(2Ag)) + sGL*q. */
template <class V>
RT_HD V sum_grup(const SetCtx<V> &c, int k, int g, typename Num<V>::Qt q) {
    const TaskRec &t = c.TR()[k];
    if (!t.isgpu) return 0;
    typename Num<V>::Qt per = q / ((typename Num<V>::Qt)2 * (typename Num<V>::Qt)c.A * g);
    return (V)t.sInfl * (V)per + Num<V>::sc(t.sGL, q);
}

/*
 * Full evaluation of task k at count g (prefix fixed), exactly as
 * analysis.py:284-296 (mem_response for every memory segment, cpu_response
 * for every CPU segment, end_to_end).  want_all: compute every value (report
 * pass); otherwise stop as soon as the verdict is known.  mr_out/cr_out (may
 * be null) receive per-segment numerators at scale q.
 */
template <class V, class TM>
RT_NI void eval_task(const TM &tm, SetCtx<V> &c, int k, int g, typename Num<V>::Qt lcm_pre,
                     bool want_all, TaskEval<V> &res, V *mr_out, V *cr_out) {
    typedef Num<V> N;
    const TaskRec &t = c.TR()[k];
    typename N::Qt q = task_scale(c, k, g, lcm_pre);
    res.q = q;
    res.pass = false;
    res.e2e = res.r1 = res.r2 = (V)-1;
    if (c.esc) return;
    c.evals++;
    RT_COUNT(g_cnt_eval);
    ensure_views(tm, c, k, q);
    const V D = N::sc(t.D, q);
    V *bases = c.SCR();
    V *outs = c.SCR() + (c.MP + c.MC + 2);
    const SegPtr sg = c.segs(t.seg);
    const SegPtr cl_hi = sg + t.m, ml_hi = sg + 2 * t.m + t.p;
    /* memory segments: analysis.py:156 (blocking = longest lp copy) */
    V sum_mr = 0;
    bool mr_none = false;
    const V grup = sum_grup(c, k, g, q);
    if (t.p > 0 && !want_all) {
        /* Verdict shortcut, exact: lfp(b') >= lfp(b) + (b' - b) gives
         * MR_j <= lfp(b_max) - (b_max - b_j), and lfp(b_max) is MR of the
         * longest copy.  One fixed point decides "some MR is None"; if R2
         * passes with the resulting upper bound on sum MR it passes exactly
         * (the least fixed point is monotone in the base). */
        i64 bmax_t = 0, bsum_t = 0;
        #pragma unroll 1
        for (int j = 0; j < t.p; j++) {
            bmax_t = tmax(bmax_t, ml_hi[j] + t.B);
            bsum_t += ml_hi[j] + t.B;
        }
        const V bmax = N::sc(bmax_t, q);
        const V rmax = lfp(tm, c, k, K_MEM, bmax, bmax, D);
        if (rmax < 0) return; /* the longest copy's MR is None: task fails */
        const V mr_ub = (V)t.p * (rmax - bmax) + N::sc(bsum_t, q);
        const V b2 = grup + mr_ub + N::sc(t.sClu, q);
        const V r2ub = lfp(tm, c, k, K_CPU, b2, b2, D);
        if (r2ub >= 0) {
            res.pass = true;
            res.e2e = r2ub; /* an upper bound; verdict mode reports no bounds */
            return;
        }
    }
    if (t.p > 0) {
        tm.pfor(t.p, [&](int j) { bases[j] = N::sc(ml_hi[j] + t.B, q); });
        lfp_many(tm, c, k, K_MEM, bases, outs, t.p, D, !want_all, mr_none);
        #pragma unroll 1
        for (int j = 0; j < t.p; j++)
            if (outs[j] >= 0) sum_mr += outs[j];
        if (mr_out) tm.pfor(t.p, [&](int j) { mr_out[j] = outs[j]; });
        tm.sync();
        if (mr_none && !want_all) return;
    }
    /* end_to_end R2 (analysis.py:214) first: it needs no per-segment CPU bounds */
    V r2 = (V)-1;
    if (!mr_none) r2 = lfp(tm, c, k, K_CPU, grup + sum_mr + N::sc(t.sClu, q),
                           grup + sum_mr + N::sc(t.sClu, q), D);
    res.r2 = r2;
    if (r2 >= 0 && !want_all) {
        res.pass = true;
        res.e2e = r2;
        return;
    }
    /* cpu_response for every CPU segment (analysis.py:175), then R1 */
    tm.pfor(t.m, [&](int j) { bases[j] = N::sc(cl_hi[j], q); });
    bool cr_none;
    lfp_many(tm, c, k, K_CPU, bases, outs, t.m, D, !want_all, cr_none);
    V sum_cr = 0;
    #pragma unroll 1
    for (int j = 0; j < t.m; j++)
        if (outs[j] >= 0) sum_cr += outs[j];
    if (cr_out) tm.pfor(t.m, [&](int j) { cr_out[j] = outs[j]; });
    tm.sync();
    V r1 = (V)-1;
    if (!mr_none && !cr_none) {
        V cand = grup + sum_mr + sum_cr;
        if (cand <= D) r1 = cand;
    }
    res.r1 = r1;
    if (mr_none) return;
    if (r1 < 0) res.e2e = r2;
    else if (r2 < 0) res.e2e = r1;
    else res.e2e = tmin(r1, r2);
    res.pass = res.e2e >= 0;
}

/* ------------------------------------------------------------ set loading */

/* Per-task sums and flags (lane-parallel).  Computes the isolated-bound
 * minimum count of analysis.py:239 _min_feasible_gn in closed form:
 * sum_j[(gw_hi*a - gl*A)/(2*A*gn) + gl] + sum ml_hi + sum cl_hi <= D. */
template <class V>
RT_NI void load_task(SetCtx<V> &c, int i, i128 *vb_out) {
    const RecP r = rec_at(c.blob, i);
    TaskRec &t = c.TR()[i];
    t.m = (int)r[0];
    t.p = (int)r[1];
    t.D = r[2];
    t.T = r[3];
    t.prio = r[4];
    t.seg = r[5];
    t.idx = i;
    t.flags = 0;
    t.g = 0;
    t.gmin = 0;
    t.isgpu = t.m > 1;
    const int m = t.m, p = t.p;
    int want_p = m < 2 ? 0 : (c.mm == RTGPU_TWO_COPY ? 2 * m - 2 : m - 1);
    /* m == 0 (no segments) and D > T are analysed as the reference does
     * without validate_taskset: a task with no segments has bound 0 and no
     * workload; D > T makes the first job's CPU gap T - D negative (used as
     * is, analysis.py:100) and its memory deadline-side gap checked
     * (analysis.py:75: InfeasibleGapError when a walk reaches it), so such
     * sets take the exact depth-first search (TF_IRREG) */
    if (m < 0 || m > c.MC || p != want_p || p > c.MP || t.T <= 0 || t.D <= 0) {
        t.flags |= TF_UNSUP;
        *vb_out = 0;
        return;
    }
    const SegPtr sg = c.segs(t.seg);
    const SegPtr cl_lo = sg, cl_hi = sg + m, ml_lo = sg + 2 * m, ml_hi = ml_lo + p;
    const int g = m - 1;
    const SegPtr gw_lo = ml_hi + p, gw_hi = gw_lo + g, gl = gw_hi + g, an = gl + g;
    i128 tot = 0;
    t.sClu = t.sCll = t.sMlu = t.sMll = t.sGWlo = t.sInfl = t.sGL = t.innerCll = t.maxMlu = 0;
    bool neg = false;
    #pragma unroll 1
    for (int j = 0; j < m; j++) {
        t.sClu += cl_hi[j];
        t.sCll += cl_lo[j];
        neg = neg || cl_hi[j] < 0 || cl_lo[j] < 0;
        if (j >= 1 && j <= m - 2) t.innerCll += cl_lo[j];
    }
    #pragma unroll 1
    for (int j = 0; j < p; j++) {
        t.sMlu += ml_hi[j];
        t.sMll += ml_lo[j];
        t.maxMlu = tmax(t.maxMlu, ml_hi[j]);
        neg = neg || ml_hi[j] < 0 || ml_lo[j] < 0;
    }
    i128 infl_hi = 0;
    #pragma unroll 1
    for (int j = 0; j < g; j++) {
        neg = neg || gw_lo[j] < 0 || gw_hi[j] < 0 || gl[j] < 0 || an[j] < 0;
        i128 w = (i128)gw_hi[j] * an[j], o = (i128)gl[j] * c.A;
        if (o > w) t.flags |= TF_INV;
        t.sInfl += (i64)(w - o);
        t.sGL += gl[j];
        t.sGWlo += gw_lo[j];
        infl_hi += w;
    }
    if (neg) {
        t.flags |= TF_UNSUP;
        *vb_out = 0;
        return;
    }
    tot = (i128)t.sClu + t.sCll + t.sMlu + t.sMll + t.sGWlo + t.sGL + infl_hi / c.A + 1;
    *vb_out = (i128)t.D + t.T + tot;
    if (t.isgpu) {
        /* infl/(2*A*gn) + fixed <= D  <=>  infl <= 2*A*gn*(D - fixed) */
        i128 X = (i128)t.D - t.sGL - t.sMlu - t.sClu;
        i128 gm = 0;
        if (c.GN >= 1) {
            if (X > 0) {
                i128 den = 2 * (i128)c.A * X;
                gm = ((i128)t.sInfl + den - 1) / den;
                if (gm < 1) gm = 1;
                if (gm > c.GN) gm = 0;
            } else if (X == 0 && t.sInfl == 0) {
                gm = 1;
            }
        }
        if (gm == 0) t.flags |= TF_ISOFAIL;
        t.gmin = (int)gm;
        if (gm > 0) {
            /* regular iff no wrap-around gap can be negative for any count >= gmin */
            i128 twog = 2 * gm;
            if (((i128)t.T - t.sClu - t.sMll) * twog - t.sGWlo < 0) t.flags |= TF_IRREG;
            if (((i128)t.T - t.sMlu - t.innerCll) * twog - t.sGWlo < 0) t.flags |= TF_IRREG;
        }
    } else {
        if (t.sClu > t.D) t.flags |= TF_ISOFAIL;
        if (t.T - t.sClu < 0) t.flags |= TF_IRREG;
    }
    if (t.D > t.T) t.flags |= TF_IRREG;
}

/* ------------------------------------------------------------ output helpers */

template <class V> struct OutPtrs {
    int32_t *vsm;   /* [n] */
    i64 *e2e, *den; /* [n] */
    i64 *detail;    /* set-blob shaped, or null */
};

/* Report pass over a fixed allocation (tr[].g) with per-task scales,
 * exactly analysis.py:280-298 evaluate(): every memory / CPU segment bound,
 * the GPU bounds of the allocation and the end-to-end bound; stops after the
 * first failing task when stop_at_fail (the reference's per_task then holds
 * the tasks up to it).  Values are written as numerators over den[k]. */
template <class V, class TM>
RT_NI bool report_pass(const TM &tm, SetCtx<V> &c, const OutPtrs<V> &o, bool stop_at_fail) {
    typedef typename Num<V>::Qt Qt;
    Qt lcm_pre = 1;
    V *mr = c.SCR() + 2 * (c.MP + c.MC + 2);
    V *cr = mr + c.MP;
    V *grl = cr + c.MC;
    V *grh = grl + c.MC;
    bool failed = false;
    int k = 0;
    #pragma unroll 1
    for (; k < c.n; k++) {
        const TaskRec &t = c.TR()[k];
        TaskEval<V> res;
        eval_task(tm, c, k, t.g, lcm_pre, true, res, mr, cr);
        if (c.esc || c.stuck) return false;
        const Qt q = res.q;
        const SegPtr sg = c.segs(t.seg);
        const int m = t.m, p = t.p, g = m - 1;
        const SegPtr gw_lo = sg + 2 * m + 2 * p, gw_hi = gw_lo + g, gl = gw_hi + g, an = gl + g;
        if (t.isgpu) {
            const Qt perlo = q / (2 * (Qt)t.g);
            const Qt perhi = q / (2 * (Qt)c.A * (Qt)t.g);
            tm.pfor(g, [&](int j) {
                grl[j] = (V)gw_lo[j] * (V)perlo;
                V infl = (V)((i128)gw_hi[j] * an[j] - (i128)gl[j] * c.A);
                grh[j] = infl * (V)perhi + Num<V>::sc(gl[j], q);
            });
        }
        /* reduce by a common gcd so numerators and den fit int64 (only the
         * 128-bit arithmetic can exceed it) */
        i128 red = 1;
        if (sizeof(V) > 8) {
            i128 gg = (i128)q;
            if (res.e2e >= 0) gg = gcdq<i128>(gg, Num<V>::wide(res.e2e));
            #pragma unroll 1
            for (int j = 0; j < p; j++)
                if (mr[j] >= 0) gg = gcdq<i128>(gg, Num<V>::wide(mr[j]));
            #pragma unroll 1
            for (int j = 0; j < m; j++)
                if (cr[j] >= 0) gg = gcdq<i128>(gg, Num<V>::wide(cr[j]));
            #pragma unroll 1
            for (int j = 0; j < g; j++) {
                gg = gcdq<i128>(gg, Num<V>::wide(grl[j]));
                gg = gcdq<i128>(gg, Num<V>::wide(grh[j]));
            }
            red = gg == 0 ? 1 : gg;
            const i128 lim = (i128)INT64_MAX;
            bool over = (i128)q / red > lim || (res.e2e >= 0 && Num<V>::wide(res.e2e) / red > lim);
            #pragma unroll 1
            for (int j = 0; j < g; j++) over = over || Num<V>::wide(grh[j]) / red > lim;
            #pragma unroll 1
            for (int j = 0; j < p; j++) over = over || (mr[j] >= 0 && Num<V>::wide(mr[j]) / red > lim);
            #pragma unroll 1
            for (int j = 0; j < m; j++) over = over || (cr[j] >= 0 && Num<V>::wide(cr[j]) / red > lim);
            if (over) {
                c.esc = 1; /* not representable even reduced */
                return false;
            }
        }
        auto num = [&](V v) -> i64 { return v < 0 ? (i64)RTGPU_NONE : (i64)(Num<V>::wide(v) / red); };
        tm.sync();
        if (tm.leader()) {
            o.e2e[k] = num(res.e2e);
            o.den[k] = (i64)((i128)q / red);
        }
        if (o.detail) {
            i64 *d = o.detail + t.seg;
            tm.pfor(2 * m + 2 * p + 4 * g, [&](int w) {
                i64 v = RTGPU_ABSENT;
                if (w < m) v = num(cr[w]);
                else if (w >= 2 * m && w < 2 * m + p) v = num(mr[w - 2 * m]);
                else if (w >= 2 * m + 2 * p && w < 2 * m + 2 * p + g) v = num(grl[w - 2 * m - 2 * p]);
                else if (w >= 2 * m + 2 * p + g && w < 2 * m + 2 * p + 2 * g) v = num(grh[w - 2 * m - 2 * p - g]);
                d[w] = v;
            });
        }
        if (t.isgpu) {
            lcm_pre = lcm_lim<Qt>(lcm_pre, (Qt)t.g, c.qlim);
            if (lcm_pre == 0) {
                c.esc = 1;
                return false;
            }
        }
        if (!res.pass) {
            failed = true;
            if (stop_at_fail) {
                k++;
                break;
            }
        }
    }
    #pragma unroll 1
    for (; k < c.n; k++) {
        if (tm.leader()) {
            o.e2e[k] = RTGPU_ABSENT;
            o.den[k] = 1;
        }
        if (o.detail) {
            const TaskRec &t = c.TR()[k];
            i64 *d = o.detail + t.seg;
            tm.pfor(2 * t.m + 2 * t.p + 4 * (t.m - 1), [&](int w) { d[w] = RTGPU_ABSENT; });
        }
    }
    tm.sync();
    return !failed;
}

/* Set the count of task k (leader write) and drop views that used the old one. */
template <class V, class TM>
RT_HD void set_g(const TM &tm, SetCtx<V> &c, int k, int g) {
    tm.sync();
    if (tm.leader()) c.TR()[k].g = g;
    tm.sync();
    if (c.vn > k) c.vn = k;
}

/* smallest passing count in [lo, hi] for task k (own-count monotone), or 0 */
template <class V, class TM>
RT_NI int find_g(const TM &tm, SetCtx<V> &c, int k, int lo, int hi, typename Num<V>::Qt lcm_pre) {
    TaskEval<V> r;
    eval_task(tm, c, k, lo, lcm_pre, false, r, (V *)nullptr, (V *)nullptr);
    if (c.esc) return 0;
    if (r.pass) return lo;
    if (lo >= hi) return 0;
    eval_task(tm, c, k, hi, lcm_pre, false, r, (V *)nullptr, (V *)nullptr);
    if (c.esc || !r.pass) return 0;
    #pragma unroll 1
    while (hi - lo > 1) {
        int mid = lo + (hi - lo) / 2;
        eval_task(tm, c, k, mid, lcm_pre, false, r, (V *)nullptr, (V *)nullptr);
        if (c.esc) return 0;
        if (r.pass) hi = mid;
        else lo = mid;
    }
    return hi;
}

/* Greedy descent (regular sets): equals the lexicographically first
 * schedulable allocation of the reference grid search. */
template <class V, class TM>
RT_NI int search_greedy(const TM &tm, SetCtx<V> &c) {
    typedef typename Num<V>::Qt Qt;
    Qt lcm_pre = 1;
    i64 used = 0, rest_min = 0;
    #pragma unroll 1
    for (int k = 0; k < c.n; k++)
        if (c.TR()[k].isgpu) rest_min += c.TR()[k].gmin;
    #pragma unroll 1
    for (int k = 0; k < c.n; k++) {
        TaskRec &t = c.TR()[k];
        if (!t.isgpu) {
            TaskEval<V> r;
            eval_task(tm, c, k, 0, lcm_pre, false, r, (V *)nullptr, (V *)nullptr);
            if (c.esc) return ST_ESCALATE;
            if (c.stuck) return RTGPU_UNDECIDED;
            if (!r.pass) return RTGPU_UNSCHEDULABLE;
            continue;
        }
        rest_min -= t.gmin;
        i64 gmax = c.GN - used - rest_min;
        if (gmax < t.gmin) return RTGPU_UNSCHEDULABLE;
        int g = find_g(tm, c, k, t.gmin, (int)gmax, lcm_pre);
        if (c.esc) return ST_ESCALATE;
        if (c.stuck) return RTGPU_UNDECIDED;
        if (g == 0) return RTGPU_UNSCHEDULABLE;
        set_g(tm, c, k, g);
        used += g;
        lcm_pre = lcm_lim<Qt>(lcm_pre, (Qt)g, c.qlim);
        if (lcm_pre == 0) return ST_ESCALATE;
    }
    return RTGPU_SCHEDULABLE;
}

/* Exact depth-first search with prefix pruning (irregular sets). */
template <class V, class TM>
RT_NI int search_dfs(const TM &tm, SetCtx<V> &c) {
    typedef typename Num<V>::Qt Qt;
    int d = 0;
    #pragma unroll 1
    for (;;) {
        if (d == c.n) return RTGPU_SCHEDULABLE;
        if (c.budget > 0 && c.evals >= c.budget) return RTGPU_UNDECIDED;
        TaskRec &t = c.TR()[d];
        Qt lcm_pre = 1;
        i64 used = 0, after = 0;
        #pragma unroll 1
        for (int i = 0; i < d; i++)
            if (c.TR()[i].isgpu) {
                lcm_pre = lcm_lim<Qt>(lcm_pre, (Qt)c.TR()[i].g, c.qlim);
                if (lcm_pre == 0) return ST_ESCALATE;
                used += c.TR()[i].g;
            }
        #pragma unroll 1
        for (int i = d + 1; i < c.n; i++)
            if (c.TR()[i].isgpu) after += c.TR()[i].gmin;
        bool ok;
        if (!t.isgpu) {
            TaskEval<V> r;
            eval_task(tm, c, d, 0, lcm_pre, false, r, (V *)nullptr, (V *)nullptr);
            ok = r.pass;
        } else {
            i64 gmax = c.GN - used - after;
            int g = gmax >= t.gmin ? find_g(tm, c, d, t.gmin, (int)gmax, lcm_pre) : 0;
            ok = g != 0;
            if (ok) set_g(tm, c, d, g);
        }
        if (c.esc) return ST_ESCALATE;
        if (c.stuck) return RTGPU_UNDECIDED;
        if (ok) {
            d++;
            continue;
        }
        /* backtrack: the deepest earlier GPU task with room for one more SM
         * (it still passes: own-count monotone) */
        #pragma unroll 1
        for (;;) {
            d--;
            if (d < 0) return RTGPU_UNSCHEDULABLE;
            TaskRec &b = c.TR()[d];
            if (!b.isgpu) continue;
            i64 u = 0, a = 0;
            #pragma unroll 1
            for (int i = 0; i < d; i++)
                if (c.TR()[i].isgpu) u += c.TR()[i].g;
            #pragma unroll 1
            for (int i = d + 1; i < c.n; i++)
                if (c.TR()[i].isgpu) a += c.TR()[i].gmin;
            if (b.g < c.GN - u - a) {
                set_g(tm, c, d, b.g + 1);
                d++;
                break;
            }
        }
    }
}

/* ------------------------------------------------------------ baselines */

template <class V> RT_HD i64 out_num(V v) { return v < 0 ? (i64)RTGPU_NONE : (i64)Num<V>::wide(v); }

/* Baselines of analysis.py:319 (self-suspension) and :355 (busy-waiting),
 * evaluated on a full allocation tr[].g at one scale q = 2*A*lcm(g).
 * Each task becomes a SuspTask (suspension.py:23); task_response
 * (suspension.py:155) uses the CPU chain views: self-suspension gaps are the
 * memory+kernel spans' lower bounds -- the same gaps as the RTGPU CPU chain
 * -- and busy-waiting collapses a task to one segment. */

/* sum over kernels of GR up at scale q (0 for pure-CPU tasks) */
template <class V> RT_HD V grup_at(const SetCtx<V> &c, const TaskRec &t, int gcount, typename Num<V>::Qt q) {
    if (!t.isgpu) return 0;
    typename Num<V>::Qt per = q / ((typename Num<V>::Qt)2 * (typename Num<V>::Qt)c.A * gcount);
    return (V)t.sInfl * (V)per + Num<V>::sc(t.sGL, q);
}

/* Largest suspension-interval upper bound of task t at scale q (the
 * self-suspension blocking a higher-priority task can suffer from it). */
template <class V> RT_HD V max_susp_hi(const SetCtx<V> &c, const TaskRec &t, int gcount, typename Num<V>::Qt q) {
    if (!t.isgpu) return 0;
    const SegPtr sg = c.segs(t.seg);
    const int m = t.m, p = t.p, g = m - 1;
    const SegPtr ml_hi = sg + 2 * m + p, gw_hi = sg + 2 * m + 2 * p + g, gl = gw_hi + g, an = gl + g;
    typename Num<V>::Qt per = q / ((typename Num<V>::Qt)2 * (typename Num<V>::Qt)c.A * gcount);
    V best = 0;
    #pragma unroll 1
    for (int j = 0; j < g; j++) {
        V gr = (V)((i128)gw_hi[j] * an[j] - (i128)gl[j] * c.A) * (V)per + Num<V>::sc(gl[j], q);
        V m1 = c.mm == RTGPU_TWO_COPY ? Num<V>::sc(ml_hi[2 * j] + ml_hi[2 * j + 1], q)
                                      : Num<V>::sc(ml_hi[j], q);
        best = tmax(best, m1 + gr);
    }
    return best;
}

/* SuspTask validity (suspension.py:35) of task t under its count, exact:
 * every lo <= hi, and sum(exec hi) + sum(susp lo) <= T. */
template <class V> RT_HD bool susp_valid(const SetCtx<V> &c, const TaskRec &t, int gcount, typename Num<V>::Qt q) {
    const SegPtr sg = c.segs(t.seg);
    const int m = t.m, p = t.p, g = m - 1;
    const SegPtr cl_lo = sg, cl_hi = sg + m, ml_lo = sg + 2 * m, ml_hi = ml_lo + p;
    const SegPtr gw_lo = ml_hi + p, gw_hi = gw_lo + g, gl = gw_hi + g, an = gl + g;
    typename Num<V>::Qt perlo = t.isgpu ? q / (2 * (typename Num<V>::Qt)gcount) : q;
    typename Num<V>::Qt perhi =
        t.isgpu ? q / ((typename Num<V>::Qt)2 * (typename Num<V>::Qt)c.A * gcount) : q;
    if (t.D > t.T) return false; /* SuspTask: 0 < D <= T (suspension.py:40) */
    auto grl = [&](int j) { return (V)gw_lo[j] * (V)perlo; };
    auto gru = [&](int j) {
        return (V)((i128)gw_hi[j] * an[j] - (i128)gl[j] * c.A) * (V)perhi + Num<V>::sc(gl[j], q);
    };
    if (c.method == RTGPU_METHOD_BUSYWAIT) {
        V lo = Num<V>::sc(t.sCll + t.sMll, q), hi = Num<V>::sc(t.sClu + t.sMlu, q);
        #pragma unroll 1
        for (int j = 0; j < g; j++) {
            lo += grl(j);
            hi += gru(j);
        }
        return lo <= hi && hi <= Num<V>::sc(t.T, q);
    }
    if (m < 1) return false; /* SuspTask: at least one execution segment */
    #pragma unroll 1
    for (int j = 0; j < m; j++)
        if (cl_lo[j] > cl_hi[j]) return false;
    V sl_sum = 0;
    #pragma unroll 1
    for (int j = 0; j < g; j++) {
        V lo, hi;
        if (c.mm == RTGPU_TWO_COPY) {
            lo = Num<V>::sc(ml_lo[2 * j] + ml_lo[2 * j + 1], q) + grl(j);
            hi = Num<V>::sc(ml_hi[2 * j] + ml_hi[2 * j + 1], q) + gru(j);
        } else {
            lo = Num<V>::sc(ml_lo[j], q) + grl(j);
            hi = Num<V>::sc(ml_hi[j], q) + gru(j);
        }
        if (lo > hi) return false;
        sl_sum += lo;
    }
    return Num<V>::sc(t.sClu, q) + sl_sum <= Num<V>::sc(t.T, q);
}

/* task_response (suspension.py:155) of task k with blocking B at scale q;
 * verdict mode computes R2 first and R1 only if needed.  Returns -1 = None. */
template <class V, class TM>
RT_NI V baseline_response(const TM &tm, SetCtx<V> &c, int k, typename Num<V>::Qt q, V B,
                          bool want_all) {
    const TaskRec &t = c.TR()[k];
    const V D = Num<V>::sc(t.D, q);
    V sum_sh = 0, sum_eh;
    if (c.single_seg) {
        sum_eh = Num<V>::sc(t.sClu + t.sMlu, q) + grup_at(c, t, t.g, q);
    } else {
        sum_eh = Num<V>::sc(t.sClu, q);
        if (t.isgpu) sum_sh = Num<V>::sc(t.sMlu, q) + grup_at(c, t, t.g, q);
    }
    V r2 = lfp(tm, c, k, K_CPU, sum_sh + sum_eh + B, sum_sh + sum_eh + B, D);
    if (c.single_seg) return r2; /* one segment, no suspension: R1 == R2 */
    if (r2 >= 0 && !want_all) return r2;
    V *bases = c.SCR();
    V *outs = c.SCR() + (c.MP + c.MC + 2);
    const SegPtr cl_hi = c.segs(t.seg) + t.m;
    tm.pfor(t.m, [&](int j) { bases[j] = Num<V>::sc(cl_hi[j], q) + B; });
    bool none;
    lfp_many(tm, c, k, K_CPU, bases, outs, t.m, D, true, none);
    V r1 = (V)-1;
    if (!none) {
        V acc = sum_sh;
        #pragma unroll 1
        for (int j = 0; j < t.m; j++) acc += outs[j];
        if (acc <= D) r1 = acc;
    }
    tm.sync();
    if (r1 < 0) return r2;
    if (r2 < 0) return r1;
    return tmin(r1, r2);
}

/* scale of a full allocation: 2*A*lcm(all GPU counts) (1 without GPU tasks) */
template <class V> RT_HD typename Num<V>::Qt alloc_scale(SetCtx<V> &c) {
    typedef typename Num<V>::Qt Qt;
    Qt L = 1;
    bool any = false;
    #pragma unroll 1
    for (int i = 0; i < c.n; i++)
        if (c.TR()[i].isgpu) {
            any = true;
            L = lcm_lim<Qt>(L, (Qt)c.TR()[i].g, c.qlim);
            if (L == 0) break;
        }
    if (!any) return 1;
    if (L == 0 || L > c.qlim / (2 * (Qt)c.A)) {
        c.esc = 1;
        return 0;
    }
    return L * 2 * (Qt)c.A;
}

/* Evaluate the current full allocation (analysis.py:323-350 / 360-390).
 * Returns n if every task passes, else the index of the first failing task,
 * or -1 if some task is not a valid SuspTask (evaluate returns (False, {})).
 * With out != null (report), writes e2e / den / GR detail per task. */
template <class V, class TM>
RT_NI int eval_alloc_baseline(const TM &tm, SetCtx<V> &c, bool want_all, const OutPtrs<V> *out) {
    typedef typename Num<V>::Qt Qt;
    Qt q = alloc_scale(c);
    if (c.esc) return -2;
    c.vn = 0;
    ensure_views(tm, c, c.n, q);
    #pragma unroll 1
    for (int i = 0; i < c.n; i++)
        if (!susp_valid(c, c.TR()[i], c.TR()[i].g, q)) return -1;
    #pragma unroll 1
    for (int k = 0; k < c.n; k++) {
        c.evals++;
        V B = 0;
        if (c.method == RTGPU_METHOD_SELFSUSP)
            #pragma unroll 1
            for (int i = 0; i < c.n; i++)
                if (c.TR()[i].prio > c.TR()[k].prio) B = tmax(B, max_susp_hi(c, c.TR()[i], c.TR()[i].g, q));
        V r = baseline_response(tm, c, k, q, B, want_all);
        if (c.esc || c.stuck) return -2;
        if (out) {
            const TaskRec &t = c.TR()[k];
            tm.sync();
            if (sizeof(V) > 8 && ((i128)q > (i128)INT64_MAX || Num<V>::wide(r) > (i128)INT64_MAX)) {
                c.esc = 1;
                return -2;
            }
            if (tm.leader()) {
                out->e2e[k] = out_num(r);
                out->den[k] = (i64)q;
            }
            if (out->detail && t.isgpu) {
                const SegPtr sg = c.segs(t.seg);
                const int m = t.m, p = t.p, g = m - 1;
                const SegPtr gw_lo = sg + 2 * m + 2 * p, gw_hi = gw_lo + g, gl = gw_hi + g, an = gl + g;
                i64 *d = out->detail + t.seg;
                const Qt perlo = q / (2 * (Qt)t.g), perhi = q / (2 * (Qt)c.A * (Qt)t.g);
                tm.pfor(g, [&](int j) {
                    d[2 * m + 2 * p + j] = out_num((V)gw_lo[j] * (V)perlo);
                    V infl = (V)((i128)gw_hi[j] * an[j] - (i128)gl[j] * c.A);
                    d[2 * m + 2 * p + g + j] = out_num(infl * (V)perhi + Num<V>::sc(gl[j], q));
                });
            }
        }
        if (r < 0) return k;
    }
    return c.n;
}

/* smallest count >= lo at which task t is a valid SuspTask (monotone), 0 if none */
template <class V> RT_HD int min_valid_g(SetCtx<V> &c, int k, int lo) {
    typedef typename Num<V>::Qt Qt;
    const TaskRec &t = c.TR()[k];
    #pragma unroll 1
    for (int g = lo; g <= c.GN; g++) {
        Qt q = (Qt)2 * (Qt)c.A * (Qt)g;
        if (q > c.qlim) {
            c.esc = 1;
            return 0;
        }
        if (susp_valid(c, t, g, q)) return g;
    }
    return 0;
}

/* Lexicographic enumeration of analysis.py:250 _grid_search for the
 * baselines with sound pruning: allocations below a task's validity minimum
 * are skipped (they fail in evaluate), and when task f fails, every
 * allocation sharing the counts of GPU tasks up to f is skipped if f fails
 * regardless of the rest -- always for busy-waiting (no blocking term), and
 * for self-suspension when f also fails under the smallest blocking any
 * completion can give (each lp kernel span is at least its copies + GL). */
template <class V, class TM>
RT_NI int search_baseline(const TM &tm, SetCtx<V> &c) {
    int ids[RTGPU_MAX_TASKS], lower[RTGPU_MAX_TASKS], nid = 0;
    #pragma unroll 1
    for (int k = 0; k < c.n; k++)
        if (c.TR()[k].isgpu) {
            int g = min_valid_g(c, k, c.TR()[k].gmin);
            if (c.esc) return ST_ESCALATE;
            if (g == 0) return RTGPU_UNSCHEDULABLE;
            ids[nid] = k;
            lower[nid++] = g;
        }
    i64 need = 0;
    #pragma unroll 1
    for (int q = 0; q < nid; q++) need += lower[q];
    if (need > c.GN) return RTGPU_UNSCHEDULABLE;
    tm.sync();
    if (tm.leader())
        #pragma unroll 1
        for (int q = 0; q < nid; q++) c.TR()[ids[q]].g = lower[q];
    tm.sync();
    #pragma unroll 1
    for (;;) {
        if (c.budget > 0 && c.evals >= c.budget) return RTGPU_UNDECIDED;
        int f = eval_alloc_baseline(tm, c, false, (const OutPtrs<V> *)nullptr);
        if (c.esc) return ST_ESCALATE;
        if (c.stuck) return RTGPU_UNDECIDED;
        if (f == c.n) return RTGPU_SCHEDULABLE;
        int pos = nid - 1; /* odometer position to advance */
        if (f >= 0) {
            bool prefix_dead = c.method == RTGPU_METHOD_BUSYWAIT;
            if (!prefix_dead) {
                /* self-suspension: retry f with the smallest possible blocking */
                typedef typename Num<V>::Qt Qt;
                Qt q = alloc_scale(c);
                if (c.esc) return ST_ESCALATE;
                V Bmin = 0;
                #pragma unroll 1
                for (int i = 0; i < c.n; i++) {
                    const TaskRec &t = c.TR()[i];
                    if (t.prio <= c.TR()[f].prio || !t.isgpu) continue;
                    const SegPtr sg = c.segs(t.seg);
                    const int m = t.m, p = t.p, g = m - 1;
                    const SegPtr ml_hi = sg + 2 * m + p, gl = sg + 2 * m + 2 * p + 2 * g;
                    #pragma unroll 1
                    for (int j = 0; j < g; j++) {
                        i64 x = c.mm == RTGPU_TWO_COPY ? ml_hi[2 * j] + ml_hi[2 * j + 1] : ml_hi[j];
                        Bmin = tmax(Bmin, Num<V>::sc(x + gl[j], q));
                    }
                }
                V r = baseline_response(tm, c, f, q, Bmin, false);
                if (c.esc) return ST_ESCALATE;
                prefix_dead = r < 0;
            }
            if (prefix_dead) {
                pos = -1;
                #pragma unroll 1
                for (int q = 0; q < nid; q++)
                    if (ids[q] <= f) pos = q;
                if (pos < 0) return RTGPU_UNSCHEDULABLE; /* fails before any choice */
            }
        }
        /* advance the odometer at pos (gpu.py:43 order) */
        int q = pos;
        #pragma unroll 1
        for (; q >= 0; q--) {
            i64 used = 0, after = 0;
            #pragma unroll 1
            for (int a = 0; a < q; a++) used += c.TR()[ids[a]].g;
            #pragma unroll 1
            for (int a = q + 1; a < nid; a++) after += lower[a];
            if (c.TR()[ids[q]].g + 1 <= c.GN - used - after) break;
        }
        if (q < 0) return RTGPU_UNSCHEDULABLE;
        tm.sync();
        if (tm.leader()) {
            c.TR()[ids[q]].g += 1;
            #pragma unroll 1
            for (int a = q + 1; a < nid; a++) c.TR()[ids[a]].g = lower[a];
        }
        tm.sync();
        c.vn = 0;
    }
}

/* ------------------------------------------------------------ verdict fast path */

/* The hot case of the benchmark -- RTGPU verdicts (status + allocation) of
 * regular task sets whose whole search fits one FP64 scale Q = 2*A*lcm(1..GN)
 * -- as one compact routine: everything warp-uniform lives in registers or
 * shared memory, the only out-of-line callee is the fixed point below, which
 * takes scalars (no context on the stack), so the hot code stays inside the
 * instruction cache.  Same algorithm as the general path (greedy descent,
 * verdict shortcut, sorted warm starts, closed-form walks); anything else
 * returns ST_ESCALATE and the general stages take the set. */

/* load_task for the fast path: int64 only.  Values beyond the guarded
 * ranges (segments >= 2^31, A >= 2^16, D or T >= 2^56) mark the task
 * TF_UNSUP, which sends the set to the general path (128-bit load). */
template <class V>
RT_HD void load_task_fast_body(SetCtx<V> &c, int i) {
    const RecP r = rec_at(c.blob, i);
    TaskRec &t = c.TR()[i];
    t.m = (int)r[0];
    t.p = (int)r[1];
    t.D = r[2];
    t.T = r[3];
    t.prio = r[4];
    t.seg = r[5];
    t.idx = i;
    t.flags = 0;
    t.g = 0;
    t.gmin = 0;
    t.isgpu = t.m > 1;
    const int m = t.m, p = t.p, g = m - 1;
    const int want_p = m < 2 ? 0 : (c.mm == RTGPU_TWO_COPY ? 2 * m - 2 : m - 1);
    const i64 big = (i64)1 << 56;
    if (m < 1 || m > c.MC || p != want_p || p > c.MP || t.T <= 0 || t.D <= 0 || t.D > t.T ||
        t.T >= big || c.A >= (1 << 16)) {
        t.flags = TF_UNSUP;
        t.B = 0;
        return;
    }
    const Seg32 sg{(const int32_t *)c.blob + t.seg}; /* compact blob (checked by the caller) */
    i64 clu = 0, cll = 0, mlu = 0, mll = 0, gwl = 0, infl = 0, gls = 0, inner = 0, mx = 0, ih = 0;
    /* one pass over the area: the sums, and an OR of every value whose sign
     * says whether any is negative (then the set is not for the fast path) */
    i64 acc = 0;
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
        if (o > w) t.flags |= TF_INV;
        infl += w - o;
        ih += w;
        gls += gl;
        gwl += lo;
    }
    if (acc < 0) {
        t.flags = TF_UNSUP;
        t.B = 0;
        return;
    }
    t.sClu = clu;
    t.sCll = cll;
    t.sMlu = mlu;
    t.sMll = mll;
    t.sGWlo = gwl;
    t.sInfl = infl;
    t.sGL = gls;
    t.innerCll = inner;
    t.maxMlu = mx;
    t.invT = t.T > 0 ? 1.0 / (double)t.T : 0.0;
    /* range bound and isolated-bound minimum count (analysis.py:239) */
    t.B = t.D + t.T + clu + cll + mlu + mll + gwl + gls + ih / c.A + 1;
    if (t.isgpu) {
        const i64 X = t.D - gls - mlu - clu;
        i64 gm = 0;
        if (c.GN >= 1) {
            if (X > 0) {
                if (X > ((i64)1 << 60) / (2 * c.A)) gm = 1; /* infl / (2 A X) < 1 */
                else {
                    const i64 den = 2 * c.A * X;
                    gm = (infl + den - 1) / den;
                    if (gm < 1) gm = 1;
                }
                if (gm > c.GN) gm = 0;
            } else if (X == 0 && infl == 0) {
                gm = 1;
            }
        }
        if (gm == 0) t.flags |= TF_ISOFAIL;
        t.gmin = (int)gm;
        if (gm > 0) {
            /* regular: no wrap-around gap negative at gm (ceil division avoids overflow) */
            const i64 need = (gwl + 2 * gm - 1) / (2 * gm);
            if (t.T - clu - mll < need) t.flags |= TF_IRREG;
            if (t.T - mlu - inner < need) t.flags |= TF_IRREG;
        }
    } else {
        if (clu > t.D) t.flags |= TF_ISOFAIL;
        if (t.T - clu < 0) t.flags |= TF_IRREG;
    }
}

/* out-of-line entry with scalar arguments (see build_view_warp_s) */
template <class V>
RT_NI void load_task_fast_s(const i64 *blob, unsigned char *hbase, int o_tr, int mm, int MC, int MP, i64 A,
                            int GN, int i) {
    SetCtx<V> c;
    c.blob = blob;
    c.hbase = hbase;
    c.o_tr = o_tr;
    c.mm = mm;
    c.MC = MC;
    c.MP = MP;
    c.A = A;
    c.GN = GN;
    load_task_fast_body(c, i);
}

/* least fixed point on a fixed scale; -1 = None, -2 = iteration cap */
template <class V, class TM>
RT_NI V lfp_fast(const TM &tm, const TaskRec *tr, const V *views, int k, int kind, int lg,
                 int PM, int half, int stride, V base, V start, V bound, int check = 0) {
    /* check = 1: is `start` a pre-fixed point (base + I(start) <= start)?
     * Then the lfp is at most f(start), which is returned; else -3.
     * Otherwise `start` is a lower bound of the lfp. */
    if (base > bound || start > bound) return (V)-1;
    RT_COUNT(g_cnt_flfp[kind]);
    V r = start;
    for (int it = 0; it < ITER_CAP; it++) {
        RT_COUNT(g_cnt_fit[kind]);
        typename TM::template Acc<V> acc;
        tm.acc_init(acc);
        if (r > 0)
            for (int i0 = 0; i0 < k; i0 += (32 >> lg)) {
                RT_COUNT(g_cnt_frounds);
                tm.group_max_round(lg, [&](int slot, V &w, V &rr, bool &es) {
                    int i = i0 + (slot >> lg), h = slot & ((1 << lg) - 1);
                    if (i < k) {
                        /* hp(k) = tasks 0..k-1: fast_verdict admits only
                         * strictly increasing priorities */
                        const TaskRec &ti = tr[i];
                        int p = kind == K_CPU ? ti.m : ti.p;
                        if (h < p) w = walk(views + (size_t)i * stride, PM, half, p, h, r, rr, es);
                    }
                }, acc);
            }
        V I;
        bool err;
        tm.acc_sum(lg, acc, I, err);
        if (err) return (V)-1;
        V nxt = base + I;
        if (check == 2) return I; /* the interference at `start` */
        if (check) return nxt <= r ? nxt : (V)-3;
        if (nxt <= r) return r;
        nxt += tm.acc_rho(acc);
        if (nxt > bound) return (V)-1;
        r = nxt;
    }
    return (V)-2;
}

#ifndef RTGPU_FAST_DCHECK
#define RTGPU_FAST_DCHECK 1 /* A/B builds: 0 turns off the deadline pre-fixed-point check */
#endif

/* ST_ESCALATE_RANGE: only the scale did not fit V (the int64 instance may) */
enum { ST_ESCALATE_RANGE = 98 };

template <class V, class TM>
RT_HD int fast_verdict(const TM &tm, SetCtx<V> &c, int32_t *vsm_out) {
    typedef i64 Qt;
    const i64 *h = c.blob;
    const int n = (int)h[0], GN = (int)h[1];
    const i64 A = h[3];
    c.n = n;
    c.GN = GN;
    c.mm = (int)h[2];
    c.A = A;
    c.segw = h[7] != 0 ? 1 : 0; /* 1 or 2: int32 segment areas */
    if (h[7] != 1 && h[7] != 2) return ST_ESCALATE; /* the fast path reads compact blobs only */
    c.single_seg = 0;
    c.vn = 0;
    c.vq = 0;
    c.esc = 0;
    c.evals = 0;
    if (n < 1 || n > c.maxn || A < 1 || (c.mm != 0 && c.mm != 1) || GN < 1 || GN > 64)
        return ST_ESCALATE; /* GN > 64: the fixed scale almost never fits (gtop > 42); skip the
                             * task loads and take the general path's per-task scales */
    TaskRec *tr = c.TR();
    {
        const i64 *blob = c.blob;
        unsigned char *hb = c.hbase;
        const int o_tr = c.o_tr, mm = c.mm, MC = c.MC, MP = c.MP;
        tm.pfor(n, [&](int i) { load_task_fast_s<V>(blob, hb, o_tr, mm, MC, MP, A, GN, i); });
    }
    i64 vb_max = 0, need = 0;
    #pragma unroll 1
    for (int k = 0; k < n; k++)
        if ((tr[k].flags & (TF_UNSUP | TF_IRREG)) || (k > 0 && tr[k].prio <= tr[k - 1].prio))
            return ST_ESCALATE; /* (equal priorities: the general path) */
    #pragma unroll 1
    for (int k = 0; k < n; k++) {
        const TaskRec &t = tr[k];
        if (t.flags & TF_INV) return ST_ESCALATE;             /* the reference raises */
        if (t.flags & TF_ISOFAIL) return RTGPU_UNSCHEDULABLE; /* first such task in order */
        vb_max = tmax(vb_max, t.B);
        if (t.isgpu) need += t.gmin;
    }
    if (need > GN) return RTGPU_UNSCHEDULABLE;
    /* One scale for the whole search: q = 2 * A * lcm(1..gtop).  Every
     * count the search evaluates for task k lies in [gmin_k, gmin_k + slack]
     * (slack = GN - sum of minimum counts: ghi = GN - used - rest_min <=
     * GN - sum_{i != k} gmin_i), and the hp views use final counts from the
     * same ranges, so every GR term's denominator divides 2 * A * g with
     * g <= gtop = max_k min(GN, gmin_k + slack).  Usually far below GN (the
     * benchmark: gtop 3-5 instead of 10), which keeps low-utilisation sets
     * (long periods) inside FP64's exact range. */
    const i128 vb = (i128)vb_max * range_factor(n, c.MC, c.MP);
    if (vb > (i128)Num<V>::limit()) return ST_ESCALATE_RANGE;
    const Qt qlim = Num<V>::limit() / (Qt)vb;
    int gtop = 1;
    #pragma unroll 1
    for (int k = 0; k < n; k++)
        if (tr[k].isgpu) gtop = tmax(gtop, (int)tmin((i64)GN, (i64)tr[k].gmin + (GN - need)));
    const Qt L = lcm_upto(gtop);
    if (L == 0 || (i128)L * (2 * A) > (i128)qlim) return ST_ESCALATE_RANGE;
    const Qt q = L * 2 * A;
    c.Vb = (i64)vb;
    c.qlim = qlim;
    c.fixed_q = q;
    c.vq = q;
    tm.sync();
    tm.pfor(n, [&](int k) {
        i64 b = 0;
        #pragma unroll 1
        for (int i = 0; i < n; i++)
            if (tr[i].prio > tr[k].prio) b = tmax(b, tr[i].maxMlu);
        tr[k].B = b;
    });
#ifndef RTGPU_FAST_NOALLQUICK
    /* floor(a / b) for 0 <= a, b < 2^52 from inv ~ 1 / b: an FP64 estimate
     * and exact corrections (products below 2^53) -- no 64-bit division */
    auto fdiv = [](i64 a, i64 b, double inv) -> i64 {
        i64 q = (i64)((double)a * inv);
        if (q * b > a) q--;
        else if ((q + 1) * b <= a) q++;
        return q;
    };
    /* ---- every task at its minimum count at once (two-copy sets whose
     * tasks all have kernels; lattice.cuh has the derivation): per hp task
     * the CPU / memory interference in a window H is at most
     * (floor(H / T_i) + 2) sClu_i / sMlu_i (a regular chain meets at most
     * floor(H / C) + 2 jobs, C = T at any count), so each task's quick test
     * -- R2 at g_min with I_cpu(D), the longest copy's offset bound r* as a
     * memory pre-fixed point -- needs no view.  Lanes test the tasks in
     * parallel; if all pass, the all-minimum allocation (the first one
     * Algorithm 2 enumerates) is schedulable. */
    if (c.mm == RTGPU_TWO_COPY) {
        bool ok = true;
#ifdef __CUDA_ARCH__
        for (int k = tm.lane; k < n; k += 32) {
#else
        for (int k = 0; k < n; k++) {
#endif
            const TaskRec &t = tr[k];
            bool pk = false;
            if (t.isgpu && t.p > 0) {
                i64 iu = 0;
                #pragma unroll 1
                for (int i = 0; i < k; i++) iu += (fdiv(t.D, tr[i].T, tr[i].invT) + 2) * tr[i].sClu;
                const i64 d = 2 * A * (i64)t.gmin;
                const i64 gr = t.sGL + t.sInfl / d + (t.sInfl % d > 0 ? 1 : 0);
                const i64 bmax = t.maxMlu + t.B, bsum = t.sMlu + (i64)t.p * t.B;
                const i64 M = t.D - iu - t.sClu - gr - bsum;
                if (M >= 0) {
                    i64 rs = M / t.p;
                    if (rs > t.D - bmax) rs = t.D - bmax;
                    if (rs >= 0) {
                        const i64 H = bmax + rs;
                        i64 um = 0;
                        #pragma unroll 1
                        for (int i = 0; i < k && um <= rs; i++) um += (fdiv(H, tr[i].T, tr[i].invT) + 2) * tr[i].sMlu;
                        pk = um <= rs;
                    }
                }
            }
            ok = ok && pk;
        }
#ifdef __CUDA_ARCH__
        ok = __all_sync(0xffffffffu, ok);
#endif
        if (ok) {
            c.evals = n;
            tm.pfor(n, [&](int i) { vsm_out[i] = 2 * tr[i].gmin; });
            return RTGPU_SCHEDULABLE;
        }
    }
#endif
    const int lgC = c.lgC, lgM = c.lgM, halfC = c.halfC, halfM = c.halfM;
    const int SC = c.L.SC, SM = c.L.SM, MC = c.MC, MP = c.MP;
    V *vc = c.VC(), *vm = c.VM();
    V *bases = c.SCR();
    V *outs = c.SCR() + (c.MP + c.MC + 2);
    int *ord = (int *)(c.SCR() + c.L.scr_n) - 32;
    /* L / g for every count g <= gtop (GR up = sInfl * L/g + GL at scale
     * q): one lane-parallel division per set instead of a 64-bit division
     * per evaluation; outs has room when gtop <= scr_n - (MP + MC + 2) - 32 */
    const bool lg_tab = gtop <= c.L.scr_n - (c.MP + c.MC + 2) - 32;
    if (lg_tab) tm.pfor(gtop, [&](int x) { outs[x] = (V)(L / (Qt)(x + 1)); });
    i64 used = 0, rest_min = need;
    V mem_prev_b = -1, mem_prev_r = 0; /* last memory fixed point (base, value) */
    V mem_guess = 0;                   /* last memory offset (or verified bound): the next guess */
    #pragma unroll 1
    for (int k = 0; k < n; k++) {
        const TaskRec &t = tr[k];
        /* views of tasks before k (their counts are final) */
#ifdef __CUDA_ARCH__
        if (k > 0)
            build_view_warp_s<V>(c.blob, c.o_tr, c.o_vc, c.o_vm, c.L.SC, c.L.SM, c.MC, c.MP, c.mm, k - 1, q,
                                 tm.lane);
#else
        if (k > 0) tm.pfor(1, [&](int) { build_view<V, Seg32>(c, k - 1, q); });
#endif
        const Seg32 sg{(const int32_t *)c.blob + t.seg};
        const Seg32 cl_hi = sg + t.m, ml_hi = sg + 2 * t.m + t.p;
        const V D = Num<V>::sc(t.D, q);
        int glo = 0, ghi = 0;
        if (t.isgpu) {
            rest_min -= t.gmin;
            const i64 gmax = GN - used - rest_min;
            if (gmax < t.gmin) return RTGPU_UNSCHEDULABLE;
            glo = t.gmin;
            ghi = (int)gmax;
        }
        int g = glo;
        bool quick = false;
#ifndef RTGPU_FAST_NOQUICK
        /* ---- quick pass at the minimum count (sufficient; two evaluations):
         * R2 (analysis.py:214) passes at glo if its base plus I_cpu(D) fits
         * D (f(D) <= D); that leaves room M for sum MR <= p r + bsum (r the
         * longest copy's offset, MR_j <= b_j + r by lfp(b') >= lfp(b) +
         * (b' - b)), and r* = floor(M / p) is verified as a memory
         * pre-fixed point (then every MR exists, analysis.py:156).  Any
         * failure falls through to the exact search below. */
        if (t.isgpu && t.p > 0) {
            const V iu = lfp_fast(tm, tr, vc, k, K_CPU, lgC, MC, halfC, SC, (V)0, D, D, 2);
            if (iu >= 0) {
                i64 bmax_t = 0, bsum_t = 0;
#if defined(__CUDA_ARCH__)
                {
                    const i64 v = tm.lane < t.p ? ml_hi[tm.lane] + t.B : 0;
                    bmax_t = v;
                    bsum_t = v;
                    #pragma unroll
                    for (int off = 16; off > 0; off >>= 1) {
                        bmax_t = tmax(bmax_t, shfl_x(bmax_t, off));
                        bsum_t += shfl_x(bsum_t, off);
                    }
                }
#else
                for (int j = 0; j < t.p; j++) {
                    bmax_t = tmax(bmax_t, ml_hi[j] + t.B);
                    bsum_t += ml_hi[j] + t.B;
                }
#endif
                const V grup = (V)t.sInfl * (lg_tab ? outs[glo - 1] : (V)(q / (2 * A * (Qt)glo))) +
                               Num<V>::sc(t.sGL, q);
                const V M = D - iu - Num<V>::sc(t.sClu, q) - grup - Num<V>::sc(bsum_t, q);
                if (M >= 0) {
                    const V bmax = Num<V>::sc(bmax_t, q);
                    V rs = Num<V>::floordiv(M, (V)t.p);
                    if (rs > D - bmax) rs = D - bmax;
                    if (rs >= 0 && lfp_fast(tm, tr, vm, k, K_MEM, lgM, MP, halfM, SM, bmax, bmax + rs, D, 1) >= 0)
                        quick = true;
                }
            }
        }
#endif
        c.evals++; /* one count evaluation per task, quick or exact */
        if (!quick) {
            /* ---- g-independent part: memory responses (Lemma 6) */
            V sum_mr = 0, mr_ub = 0;
            bool have_exact_mr = t.p == 0, rmax_exact = true;
            i64 bsum_k = 0;
            V bmax_k = 0;
            if (t.p > 0) {
                i64 bmax_t = 0, bsum_t = 0;
    #if defined(__CUDA_ARCH__) && !defined(RTGPU_FAST_NO_LANESUMS)
                { /* one load per lane and two butterflies (p <= 30): +1.1% on the
                   * 8 x 5 sweep over the sequential loop (scripts/gpu_lat_ab.sh r2u) */
                    const i64 v = tm.lane < t.p ? ml_hi[tm.lane] + t.B : 0;
                    bmax_t = v;
                    bsum_t = v;
                    #pragma unroll
                    for (int off = 16; off > 0; off >>= 1) {
                        bmax_t = tmax(bmax_t, shfl_x(bmax_t, off));
                        bsum_t += shfl_x(bsum_t, off);
                    }
                }
    #else
                #pragma unroll 1
                for (int j = 0; j < t.p; j++) {
                    bmax_t = tmax(bmax_t, ml_hi[j] + t.B);
                    bsum_t += ml_hi[j] + t.B;
                }
    #endif
                const V bmax = Num<V>::sc(bmax_t, q);
                bsum_k = bsum_t;
                bmax_k = bmax;
                /* warm start across tasks: hp(k) grows with k, so the memory
                 * interference of task k is pointwise >= that of any earlier
                 * task, and lfp(b') >= lfp(b) + (b' - b) for b' >= b: the
                 * previous task's fixed point shifted by the base difference is
                 * below this one */
                V rmax = -1;
                /* off by default: on the 8 x 5 benchmark the longer code costs more
                 * than the saved iterations (scripts/gpu_lat_ab.sh r2l: 24.4 vs
                 * 25.5 M sets/s); the lattice path keeps it (alloc64 +14%) */
    #ifdef RTGPU_FAST_GUESS
                if (mem_guess > 0) {
    #else
                if (false) {
    #endif
                    /* the previous task's memory offset grown by half, verified
                     * as a pre-fixed point in one evaluation (then the lfp is at
                     * most f(U) <= D: every MR exists, bounded via f(U)); the
                     * exact fixed point only if R2 needs it (lattice.cuh) */
                    const V U = bmax + Num<V>::sc(1, q) + floor(mem_guess * 1.5);
                    if (U <= D) rmax = lfp_fast(tm, tr, vm, k, K_MEM, lgM, MP, halfM, SM, bmax, U, D, 1);
                    rmax_exact = rmax < 0;
                }
                if (rmax < 0) {
                    V start = bmax;
                    if (mem_prev_b >= 0 && bmax >= mem_prev_b) start = tmax(bmax, mem_prev_r + (bmax - mem_prev_b));
                    rmax = start > D ? (V)-1 : lfp_fast(tm, tr, vm, k, K_MEM, lgM, MP, halfM, SM, bmax, start, D);
                    if (rmax == (V)-2) return ST_ESCALATE;
                    if (rmax < 0) return RTGPU_UNSCHEDULABLE; /* the longest copy's MR is None */
                    mem_prev_b = bmax;
                    mem_prev_r = rmax;
                }
                mem_guess = rmax - bmax;
                mr_ub = (V)t.p * (rmax - bmax) + Num<V>::sc(bsum_t, q);
            }
            V sum_cr = -1; /* not computed yet; -2: some CR is None */
            /* task k passes at count g?  (R2 with the MR upper bound, then exact) */
            auto passes = [&](int g) -> int {
                RT_COUNT(g_cnt_passes);
                const V grup = t.isgpu ? (V)t.sInfl * (lg_tab ? outs[g - 1] : (V)(q / (2 * A * (Qt)g))) +
                                             Num<V>::sc(t.sGL, q)
                                       : (V)0;
                const V cl = Num<V>::sc(t.sClu, q);
                if (t.p > 0 || !have_exact_mr) {
                    V b2 = grup + mr_ub + cl;
                    /* R2 proven at the deadline itself (f(D) <= D) in one evaluation */
                    if (RTGPU_FAST_DCHECK && b2 <= D && lfp_fast(tm, tr, vc, k, K_CPU, lgC, MC, halfC, SC, b2, D, D, 1) >= 0)
                        return 1;
                    if (!rmax_exact) {
                        /* the verified memory bound was loose: the exact one */
                        const V rm = lfp_fast(tm, tr, vm, k, K_MEM, lgM, MP, halfM, SM, bmax_k, bmax_k, D);
                        if (rm < 0) return -1; /* cannot be None below a verified bound */
                        rmax_exact = true;
                        mem_prev_b = bmax_k;
                        mem_prev_r = rm;
                        mem_guess = rm - bmax_k;
                        mr_ub = (V)t.p * (rm - bmax_k) + Num<V>::sc(bsum_k, q);
                        b2 = grup + mr_ub + cl;
                        if (RTGPU_FAST_DCHECK && b2 <= D && lfp_fast(tm, tr, vc, k, K_CPU, lgC, MC, halfC, SC, b2, D, D, 1) >= 0)
                            return 1;
                    }
                    const V r = lfp_fast(tm, tr, vc, k, K_CPU, lgC, MC, halfC, SC, b2, b2, D);
                    if (r == (V)-2) return -1;
                    if (r >= 0) return 1;
                    if (!have_exact_mr) {
                        /* exact memory responses, ascending bases with warm starts */
                        tm.pfor(t.p, [&](int j) { bases[j] = Num<V>::sc(ml_hi[j] + t.B, q); });
                        tm.pfor(t.p, [&](int j) {
                            int rk = 0;
                            #pragma unroll 1
                            for (int x = 0; x < t.p; x++)
                                rk += (bases[x] < bases[j] || (bases[x] == bases[j] && x < j)) ? 1 : 0;
                            ord[rk] = j;
                        });
                        V pb = 0, pr = 0, acc = 0;
                        #pragma unroll 1
                        for (int st = 0; st < t.p; st++) {
                            const V b = bases[ord[st]];
                            const V r0 = lfp_fast(tm, tr, vm, k, K_MEM, lgM, MP, halfM, SM, b,
                                                  st ? tmax(b, pr + (b - pb)) : b, D);
                            if (r0 < 0) return r0 == (V)-2 ? -1 : 0; /* cannot be None: rmax was not */
                            acc += r0;
                            pb = b;
                            pr = r0;
                        }
                        sum_mr = acc;
                        have_exact_mr = true;
                    }
                    if (sum_mr != mr_ub) {
                        const V b3 = grup + sum_mr + cl;
                        const V r3 = lfp_fast(tm, tr, vc, k, K_CPU, lgC, MC, halfC, SC, b3, b3, D);
                        if (r3 == (V)-2) return -1;
                        if (r3 >= 0) return 1;
                    }
                } else {
                    const V b3 = grup + cl;
                    if (RTGPU_FAST_DCHECK && b3 <= D && lfp_fast(tm, tr, vc, k, K_CPU, lgC, MC, halfC, SC, b3, D, D, 1) >= 0)
                        return 1;
                    const V r3 = lfp_fast(tm, tr, vc, k, K_CPU, lgC, MC, halfC, SC, b3, b3, D);
                    if (r3 == (V)-2) return -1;
                    if (r3 >= 0) return 1;
                }
                /* R1 = GR up + sum MR + sum CR (analysis.py:207) */
                if (sum_cr == -1) {
                    tm.pfor(t.m, [&](int j) { bases[j] = Num<V>::sc(cl_hi[j], q); });
                    tm.pfor(t.m, [&](int j) {
                        int rk = 0;
                        #pragma unroll 1
                        for (int x = 0; x < t.m; x++)
                            rk += (bases[x] < bases[j] || (bases[x] == bases[j] && x < j)) ? 1 : 0;
                        ord[rk] = j;
                    });
                    V pb = 0, pr = 0, acc = 0;
                    #pragma unroll 1
                    for (int st = 0; st < t.m; st++) {
                        const V b = bases[ord[st]];
                        const V r0 = lfp_fast(tm, tr, vc, k, K_CPU, lgC, MC, halfC, SC, b,
                                              st ? tmax(b, pr + (b - pb)) : b, D);
                        if (r0 == (V)-2) return -1;
                        if (r0 < 0) {
                            acc = -2;
                            break;
                        }
                        acc += r0;
                        pb = b;
                        pr = r0;
                    }
                    sum_cr = acc;
                }
                if (sum_cr < 0) return 0;
                return grup + sum_mr + sum_cr <= D ? 1 : 0;
            };
            /* smallest passing count: glo, else ghi, else bisection -- one call
             * site for `passes` keeps a single inlined copy */
            g = 0;
            int lo = glo, hi = ghi, phase = t.isgpu ? 0 : 3;
            int cand = t.isgpu ? glo : 0;
            #pragma unroll 1
            for (;;) {
                const int o = passes(cand);
                if (o < 0) return ST_ESCALATE;
                if (phase == 3) { /* pure-CPU task: one evaluation */
                    if (!o) return RTGPU_UNSCHEDULABLE;
                    break;
                }
                if (phase == 0) {
                    if (o) {
                        g = glo;
                        break;
                    }
                    if (glo >= ghi) return RTGPU_UNSCHEDULABLE;
                    phase = 1;
                    cand = ghi;
                    continue;
                }
                if (phase == 1) {
                    if (!o) return RTGPU_UNSCHEDULABLE;
                    phase = 2;
                } else if (o) {
                    hi = cand;
                } else {
                    lo = cand;
                }
                if (hi - lo <= 1) {
                    g = hi;
                    break;
                }
                cand = lo + (hi - lo) / 2;
            }
        }
        if (!t.isgpu) continue;
        tm.sync();
        if (tm.leader()) tr[k].g = g;
        tm.sync();
        used += g;
    }
    tm.pfor(n, [&](int i) { vsm_out[i] = tr[i].isgpu ? 2 * tr[i].g : 0; });
    return RTGPU_SCHEDULABLE;
}

/* ------------------------------------------------------------ point queries */

/* One query of include/rtgpu.h rtgpu_query_*: a building block of the
 * analysis evaluated on a packed set whose kernels carry explicit response
 * bounds (one physical SM each, alpha = 1, GL = 0, GW = 2 * GR), so every
 * value lives on the scale q = 2 * A.  Returns a status; *res is the
 * numerator over q (-1 = None). */
template <class V, class TM>
RT_NI int run_query(const TM &tm, SetCtx<V> &c, int kind, int k, int idx, i64 horizon, i64 blocking,
                    i64 *res_num, i64 *res_den) {
    typedef typename Num<V>::Qt Qt;
    const i64 *h = c.blob;
    c.n = (int)h[0];
    c.GN = (int)h[1];
    c.mm = (int)h[2];
    c.A = h[3];
    c.segw = (int)h[7];
    c.vn = 0;
    c.vq = 0;
    c.esc = 0;
    c.stuck = 0;
    c.evals = 0;
    c.single_seg = 0;
    c.fixed_q = 0;
    if (c.n < 1 || c.n > c.maxn || c.A < 1 || k < 0 || k >= c.n) return RTGPU_INVALID;
    i128 vb_max = 0;
    tm.pfor(c.n, [&](int i) {
        i128 vb;
        load_task(c, i, &vb);
        c.TR()[i].B = vb > (i128)((i64)1 << 62) ? ((i64)1 << 62) : (i64)vb;
        c.TR()[i].g = 1;
    });
    #pragma unroll 1
    for (int i = 0; i < c.n; i++) {
        if (c.TR()[i].flags & TF_UNSUP) return RTGPU_INVALID;
        vb_max = tmax(vb_max, (i128)c.TR()[i].B);
    }
    i128 hz = (i128)(horizon < 0 ? 0 : horizon) + (blocking < 0 ? 0 : blocking);
    i128 vb = (vb_max + hz) * ((i128)c.n + 2 * RTGPU_MAX_M + 4);
    if (vb > (i128)Num<V>::limit()) return ST_ESCALATE;
    c.Vb = (i64)vb;
    c.qlim = (Qt)(Num<V>::limit() / (Qt)c.Vb);
    tm.sync();
    tm.pfor(c.n, [&](int kk) {
        i64 b = 0;
        #pragma unroll 1
        for (int i = 0; i < c.n; i++)
            if (c.TR()[i].prio > c.TR()[kk].prio) b = tmax(b, c.TR()[i].maxMlu);
        c.TR()[kk].B = b;
    });
    const Qt q = (Qt)2 * (Qt)c.A;
    if (q > c.qlim) return ST_ESCALATE;
    ensure_views(tm, c, c.n, q);
    const TaskRec &t = c.TR()[k];
    const SegPtr sg = c.segs(t.seg);
    const V D = Num<V>::sc(t.D, q);
    V r = (V)-1;
    *res_den = (i64)q;
    if (kind == RTGPU_Q_WORKLOAD || kind == RTGPU_Q_MAX_WORKLOAD || kind == RTGPU_Q_CPU_WORKLOAD ||
        kind == RTGPU_Q_MEM_WORKLOAD) {
        const bool mem = kind == RTGPU_Q_MEM_WORKLOAD;
        const int p = mem ? t.p : t.m;
        if (p == 0) {
            *res_num = 0;
            return RTGPU_SCHEDULABLE;
        }
        const int PM = mem ? c.MP : c.MC;
        const V *view = (mem ? c.VM() + (size_t)k * c.L.SM : c.VC() + (size_t)k * c.L.SC);
        const int half = mem ? c.halfM : c.halfC;
        const V H = Num<V>::sc(horizon, q);
        V best = 0;
        bool err = false;
        const int h0 = kind == RTGPU_Q_MAX_WORKLOAD ? 0 : idx;
        const int h1 = kind == RTGPU_Q_MAX_WORKLOAD ? p : idx + 1;
        if (h0 < 0 || h1 > p) return RTGPU_INVALID;
        #pragma unroll 1
        for (int hh = h0; hh < h1; hh++) {
            V rho;
            V w = walk(view, PM, half, p, hh, H, rho, err);
            if (hh == h0 || w > best) best = w;
        }
        if (err) return RTGPU_GAP_ERROR;
        r = best;
    } else if (kind == RTGPU_Q_SEGMENT_RESPONSE) {
        if (idx < 0 || idx >= t.m) return RTGPU_INVALID;
        V b = Num<V>::sc(sg[t.m + idx] + blocking, q);
        r = lfp(tm, c, k, K_CPU, b, b, D);
    } else if (kind == RTGPU_Q_TASK_RESPONSE) {
        r = baseline_response(tm, c, k, q, Num<V>::sc(blocking, q), true);
    } else if (kind == RTGPU_Q_MEM_RESPONSE) {
        if (idx < 0 || idx >= t.p) return RTGPU_INVALID;
        V b = Num<V>::sc(sg[2 * t.m + t.p + idx] + t.B, q);
        r = lfp(tm, c, k, K_MEM, b, b, D);
    } else if (kind == RTGPU_Q_CPU_RESPONSE) {
        if (idx < 0 || idx >= t.m) return RTGPU_INVALID;
        V b = Num<V>::sc(sg[t.m + idx], q);
        r = lfp(tm, c, k, K_CPU, b, b, D);
    } else if (kind == RTGPU_Q_END_TO_END) {
        TaskEval<V> res;
        eval_task(tm, c, k, 1, (Qt)1, true, res, (V *)nullptr, (V *)nullptr);
        r = res.e2e;
    } else if (kind == RTGPU_Q_R2) {
        V b = Num<V>::sc(horizon, q);
        r = lfp(tm, c, k, K_CPU, b, b, D);
    } else {
        return RTGPU_INVALID;
    }
    if (c.esc) return ST_ESCALATE;
    if (c.stuck) return RTGPU_UNDECIDED;
    if (sizeof(V) > 8 && Num<V>::wide(r) > (i128)INT64_MAX) return ST_ESCALATE;
    *res_num = r < 0 ? (i64)RTGPU_NONE : (i64)Num<V>::wide(r);
    return RTGPU_SCHEDULABLE;
}

/* Whole pipeline for one set; returns the status (or ST_ESCALATE). */
template <class V, class TM>
RT_NI int analyze_set(const TM &tm, SetCtx<V> &c, unsigned flags, const OutPtrs<V> &o) {
    typedef typename Num<V>::Qt Qt;
    const i64 *h = c.blob;
    c.n = (int)h[0];
    c.GN = (int)h[1];
    c.mm = (int)h[2];
    c.A = h[3];
    c.segw = (int)h[7];
    c.vn = 0;
    c.vq = 0;
    c.esc = 0;
    c.stuck = 0;
    c.evals = 0;
    c.budget_hit = 0;
    c.single_seg = c.method == RTGPU_METHOD_BUSYWAIT;
    tm.pfor(c.n, [&](int i) {
        o.vsm[i] = 0;
        o.e2e[i] = RTGPU_ABSENT;
        o.den[i] = 1;
    });
    if (c.n < 0 || c.n > c.maxn || c.A < 1 || (c.mm != 0 && c.mm != 1) || c.segw < 0 ||
        c.segw > 2 || (c.segw >= 1 && o.detail))
        return RTGPU_INVALID; /* the detail output mirrors the int64 layout */
    /* per-task loading; range bound = (n + 2M + 4) * max(D + T + sums) */
    i128 vb_max = 0;
    {
        /* lanes load tasks; reduce the bound through the TaskRec B field */
        tm.pfor(c.n, [&](int i) {
            i128 vb;
            load_task(c, i, &vb);
            /* store the clamped bound temporarily in B (recomputed below) */
            c.TR()[i].B = vb > (i128)((i64)1 << 62) ? ((i64)1 << 62) : (i64)vb;
        });
        #pragma unroll 1
        for (int i = 0; i < c.n; i++) vb_max = tmax(vb_max, (i128)c.TR()[i].B);
    }
    #pragma unroll 1
    for (int k = 0; k < c.n; k++)
        if (c.TR()[k].flags & TF_UNSUP) return RTGPU_INVALID;
    /* reference order: the first task whose min-SM search raises or fails */
    #pragma unroll 1
    for (int k = 0; k < c.n; k++) {
        if (c.TR()[k].flags & TF_INV) return RTGPU_INVALID;
        if (c.TR()[k].flags & TF_ISOFAIL) return RTGPU_UNSCHEDULABLE;
    }
    i64 need = 0;
    bool irregular = false;
    #pragma unroll 1
    for (int k = 0; k < c.n; k++) {
        if (c.TR()[k].isgpu) need += c.TR()[k].gmin;
        if (c.TR()[k].flags & TF_IRREG) irregular = true;
    }
    if (need > c.GN) return RTGPU_UNSCHEDULABLE;
    i128 factor = range_factor(c.n, c.MC, c.MP);
    i128 vb = vb_max * factor;
    if (vb > (i128)Num<V>::limit()) return ST_ESCALATE;
    c.Vb = (i64)vb;
    c.qlim = (Qt)(Num<V>::limit() / (Qt)c.Vb);
    c.fixed_q = 0;
#ifndef RTGPU_NO_FIXED_Q
    if (c.method == RTGPU_METHOD_RTGPU && c.GN >= 1 && c.GN <= 64) {
        Qt L = 1;
        #pragma unroll 1
        for (int g = 2; g <= c.GN && L != 0; g++) L = lcm_lim<Qt>(L, (Qt)g, c.qlim);
        if (L != 0 && L <= c.qlim / (2 * (Qt)c.A)) c.fixed_q = L * 2 * (Qt)c.A;
    }
#endif
    tm.sync();
    /* mem blocking term of analysis.py:162: longest copy of any lower-priority task */
    tm.pfor(c.n, [&](int k) {
        i64 b = 0;
        #pragma unroll 1
        for (int i = 0; i < c.n; i++)
            if (c.TR()[i].prio > c.TR()[k].prio) b = tmax(b, c.TR()[i].maxMlu);
        c.TR()[k].B = b;
    });
    const bool rtg = c.method == RTGPU_METHOD_RTGPU;
    int st = !rtg ? search_baseline(tm, c) : irregular ? search_dfs(tm, c) : search_greedy(tm, c);
    if (st == ST_ESCALATE) return st;
    if (st == RTGPU_SCHEDULABLE) {
        tm.pfor(c.n, [&](int i) { o.vsm[i] = c.TR()[i].isgpu ? 2 * c.TR()[i].g : 0; });
    }
    if ((flags & (RTGPU_F_BOUNDS | RTGPU_F_DETAIL)) &&
        (st == RTGPU_SCHEDULABLE || st == RTGPU_UNSCHEDULABLE)) {
        if (st == RTGPU_UNSCHEDULABLE) {
            /* the reference reports the last allocation it tried: the
             * lexicographically largest one (first GPU task takes the rest) */
            int first = -1;
            i64 others = 0;
            #pragma unroll 1
            for (int k = 0; k < c.n; k++)
                if (c.TR()[k].isgpu) {
                    if (first < 0) first = k;
                    else others += c.TR()[k].gmin;
                }
            tm.sync();
            if (tm.leader())
                #pragma unroll 1
                for (int k = 0; k < c.n; k++)
                    c.TR()[k].g = c.TR()[k].isgpu ? (k == first ? (int)(c.GN - others) : c.TR()[k].gmin) : 0;
            tm.sync();
            c.vn = 0;
        }
        c.stuck = 0;
        if (rtg) {
            report_pass(tm, c, o, st == RTGPU_UNSCHEDULABLE);
        } else {
            int f = eval_alloc_baseline(tm, c, true, &o);
            if (f >= 0) /* tasks after the first failing one are not in per_task */
                #pragma unroll 1
                for (int k = f + 1; k < c.n; k++)
                    if (tm.leader()) {
                        o.e2e[k] = RTGPU_ABSENT;
                        o.den[k] = 1;
                    }
            tm.sync();
        }
        if (c.esc) return ST_ESCALATE;
        if (c.stuck) return RTGPU_UNDECIDED;
    }
    return st;
}

}  // namespace rtgpu
