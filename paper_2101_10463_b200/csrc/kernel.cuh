/*
 * kernel.cuh -- persistent warp-per-set kernels and their launchers,
 * instantiated once per arithmetic in rtgpu_k_{f64,i64,i128}.cu (separate
 * translation units so the instantiations compile in parallel).
 *
 * Stages (one stream, no host round trip; each stage reads the sets the
 * previous one escalated from a device-side list):
 *   0  front_kernel        FP64  every set: verdict fast path or general path
 *   1  analyze_kernel<f64> FP64  general path
 *   2  analyze_kernel<i64> int64
 *   3  analyze_kernel<i128> int128 (beyond: RTGPU_RANGE)
 */
#pragma once
#include <cuda_runtime.h>
#include <stdio.h>

#include "engine_core.cuh"

namespace rtgpu {

#ifndef RTGPU_MAX_CHUNKS
#define RTGPU_MAX_CHUNKS 32
#endif

struct KParams {
    const i64 *blobs, *set_off, *task_base;
    i64 n_sets;
    Dims dims;
    int GC, GM;
    unsigned flags;
    int method;
    i64 budget;
    int32_t *status;
    i64 *evals;
    int32_t *vsm;
    i64 *e2e, *den, *detail;
    /* ctr[0] front-stage work counter (unchunked launch), ctr[1..3]
     * general-stage work counters, ctr[4..6] lengths of esc[0..2]; esc[s]
     * holds the sets stage s hands to stage s+1 */
    unsigned long long *ctr;
    i64 *esc[3];
    int use_fast;              /* front stage runs the verdict fast path */
    int last_stage = 3;        /* escalating past this general stage is RTGPU_RANGE (3; 2 in
                                * verdict runs, whose general stages are int64 then int128) */
    /* streamed input (end-to-end path): set s of chunk c = the c with
     * chunk_begin[c] <= s < chunk_begin[c + 1] is readable once
     * chunk_flag[c] == epoch (the copy stream writes it after the chunk's
     * H2D copy) */
    const unsigned long long *chunk_flag = nullptr;
    i64 chunk_begin[RTGPU_MAX_CHUNKS + 1];
    /* set to epoch by the first warp whose wait times out: every other warp
     * then stops waiting at once and the host re-runs the batch unstreamed */
    unsigned long long *chunk_abort = nullptr;
    unsigned long long epoch = 0;
    int chunks = 1;
    i64 set_base;              /* front stage: first set of this launch (chunked e2e path) */
    unsigned long long *wctr0; /* front stage: this launch's work counter */
    unsigned long long *lat_ctr = nullptr; /* lattice list stage's work counter */
};

/* minimum resident CTAs per SM the register allocation must allow */
#ifndef RTGPU_MINB
#define RTGPU_MINB 4
#endif
template <class V> struct MinBlocks { static constexpr int value = RTGPU_MINB; };
template <> struct MinBlocks<i128> { static constexpr int value = 2; };

template <class V>
__device__ __forceinline__ void kernel_ctx(SetCtx<V> &c, const Dims &dims, const Layout<V> &L, int warp) {
    c.hbase = nullptr;
    c.o_tr = warp * L.bytes;
    c.o_vc = c.o_tr + L.off_views_c;
    c.o_vm = c.o_tr + L.off_views_m;
    c.o_scr = c.o_tr + L.off_scr;
    c.L = L;
    c.maxn = dims.maxn;
    c.MC = dims.MC;
    c.MP = dims.MP;
    set_groups(c);
}

/* Stages 1..3 (V = double, int64, int128): the general path over the sets
 * the previous stage escalated. */
template <class V>
__global__ void __launch_bounds__(256, MinBlocks<V>::value) analyze_kernel(KParams p, int stage) {
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    Layout<V> L;
    L.init(p.dims);
    SetCtx<V> c;
    kernel_ctx(c, p.dims, L, warp);
    c.budget = p.budget;
    c.method = p.method;
    WarpTeam tm{lane};
    const i64 count = (i64)p.ctr[4 + stage - 1];
    const i64 *list = p.esc[stage - 1];
    for (;;) {
        unsigned long long idx = 0;
        if (lane == 0) idx = atomicAdd(&p.ctr[stage], 1ull);
        idx = __shfl_sync(0xffffffffu, idx, 0);
        if ((i64)idx >= count) break;
        const i64 s = list[idx];
        if (s < 0) continue; /* decided by stage 1a (the int64 fast path) */
        c.blob = p.blobs + p.set_off[s];
        const i64 tb = p.task_base[s];
        OutPtrs<V> o;
        o.vsm = p.vsm + tb;
        o.e2e = p.e2e + tb;
        o.den = p.den + tb;
        o.detail = p.detail ? p.detail + p.set_off[s] : nullptr;
        const bool force = (stage == 1 && (p.flags & (RTGPU_F_FIRST_I64 | RTGPU_F_FIRST_I128))) ||
                           (stage == 2 && (p.flags & RTGPU_F_FIRST_I128));
        int st = force ? (int)ST_ESCALATE : analyze_set(tm, c, p.flags, o);
        if (st == ST_ESCALATE) {
            if (stage < p.last_stage) {
                if (lane == 0) {
                    unsigned long long pos = atomicAdd(&p.ctr[4 + stage], 1ull);
                    p.esc[stage][pos] = s;
                }
                __syncwarp();
                continue;
            }
            st = RTGPU_RANGE;
        }
        if (lane == 0) {
            p.status[s] = st;
            p.evals[s] = c.evals;
        }
        __syncwarp();
    }
}

/* Stage 1a (verdict runs): the fast path in int64 over stage 0's
 * escalations.  With the fixed scale from the candidate counts (gtop) the
 * only sets stage 0 still escalates are range escalations (a handful per
 * 100 000: periods so long that the FP64 scale does not fit), which the
 * int64 instance decides in fast-path time instead of a general-path
 * latency; it is a separate kernel so the FP64 fast kernel keeps its
 * registers.  Decided entries of stage 0's list become -1 and the general
 * stage skips them. */
template <class V>
__global__ void __launch_bounds__(256, MinBlocks<V>::value) fast_list_kernel(KParams p) {
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    Layout<V> L;
    L.init(p.dims);
    SetCtx<V> c;
    kernel_ctx(c, p.dims, L, warp);
    c.budget = p.budget;
    c.method = p.method;
    WarpTeam tm{lane};
    const i64 count = (i64)p.ctr[4];
    for (;;) {
        unsigned long long idx = 0;
        if (lane == 0) idx = atomicAdd(&p.ctr[7], 1ull);
        idx = __shfl_sync(0xffffffffu, idx, 0);
        if ((i64)idx >= count) break;
        const i64 s = p.esc[0][idx];
        if (s < 0) continue; /* decided by the lattice stage */
        c.blob = p.blobs + p.set_off[s];
        const i64 tb = p.task_base[s];
        const int st = fast_verdict(tm, c, p.vsm + tb);
        if (st == ST_ESCALATE || st == ST_ESCALATE_RANGE) continue; /* the general stage's */
        if (st != RTGPU_SCHEDULABLE) {
            const int n = (int)c.blob[0];
            for (int i = lane; i < n; i += 32) p.vsm[tb + i] = 0; /* no allocation */
        }
        __syncwarp();
        if (lane == 0) {
            p.status[s] = st;
            p.evals[s] = c.evals;
            p.esc[0][idx] = -1;
        }
        __syncwarp();
    }
}

#ifdef RTGPU_FRONT_TU /* defined only in rtgpu_k_f64.cu */
/* Stage 0: sets [set_base, set_base + n_sets) in FP64 -- the verdict fast
 * path when it applies (RTGPU, verdict only), else the general path. */
__global__ void __launch_bounds__(256, MinBlocks<double>::value) front_kernel(KParams p) {
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    Layout<double> L;
    L.init(p.dims);
    SetCtx<double> c;
    kernel_ctx(c, p.dims, L, warp);
    c.budget = p.budget;
    c.method = p.method;
    WarpTeam tm{lane};
    for (;;) {
        unsigned long long idx = 0;
        if (lane == 0) idx = atomicAdd(p.wctr0, 1ull);
        idx = __shfl_sync(0xffffffffu, idx, 0);
        if ((i64)idx >= p.n_sets) break;
        const i64 s = p.set_base + (i64)idx;
        c.blob = p.blobs + p.set_off[s];
        const i64 tb = p.task_base[s];
        int st;
        if (p.flags & (RTGPU_F_FIRST_I64 | RTGPU_F_FIRST_I128)) {
            st = ST_ESCALATE;
        } else if (p.use_fast) {
            st = fast_verdict(tm, c, p.vsm + tb);
            /* a scale beyond FP64: the general path's per-task scales are
             * cheaper than an int64 fast path (measured) */
            if (st == ST_ESCALATE_RANGE) st = ST_ESCALATE;
            if (st != RTGPU_SCHEDULABLE && st != ST_ESCALATE) {
                const int n = (int)c.blob[0];
                for (int i = lane; i < n; i += 32) p.vsm[tb + i] = 0; /* no allocation */
                __syncwarp();
            }
        } else {
            OutPtrs<double> o;
            o.vsm = p.vsm + tb;
            o.e2e = p.e2e + tb;
            o.den = p.den + tb;
            o.detail = p.detail ? p.detail + p.set_off[s] : nullptr;
            st = analyze_set(tm, c, p.flags, o);
        }
        if (st == ST_ESCALATE) {
            if (lane == 0) {
                unsigned long long pos = atomicAdd(&p.ctr[4], 1ull);
                p.esc[0][pos] = s;
            }
            __syncwarp();
            continue;
        }
        if (lane == 0) {
            p.status[s] = st;
            p.evals[s] = c.evals;
        }
        __syncwarp();
    }
}

/* Wait until the chunk holding set s has arrived (streamed input).  Lane 0
 * polls the chunk's flag, backing off with nanosleep.  The first set of a
 * chunk always takes an acquire load plus an acquire fence: a 128-byte line
 * spanning the chunk boundary may sit in this SM's L1 from the previous
 * chunk's last set, loaded before this chunk's bytes arrived, and the
 * acquire invalidates it.  Lines of any other set lie wholly in its chunk and
 * are never loaded before the chunk's flag is seen. */
__device__ __forceinline__ bool wait_chunk(const KParams &p, i64 s, int lane) {
    /* bounded: a chunk that never arrives (a failed copy) must not hang the
     * GPU -- after ~2^23 polls (seconds) the set is reported undecided */
    int ok = 1;
    if (lane == 0) {
        int c = 0;
        #pragma unroll 1
        for (int st = 16; st > 0; st >>= 1) /* last chunk with chunk_begin[c] <= s */
            if (c + st < p.chunks && p.chunk_begin[c + st] <= s) c += st;
        const bool first = s == p.chunk_begin[c];
        const unsigned long long *f = p.chunk_flag + c;
        unsigned long long v;
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(f) : "memory");
        if (v != p.epoch || first) {
            for (int polls = 0;; polls++) {
                asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(f) : "memory");
                if (v == p.epoch) break;
                unsigned long long a;
                asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(a) : "l"(p.chunk_abort) : "memory");
                if (a == p.epoch || polls > (1 << 22)) {
                    if (a != p.epoch)
                        asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p.chunk_abort), "l"(p.epoch) : "memory");
                    ok = 0;
                    break;
                }
                __nanosleep(256);
            }
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
        }
    }
    return __shfl_sync(0xffffffffu, ok, 0) != 0;
}

/* Stage 0 when the fast path applies (RTGPU, verdict only): the fast path
 * and nothing else, so neither the general path's stack frame and
 * registers nor its code sit in this kernel -- sets it cannot decide go to
 * stage 1's list like the front kernel's escalations. */
#ifndef RTGPU_FAST_MINB
#define RTGPU_FAST_MINB RTGPU_MINB
#endif
template <bool STREAM>
__global__ void __launch_bounds__(256, RTGPU_FAST_MINB) fast_kernel(KParams p) {
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    Layout<double> L;
    L.init(p.dims);
    SetCtx<double> c;
    kernel_ctx(c, p.dims, L, warp);
    c.budget = p.budget;
    c.method = p.method;
    WarpTeam tm{lane};
    for (;;) {
        unsigned long long idx = 0;
        if (lane == 0) idx = atomicAdd(p.wctr0, 1ull);
        idx = __shfl_sync(0xffffffffu, idx, 0);
        if ((i64)idx >= p.n_sets) break;
        const i64 s = p.set_base + (i64)idx;
        if (STREAM) {
            if (!wait_chunk(p, s, lane)) {
                if (lane == 0) p.status[s] = RTGPU_UNDECIDED;
                __syncwarp();
                continue;
            }
            /* the layout was sized from a sample of the batch: a set beyond
             * it goes to the oversize list (esc[2], unused by verdict runs)
             * and the host re-runs it with the batch's true dims */
            const i64 *h = p.blobs + p.set_off[s];
            if (h[0] > p.dims.maxn || h[5] > p.dims.MC || h[6] > p.dims.MP) {
                if (lane == 0) {
                    unsigned long long pos = atomicAdd(&p.ctr[6], 1ull);
                    p.esc[2][pos] = s;
                }
                __syncwarp();
                continue;
            }
        }
        c.blob = p.blobs + p.set_off[s];
        const i64 tb = p.task_base[s];
        int st = fast_verdict(tm, c, p.vsm + tb);
        if (st == ST_ESCALATE_RANGE) st = ST_ESCALATE;
        if (st == ST_ESCALATE) {
            if (lane == 0) {
                unsigned long long pos = atomicAdd(&p.ctr[4], 1ull);
                p.esc[0][pos] = s;
            }
            __syncwarp();
            continue;
        }
        if (st != RTGPU_SCHEDULABLE) {
            const int n = (int)c.blob[0];
            for (int i = lane; i < n; i += 32) p.vsm[tb + i] = 0; /* no allocation */
        }
        if (lane == 0) {
            p.status[s] = st;
            p.evals[s] = c.evals;
        }
        __syncwarp();
    }
}
#endif

/* ------------------------------------------------------------ point queries */

struct QParams {
    const i64 *blobs, *set_off;
    const rtgpu_query *queries;
    i64 n;
    Dims dims;
    int32_t *status;
    i64 *num, *den;
    unsigned long long *ctr;
    i64 *esc0, *esc1;
};

template <class V>
__global__ void __launch_bounds__(256, MinBlocks<V>::value) query_kernel(QParams p, int stage) {
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    Layout<V> L;
    L.init(p.dims);
    SetCtx<V> c;
    c.hbase = nullptr;
    c.o_tr = warp * L.bytes;
    c.o_vc = c.o_tr + L.off_views_c;
    c.o_vm = c.o_tr + L.off_views_m;
    c.o_scr = c.o_tr + L.off_scr;
    c.L = L;
    c.maxn = p.dims.maxn;
    c.MC = p.dims.MC;
    c.MP = p.dims.MP;
    set_groups(c);
    c.budget = 0;
    c.method = RTGPU_METHOD_RTGPU;
    WarpTeam tm{lane};
    const i64 count = stage == 0 ? p.n : (i64)(stage == 1 ? p.ctr[3] : p.ctr[4]);
    const i64 *list = stage == 0 ? nullptr : (stage == 1 ? p.esc0 : p.esc1);
    for (;;) {
        unsigned long long idx = 0;
        if (lane == 0) idx = atomicAdd(&p.ctr[stage], 1ull);
        idx = __shfl_sync(0xffffffffu, idx, 0);
        if ((i64)idx >= count) break;
        const i64 qi = list ? list[idx] : (i64)idx;
        const rtgpu_query qq = p.queries[qi];
        c.blob = p.blobs + p.set_off[qq.set];
        i64 num = RTGPU_NONE, den = 1;
        int st = run_query(tm, c, qq.kind, qq.task, qq.index, qq.horizon, qq.blocking, &num, &den);
        if (st == ST_ESCALATE) {
            if (stage < 2) {
                if (lane == 0) {
                    unsigned long long pos = atomicAdd(&p.ctr[3 + stage], 1ull);
                    (stage == 0 ? p.esc0 : p.esc1)[pos] = qi;
                }
                __syncwarp();
                continue;
            }
            st = RTGPU_RANGE;
        }
        if (lane == 0) {
            p.status[qi] = st;
            p.num[qi] = num;
            p.den[qi] = den;
        }
        __syncwarp();
    }
}

template <class V> inline int launch_query_stage(const QParams &p, int stage, cudaStream_t st);

void set_err(const char *what, cudaError_t e);
void set_err_msg(const char *msg);
void count_launch();

inline int pow2_group(int p) {
    int g = 1;
    while (g < p) g <<= 1;
    return g < 1 ? 1 : (g > 32 ? 32 : g);
}

template <class V> inline int warps_per_block(const Dims &d, int *bytes_out) {
    Layout<V> L;
    L.init(d);
    int wpb = 8;
    while (wpb > 1 && (size_t)L.bytes * wpb > 200 * 1024) wpb >>= 1;
    *bytes_out = L.bytes * wpb;
    return (size_t)L.bytes * wpb > 220 * 1024 ? 0 : wpb;
}

template <class K> inline int launch_persistent(K kernel, const Dims &dims, int wpb_bytes_for, i64 want,
                                                int wpb, int bytes, cudaStream_t st, const char *name,
                                                const KParams &p, int stage, bool front) {
    (void)wpb_bytes_for;
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) {
        set_err("cudaFuncSetAttribute", e);
        return -4;
    }
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, 32 * wpb, bytes);
    if (per_sm < 1) per_sm = 1;
    i64 grid = (i64)sms * per_sm;
    if (want >= 0 && want < grid) grid = want;
    if (grid < 1) grid = 1;
    if (front) ((void (*)(KParams))kernel)<<<(unsigned)grid, 32 * wpb, bytes, st>>>(p);
    else ((void (*)(KParams, int))kernel)<<<(unsigned)grid, 32 * wpb, bytes, st>>>(p, stage);
    count_launch();
    e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_err(name, e);
        return -5;
    }
    return 0;
}

template <class V> inline int launch_stage(const KParams &p, int stage, cudaStream_t st) {
    int bytes = 0;
    int wpb = warps_per_block<V>(p.dims, &bytes);
    if (wpb == 0) {
        set_err_msg("task sets too large for shared memory");
        return -3;
    }
    /* the list length is only known on the device: a persistent grid at
     * full occupancy (a hard set takes one warp ~0.4 ms in the general path,
     * so the stage's time is its longest warp: spread the list over every
     * resident warp; idle warps exit at once) */
    return launch_persistent((void *)analyze_kernel<V>, p.dims, 0, -1, wpb, bytes, st,
                             "analyze_kernel launch", p, stage, false);
}

template <class V> inline int launch_fast_list(const KParams &p, cudaStream_t st) {
    int bytes = 0;
    const int wpb = warps_per_block<V>(p.dims, &bytes);
    if (wpb == 0) return 0; /* the general stage takes the list */
    /* persistent over the list (its length is on the device): a few CTAs
     * suffice, the list is short */
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return launch_persistent((void *)fast_list_kernel<V>, p.dims, 0, (i64)sms, wpb, bytes, st,
                             "fast_list_kernel launch", p, 0, true);
}

#ifdef RTGPU_FRONT_TU
inline int launch_front(const KParams &p, cudaStream_t st) {
    int bytes = 0;
    int wpb = warps_per_block<double>(p.dims, &bytes);
    if (wpb == 0) {
        set_err_msg("task sets too large for shared memory");
        return -3;
    }
    if (p.use_fast && !(p.flags & (RTGPU_F_FIRST_I64 | RTGPU_F_FIRST_I128)))
        return launch_persistent(p.chunk_flag ? (void *)fast_kernel<true> : (void *)fast_kernel<false>, p.dims,
                                 0, (p.n_sets + wpb - 1) / wpb, wpb, bytes, st, "fast_kernel launch", p, 0, true);
    return launch_persistent((void *)front_kernel, p.dims, 0, (p.n_sets + wpb - 1) / wpb, wpb, bytes,
                             st, "front_kernel launch", p, 0, true);
}
#endif

template <class V> inline int launch_query_stage(const QParams &p, int stage, cudaStream_t st) {
    int bytes = 0;
    int wpb = warps_per_block<V>(p.dims, &bytes);
    if (wpb == 0) {
        set_err_msg("task sets too large for shared memory");
        return -3;
    }
    cudaError_t e = cudaFuncSetAttribute(query_kernel<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) {
        set_err("cudaFuncSetAttribute", e);
        return -4;
    }
    i64 grid = stage == 0 ? (p.n + wpb - 1) / wpb : 148;
    if (grid > 148 * 8) grid = 148 * 8;
    if (grid < 1) grid = 1;
    query_kernel<V><<<(unsigned)grid, 32 * wpb, bytes, st>>>(p, stage);
    count_launch();
    e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_err("query_kernel launch", e);
        return -5;
    }
    return 0;
}

int launch_query_f64(const QParams &p, int stage, cudaStream_t st);
int launch_query_i64(const QParams &p, int stage, cudaStream_t st);
int launch_query_i128(const QParams &p, int stage, cudaStream_t st);
int launch_front_f64(const KParams &p, cudaStream_t st);
int launch_stage_f64(const KParams &p, int stage, cudaStream_t st);
int launch_stage_i64(const KParams &p, int stage, cudaStream_t st);
int launch_fast_list_i64(const KParams &p, cudaStream_t st);
int launch_stage_i128(const KParams &p, int stage, cudaStream_t st);
int launch_lattice_front(const KParams &p, cudaStream_t st);
int launch_lattice_list(const KParams &p, cudaStream_t st);

}  // namespace rtgpu
