/*
 * simulator.cu -- batched discrete-event simulation on the GPU
 * (include/rtgpu_sim.h): the reference's gpusched.simulator.simulate
 * (/root/reference/pkg/src/gpusched/simulator.py:160) restated as one GPU
 * thread per simulation over integer (scaled) time.
 *
 * The reference keeps one heap of (time, order, seq, payload).  Here the
 * pending events are kept by kind and the next one is the lexicographic
 * minimum of (time, order, seq):
 *   order 0  finishes: the running CPU segment (one valid finish at a time;
 *            a preempted segment's stale heap entry is never popped as
 *            valid, simulator.py:323), the bus transfer, every job in a GPU
 *            segment -- tie-broken by push sequence number;
 *   order 1  deadlines: at most one per task pending (D <= T, validated);
 *   order 2  releases: task i's next k*T_i < horizon, tie-broken by
 *            priority -- exactly the order of the reference's pre-pushed,
 *            (time, priority)-sorted release points (simulator.py:186).
 * The push counter starts at R (the release pushes) and advances on every
 * deadline and finish push, so equal-time ties resolve as in the heap.
 * Ready queues are insertion-ordered; "stable sort by priority, pop(0)"
 * (simulator.py:222, 249) is "first entry of the best priority".  Uniform
 * lengths are drawn at release time, in plan order, from a per-simulation
 * MT19937 seeded like random.Random(seed) with Python's randint algorithm
 * (simulator.py:122), so traces are bit-identical.
 */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <mutex>
#include <vector>

#include "../../include/rtgpu_sim.h"

namespace {

typedef int64_t i64;

constexpr int JW0 = 12; /* job record: fixed fields before lens[] / segr[] */
/* J_SLOT: the job's output slot (release order); J_DLP: its deadline event
 * is still pending (the record is recycled once done and past it) */
enum { J_TASK = 0, J_K, J_REL, J_DL, J_POS, J_REM, J_DONE, J_GFIN, J_GSEQ, J_S, J_SLOT, J_DLP };

__host__ __device__ inline i64 job_words(int s_max) { return JW0 + 2 * (i64)s_max; }

/* job-record pool: header [8] records (0: one per release point) */
__host__ __device__ inline i64 pool_of(const i64 *b) { return b[8] > 0 && b[8] < b[3] ? b[8] : b[3]; }

__host__ __device__ inline i64 scratch_words(const i64 *b) {
    const i64 P = pool_of(b), smax = b[6];
    /* job records, three queues (cpu, bus, gpu) and the free stack (int32),
     * per-task state (4 x 64), MT19937 state (624 x u32 + index) */
    return P * job_words((int)smax) + 2 * P + 2 + 4 * RTGPU_SIM_MAX_TASKS + 320;
}

/* ------------------------------------------------------------ MT19937 */

struct MT {
    uint32_t *mt;
    int idx;
    __device__ void init_genrand(uint32_t s) {
        mt[0] = s;
        for (int i = 1; i < 624; i++) mt[i] = 1812433253u * (mt[i - 1] ^ (mt[i - 1] >> 30)) + (uint32_t)i;
        idx = 624;
    }
    /* CPython _random init_by_array; key words held one per int64 */
    __device__ void init_by_array(const i64 *key, int n) {
        init_genrand(19650218u);
        int i = 1, j = 0;
        for (int k = n > 624 ? n : 624; k; k--) {
            mt[i] = (mt[i] ^ ((mt[i - 1] ^ (mt[i - 1] >> 30)) * 1664525u)) + (uint32_t)key[j] + (uint32_t)j;
            if (++i >= 624) {
                mt[0] = mt[623];
                i = 1;
            }
            if (++j >= n) j = 0;
        }
        for (int k = 623; k; k--) {
            mt[i] = (mt[i] ^ ((mt[i - 1] ^ (mt[i - 1] >> 30)) * 1566083941u)) - (uint32_t)i;
            if (++i >= 624) {
                mt[0] = mt[623];
                i = 1;
            }
        }
        mt[0] = 0x80000000u;
        idx = 624;
    }
    __device__ uint32_t next() {
        if (idx >= 624) {
            for (int k = 0; k < 624; k++) {
                const uint32_t y = (mt[k] & 0x80000000u) | (mt[k + 1 < 624 ? k + 1 : 0] & 0x7fffffffu);
                mt[k] = mt[k + 397 < 624 ? k + 397 : k + 397 - 624] ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
            }
            idx = 0;
        }
        uint32_t y = mt[idx++];
        y ^= y >> 11;
        y ^= (y << 7) & 0x9d2c5680u;
        y ^= (y << 15) & 0xefc60000u;
        y ^= y >> 18;
        return y;
    }
    /* random.getrandbits(k), 1 <= k <= 64: little-endian 32-bit words, the
     * last one shifted down */
    __device__ uint64_t getrandbits(int k) {
        if (k <= 32) return next() >> (32 - k);
        const uint64_t w0 = next();
        const uint64_t w1 = next() >> (64 - k);
        return w0 | (w1 << 32);
    }
    /* random.randint(a, b) = a + _randbelow(b - a + 1) (rejection sampling
     * on bit_length(n) bits) */
    __device__ i64 randint(i64 a, i64 b) {
        const uint64_t n = (uint64_t)(b - a) + 1;
        int k = 64 - __clzll((long long)n);
        uint64_t r = getrandbits(k);
        while (r >= n) r = getrandbits(k);
        return a + (i64)r;
    }
};

/* ------------------------------------------------------------ simulation */

/* One warp per simulation.  Every lane runs the same (warp-uniform) event
 * loop on the same state -- no divergence -- and the scans are lane-
 * parallel: task t's next release and pending deadline live in the
 * registers of lane t % 32 (two per lane: tasks t and t + 32), the next
 * event is a butterfly min over lanes, ready queues and the GPU set are
 * scanned 32 entries at a time.  Job records live in a recycled pool in
 * global scratch (L1-resident for the live jobs); all lanes store the same
 * values, so each lane reads its own writes without synchronisation. */
constexpr i64 INF = 0x7fffffffffffffffLL;

__device__ __forceinline__ i64 shfl64(i64 v, int m) { return (i64)__shfl_xor_sync(0xffffffffu, (long long)v, m); }

struct Sim {
    const i64 *blob, *tr;
    int n, policy, smax, jw, sstride, lane; /* sstride: seg_max row width */
    i64 H, R, evcap;
    i64 *jobs;
    int *cq, *bq, *gq, *freel;
    int cn, bn, gn, fn;
    bool pool_out;
    /* lane-held state of tasks a = lane and b = lane + 32 */
    i64 TA, TB, DA, DB;      /* period, relative deadline        */
    i64 relA, relB;          /* next release time (INF: none)    */
    i64 kA, kB;              /* next job index                   */
    i64 dlA, dlB, dsA, dsB;  /* pending deadline: time, seq      */
    int djA, djB;            /* its job record (-1: none)        */
    MT rng;
    int cpu_run, bus_run;
    i64 run_fin, run_seq, bus_fin, bus_seq;
    i64 seq, n_jobs, rank, nev, misses;
    bool overflow;
    /* outputs */
    rtgpu_sim_event *ev;
    int32_t *job_task, *job_k, *job_rank;
    i64 *job_resp, *seg_max, *resp_max;

    __device__ i64 *J(int j) const { return jobs + (i64)j * jw; }
    __device__ const i64 *plan(int task, int pos) const {
        return blob + tr[task * RTGPU_SIM_TASK + 4] + (i64)pos * RTGPU_SIM_SEG;
    }
    __device__ int kind_of(const i64 *e) const { return (int)(e[0] & 0xff); }
    __device__ int idx_of(const i64 *e) const { return (int)((e[0] >> 8) & 0xff); }

    __device__ void emit(i64 time, int j, int kind, int seg, int action) {
        if (nev < evcap) {
            if (ev && lane == 0) {
                const i64 *jr = J(j);
                ev[nev].time = time;
                ev[nev].packed = (uint64_t)(uint32_t)jr[J_K] | ((uint64_t)(jr[J_TASK] & 0xff) << 32) |
                                 ((uint64_t)kind << 40) | ((uint64_t)action << 44) |
                                 ((uint64_t)((seg + 1) & 0xff) << 48);
            }
        } else {
            overflow = true;
        }
        nev++;
    }
    __device__ i64 &seg_start(int j, int pos) { return J(j)[JW0 + smax + pos]; }

    /* first index of the best priority (lowest task index) in a queue:
     * warp min of (task, position) */
    __device__ int best_in(const int *q, int cnt) const {
        int best = 0x7fffffff;
        for (int x = lane; x < cnt; x += 32) {
            const int key = ((int)J(q[x])[J_TASK] << 20) | x;
            best = key < best ? key : best;
        }
        for (int m = 16; m; m >>= 1) {
            const int o = __shfl_xor_sync(0xffffffffu, best, m);
            best = o < best ? o : best;
        }
        return best & 0xfffff;
    }
    /* order-preserving removal (ties among one task's jobs keep FIFO order) */
    __device__ void remove_at(int *q, int &cnt, int at) const {
        for (int base = at; base + 1 < cnt; base += 32) {
            const int x = base + lane;
            const int v = x + 1 < cnt ? q[x + 1] : 0;
            __syncwarp();
            if (x + 1 < cnt) q[x] = v;
            __syncwarp();
        }
        cnt--;
    }

    __device__ void start_cpu(i64 time, int j, bool resumed) {
        __syncwarp();
        i64 *jr = J(j);
        cpu_run = j;
        const i64 *e = plan((int)jr[J_TASK], (int)jr[J_POS]);
        emit(time, j, RTGPU_KIND_CPU, idx_of(e), resumed ? RTGPU_EV_RESUME : RTGPU_EV_START);
        if (!resumed && seg_start(j, (int)jr[J_POS]) < 0) seg_start(j, (int)jr[J_POS]) = time;
        run_fin = time + jr[J_REM];
        run_seq = seq++;
    }

    __device__ i64 cur_dur(int j) const {
        const i64 *jr = J(j);
        return jr[JW0 + jr[J_POS]];
    }

    __device__ void sched_cpu(i64 time) {
        if (cn == 0) return;
        const int t = best_in(cq, cn);
        const int top = cq[t];
        if (cpu_run < 0) {
            remove_at(cq, cn, t);
            start_cpu(time, top, J(top)[J_REM] != cur_dur(top));
        } else if (J(top)[J_TASK] < J(cpu_run)[J_TASK]) {
            const int v = cpu_run;
            i64 *vr = J(v);
            __syncwarp();
            vr[J_REM] = run_fin - time;
            emit(time, v, RTGPU_KIND_CPU, idx_of(plan((int)vr[J_TASK], (int)vr[J_POS])), RTGPU_EV_PREEMPT);
            __syncwarp();
            cq[cn++] = v;
            __syncwarp();
            remove_at(cq, cn, t);
            cpu_run = -1;
            start_cpu(time, top, J(top)[J_REM] != cur_dur(top));
        }
    }

    __device__ void grant_bus(i64 time) {
        if (bus_run >= 0 || bn == 0) return;
        const int t = best_in(bq, bn);
        const int j = bq[t];
        remove_at(bq, bn, t);
        bus_run = j;
        i64 *jr = J(j);
        emit(time, j, RTGPU_KIND_MEM, idx_of(plan((int)jr[J_TASK], (int)jr[J_POS])), RTGPU_EV_START);
        if (seg_start(j, (int)jr[J_POS]) < 0) seg_start(j, (int)jr[J_POS]) = time;
        bus_fin = time + cur_dur(j);
        bus_seq = seq++;
    }

    __device__ void dispatch(i64 time, int j) {
        __syncwarp();
        i64 *jr = J(j);
        const int pos = (int)jr[J_POS];
        const i64 *e = plan((int)jr[J_TASK], pos);
        const int kind = kind_of(e);
        if (kind == RTGPU_KIND_CPU) {
            jr[J_REM] = cur_dur(j);
            __syncwarp();
            cq[cn++] = j;
            __syncwarp();
            sched_cpu(time);
        } else if (kind == RTGPU_KIND_MEM) {
            __syncwarp();
            bq[bn++] = j;
            __syncwarp();
            grant_bus(time);
        } else { /* dedicated virtual SMs: starts at once */
            emit(time, j, RTGPU_KIND_GPU, idx_of(e), RTGPU_EV_START);
            if (seg_start(j, pos) < 0) seg_start(j, pos) = time;
            jr[J_GFIN] = time + cur_dur(j);
            jr[J_GSEQ] = seq++;
            __syncwarp();
            gq[gn++] = j;
            __syncwarp();
        }
    }

    __device__ void advance(i64 time, int j) {
        __syncwarp();
        i64 *jr = J(j);
        const int task = (int)jr[J_TASK];
        const int pos = (int)jr[J_POS];
        const i64 *e = plan(task, pos);
        emit(time, j, kind_of(e), idx_of(e), RTGPU_EV_FINISH);
        const i64 st0 = seg_start(j, pos);
        __syncwarp(); /* every lane has read the record before any rewrites it */
        seg_start(j, pos) = time - st0; /* start -> finish response */
        jr[J_POS] = pos + 1;
        if (pos + 1 == (int)jr[J_S]) {
            jr[J_DONE] = 1;
            const i64 resp = time - jr[J_REL];
            if (lane == 0) {
                job_resp[jr[J_SLOT]] = resp;
                job_rank[jr[J_SLOT]] = (int32_t)rank;
            }
            rank++;
            if (time > jr[J_DL]) {
                emit(time, j, RTGPU_KIND_JOB, -1, RTGPU_EV_DEADLINE_MISS);
                misses++;
            }
            __syncwarp();
            i64 *sm = seg_max + (i64)task * sstride;
            for (int p = lane; p < (int)jr[J_S]; p += 32) {
                const i64 v = seg_start(j, p);
                if (v > sm[p]) sm[p] = v;
            }
            if (lane == 0 && resp > resp_max[task]) resp_max[task] = resp;
            __syncwarp();
            if (!jr[J_DLP]) {
                freel[fn++] = j;
                __syncwarp();
            }
        } else {
            dispatch(time, j);
        }
    }

    __device__ void release(i64 time, int task) {
        const i64 *t = tr + task * RTGPU_SIM_TASK;
        if (fn == 0) { /* more live jobs than the pool holds: the host re-runs */
            pool_out = true;
            return;
        }
        const int j = freel[--fn];
        const i64 slot = n_jobs++;
        i64 *jr = J(j);
        const int S = (int)t[0];
        const bool mine = lane == (task & 31), hi = task >= 32;
        const i64 k = hi ? kB : kA; /* valid in the owning lane */
        const i64 kk = (i64)__shfl_sync(0xffffffffu, (long long)k, task & 31);
        if (mine) {
            if (hi) {
                kB++;
                relB = kB * TB < H ? kB * TB : INF;
            } else {
                kA++;
                relA = kA * TA < H ? kA * TA : INF;
            }
        }
        jr[J_SLOT] = slot;
        jr[J_DLP] = 1;
        jr[J_TASK] = task;
        jr[J_K] = kk;
        jr[J_REL] = time;
        jr[J_DL] = time + t[2];
        jr[J_POS] = 0;
        jr[J_REM] = 0;
        jr[J_DONE] = 0;
        jr[J_S] = S;
        __syncwarp();
        for (int p = lane; p < S; p += 32) { /* fixed lengths, in parallel */
            jr[JW0 + p] = plan(task, p)[3];
            seg_start(j, p) = -1;
        }
        __syncwarp();
        if (policy == 1) /* draws in plan order, one stream, lane 0's generator */
            for (int p = 0; p < S; p++) {
                const i64 *e = plan(task, p);
                if ((e[0] >> 16) & 1) {
                    i64 d = 0;
                    if (lane == 0) d = rng.randint(e[1], e[2]) * e[4] + e[5];
                    d = (i64)__shfl_sync(0xffffffffu, (long long)d, 0);
                    jr[JW0 + p] = d;
                }
            }
        __syncwarp();
        if (lane == 0) {
            job_task[slot] = task;
            job_k[slot] = (int32_t)kk;
            job_resp[slot] = -1;
            job_rank[slot] = -1;
        }
        emit(time, j, RTGPU_KIND_JOB, -1, RTGPU_EV_RELEASE);
        const i64 dseq = seq++;
        if (mine) {
            if (hi) {
                dlB = jr[J_DL];
                dsB = dseq;
                djB = j;
            } else {
                dlA = jr[J_DL];
                dsA = dseq;
                djA = j;
            }
        }
        dispatch(time, j);
    }

    __device__ void run() {
        for (;;) {
            /* next event: lexicographic min of (time, order << 58 | seq) over
             * lanes (GPU finishes, deadlines, releases), then the CPU and bus
             * finishes every lane holds */
            i64 bt = INF, bk = INF;
            int bp = -1; /* type << 16 | arg */
            auto consider = [&](i64 t, i64 key, int p) {
                if (t < bt || (t == bt && key < bk)) {
                    bt = t;
                    bk = key;
                    bp = p;
                }
            };
            for (int x = lane; x < gn; x += 32) {
                const i64 *jr = J(gq[x]);
                consider(jr[J_GFIN], jr[J_GSEQ], (2 << 16) | x);
            }
            if (lane < n) {
                if (djA >= 0) consider(dlA, ((i64)1 << 58) | dsA, (3 << 16) | lane);
                if (relA != INF) consider(relA, ((i64)2 << 58) | lane, (4 << 16) | lane);
            }
            if (lane + 32 < n) {
                if (djB >= 0) consider(dlB, ((i64)1 << 58) | dsB, (3 << 16) | (lane + 32));
                if (relB != INF) consider(relB, ((i64)2 << 58) | (lane + 32), (4 << 16) | (lane + 32));
            }
            for (int m = 16; m; m >>= 1) {
                const i64 t2 = shfl64(bt, m), k2 = shfl64(bk, m);
                const int p2 = __shfl_xor_sync(0xffffffffu, bp, m);
                if (t2 < bt || (t2 == bt && k2 < bk)) {
                    bt = t2;
                    bk = k2;
                    bp = p2;
                }
            }
            if (cpu_run >= 0) consider(run_fin, run_seq, 0);
            if (bus_run >= 0) consider(bus_fin, bus_seq, 1 << 16);
            if (bp < 0 || bt > H) break;
            const int type = bp >> 16, arg = bp & 0xffff;
            if (type == 0) {
                const int j = cpu_run;
                cpu_run = -1;
                advance(bt, j);
                sched_cpu(bt);
            } else if (type == 1) {
                const int j = bus_run;
                bus_run = -1;
                advance(bt, j);
                grant_bus(bt);
            } else if (type == 2) {
                const int j = gq[arg];
                __syncwarp();
                gq[arg] = gq[gn - 1]; /* the GPU set is unordered: ties use seq */
                gn--;
                __syncwarp();
                advance(bt, j);
            } else if (type == 3) {
                const bool hi = arg >= 32;
                const int j = __shfl_sync(0xffffffffu, hi ? djB : djA, arg & 31);
                if (lane == (arg & 31)) {
                    if (hi) djB = -1;
                    else djA = -1;
                }
                J(j)[J_DLP] = 0;
                if (!J(j)[J_DONE]) {
                    emit(bt, j, RTGPU_KIND_JOB, -1, RTGPU_EV_DEADLINE_MISS);
                    misses++;
                } else {
                    __syncwarp();
                    freel[fn++] = j;
                    __syncwarp();
                }
            } else {
                release(bt, arg);
                if (pool_out) break;
            }
        }
    }
};

/* One single-warp block per simulation: the block scheduler hands blocks to
 * SMs as they free up, so with `order` = longest-first (the host's estimate
 * from release points x plan length) the batch is list-scheduled and the
 * longest simulations do not start last. */
__global__ void __launch_bounds__(32) sim_kernel(const i64 *blobs, const i64 *set_off, i64 n_sims,
                                                 const i64 *job_base, const i64 *task_base,
                                                 const i64 *ev_base, const i64 *scr_off, i64 *scratch,
                                                 const i64 *order, int s_max_out, rtgpu_sim_out o) {
    const int lane = threadIdx.x & 31;
    {
        const i64 s = order ? order[blockIdx.x] : (i64)blockIdx.x;
        const i64 *b = blobs + set_off[s];
        Sim m;
        m.lane = lane;
        m.blob = b;
        m.n = (int)b[0];
        m.policy = (int)b[1];
        m.H = b[2];
        m.R = b[3];
        m.evcap = b[4];
        m.smax = (int)b[6];
        m.jw = (int)job_words(m.smax);
        m.tr = b + RTGPU_SIM_HDR;
        const i64 tb = task_base[s], jb = job_base[s];
        int st = RTGPU_SIM_OK;
        if (m.n < 0 || m.n > RTGPU_SIM_MAX_TASKS || m.smax > s_max_out || m.R != job_base[s + 1] - jb ||
            task_base[s + 1] - tb != m.n || (m.policy == 1 && (b[5] < 1 || b[5] > RTGPU_SIM_MAX_KEY)))
            st = RTGPU_SIM_BAD_INPUT;
        if (st != RTGPU_SIM_OK) {
            if (lane == 0) {
                o.n_events[s] = 0;
                o.misses[s] = 0;
                o.status[s] = st;
            }
            return;
        }
        const i64 P = pool_of(b);
        i64 *w = scratch + scr_off[s];
        m.jobs = w;
        w += P * m.jw;
        m.cq = (int *)w;
        m.bq = m.cq + P;
        m.gq = m.bq + P;
        m.freel = m.gq + P;
        w += 2 * P + 2;
        for (i64 x = lane; x < P; x += 32) m.freel[x] = (int)(P - 1 - x);
        m.fn = (int)P;
        m.pool_out = false;
        w += 4 * RTGPU_SIM_MAX_TASKS;
        m.rng.mt = (uint32_t *)w;
        if (m.policy == 1 && lane == 0) m.rng.init_by_array(b + b[7], (int)b[5]);
        __syncwarp();
        const int ta = lane, tbb = lane + 32;
        m.TA = ta < m.n ? m.tr[ta * RTGPU_SIM_TASK + 1] : 1;
        m.DA = ta < m.n ? m.tr[ta * RTGPU_SIM_TASK + 2] : 0;
        m.TB = tbb < m.n ? m.tr[tbb * RTGPU_SIM_TASK + 1] : 1;
        m.DB = tbb < m.n ? m.tr[tbb * RTGPU_SIM_TASK + 2] : 0;
        m.kA = m.kB = 0;
        m.relA = (ta < m.n && 0 < m.H) ? 0 : INF;
        m.relB = (tbb < m.n && 0 < m.H) ? 0 : INF;
        m.djA = m.djB = -1;
        m.dlA = m.dlB = m.dsA = m.dsB = 0;
        for (int i = lane; i < m.n; i += 32) {
            o.resp_max[tb + i] = -1;
            for (int p = 0; p < s_max_out; p++) o.seg_max[(tb + i) * s_max_out + p] = -1;
        }
        __syncwarp();
        m.cn = m.bn = m.gn = 0;
        m.cpu_run = m.bus_run = -1;
        m.run_fin = m.run_seq = m.bus_fin = m.bus_seq = 0;
        m.seq = m.R; /* the reference pushes every release point first */
        m.n_jobs = m.rank = m.nev = m.misses = 0;
        m.overflow = false;
        m.ev = o.events ? o.events + ev_base[s] : nullptr;
        m.job_task = o.job_task + jb;
        m.job_k = o.job_k + jb;
        m.job_rank = o.job_rank + jb;
        m.job_resp = o.job_resp + jb;
        m.seg_max = o.seg_max + tb * s_max_out;
        m.sstride = s_max_out;
        m.resp_max = o.resp_max + tb;
        m.run();
        __syncwarp();
        if (lane == 0) {
            o.status[s] = m.pool_out ? RTGPU_SIM_POOL_OVERFLOW
                                     : (m.overflow ? RTGPU_SIM_EVENT_OVERFLOW : RTGPU_SIM_OK);
            o.n_events[s] = m.nev;
            o.misses[s] = m.misses;
        }
    }
}

char g_err[256] = "";
std::mutex g_mu;

int launch(const i64 *blobs, const i64 *set_off, i64 n_sims, const i64 *job_base, const i64 *task_base,
           const i64 *ev_base, const i64 *scr_off, i64 *scratch, const i64 *order, int s_max,
           const rtgpu_sim_out &o, cudaStream_t st) {
    if (n_sims <= 0) return 0;
    if (n_sims > 0x7fffffffLL) {
        snprintf(g_err, sizeof g_err, "too many simulations in one launch");
        return -3;
    }
    sim_kernel<<<(unsigned)n_sims, 32, 0, st>>>(blobs, set_off, n_sims, job_base, task_base, ev_base, scr_off,
                                               scratch, order, s_max, o);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        snprintf(g_err, sizeof g_err, "sim_kernel launch: %s", cudaGetErrorString(e));
        return -5;
    }
    return 0;
}

}  // namespace

extern "C" {

const char *rtgpu_sim_last_error(void) { return g_err; }

int64_t rtgpu_sim_scratch_words(const int64_t *blob) { return scratch_words((const i64 *)blob); }

int rtgpu_sim_device(const int64_t *blobs, const int64_t *set_off, int64_t n_sims, const int64_t *job_base,
                     const int64_t *task_base, const int64_t *ev_base, const int64_t *scr_off,
                     int64_t *scratch, const int64_t *order, int32_t s_max, const rtgpu_sim_out *out,
                     void *stream) {
    return launch((const i64 *)blobs, (const i64 *)set_off, n_sims, (const i64 *)job_base,
                  (const i64 *)task_base, (const i64 *)ev_base, (const i64 *)scr_off, (i64 *)scratch,
                  (const i64 *)order, s_max, *out, (cudaStream_t)stream);
}

int rtgpu_sim_host(const int64_t *blobs, const int64_t *set_off, int64_t n_sims, const int64_t *job_base,
                   const int64_t *task_base, const int64_t *ev_base, int32_t s_max, rtgpu_sim_out *out) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (n_sims <= 0) return 0;
    const i64 W = set_off[n_sims], NJ = job_base[n_sims], NT = task_base[n_sims];
    const i64 NE = (out->events && ev_base) ? ev_base[n_sims] : 0;
    std::vector<i64> scr(n_sims + 1, 0), order(n_sims);
    for (i64 s = 0; s < n_sims; s++) scr[s + 1] = scr[s] + scratch_words((const i64 *)blobs + set_off[s]);
    for (i64 s = 0; s < n_sims; s++) order[s] = s;
    std::stable_sort(order.begin(), order.end(), [&](i64 a, i64 b) {
        return blobs[set_off[a] + 4] > blobs[set_off[b] + 4]; /* event capacity: longest first */
    });
    struct Buf {
        void *p = nullptr;
        ~Buf() { cudaFree(p); }
    } d_blob, d_off, d_jb, d_tb, d_eb, d_scro, d_scr, d_out, d_ord;
    const size_t n1 = (size_t)(n_sims + 1) * 8;
    size_t out_bytes = 0;
    const size_t o_status = out_bytes;
    out_bytes += (size_t)n_sims * 4 + 4;
    const size_t o_nev = (out_bytes = (out_bytes + 7) & ~(size_t)7);
    out_bytes += (size_t)n_sims * 8;
    const size_t o_miss = out_bytes;
    out_bytes += (size_t)n_sims * 8;
    const size_t o_jt = out_bytes;
    out_bytes += (size_t)NJ * 4 + 4;
    const size_t o_jk = (out_bytes = (out_bytes + 7) & ~(size_t)7);
    out_bytes += (size_t)NJ * 4 + 4;
    const size_t o_jr = (out_bytes = (out_bytes + 7) & ~(size_t)7);
    out_bytes += (size_t)NJ * 8;
    const size_t o_jrank = out_bytes;
    out_bytes += (size_t)NJ * 4 + 4;
    const size_t o_sm = (out_bytes = (out_bytes + 7) & ~(size_t)7);
    out_bytes += (size_t)NT * s_max * 8;
    const size_t o_rm = out_bytes;
    out_bytes += (size_t)NT * 8;
    const size_t o_ev = out_bytes;
    out_bytes += (size_t)NE * sizeof(rtgpu_sim_event);
    if (cudaMalloc(&d_blob.p, (size_t)W * 8 + 8) || cudaMalloc(&d_off.p, n1) || cudaMalloc(&d_jb.p, n1) ||
        cudaMalloc(&d_tb.p, n1) || cudaMalloc(&d_eb.p, n1) || cudaMalloc(&d_scro.p, n1) ||
        cudaMalloc(&d_scr.p, (size_t)scr[n_sims] * 8 + 8) || cudaMalloc(&d_out.p, out_bytes + 8) ||
        cudaMalloc(&d_ord.p, (size_t)n_sims * 8)) {
        snprintf(g_err, sizeof g_err, "cudaMalloc: %s", cudaGetErrorString(cudaGetLastError()));
        return -6;
    }
    cudaMemcpy(d_blob.p, blobs, (size_t)W * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(d_off.p, set_off, n1, cudaMemcpyHostToDevice);
    cudaMemcpy(d_jb.p, job_base, n1, cudaMemcpyHostToDevice);
    cudaMemcpy(d_tb.p, task_base, n1, cudaMemcpyHostToDevice);
    if (NE) cudaMemcpy(d_eb.p, ev_base, n1, cudaMemcpyHostToDevice);
    cudaMemcpy(d_scro.p, scr.data(), n1, cudaMemcpyHostToDevice);
    cudaMemcpy(d_ord.p, order.data(), (size_t)n_sims * 8, cudaMemcpyHostToDevice);
    char *ob = (char *)d_out.p;
    rtgpu_sim_out d;
    d.status = (int32_t *)(ob + o_status);
    d.n_events = (int64_t *)(ob + o_nev);
    d.misses = (int64_t *)(ob + o_miss);
    d.job_task = (int32_t *)(ob + o_jt);
    d.job_k = (int32_t *)(ob + o_jk);
    d.job_resp = (int64_t *)(ob + o_jr);
    d.job_rank = (int32_t *)(ob + o_jrank);
    d.seg_max = (int64_t *)(ob + o_sm);
    d.resp_max = (int64_t *)(ob + o_rm);
    d.events = NE ? (rtgpu_sim_event *)(ob + o_ev) : nullptr;
    int rc = launch((const i64 *)d_blob.p, (const i64 *)d_off.p, n_sims, (const i64 *)d_jb.p,
                    (const i64 *)d_tb.p, NE ? (const i64 *)d_eb.p : nullptr, (const i64 *)d_scro.p,
                    (i64 *)d_scr.p, (const i64 *)d_ord.p, s_max, d, 0);
    if (rc) return rc;
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        snprintf(g_err, sizeof g_err, "sim_kernel: %s", cudaGetErrorString(e));
        return -7;
    }
    cudaMemcpy(out->status, d.status, (size_t)n_sims * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(out->n_events, d.n_events, (size_t)n_sims * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(out->misses, d.misses, (size_t)n_sims * 8, cudaMemcpyDeviceToHost);
    if (NJ) {
        cudaMemcpy(out->job_task, d.job_task, (size_t)NJ * 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(out->job_k, d.job_k, (size_t)NJ * 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(out->job_resp, d.job_resp, (size_t)NJ * 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(out->job_rank, d.job_rank, (size_t)NJ * 4, cudaMemcpyDeviceToHost);
    }
    if (NT) {
        cudaMemcpy(out->seg_max, d.seg_max, (size_t)NT * s_max * 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(out->resp_max, d.resp_max, (size_t)NT * 8, cudaMemcpyDeviceToHost);
    }
    if (NE) cudaMemcpy(out->events, d.events, (size_t)NE * sizeof(rtgpu_sim_event), cudaMemcpyDeviceToHost);
    e = cudaGetLastError();
    if (e != cudaSuccess) {
        snprintf(g_err, sizeof g_err, "copy: %s", cudaGetErrorString(e));
        return -8;
    }
    return 0;
}

}  // extern "C"
