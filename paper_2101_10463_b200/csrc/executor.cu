/*
 * executor.cu -- the paper's accelerator mechanism on a B200: a
 * persistent-thread, %smid-pinned virtual-SM executor (RTGPU section 4,
 * Algorithm 1), with a host runtime that releases periodic jobs of
 * CPU / memory-copy / GPU segments and measures response times so they can
 * be checked against the analysis bounds (reference simulator.py plays this
 * role in software).
 *
 * Kernel.  Every GPU segment is one launch of `persistent_segment` with a
 * grid covering every SM several times.  A block reads %smid and exits at
 * once unless the SM belongs to the task's partition; on a partition SM the
 * first `slots` blocks to arrive stay (slots = 2: the two virtual SMs of one
 * physical SM interleave, paper section 4.3) and pull work items from a
 * global counter until the segment's work is done.  Blocks are small (128
 * threads, no shared memory) so exiting blocks of other tasks always find
 * room on an occupied SM and cannot delay a partition.
 */
#include <cuda.h> /* types of the driver entry point fetched at run time */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <dirent.h>
#include <pthread.h>
#include <stdlib.h>
#include <sched.h>
#include <time.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <mutex>
#include <set>
#include <thread>
#include <vector>

#include "../../include/rtgpu_exec.h"

namespace {

__device__ __forceinline__ unsigned smid() {
    unsigned r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}

/* per-lane control block, cleared by one memset before every launch */
struct Ctl {
    unsigned slots[256];          /* per-SM slot counters                       */
    unsigned long long work;      /* work-item counter                          */
    unsigned long long inv_start; /* ~(first participating block's start), max  */
    unsigned long long end;       /* last participating block's end, max        */
    unsigned long long last_start;/* last participating block's start           */
    unsigned trace_n;             /* participating blocks traced                */
    unsigned pad;
    unsigned bitems[16];          /* items of the first 16 participating blocks */
    unsigned long long cyc0, ns0; /* block 0 of the participants: SM clock and */
    unsigned long long cyc1, ns1; /* global time at its start and end           */
    unsigned smsp[256];           /* per SM: participating warps per SM sub-
                                   * partition (%warpid % 4), 8 bits each       */
};

struct SegArgs {
    uint32_t mask[RTGPU_EXEC_MASK_WORDS]; /* partition, by value (no H2D per launch) */
    Ctl *ctl;
    long long items;
    int iters;
    int nslots;
    float *sink;
    unsigned *trace; /* optional: SM of every participating block */
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

/* work-item claim in the global state space: a generic-address atomic on
 * sm_100 compiles to ATOM + a shared-window fallback whose branch waits for
 * the result, putting the round trip on the critical path */
__device__ __forceinline__ unsigned long long claim(unsigned long long *p) {
    unsigned long long r;
    asm volatile("atom.global.add.u64 %0, [%1], 1;"
                 : "=l"(r)
                 : "l"(__cvta_generic_to_global(p))
                 : "memory");
    return r;
}

__device__ __forceinline__ void gmax(unsigned long long *p, unsigned long long v) {
    asm volatile("red.global.max.u64 [%0], %1;" ::"l"(__cvta_generic_to_global(p)), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned gadd32(unsigned *p, unsigned v) {
    unsigned r;
    asm volatile("atom.global.add.u32 %0, [%1], %2;" : "=r"(r) : "l"(__cvta_generic_to_global(p)), "r"(v) : "memory");
    return r;
}

/* Blocks outside the partition read %smid and exit without touching memory:
 * a launch's other ~6*148 blocks land on every SM, including other tasks'
 * partitions, and must not steal their issue slots. */
__global__ void __launch_bounds__(128) persistent_segment(SegArgs a) {
    __shared__ unsigned slot;
    const unsigned sm = smid();
    if (!((a.mask[sm >> 5] >> (sm & 31)) & 1u)) return;
    const unsigned long long t_in = gtimer();
    if (threadIdx.x == 0) slot = gadd32(&a.ctl->slots[sm], 1u);
    __syncthreads();
    if (slot >= (unsigned)a.nslots) return;
    __shared__ unsigned tpos;
    if (threadIdx.x == 0) {
        gmax(&a.ctl->inv_start, ~t_in);
        gmax(&a.ctl->last_start, t_in);
        tpos = gadd32(&a.ctl->trace_n, 1u);
        if (a.trace && tpos < 4096) a.trace[tpos] = sm;
        if (tpos == 0) {
            a.ctl->cyc0 = clock64();
            a.ctl->ns0 = gtimer();
        }
    }
    /* synthetic compute work: three dependent FMA chains per thread, so one
     * block (one warp per SM sub-partition) keeps the FMA pipe ~3/4 busy and
     * the second slot's block fills the rest: interleave ratio
     * alpha = 2 t2 / t1 ~ 1.3-1.5, inside the model's [1, 1.8] (model.py:17).
     * Every WARP claims its own work items (a segment's `items` are block
     * items of blockDim/32 warp items each): no block-wide barrier per item,
     * so a warp slowed by an unlucky sub-partition placement (the warp slots
     * exiting blocks of other grids leave behind) costs only its own share
     * and the others absorb the rest.  The next item is claimed before the
     * current one is computed and only consumed after it, so the atomic's
     * round trip never sits on the critical path. */
    const int lane = threadIdx.x & 31;
    if (lane == 0) {
        unsigned wid;
        asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
        gadd32(&a.ctl->smsp[sm & 255], 1u << (8 * (wid & 3)));
    }
    const long long witems = a.items * (long long)(blockDim.x >> 5);
    float x0 = threadIdx.x, x1 = x0 + 1.f, x2 = x0 + 2.f;
    /* two claims in flight: a claim is consumed two items after it was
     * issued, so an atomic delayed by copy traffic at the L2 (up to two
     * items of compute) does not stall the warp */
    unsigned long long it = 0, nx = 0;
    if (lane == 0) {
        it = claim(&a.ctl->work);
        nx = claim(&a.ctl->work);
    }
    it = __shfl_sync(0xffffffffu, it, 0);
    unsigned done = 0;
    while ((long long)it < witems) {
        done++;
        unsigned long long nn = 0;
        if (lane == 0) nn = claim(&a.ctl->work); /* in flight for two items */
        const int iters = a.iters;
#pragma unroll 4
        for (int k = 0; k < iters; k++) {
            x0 = fmaf(x0, 0.9999999f, 0.5f);
            x1 = fmaf(x1, 0.9999999f, 0.5f);
            x2 = fmaf(x2, 0.9999999f, 0.5f);
        }
        it = __shfl_sync(0xffffffffu, nx, 0);
        nx = nn;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        gmax(&a.ctl->end, gtimer());
        if (tpos < 16) a.ctl->bitems[tpos] = done;
        if (tpos == 0) {
            a.ctl->cyc1 = clock64();
            a.ctl->ns1 = gtimer();
        }
    }
    if (x0 + x1 + x2 == 12345.f) a.sink[blockIdx.x] = x0;
}

/* Stall sentinel: one thread on an SM no partition uses reads %globaltimer
 * every ~2 us for the whole run and logs every gap above `thresh_ns` -- the
 * intervals in which that SM (with the rest of the GPU, if the pause is
 * GPU-wide) did not execute.  Every other block exits at once. */
struct StallGap {
    unsigned long long a, b;
};

__global__ void stall_sentinel(unsigned target_sm, const volatile int *stop, int *claim, StallGap *gaps,
                               unsigned *ngaps, unsigned cap, unsigned long long thresh_ns,
                               unsigned long long max_ns) {
    if (smid() != target_sm || threadIdx.x != 0) return;
    if (atomicCAS(claim, 0, 1) != 0) return;
    unsigned long long prev = gtimer();
    const unsigned long long t_end = prev + max_ns; /* never outlives the run by much */
    for (unsigned it = 0;; it++) {
        if ((it & 63) == 0 && (*stop || prev > t_end)) break;
        __nanosleep(2000);
        const unsigned long long now = gtimer();
        if (now - prev > thresh_ns) {
            const unsigned k = atomicAdd(ngaps, 1u);
            if (k < cap) gaps[k] = StallGap{prev, now};
        }
        prev = now;
    }
}

char g_err[256] = "";

/* every kernel launch of the last rtgpu_exec_run: task, segment, first
 * participating block's start (%globaltimer ns), span (us), fewest / most
 * items of a traced warp, SM clock -- read by rtgpu_exec_launch_log */
struct LaunchRec {
    int task, seg;
    unsigned long long t0_ns;
    double span_us;
    int items_min, items_max;
    double mhz;
};
std::mutex g_log_mu;
std::vector<LaunchRec> g_log;
std::vector<StallGap> g_stalls; /* the last run's sentinel gaps */
int g_sentinel_sm = -1;         /* the SM it ran on, -1 = none free */

constexpr int RING = 16; /* control blocks / event pairs per lane: one per kernel of a job */

struct Lane {
    cudaStream_t st = nullptr;
    Ctl *ring = nullptr;  /* device control blocks, one per kernel segment of a job */
    Ctl *hring = nullptr; /* pinned host copies, read back after the job */
    Ctl *ctl = nullptr;   /* the control block of the next launch */
    Ctl *hctl = nullptr;
    float *sink = nullptr;
    unsigned *trace = nullptr;
    void *hbuf = nullptr, *dbuf = nullptr;
    size_t buf = 0;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    cudaEvent_t k0[RING] = {}, k1[RING] = {};
    cudaEvent_t ev_wait = nullptr; /* blocking-sync: a waiting thread sleeps */
    bool spin = false;             /* waits poll instead of sleeping (own core) */
    /* completion flag: the stream writes `seq` into pinned host memory
     * (cuStreamWriteValue32), so a polling thread makes no CUDA call --
     * polling cudaEventQuery from several threads contends on the driver
     * lock and delays the other tasks' launches */
    volatile uint32_t *hflag = nullptr;
    CUdeviceptr dflag = 0;
    uint32_t seq = 0;
    void use(int k) {
        ctl = ring + k;
        hctl = hring + k;
    }
};

int sm_count() {
    int dev = 0, n = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
}

typedef CUresult (*WriteValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

WriteValue32 write_value32() {
    static WriteValue32 fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (WriteValue32)p;
        cudaGetLastError();
    }
    return fn;
}

int lane_init(Lane &L, size_t buf) {
    if (cudaStreamCreateWithFlags(&L.st, cudaStreamNonBlocking) != cudaSuccess) return -1;
    if (cudaMalloc(&L.ring, RING * sizeof(Ctl)) != cudaSuccess) return -1;
    if (cudaMallocHost(&L.hring, RING * sizeof(Ctl)) != cudaSuccess) return -1;
    L.use(0);
    if (cudaMalloc(&L.sink, 8192 * sizeof(float)) != cudaSuccess) return -1;
    if (cudaMalloc(&L.trace, 4096 * sizeof(unsigned)) != cudaSuccess) return -1;
    L.buf = buf < 64 ? 64 : buf;
    if (cudaMallocHost(&L.hbuf, L.buf) != cudaSuccess) return -1;
    if (cudaMalloc(&L.dbuf, L.buf) != cudaSuccess) return -1;
    memset(L.hbuf, 1, L.buf);
    cudaEventCreate(&L.e0);
    cudaEventCreate(&L.e1);
    for (int k = 0; k < RING; k++) {
        cudaEventCreate(&L.k0[k]);
        cudaEventCreate(&L.k1[k]);
    }
    cudaEventCreateWithFlags(&L.ev_wait, cudaEventBlockingSync | cudaEventDisableTiming);
    void *hf = nullptr;
    if (write_value32() && cudaHostAlloc(&hf, 64, cudaHostAllocMapped) == cudaSuccess) {
        void *df = nullptr;
        if (cudaHostGetDevicePointer(&df, hf, 0) == cudaSuccess) {
            L.hflag = (volatile uint32_t *)hf;
            *L.hflag = 0;
            L.dflag = (CUdeviceptr)df;
        } else {
            cudaFreeHost(hf);
        }
    }
    cudaGetLastError();
    return 0;
}

void lane_free(Lane &L) {
    if (L.st) cudaStreamDestroy(L.st);
    cudaFree(L.ring);
    cudaFreeHost(L.hring);
    cudaFree(L.sink);
    cudaFree(L.trace);
    cudaFreeHost(L.hbuf);
    cudaFree(L.dbuf);
    if (L.e0) cudaEventDestroy(L.e0);
    if (L.e1) cudaEventDestroy(L.e1);
    for (int k = 0; k < RING; k++) {
        if (L.k0[k]) cudaEventDestroy(L.k0[k]);
        if (L.k1[k]) cudaEventDestroy(L.k1[k]);
    }
    if (L.ev_wait) cudaEventDestroy(L.ev_wait);
    if (L.hflag) cudaFreeHost((void *)L.hflag);
}

/* wait for the lane's stream: poll when the thread owns its core (no
 * wake-up latency), else sleep so lower-priority threads on the core run */
void lane_wait(Lane &L) {
    if (L.spin && L.hflag) {
        const uint32_t want = ++L.seq;
        if (write_value32()((CUstream)L.st, L.dflag, want, CU_STREAM_WRITE_VALUE_DEFAULT) == CUDA_SUCCESS) {
            while (*L.hflag != want) {
            }
            return;
        }
    }
    cudaEventRecord(L.ev_wait, L.st);
    if (L.spin) {
        while (cudaEventQuery(L.ev_wait) == cudaErrorNotReady) {
        }
    } else {
        cudaEventSynchronize(L.ev_wait);
    }
}

/* enqueue one GPU segment on the lane's stream */
void enqueue_segment(Lane &L, const uint32_t *mask, int nslots, long long items, int iters,
                     bool trace) {
    SegArgs a;
    memcpy(a.mask, mask, sizeof a.mask);
    a.ctl = L.ctl;
    a.items = items;
    a.iters = iters;
    a.nslots = nslots;
    a.sink = L.sink;
    a.trace = trace ? L.trace : nullptr;
    cudaMemsetAsync(L.ctl, 0, sizeof(Ctl), L.st);
    const int grid = sm_count() * RTGPU_EXEC_BLOCKS_PER_SM;
    persistent_segment<<<grid, 128, 0, L.st>>>(a);
}

/* the last launch's participating blocks and on-GPU span (us); enqueues a
 * D2H of the control block and waits */
struct LaunchDetail {
    double skew_us;     /* first -> last participating block start             */
    int items_min, items_max;
    double mhz;         /* SM clock over the first participant's run            */
    int smsp_max;       /* most participating warps on one SM sub-partition     */
};

void decode_ctl(const Ctl &c, unsigned *nb, double *span_us, LaunchDetail *d);

void lane_readback(Lane &L, unsigned *nb, double *span_us, LaunchDetail *d = nullptr) {
    cudaMemcpyAsync(L.hctl, L.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, L.st);
    lane_wait(L);
    decode_ctl(*L.hctl, nb, span_us, d);
}

void decode_ctl(const Ctl &c, unsigned *nb, double *span_us, LaunchDetail *d) {
    *nb = c.trace_n;
    const unsigned long long t0 = ~c.inv_start, t1 = c.end;
    *span_us = (c.inv_start && t1 >= t0) ? (double)(t1 - t0) * 1e-3 : 0.0;
    if (d) {
        d->skew_us = (c.inv_start && c.last_start >= t0) ? (double)(c.last_start - t0) * 1e-3 : 0.0;
        d->mhz = (c.ns1 > c.ns0 && c.cyc1 > c.cyc0) ? (double)(c.cyc1 - c.cyc0) * 1e3 / (double)(c.ns1 - c.ns0)
                                                   : 0.0;
        d->items_min = 1 << 30;
        d->items_max = 0;
        for (unsigned b = 0; b < std::min(c.trace_n, 16u); b++) {
            d->items_min = std::min(d->items_min, (int)c.bitems[b]);
            d->items_max = std::max(d->items_max, (int)c.bitems[b]);
        }
        d->smsp_max = 0;
        for (int sm = 0; sm < 256; sm++)
            for (int k = 0; k < 4; k++) d->smsp_max = std::max(d->smsp_max, (int)((c.smsp[sm] >> (8 * k)) & 255));
    }
}

typedef std::chrono::steady_clock clk;

inline double us_since(clk::time_point t0) {
    return std::chrono::duration<double, std::micro>(clk::now() - t0).count();
}

double thread_cpu_us() {
    timespec ts;
    clock_gettime(CLOCK_THREAD_CPUTIME_ID, &ts);
    return (double)ts.tv_sec * 1e6 + (double)ts.tv_nsec * 1e-3;
}

/* execute `us` of CPU work: spin until the thread has consumed that much CPU
 * time (a preempted segment resumes where it stopped, as in the model) */
void spin_us(double us) {
    const double t0 = thread_cpu_us();
    while (thread_cpu_us() - t0 < us) {
    }
}

/* One non-preemptive fixed-priority bus (simulator.py grant_bus): a copy
 * starts when the bus is free and no higher-priority copy is waiting. */
struct Bus {
    std::mutex mu;
    std::condition_variable cv;
    bool busy = false;
    std::multiset<int> waiting; /* priorities: lower value = higher priority */
    void acquire(int prio, bool poll) {
        std::unique_lock<std::mutex> lk(mu);
        auto it = waiting.insert(prio);
        if (poll) { /* the thread owns its core: no wake-up latency */
            while (busy || *waiting.begin() != prio) {
                lk.unlock();
                lk.lock();
            }
        } else {
            cv.wait(lk, [&] { return !busy && *waiting.begin() == prio; });
        }
        waiting.erase(it);
        busy = true;
    }
    void release() {
        {
            std::lock_guard<std::mutex> lk(mu);
            busy = false;
        }
        cv.notify_all();
    }
};

int g_cpu_mode = RTGPU_EXEC_CPU_PARALLEL;
int g_bus_mode = RTGPU_EXEC_BUS_FP;

/* the CPUs this process may run on, highest first */
std::vector<int> allowed_cpus() {
    std::vector<int> out;
    cpu_set_t set;
    CPU_ZERO(&set);
    if (sched_getaffinity(0, sizeof set, &set) == 0)
        for (int c = CPU_SETSIZE - 1; c >= 0; c--)
            if (CPU_ISSET(c, &set)) out.push_back(c);
    return out;
}

/* Keep every other thread of the process (the caller, the CUDA driver's
 * helpers) off the task threads' cores for the run, so a polling task
 * thread is never time-sliced away; restore() puts the old masks back. */
struct CoreFence {
    std::vector<std::pair<pid_t, cpu_set_t>> saved;
    void apply(const std::vector<int> &reserved, const std::vector<int> &all) {
        cpu_set_t others;
        CPU_ZERO(&others);
        int n_others = 0;
        for (int c : all)
            if (std::find(reserved.begin(), reserved.end(), c) == reserved.end()) {
                CPU_SET(c, &others);
                n_others++;
            }
        if (n_others == 0) return;
        DIR *d = opendir("/proc/self/task");
        if (!d) return;
        while (dirent *e = readdir(d)) {
            const pid_t tid = (pid_t)atoi(e->d_name);
            if (tid <= 0) continue;
            cpu_set_t old;
            if (sched_getaffinity(tid, sizeof old, &old) != 0) continue;
            if (sched_setaffinity(tid, sizeof others, &others) == 0) saved.push_back({tid, old});
        }
        closedir(d);
    }
    void restore() {
        for (auto &x : saved) sched_setaffinity(x.first, sizeof x.second, &x.second);
        saved.clear();
    }
};

bool pin_thread(int cpu) {
    cpu_set_t set;
    CPU_ZERO(&set);
    CPU_SET(cpu, &set);
    return pthread_setaffinity_np(pthread_self(), sizeof set, &set) == 0;
}

}  // namespace

extern "C" {

const char *rtgpu_exec_last_error(void) { return g_err; }

int rtgpu_exec_kernel_ms(const uint32_t *mask, int nslots, int64_t items, int iters, int reps,
                         float *ms_out, int32_t *blocks_out, int32_t *sms_out) {
    return rtgpu_exec_kernel_ms_idle(mask, nslots, items, iters, reps, 0, ms_out, blocks_out, sms_out);
}

int rtgpu_exec_kernel_ms_idle(const uint32_t *mask, int nslots, int64_t items, int iters, int reps,
                              int idle_us, float *ms_out, int32_t *blocks_out, int32_t *sms_out) {
    return rtgpu_exec_kernel_ms_loaded(mask, nslots, items, iters, reps, idle_us, nullptr, ms_out,
                                       blocks_out, sms_out);
}

int rtgpu_exec_kernel_ms_loaded(const uint32_t *mask, int nslots, int64_t items, int iters, int reps,
                                int idle_us, const uint32_t *bg_mask, float *ms_out,
                                int32_t *blocks_out, int32_t *sms_out) {
    return rtgpu_exec_kernel_ms_stress(mask, nslots, items, iters, reps, idle_us, bg_mask, 0, ms_out,
                                       blocks_out, sms_out);
}

int rtgpu_exec_kernel_ms_stress(const uint32_t *mask, int nslots, int64_t items, int iters, int reps,
                                int idle_us, const uint32_t *bg_mask, int64_t copy_bytes, float *ms_out,
                                int32_t *blocks_out, int32_t *sms_out) {
    /* copy load: a host thread keeps alternating H2D / D2H copies of
     * copy_bytes (pinned) on its own stream for the whole measurement -- the
     * executor's other tasks move their data while a kernel runs, loading
     * the copy engines, L2 and the memory controllers */
    std::atomic<bool> stop_copies{false};
    std::thread copier;
    Lane C;
    if (copy_bytes > 0) {
        if (lane_init(C, (size_t)copy_bytes)) {
            strcpy(g_err, "executor allocation failed");
            return -1;
        }
        copier = std::thread([&]() {
            for (int k = 0; !stop_copies.load(std::memory_order_relaxed); k++) {
                if (k & 1) cudaMemcpyAsync(C.hbuf, C.dbuf, (size_t)copy_bytes, cudaMemcpyDeviceToHost, C.st);
                else cudaMemcpyAsync(C.dbuf, C.hbuf, (size_t)copy_bytes, cudaMemcpyHostToDevice, C.st);
                cudaStreamSynchronize(C.st);
            }
        });
    }
    struct Joiner {
        std::atomic<bool> &stop;
        std::thread &t;
        Lane &c;
        bool on;
        ~Joiner() {
            if (!on) return;
            stop.store(true);
            t.join();
            lane_free(c);
        }
    } joiner{stop_copies, copier, C, copy_bytes > 0};
    Lane L;
    if (lane_init(L, 64)) {
        strcpy(g_err, "executor allocation failed");
        return -1;
    }
    /* co-runner load: persistent segments on bg_mask (other partitions), kept
     * running for the whole measurement and stopped by advancing their work
     * counter past the end */
    Lane B;
    const bool loaded = bg_mask != nullptr;
    if (loaded) {
        if (lane_init(B, 64)) {
            strcpy(g_err, "executor allocation failed");
            return -1;
        }
        enqueue_segment(B, bg_mask, 2, (long long)1 << 40, iters, false);
    }
    /* warm up once, then time reps launches individually */
    enqueue_segment(L, mask, nslots, items, iters, false);
    cudaStreamSynchronize(L.st);
    for (int r = 0; r < reps; r++) {
        if (idle_us > 0) std::this_thread::sleep_for(std::chrono::microseconds(idle_us));
        cudaEventRecord(L.e0, L.st);
        enqueue_segment(L, mask, nslots, items, iters, r == 0);
        cudaEventRecord(L.e1, L.st);
        cudaEventSynchronize(L.e1);
        cudaEventElapsedTime(&ms_out[r], L.e0, L.e1);
        if (r == 0 && (blocks_out || sms_out)) {
            std::vector<unsigned> tr(4096);
            unsigned nb = 0;
            double span = 0;
            lane_readback(L, &nb, &span);
            nb = std::min(nb, 4096u);
            cudaMemcpy(tr.data(), L.trace, 4096 * sizeof(unsigned), cudaMemcpyDeviceToHost);
            std::vector<int> per(256, 0);
            int distinct = 0;
            bool outside = false;
            for (unsigned b = 0; b < nb; b++) {
                unsigned s = tr[b];
                if (s >= 256 || !((mask[s >> 5] >> (s & 31)) & 1u)) outside = true;
                else if (per[s]++ == 0) distinct++;
            }
            if (blocks_out) *blocks_out = outside ? -1 : (int)nb;
            if (sms_out) *sms_out = distinct;
        }
    }
    if (loaded) {
        const unsigned long long stop = (unsigned long long)1 << 62; /* past any segment's warp items */
        cudaMemcpy(&B.ctl->work, &stop, sizeof stop, cudaMemcpyHostToDevice);
        cudaStreamSynchronize(B.st);
        lane_free(B);
    }
    cudaError_t e = cudaGetLastError();
    lane_free(L);
    if (e != cudaSuccess) {
        snprintf(g_err, sizeof g_err, "kernel: %s", cudaGetErrorString(e));
        return -2;
    }
    return 0;
}

int rtgpu_exec_copy_ms(int64_t bytes, int to_device, int reps, float *ms_out) {
    Lane L;
    if (lane_init(L, (size_t)bytes)) {
        strcpy(g_err, "executor allocation failed");
        return -1;
    }
    L.spin = true;
    for (int r = -1; r < reps; r++) {
        /* host wall time of the run loop's copy path: enqueue + polled completion */
        const auto t0 = clk::now();
        if (to_device) cudaMemcpyAsync(L.dbuf, L.hbuf, bytes, cudaMemcpyHostToDevice, L.st);
        else cudaMemcpyAsync(L.hbuf, L.dbuf, bytes, cudaMemcpyDeviceToHost, L.st);
        lane_wait(L);
        if (r >= 0) ms_out[r] = (float)(us_since(t0) * 1e-3);
    }
    lane_free(L);
    return 0;
}

int rtgpu_exec_launch_us(const uint32_t *mask, int reps, float *us_out) {
    Lane L;
    if (lane_init(L, 64)) {
        strcpy(g_err, "executor allocation failed");
        return -1;
    }
    L.spin = true;
    for (int r = -1; r < reps; r++) {
        /* the run loop's kernel path with no work: memset, launch, polled completion */
        const auto t0 = clk::now();
        enqueue_segment(L, mask, 2, 0, 1, false);
        lane_wait(L);
        if (r >= 0) us_out[r] = (float)us_since(t0);
    }
    cudaError_t e = cudaGetLastError();
    lane_free(L);
    if (e != cudaSuccess) {
        snprintf(g_err, sizeof g_err, "launch: %s", cudaGetErrorString(e));
        return -2;
    }
    return 0;
}

/* Interference probe: `reps` launches of a segment on `mask` (nslots, items,
 * iters) while a background host thread keeps one load running until done:
 * load 0 none, 1 back-to-back H2D+D2H copies of `bytes`, 2 back-to-back
 * launches of an empty segment whose blocks all exit (other partitions'
 * grids), 3 a long segment on bg_mask.  Outputs each launch's on-GPU span. */
int rtgpu_exec_probe(const uint32_t *mask, int nslots, int64_t items, int iters, int reps, int load,
                     int64_t bytes, const uint32_t *bg_mask, float *span_us_out) {
    Lane L, B;
    if (lane_init(L, 64) || lane_init(B, (size_t)std::max<int64_t>(bytes, 64))) {
        strcpy(g_err, "executor allocation failed");
        return -1;
    }
    L.spin = B.spin = true;
    std::atomic<bool> stop{false};
    uint32_t none[RTGPU_EXEC_MASK_WORDS] = {0};
    std::thread bg([&]() {
        if (load == 3) enqueue_segment(B, bg_mask, 2, (long long)1 << 40, iters, false);
        while (!stop.load()) {
            if (load == 1) {
                cudaMemcpyAsync(B.dbuf, B.hbuf, (size_t)bytes, cudaMemcpyHostToDevice, B.st);
                cudaMemcpyAsync(B.hbuf, B.dbuf, (size_t)bytes, cudaMemcpyDeviceToHost, B.st);
                lane_wait(B);
            } else if (load == 2) {
                enqueue_segment(B, none, 2, 0, 1, false);
                lane_wait(B);
            } else {
                std::this_thread::sleep_for(std::chrono::microseconds(200));
            }
        }
    });
    std::this_thread::sleep_for(std::chrono::milliseconds(5));
    for (int r = 0; r < reps; r++) {
        enqueue_segment(L, mask, nslots, items, iters, false);
        unsigned nb;
        double span;
        lane_readback(L, &nb, &span);
        span_us_out[r] = (float)span;
    }
    stop = true;
    bg.join();
    if (load == 3) {
        const unsigned long long stopw = (unsigned long long)1 << 62; /* past any segment's warp items */
        cudaMemcpy(&B.ctl->work, &stopw, sizeof stopw, cudaMemcpyHostToDevice);
    }
    cudaDeviceSynchronize();
    cudaError_t e = cudaGetLastError();
    lane_free(L);
    lane_free(B);
    if (e != cudaSuccess) {
        snprintf(g_err, sizeof g_err, "probe: %s", cudaGetErrorString(e));
        return -2;
    }
    return 0;
}

int rtgpu_exec_launch_log(double *out, int max_records) {
    std::lock_guard<std::mutex> g(g_log_mu);
    const int n = (int)std::min<size_t>(g_log.size(), (size_t)std::max(0, max_records));
    for (int k = 0; k < n; k++) {
        const LaunchRec &r = g_log[k];
        double *o = out + 7 * (size_t)k;
        o[0] = r.task;
        o[1] = r.seg;
        o[2] = (double)r.t0_ns * 1e-3;
        o[3] = r.span_us;
        o[4] = r.items_min;
        o[5] = r.items_max;
        o[6] = r.mhz;
    }
    return (int)g_log.size();
}

int rtgpu_exec_stall_log(double *out, int max_records, int *sentinel_sm) {
    std::lock_guard<std::mutex> g(g_log_mu);
    if (sentinel_sm) *sentinel_sm = g_sentinel_sm;
    const int n = (int)std::min<size_t>(g_stalls.size(), (size_t)std::max(0, max_records));
    for (int k = 0; k < n; k++) {
        out[2 * k] = (double)g_stalls[k].a * 1e-3;
        out[2 * k + 1] = (double)g_stalls[k].b * 1e-3;
    }
    return (int)g_stalls.size();
}

int rtgpu_exec_configure(int cpu_mode, int bus_mode) {
    if (cpu_mode < 0 || cpu_mode > 1 || bus_mode < 0 || bus_mode > 1) {
        strcpy(g_err, "rtgpu_exec_configure: unknown mode");
        return -1;
    }
    g_cpu_mode = cpu_mode;
    g_bus_mode = bus_mode;
    return 0;
}

/*
 * Run the task set for `horizon_us`: each task is a host thread releasing
 * jobs every period; a job runs its segments in order (CPU: thread CPU time
 * on the host; copy: cudaMemcpyAsync on the task's stream, through the bus
 * arbiter in bus mode 1; kernel: persistent segment pinned to the task's SM
 * partition) and its response time is release -> end of the last CPU
 * segment.  Jobs of one task run in order; a release while the previous job
 * still runs waits for it (constrained deadlines make this rare).
 */
int rtgpu_exec_run(const rtgpu_exec_task *tasks, int n_tasks, double horizon_us,
                   rtgpu_exec_result *results) {
    if (n_tasks < 1 || n_tasks > 64) {
        strcpy(g_err, "1..64 tasks");
        return -1;
    }
    {
        std::lock_guard<std::mutex> g(g_log_mu);
        g_log.clear();
    }
    std::vector<Lane> lanes(n_tasks);
    for (int i = 0; i < n_tasks; i++) {
        int64_t mx = 64;
        for (int j = 0; j < tasks[i].n_copies; j++) mx = std::max(mx, tasks[i].copy_bytes[j]);
        if (lane_init(lanes[i], (size_t)mx)) {
            strcpy(g_err, "executor allocation failed");
            return -1;
        }
        memset(&results[i], 0, sizeof(rtgpu_exec_result));
    }
    /* priority rank of every task (0 = highest) */
    std::vector<int> rank(n_tasks, 0);
    for (int i = 0; i < n_tasks; i++)
        for (int j = 0; j < n_tasks; j++)
            if (tasks[j].priority < tasks[i].priority || (tasks[j].priority == tasks[i].priority && j < i))
                rank[i]++;
    const std::vector<int> cpus = allowed_cpus();
    const int cpu_mode = g_cpu_mode, bus_mode = g_bus_mode;
    std::atomic<int> fifo_fail{0};
    Bus bus;
    CoreFence fence;
    if (cpu_mode == RTGPU_EXEC_CPU_PARALLEL && (int)cpus.size() > n_tasks)
        fence.apply(std::vector<int>(cpus.begin(), cpus.begin() + n_tasks), cpus);
    /* the stall sentinel on the first SM no task uses */
    const int nsm = sm_count();
    int free_sm = -1;
    for (int sm = 0; sm < nsm && free_sm < 0; sm++) {
        bool used = false;
        for (int i = 0; i < n_tasks; i++) used = used || ((tasks[i].sm_mask[sm >> 5] >> (sm & 31)) & 1u);
        if (!used) free_sm = sm;
    }
    const unsigned STALL_CAP = 4096;
    cudaStream_t sst = nullptr;
    char *sbuf = nullptr; /* stop flag, claim, count, gaps */
    if (free_sm >= 0 && cudaStreamCreateWithFlags(&sst, cudaStreamNonBlocking) == cudaSuccess &&
        cudaMalloc(&sbuf, 64 + STALL_CAP * sizeof(StallGap)) == cudaSuccess) {
        cudaMemsetAsync(sbuf, 0, 64, sst);
        stall_sentinel<<<2 * nsm, 32, 0, sst>>>((unsigned)free_sm, (const volatile int *)sbuf, (int *)(sbuf + 4),
                                                (StallGap *)(sbuf + 64), (unsigned *)(sbuf + 8), STALL_CAP,
                                                50000ull, (unsigned long long)((horizon_us + 30e6) * 1e3));
    } else {
        free_sm = -1;
    }
    auto t_start = clk::now() + std::chrono::milliseconds(50);
    std::vector<std::thread> th;
    for (int i = 0; i < n_tasks; i++) {
        th.emplace_back([&, i]() {
            const rtgpu_exec_task &t = tasks[i];
            Lane &L = lanes[i];
            rtgpu_exec_result &R = results[i];
            bool own_core = true;
            if (!cpus.empty()) {
                if (cpu_mode == RTGPU_EXEC_CPU_FP_ONE_CORE) {
                    pin_thread(cpus[0]);
                    sched_param sp;
                    sp.sched_priority = 80 - rank[i];
                    if (pthread_setschedparam(pthread_self(), SCHED_FIFO, &sp) == 0) {
                        own_core = false;
                    } else {
                        fifo_fail++; /* no FP CPU: do not time-share one core */
                        pin_thread(cpus[(size_t)rank[i] % cpus.size()]);
                    }
                } else {
                    pin_thread(cpus[(size_t)rank[i] % cpus.size()]);
                }
            }
            /* a thread that owns its core polls every wait (bus, stream,
             * release): no wake-up latency enters the response times */
            L.spin = own_core;
            double sum = 0;
            auto copy = [&](int idx, bool h2d) {
                const auto w0 = clk::now();
                if (bus_mode == RTGPU_EXEC_BUS_FP) bus.acquire(t.priority, own_core);
                R.max_bus_wait_us = std::max(R.max_bus_wait_us, us_since(w0));
                const auto c0 = clk::now();
                if (h2d)
                    cudaMemcpyAsync(L.dbuf, L.hbuf, (size_t)t.copy_bytes[idx], cudaMemcpyHostToDevice, L.st);
                else
                    cudaMemcpyAsync(L.hbuf, L.dbuf, (size_t)t.copy_bytes[idx], cudaMemcpyDeviceToHost, L.st);
                lane_wait(L);
                if (bus_mode == RTGPU_EXEC_BUS_FP) bus.release();
                R.max_copy_us = std::max(R.max_copy_us, us_since(c0));
            };
            for (int64_t k = 0;; k++) {
                double release = (double)k * t.period_us;
                if (release >= horizon_us) break;
                auto rel_tp = t_start + std::chrono::microseconds((int64_t)release);
                if (own_core) {
                    std::this_thread::sleep_until(rel_tp - std::chrono::microseconds(500));
                    while (clk::now() < rel_tp) {
                    }
                } else {
                    std::this_thread::sleep_until(rel_tp);
                }
                int cp = 0;
                double wall[RING] = {0};
                for (int s = 0; s < t.m; s++) {
                    spin_us((double)t.cpu_us[s]);
                    if (s == t.m - 1) break;
                    /* memory copies and the kernel between CPU segments s and s+1 */
                    if (cp < t.n_copies) copy(cp++, true);
                    auto k0 = clk::now();
                    L.use(s);
                    cudaEventRecord(L.k0[s], L.st);
                    enqueue_segment(L, t.sm_mask, t.slots_per_sm, t.kernel_items[s], t.kernel_iters,
                                    true);
                    cudaEventRecord(L.k1[s], L.st);
                    lane_wait(L);
                    wall[s] = us_since(k0);
                    if (t.two_copy && cp < t.n_copies) copy(cp++, false);
                }
                double resp = std::chrono::duration<double, std::micro>(clk::now() - rel_tp).count();
                R.jobs++;
                sum += resp;
                R.max_response_us = std::max(R.max_response_us, resp);
                if (resp > (double)t.deadline_us) R.deadline_misses++;
                /* the job's kernel records, read back off its critical path */
                const int nk = t.m - 1;
                if (nk > 0) {
                    cudaMemcpyAsync(L.hring, L.ring, nk * sizeof(Ctl), cudaMemcpyDeviceToHost, L.st);
                    lane_wait(L);
                }
                for (int s = 0; s < nk; s++) {
                    unsigned nb = 0;
                    double span = 0;
                    LaunchDetail det;
                    decode_ctl(L.hring[s], &nb, &span, &det);
                    {
                        std::lock_guard<std::mutex> g(g_log_mu);
                        if (g_log.size() < (1u << 20))
                            g_log.push_back({i, s, ~L.hring[s].inv_start, span, det.items_min, det.items_max,
                                             det.mhz});
                    }
                    if (span > R.seg_max_span_us[s]) {
                        R.seg_worst_skew_us[s] = det.skew_us;
                        R.seg_worst_items[s][0] = det.items_min;
                        R.seg_worst_items[s][1] = det.items_max;
                        R.seg_worst_mhz[s] = det.mhz;
                        R.seg_worst_smsp[s] = det.smsp_max;
                    }
                    R.smsp_max = std::max(R.smsp_max, det.smsp_max);
                    if (det.mhz > 0 && (R.min_mhz == 0 || det.mhz < R.min_mhz)) R.min_mhz = det.mhz;
                    float kms = 0;
                    cudaEventElapsedTime(&kms, L.k0[s], L.k1[s]);
                    R.max_kernel_us = std::max(R.max_kernel_us, (double)kms * 1e3);
                    R.seg_max_kernel_us[s] = std::max(R.seg_max_kernel_us[s], (double)kms * 1e3);
                    R.seg_max_wall_us[s] = std::max(R.seg_max_wall_us[s], wall[s]);
                    R.seg_max_span_us[s] = std::max(R.seg_max_span_us[s], span);
                    if (R.min_blocks == 0 || (int)nb < R.min_blocks) R.min_blocks = (int)nb;
                    R.max_blocks = std::max(R.max_blocks, (int)nb);
                    R.max_kernel_wall_us = std::max(R.max_kernel_wall_us, wall[s]);
                }
            }
            R.mean_response_us = R.jobs ? sum / (double)R.jobs : 0;
        });
    }
    for (auto &x : th) x.join();
    fence.restore();
    {
        std::lock_guard<std::mutex> g(g_log_mu);
        g_stalls.clear();
        g_sentinel_sm = free_sm;
        if (free_sm >= 0) {
            /* the stop flag goes through a second stream: sst is occupied by
             * the sentinel itself until it sees the flag */
            static const int one = 1;
            cudaStream_t s2 = nullptr;
            cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
            cudaMemcpyAsync(sbuf, &one, sizeof one, cudaMemcpyHostToDevice, s2);
            cudaStreamSynchronize(s2);
            cudaStreamDestroy(s2);
            unsigned n = 0;
            cudaMemcpyAsync(&n, sbuf + 8, sizeof n, cudaMemcpyDeviceToHost, sst);
            cudaStreamSynchronize(sst);
            n = std::min(n, STALL_CAP);
            g_stalls.resize(n);
            if (n) cudaMemcpy(g_stalls.data(), sbuf + 64, n * sizeof(StallGap), cudaMemcpyDeviceToHost);
        }
    }
    if (sbuf) cudaFree(sbuf);
    if (sst) cudaStreamDestroy(sst);
    for (int i = 0; i < n_tasks; i++) {
        results[i].cpu_mode = (cpu_mode == RTGPU_EXEC_CPU_FP_ONE_CORE && fifo_fail == 0)
                                  ? RTGPU_EXEC_CPU_FP_ONE_CORE : RTGPU_EXEC_CPU_PARALLEL;
        results[i].bus_mode = bus_mode;
    }
    cudaError_t e = cudaGetLastError();
    for (auto &L : lanes) lane_free(L);
    if (e != cudaSuccess) {
        snprintf(g_err, sizeof g_err, "run: %s", cudaGetErrorString(e));
        return -2;
    }
    if (cpu_mode == RTGPU_EXEC_CPU_FP_ONE_CORE && fifo_fail > 0) {
        snprintf(g_err, sizeof g_err, "SCHED_FIFO unavailable: ran with a core per task");
    }
    return 0;
}

}  // extern "C"
