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
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/rtgpu_exec.h"

namespace {

__device__ __forceinline__ unsigned smid() {
    unsigned r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}

struct SegArgs {
    uint32_t mask[RTGPU_EXEC_MASK_WORDS]; /* partition, by value (no H2D per launch) */
    unsigned *slots;                      /* per-SM slot counters, zeroed per launch */
    unsigned long long *work;             /* work counter, zeroed per launch */
    long long items;
    int iters;
    int nslots;
    float *sink;
    unsigned *trace; /* optional: SM of every participating block (+ count at [0]) */
};

__global__ void __launch_bounds__(128) persistent_segment(SegArgs a) {
    __shared__ unsigned slot;
    __shared__ unsigned long long item;
    const unsigned sm = smid();
    if (!((a.mask[sm >> 5] >> (sm & 31)) & 1u)) return;
    if (threadIdx.x == 0) slot = atomicAdd(&a.slots[sm], 1u);
    __syncthreads();
    if (slot >= (unsigned)a.nslots) return;
    if (a.trace && threadIdx.x == 0) {
        unsigned pos = atomicAdd(&a.trace[0], 1u);
        if (pos < 4095) a.trace[1 + pos] = sm;
    }
    /* synthetic compute work: dependent FMA chains, 4 per thread (ILP).
     * The next item is claimed before the current one is computed, so the
     * atomic's round trip (L2-die and contention dependent) overlaps work. */
    float x0 = threadIdx.x, x1 = x0 + 1.f, x2 = x0 + 2.f, x3 = x0 + 3.f;
    __shared__ unsigned long long next;
    if (threadIdx.x == 0) item = atomicAdd(a.work, 1ull);
    __syncthreads();
    unsigned long long it = item;
    while ((long long)it < a.items) {
        if (threadIdx.x == 0) next = atomicAdd(a.work, 1ull);
        for (int k = 0; k < a.iters; k++) {
            x0 = fmaf(x0, 0.9999999f, 0.5f);
            x1 = fmaf(x1, 0.9999999f, 0.5f);
            x2 = fmaf(x2, 0.9999999f, 0.5f);
            x3 = fmaf(x3, 0.9999999f, 0.5f);
        }
        __syncthreads();
        it = next;
        __syncthreads();
    }
    if (x0 + x1 + x2 + x3 == 12345.f) a.sink[blockIdx.x] = x0;
}

char g_err[256] = "";

struct Lane {
    cudaStream_t st = nullptr;
    unsigned *slots = nullptr;
    unsigned long long *work = nullptr;
    float *sink = nullptr;
    unsigned *trace = nullptr;
    void *hbuf = nullptr, *dbuf = nullptr;
    size_t buf = 0;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
};

int sm_count() {
    int dev = 0, n = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
}

int lane_init(Lane &L, size_t buf) {
    if (cudaStreamCreateWithFlags(&L.st, cudaStreamNonBlocking) != cudaSuccess) return -1;
    if (cudaMalloc(&L.slots, 256 * sizeof(unsigned)) != cudaSuccess) return -1;
    if (cudaMalloc(&L.work, sizeof(unsigned long long)) != cudaSuccess) return -1;
    if (cudaMalloc(&L.sink, 8192 * sizeof(float)) != cudaSuccess) return -1;
    if (cudaMalloc(&L.trace, 4096 * sizeof(unsigned)) != cudaSuccess) return -1;
    L.buf = buf < 64 ? 64 : buf;
    if (cudaMallocHost(&L.hbuf, L.buf) != cudaSuccess) return -1;
    if (cudaMalloc(&L.dbuf, L.buf) != cudaSuccess) return -1;
    memset(L.hbuf, 1, L.buf);
    cudaEventCreate(&L.e0);
    cudaEventCreate(&L.e1);
    return 0;
}

void lane_free(Lane &L) {
    if (L.st) cudaStreamDestroy(L.st);
    cudaFree(L.slots);
    cudaFree(L.work);
    cudaFree(L.sink);
    cudaFree(L.trace);
    cudaFreeHost(L.hbuf);
    cudaFree(L.dbuf);
    if (L.e0) cudaEventDestroy(L.e0);
    if (L.e1) cudaEventDestroy(L.e1);
}

/* enqueue one GPU segment on the lane's stream */
void enqueue_segment(Lane &L, const uint32_t *mask, int nslots, long long items, int iters,
                     bool trace) {
    SegArgs a;
    memcpy(a.mask, mask, sizeof a.mask);
    a.slots = L.slots;
    a.work = L.work;
    a.items = items;
    a.iters = iters;
    a.nslots = nslots;
    a.sink = L.sink;
    a.trace = trace ? L.trace : nullptr;
    cudaMemsetAsync(L.slots, 0, 256 * sizeof(unsigned), L.st);
    cudaMemsetAsync(L.work, 0, sizeof(unsigned long long), L.st);
    if (trace) cudaMemsetAsync(L.trace, 0, sizeof(unsigned), L.st);
    const int grid = sm_count() * RTGPU_EXEC_BLOCKS_PER_SM;
    persistent_segment<<<grid, 128, 0, L.st>>>(a);
}

typedef std::chrono::steady_clock clk;

inline double us_since(clk::time_point t0) {
    return std::chrono::duration<double, std::micro>(clk::now() - t0).count();
}

void spin_us(double us) {
    auto t0 = clk::now();
    while (us_since(t0) < us) {
    }
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
            cudaMemcpy(tr.data(), L.trace, 4096 * sizeof(unsigned), cudaMemcpyDeviceToHost);
            unsigned nb = std::min(tr[0], 4095u);
            std::vector<int> per(256, 0);
            int distinct = 0;
            bool outside = false;
            for (unsigned b = 0; b < nb; b++) {
                unsigned s = tr[1 + b];
                if (s >= 256 || !((mask[s >> 5] >> (s & 31)) & 1u)) outside = true;
                else if (per[s]++ == 0) distinct++;
            }
            if (blocks_out) *blocks_out = outside ? -1 : (int)nb;
            if (sms_out) *sms_out = distinct;
        }
    }
    if (loaded) {
        const unsigned long long stop = (unsigned long long)1 << 41;
        cudaMemcpy(B.work, &stop, sizeof stop, cudaMemcpyHostToDevice);
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
    for (int r = -1; r < reps; r++) {
        cudaEventRecord(L.e0, L.st);
        if (to_device) cudaMemcpyAsync(L.dbuf, L.hbuf, bytes, cudaMemcpyHostToDevice, L.st);
        else cudaMemcpyAsync(L.hbuf, L.dbuf, bytes, cudaMemcpyDeviceToHost, L.st);
        cudaEventRecord(L.e1, L.st);
        cudaEventSynchronize(L.e1);
        if (r >= 0) cudaEventElapsedTime(&ms_out[r], L.e0, L.e1);
    }
    lane_free(L);
    return 0;
}

/*
 * Run the task set for `horizon_us`: each task is a host thread releasing
 * jobs every period; a job runs its segments in order (CPU: busy wait on the
 * host; copy: cudaMemcpyAsync on the task's stream; kernel: persistent
 * segment pinned to the task's SM partition) and its response time is
 * release -> end of the last CPU segment.  Jobs of one task run in order;
 * a release while the previous job still runs waits for it (the sporadic
 * task model's constrained deadlines make this rare).
 */
int rtgpu_exec_run(const rtgpu_exec_task *tasks, int n_tasks, double horizon_us,
                   rtgpu_exec_result *results) {
    if (n_tasks < 1 || n_tasks > 64) {
        strcpy(g_err, "1..64 tasks");
        return -1;
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
    std::atomic<int> ready{0};
    auto t_start = clk::now() + std::chrono::milliseconds(50);
    std::vector<std::thread> th;
    for (int i = 0; i < n_tasks; i++) {
        th.emplace_back([&, i]() {
            const rtgpu_exec_task &t = tasks[i];
            Lane &L = lanes[i];
            rtgpu_exec_result &R = results[i];
            ready++;
            std::this_thread::sleep_until(t_start);
            double sum = 0;
            for (int64_t k = 0;; k++) {
                double release = (double)k * t.period_us;
                if (release >= horizon_us) break;
                auto rel_tp = t_start + std::chrono::microseconds((int64_t)release);
                std::this_thread::sleep_until(rel_tp);
                int copy = 0;
                for (int s = 0; s < t.m; s++) {
                    spin_us((double)t.cpu_us[s]);
                    if (s == t.m - 1) break;
                    /* memory copies and the kernel between CPU segments s and s+1 */
                    auto seg_t0 = clk::now();
                    if (copy < t.n_copies) {
                        cudaMemcpyAsync(L.dbuf, L.hbuf, (size_t)t.copy_bytes[copy++],
                                        cudaMemcpyHostToDevice, L.st);
                        cudaStreamSynchronize(L.st);
                    }
                    double c0 = us_since(seg_t0);
                    R.max_copy_us = std::max(R.max_copy_us, c0);
                    auto k0 = clk::now();
                    cudaMemsetAsync(L.trace, 0, sizeof(unsigned), L.st);
                    cudaEventRecord(L.e0, L.st);
                    enqueue_segment(L, t.sm_mask, t.slots_per_sm, t.kernel_items[s], t.kernel_iters,
                                    true);
                    cudaEventRecord(L.e1, L.st);
                    unsigned nb = 0;
                    cudaMemcpyAsync(&nb, L.trace, sizeof(unsigned), cudaMemcpyDeviceToHost, L.st);
                    cudaStreamSynchronize(L.st);
                    float kms = 0;
                    cudaEventElapsedTime(&kms, L.e0, L.e1);
                    R.max_kernel_us = std::max(R.max_kernel_us, (double)kms * 1e3);
                    R.seg_max_kernel_us[s] = std::max(R.seg_max_kernel_us[s], (double)kms * 1e3);
                    if (R.min_blocks == 0 || (int)nb < R.min_blocks) R.min_blocks = (int)nb;
                    R.max_blocks = std::max(R.max_blocks, (int)nb);
                    R.max_kernel_wall_us = std::max(R.max_kernel_wall_us, us_since(k0));
                    if (t.two_copy && copy < t.n_copies) {
                        auto d0 = clk::now();
                        cudaMemcpyAsync(L.hbuf, L.dbuf, (size_t)t.copy_bytes[copy++],
                                        cudaMemcpyDeviceToHost, L.st);
                        cudaStreamSynchronize(L.st);
                        R.max_copy_us = std::max(R.max_copy_us, us_since(d0));
                    }
                }
                double resp = std::chrono::duration<double, std::micro>(clk::now() - rel_tp).count();
                R.jobs++;
                sum += resp;
                R.max_response_us = std::max(R.max_response_us, resp);
                if (resp > (double)t.deadline_us) R.deadline_misses++;
            }
            R.mean_response_us = R.jobs ? sum / (double)R.jobs : 0;
        });
    }
    for (auto &x : th) x.join();
    cudaError_t e = cudaGetLastError();
    for (auto &L : lanes) lane_free(L);
    if (e != cudaSuccess) {
        snprintf(g_err, sizeof g_err, "run: %s", cudaGetErrorString(e));
        return -2;
    }
    return 0;
}

}  // extern "C"
