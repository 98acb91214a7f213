/*
 * rtgpu_exec.h -- C-ABI of the SM-partitioned persistent-thread executor
 * (csrc/executor.cu): the paper's accelerator mechanism (RTGPU section 4,
 * Algorithm 1) on the GPU, whose measured response times are checked against
 * the analysis (the reference checks its discrete-event simulator the same
 * way: simulator.py check_against_analysis).
 */
#ifndef RTGPU_EXEC_H
#define RTGPU_EXEC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RTGPU_EXEC_MASK_WORDS 8    /* SM bitmap: up to 256 SMs            */
#ifndef RTGPU_EXEC_BLOCKS_PER_SM
#define RTGPU_EXEC_BLOCKS_PER_SM 6 /* launch width per SM (>= 2 slots)    */
#endif

typedef struct {
    int32_t m;                    /* CPU segments                              */
    int32_t two_copy;             /* 1: H2D before and D2H after each kernel   */
    int32_t n_copies;             /* memory copies (2m-2 or m-1)               */
    int32_t slots_per_sm;         /* virtual SMs per physical SM (2)           */
    int64_t cpu_us[16];           /* CPU segment lengths (host busy wait)      */
    int64_t copy_bytes[30];       /* bytes of each copy                        */
    int64_t kernel_items[15];     /* work items of each kernel                 */
    int32_t kernel_iters;         /* FMA iterations per item                   */
    int32_t priority;
    uint32_t sm_mask[RTGPU_EXEC_MASK_WORDS]; /* the task's physical SMs        */
    int64_t period_us;
    int64_t deadline_us;
} rtgpu_exec_task;

typedef struct {
    int64_t jobs;
    int64_t deadline_misses;
    double max_response_us;       /* measured worst-case response time        */
    double mean_response_us;
    double max_kernel_us;         /* worst kernel time (CUDA events)          */
    double max_kernel_wall_us;    /* worst kernel time incl. launch (host)    */
    double max_copy_us;
    double seg_max_kernel_us[15]; /* worst time of each kernel segment        */
    int32_t min_blocks;           /* fewest participating blocks in a launch  */
    int32_t max_blocks;           /* most participating blocks in a launch    */
    double seg_max_span_us[15];   /* worst on-GPU span of each kernel segment:
                                   * first participating block's start to the
                                   * last one's end (%globaltimer)            */
    double max_bus_wait_us;       /* worst wait for the bus (arbiter mode)    */
    int32_t cpu_mode;             /* CPU mode actually applied (see below)    */
    int32_t bus_mode;             /* bus mode actually applied                */
    /* the launch with the worst span of each kernel segment: first -> last
     * participating block start, fewest / most work items a participating
     * block ran */
    double seg_worst_skew_us[15];
    int32_t seg_worst_items[15][2];
    double seg_max_wall_us[15];   /* worst host-observed kernel segment: launch
                                   * to observed completion (the segment's
                                   * response as the job sees it)            */
    double seg_worst_mhz[15];     /* SM clock during the worst-span launch     */
    double min_mhz;               /* lowest SM clock seen in any launch        */
    int32_t seg_worst_smsp[15];   /* worst-span launch: most participating warps
                                   * on one SM sub-partition (%warpid % 4) of
                                   * any of its SMs (2 = even, two 4-warp
                                   * blocks per SM)                           */
    int32_t smsp_max;             /* the same over every launch                */
} rtgpu_exec_result;

/* Host-side resource models of rtgpu_exec_run (rtgpu_exec_configure):
 *  cpu_mode 0  every task thread on its own core (no CPU interference: the
 *              analysis' single preemptive CPU is an over-approximation)
 *  cpu_mode 1  all task threads on one core under SCHED_FIFO, priorities in
 *              the tasks' order -- the analysis' preemptive fixed-priority
 *              CPU (falls back to mode 0 without CAP_SYS_NICE)
 *  bus_mode 0  copies of different tasks may overlap on the copy engines
 *  bus_mode 1  one non-preemptive fixed-priority bus: a copy waits until the
 *              bus is free and it is the highest-priority waiter (Lemma 6's
 *              model; simulator.py grant_bus)
 * CPU segments consume thread CPU time (CLOCK_THREAD_CPUTIME_ID), so a
 * preempted segment still executes its full length. */
#define RTGPU_EXEC_CPU_PARALLEL 0
#define RTGPU_EXEC_CPU_FP_ONE_CORE 1
#define RTGPU_EXEC_BUS_FREE 0
#define RTGPU_EXEC_BUS_FP 1

const char *rtgpu_exec_last_error(void);

/* Time `reps` launches of one persistent segment on partition `mask` with
 * `nslots` blocks per SM; blocks_out = participating blocks of the first
 * launch (-1 if any ran outside the mask), sms_out = distinct SMs used. */
int rtgpu_exec_kernel_ms(const uint32_t *mask, int nslots, int64_t items, int iters, int reps,
                         float *ms_out, int32_t *blocks_out, int32_t *sms_out);

/* Same, with the GPU left idle for idle_us before every timed launch (the
 * clock may have dropped: worst-case calibration without locked clocks). */
int rtgpu_exec_kernel_ms_idle(const uint32_t *mask, int nslots, int64_t items, int iters, int reps,
                              int idle_us, float *ms_out, int32_t *blocks_out, int32_t *sms_out);

/* Same, while persistent segments keep the SMs of bg_mask busy (co-runner
 * interference of concurrent partitions: launch path, L2, power). */
int rtgpu_exec_kernel_ms_loaded(const uint32_t *mask, int nslots, int64_t items, int iters, int reps,
                                int idle_us, const uint32_t *bg_mask, float *ms_out,
                                int32_t *blocks_out, int32_t *sms_out);

/* Same, with a host thread alternating H2D / D2H pinned copies of
 * copy_bytes on its own stream throughout (copy-engine, L2 and memory
 * load of the other tasks' copies); copy_bytes <= 0: no copies. */
int rtgpu_exec_kernel_ms_stress(const uint32_t *mask, int nslots, int64_t items, int iters, int reps,
                                int idle_us, const uint32_t *bg_mask, int64_t copy_bytes, float *ms_out,
                                int32_t *blocks_out, int32_t *sms_out);

/* Host wall time (us) of `reps` empty segment launches on `mask`: memset,
 * launch and polled completion -- the executor's per-kernel overhead. */
int rtgpu_exec_launch_us(const uint32_t *mask, int reps, float *us_out);

/* The kernel launches of the last rtgpu_exec_run, 7 doubles each: task
 * index, kernel segment, first participating block's start (us of
 * %globaltimer), on-GPU span (us), fewest / most work items of a traced
 * warp, SM clock (MHz).  Writes min(count, max_records) records and returns
 * the count. */
int rtgpu_exec_launch_log(double *out, int max_records);

/* The last rtgpu_exec_run's stall sentinel: one thread on an SM no task used
 * read %globaltimer every ~2 us for the whole run; each record (2 doubles,
 * us of %globaltimer, the launch log's time base) is an interval over 50 us
 * in which it did not run.  *sentinel_sm = that SM, -1 if every SM was in a
 * partition (no sentinel).  Returns the count. */
int rtgpu_exec_stall_log(double *out, int max_records, int *sentinel_sm);

/* Host wall time (ms) of `reps` pinned-host copies of `bytes` (to_device:
 * H2D, else D2H): enqueue and polled completion, as the run loop does. */
int rtgpu_exec_copy_ms(int64_t bytes, int to_device, int reps, float *ms_out);

/* Select the host resource models for subsequent rtgpu_exec_run calls. */
int rtgpu_exec_configure(int cpu_mode, int bus_mode);

/* Run the task set for horizon_us with periodic releases; per-task results. */
int rtgpu_exec_run(const rtgpu_exec_task *tasks, int n_tasks, double horizon_us,
                   rtgpu_exec_result *results);

#ifdef __cplusplus
}
#endif

#endif
