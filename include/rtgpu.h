/*
 * rtgpu.h -- C-ABI of the B200 batched RTGPU schedulability engine.
 *
 * This is the drop-in boundary for the data-parallel hot path of the
 * reference package `gpusched` (reference: pkg/src/gpusched/).  The
 * reference is pure Python, so "its FFI" is the ctypes binding its public
 * API would use; INTEGRATION.md shows that binding.  Every entry point is
 * plain C: int64/int32 pointers and sizes, no torch or CUDA types.
 *
 *   reference function (file:line)                     replaced by
 *   -----------------------------------------------    -------------------------
 *   analysis.analyze_rtgpu            analysis.py:275  rtgpu_analyze_{host,device}
 *   analysis._grid_search             analysis.py:250    (method RTGPU_METHOD_RTGPU)
 *   analysis._min_feasible_gn         analysis.py:239
 *   gpu.feasible_allocations          gpu.py:69
 *   gpu.gpu_bounds_cache              gpu.py:91
 *   gpu.gpu_response_bounds           gpu.py:25
 *   analysis.mem_response             analysis.py:156
 *   analysis.cpu_response             analysis.py:175
 *   analysis.end_to_end               analysis.py:191
 *   analysis.{mem,cpu}_workload       analysis.py:109,118
 *   analysis.{mem,cpu}_inter_arrival  analysis.py:57,89
 *   suspension.chain_workload         suspension.py:77
 *   suspension.fixed_point            suspension.py:123
 *   analysis.analyze_self_suspension_baseline  analysis.py:319  (RTGPU_METHOD_SELFSUSP)
 *   analysis.analyze_busy_waiting_baseline     analysis.py:355  (RTGPU_METHOD_BUSYWAIT)
 *   suspension.{workload,max_workload,         suspension.py:107-176
 *               segment_response,task_response}   rtgpu_query_host (RTGPU_Q_*)
 *
 * ---------------------------------------------------------------------
 * Packed task-set layout ("blob"), shared by the engine and the oracle.
 * ---------------------------------------------------------------------
 * A batch is a flat int64 array holding S blobs back to back; set_off[s]
 * is the word offset of blob s (set_off[S] = total words) and
 * task_base[s] the index of its first task in the per-task result arrays
 * (task_base[S] = total tasks).  Every duration is an integer count of
 * "input ticks" (1 tick = 1/time_scale us; the engine is scale free, the
 * host multiplies result denominators by time_scale).
 *
 *   header (RTGPU_HDR_WORDS):
 *     [0] n_tasks  [1] physical_sms (GN)  [2] mem_model (0 two_copy, 1 one_copy)
 *     [3] alpha_den (A: interleave ratio = alpha_num / A)  [4] blob words
 *     [5] max m over tasks  [6] max p over tasks
 *     [7] segment word: 0 = int64; 1 = int32 (compact: segment areas hold
 *         int32 values and seg_off counts int32 elements from the blob
 *         start; not combinable with RTGPU_F_DETAIL); 2 = compact with
 *         packed task records (4 int64 words per task: D, T,
 *         m | p << 8 | index << 16, priority (int32, low half) | seg_off << 32):
 *         15% fewer bytes per 8 x 5 set to copy; read records through
 *         rtgpu_rec_word(), which returns the 8-word record's fields
 *   n task records (RTGPU_TASK_WORDS each), in TaskSet.by_priority() order:
 *     [0] m (CPU segments)  [1] p (memory segments)  [2] D  [3] T
 *     [4] priority  [5] seg_off (word offset of the segment area from the
 *     blob start)  [6] index of the task in TaskSet.tasks  [7] 0
 *   segment area of a task (g = m - 1 GPU segments):
 *     cl_lo[m] cl_hi[m] ml_lo[p] ml_hi[p] gw_lo[g] gw_hi[g] gl[g] alpha_num[g]
 *
 * Results (per set s / per task t / per blob word w):
 *   status[s]   RTGPU_* status below
 *   evals[s]    number of task evaluations the search performed
 *   vsm[t]      virtual SMs (2*GN_i) of the reported allocation, 0 if none
 *   e2e_num[t]  end-to-end bound numerator; RTGPU_NONE if the analysis
 *               returned None, RTGPU_ABSENT if the task is not in per_task
 *   den[t]      denominator (in input ticks) shared by all values of task t
 *   detail[w]   optional, same shape as the blob buffer: at the task's
 *               segment area, the cl_lo slots hold cpu_r_up[m], the ml_lo
 *               slots mem_r_up[p], the gw_lo / gw_hi slots the GPU response
 *               bounds GR lo / hi; numerators over den[t], RTGPU_NONE = None.
 */
#ifndef RTGPU_H
#define RTGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RTGPU_ABI_VERSION 1

#define RTGPU_HDR_WORDS 8
#define RTGPU_TASK_WORDS 8

/* int64 words of the record area per task: 8, or 4 with int32 records */
#define RTGPU_REC_WORDS(seg_word) ((seg_word) == 2 ? RTGPU_TASK_WORDS / 2 : RTGPU_TASK_WORDS)

/* field f (the 8-word record's numbering) of task record i, either form */
static inline int64_t rtgpu_rec_packed(const int64_t *w, int f) {
    switch (f) {
    case 0: return w[2] & 0xff;
    case 1: return (w[2] >> 8) & 0xff;
    case 2: return w[0];
    case 3: return w[1];
    case 4: return (int64_t)(int32_t)(uint32_t)((uint64_t)w[3] & 0xffffffffu);
    case 5: return w[3] >> 32;
    case 6: return w[2] >> 16;
    default: return 0;
    }
}
static inline int64_t rtgpu_rec_word(const int64_t *blob, int i, int f) {
    return blob[7] == 2 ? rtgpu_rec_packed(blob + RTGPU_HDR_WORDS + (RTGPU_TASK_WORDS / 2) * i, f)
                        : blob[RTGPU_HDR_WORDS + RTGPU_TASK_WORDS * i + f];
}

#define RTGPU_TWO_COPY 0
#define RTGPU_ONE_COPY 1

/* analysis methods (model.AnalysisMethod) */
#define RTGPU_METHOD_RTGPU 0
#define RTGPU_METHOD_SELFSUSP 1
#define RTGPU_METHOD_BUSYWAIT 2

/* per-set status */
#define RTGPU_UNSCHEDULABLE 0
#define RTGPU_SCHEDULABLE 1
#define RTGPU_UNDECIDED 2  /* allocation search exceeded eval_budget         */
#define RTGPU_RANGE 3      /* exact values exceed the 127-bit range          */
#define RTGPU_INVALID 4    /* input the reference rejects with an exception  */

/* sentinels in e2e_num / detail */
#define RTGPU_NONE (-1LL)
#define RTGPU_ABSENT (-2LL)

/* flags */
#define RTGPU_F_BOUNDS 1u  /* fill e2e_num/den for the reported allocation   */
#define RTGPU_F_DETAIL 2u  /* also the per-segment report (implies BOUNDS)   */
#define RTGPU_F_FIRST_I64 4u  /* testing: start at the int64 stage          */
#define RTGPU_F_FIRST_I128 8u /* testing: start at the int128 stage         */

/* limits of the engine (checked on entry; larger sets -> RTGPU_INVALID) */
#define RTGPU_MAX_TASKS 64
#define RTGPU_MAX_M 16

int rtgpu_abi_version(void);
const char *rtgpu_last_error(void);
/* number of visible CUDA devices, SM count and compute capability of device 0 */
int rtgpu_device_info(int *n_devices, int *sm_count, int *cc_major, int *cc_minor);

/*
 * Batched allocation search + response-time analysis (Algorithm 2) of S
 * packed task sets, each exactly as gpusched.analysis.analyze(ts, method).
 * Host pointers: the call copies the batch to the current device in chunks
 * overlapped with the analysis of the chunks already resident, and copies
 * the results back (the end-to-end path; pass pinned host memory for the
 * overlap).  Verdict runs (flags 0, RTGPU method) stream: one persistent
 * kernel starts after the first chunk and waits per set on device-side
 * arrival flags the copy stream writes; its shared-memory layout is sized
 * from a sample of the batch and sets beyond it are re-run at the batch's
 * true sizes.  Other runs pipeline per-chunk launches over two streams.
 * e2e_num / den are written only with RTGPU_F_BOUNDS or RTGPU_F_DETAIL.
 * eval_budget <= 0 means unlimited (the search always ends: the allocation
 * space is finite); > 0 caps the task evaluations of an irregular set's
 * depth-first search (RTGPU_UNDECIDED beyond).  Returns 0 or a negative
 * error code.
 */
int rtgpu_analyze_host(const int64_t *blobs, const int64_t *set_off,
                       const int64_t *task_base, int64_t n_sets, int method,
                       unsigned flags, int64_t eval_budget, int32_t *status,
                       int64_t *evals, int32_t *vsm, int64_t *e2e_num,
                       int64_t *den, int64_t *detail);

/* Same on device-resident buffers, enqueued on `stream` (cudaStream_t or
 * NULL for the legacy default stream).  Asynchronous.  max_tasks / max_m /
 * max_p bound n, m and p over the batch (they size shared memory; a set
 * exceeding them reports RTGPU_INVALID). */
int rtgpu_analyze_device(const int64_t *d_blobs, const int64_t *d_set_off,
                         const int64_t *d_task_base, int64_t n_sets,
                         int max_tasks, int max_m, int max_p,
                         int method, unsigned flags, int64_t eval_budget,
                         int32_t *d_status, int64_t *d_evals, int32_t *d_vsm,
                         int64_t *d_e2e_num, int64_t *d_den,
                         int64_t *d_detail, void *stream);

/*
 * Point queries: the analysis building blocks on packed sets, one query per
 * warp.  The sets use the blob layout with explicit GPU response bounds:
 * every kernel is packed with GW = [2*GR_lo, 2*GR_up], GL = 0, alpha = 1
 * (alpha_den 1) and the engine gives it one physical SM, so Lemma 4 returns
 * exactly [GR_lo, GR_up].  A SuspTask (suspension.py:23) is packed as a
 * two-copy task whose copies carry its suspension bounds (even copies) and
 * zero (odd copies), with zero-length kernels.  Results are numerators over
 * den (a multiple of the input tick), RTGPU_NONE for None.
 *
 *   kind                      reference (file:line)            task / index / horizon / blocking
 *   RTGPU_Q_WORKLOAD          suspension.workload:107          k / h / t / -
 *   RTGPU_Q_MAX_WORKLOAD      suspension.max_workload:116      k / - / t / -
 *   RTGPU_Q_SEGMENT_RESPONSE  suspension.segment_response:140  k / j / - / blocking (hp = prio < k)
 *   RTGPU_Q_TASK_RESPONSE     suspension.task_response:155     k / - / - / blocking
 *   RTGPU_Q_MEM_RESPONSE      analysis.mem_response:156        k / j / - / -
 *   RTGPU_Q_CPU_RESPONSE      analysis.cpu_response:175        k / j / - / -
 *   RTGPU_Q_END_TO_END        analysis.end_to_end:191          k / - / - / -
 *   RTGPU_Q_MEM_WORKLOAD      analysis.mem_workload:109        i / h / t / -
 *   RTGPU_Q_CPU_WORKLOAD      analysis.cpu_workload:118        i / h / t / -
 *   RTGPU_Q_R2                end_to_end's R2 recurrence:214   k / - / base / -
 */
#define RTGPU_Q_WORKLOAD 0
#define RTGPU_Q_MAX_WORKLOAD 1
#define RTGPU_Q_SEGMENT_RESPONSE 2
#define RTGPU_Q_TASK_RESPONSE 3
#define RTGPU_Q_MEM_RESPONSE 4
#define RTGPU_Q_CPU_RESPONSE 5
#define RTGPU_Q_END_TO_END 6
#define RTGPU_Q_MEM_WORKLOAD 7
#define RTGPU_Q_CPU_WORKLOAD 8
#define RTGPU_Q_R2 9

#define RTGPU_GAP_ERROR 5 /* query status: the reference raises InfeasibleGapError */

typedef struct {
    int64_t set;      /* index of the set in the batch */
    int32_t kind;     /* RTGPU_Q_* */
    int32_t task;     /* task position in the blob (priority order) */
    int32_t index;    /* start segment h or segment j */
    int32_t pad;
    int64_t horizon;  /* window length t (ticks), or the R2 base */
    int64_t blocking; /* constant blocking term (ticks) */
} rtgpu_query;

int rtgpu_query_host(const int64_t *blobs, const int64_t *set_off, int64_t n_sets,
                     const rtgpu_query *queries, int64_t n_queries, int32_t *status,
                     int64_t *num, int64_t *den);

/* number of kernel launches the last rtgpu_analyze_* call enqueued */
int64_t rtgpu_last_launch_count(void);

/* Stage timing: when enabled, each rtgpu_analyze_* call records CUDA events
 * around its three stage kernels on the launching stream;
 * rtgpu_last_stage_ms (which synchronises on the last event) returns their
 * durations in ms and the number of sets each stage processed. */
void rtgpu_set_stage_timing(int enable);
int rtgpu_last_stage_ms(float *ms3, int64_t *sets3);

#ifdef __cplusplus
}
#endif

#endif /* RTGPU_H */
