/*
 * rtgpu_sim.h -- C-ABI of the batched discrete-event simulator
 * (csrc/simulator.cu): one preemptive fixed-priority CPU, one non-preemptive
 * fixed-priority bus and per-task dedicated virtual SMs, exactly the
 * semantics of the reference's gpusched.simulator.simulate
 * (/root/reference/pkg/src/gpusched/simulator.py:160) -- same event order,
 * same tie-breaking (finishes, then deadlines, then releases at equal
 * times; push order within a kind), same Mersenne-Twister draws for the
 * uniform length policy -- run on the GPU, one thread per simulation.
 *
 * Replaces: simulate() (simulator.py:160) for one task set (a batch of one,
 * the drop-in path) and for many (validation sweeps).  check_against_analysis
 * (simulator.py:340) is host post-processing over the returned trace; the
 * per-task maxima below give the same verdict for whole batches.
 *
 * Times are integers: every duration, period, deadline and the horizon is
 * scaled by one per-simulation factor Q chosen by the caller so that all of
 * them (and the uniform policy's GPU durations work*A + B) are integral.
 */
#ifndef RTGPU_SIM_H
#define RTGPU_SIM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- input: one blob of int64 words per simulation -----------------------
 * header (RTGPU_SIM_HDR words):
 *   [0] n_tasks (<= 64)      [1] policy (0 worst case, 1 uniform random)
 *   [2] horizon (scaled)     [3] release points R (sum over tasks)
 *   [4] event capacity       [5] MT19937 key length L (uniform only)
 *   [6] S_max (longest job segment plan)
 *   [7] word offset of the key from the blob start: L words, the 32-bit
 *       init_by_array key random.Random(seed) derives from the seed
 *   [8] job-record pool size P (0 = R): records of finished jobs past
 *       their deadline are recycled; a run needing more than P live jobs
 *       stops with RTGPU_SIM_POOL_OVERFLOW (re-run it with P = R)
 *   [9..15] reserved
 * task records (RTGPU_SIM_TASK words, priority order, highest first):
 *   [0] S plan length  [1] period  [2] deadline  [3] priority
 *   [4] word offset of the task's plan entries from the blob start
 *   [5] CPU segments m  [6..7] reserved
 * plan entries (RTGPU_SIM_SEG words each, job_segment_plan order,
 * simulator.py:106):
 *   [0] kind | index << 8 | random << 16   (kind 0 cpu, 1 mem, 2 gpu)
 *   [1] lo  [2] hi   (integer bounds for randint when random)
 *   [3] fixed duration (scaled; used when not random)
 *   [4] A  [5] B     (random: duration = randint(lo, hi) * A + B, scaled)
 */
#define RTGPU_SIM_HDR 16
#define RTGPU_SIM_TASK 8
#define RTGPU_SIM_SEG 6
#define RTGPU_SIM_MAX_TASKS 64
#define RTGPU_SIM_MAX_KEY 4096

/* event actions and kinds (SimEvent.action / .kind) */
enum { RTGPU_EV_RELEASE = 0, RTGPU_EV_START, RTGPU_EV_PREEMPT, RTGPU_EV_RESUME, RTGPU_EV_FINISH,
       RTGPU_EV_DEADLINE_MISS };
enum { RTGPU_KIND_CPU = 0, RTGPU_KIND_MEM, RTGPU_KIND_GPU, RTGPU_KIND_JOB };

/* per-simulation status */
enum { RTGPU_SIM_OK = 0, RTGPU_SIM_BAD_INPUT = 1, RTGPU_SIM_EVENT_OVERFLOW = 2,
       RTGPU_SIM_POOL_OVERFLOW = 3 };

/* One event: time (scaled) and packed fields
 *   bits 0..31 job index, 32..39 task (priority order), 40..43 kind,
 *   44..47 action, 48..55 segment + 1 (0 = job-level event). */
typedef struct {
    int64_t time;
    uint64_t packed;
} rtgpu_sim_event;

/* Outputs.  Per simulation s: status[s], n_events[s], misses[s] (deadline-
 * miss events).  Per job slot j in [job_base[s], job_base[s+1]) -- slots in
 * release order (time, then priority): job_task, job_k, job_resp (end-to-end
 * response, scaled; -1 if unfinished at the horizon = truncated) and
 * job_rank (completion order; -1 if unfinished).  Per task i in
 * [task_base[s], task_base[s+1]) and plan position: seg_max[i * s_max + pos]
 * = largest start-to-finish response of that segment over finished jobs
 * (-1 if none; what check_against_analysis compares per segment) and
 * resp_max[i] over finished jobs.  events (optional, may be NULL): events
 * of simulation s at ev_base[s] .. ev_base[s] + n_events[s]. */
typedef struct {
    int32_t *status;
    int64_t *n_events;
    int64_t *misses;
    int32_t *job_task;
    int32_t *job_k;
    int64_t *job_resp;
    int32_t *job_rank;
    int64_t *seg_max;
    int64_t *resp_max;
    rtgpu_sim_event *events;
} rtgpu_sim_out;

/* Scratch words simulation s needs (device working state: jobs, queues,
 * Mersenne-Twister state). */
int64_t rtgpu_sim_scratch_words(const int64_t *blob);

/* Host path: host buffers in, host buffers out (copies inside).  set_off,
 * job_base, task_base, ev_base: n_sims + 1 entries (ev_base may be NULL when
 * out->events is NULL).  s_max: stride of seg_max.  0 on success. */
int rtgpu_sim_host(const int64_t *blobs, const int64_t *set_off, int64_t n_sims,
                   const int64_t *job_base, const int64_t *task_base, const int64_t *ev_base,
                   int32_t s_max, rtgpu_sim_out *out);

/* Device path: every pointer (including those inside *out) is device
 * memory; scratch holds sum of rtgpu_sim_scratch_words at scr_off[s].
 * order (may be NULL): a permutation of the simulations, started in that
 * order -- longest first (e.g. by event capacity) list-schedules the batch. */
int rtgpu_sim_device(const int64_t *blobs, const int64_t *set_off, int64_t n_sims,
                     const int64_t *job_base, const int64_t *task_base, const int64_t *ev_base,
                     const int64_t *scr_off, int64_t *scratch, const int64_t *order,
                     int32_t s_max, const rtgpu_sim_out *out, void *stream);

const char *rtgpu_sim_last_error(void);

#ifdef __cplusplus
}
#endif

#endif
