/*
 * rtgpu_gen.h -- C-ABI of the bulk task-set generator (host code).
 *
 * Replaces gpusched.workbench.generate_taskset (workbench.py:101) for bulk
 * use: for the same parameters and seed it produces the same task set,
 * written straight into the engine's blob layout (include/rtgpu.h), tasks in
 * priority order.  Seeds are Python int seeds or Python str seeds (the
 * sweep's cell seeds "master:utilization:index", workbench.py:220).
 */
#ifndef RTGPU_GEN_H
#define RTGPU_GEN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* GenParams (workbench.py:43); Fractions as num/den; mem range already
 * resolved through GenParams.effective_mem_range(). */
typedef struct {
    int32_t n_tasks, n_subtasks;
    int64_t cpu_lo, cpu_hi, gpu_lo, gpu_hi, mem_lo, mem_hi;
    int64_t util_num, util_den;
    int32_t mem_model; /* RTGPU_TWO_COPY / RTGPU_ONE_COPY */
    int32_t physical_sms;
    int64_t eps_num, eps_den;       /* launch_overhead_frac */
    int64_t lofrac_num, lofrac_den; /* lo_frac */
    int32_t seg_int32;              /* 1: compact blobs (int32 segment areas) */
    int32_t pad;
} rtgpu_gen_params;

/* words of one generated blob (all sets of a call have the same size) */
int64_t rtgpu_gen_blob_words(const rtgpu_gen_params *p);

/* Generate n_sets task sets; exactly one of int_seeds / str_seeds is
 * non-null.  blobs must hold n_sets * rtgpu_gen_blob_words(p) words;
 * set_off / task_base receive n_sets + 1 entries.  0 on success. */
int rtgpu_generate(const rtgpu_gen_params *p, int64_t n_sets, const int64_t *int_seeds,
                   const char *const *str_seeds, int n_threads, int64_t *blobs,
                   int64_t *set_off, int64_t *task_base);

void rtgpu_sha512(const unsigned char *msg, int64_t len, unsigned char *out64);

#ifdef __cplusplus
}
#endif

#endif
