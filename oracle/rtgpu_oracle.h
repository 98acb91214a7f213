/* rtgpu_oracle.h -- TEST INFRASTRUCTURE ONLY (see rtgpu_oracle.c). */
#ifndef RTGPU_ORACLE_H
#define RTGPU_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif
/* One packed set (include/rtgpu.h layout); outputs for that set only. */
int oracle_analyze_set(const int64_t *blob, int method, unsigned flags, int64_t budget,
                       int32_t *status, int64_t *evals, int32_t *vsm, int64_t *e2e_num,
                       int64_t *den, int64_t *blob_detail);
/* A batch, same argument meaning as rtgpu_analyze_host, on n_threads host threads. */
int oracle_analyze_batch(const int64_t *blobs, const int64_t *set_off, const int64_t *task_base,
                         int64_t n_sets, int method, unsigned flags, int64_t budget,
                         int n_threads, int32_t *status, int64_t *evals, int32_t *vsm,
                         int64_t *e2e_num, int64_t *den, int64_t *detail);
#ifdef __cplusplus
}
#endif
#endif
