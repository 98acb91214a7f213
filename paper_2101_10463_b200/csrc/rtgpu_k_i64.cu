/* rtgpu_k_i64.cu -- stage kernel instantiated for V = i64 (see kernel.cuh). */
#include "kernel.cuh"

namespace rtgpu {
int launch_stage_i64(const KParams &p, int stage, cudaStream_t st) { return launch_stage<i64>(p, stage, st); }
int launch_fast_list_i64(const KParams &p, cudaStream_t st) { return launch_fast_list<i64>(p, st); }
int launch_query_i64(const QParams &p, int stage, cudaStream_t st) { return launch_query_stage<i64>(p, stage, st); }
}  // namespace rtgpu
