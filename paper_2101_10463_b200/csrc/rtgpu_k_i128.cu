/* rtgpu_k_i128.cu -- stage kernel instantiated for V = i128 (see kernel.cuh). */
#include "kernel.cuh"

namespace rtgpu {
int launch_stage_i128(const KParams &p, int stage, cudaStream_t st) { return launch_stage<i128>(p, stage, st); }
int launch_query_i128(const QParams &p, int stage, cudaStream_t st) { return launch_query_stage<i128>(p, stage, st); }
}  // namespace rtgpu
