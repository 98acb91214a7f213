/* rtgpu_k_f64.cu -- stage kernel instantiated for V = double (see kernel.cuh). */
#define RTGPU_FRONT_TU 1
#include "kernel.cuh"

namespace rtgpu {
int launch_front_f64(const KParams &p, cudaStream_t st) { return launch_front(p, st); }
int launch_stage_f64(const KParams &p, int stage, cudaStream_t st) { return launch_stage<double>(p, stage, st); }
int launch_query_f64(const QParams &p, int stage, cudaStream_t st) { return launch_query_stage<double>(p, stage, st); }
}  // namespace rtgpu
