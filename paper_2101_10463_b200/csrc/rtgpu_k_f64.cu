/* rtgpu_k_f64.cu -- stage kernel instantiated for V = double (see kernel.cuh). */
#include "kernel.cuh"

namespace rtgpu {
int launch_stage_f64(const KParams &p, int stage, cudaStream_t st) { return launch_stage<double>(p, stage, st); }
}  // namespace rtgpu
