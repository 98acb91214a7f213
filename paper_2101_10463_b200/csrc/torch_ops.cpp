/*
 * torch_ops.cpp -- the engine's device entry point as a PyTorch operator:
 * torch.ops.rtgpu.analyze_out runs rtgpu_analyze_device (include/rtgpu.h)
 * on CUDA tensors, enqueued on PyTorch's current stream of the tensors'
 * device, so it orders with the caller's other work like any torch op.
 * A thin shim over the C-ABI (no analysis code here): argument checks,
 * the stream, and the error text of a failed call.
 */
#include <ATen/ATen.h>
#include <c10/cuda/CUDAGuard.h>
#include <c10/cuda/CUDAStream.h>
#include <torch/library.h>

#include "rtgpu.h"

namespace {

void check(const at::Tensor &t, at::ScalarType ty, const char *name, const at::Device &dev) {
    TORCH_CHECK(t.is_cuda(), name, " must be a CUDA tensor");
    TORCH_CHECK(t.device() == dev, name, " must be on ", dev);
    TORCH_CHECK(t.scalar_type() == ty, name, " has dtype ", t.scalar_type(), ", expected ", ty);
    TORCH_CHECK(t.is_contiguous(), name, " must be contiguous");
}

/* analysis of the packed batch (blobs, set_off, task_base) into the
 * caller's result tensors; detail may be an empty tensor */
void analyze_out(const at::Tensor &blobs, const at::Tensor &set_off, const at::Tensor &task_base,
                 int64_t max_tasks, int64_t max_m, int64_t max_p, int64_t method, int64_t flags,
                 int64_t budget, at::Tensor &status, at::Tensor &evals, at::Tensor &vsm, at::Tensor &e2e_num,
                 at::Tensor &den, at::Tensor &detail) {
    const at::Device dev = blobs.device();
    check(blobs, at::kLong, "blobs", dev);
    check(set_off, at::kLong, "set_off", dev);
    check(task_base, at::kLong, "task_base", dev);
    check(status, at::kInt, "status", dev);
    check(evals, at::kLong, "evals", dev);
    check(vsm, at::kInt, "vsm", dev);
    check(e2e_num, at::kLong, "e2e_num", dev);
    check(den, at::kLong, "den", dev);
    const int64_t S = set_off.numel() - 1;
    TORCH_CHECK(S >= 0 && task_base.numel() == S + 1, "set_off / task_base sizes");
    TORCH_CHECK(status.numel() >= S && evals.numel() >= S, "status / evals too small");
    const bool want_detail = (flags & RTGPU_F_DETAIL) != 0;
    if (want_detail) {
        check(detail, at::kLong, "detail", dev);
        TORCH_CHECK(detail.numel() >= blobs.numel(), "detail must be blob-shaped");
    }
    c10::cuda::CUDAGuard guard(dev);
    cudaStream_t st = c10::cuda::getCurrentCUDAStream(dev.index()).stream();
    const int rc = rtgpu_analyze_device(
        blobs.data_ptr<int64_t>(), set_off.data_ptr<int64_t>(), task_base.data_ptr<int64_t>(), S,
        (int)max_tasks, (int)max_m, (int)max_p, (int)method, (unsigned)flags, budget,
        status.data_ptr<int32_t>(), evals.data_ptr<int64_t>(), vsm.data_ptr<int32_t>(),
        e2e_num.data_ptr<int64_t>(), den.data_ptr<int64_t>(),
        want_detail ? detail.data_ptr<int64_t>() : nullptr, (void *)st);
    TORCH_CHECK(rc == 0, "rtgpu_analyze_device failed (", rc, "): ", rtgpu_last_error());
}

}  // namespace

TORCH_LIBRARY(rtgpu, m) {
    m.def("analyze_out(Tensor blobs, Tensor set_off, Tensor task_base, int max_tasks, int max_m, "
          "int max_p, int method, int flags, int budget, Tensor(a!) status, Tensor(b!) evals, "
          "Tensor(c!) vsm, Tensor(d!) e2e_num, Tensor(e!) den, Tensor(f!) detail) -> ()");
}

TORCH_LIBRARY_IMPL(rtgpu, CUDA, m) { m.impl("analyze_out", &analyze_out); }
