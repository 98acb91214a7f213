"""Batched, device-resident front end of the CUDA engine.

``DeviceBatch`` keeps a packed batch of task sets in HBM (torch tensors are
used only as device allocations) and runs the allocation search +
response-time analysis on it with ``rtgpu_analyze_device`` on a CUDA stream.
``analyze_packed`` is the end-to-end path from host buffers (pinned or not)
through ``rtgpu_analyze_host``.
"""
from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _native
from .pack import F_BOUNDS, F_DETAIL, RawResults

METHOD_RTGPU, METHOD_SELFSUSP, METHOD_BUSYWAIT = 0, 1, 2

_OP_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "rtgpu_torch.so")
_op = None


def torch_op():
    """torch.ops.rtgpu.analyze_out (csrc/torch_ops.cpp: rtgpu_analyze_device as
    a PyTorch operator on the current stream), or None when an A/B build is
    selected with RTGPU_LIB (the operator links the in-tree library) or the
    operator is not built."""
    global _op
    if _op is None:
        if os.environ.get("RTGPU_LIB") or not os.path.exists(_OP_PATH):
            _op = False
        else:
            import torch
            _native.lib()  # the same librtgpu.so instance the operator links
            torch.ops.load_library(_OP_PATH)
            _op = torch.ops.rtgpu.analyze_out
    return _op or None


def batch_dims(blobs: np.ndarray, set_off: np.ndarray) -> tuple[int, int, int]:
    """(max tasks, max CPU segments, max memory segments) over a batch."""
    hdr = np.asarray(set_off[:-1], dtype=np.int64)
    if len(hdr) == 0:
        return (1, 1, 0)
    n = blobs[hdr]
    mc = blobs[hdr + 5]
    mp = blobs[hdr + 6]
    return (max(1, int(n.max())), max(1, int(mc.max())), int(mp.max()))


@dataclass
class DeviceResults:
    status: "object"   # torch int32 [S]
    evals: "object"    # torch int64 [S]
    vsm: "object"      # torch int32 [T]
    e2e_num: "object"  # torch int64 [T]
    den: "object"      # torch int64 [T]
    detail: Optional["object"] = None

    def to_host(self) -> RawResults:
        return RawResults(self.status.cpu().numpy(), self.evals.cpu().numpy(),
                          self.vsm.cpu().numpy(), self.e2e_num.cpu().numpy(),
                          self.den.cpu().numpy(),
                          None if self.detail is None else self.detail.cpu().numpy())


class DeviceBatch:
    """A packed batch resident on one CUDA device."""

    def __init__(self, blobs: np.ndarray, set_off: np.ndarray, task_base: np.ndarray,
                 device: str = "cuda"):
        import torch
        _native.require_device()
        self.device = torch.device(device)
        self.n_sets = len(set_off) - 1
        self.n_tasks = int(task_base[-1])
        self.words = int(set_off[-1])
        self.dims = batch_dims(blobs, set_off)
        self.blobs = torch.from_numpy(np.ascontiguousarray(blobs, np.int64)).to(self.device)
        self.set_off = torch.from_numpy(np.ascontiguousarray(set_off, np.int64)).to(self.device)
        self.task_base = torch.from_numpy(np.ascontiguousarray(task_base, np.int64)).to(self.device)
        self.input_bytes = 8 * (self.words + 2 * (self.n_sets + 1))

    def alloc_results(self, detail: bool = False) -> DeviceResults:
        import torch
        d = self.device
        return DeviceResults(
            torch.empty(self.n_sets, dtype=torch.int32, device=d),
            torch.empty(self.n_sets, dtype=torch.int64, device=d),
            torch.empty(self.n_tasks, dtype=torch.int32, device=d),
            torch.empty(self.n_tasks, dtype=torch.int64, device=d),
            torch.empty(self.n_tasks, dtype=torch.int64, device=d),
            torch.empty(self.words, dtype=torch.int64, device=d) if detail else None)

    def _no_detail(self):
        import torch
        if getattr(self, "_empty", None) is None:
            self._empty = torch.empty(0, dtype=torch.int64, device=self.device)
        return self._empty

    def output_bytes(self, flags: int) -> int:
        b = 4 * self.n_sets + 8 * self.n_sets + 4 * self.n_tasks
        if flags & (F_BOUNDS | F_DETAIL):
            b += 16 * self.n_tasks
        if flags & F_DETAIL:
            b += 8 * self.words
        return b

    def run(self, out: DeviceResults, method: int = METHOD_RTGPU, flags: int = 0,
            budget: int = 0, stream=None) -> None:
        """Enqueue the analysis on `stream` (default: torch's current stream)."""
        import torch
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        op = torch_op()
        if op is not None:
            with torch.cuda.stream(stream):
                op(self.blobs, self.set_off, self.task_base, self.dims[0], self.dims[1], self.dims[2],
                   method, flags, budget, out.status, out.evals, out.vsm, out.e2e_num, out.den,
                   out.detail if out.detail is not None else self._no_detail())
            return
        _native.analyze_device(
            self.blobs.data_ptr(), self.set_off.data_ptr(), self.task_base.data_ptr(),
            self.n_sets, self.dims, method, flags, budget, out.status.data_ptr(),
            out.evals.data_ptr(), out.vsm.data_ptr(), out.e2e_num.data_ptr(),
            out.den.data_ptr(), out.detail.data_ptr() if out.detail is not None else None,
            stream.cuda_stream)


def analyze_packed(blobs: np.ndarray, set_off: np.ndarray, task_base: np.ndarray,
                   method: int = METHOD_RTGPU, flags: int = F_DETAIL, budget: int = 0) -> RawResults:
    """End-to-end: host buffers in, host results out (rtgpu_analyze_host)."""
    out = _native.analyze_host(blobs, set_off, task_base, method, flags, budget,
                               detail=bool(flags & F_DETAIL))
    return RawResults(out["status"], out["evals"], out["vsm"], out["e2e_num"], out["den"],
                      out["detail"])
