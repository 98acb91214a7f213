"""The end-to-end verdict call's stream timeline (RTGPU_E2E_TRACE=1) on the
benchmark batch: python scripts/e2e_trace.py [reps]"""
import ctypes
import os
import sys
import time
from fractions import Fraction

os.environ["RTGPU_E2E_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2101_10463_b200 import _native  # noqa: E402

wl = bench.WORKLOADS["sweep8x5"]
blobs, set_off, task_base = bench.gen_workload(wl, 1000, bench.cell_indices(wl, 0, 1))
S, T = len(set_off) - 1, int(task_base[-1])
pin = torch.empty(len(blobs), dtype=torch.int64, pin_memory=True)
pin.numpy()[:] = blobs
po = torch.empty(len(set_off), dtype=torch.int64, pin_memory=True)
po.numpy()[:] = set_off
pt = torch.empty(len(task_base), dtype=torch.int64, pin_memory=True)
pt.numpy()[:] = task_base
st = torch.empty(S, dtype=torch.int32, pin_memory=True).numpy()
ev = torch.empty(S, dtype=torch.int64, pin_memory=True).numpy()
vs = torch.empty(T, dtype=torch.int32, pin_memory=True).numpy()
e2 = torch.empty(T, dtype=torch.int64, pin_memory=True).numpy()
dn = torch.empty(T, dtype=torch.int64, pin_memory=True).numpy()
L = _native.lib()
P = lambda a, ty: a.ctypes.data_as(ctypes.POINTER(ty))  # noqa: E731
args = (P(pin.numpy(), ctypes.c_int64), P(po.numpy(), ctypes.c_int64), P(pt.numpy(), ctypes.c_int64), S, 0, 0, 0,
        P(st, ctypes.c_int32), P(ev, ctypes.c_int64), P(vs, ctypes.c_int32), P(e2, ctypes.c_int64),
        P(dn, ctypes.c_int64), None)
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 5):
    t0 = time.perf_counter()
    rc = L.rtgpu_analyze_host(*args)
    dt = time.perf_counter() - t0
    print(f"call {i}: rc {rc} host wall {dt * 1e3:.3f} ms ({S / dt / 1e6:.2f} M sets/s)", file=sys.stderr, flush=True)
