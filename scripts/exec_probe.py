"""Interference probe for the executor kernel (see rtgpu_exec_probe)."""
import ctypes
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2101_10463_b200 import executor as ex  # noqa: E402

L = ex._lib()
L.rtgpu_exec_probe.argtypes = [ctypes.POINTER(ctypes.c_uint32), ctypes.c_int, ctypes.c_int64,
                               ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64,
                               ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_float)]
reps = 60
for sms, bg in (([0], [1]), ([0], range(1, 148)), ([0], range(2, 148)), ([0], [2, 3, 4]),
                ([2], [0, 1, 3, 4]), ([74], [75])):
    out = (ctypes.c_float * reps)()
    rc = L.rtgpu_exec_probe(ex.mask_of(sms), 2, 500, 2048, reps, 3, 4 << 20, ex.mask_of(bg), out)
    a = np.array(out[:])
    print(sms, "bg", list(bg)[:6], "rc", rc, "span us min/med/max", a.min().round(1),
          np.median(a).round(1), a.max().round(1), flush=True)
