"""A/B timing of the lattice path on the 148-SM shapes and the bounds run
(resident inputs, CUDA events): python scripts/lat_ab.py [reps]
Select a library build with RTGPU_LIB=path."""
import os
import sys
import time
from fractions import Fraction

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2101_10463_b200 import _native  # noqa: E402
from paper_2101_10463_b200.engine import DeviceBatch  # noqa: E402
from paper_2101_10463_b200.pack import F_BOUNDS  # noqa: E402


def gen(n, ms, gn, utils, per):
    from paper_2101_10463_b200.distributed import concat_batches
    parts = []
    for m in ms:
        for u in utils:
            gp = _native.gen_params_c(n, m, (1000, 20000), (1000, 20000), (250, 5000), u, 0, gn,
                                      Fraction(12, 100), Fraction(1), compact=True)
            parts.append(_native.generate(gp, [f"1000:{u}:{i}" for i in range(per)]))
    return concat_batches(parts)


U20 = [Fraction(k, 20) for k in range(1, 11)]
U10 = [Fraction(k, 10) for k in range(1, 11)]
cases = {"sweep16x9": (16, list(range(2, 10)), 148, U20, 2500, 0),
         "alloc64": (64, [5], 148, U20, 2000, 0),
         "bounds8x5": (8, [5], 10, U10, 10000, F_BOUNDS),
         "verdict8x5": (8, [5], 10, U10, 10000, 0)}
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
want = sys.argv[2].split(",") if len(sys.argv) > 2 else list(cases)
for name in want:
    n, ms, gn, utils, per, flags = cases[name]
    b, so, tb = gen(n, ms, gn, utils, per)
    batch = DeviceBatch(b, so, tb)
    out = batch.alloc_results()
    st = torch.cuda.current_stream()
    batch.run(out, flags=flags, stream=st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        batch.run(out, flags=flags, stream=st)
    e1.record(st)
    torch.cuda.synchronize()
    ms_ = e0.elapsed_time(e1) / reps
    S = len(so) - 1
    sched = int((out.status == 1).sum().item())
    print(f"{name:10s} {S:7d} sets  {ms_:8.2f} ms  {S / ms_ / 1e3:7.3f} M sets/s  sched {sched}  "
          f"lib {os.path.basename(os.environ.get('RTGPU_LIB', 'librtgpu.so'))}", flush=True)
