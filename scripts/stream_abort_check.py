"""Run under `ncu` (which serialises kernels): the streamed end-to-end
verdict kernel waits for chunk copies queued behind it, its bounded wait
times out, the abort word stops every warp, and the host re-runs the batch
unstreamed.  Verdicts and allocations must still equal the device path's."""
import os
import sys
import time

import numpy as np
from fractions import Fraction

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2101_10463_b200 import _native  # noqa: E402
from paper_2101_10463_b200.engine import DeviceBatch, analyze_packed

gp = _native.gen_params_c(8, 5, (1000, 20000), (1000, 20000), (250, 5000), Fraction(1, 2), 0, 10,
                          Fraction(12, 100), Fraction(1), compact=True)
b, so, tb = _native.generate(gp, [f"abort:{i}" for i in range(40000)])
t0 = time.time()
h = analyze_packed(b, so, tb, 0, 0)
t1 = time.time()
batch = DeviceBatch(b, so, tb)
out = batch.alloc_results()
batch.run(out, flags=0)
g = out.to_host()
ok = np.array_equal(g.status, h.status) and np.array_equal(g.vsm, h.vsm)
print(f"streamed call {t1 - t0:.2f} s; undecided {int((h.status == 2).sum())}; equal to device path: {ok}")
assert ok
