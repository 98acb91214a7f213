"""Randomised verdict parity: GPU fast path / streamed e2e vs the oracle's
greedy mode (equal to full enumeration, tests/test_fullsize.py) over many
shapes.  python scripts/parity_sweep.py [sets_per_shape]"""
import random
import sys
import time
from fractions import Fraction

import numpy as np

sys.path.insert(0, ".")
from oracle import oracle  # noqa: E402
from paper_2101_10463_b200 import _native  # noqa: E402
from paper_2101_10463_b200.engine import DeviceBatch, analyze_packed  # noqa: E402

GREEDY = 0x100
per = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 2101)
total = bad = 0
t0 = time.time()
for shape in range(40):
    n, m = rng.randint(2, 12), rng.randint(1, 6)
    gn = rng.randint(max(2, n // 2), 24)
    u = Fraction(rng.randint(2, 12), 10) * n / 8  # around the schedulability boundary
    mm = rng.randint(0, 1)
    lo = Fraction(rng.choice([10, 10, 7, 5]), 10)
    gp = _native.gen_params_c(n, m, (1000, 20000), (1000, 20000), (250, 5000), u, mm, gn,
                              Fraction(12, 100), lo, compact=True)
    b, so, tb = _native.generate(gp, [f"par:{shape}:{i}" for i in range(per)])
    o = oracle.analyze_batch(b, so, tb, flags=1 | GREEDY, threads=16, detail=False)
    batch = DeviceBatch(b, so, tb)
    out = batch.alloc_results()
    batch.run(out, flags=0)
    g = out.to_host()
    h = analyze_packed(b, so, tb, 0, 0)
    sched = np.repeat(o["status"] == 1, np.diff(tb))
    ok = (np.array_equal(o["status"], g.status) and np.array_equal(o["vsm"][sched], g.vsm[sched])
          and np.array_equal(g.status, h.status) and np.array_equal(g.vsm, h.vsm))
    total += per
    if not ok:
        bad += 1
        diff = np.nonzero(o["status"] != g.status)[0][:5]
        print("MISMATCH", dict(n=n, m=m, gn=gn, u=str(u), mm=mm, lo=str(lo)), diff, flush=True)
    print(f"shape {shape}: n={n} m={m} gn={gn} u={u} mm={mm} lo={lo} "
          f"sched={float(np.mean(o['status'] == 1)):.2f} ok={ok}", flush=True)
print(f"{total} sets over 40 shapes, {bad} mismatching shapes, {time.time() - t0:.0f} s")
