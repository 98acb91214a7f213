"""Algorithmic work of the lattice path per task set (host harness built with
RT_COUNTERS; no GPU): fixed points and iterations by resource and mode,
walks, count evaluations.  python scripts/lat_counters.py [sweep16x9|alloc64] [sets]"""
import ctypes
import os
import subprocess
import sys
from fractions import Fraction

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2101_10463_b200 import _native  # noqa: E402
from paper_2101_10463_b200.distributed import concat_batches  # noqa: E402
sys.path.insert(0, os.path.join(ROOT, "tests"))
from harness import harness  # noqa: E402

LIB = "/tmp/libenginehost_cnt.so"
subprocess.run(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-DRT_COUNTERS", *(sys.argv[3].split() if len(sys.argv) > 3 else []), "-o", LIB,
                harness.SRC], check=True)
harness._lib = None
harness.LIB = LIB
harness.build = lambda: LIB
lib = harness.lib()
lib.host_counters.argtypes = [ctypes.POINTER(ctypes.c_longlong), ctypes.c_int]

name = sys.argv[1] if len(sys.argv) > 1 else "sweep16x9"
per = int(sys.argv[2]) if len(sys.argv) > 2 else 40
n, ms, gn, den = {"sweep16x9": (16, range(2, 10), 148, 20), "alloc64": (64, [5], 148, 20),
                  "sweep8x5": (8, [5], 10, 10)}[name]
parts = []
for m in ms:
    for k in range(1, 11):
        u = Fraction(k, den)
        gp = _native.gen_params_c(n, m, (1000, 20000), (1000, 20000), (250, 5000), u, 0, gn,
                                  Fraction(12, 100), Fraction(1), compact=True)
        parts.append(_native.generate(gp, [f"1000:{u}:{i}" for i in range(per)]))
b, so, tb = concat_batches(parts)
S = len(so) - 1
cnt = (ctypes.c_longlong * 22)()
lib.host_counters(cnt, 1)
if name == "sweep8x5" and not os.environ.get("LAT"):  # the fast path (fast_verdict), as the fast kernel runs it
    out = harness.analyze_batch(b, so, tb, flags=0, detail=False)
else:
    out = harness.lattice_batch(b, so, tb)
lib.host_counters(cnt, 0)
v = list(cnt)
names = ["interf0", "interf1", "lfp0", "R2_full_lfp", "allquick_sets", "rounds", "site_guessfail", "site_rmaxexact", "fit0", "fit1",
         "walks", "passes", "lat_lfp_cpu", "lat_lfp_mem", "lat_pre_cpu", "lat_pre_mem", "lat_it_cpu",
         "lat_it_mem", "lat_preit_cpu", "lat_preit_mem", "site_summr_chains", "site_sumcr_chains"]
print(f"{name}: {S} sets, sched {(out['status'] == 1).sum()}, esc {(out['status'] == 99).sum()}")
for k, x in zip(names, v):
    if x == 0:
        continue
    print(f"  {k:12s} {x / S:10.2f} per set")
