"""The bulk generator (csrc/taskgen.cpp) reproduces the reference generator
(workbench.generate_taskset) bit for bit: every 'gen' golden case, generated
by the reference with int and str seeds, is re-generated and packed."""
from fractions import Fraction

import numpy as np

from golden_io import load_cases, ts_from_exact
from paper_2101_10463_b200 import _native
from paper_2101_10463_b200.pack import pack_tasksets


def test_generator_matches_reference_golden():
    cases = [c for c in load_cases() if c["kind"] == "gen"]
    assert len(cases) > 100
    assert any(isinstance(c["seed"], str) for c in cases)
    bad = []
    for c in cases:
        p = c["params"]
        gpu = tuple(p.get("gpu", (1000, 20000)))
        mem = (max(1, gpu[0] // 4), gpu[1] // 4)
        gp = _native.gen_params_c(p["n"], p["m"], (1000, 20000), gpu, mem, Fraction(p["u"]),
                                  0 if p["mm"] == "two_copy" else 1, p["gn"], Fraction(12, 100),
                                  Fraction(p["lo"]))
        blobs, _, _ = _native.generate(gp, [c["seed"]])
        ref = pack_tasksets([ts_from_exact(c["taskset"])])
        if not np.array_equal(blobs, ref.blobs):
            bad.append((c["seed"], p))
    assert not bad, bad[:3]


def test_generator_threads_deterministic():
    gp = _native.gen_params_c(8, 5, (1000, 20000), (1000, 20000), (250, 5000), Fraction(1, 2), 0,
                              10, Fraction(12, 100), Fraction(1))
    a = _native.generate(gp, list(range(300)), n_threads=1)[0]
    b = _native.generate(gp, list(range(300)), n_threads=7)[0]
    assert np.array_equal(a, b)
