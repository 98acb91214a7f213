"""Parity of the CUDA engine (librtgpu.so on the B200) with the reference:
golden reports produced by the reference itself, and the oracle on the
reference generator's task sets.  Bit-exact: verdicts, allocations and every
bound as an exact rational."""
from fractions import Fraction

import numpy as np
import pytest

from golden_io import load_cases, ts_from_exact
from oracle import oracle
from paper_2101_10463_b200 import _native
from paper_2101_10463_b200.analysis import analyze_batch, analyze_rtgpu
from paper_2101_10463_b200.engine import DeviceBatch, analyze_packed
from paper_2101_10463_b200.model import AnalysisMethod, report_to_dict
from paper_2101_10463_b200.pack import (F_BOUNDS, F_DETAIL, INVALID, pack_tasksets,
                                        unpack_report)

pytestmark = pytest.mark.gpu

F_FIRST_I64, F_FIRST_I128 = 4, 8


@pytest.fixture(scope="module")
def golden():
    cases = load_cases()
    return cases, pack_tasksets([ts_from_exact(c["taskset"]) for c in cases])


METHODS = [AnalysisMethod.RTGPU, AnalysisMethod.SELF_SUSPENSION, AnalysisMethod.BUSY_WAITING]


def _check_golden(cases, batch, res, method=AnalysisMethod.RTGPU):
    bad = []
    for s, c in enumerate(cases):
        want = c[method.value]
        if "raises" in want:
            if res.status[s] != INVALID:
                bad.append(s)
            continue
        if report_to_dict(unpack_report(batch, res, s, method)) != want:
            bad.append(s)
    return bad


@pytest.mark.parametrize("mi", [0, 1, 2])
@pytest.mark.parametrize("first", [0, F_FIRST_I64, F_FIRST_I128])
def test_gpu_matches_reference_reports(golden, first, mi):
    cases, batch = golden
    res = analyze_packed(batch.blobs, batch.set_off, batch.task_base, mi, F_DETAIL | first)
    assert not _check_golden(cases, batch, res, METHODS[mi])
    assert _native.last_launch_count() >= 3


def test_dropin_api_matches_reference(golden):
    cases, _ = golden
    some = [c for c in cases if "raises" not in c["rtgpu"]][:60]
    for c in some:
        got = report_to_dict(analyze_rtgpu(ts_from_exact(c["taskset"])))
        assert got == c["rtgpu"]
    reps = analyze_batch([ts_from_exact(c["taskset"]) for c in some])
    assert [report_to_dict(r) for r in reps] == [c["rtgpu"] for c in some]


def _cmp(o, g_status, g_vsm, g_e2e, g_den):
    assert np.array_equal(o["status"], g_status)
    assert np.array_equal(o["vsm"], g_vsm)
    for i in range(len(o["e2e_num"])):
        a, b = int(o["e2e_num"][i]), int(g_e2e[i])
        if a < 0 or b < 0:
            assert a == b, i
        else:
            assert Fraction(a, int(o["den"][i])) == Fraction(b, int(g_den[i])), i


@pytest.mark.parametrize("mi", [1, 2])
@pytest.mark.parametrize("n,m,gn,u", [(8, 5, 10, "2/5"), (5, 3, 10, "1"), (6, 2, 12, "4/5")])
def test_gpu_baselines_match_oracle(n, m, gn, u, mi):
    gp = _native.gen_params_c(n, m, (1000, 20000), (1000, 20000), (250, 5000), Fraction(u), 0,
                              gn, Fraction(12, 100), Fraction(1))
    b, so, tb = _native.generate(gp, [f"5:{u}:{i}" for i in range(300)])
    o = oracle.analyze_batch(b, so, tb, method=mi, flags=1, threads=8, detail=False)
    batch = DeviceBatch(b, so, tb)
    out = batch.alloc_results()
    batch.run(out, method=mi, flags=F_BOUNDS)
    g = out.to_host()
    _cmp({k: v for k, v in o.items() if k not in ("detail", "evals")},
         g.status, g.vsm, g.e2e_num, g.den)


@pytest.mark.parametrize("n,m,gn,u,mm,lo", [
    (8, 5, 10, "1/5", 0, "1"), (8, 5, 10, "2/5", 0, "1"), (8, 5, 10, "3/5", 0, "1"),
    (8, 5, 10, "4/5", 1, "7/10"), (5, 5, 10, "1/2", 1, "1"), (5, 3, 10, "1", 0, "3/5"),
    (3, 3, 4, "1", 1, "1"), (6, 2, 20, "4/5", 0, "1"), (10, 4, 16, "1/2", 0, "1")])
def test_gpu_matches_oracle_generated(n, m, gn, u, mm, lo):
    gp = _native.gen_params_c(n, m, (1000, 20000), (1000, 20000), (250, 5000), Fraction(u), mm,
                              gn, Fraction(12, 100), Fraction(lo))
    seeds = [f"9:{u}:{i}" for i in range(400)]
    b, so, tb = _native.generate(gp, seeds)
    o = oracle.analyze_batch(b, so, tb, flags=1, threads=8, detail=False, budget=3_000_000)
    decided = o["status"] != 2
    batch = DeviceBatch(b, so, tb)
    out = batch.alloc_results()
    batch.run(out, flags=F_BOUNDS)
    g = out.to_host()
    assert decided.mean() > 0.9
    idx = np.nonzero(decided)[0]
    tmask = np.repeat(decided, n)
    _cmp({k: (v[idx] if k == "status" else v[tmask]) for k, v in o.items() if k != "detail"
          and k != "evals"},
         g.status[idx], g.vsm[tmask], g.e2e_num[tmask], g.den[tmask])


def test_device_batch_all_stages_agree():
    gp = _native.gen_params_c(8, 5, (1000, 20000), (1000, 20000), (250, 5000), Fraction(2, 5), 0,
                              10, Fraction(12, 100), Fraction(1))
    b, so, tb = _native.generate(gp, list(range(2000)))
    batch = DeviceBatch(b, so, tb)
    outs = []
    for first in (0, F_FIRST_I64, F_FIRST_I128):
        out = batch.alloc_results()
        batch.run(out, flags=F_BOUNDS | first)
        outs.append(out.to_host())
    for r in outs[1:]:
        assert np.array_equal(r.status, outs[0].status)
        assert np.array_equal(r.vsm, outs[0].vsm)
        f0 = [Fraction(int(a), int(d)) for a, d in zip(outs[0].e2e_num, outs[0].den) if a >= 0]
        f1 = [Fraction(int(a), int(d)) for a, d in zip(r.e2e_num, r.den) if a >= 0]
        assert f0 == f1


def test_e2e_chunked_path_equals_device_path():
    """rtgpu_analyze_host pipelines chunks over two streams; same results."""
    gp = _native.gen_params_c(8, 5, (1000, 20000), (1000, 20000), (250, 5000), Fraction(1, 2), 0,
                              10, Fraction(12, 100), Fraction(1))
    b, so, tb = _native.generate(gp, list(range(40000)))
    batch = DeviceBatch(b, so, tb)
    out = batch.alloc_results()
    batch.run(out, flags=F_BOUNDS)
    g = out.to_host()
    h = analyze_packed(b, so, tb, 0, F_BOUNDS)
    assert _native.last_launch_count() > 3
    assert np.array_equal(g.status, h.status) and np.array_equal(g.vsm, h.vsm)
    assert np.array_equal(g.e2e_num, h.e2e_num) and np.array_equal(g.den, h.den)


@pytest.mark.parametrize("u", ["1/10", "3/10", "1/2", "7/10", "1"])
def test_gpu_verdict_fast_path_matches_oracle(u):
    """The benchmark's mode: flags = 0 (verdict + allocation), front-stage
    fast path, on the benchmark's own shape and seeds."""
    gp = _native.gen_params_c(8, 5, (1000, 20000), (1000, 20000), (250, 5000), Fraction(u), 0,
                              10, Fraction(12, 100), Fraction(1))
    b, so, tb = _native.generate(gp, [f"1000:{u}:{i}" for i in range(2000)])
    o = oracle.analyze_batch(b, so, tb, flags=0, threads=16, detail=False)
    batch = DeviceBatch(b, so, tb)
    out = batch.alloc_results()
    batch.run(out, flags=0)
    g = out.to_host()
    assert np.array_equal(o["status"], g.status)
    sched = np.repeat(o["status"] == 1, 8)
    assert np.array_equal(o["vsm"][sched], g.vsm[sched])


def test_gpu_compact_blobs_equal_int64_blobs():
    """Compact (int32 segment) blobs give the same results as int64 blobs."""
    res = []
    for compact in (False, True):
        gp = _native.gen_params_c(8, 5, (1000, 20000), (1000, 20000), (250, 5000), Fraction(1, 2),
                                  0, 10, Fraction(12, 100), Fraction(1), compact=compact)
        b, so, tb = _native.generate(gp, [f"8:{i}" for i in range(3000)])
        batch = DeviceBatch(b, so, tb)
        for flags in (0, F_BOUNDS):
            out = batch.alloc_results()
            batch.run(out, flags=flags)
            res.append(out.to_host())
    for a, b in ((res[0], res[2]), (res[1], res[3])):
        assert np.array_equal(a.status, b.status) and np.array_equal(a.vsm, b.vsm)
    # the same bounds as exact rationals (the paths may pick different denominators)
    for a, d, b, e in zip(res[1].e2e_num, res[1].den, res[3].e2e_num, res[3].den):
        if a < 0 or b < 0:
            assert a == b
        else:
            assert Fraction(int(a), int(d)) == Fraction(int(b), int(e))


def _cat_batches(parts):
    """Concatenate packed batches (blobs, set_off, task_base)."""
    blobs, offs, tbs = [], [0], [0]
    for b, so, tb in parts:
        blobs.append(b)
        offs += list(so[1:] + offs[-1])
        tbs += list(tb[1:] + tbs[-1])
    return np.concatenate(blobs), np.asarray(offs, np.int64), np.asarray(tbs, np.int64)


def test_e2e_streamed_verdicts_mixed_dims():
    """The end-to-end verdict path streams chunks into one persistent kernel
    whose layout is sized from a sample of the batch: sets beyond it (here
    16x9 sets in the middle of 4x3 sets, and 8x5 sets at the end) go to the
    oversize list and are re-run with the true dims; verdicts and
    allocations equal the oracle's and the device path's."""
    parts = []
    for (n, m, k, seed) in ((4, 3, 9000, 1), (16, 9, 300, 2), (4, 3, 9000, 3), (8, 5, 500, 4)):
        gp = _native.gen_params_c(n, m, (1000, 20000), (1000, 20000), (250, 5000),
                                  Fraction(1, 2), 0, 10, Fraction(12, 100), Fraction(1),
                                  compact=True)
        parts.append(_native.generate(gp, [f"mix:{seed}:{i}" for i in range(k)]))
    b, so, tb = _cat_batches(parts)
    # the sample (first, middle, last set) sees 4x3 and 8x5 sets, not 16x9
    h = analyze_packed(b, so, tb, 0, 0)
    batch = DeviceBatch(b, so, tb)
    out = batch.alloc_results()
    batch.run(out, flags=0)
    g = out.to_host()
    assert np.array_equal(g.status, h.status) and np.array_equal(g.vsm, h.vsm)
    idx = np.r_[0:200, 18000:18300, 18300:18500, len(so) - 400:len(so) - 1]
    sub = [b[so[s]:so[s + 1]] for s in idx]
    sb = np.concatenate(sub)
    sso = np.concatenate([[0], np.cumsum([len(x) for x in sub])]).astype(np.int64)
    ntask = [int(tb[s + 1] - tb[s]) for s in idx]
    stb = np.concatenate([[0], np.cumsum(ntask)]).astype(np.int64)
    o = oracle.analyze_batch(sb, sso, stb, flags=0, threads=16, detail=False)
    assert np.array_equal(o["status"], h.status[idx])
    hv = np.concatenate([h.vsm[tb[s]:tb[s + 1]] for s in idx])
    sched = np.repeat(o["status"] == 1, ntask)
    assert np.array_equal(o["vsm"][sched], hv[sched])


_NO_STREAM_CHILD = r"""
import sys, numpy as np
from fractions import Fraction
from paper_2101_10463_b200 import _native
from paper_2101_10463_b200.engine import analyze_packed
gp = _native.gen_params_c(8, 5, (1000, 20000), (1000, 20000), (250, 5000), Fraction(1, 2), 0, 10,
                          Fraction(12, 100), Fraction(1), compact=True)
b = _native.generate(gp, [f"ns:{i}" for i in range(20000)])
h = analyze_packed(*b, 0, 0)
np.save(sys.argv[1], np.concatenate([h.status.astype(np.int64), h.vsm.astype(np.int64)]))
"""


@pytest.mark.gpu
def test_e2e_no_stream_override_matches_streamed(tmp_path):
    """RTGPU_NO_STREAM=1 (used for profiler runs, which serialise kernels)
    switches the end-to-end verdict path to per-chunk launches; verdicts and
    allocations are identical to the streamed path's."""
    import os
    import subprocess
    import sys
    outs = []
    for env_val in ("0", "1"):
        f = tmp_path / f"o{env_val}.npy"
        env = dict(os.environ, RTGPU_NO_STREAM=env_val)
        subprocess.run([sys.executable, "-c", _NO_STREAM_CHILD, str(f)], check=True, env=env,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))), timeout=300)
        outs.append(np.load(f))
    assert np.array_equal(outs[0], outs[1])


def _no_detail(d):
    return {**d, "per_task": {k: {**v, "gpu_r": [], "mem_r_up": [], "cpu_r_up": []}
                              for k, v in d["per_task"].items()}}


@pytest.mark.parametrize("fixture", ["rtgpu_golden.json", "ood_golden.json"])
@pytest.mark.parametrize("mi", [0, 1, 2])
def test_batch_without_detail_matches_reference(fixture, mi):
    """analyze_batch(detail=False) packs compact blobs (the fast / lattice
    kernels' form, csrc/packer.cpp compact_set): verdicts, allocations and
    end-to-end bounds equal the reference's reports, in and out of the
    reference's validation domain."""
    method = METHODS[mi]
    cases = [c for c in load_cases(fixture) if "raises" not in c[method.value]]
    reps = analyze_batch([ts_from_exact(c["taskset"]) for c in cases], method, detail=False)
    bad = [s for s, (c, r) in enumerate(zip(cases, reps))
           if report_to_dict(r) != _no_detail(c[method.value])]
    assert not bad, bad[:8]
