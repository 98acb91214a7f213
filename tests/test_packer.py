"""The native TaskSet packer (csrc/packer.cpp) writes exactly the Python
packer's words, task order and time scales -- on the reference's golden
task sets (Fraction-valued, odd shapes, sets the engine refuses) and on
generated sets -- and falls back to the Python packer's exceptions."""
from fractions import Fraction

import numpy as np
import pytest

from golden_io import load_cases, ts_from_exact
from paper_2101_10463_b200.pack import pack_tasksets, pack_tasksets_py
from paper_2101_10463_b200.workbench import GenParams, generate_taskset


def same(a, b):
    assert np.array_equal(a.blobs, b.blobs)
    assert np.array_equal(a.set_off, b.set_off) and np.array_equal(a.task_base, b.task_base)
    for x, y in zip(a.metas, b.metas):
        assert x.order == y.order and x.time_scale == y.time_scale and x.word_off == y.word_off


def test_native_packer_is_built():
    from paper_2101_10463_b200 import _packer  # noqa: F401


def test_native_equals_python_on_golden():
    for c in load_cases():
        ts = ts_from_exact(c["taskset"])
        try:
            want = pack_tasksets_py([ts])
        except Exception as exc:  # the engine refuses this shape: same exception either way
            with pytest.raises(type(exc)):
                pack_tasksets([ts])
            continue
        same(pack_tasksets([ts]), want)


@pytest.mark.parametrize("n,m,u,mm", [(8, 5, "1/2", "two_copy"), (16, 9, "1/5", "one_copy"),
                                      (3, 1, "1", "two_copy")])
def test_native_equals_python_generated(n, m, u, mm):
    from paper_2101_10463_b200.model import MemModel
    gp = GenParams(n_tasks=n, n_subtasks=m, physical_sms=20, target_utilization=Fraction(u),
                   mem_model=MemModel(mm), lo_frac=Fraction(7, 10))
    sets = [generate_taskset(gp, i) for i in range(200)]
    same(pack_tasksets(sets), pack_tasksets_py(sets))


def test_native_compact_equals_compacted_python():
    """pack(compact=True) writes tests/blobtools.compact's words: int32 segment
    areas wherever every value of the set fits, int64 elsewhere."""
    from blobtools import compact
    gp = GenParams(n_tasks=6, n_subtasks=4, target_utilization=Fraction(1, 2))
    sets = [generate_taskset(gp, f"c{i}") for i in range(30)]
    want = pack_tasksets_py(sets)
    cb, co, ct = compact(want.blobs, want.set_off, want.task_base)
    got = pack_tasksets(sets, compact=True)
    assert np.array_equal(got.blobs, cb) and np.array_equal(got.set_off, co)
    assert np.array_equal(got.task_base, ct)
