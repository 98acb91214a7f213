"""Host helpers of gpu.py (reference gpu.py:16-99): the allocation grid
order, Eq. (1) and Lemma 4 on small exact cases (no GPU needed)."""
import itertools
import random
from fractions import Fraction

import pytest

from paper_2101_10463_b200.gpu import _compositions, gpu_response_bounds, kernel_time
from paper_2101_10463_b200.model import GpuKernelModel, ExecBounds


def _nested_loops(total, mins):
    """The reference's grid: nested loops, first position outermost, each
    ascending, sum within the total."""
    k = len(mins)
    ranges = [range(lo, total + 1) for lo in mins]
    return [c for c in itertools.product(*ranges) if sum(c) <= total] if k else [()]


def test_compositions_match_nested_loops():
    rng = random.Random(10463)
    for _ in range(300):
        k = rng.randint(0, 4)
        mins = [rng.randint(1, 4) for _ in range(k)]
        total = rng.randint(0, 12)
        want = _nested_loops(total, mins) if sum(mins) <= total else []
        assert list(_compositions(total, mins)) == want


def test_kernel_time_and_errors():
    assert kernel_time(Fraction(10), Fraction(2), 4) == Fraction(4)
    with pytest.raises(ValueError, match="sms must be >= 1"):
        kernel_time(Fraction(10), Fraction(2), 0)
    with pytest.raises(ValueError, match=r"overhead must be in \[0, work\]"):
        kernel_time(Fraction(10), Fraction(11), 1)


def test_lemma4_bounds():
    g = GpuKernelModel(work=ExecBounds(Fraction(6), Fraction(12)),
                       critical_path_overhead=Fraction(1), interleave_ratio=Fraction(3, 2))
    b = gpu_response_bounds(g, 4)
    assert b == ExecBounds(Fraction(6, 4), 1 + (Fraction(18) - 1) / 4)
    with pytest.raises(ValueError, match="even count"):
        gpu_response_bounds(g, 3)
