"""The ctypes stub INTEGRATION.md shows a maintainer adding to gpusched is
runnable as written: the block is executed against the in-tree library and
must reproduce the reference's golden reports."""
import os
import re

import pytest

from golden_io import load_cases, ts_from_exact
from paper_2101_10463_b200.model import AnalysisMethod, report_to_dict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def stub_source():
    with open(os.path.join(ROOT, "INTEGRATION.md")) as fh:
        text = fh.read()
    blocks = re.findall(r"```python\n(# gpusched/_b200\.py.*?)```", text, re.S)
    assert len(blocks) == 1
    return blocks[0]


def test_stub_is_complete_python():
    src = stub_source()
    compile(src, "INTEGRATION.md", "exec")
    assert "..." not in src


@pytest.mark.gpu
def test_stub_reproduces_golden_reports():
    os.environ["RTGPU_LIB"] = os.path.join(ROOT, "paper_2101_10463_b200", "librtgpu.so")
    ns = {}
    exec(stub_source(), ns)
    bad = 0
    for c in load_cases()[:120]:
        ts = ts_from_exact(c["taskset"])
        for method in (AnalysisMethod.RTGPU, AnalysisMethod.BUSY_WAITING):
            want = c[method.value]
            try:
                got = report_to_dict(ns["analyze_b200"](ts, method))
            except ValueError:
                got = "raises"
            if ("raises" in want) != (got == "raises") or ("raises" not in want and got != want):
                bad += 1
    assert bad == 0
