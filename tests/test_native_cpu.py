"""CPU-side checks of the native library: it loads, exports every entry
point the public headers declare, and refuses to analyse without a GPU."""
import ctypes
import glob
import os
import re

import pytest

from paper_2101_10463_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = open(h).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        names |= set(re.findall(r"\b(rtgpu_\w+)\s*\(", text))
        # header-only helpers (static inline, e.g. rtgpu_rec_word) are not exports
        names -= set(re.findall(r"static\s+inline\s+[\w\s\*]*?\b(rtgpu_\w+)\s*\(", text))
    return names


def test_library_exports_every_header_symbol():
    lib = _native.lib()
    missing = [n for n in sorted(declared_symbols()) if not hasattr(lib, n)]
    assert not missing, missing
    assert set(_native.EXPORTS) <= declared_symbols()


def test_abi_version():
    assert _native.lib().rtgpu_abi_version() == 1


def test_sha512_known_answer():
    out = ctypes.create_string_buffer(64)
    _native.lib().rtgpu_sha512(b"abc", 3, out)
    assert out.raw.hex().startswith("ddaf35a193617aba")


@pytest.mark.skipif(_native.device_info()["n_devices"] > 0, reason="GPU present")
def test_no_cpu_fallback():
    from paper_2101_10463_b200.analysis import analyze_rtgpu
    from paper_2101_10463_b200.model import PlatformConfig, TaskSet, MemModel
    with pytest.raises(_native.EngineUnavailable):
        analyze_rtgpu(TaskSet((), MemModel.TWO_COPY, PlatformConfig(4)))


def test_torch_operator_registers():
    """The PyTorch operator (csrc/torch_ops.cpp) loads and registers
    rtgpu::analyze_out with its schema (no compute without a GPU)."""
    import torch
    from paper_2101_10463_b200 import build
    torch.ops.load_library(build.build_torch_op())
    op = torch.ops.rtgpu.analyze_out
    schema = str(op.default._schema)
    assert "Tensor(a!) status" in schema and "int budget" in schema
