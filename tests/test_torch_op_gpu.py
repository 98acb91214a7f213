"""torch.ops.rtgpu.analyze_out (csrc/torch_ops.cpp) on the GPU: it is the
binding DeviceBatch uses, it runs on the caller's stream, and it gives the
ctypes binding's results bit for bit."""
from fractions import Fraction

import numpy as np
import pytest

from paper_2101_10463_b200 import _native, engine
from paper_2101_10463_b200.pack import F_BOUNDS

pytestmark = pytest.mark.gpu


def test_operator_is_the_device_binding_and_matches_ctypes():
    import torch
    assert engine.torch_op() is not None
    gp = _native.gen_params_c(16, 9, (1000, 20000), (1000, 20000), (250, 5000), Fraction(1, 5), 0, 148,
                              Fraction(12, 100), Fraction(1), compact=True)
    b, so, tb = _native.generate(gp, list(range(4000)))
    batch = engine.DeviceBatch(b, so, tb)
    for flags in (0, F_BOUNDS):
        side = torch.cuda.Stream()
        a = batch.alloc_results()
        with torch.cuda.stream(side):
            batch.run(a, flags=flags)  # the operator, on `side`
        side.synchronize()
        c = batch.alloc_results()
        _native.analyze_device(batch.blobs.data_ptr(), batch.set_off.data_ptr(), batch.task_base.data_ptr(),
                               batch.n_sets, batch.dims, 0, flags, 0, c.status.data_ptr(), c.evals.data_ptr(),
                               c.vsm.data_ptr(), c.e2e_num.data_ptr(), c.den.data_ptr(), None,
                               torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        for x, y in zip((a.status, a.vsm, a.e2e_num, a.den), (c.status, c.vsm, c.e2e_num, c.den)):
            if flags or x.dtype == torch.int32:
                assert torch.equal(x, y)


def test_operator_rejects_host_tensors():
    import torch
    op = engine.torch_op()
    cpu = torch.zeros(4, dtype=torch.int64)
    with pytest.raises((RuntimeError, NotImplementedError)):  # no CPU kernel is registered
        op(cpu, cpu, cpu, 1, 1, 0, 0, 0, 0, cpu.int(), cpu, cpu.int(), cpu, cpu, cpu)
