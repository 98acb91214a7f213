"""Host-side logic of the executor report (no GPU): how launch spans are
judged net of the stall sentinel's measured GPU pauses, and how an overrun
is put in context (paper_2101_10463_b200/executor.py)."""
import ctypes

from paper_2101_10463_b200 import executor as ex


def test_stalled_time_is_the_overlap():
    stalls = [(100.0, 1700.0), (5000.0, 5100.0)]
    assert ex._stalled_us(0.0, 50.0, stalls) == 0.0
    assert ex._stalled_us(0.0, 1000.0, stalls) == 900.0
    assert ex._stalled_us(1500.0, 5050.0, stalls) == 200.0 + 50.0
    assert ex._stalled_us(0.0, 10000.0, stalls) == 1600.0 + 100.0
    assert ex._stalled_us(0.0, 10000.0, []) == 0.0


def test_overrun_context_pairs_concurrent_launches():
    # two tasks' kernels overlap a 1.5 ms pause; a third launch is elsewhere in time
    log = [{"task": 0, "seg": 0, "t0_us": 1000.0, "span_us": 5500.0, "items": (10, 11), "mhz": 1965.0},
           {"task": 1, "seg": 1, "t0_us": 2000.0, "span_us": 4000.0, "items": (8, 8), "mhz": 1965.0},
           {"task": 1, "seg": 0, "t0_us": 20000.0, "span_us": 3000.0, "items": (8, 8), "mhz": 1965.0}]
    grs = [[5000.0], [3900.0, 3800.0]]
    out = ex._overrun_context(log, grs, stalls=[(3000.0, 4500.0)])
    assert [(o["task"], o["seg"]) for o in out] == [(0, 0), (1, 1)]  # worst first
    top = out[0]
    assert top["ratio"] == 1.1 and top["stalled_us"] == 1500.0
    assert [(b["task"], b["seg"]) for b in top["beside"]] == [(1, 1)]
    assert top["beside"][0]["overlap_us"] == 4000.0
    # net of the pause both launches are inside their bounds
    for o, e in zip(out, log[:2]):
        assert (e["span_us"] - o["stalled_us"]) / grs[e["task"]][e["seg"]] <= 1.0


def test_result_struct_matches_header():
    """ExecResultC mirrors include/rtgpu_exec.h's rtgpu_exec_result field for
    field (the tail fields added in round 2 included)."""
    names = [f[0] for f in ex.ExecResultC._fields_]
    assert names[-2:] == ["seg_worst_smsp", "smsp_max"]
    with open(__file__.replace("tests/test_executor_host.py", "include/rtgpu_exec.h")) as fh:
        hdr = fh.read()
    body = hdr[hdr.index("typedef struct {\n    int64_t jobs;"):hdr.index("} rtgpu_exec_result;")]
    for n in names:
        assert n in body, n
    assert ctypes.sizeof(ex.ExecResultC) % 8 == 0
