"""SM-partitioned persistent-thread executor (include/rtgpu_exec.h) and the
measured-WCRT-vs-bound experiment (BASELINE config 4).

Pipeline:
  1. calibrate the GPU timing model on the device: single-SM time of each
     kernel (GW), the two-slot interleave ratio (alpha = 2 t2 / t1, section
     4.3), the launch / critical-path overhead (GL) and copy times (ML);
  2. build the task set in the analysis' model from those measurements
     (upper bounds rounded up with a safety margin) and run analyze_rtgpu on
     the GPU engine to get an SM allocation and the bounds R_k;
  3. pin each task's kernels to its disjoint SM partition and run the tasks
     concurrently with periodic releases, measuring every job's response;
  4. check measured WCRT <= R_k and measured kernel times <= GR_up.
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field
from fractions import Fraction
from typing import Optional

import numpy as np

from . import _native
from .analysis import analyze_rtgpu
from .gpu import gpu_response_bounds
from .model import ExecBounds, GpuKernelModel, MemModel, PlatformConfig, TaskSet, TaskSpec

MASK_WORDS = 8


class ExecTaskC(ctypes.Structure):
    _fields_ = [("m", ctypes.c_int32), ("two_copy", ctypes.c_int32),
                ("n_copies", ctypes.c_int32), ("slots_per_sm", ctypes.c_int32),
                ("cpu_us", ctypes.c_int64 * 16), ("copy_bytes", ctypes.c_int64 * 30),
                ("kernel_items", ctypes.c_int64 * 15), ("kernel_iters", ctypes.c_int32),
                ("priority", ctypes.c_int32), ("sm_mask", ctypes.c_uint32 * MASK_WORDS),
                ("period_us", ctypes.c_int64), ("deadline_us", ctypes.c_int64)]


class ExecResultC(ctypes.Structure):
    _fields_ = [("jobs", ctypes.c_int64), ("deadline_misses", ctypes.c_int64),
                ("max_response_us", ctypes.c_double), ("mean_response_us", ctypes.c_double),
                ("max_kernel_us", ctypes.c_double), ("max_kernel_wall_us", ctypes.c_double),
                ("max_copy_us", ctypes.c_double), ("seg_max_kernel_us", ctypes.c_double * 15),
                ("min_blocks", ctypes.c_int32), ("max_blocks", ctypes.c_int32),
                ("seg_max_span_us", ctypes.c_double * 15), ("max_bus_wait_us", ctypes.c_double),
                ("cpu_mode", ctypes.c_int32), ("bus_mode", ctypes.c_int32),
                ("seg_worst_skew_us", ctypes.c_double * 15),
                ("seg_worst_items", (ctypes.c_int32 * 2) * 15),
                ("seg_max_wall_us", ctypes.c_double * 15),
                ("seg_worst_mhz", ctypes.c_double * 15), ("min_mhz", ctypes.c_double),
                ("seg_worst_smsp", ctypes.c_int32 * 15), ("smsp_max", ctypes.c_int32)]

CPU_PARALLEL, CPU_FP_ONE_CORE = 0, 1   # include/rtgpu_exec.h host resource models
BUS_FREE, BUS_FP = 0, 1


def _lib():
    L = _native.lib()
    if not getattr(L, "_exec_ready", False):
        L.rtgpu_exec_kernel_ms.argtypes = [ctypes.POINTER(ctypes.c_uint32), ctypes.c_int,
                                           ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                           ctypes.POINTER(ctypes.c_float),
                                           ctypes.POINTER(ctypes.c_int32),
                                           ctypes.POINTER(ctypes.c_int32)]
        L.rtgpu_exec_kernel_ms_idle.argtypes = [ctypes.POINTER(ctypes.c_uint32), ctypes.c_int,
                                                ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                                ctypes.c_int, ctypes.POINTER(ctypes.c_float),
                                                ctypes.POINTER(ctypes.c_int32),
                                                ctypes.POINTER(ctypes.c_int32)]
        L.rtgpu_exec_kernel_ms_loaded.argtypes = [ctypes.POINTER(ctypes.c_uint32), ctypes.c_int,
                                                  ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                                  ctypes.c_int, ctypes.POINTER(ctypes.c_uint32),
                                                  ctypes.POINTER(ctypes.c_float),
                                                  ctypes.POINTER(ctypes.c_int32),
                                                  ctypes.POINTER(ctypes.c_int32)]
        L.rtgpu_exec_kernel_ms_stress.argtypes = [ctypes.POINTER(ctypes.c_uint32), ctypes.c_int,
                                                  ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                                  ctypes.c_int, ctypes.POINTER(ctypes.c_uint32),
                                                  ctypes.c_int64, ctypes.POINTER(ctypes.c_float),
                                                  ctypes.POINTER(ctypes.c_int32),
                                                  ctypes.POINTER(ctypes.c_int32)]
        L.rtgpu_exec_copy_ms.argtypes = [ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                         ctypes.POINTER(ctypes.c_float)]
        L.rtgpu_exec_run.argtypes = [ctypes.POINTER(ExecTaskC), ctypes.c_int, ctypes.c_double,
                                     ctypes.POINTER(ExecResultC)]
        L.rtgpu_exec_launch_us.argtypes = [ctypes.POINTER(ctypes.c_uint32), ctypes.c_int,
                                           ctypes.POINTER(ctypes.c_float)]
        L.rtgpu_exec_configure.argtypes = [ctypes.c_int, ctypes.c_int]
        L.rtgpu_exec_last_error.restype = ctypes.c_char_p
        L._exec_ready = True
    return L


def mask_of(sms) -> "ctypes.Array":
    m = (ctypes.c_uint32 * MASK_WORDS)()
    for s in sms:
        m[s >> 5] |= 1 << (s & 31)
    return m


def kernel_ms_loaded(sms, bg_sms, nslots: int, items: int, iters: int, reps: int = 3):
    """Like kernel_ms while the SMs bg_sms run co-runner persistent segments."""
    _native.require_device()
    out = (ctypes.c_float * reps)()
    nb, ns = ctypes.c_int32(0), ctypes.c_int32(0)
    rc = _lib().rtgpu_exec_kernel_ms_loaded(mask_of(sms), nslots, items, iters, reps, 0,
                                            mask_of(bg_sms), out, ctypes.byref(nb),
                                            ctypes.byref(ns))
    if rc:
        raise RuntimeError(_lib().rtgpu_exec_last_error().decode())
    return [float(x) for x in out], nb.value, ns.value


def kernel_ms_stress(sms, bg_sms, copy_bytes: int, nslots: int, items: int, iters: int, reps: int = 3):
    """Like kernel_ms_loaded with, in addition, H2D / D2H copies of copy_bytes
    running back to back on another stream (the other tasks' copies)."""
    _native.require_device()
    out = (ctypes.c_float * reps)()
    nb, ns = ctypes.c_int32(0), ctypes.c_int32(0)
    rc = _lib().rtgpu_exec_kernel_ms_stress(mask_of(sms), nslots, items, iters, reps, 0,
                                            mask_of(bg_sms) if bg_sms else None, copy_bytes, out,
                                            ctypes.byref(nb), ctypes.byref(ns))
    if rc:
        raise RuntimeError(_lib().rtgpu_exec_last_error().decode())
    return [float(x) for x in out], nb.value, ns.value


def kernel_ms(sms, nslots: int, items: int, iters: int, reps: int = 5, idle_us: int = 0):
    """Times (ms) of `reps` launches on the SM list (each after idle_us of an
    idle GPU); also participating blocks of the first launch (-1 if a block
    ran outside the partition) and the number of distinct SMs that ran it."""
    _native.require_device()
    out = (ctypes.c_float * reps)()
    nb, ns = ctypes.c_int32(0), ctypes.c_int32(0)
    rc = _lib().rtgpu_exec_kernel_ms_idle(mask_of(sms), nslots, items, iters, reps, idle_us, out,
                                          ctypes.byref(nb), ctypes.byref(ns))
    if rc:
        raise RuntimeError(_lib().rtgpu_exec_last_error().decode())
    return [float(x) for x in out], nb.value, ns.value


def launch_us(sms, reps: int = 20):
    """Host wall time (us) of empty segment launches: the per-kernel overhead
    the job path pays (memset, launch, polled completion)."""
    _native.require_device()
    out = (ctypes.c_float * reps)()
    if _lib().rtgpu_exec_launch_us(mask_of(sms), reps, out):
        raise RuntimeError(_lib().rtgpu_exec_last_error().decode())
    return [float(x) for x in out]


def copy_ms(nbytes: int, to_device: bool, reps: int = 5):
    out = (ctypes.c_float * reps)()
    if _lib().rtgpu_exec_copy_ms(nbytes, 1 if to_device else 0, reps, out):
        raise RuntimeError(_lib().rtgpu_exec_last_error().decode())
    return [float(x) for x in out]


@dataclass
class KernelCal:
    items: int
    iters: int
    t1_us: float      # one SM, one slot (the paper's single-SM time GW)
    t2_us: float      # one SM, two slots
    alpha: Fraction   # 2 t2 / t1, rounded up to a percent
    lo_us: int
    hi_us: int


@dataclass
class ExecTaskDef:
    cpu_us: list
    copy_bytes: list
    kernel_items: list
    period_us: int = 0
    deadline_us: int = 0


@dataclass
class WcrtReport:
    tasks: list = field(default_factory=list)
    allocation: dict = field(default_factory=dict)
    schedulable: bool = False
    all_within_bound: bool = False
    kernels_within_bound: bool = False
    max_ratio: float = 0.0
    max_kernel_ratio: float = 0.0  # worst measured kernel time / its Lemma-4 bound
    sms_used: int = 0              # physical SMs covered by the partitions
    horizon_us: float = 0.0
    cpu_mode: int = CPU_PARALLEL
    bus_mode: int = BUS_FP
    calibration: list = field(default_factory=list)  # per kernel: items, t1, t2, alpha
    note: str = ""
    # launches over their Lemma-4 bound, each with the other tasks' launches
    # that overlapped it in GPU time (span / GR_up of each) -- is a slowdown
    # one partition's, or GPU-wide?
    overruns: list = field(default_factory=list)
    launch_ratio_pcts: dict = field(default_factory=dict)  # span / GR_up percentiles over all launches
    # the stall sentinel (an SM outside every partition reading %globaltimer):
    # GPU pauses during the run, and every launch's span with the paused time
    # it overlapped taken out -- Lemma 4 bounds execution, not platform pauses
    stalls: dict = field(default_factory=dict)
    max_kernel_ratio_net: Optional[float] = None
    kernels_within_bound_net: Optional[bool] = None


def _ceil_margin(x_us: float, margin: float) -> int:
    return int(math.ceil(x_us * (1 + margin))) + 1


CAL_SMS = (0, 74)  # one SM on each die: L2 distance differs per die
_CAL_CACHE: dict = {}


# Safety margin on measured worst cases.  A kernel's speed on its SMs depends
# on how its warps land on the four SM sub-partitions (the warp slots other
# grids' exiting blocks leave free): with two 4-warp blocks per SM an uneven
# placement costs up to 1/8 of the FMA throughput, which calibration on an
# otherwise idle GPU does not see.  25% covers it.
MARGIN = 0.25


def calibrate_kernel(items: int, iters: int, reps: int = 4, margin: float = MARGIN,
                     idle_us: int = 20000, copy_bytes: int = 4 << 20) -> KernelCal:
    """Worst case over SMs of both dies, warm launches and launches after an
    idle GPU (the SM clock may have dropped; clocks are not locked here), with
    co-runners on every other SM, and with co-runners plus back-to-back
    H2D / D2H copies (the conditions of a run: other partitions compute while
    other tasks copy)."""
    t1, t2 = [], []
    for sm in CAL_SMS:
        others = [x for x in range(148) if x != sm]
        t1 += kernel_ms([sm], 1, items, iters, reps)[0] + kernel_ms([sm], 1, items, iters, 2, idle_us)[0]
        t2 += kernel_ms([sm], 2, items, iters, reps)[0] + kernel_ms([sm], 2, items, iters, 2, idle_us)[0]
        # co-runners on every other SM (the executor's concurrent partitions)
        t1 += kernel_ms_loaded([sm], others, 1, items, iters, 2)[0]
        t2 += kernel_ms_loaded([sm], others, 2, items, iters, 2)[0]
        if copy_bytes > 0:
            t1 += kernel_ms_stress([sm], others, copy_bytes, 1, items, iters, 2)[0]
            t2 += kernel_ms_stress([sm], others, copy_bytes, 2, items, iters, 2)[0]
    t1u, t2u = max(t1) * 1e3, max(t2) * 1e3
    pct = math.ceil(200 * t2u / t1u)
    if pct > 180:  # MAX_INTERLEAVE_RATIO (model.py:17): the model cannot bound this kernel
        raise ValueError(f"measured interleave ratio {pct / 100} exceeds the model's 1.8")
    alpha = Fraction(max(100, pct), 100)
    return KernelCal(items, iters, t1u, t2u, alpha, int(min(t1) * 1e3 * 0.95),
                     _ceil_margin(t1u, margin))


def launch_log():
    """The last run's kernel launches (rtgpu_exec_launch_log): dicts with task,
    seg, t0_us (%globaltimer), span_us, items (min, max of traced warps), mhz."""
    L = _lib()
    L.rtgpu_exec_launch_log.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.c_int]
    n = L.rtgpu_exec_launch_log(None, 0)
    buf = (ctypes.c_double * (7 * max(n, 1)))()
    n = L.rtgpu_exec_launch_log(buf, n)
    return [{"task": int(buf[7 * k]), "seg": int(buf[7 * k + 1]), "t0_us": buf[7 * k + 2],
             "span_us": buf[7 * k + 3], "items": (int(buf[7 * k + 4]), int(buf[7 * k + 5])),
             "mhz": buf[7 * k + 6]} for k in range(n)]


def stall_log():
    """The last run's stall sentinel (rtgpu_exec_stall_log): (sentinel SM or
    None, [(start_us, end_us), ...] intervals over 50 us in which an SM no
    task used did not execute), in the launch log's %globaltimer time base."""
    L = _lib()
    L.rtgpu_exec_stall_log.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.c_int,
                                       ctypes.POINTER(ctypes.c_int)]
    sm = ctypes.c_int(-1)
    n = L.rtgpu_exec_stall_log(None, 0, ctypes.byref(sm))
    buf = (ctypes.c_double * (2 * max(n, 1)))()
    n = L.rtgpu_exec_stall_log(buf, n, ctypes.byref(sm))
    return (None if sm.value < 0 else sm.value), [(buf[2 * k], buf[2 * k + 1]) for k in range(n)]


def _stalled_us(t0: float, t1: float, stalls) -> float:
    return sum(max(0.0, min(t1, b) - max(t0, a)) for a, b in stalls)


def _overrun_context(log, grs_of, limit: int = 12, stalls=None):
    """Launches over their bound, the sentinel's paused time inside them, and
    what ran beside them."""
    ratio = lambda e: e["span_us"] / grs_of[e["task"]][e["seg"]]  # noqa: E731
    out = []
    for e in sorted((e for e in log if ratio(e) > 1.0), key=ratio, reverse=True)[:limit]:
        a0, a1 = e["t0_us"], e["t0_us"] + e["span_us"]
        beside = [{"task": o["task"], "seg": o["seg"], "ratio": round(ratio(o), 3),
                   "overlap_us": round(min(a1, o["t0_us"] + o["span_us"]) - max(a0, o["t0_us"]), 1)}
                  for o in log if o is not e and o["t0_us"] < a1 and o["t0_us"] + o["span_us"] > a0]
        out.append({"task": e["task"], "seg": e["seg"], "ratio": round(ratio(e), 3),
                    "stalled_us": round(_stalled_us(a0, a1, stalls), 1) if stalls is not None else None,
                    "span_us": round(e["span_us"], 1), "t0_ms": round((a0 - log[0]["t0_us"]) * 1e-3, 3),
                    "items": e["items"], "mhz": round(e["mhz"]), "beside": beside})
    return out


def run_tasks(defs, partitions, iters: int, horizon_us: float, two_copy: bool = True,
              cpu_mode: int = CPU_PARALLEL, bus_mode: int = BUS_FP, priorities=None):
    """Run the tasks on their SM partitions.  priorities[i] is task i's fixed
    priority (smaller = higher, as TaskSpec.priority): the bus arbiter and the
    CPU ranks use it, so it must be the priority the analysis assumed
    (default: the order of defs)."""
    L = _lib()
    if L.rtgpu_exec_configure(cpu_mode, bus_mode):
        raise ValueError(L.rtgpu_exec_last_error().decode())
    n = len(defs)
    arr = (ExecTaskC * n)()
    for i, (d, sms) in enumerate(zip(defs, partitions)):
        t = arr[i]
        t.m = len(d.cpu_us)
        t.two_copy = 1 if two_copy else 0
        t.n_copies = len(d.copy_bytes)
        t.slots_per_sm = 2
        for j, v in enumerate(d.cpu_us):
            t.cpu_us[j] = int(v)
        for j, v in enumerate(d.copy_bytes):
            t.copy_bytes[j] = int(v)
        for j, v in enumerate(d.kernel_items):
            t.kernel_items[j] = int(v)
        t.kernel_iters = iters
        t.priority = int(priorities[i]) if priorities is not None else i + 1
        mk = mask_of(sms)
        for w in range(MASK_WORDS):
            t.sm_mask[w] = mk[w]
        t.period_us = int(d.period_us)
        t.deadline_us = int(d.deadline_us)
    res = (ExecResultC * n)()
    if L.rtgpu_exec_run(arr, n, float(horizon_us), res):
        raise RuntimeError(L.rtgpu_exec_last_error().decode())
    return [res[i] for i in range(n)]


def wcrt_experiment(n_tasks: int = 4, m: int = 3, iters: int = 2048, seed: int = 0,
                    utilization: float = 3.0, horizon_us: float = 3e6, n_sm: int = 148,
                    margin: float = MARGIN, cpu_mode: int = CPU_PARALLEL,
                    bus_mode: int = BUS_FP, layout: str = "", width=None) -> WcrtReport:
    """BASELINE config 4: n concurrent tasks on disjoint SM partitions of the
    GPU; measured WCRT vs the RTGPU bound R_k.  layout "consecutive" packs
    the partitions on consecutive SM ids; "tpc" gives each task whole TPCs
    (SM pairs 2t, 2t+1), so no two tasks share a TPC (default: $RTGPU_EXEC_LAYOUT,
    else "tpc").  Over 72 robustness runs each layout saw occasional kernel
    overruns of Lemma 4 (tpc 4, consecutive 4 in 48); only consecutive
    partitions pushed a job past R_k (2 runs) -- profiles/r1m_exec_*.jsonl.

    width = (lo, hi): wide partitions -- kernels sized so that one SM would
    need tens of milliseconds, and every task's deadline set from a target
    SM count drawn from [lo, hi] (its own segments at that count, times a
    slack for the interference of higher-priority tasks), so the analysis
    gives each task a partition of several to tens of SMs; `utilization`
    is then unused."""
    _native.require_device()
    rng = np.random.default_rng(seed)
    defs = []
    items_rng = (400, 3000) if width is None else (6000, 20000)
    for i in range(n_tasks):
        items = rng.integers(*items_rng, m - 1)
        if width is not None:
            items = (items // 2000) * 2000  # a few sizes: calibrations are reused across runs
        defs.append(ExecTaskDef(
            cpu_us=[int(x) for x in rng.integers(100, 600, m)],
            copy_bytes=[int(x) for x in rng.integers(1 << 18, 4 << 20, 2 * m - 2)],
            kernel_items=[int(x) for x in items]))
    # calibrate every kernel and copy on the device (kept per process: the
    # same kernel size is not re-timed by the next experiment)
    cal = {}
    for d in defs:
        for it in d.kernel_items:
            if it not in cal:
                key = (it, iters, margin)
                if key not in _CAL_CACHE:
                    _CAL_CACHE[key] = calibrate_kernel(it, iters, margin=margin)
                cal[it] = _CAL_CACHE[key]
    # critical-path overhead GL: host wall time of an empty launch (what the
    # job path adds around every kernel), worst of many
    overhead = max(launch_us(list(range(8)), 50) +
                   [x * 1e3 for x in kernel_ms(list(range(8)), 2, 0, iters, 3, 20000)[0]])
    GL = _ceil_margin(overhead, margin)
    # a kernel's blocks claim work items one at a time, so the last item
    # can end up to one item's two-slot time tau2 = 2 t2 / items after the
    # perfectly divided (C - L)/m of Lemma 4: the critical-path term of a
    # kernel carries it (L (1 - 1/2g) >= launch + tau2 for L = 2 (launch +
    # tau2)); it matters once partitions are wide and items per block few
    gl_of = {it: _ceil_margin(2 * (overhead + 2 * c.t2_us / c.items), margin) for it, c in cal.items()}
    copy_cal = {}
    for d in defs:
        for j, b in enumerate(d.copy_bytes):
            key = (b, j % 2 == 0)
            if key not in copy_cal:
                ts = copy_ms(b, j % 2 == 0, 5)
                copy_cal[key] = (int(min(ts) * 1e3 * 0.9), _ceil_margin(max(ts) * 1e3, margin + 0.5))
    # the analysis' task set (integer microseconds; upper bounds padded)
    specs = []
    util = rng.uniform(0.5, 1.5, n_tasks)
    util = util / util.sum() * utilization
    targets = None
    if width is not None:
        targets = rng.integers(width[0], width[1] + 1, n_tasks)
        while targets.sum() > n_sm - 2 * n_tasks:  # room for TPC alignment
            targets = np.maximum(1, targets - 1)
    for i, d in enumerate(defs):
        cpu = tuple(ExecBounds.exact(c) for c in d.cpu_us)
        mem = tuple(ExecBounds(Fraction(copy_cal[(b, j % 2 == 0)][0]),
                               Fraction(copy_cal[(b, j % 2 == 0)][1]))
                    for j, b in enumerate(d.copy_bytes))
        gpu = tuple(GpuKernelModel(ExecBounds(Fraction(min(cal[it].lo_us, cal[it].hi_us)),
                                              Fraction(cal[it].hi_us)),
                                   Fraction(min(gl_of[it], cal[it].lo_us)), cal[it].alpha)
                    for it in d.kernel_items)
        demand = sum(c.hi for c in cpu) + sum(x.hi for x in mem) + sum(g.work.hi for g in gpu)
        if targets is None:
            D = int(demand / Fraction(util[i]).limit_denominator(10**6))
        else:
            own = (sum(c.hi for c in cpu) + sum(x.hi for x in mem) +
                   sum(gpu_response_bounds(g, 2 * int(targets[i])).hi for g in gpu))
            D = int(own * Fraction(rng.uniform(1.5, 2.2)).limit_denominator(1000)) + 1
        d.period_us = d.deadline_us = D
        specs.append(TaskSpec(f"x{i}", cpu, mem, gpu, Fraction(D), Fraction(D), 0))
    order = sorted(range(n_tasks), key=lambda i: (specs[i].deadline, i))
    specs = [TaskSpec(s.id, s.cpu_segments, s.mem_segments, s.gpu_segments, s.deadline, s.period,
                      order.index(i) + 1) for i, s in enumerate(specs)]
    ts = TaskSet(tuple(specs), MemModel.TWO_COPY, PlatformConfig(n_sm, Fraction(3, 25)))
    report = analyze_rtgpu(ts)
    out = WcrtReport(schedulable=report.schedulable, horizon_us=horizon_us)
    out.calibration = [{"items": c.items, "t1_us": round(c.t1_us, 1), "t2_us": round(c.t2_us, 1),
                        "alpha": str(c.alpha), "gw_hi_us": c.hi_us, "gl_us": gl_of[it]}
                       for it, c in cal.items()]
    if targets is not None:
        out.note = f"target SM counts {[int(x) for x in targets]}"
    if not report.schedulable:
        out.note = "analysis rejects the calibrated task set; nothing to execute"
        return out
    # disjoint partitions in priority order
    alloc = report.allocation.per_task_virtual_sms
    layout = layout or os.environ.get("RTGPU_EXEC_LAYOUT", "tpc")
    parts, nxt = [], 0
    for s in specs:
        gn = alloc[s.id] // 2
        parts.append(list(range(nxt, nxt + gn)))
        nxt += gn
        if layout == "tpc":
            nxt += nxt % 2  # the next task starts on a fresh TPC
    if nxt > n_sm:
        raise ValueError(f"partitions need {nxt} SMs, the GPU has {n_sm}")
    out.sms_used = sum(len(p) for p in parts)
    out.allocation = {s.id: alloc[s.id] for s in specs}
    # the executor arbitrates the bus and the CPU with the analysis' own
    # (deadline-monotonic) priorities, not the order tasks were drawn in
    res = run_tasks(defs, parts, iters, horizon_us, cpu_mode=cpu_mode, bus_mode=bus_mode,
                    priorities=[s.priority for s in specs])
    out.cpu_mode, out.bus_mode = int(res[0].cpu_mode), int(res[0].bus_mode)
    ratios, kok = [], True
    for s, d, r, sms in zip(specs, defs, res, parts):
        bound = report.per_task[s.id].end_to_end_up
        grs = [gpu_response_bounds(g, 2 * len(sms)).hi for g in s.gpu_segments]
        ratio = r.max_response_us / float(bound)
        ratios.append(ratio)
        # Lemma 4 bounds the kernel's execution on its partition: the on-GPU
        # span from the first participating block's start to the last one's
        # end (%globaltimer).  Event and host-observed times, which add launch
        # latency (and the VM's scheduling jitter), are reported beside it;
        # the end-to-end check covers them.
        seg = [r.seg_max_span_us[j] for j in range(len(grs))]
        kern_ok = all(x <= float(b) for x, b in zip(seg, grs))
        kok = kok and kern_ok
        out.max_kernel_ratio = max([out.max_kernel_ratio] + [x / float(b) for x, b in zip(seg, grs)])
        out.tasks.append({"task": s.id, "priority": s.priority, "sms": len(sms),
                          "jobs": int(r.jobs), "wcrt_us": round(r.max_response_us, 1),
                          "bound_us": float(bound), "ratio": round(ratio, 4),
                          "mean_us": round(r.mean_response_us, 1),
                          "max_kernel_us": round(r.max_kernel_us, 1),
                          "kernel_span_us_vs_gr_up": [[round(x, 1), round(float(b), 1)]
                                                 for x, b in zip(seg, grs)],
                          "kernel_event_us": [round(r.seg_max_kernel_us[j], 1)
                                              for j in range(len(grs))],
                          "kernel_wall_us": [round(r.seg_max_wall_us[j], 1)
                                             for j in range(len(grs))],
                          "worst_launch": [{"skew_us": round(r.seg_worst_skew_us[j], 1),
                                            "sm_mhz": round(r.seg_worst_mhz[j]),
                                            "items": [int(r.seg_worst_items[j][0]),
                                                      int(r.seg_worst_items[j][1])],
                                            "smsp_max_warps": int(r.seg_worst_smsp[j])}
                                           for j in range(len(grs))],
                          "smsp_max_warps": int(r.smsp_max),
                          "min_sm_mhz": round(r.min_mhz),
                          "max_copy_us": round(r.max_copy_us, 1),
                          "max_bus_wait_us": round(r.max_bus_wait_us, 1),
                          "blocks_per_launch": [int(r.min_blocks), int(r.max_blocks)],
                          "gr_up_us": float(max(grs)), "deadline_us": d.deadline_us,
                          "deadline_misses": int(r.deadline_misses)})
    grs_of = [[float(gpu_response_bounds(g, 2 * len(sms)).hi) for g in s.gpu_segments]
              for s, sms in zip(specs, parts)]
    log = launch_log()
    sentinel, stalls = stall_log()
    if log and sentinel is not None:
        net = [(e["span_us"] - _stalled_us(e["t0_us"], e["t0_us"] + e["span_us"], stalls))
               / grs_of[e["task"]][e["seg"]] for e in log]
        out.max_kernel_ratio_net = round(max(net), 4)
        out.kernels_within_bound_net = bool(max(net) <= 1.0)
        dur = [b - a for a, b in stalls]
        out.stalls = {"sentinel_sm": sentinel, "count": len(stalls),
                      "max_us": round(max(dur), 1) if dur else 0.0,
                      "total_us": round(sum(dur), 1),
                      "launches_overlapping": sum(1 for e in log if _stalled_us(
                          e["t0_us"], e["t0_us"] + e["span_us"], stalls) > 0)}
    if log:
        out.overruns = _overrun_context(log, grs_of, stalls=stalls if sentinel is not None else None)
        rs = np.array([e["span_us"] / grs_of[e["task"]][e["seg"]] for e in log])
        out.launch_ratio_pcts = {"launches": len(rs), "p50": round(float(np.percentile(rs, 50)), 3),
                                 "p99": round(float(np.percentile(rs, 99)), 3),
                                 "max": round(float(rs.max()), 3), "over_1": int((rs > 1).sum())}
    out.max_ratio = max(ratios)
    out.all_within_bound = all(x <= 1.0 for x in ratios)
    out.kernels_within_bound = kok
    return out
