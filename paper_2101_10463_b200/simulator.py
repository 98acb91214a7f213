"""Discrete-event simulation of one preemptive fixed-priority CPU, one
non-preemptive fixed-priority bus and per-task dedicated virtual SMs -- the
drop-in for gpusched.simulator (/root/reference/pkg/src/gpusched/simulator.py)
with the simulation itself on the GPU (include/rtgpu_sim.h, csrc/simulator.cu:
one thread per simulation, integer time scaled by an exact common factor).

`simulate` (simulator.py:160) runs a batch of one and returns the same
SimTrace -- same events in the same order, same responses, same truncation
list; `check_against_analysis` (simulator.py:340) is the same host-side check
over a trace.  `simulate_batch` / `SimBatch.check` run many simulations in
one launch and give check_against_analysis's verdict per task set from the
device-side per-segment maxima, without materialising traces.
"""
from __future__ import annotations

import ctypes
import hashlib
import json
import math
import os
from dataclasses import dataclass, field
from enum import Enum
from fractions import Fraction
from typing import Optional, Sequence

import numpy as np

from . import _native
from .gpu import gpu_response_bounds
from .model import (AnalysisReport, SmAllocation, TaskSet, TaskSpec, duration_to_str,
                    validate_taskset)

HDR, TASKW, SEGW = 16, 8, 6          # include/rtgpu_sim.h
KINDS = ("cpu", "mem", "gpu", "job")
ACTIONS = ("release", "start", "preempt", "resume", "finish", "deadline-miss")
LIMIT = 1 << 62


class LengthPolicy(str, Enum):
    WORST_CASE = "worst"
    UNIFORM_RANDOM = "uniform"


class ReleasePolicy(str, Enum):
    PERIODIC = "periodic"


@dataclass(frozen=True)
class SimConfig:
    horizon: Optional[Fraction] = None  # default: 20 x max period
    seed: int = 0
    length_policy: LengthPolicy = LengthPolicy.WORST_CASE
    release_policy: ReleasePolicy = ReleasePolicy.PERIODIC


@dataclass(frozen=True)
class SimEvent:
    time: Fraction
    task: str
    job: int
    kind: str  # "cpu" | "mem" | "gpu" | "job"
    segment: int
    action: str  # release/start/preempt/resume/finish/deadline-miss


@dataclass
class SimTrace:
    events: list = field(default_factory=list)
    responses: dict = field(default_factory=dict)
    releases: dict = field(default_factory=dict)
    truncated: list = field(default_factory=list)

    def to_jsonl(self) -> str:
        lines = [json.dumps({"time": duration_to_str(e.time), "task": e.task, "job": e.job,
                             "kind": e.kind, "segment": e.segment, "action": e.action})
                 for e in self.events]
        return "\n".join(lines) + ("\n" if lines else "")


class SimRangeError(OverflowError):
    """The simulation's exact time scale does not fit 62-bit integers."""


# ---------------------------------------------------------------- packing

def job_segment_plan(task: TaskSpec, two_copy: bool) -> list:
    """Execution order of (kind, index) segments of one job (simulator.py:106)."""
    m = task.n_subtasks
    plan = []
    for j in range(m - 1):
        plan.append(("cpu", j))
        if two_copy:
            plan += [("mem", 2 * j), ("gpu", j), ("mem", 2 * j + 1)]
        else:
            plan += [("mem", j), ("gpu", j)]
    plan.append(("cpu", m - 1))
    return plan


def check_allocation(ts: TaskSet, alloc: SmAllocation) -> None:
    """Same rules and messages as simulator.py:145."""
    for t in ts.tasks:
        vs = alloc.virtual_sms(t.id)
        if t.gpu_segments:
            if vs < 2 or vs % 2 != 0:
                raise ValueError(f"task {t.id}: needs an even virtual-SM count >= 2, got {vs}")
        elif vs != 0:
            raise ValueError(f"task {t.id}: pure-CPU task allocated SMs")
    if alloc.total_physical() > ts.platform.physical_sms:
        raise ValueError("allocation exceeds available physical SMs")


def _seed_key(seed) -> list:
    """The 32-bit init_by_array key random.Random(seed) uses (CPython
    random_seed: |int| as little-endian words; str/bytes through sha512;
    float through hash())."""
    if seed is None:
        seed = int.from_bytes(os.urandom(32), "little")
    if isinstance(seed, (str, bytes, bytearray)):
        raw = seed.encode() if isinstance(seed, str) else bytes(seed)
        seed = int.from_bytes(raw + hashlib.sha512(raw).digest(), "big")
    elif isinstance(seed, float):
        seed = hash(seed)
    elif not isinstance(seed, int):
        raise TypeError("The only supported seed types are:\nNoneType, int, float, str, bytes, "
                        "and bytearray.")
    a = abs(int(seed))
    words = []
    while a:
        words.append(a & 0xFFFFFFFF)
        a >>= 32
    return words or [0]


@dataclass
class _Packed:
    blob: np.ndarray
    Q: int
    tasks: tuple
    R: int
    evcap: int
    smax: int
    plans: list


def _lcm(a: int, b: int) -> int:
    return a // math.gcd(a, b) * b


def pack_simulation(ts: TaskSet, alloc: SmAllocation, cfg: SimConfig,
                    pool: Optional[int] = 0) -> _Packed:
    """Validate like simulate() and build the simulator blob (rtgpu_sim.h).
    pool: job records on the device (0: one per release point, always
    enough; None: 4 per task + 16, recycled -- RTGPU_SIM_POOL_OVERFLOW if an
    overloaded run needs more, and simulate_batch re-runs it with pool 0)."""
    violations = validate_taskset(ts)
    if violations:
        raise ValueError("invalid taskset: " + "; ".join(violations))
    check_allocation(ts, alloc)
    two_copy = ts.mem_model.value == "two_copy"
    horizon = cfg.horizon
    if horizon is None:
        horizon = 20 * max((t.period for t in ts.tasks), default=Fraction(1))
    horizon = Fraction(horizon)
    uniform = LengthPolicy(cfg.length_policy) is LengthPolicy.UNIFORM_RANDOM
    tasks = ts.by_priority()
    plans, entries = [], []
    dens = {horizon.denominator}
    for t in tasks:
        dens |= {Fraction(t.period).denominator, Fraction(t.deadline).denominator}
        vs = alloc.virtual_sms(t.id)
        plan = job_segment_plan(t, two_copy)
        plans.append(plan)
        ent = []
        for kind, idx in plan:
            if kind in ("cpu", "mem"):
                b = (t.cpu_segments if kind == "cpu" else t.mem_segments)[idx]
                rnd = uniform and b.lo != b.hi
                fixed, A, B = Fraction(b.hi), Fraction(1), Fraction(0)
                lo, hi = int(b.lo), int(b.hi)
            else:
                g = t.gpu_segments[idx]
                lo, hi = int(g.work.lo), int(g.work.hi)
                A = Fraction(g.interleave_ratio) / vs
                B = Fraction(g.critical_path_overhead) - Fraction(g.critical_path_overhead) / vs
                if not uniform:
                    fixed, rnd = gpu_response_bounds(g, vs).hi, False
                else:
                    rnd = g.work.lo != g.work.hi
                    fixed = ((Fraction(g.work.hi) * g.interleave_ratio - g.critical_path_overhead)
                             / vs + g.critical_path_overhead)
            dens.add(Fraction(fixed).denominator)
            if rnd:
                dens |= {A.denominator, B.denominator}
            ent.append((kind, idx, rnd, lo, hi, Fraction(fixed), A, B))
        entries.append(ent)
    Q = 1
    for d in dens:
        Q = _lcm(Q, d)
    H = horizon * Q
    assert H.denominator == 1
    H = int(H)
    n = len(tasks)
    key = _seed_key(cfg.seed) if uniform else []
    counts = []
    for t in tasks:
        T = int(Fraction(t.period) * Q)
        counts.append((H + T - 1) // T if H > 0 else 0)
    R = sum(counts)
    smax = max((len(p) for p in plans), default=0)
    evcap = sum(c * (3 + 2 * len(p) + 2 * t.n_subtasks) for c, p, t in zip(counts, plans, tasks))
    seg_off = HDR + TASKW * n
    words = seg_off + SEGW * sum(len(p) for p in plans) + len(key)
    blob = np.zeros(words, dtype=np.int64)
    big = H + max((Fraction(t.deadline) * Q for t in tasks), default=0)
    for i, (t, ent) in enumerate(zip(tasks, entries)):
        r = HDR + TASKW * i
        blob[r:r + 6] = [len(ent), int(Fraction(t.period) * Q), int(Fraction(t.deadline) * Q),
                         t.priority, seg_off, t.n_subtasks]
        for p, (kind, idx, rnd, lo, hi, fixed, A, B) in enumerate(ent):
            k = ("cpu", "mem", "gpu").index(kind)
            vals = [k | (idx << 8) | (int(rnd) << 16), lo, hi, int(fixed * Q),
                    int(A * Q) if rnd else 0, int(B * Q) if rnd else 0]
            blob[seg_off + SEGW * p:seg_off + SEGW * (p + 1)] = vals
            dmax = (abs(hi) * abs(A) + abs(B)) * Q if rnd else fixed * Q
            big = max(big, H + dmax)
        seg_off += SEGW * len(ent)
    if 2 * big >= LIMIT:
        raise SimRangeError(f"simulation time scale {Q} x horizon exceeds 62-bit integers")
    blob[:9] = [n, int(uniform), H, R, evcap, len(key), smax, seg_off,
                4 * n + 16 if pool is None else pool]
    blob[seg_off:seg_off + len(key)] = key
    return _Packed(blob, Q, tasks, R, evcap, smax, plans)


# ---------------------------------------------------------------- native call

class _SimOut(ctypes.Structure):
    _fields_ = [(name, ctypes.c_void_p) for name in
                ("status", "n_events", "misses", "job_task", "job_k", "job_resp", "job_rank",
                 "seg_max", "resp_max", "events")]


def _lib():
    L = _native.lib()
    if not getattr(L, "_sim_ready", False):
        p64 = ctypes.POINTER(ctypes.c_int64)
        L.rtgpu_sim_host.argtypes = [p64, p64, ctypes.c_int64, p64, p64, p64, ctypes.c_int32,
                                     ctypes.POINTER(_SimOut)]
        L.rtgpu_sim_device.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64] + \
            [ctypes.c_void_p] * 6 + [ctypes.c_int32, ctypes.POINTER(_SimOut), ctypes.c_void_p]
        L.rtgpu_sim_scratch_words.argtypes = [p64]
        L.rtgpu_sim_scratch_words.restype = ctypes.c_int64
        L.rtgpu_sim_last_error.restype = ctypes.c_char_p
        L._sim_ready = True
    return L


@dataclass
class SimBatch:
    """Device results of simulate_batch (arrays per simulation / job / task)."""
    packs: list
    status: np.ndarray
    n_events: np.ndarray
    misses: np.ndarray
    job_base: np.ndarray
    task_base: np.ndarray
    job_task: np.ndarray
    job_k: np.ndarray
    job_resp: np.ndarray
    job_rank: np.ndarray
    seg_max: np.ndarray     # [total tasks, smax]
    resp_max: np.ndarray
    ev_base: Optional[np.ndarray] = None
    events: Optional[np.ndarray] = None  # [total events, 2] int64 (time, packed)

    def trace(self, s: int) -> SimTrace:
        """SimTrace of simulation s (needs events=True)."""
        pk = self.packs[s]
        Q, tasks = pk.Q, pk.tasks
        out = SimTrace()
        if self.events is not None:
            ev = self.events[self.ev_base[s]:self.ev_base[s] + self.n_events[s]]
            for tm, pw in ev.tolist():
                pw &= (1 << 64) - 1
                out.events.append(SimEvent(Fraction(tm, Q), tasks[(pw >> 32) & 0xFF].id,
                                           pw & 0xFFFFFFFF, KINDS[(pw >> 40) & 0xF],
                                           ((pw >> 48) & 0xFF) - 1, ACTIONS[(pw >> 44) & 0xF]))
        a, b = self.job_base[s], self.job_base[s + 1]
        jt, jk = self.job_task[a:b].tolist(), self.job_k[a:b].tolist()
        jr, jn = self.job_resp[a:b].tolist(), self.job_rank[a:b].tolist()
        done = sorted((jn[x], x) for x in range(b - a) if jr[x] >= 0)
        for _, x in done:
            out.responses[(tasks[jt[x]].id, jk[x])] = Fraction(jr[x], Q)
        for x in range(b - a):
            t = tasks[jt[x]]
            out.releases[(t.id, jk[x])] = jk[x] * Fraction(t.period)
            if jr[x] < 0:
                out.truncated.append((t.id, jk[x]))
        return out

    def check(self, s: int, report: AnalysisReport) -> list:
        """check_against_analysis's violations for simulation s, from the
        device-side maxima (one line per task/segment bound exceeded, per task
        whose end-to-end bound is exceeded, and the deadline-miss count)."""
        if not report.schedulable:
            raise ValueError("report must be from an accepting analysis")
        pk = self.packs[s]
        out = []
        if self.misses[s]:
            out.append(f"{int(self.misses[s])} deadline-miss events")
        for i, t in enumerate(pk.tasks):
            tr = report.per_task.get(t.id)
            if tr is None:
                continue
            row = self.seg_max[self.task_base[s] + i]
            for p, (kind, seg) in enumerate(pk.plans[i]):
                v = int(row[p])
                if v < 0:
                    continue
                bound = _segment_bound(tr, kind, seg)
                if bound is not None and Fraction(v, pk.Q) > bound:
                    out.append(f"task {t.id}: {kind} segment {seg} response "
                               f"{Fraction(v, pk.Q)} > bound {bound}")
            rm = int(self.resp_max[self.task_base[s] + i])
            if tr.end_to_end_up is not None and rm >= 0 and Fraction(rm, pk.Q) > tr.end_to_end_up:
                out.append(f"task {t.id}: end-to-end response {Fraction(rm, pk.Q)} > bound "
                           f"{tr.end_to_end_up}")
        return out


def simulate_batch(items: Sequence, cfg=SimConfig(), events: bool = False,
                   pool: Optional[int] = None) -> SimBatch:
    """Simulate many (TaskSet, SmAllocation) pairs in one GPU launch; cfg is
    one SimConfig or one per item.  events=True also returns every trace.
    Runs whose live jobs outgrow the recycled record pool are re-run with
    one record per release point."""
    _native.require_device()
    cfgs = list(cfg) if isinstance(cfg, (list, tuple)) else [cfg] * len(items)
    packs = [pack_simulation(ts, al, c, pool) for (ts, al), c in zip(items, cfgs)]
    res = _run_packs(packs, events)
    redo = [s for s in range(len(packs)) if res.status[s] == 3]
    if redo:
        again = _run_packs([pack_simulation(*items[s], cfgs[s], 0) for s in redo], events)
        res = _merge(res, redo, again)
    bad = np.nonzero(res.status)[0]
    if len(bad):
        raise RuntimeError(f"simulator: status {int(res.status[bad[0]])} for simulation "
                           f"{int(bad[0])}")
    return res


def _merge(res: SimBatch, redo: list, again: SimBatch) -> SimBatch:
    """Replace the results of simulations `redo` by those of `again`."""
    packs = list(res.packs)
    for x, s in enumerate(redo):
        packs[s] = again.packs[x]
    pick = {s: x for x, s in enumerate(redo)}
    src = [(again, pick[s]) if s in pick else (res, s) for s in range(len(packs))]

    def cat(name, base):
        parts = []
        for b, s in src:
            bb = getattr(b, base)
            parts.append(getattr(b, name)[bb[s]:bb[s + 1]])
        return np.concatenate(parts) if parts else getattr(res, name)

    def bases(key):
        return np.concatenate([[0], np.cumsum([getattr(b, key)[s + 1] - getattr(b, key)[s]
                                               for b, s in src])]).astype(np.int64)
    out = SimBatch(packs, np.array([b.status[s] for b, s in src], np.int32),
                   np.array([b.n_events[s] for b, s in src], np.int64),
                   np.array([b.misses[s] for b, s in src], np.int64),
                   bases("job_base"), bases("task_base"),
                   cat("job_task", "job_base"), cat("job_k", "job_base"),
                   cat("job_resp", "job_base"), cat("job_rank", "job_base"),
                   np.zeros((0, 1), np.int64), cat("resp_max", "task_base"))
    w = max(res.seg_max.shape[1], again.seg_max.shape[1])
    rows = []
    for b, s in src:
        r = b.seg_max[b.task_base[s]:b.task_base[s + 1]]
        rows.append(np.pad(r, ((0, 0), (0, w - r.shape[1])), constant_values=-1))
    out.seg_max = np.concatenate(rows) if rows else np.zeros((0, w), np.int64)
    if res.events is not None:
        out.events = np.concatenate([b.events[b.ev_base[s]:b.ev_base[s] + b.n_events[s]]
                                     for b, s in src]) if src else res.events
        out.ev_base = np.concatenate([[0], np.cumsum([b.n_events[s] for b, s in src])]
                                     ).astype(np.int64)
    return out


def _run_packs(packs: list, events: bool) -> SimBatch:
    S = len(packs)
    set_off = np.zeros(S + 1, np.int64)
    job_base = np.zeros(S + 1, np.int64)
    task_base = np.zeros(S + 1, np.int64)
    ev_base = np.zeros(S + 1, np.int64)
    for s, pk in enumerate(packs):
        set_off[s + 1] = set_off[s] + len(pk.blob)
        job_base[s + 1] = job_base[s] + pk.R
        task_base[s + 1] = task_base[s] + len(pk.tasks)
        ev_base[s + 1] = ev_base[s] + (pk.evcap if events else 0)
    blobs = np.concatenate([pk.blob for pk in packs]) if packs else np.zeros(1, np.int64)
    smax = max([pk.smax for pk in packs] + [1])
    NJ, NT, NE = int(job_base[-1]), int(task_base[-1]), int(ev_base[-1])
    res = SimBatch(packs, np.zeros(S, np.int32), np.zeros(S, np.int64), np.zeros(S, np.int64),
                   job_base, task_base, np.zeros(NJ, np.int32), np.zeros(NJ, np.int32),
                   np.zeros(NJ, np.int64), np.zeros(NJ, np.int32),
                   np.zeros((NT, smax), np.int64), np.zeros(NT, np.int64),
                   ev_base if events else None,
                   np.zeros((NE, 2), np.int64) if events else None)
    if S == 0:
        return res
    o = _SimOut(*[a.ctypes.data for a in (res.status, res.n_events, res.misses, res.job_task,
                                          res.job_k, res.job_resp, res.job_rank, res.seg_max,
                                          res.resp_max)],
                res.events.ctypes.data if events and NE else None)
    p64 = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))  # noqa: E731
    L = _lib()
    rc = L.rtgpu_sim_host(p64(blobs), p64(set_off), S, p64(job_base), p64(task_base),
                          p64(ev_base) if events else None, smax, ctypes.byref(o))
    if rc != 0:
        raise RuntimeError("simulator: " + L.rtgpu_sim_last_error().decode())
    return res


class DeviceSimBatch:
    """Packed simulations resident in HBM (torch tensors as allocations),
    run with rtgpu_sim_device on a CUDA stream -- the bulk validation path."""

    def __init__(self, packs: list, device: str = "cuda", events: bool = False):
        import torch
        _native.require_device()
        L = _lib()
        self.packs = packs
        S = self.n = len(packs)
        self.events = events
        self.device = torch.device(device)
        off = np.zeros((6, S + 1), np.int64)   # set_off, job_base, task_base, ev_base, scr_off,
        # and the launch order: longest simulations (most events) first
        for s, pk in enumerate(packs):
            off[:5, s + 1] = off[:5, s] + [len(pk.blob), pk.R, len(pk.tasks),
                                         pk.evcap if events else 0,
                                         L.rtgpu_sim_scratch_words(pk.blob.ctypes.data_as(
                                             ctypes.POINTER(ctypes.c_int64)))]
        off[5, :S] = np.argsort([-pk.evcap for pk in packs], kind="stable")
        self.offsets = off
        self.smax = max([pk.smax for pk in packs] + [1])
        blobs = np.concatenate([pk.blob for pk in packs]) if packs else np.zeros(1, np.int64)
        dev = self.device
        t64 = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.int64)).to(dev)  # noqa: E731
        self.d_blobs, self.d_off = t64(blobs), t64(off)
        self.scratch = torch.empty(int(off[4, -1]) + 1, dtype=torch.int64, device=dev)
        NJ, NT, NE = int(off[1, -1]), int(off[2, -1]), int(off[3, -1])
        e = lambda n, dt: torch.empty(max(n, 1), dtype=dt, device=dev)  # noqa: E731
        self.out = {"status": e(S, torch.int32), "n_events": e(S, torch.int64),
                    "misses": e(S, torch.int64), "job_task": e(NJ, torch.int32),
                    "job_k": e(NJ, torch.int32), "job_resp": e(NJ, torch.int64),
                    "job_rank": e(NJ, torch.int32), "seg_max": e(NT * self.smax, torch.int64),
                    "resp_max": e(NT, torch.int64),
                    "events": e(2 * NE, torch.int64) if events else None}
        self.input_bytes = 8 * (len(blobs) + 6 * (S + 1))

    def run(self, stream=None) -> None:
        import torch
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        o = self.out
        so = _SimOut(*[o[k].data_ptr() for k in ("status", "n_events", "misses", "job_task",
                                                  "job_k", "job_resp", "job_rank", "seg_max",
                                                  "resp_max")],
                     o["events"].data_ptr() if self.events else None)
        base = self.d_off.data_ptr()
        row = 8 * (self.n + 1)
        L = _lib()
        rc = L.rtgpu_sim_device(self.d_blobs.data_ptr(), base, self.n, base + row,
                                base + 2 * row, base + 3 * row if self.events else None,
                                base + 4 * row, self.scratch.data_ptr(), base + 5 * row,
                                self.smax, ctypes.byref(so), stream.cuda_stream)
        if rc:
            raise RuntimeError("simulator: " + L.rtgpu_sim_last_error().decode())

    def to_host(self) -> SimBatch:
        o = {k: (None if v is None else v.cpu().numpy()) for k, v in self.out.items()}
        off = self.offsets
        NJ, NT, NE = int(off[1, -1]), int(off[2, -1]), int(off[3, -1])
        return SimBatch(self.packs, o["status"][:self.n], o["n_events"][:self.n],
                        o["misses"][:self.n], off[1], off[2], o["job_task"][:NJ],
                        o["job_k"][:NJ], o["job_resp"][:NJ], o["job_rank"][:NJ],
                        o["seg_max"][:NT * self.smax].reshape(NT, self.smax), o["resp_max"][:NT],
                        off[3] if self.events else None,
                        o["events"][:2 * NE].reshape(NE, 2) if self.events else None)


def simulate(ts: TaskSet, alloc: SmAllocation, cfg: SimConfig) -> SimTrace:
    """The reference's simulate (simulator.py:160), run on the GPU."""
    return simulate_batch([(ts, alloc)], cfg, events=True).trace(0)


def _segment_bound(tr, kind: str, seg: int):
    """The report's bound for one segment (None: not bounded)."""
    table = {"mem": tr.mem_r_up, "cpu": tr.cpu_r_up,
             "gpu": tuple(b.hi for b in tr.gpu_r)}.get(kind, ())
    return table[seg] if 0 <= seg < len(table) else None


def check_against_analysis(trace: SimTrace, report: AnalysisReport) -> list:
    """Observed responses above their bounds and deadline misses
    (simulator.py:340): first every deadline miss in trace order, then every
    finished segment of a non-truncated job (start-to-finish, in order of
    completion), then every end-to-end response (in completion order)."""
    if not report.schedulable:
        raise ValueError("report must be from an accepting analysis")
    skip = set(trace.truncated)
    misses, first_start, finished = [], {}, {}
    for e in trace.events:
        if e.action == "deadline-miss":
            misses.append(f"task {e.task} job {e.job}: deadline miss at {e.time}")
        if e.kind == "job":
            continue
        key = (e.task, e.job, e.kind, e.segment)
        if e.action == "start" and key not in first_start:
            first_start[key] = e.time
        elif e.action == "finish":
            finished[key] = e.time
    seg_lines = []
    for key, t_end in finished.items():
        task, job, kind, seg = key
        tr = report.per_task.get(task)
        if (task, job) in skip or tr is None:
            continue
        bound = _segment_bound(tr, kind, seg)
        took = t_end - first_start[key]
        if bound is not None and took > bound:
            seg_lines.append(f"task {task} job {job}: {kind} segment {seg} response {took} > "
                             f"bound {bound}")
    e2e_lines = [f"task {task} job {job}: end-to-end response {r} > bound "
                 f"{report.per_task[task].end_to_end_up}"
                 for (task, job), r in trace.responses.items()
                 if report.per_task.get(task) is not None
                 and report.per_task[task].end_to_end_up is not None
                 and r > report.per_task[task].end_to_end_up]
    return misses + seg_lines + e2e_lines
