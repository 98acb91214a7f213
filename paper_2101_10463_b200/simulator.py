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
from .model import AnalysisReport, SmAllocation, TaskSet, TaskSpec, duration_to_str, validate_taskset

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


def pack_simulation(ts: TaskSet, alloc: SmAllocation, cfg: SimConfig) -> _Packed:
    """Validate like simulate() and build the simulator blob (rtgpu_sim.h)."""
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
    blob[:8] = [n, int(uniform), H, R, evcap, len(key), smax, seg_off]
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
                bound = None
                if kind == "mem" and seg < len(tr.mem_r_up):
                    bound = tr.mem_r_up[seg]
                elif kind == "cpu" and seg < len(tr.cpu_r_up):
                    bound = tr.cpu_r_up[seg]
                elif kind == "gpu" and seg < len(tr.gpu_r):
                    bound = tr.gpu_r[seg].hi
                if bound is not None and Fraction(v, pk.Q) > bound:
                    out.append(f"task {t.id}: {kind} segment {seg} response "
                               f"{Fraction(v, pk.Q)} > bound {bound}")
            rm = int(self.resp_max[self.task_base[s] + i])
            if tr.end_to_end_up is not None and rm >= 0 and Fraction(rm, pk.Q) > tr.end_to_end_up:
                out.append(f"task {t.id}: end-to-end response {Fraction(rm, pk.Q)} > bound "
                           f"{tr.end_to_end_up}")
        return out


def simulate_batch(items: Sequence, cfg=SimConfig(), events: bool = False) -> SimBatch:
    """Simulate many (TaskSet, SmAllocation) pairs in one GPU launch; cfg is
    one SimConfig or one per item.  events=True also returns every trace."""
    _native.require_device()
    cfgs = list(cfg) if isinstance(cfg, (list, tuple)) else [cfg] * len(items)
    packs = [pack_simulation(ts, al, c) for (ts, al), c in zip(items, cfgs)]
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
    bad = np.nonzero(res.status)[0]
    if len(bad):
        raise RuntimeError(f"simulator: status {int(res.status[bad[0]])} for simulation "
                           f"{int(bad[0])}")
    return res


def simulate(ts: TaskSet, alloc: SmAllocation, cfg: SimConfig) -> SimTrace:
    """The reference's simulate (simulator.py:160), run on the GPU."""
    return simulate_batch([(ts, alloc)], cfg, events=True).trace(0)


def check_against_analysis(trace: SimTrace, report: AnalysisReport) -> list:
    """Observed responses above their bounds and deadline misses, in the
    reference's order and wording (simulator.py:340)."""
    if not report.schedulable:
        raise ValueError("report must be from an accepting analysis")
    out = []
    truncated = set(trace.truncated)
    for e in trace.events:
        if e.action == "deadline-miss":
            out.append(f"task {e.task} job {e.job}: deadline miss at {e.time}")
    ready, finish = {}, {}
    for e in trace.events:
        if e.kind == "job":
            continue
        key = (e.task, e.job, e.kind, e.segment)
        if e.action == "start":
            ready.setdefault(key, e.time)
        elif e.action == "finish":
            finish[key] = e.time
    for (task, jobidx, kind, seg), t_fin in finish.items():
        if (task, jobidx) in truncated:
            continue
        tr = report.per_task.get(task)
        if tr is None:
            continue
        resp = t_fin - ready[(task, jobidx, kind, seg)]
        bound = None
        if kind == "mem" and seg < len(tr.mem_r_up):
            bound = tr.mem_r_up[seg]
        elif kind == "cpu" and seg < len(tr.cpu_r_up):
            bound = tr.cpu_r_up[seg]
        elif kind == "gpu" and seg < len(tr.gpu_r):
            bound = tr.gpu_r[seg].hi
        if bound is not None and resp > bound:
            out.append(f"task {task} job {jobidx}: {kind} segment {seg} response {resp} > bound "
                       f"{bound}")
    for (task, jobidx), resp in trace.responses.items():
        tr = report.per_task.get(task)
        if tr is None or tr.end_to_end_up is None:
            continue
        if resp > tr.end_to_end_up:
            out.append(f"task {task} job {jobidx}: end-to-end response {resp} > bound "
                       f"{tr.end_to_end_up}")
    return out
