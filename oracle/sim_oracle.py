"""TEST INFRASTRUCTURE -- the checker, never the product.

CPU restatement of the reference's discrete-event simulator
(/root/reference/pkg/src/gpusched/simulator.py), used only by tests/ and
bench.py's cpu_baseline to check the GPU simulator (csrc/simulator.cu).
Pinned against the reference's own traces (tests/golden/sim_golden.json,
made by tests/golden/make_golden_sim.py) in tests/test_sim_oracle.py.

Semantics restated (simulator.py line refs):
  * release points k*T < horizon for every task, processed in (time,
    priority) order (:186-193); at release the job's segment lengths are
    drawn in plan order (:114-139), a deadline event is queued (:303) and
    the first segment dispatched;
  * one preemptive fixed-priority CPU (:200-239), one non-preemptive
    fixed-priority bus (:241-251), dedicated SMs: a GPU segment starts at
    once (:266-268);
  * equal-time order: finishes, deadlines, releases; within a kind, queue
    push order (:34, :181-184);
  * a job finishing after its deadline logs a second deadline miss (:277);
  * events past the horizon end the run; unfinished jobs are truncated.
Time is exact (Fraction); the heap holds (time, order, seq, item).
"""
from __future__ import annotations

import heapq
import random
from fractions import Fraction

FIN, DL, REL = 0, 1, 2


def plan_of(task, two_copy):
    out = []
    for j in range(task.n_subtasks - 1):
        out.append(("cpu", j))
        out.extend([("mem", 2 * j), ("gpu", j), ("mem", 2 * j + 1)] if two_copy
                   else [("mem", j), ("gpu", j)])
    out.append(("cpu", task.n_subtasks - 1))
    return out


def gpu_hi(g, vs):
    infl = g.work.hi * g.interleave_ratio
    if g.critical_path_overhead > infl:
        raise ValueError("critical-path overhead exceeds inflated work")
    return (infl - g.critical_path_overhead) / vs + g.critical_path_overhead


class _J:
    def __init__(self, task, k, rel, lens):
        self.task, self.k, self.rel = task, k, rel
        self.dl = rel + task.deadline
        self.lens = lens
        self.pos = 0
        self.rem = Fraction(0)
        self.done = False


def simulate(ts, alloc, horizon=None, seed=0, uniform=False):
    """Returns (events, responses, releases, truncated) like SimTrace:
    events are (time, task id, job, kind, segment, action)."""
    two = ts.mem_model.value == "two_copy"
    if horizon is None:
        horizon = 20 * max((t.period for t in ts.tasks), default=Fraction(1))
    rng = random.Random(seed)
    tasks = sorted(ts.tasks, key=lambda t: t.priority)
    plans = {t.id: plan_of(t, two) for t in tasks}
    ev, resp, rels, jobs = [], {}, {}, []
    heap, ctr = [], [0]

    def push(t, order, item):
        heapq.heappush(heap, (t, order, ctr[0], item))
        ctr[0] += 1

    pts = []
    for t in tasks:
        k = 0
        while k * t.period < horizon:
            pts.append((Fraction(k) * t.period, t.priority, t, k))
            k += 1
    for tm, _, t, k in sorted(pts, key=lambda x: (x[0], x[1])):
        push(tm, REL, ("rel", t, k))

    cpu = {"run": None, "tok": 0, "fin": None, "ready": []}
    bus = {"busy": None, "q": []}

    def log(tm, j, kind, seg, act):
        ev.append((tm, j.task.id, j.k, kind, seg, act))

    def draw(t):
        vs = alloc.virtual_sms(t.id)
        out = []
        for kind, idx in plans[t.id]:
            if kind == "gpu":
                g = t.gpu_segments[idx]
                if not uniform:
                    out.append(gpu_hi(g, vs))
                    continue
                w = g.work.hi if g.work.lo == g.work.hi else Fraction(
                    rng.randint(int(g.work.lo), int(g.work.hi)))
                out.append((w * g.interleave_ratio - g.critical_path_overhead) / vs
                           + g.critical_path_overhead)
            else:
                b = (t.cpu_segments if kind == "cpu" else t.mem_segments)[idx]
                out.append(b.hi if (not uniform or b.lo == b.hi)
                           else Fraction(rng.randint(int(b.lo), int(b.hi))))
        return out

    def first_best(lst):
        return min(range(len(lst)), key=lambda x: (lst[x].task.priority, x))

    def run_cpu(tm, j):
        cpu["run"] = j
        cpu["tok"] += 1
        fresh = j.rem == j.lens[j.pos]
        log(tm, j, "cpu", plans[j.task.id][j.pos][1], "start" if fresh else "resume")
        cpu["fin"] = tm + j.rem
        push(tm + j.rem, FIN, ("cpu", j, cpu["tok"]))

    def cpu_sched(tm):
        if not cpu["ready"]:
            return
        x = first_best(cpu["ready"])
        top = cpu["ready"][x]
        cur = cpu["run"]
        if cur is None:
            cpu["ready"].pop(x)
            run_cpu(tm, top)
        elif top.task.priority < cur.task.priority:
            cur.rem = cpu["fin"] - tm
            log(tm, cur, "cpu", plans[cur.task.id][cur.pos][1], "preempt")
            cpu["ready"].pop(x)
            cpu["ready"].append(cur)
            cpu["run"] = None
            run_cpu(tm, top)

    def bus_grant(tm):
        if bus["busy"] is not None or not bus["q"]:
            return
        j = bus["q"].pop(first_best(bus["q"]))
        bus["busy"] = j
        log(tm, j, "mem", plans[j.task.id][j.pos][1], "start")
        push(tm + j.lens[j.pos], FIN, ("bus", j))

    def route(tm, j):
        kind, idx = plans[j.task.id][j.pos]
        if kind == "cpu":
            j.rem = j.lens[j.pos]
            cpu["ready"].append(j)
            cpu_sched(tm)
        elif kind == "mem":
            bus["q"].append(j)
            bus_grant(tm)
        else:
            log(tm, j, "gpu", idx, "start")
            push(tm + j.lens[j.pos], FIN, ("gpu", j))

    def step(tm, j):
        kind, idx = plans[j.task.id][j.pos]
        log(tm, j, kind, idx, "finish")
        j.pos += 1
        if j.pos < len(j.lens):
            route(tm, j)
            return
        j.done = True
        resp[(j.task.id, j.k)] = tm - j.rel
        if tm > j.dl:
            log(tm, j, "job", -1, "deadline-miss")

    while heap:
        tm, _, _, item = heapq.heappop(heap)
        if tm > horizon:
            break
        what = item[0]
        if what == "rel":
            t, k = item[1], item[2]
            j = _J(t, k, tm, draw(t))
            jobs.append(j)
            rels[(t.id, k)] = tm
            log(tm, j, "job", -1, "release")
            push(j.dl, DL, ("dl", j))
            route(tm, j)
        elif what == "cpu":
            if item[2] != cpu["tok"] or cpu["run"] is not item[1]:
                continue
            cpu["run"] = None
            step(tm, item[1])
            cpu_sched(tm)
        elif what == "bus":
            bus["busy"] = None
            step(tm, item[1])
            bus_grant(tm)
        elif what == "gpu":
            step(tm, item[1])
        elif not item[1].done:
            log(tm, item[1], "job", -1, "deadline-miss")
    trunc = [(j.task.id, j.k) for j in jobs if not j.done]
    return ev, resp, rels, trunc
