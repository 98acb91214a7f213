"""TEST HELPERS: blob conversion and an adversarial task-set generator.

compact(): int64 blobs -> the compact (int32 segment) blob form the fast and
lattice paths read.

adversarial(): packed task sets built to stress the allocation-search
argument rather than to look like the benchmark:

* tight tasks -- interleave ratio 1, no launch overhead, lo == hi and
  D = T = the task's isolated bound at a chosen count g0 plus 0..2 ticks,
  so the wrap-around gaps (analysis.py:89, :57) are within a few ticks of
  zero at g_min: the boundary of the regularity the greedy descent needs;
* lo < hi segments (gaps use lo, demand uses hi);
* irregular tasks -- copy lower bounds above their upper bounds, the only
  way (besides D > T) a task passing its isolated bound gets a negative
  wrap-around gap, which sends the set to the exact depth-first search;
* CPU-only tasks (one segment) and equal priorities (the reference's
  by_priority is a stable sort on the priority value, model.py:107).
"""
from __future__ import annotations

import numpy as np

from paper_2101_10463_b200.pack import build_blob

HDR, TW = 8, 8


def compact(blobs, set_off, task_base):
    """int64 blobs -> the compact form (int32 segment areas, header word 7 =
    1) wherever every segment value fits int32 (others stay int64)."""
    words, offs = [], [0]
    for s in range(len(set_off) - 1):
        b = [int(x) for x in blobs[set_off[s]:set_off[s + 1]]]
        n = b[0]
        base = HDR + TW * n
        seg = b[base:]
        if b[7] == 0 and all(-2**31 <= v < 2**31 for v in seg):
            recs = b[HDR:base]
            for i in range(n):
                recs[TW * i + 5] = 2 * base + (recs[TW * i + 5] - base)  # int32 element offset
            if len(seg) % 2:
                seg = seg + [0]
            packed = np.asarray(seg, np.int32).view(np.int64).tolist()
            b = b[:HDR] + recs + packed
            b[7] = 1
            b[4] = len(b)
        words += b
        offs.append(len(words))
    return np.asarray(words, np.int64), np.asarray(offs, np.int64), np.asarray(task_base, np.int64)


def _task(rng, m, mm, A, kind, gn, n, u_hi):
    p = 0 if m < 2 else (2 * m - 2 if mm == 0 else m - 1)
    cl_hi = rng.integers(1000, 20001, m)
    ml_hi = rng.integers(250, 5001, p)
    gw_hi = rng.integers(1000, 20001, m - 1)
    if kind == "tight":
        cl_lo, ml_lo, gw_lo = cl_hi.copy(), ml_hi.copy(), gw_hi.copy()
        gl = np.zeros(m - 1, np.int64)
        an = np.full(m - 1, A, np.int64)  # interleave ratio 1
        g0 = int(rng.integers(1, max(2, gn // max(1, n)) + 1))
        # isolated bound at g0: sum cl_hi + sum ml_hi + sum_j GW_j / (2 g0)
        iso = int(cl_hi.sum() + ml_hi.sum()) + (-(-int(gw_hi.sum()) // (2 * g0)) if m > 1 else 0)
        D = iso + int(rng.integers(0, 3))
        return dict(m=m, p=p, D=D, T=D, cl_lo=cl_lo, cl_hi=cl_hi, ml_lo=ml_lo, ml_hi=ml_hi,
                    gw_lo=gw_lo, gw_hi=gw_hi, gl=gl, an=an)
    lo_f = rng.uniform(0.5, 1.0) if kind in ("lohi", "irregular") else 1.0
    cl_lo = np.minimum(cl_hi, (cl_hi * lo_f).astype(np.int64))
    gw_lo = np.minimum(gw_hi, (gw_hi * lo_f).astype(np.int64))
    ml_lo = np.minimum(ml_hi, (ml_hi * lo_f).astype(np.int64))
    if kind == "irregular" and p > 0:
        ml_lo = (ml_hi * rng.uniform(1.0, 3.0, p)).astype(np.int64)  # lo > hi
    pct = rng.integers(100, 181, m - 1)
    an = pct * A // 100
    gl = np.minimum((gw_hi * 12) // 100, gw_lo)
    demand = int(cl_hi.sum() + ml_hi.sum() + gw_hi.sum())
    u = rng.uniform(0.1 * u_hi, u_hi)
    D = max(1, int(demand / u))
    return dict(m=m, p=p, D=D, T=D, cl_lo=cl_lo, cl_hi=cl_hi, ml_lo=ml_lo, ml_hi=ml_hi,
                gw_lo=gw_lo, gw_hi=gw_hi, gl=gl, an=an)


def adversarial(seed: int, count: int, n: int, m_max: int, gn: int, mm: int,
                p_tight=0.15, p_lohi=0.3, p_irreg=0.0, p_cpu=0.15, p_eq=0.3, u_total=1.0):
    """(blobs, set_off, task_base) of `count` adversarial sets (int64 blobs)."""
    rng = np.random.default_rng(seed)
    A = 100
    words, offs, tbs = [], [0], [0]
    for _ in range(count):
        rows = []
        for i in range(n):
            m = 1 if rng.random() < p_cpu else int(rng.integers(2, m_max + 1))
            r = rng.random()
            kind = ("tight" if r < p_tight else "lohi" if r < p_tight + p_lohi
                    else "irregular" if r < p_tight + p_lohi + p_irreg else "plain")
            t = _task(rng, m, mm, A, kind if m > 1 else "plain", gn, n, 2.0 * u_total / n)
            t["idx"] = i
            rows.append(t)
        # deadline-monotonic priorities, some merged into ties
        order = sorted(range(n), key=lambda i: (rows[i]["D"], i))
        prio, cur = [0] * n, 0
        for rank, i in enumerate(order):
            if rank == 0 or rng.random() >= p_eq:
                cur += 1
            prio[i] = cur
        for i in range(n):
            rows[i]["prio"] = prio[i]
        rows.sort(key=lambda t: (t["prio"], t["idx"]))  # by_priority: stable sort on priority
        rows = [{k: (list(int(x) for x in v) if isinstance(v, np.ndarray) else int(v))
                 for k, v in t.items()} for t in rows]
        b = build_blob(rows, gn, mm, A)
        words += b
        offs.append(len(words))
        tbs.append(tbs[-1] + n)
    return np.asarray(words, np.int64), np.asarray(offs, np.int64), np.asarray(tbs, np.int64)
