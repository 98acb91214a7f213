"""Summarise ncu captures into profiles/ (run on the CPU box after gpurun).

    python scripts/make_profiles.py gpurun_out/prof_X.ncu-rep [gpurun_out/launches.csv] --tag r1

Writes profiles/ncu_summary.json (read by bench.py: DRAM traffic per launch
and the issue-rate evidence of the dominant kernel) and
profiles/<tag>_front_kernel.json (the full counter summary); with a launch
list, profiles/<tag>_launches.csv (per-launch device times, cold-cache and
serialised: compare shares, not absolutes) plus the per-kernel share.
"""
from __future__ import annotations

import csv
import io
import json
import os
import shutil
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

METRICS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "sm__inst_executed.avg.per_cycle_active": "ipc_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "smsp__inst_executed.sum": "warp_instructions",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "sm__maximum_warps_per_active_cycle_pct": "theoretical_occupancy_pct",
    "launch__registers_per_thread": "registers_per_thread",
    "launch__occupancy_limit_registers": "occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem": "occupancy_limit_shared_mem",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "active_threads_per_warp_inst",
    "smsp__sass_average_branch_targets_threads_uniform.pct": "branch_uniform_pct",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu_pipe_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "launch__grid_size": "grid_size",
    "launch__block_size": "block_size",
}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    return {h[i]: (v[i], u[i]) for i in range(len(h))}


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return None


SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "usecond": 1e3,
         "ms": 1e6, "msecond": 1e6, "nsecond": 1, "s": 1e9, "second": 1e9}


def to_base(v, unit):
    """ncu scales units per value (Mbyte, ms ...): back to bytes / ns."""
    if v is None:
        return None
    return v * SCALE.get(unit, 1)


def summarise(rep):
    d = raw(rep)
    s = {"kernel": d.get("Kernel Name", ("?", ""))[0]}
    for k, name in METRICS.items():
        if k in d:
            s[name] = to_base(num(d[k][0]), d[k][1])
    stalls = {}
    for k, (val, _) in d.items():
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            v = num(val)
            if v:
                stalls[k.replace("smsp__pcsamp_warps_issue_stalled_", "")] = v
    tot = sum(stalls.values()) or 1
    s["stall_share"] = {k: round(v / tot, 3) for k, v in sorted(stalls.items(), key=lambda x: -x[1])
                        if v / tot >= 0.01}
    return s


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and "Kernel Name" in r)
    h = rows[hi]
    kn, mv, mn = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    per = defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) > mv and r[mn] == "gpu__time_duration.sum":
            name = r[kn].split("(")[0]
            per[name][0] += 1
            per[name][1] += num(r[mv]) or 0.0
    total = sum(v[1] for v in per.values()) or 1
    return {k: {"launches": v[0], "time_ns": v[1], "share": round(v[1] / total, 4)}
            for k, v in sorted(per.items(), key=lambda x: -x[1][1])}


def main():
    """python scripts/make_profiles.py REP [LAUNCHES.csv] --tag T [--key fast_kernel]
    [--sets N] [--lib-sha SHA]: the capture's summary is merged into
    profiles/ncu_summary.json under kernels[key] (bench.py reads it and checks
    lib_sha against the library it benches)."""
    argv = sys.argv[1:]
    opt = {}
    for name in ("--tag", "--key", "--sets", "--lib-sha"):
        if name in argv:
            i = argv.index(name)
            opt[name] = argv[i + 1]
            del argv[i:i + 2]
    args = [a for a in argv if not a.startswith("--")]
    tag = opt.get("--tag", "r1")
    key = opt.get("--key", "fast_kernel")
    rep = args[0]
    os.makedirs(PROF, exist_ok=True)
    s = summarise(rep)
    with open(os.path.join(PROF, f"{tag}_{key}.json"), "w") as fh:
        json.dump(s, fh, indent=1)
    launch = None
    if len(args) > 1 and os.path.exists(args[1]):
        shutil.copy(args[1], os.path.join(PROF, f"{tag}_launches.csv"))
        launch = launches(args[1])
        with open(os.path.join(PROF, f"{tag}_launch_shares.json"), "w") as fh:
            json.dump(launch, fh, indent=1)
    traffic = (s.get("dram_read_bytes") or 0) + (s.get("dram_write_bytes") or 0)
    entry = {
        "source": os.path.basename(rep),
        "tag": tag,
        "kernel": s["kernel"],
        "duration_ns": s.get("duration_ns"),
        "dram_bytes_per_launch": traffic,
        "dram_read_bytes": s.get("dram_read_bytes"),
        "dram_write_bytes": s.get("dram_write_bytes"),
        "warp_instructions": s.get("warp_instructions"),
        "lib_sha": opt.get("--lib-sha"),
        "issue": {"ipc_active": s.get("ipc_active"), "issue_slots_busy_pct": s.get("issue_active_pct"),
                  "peak_ipc": 4.0, "fp64_pipe_pct": s.get("fp64_pipe_pct"),
                  "alu_pipe_pct": s.get("alu_pipe_pct"), "fma_pipe_pct": s.get("fma_pipe_pct"),
                  "lsu_pipe_pct": s.get("lsu_pipe_pct"),
                  "achieved_occupancy_pct": s.get("achieved_occupancy_pct"),
                  "registers_per_thread": s.get("registers_per_thread"),
                  "active_threads_per_warp_inst": s.get("active_threads_per_warp_inst"),
                  "branch_uniform_pct": s.get("branch_uniform_pct"),
                  "top_stalls": s["stall_share"]},
        "launch_shares": launch,
    }
    if "--sets" in opt and s.get("warp_instructions"):
        entry["sets_per_launch"] = int(opt["--sets"])
        entry["warp_instructions_per_set"] = s["warp_instructions"] / int(opt["--sets"])
    path = os.path.join(PROF, "ncu_summary.json")
    summary = {}
    if os.path.exists(path):
        with open(path) as fh:
            summary = json.load(fh)
    if "kernels" not in summary:
        summary = {"kernels": {}}
    summary["kernels"][key] = entry
    with open(path, "w") as fh:
        json.dump(summary, fh, indent=1)
    print(json.dumps(entry, indent=1))


if __name__ == "__main__":
    main()
