"""Simulator throughput probe: generation, packing and kernel time."""
import sys
import time
from fractions import Fraction

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2101_10463_b200.analysis import analyze_batch  # noqa: E402
from paper_2101_10463_b200.simulator import DeviceSimBatch, SimConfig, pack_simulation  # noqa: E402
from paper_2101_10463_b200.workbench import GenParams, generate_taskset  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
t0 = time.time()
gp = GenParams(n_tasks=8, n_subtasks=5, physical_sms=10, target_utilization=Fraction(1, 2))
sets = [generate_taskset(gp, f"1000:1/2:{i}") for i in range(n)]
t1 = time.time()
reps = analyze_batch(sets)
acc = [(s, r) for s, r in zip(sets, reps) if r.schedulable]
t2 = time.time()
packs = [pack_simulation(s, r.allocation, SimConfig(), None) for s, r in acc]
t3 = time.time()
print(f"gen {t1 - t0:.1f}s analyze {t2 - t1:.1f}s pack {t3 - t2:.1f}s accepted {len(acc)}", flush=True)
for k in (1, 16, 128, len(packs)):
    d = DeviceSimBatch(packs[:k])
    torch.cuda.synchronize()
    a = time.time()
    d.run()
    torch.cuda.synchronize()
    dt = time.time() - a
    h = d.to_host()
    print(f"{k} sims: {dt * 1e3:.1f} ms, events {int(h.n_events.sum())}, "
          f"{k / dt:.1f} sims/s, {h.n_events.sum() / dt / 1e6:.2f} M events/s, "
          f"status {set(h.status.tolist())}", flush=True)
