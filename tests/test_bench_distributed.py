"""bench.py's N>1 path on CPU: world-size-2 gloo processes run the same
sharding (cell_indices), histogram all_reduce (status_hist) and max-over-
ranks timing (max_over_ranks) that the NCCL bench runs use, with the oracle
as the analysis.  A fixed workload split across ranks (strong scaling,
BASELINE configs[2]'s protocol) must reproduce the single-process histogram."""
import os
import socket
import sys
from fractions import Fraction

import numpy as np
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WL_STRONG = dict(n=4, ms=[2, 3], gn=10, utils=[Fraction(1, 2), Fraction(9, 10)], per_cell=40, strong=True,
                 desc="test")
WL_WEAK = dict(WL_STRONG, strong=False, per_cell=20)


def oracle_status(blobs, set_off, task_base):
    from oracle import oracle
    return oracle.analyze_batch(blobs, set_off, task_base, method=0, flags=0x100, threads=2,
                                detail=False)["status"]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_path):
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    hs = bench.sweep_histogram(WL_STRONG, 7, rank, world, oracle_status).numpy()
    hw = bench.sweep_histogram(WL_WEAK, 7, rank, world, oracle_status).numpy()
    mx = bench.max_over_ranks(float(rank + 1), world)
    np.savez(f"{out_path}.{rank}.npz", strong=hs, weak=hw, mx=mx,
             idx=np.asarray(bench.cell_indices(WL_STRONG, rank, world)))
    dist.destroy_process_group()


def test_bench_world2_gloo_matches_single_process(tmp_path):
    sys.path.insert(0, ROOT)
    import bench
    single = bench.sweep_histogram(WL_STRONG, 7, 0, 1, oracle_status).numpy()
    out = str(tmp_path / "h")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    r = [np.load(f"{out}.{k}.npz") for k in range(2)]
    # every rank holds the global histogram; the fixed workload's equals the single-GPU one
    for k in range(2):
        assert np.array_equal(r[k]["strong"], single)
        assert np.array_equal(r[k]["weak"], r[0]["weak"])
        assert float(r[k]["mx"]) == 2.0
    ncell = len(WL_STRONG["ms"]) * len(WL_STRONG["utils"])
    assert r[0]["weak"].sum() == 2 * WL_WEAK["per_cell"] * ncell  # weak: fresh sets per rank
    # the strong shards partition the cell
    assert sorted(list(r[0]["idx"]) + list(r[1]["idx"])) == list(range(WL_STRONG["per_cell"]))
