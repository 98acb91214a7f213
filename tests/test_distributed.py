"""The N>1 path on CPU: world-size-2 gloo processes run the sharded sweep
(each rank analyses its slice of every cell -- here with the oracle as the
analysis function, since this box has no GPU) and must reproduce the
single-process sweep and the reference's golden CSV after the all_reduce."""
import json
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from golden_io import GOLDEN_DIR


def oracle_status(blobs, set_off, task_base, method):
    from oracle import oracle
    return oracle.analyze_batch(blobs, set_off, task_base, method=method, flags=0, threads=2,
                                detail=False)["status"]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg_dict, out_path):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2101_10463_b200.distributed import sharded_sweep
    from paper_2101_10463_b200.workbench import sweep_config_from_dict, sweep_to_csv
    rows = sharded_sweep(sweep_config_from_dict(cfg_dict), rank, world, analyze=oracle_status)
    with open(f"{out_path}.{rank}", "w") as fh:
        fh.write(sweep_to_csv(rows))
    dist.destroy_process_group()


def test_shard_range_partitions():
    from paper_2101_10463_b200.distributed import shard_range
    for n in (0, 1, 7, 100, 101):
        for w in (1, 2, 3, 8):
            parts = [shard_range(n, r, w) for r in range(w)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(w - 1))


@pytest.mark.parametrize("which", [0, 1])
def test_gloo_world2_sweep_equals_reference(tmp_path, which):
    with open(os.path.join(GOLDEN_DIR, "sweep_golden.json")) as fh:
        golden = json.load(fh)["sweeps"][which]
    out = str(tmp_path / "sweep.csv")
    mp.spawn(_worker, args=(2, _free_port(), golden["config"], out), nprocs=2, join=True)
    for r in range(2):
        with open(f"{out}.{r}") as fh:
            assert fh.read() == golden["csv"]


def undecided_on_rank1(blobs, set_off, task_base, method):
    import torch.distributed as dist
    st = oracle_status(blobs, set_off, task_base, method)
    if dist.get_rank() == 1:
        st = st.copy()
        st[0] = 2  # RTGPU_UNDECIDED
    return st


def _worker_fail(rank, world, port, cfg_dict, out_path):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2101_10463_b200.distributed import sharded_sweep
    from paper_2101_10463_b200.workbench import sweep_config_from_dict
    try:
        sharded_sweep(sweep_config_from_dict(cfg_dict), rank, world, analyze=undecided_on_rank1)
        msg = "no error"
    except RuntimeError as exc:
        msg = str(exc)
    with open(f"{out_path}.{rank}", "w") as fh:
        fh.write(msg)
    dist.destroy_process_group()


def test_gloo_world2_undecided_raises_on_every_rank(tmp_path):
    """An undecided set on one rank is reduced with the counts: every rank
    raises after the collective, none is left waiting in all_reduce."""
    with open(os.path.join(GOLDEN_DIR, "sweep_golden.json")) as fh:
        golden = json.load(fh)["sweeps"][0]
    out = str(tmp_path / "fail")
    mp.spawn(_worker_fail, args=(2, _free_port(), golden["config"], out), nprocs=2, join=True)
    for r in range(2):
        with open(f"{out}.{r}") as fh:
            assert "undecided task sets" in fh.read()
