"""N > 1 host logic of bench.py on CPU: world_size 2 over gloo.

The product path shards the batch across ranks with no data-path collective; the only
cross-rank operations are the timing barrier and the max-over-ranks reduction.  This checks
that each rank draws different instances of the same configuration, that the reduction
returns the slowest rank's time on every rank, and the whole-job throughput formula.
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    import synth
    cfg = {k: v for k, v in synth.CONFIGS["C1"].items() if k != "kind"}
    inp = synth.matvec_inputs(**bench.rank_config(cfg, rank))
    ms_local = 10.0 + 5.0 * rank
    ms_max = bench.max_over_ranks(ms_local, world, device="cpu")
    dist.barrier()
    out[rank] = (ms_max, int(inp["a"][0, :8].sum()), int(inp["f"]), bench.whole_job_gelems(world, 1, 1024, 4, ms_max))
    dist.destroy_process_group()


def test_two_ranks_gloo():
    world = 2
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
        res = dict(out)
    assert res[0][0] == res[1][0] == 15.0          # slowest rank on every rank
    assert res[0][1] != res[1][1] or res[0][2] != res[1][2]   # independent instances per rank
    assert res[0][3] == pytest.approx(2 * 1024 * 4 / 15e-3 / 1e9)


def test_single_rank_no_collective():
    import bench
    assert bench.max_over_ranks(3.5, 1) == 3.5
    assert bench.whole_job_gelems(1, 64, 1 << 20, 10, 5.0) == pytest.approx(64 * (1 << 20) * 10 / 5e-3 / 1e9)
