"""The N > 1 bench plumbing (replicas; paper_2401_00228_b200/dist.py) with
world_size 2 over gloo on CPU."""

import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import numpy as np

    from paper_2401_00228_b200 import dist
    from tests.cases import BASELINE

    dist.init("gloo")
    r, w, lr = dist.rank_info()
    case = BASELINE["c3"].scaled(seed=dist.instance_seed(0, r))
    u0 = case.u0_vector()
    # each rank "times" a different amount; everyone must see the max
    t = dist.max_over_ranks(10.0 + r)
    dist.barrier()
    out[rank] = (r, w, lr, t, float(np.sum(u0)))
    import torch.distributed as tdist

    tdist.destroy_process_group()


def test_replicas_max_over_ranks_gloo():
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
        res = dict(out)
    assert sorted(res) == [0, 1]
    assert res[0][:3] == (0, 2, 0) and res[1][:3] == (1, 2, 1)
    assert res[0][3] == res[1][3] == 11.0          # max over ranks
    assert res[0][4] != res[1][4]                 # independent seeded instances


def test_single_process_identity():
    from paper_2401_00228_b200 import dist

    assert dist.max_over_ranks(3.5) == 3.5
    assert dist.instance_seed(7, 0) == 7
