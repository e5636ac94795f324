"""Host side of the multi-GPU path on CPU: two gloo ranks (world_size 2,
127.0.0.1) share an NCCL clique id and agree on the z-slab plan.  The device
exchanges themselves are covered by tests/test_gpu_slabs.py (in-process
clique on one GPU, bit-identical to the single-GPU solve)."""
import os
import socket

import pytest
import torch.distributed as td
import torch.multiprocessing as mp

import paper_1703_07206_b200 as S
from paper_1703_07206_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    td.init_process_group("gloo", rank=rank, world_size=world)
    try:
        uid = D.share_unique_id(rank)
        ids = [None] * world
        td.all_gather_object(ids, uid)
        plans = [None] * world
        td.all_gather_object(plans, [S.slab_plan(n, world, rank) for n in (3, 5, 9, 10)])
        if rank == 0:
            out.put((ids, plans))
    finally:
        td.destroy_process_group()


def test_two_gloo_ranks_share_id_and_plan():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ids, plans = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert len(ids[0]) == 128 and ids[0] == ids[1]
    for k, n in enumerate((3, 5, 9, 10)):
        table = [plans[r][k] for r in range(2)]
        assert table == D.plan_table(n, 2)
        D.check_plan(n, 2)


@pytest.mark.parametrize("replicate_n", [0, 3])
@pytest.mark.parametrize("n,nranks", [(3, 4), (4, 8), (9, 2), (9, 8), (10, 8), (13, 4096)])
def test_slab_plans_tile_every_level(n, nranks, replicate_n):
    D.check_plan(n, nranks, replicate_n)


@pytest.mark.parametrize("n,nranks,rn,vrep", [
    (10, 8, 0, 4),   # 1025^3 on 8 ranks: levels 0..3 (1025..129) slabs, 65^3 and coarser replicated
    (10, 8, 3, 7),   # replicate only where a rank would hold < 2 planes
    (9, 2, 0, 3), (6, 2, 0, 0), (9, 8, 129, 2)])
def test_replicated_levels_start_at_65_nodes(n, nranks, rn, vrep):
    assert S.slab_plan(n, nranks, 0, rn)[0] == vrep
