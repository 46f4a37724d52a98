"""The N>1 host path on CPU: world_size-2 gloo processes run the collective congruence check of
tc_plan_create through the same torch.distributed allgather callback tc.Comm uses."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, numels_per_rank, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1801_03855_b200 as tc
    try:
        plan = tc.Plan(numels_per_rank[rank], nranks=world, rank=rank, pg=dist.group.WORLD)
        q.put((rank, "ok", plan.num_slots, [plan.owner_range(r) for r in range(world)]))
    except tc.TcError as e:
        q.put((rank, "err", e.status, None))
    dist.destroy_process_group()


def _run(numels_per_rank, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, numels_per_rank, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def test_congruent_plans_agree():
    res = _run([[7, 13, 1000], [7, 13, 1000]])
    assert [r[1] for r in res] == ["ok", "ok"]
    assert res[0][2:] == res[1][2:]
    assert res[0][3] == [(0, 128), (128, 256)]


def test_shape_mismatch_reported_on_every_rank():
    res = _run([[7, 13, 1000], [7, 14, 1000]])
    import paper_1801_03855_b200 as tc
    assert [r[1:3] for r in res] == [("err", tc.tc.TC_ERR_SHAPE_MISMATCH)] * 2


def test_invalid_input_on_one_rank_fails_everywhere():
    res = _run([[7, 13], [7, -13]])
    assert all(r[1] == "err" for r in res)
