"""Multi-process stress of the epoch / staging-parity bookkeeping (diagnostics).

    torchrun --nproc-per-node N tools/stress_mp.py [iters]

Every rank starts from its own integer-valued group; the first tc_allreduce(scale 1/p) leaves
the exact mean on every rank, and every later call must reproduce it bit for bit, whatever the
algorithm (rotating auto / pull / push / TMA / claimed / one-shot / LL) and interleaved with
broadcasts (which must also leave the mean).  Checked on the GPU every call."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1801_03855_b200 as tc  # noqa: E402
import tc_workloads as W  # noqa: E402


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 400
    dist.init_process_group("gloo")
    rank, p = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    comm = tc.Comm.from_process_group(device=local)
    numels = [7, 13, 1000, 0, 50001, 3, 262144, 2048, 4099]
    flat = torch.from_numpy(np.concatenate(W.group(numels, "int", 90, 0, rank, W.GRAD))).cuda()
    views = list(torch.split(flat, numels))
    g = tc.Group(comm, views)
    tc.allreduce(g, 1.0 / p)
    ref = flat.clone()
    settings = [(0, -1, -1), (1, 0, 0), (3, 0, 0), (6, 0, 0), (7, 0, 0), (0, 1 << 30, 0),
                (0, 0, 1 << 30)]
    bad = 0
    for i in range(iters):
        a, oneshot, ll = settings[i % len(settings)]
        comm.set_algorithm(a)
        comm.set_tuning(0, 0, oneshot)
        comm.set_ll_max(ll)
        if i % 5 == 4:
            tc.broadcast(g, i % p)
        else:
            tc.allreduce(g, 1.0 / p)
        if not torch.equal(flat, ref):
            bad += 1
    torch.cuda.synchronize()
    err = comm.async_error()
    t = torch.tensor([bad, err], dtype=torch.int64)
    dist.all_reduce(t)
    if rank == 0:
        print(f"stress p={p} iters={iters}: mismatching calls {int(t[0])}, async errors {int(t[1])}",
              flush=True)
    g.destroy()
    comm.destroy()
    dist.destroy_process_group()
    assert int(t[0]) == 0 and int(t[1]) == 0


if __name__ == "__main__":
    main()
