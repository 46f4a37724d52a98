"""Multi-process stress of the epoch / staging-parity bookkeeping (diagnostics).

    torchrun --nproc-per-node N tools/stress_mp.py [iters]     (N a power of two: 1/N exact)

Every rank holds an integer-valued group (in symmetric memory, so NVLS can run too).  Every call
changes the data: before call i each rank adds d_r = 2k(r + 1) (k = 1 + i mod 7) to every element,
then
  * allreduce(scale 1/p):   x := x + k(p + 1)          (the mean of the d_r, exact in fp32)
  * broadcast(root q):      x := x + 2k(q + 1)         (every rank takes the root's copy)
so a call that did nothing, ran twice, read a stale stage or mixed epochs leaves a wrong value.
The algorithm rotates (automatic / register pull / TMA two-shot / NVLS / one-shot / LL) and every
call is checked against the running reference on the GPU."""
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
    n = sum(numels)
    flat = comm.alloc_symmetric(n)
    flat.copy_(torch.from_numpy(np.concatenate(W.group(numels, "int", 90, 0, rank, W.GRAD))))
    views = list(torch.split(flat, numels))
    g = tc.Group(comm, views)
    tc.allreduce(g, 1.0 / p)  # a common (exact) starting point: integers, then their mean
    ref = flat.clone()
    settings = [(0, -1, -1), (1, 0, 0), (6, 0, 0), (0, 1 << 30, 0), (0, 0, 1 << 30)]
    if comm.multicast_supported:
        settings.append((4, 0, 0))
    bad, counts = 0, {}
    for i in range(iters):
        a, oneshot, ll = settings[i % len(settings)]
        comm.set_algorithm(a)
        comm.set_tuning(0, 0, oneshot)
        comm.set_ll_max(ll)
        k = 1 + i % 7
        flat.add_(2.0 * k * (rank + 1))
        if i % 5 == 4:
            q = i % p
            tc.broadcast(g, q)
            ref.add_(2.0 * k * (q + 1))
        else:
            tc.allreduce(g, 1.0 / p)
            ref.add_(float(k * (p + 1)))
        name = comm.last_launch()[0]
        counts[name] = counts.get(name, 0) + 1
        if not torch.equal(flat, ref):
            bad += 1
            flat.copy_(ref)
    torch.cuda.synchronize()
    err = comm.async_error()
    t = torch.tensor([bad, err], dtype=torch.int64)
    dist.all_reduce(t)
    if rank == 0:
        print(f"stress p={p} iters={iters}: mismatching calls {int(t[0])}, async errors "
              f"{int(t[1])}, launches per algorithm {counts}", flush=True)
    g.destroy()
    comm.free_symmetric(flat)
    comm.destroy()
    dist.destroy_process_group()
    assert int(t[0]) == 0 and int(t[1]) == 0


if __name__ == "__main__":
    main()
