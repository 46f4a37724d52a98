"""Does a collective kernel run beside computation?  (diagnostics for NEXT row f1)

    torchrun --nproc-per-node N tools/overlap_probe.py
    env: GEMM_ONLY=1, NO_CARVEOUT=1, SYM=1 (gradients in tc_mem_alloc memory), ALGO=4 (NVLS),
         THREADS=128 (NVLS allreduce block size), CTAS=148,296, PRIO=1 (side stream priority)

Times, max over ranks: a compute burst alone (FMA kernel, or cuBLAS GEMMs with an SM carveout
equal to the collective's CTAs), tc_allreduce of the ResNet-50 group alone with C CTAs, and both
launched together on two streams.  Ideal overlap: both = max(compute, allreduce).
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1801_03855_b200 as tc  # noqa: E402
import tc_workloads as W  # noqa: E402
from bench_overlap import Burn, timed  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    numels = W.RESNET50
    g = torch.from_numpy(np.concatenate(W.group(numels, "grad", 2, 0, rank, W.GRAD))).cuda()
    comm = tc.Comm.from_process_group(device=local)
    if os.environ.get("SYM"):
        gs = comm.alloc_symmetric(g.numel())
        gs.copy_(g)
        g = gs
    views = list(torch.split(g, numels))
    comm.set_algorithm(int(os.environ.get("ALGO", "0")))
    thr = int(os.environ.get("THREADS", "0"))
    G = tc.Group(comm, views)
    side = (torch.cuda.Stream(priority=torch.cuda.Stream.priority_range()[1])
            if os.environ.get("PRIO") else torch.cuda.Stream())
    burn = Burn(local)
    torch.backends.cuda.preferred_blas_library("cublaslt")
    A = torch.randn(2048, 2048, device="cuda", dtype=torch.bfloat16)
    B = torch.randn(2048, 2048, device="cuda", dtype=torch.bfloat16)
    Cm = torch.empty_like(A)
    for kind in (("gemm",) if os.environ.get("GEMM_ONLY") else ("burn", "gemm")):
        for ctas in [int(c) for c in os.environ.get("CTAS", "16,32,64,0").split(",")]:
            comm.set_tuning(ctas, thr, -1)
            carve = ctas if (kind == "gemm" and ctas and not os.environ.get("NO_CARVEOUT")) else None
            torch._C._set_sm_carveout_experimental(carve)

            def compute():
                if kind == "burn":
                    burn(60000)
                else:
                    for _ in range(12):
                        torch.mm(A, B, out=Cm)

            def ar():
                tc.allreduce(G, 1.0 / world)

            def both():
                ev = torch.cuda.Event()
                ev.record()
                side.wait_event(ev)
                with torch.cuda.stream(side):
                    tc.allreduce(G, 1.0 / world, stream=side)
                compute()
                ev2 = torch.cuda.Event()
                ev2.record(side)
                torch.cuda.current_stream().wait_event(ev2)

            tcomp, tar, tboth = timed(compute, 10, world), timed(ar, 10, world), timed(both, 10, world)
            torch._C._set_sm_carveout_experimental(None)
            if rank == 0:
                print(f"p={world} {kind:4s} algo={comm.last_launch()} ctas={ctas or 'auto':>4} "
                      f"compute {tcomp:7.1f} us  "
                      f"allreduce {tar:7.1f} us  both {tboth:7.1f} us  "
                      f"(ideal {max(tcomp, tar):7.1f}, serial {tcomp + tar:7.1f})", flush=True)
    G.destroy()
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
