#!/usr/bin/env python
"""Grid-size probe for the TMA two-shot on the ResNet-50 group (config 2).

    torchrun --nproc-per-node N tools/ctas_probe.py

For CTAs per rank in a list: tc_allreduce and the fused tc_sgd_step on the ResNet-50 gradient
group, each timed as a CUDA-graph replay with CUDA events (max over ranks, us).  The gradients
are not refreshed between calls (scale 1/p keeps their magnitude; timing only).  Rank 0 prints
one JSON line per grid size.
"""
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1801_03855_b200 as tc  # noqa: E402
import tc_workloads as W  # noqa: E402
from bench_sweep import timed  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, p = dist.get_rank(), dist.get_world_size()
    comm = tc.Comm.from_process_group(device=local)
    numels = W.RESNET50
    n = sum(numels)
    flat_g = torch.randn(n, device="cuda") * 1e-3
    flat_w = torch.randn(n, device="cuda") * 0.05
    flat_dw = torch.zeros(n, device="cuda")
    g = tc.Group(comm, list(torch.split(flat_g, numels)))
    w = tc.Group(comm, list(torch.split(flat_w, numels)))
    dw = tc.Group(comm, list(torch.split(flat_dw, numels)))
    s = torch.cuda.current_stream
    for ctas in (0, 64, 96, 112, 120, 128, 136, 144, 148):  # (one CTA per SM at most)
        comm.set_tuning(ctas, 0, -1)
        t_ar = timed(lambda: tc.allreduce(g, 1.0 / p, stream=s()), 20, graph=True)
        ar_algo = comm.last_launch()
        t_sgd = timed(lambda: tc.sgd_step(w, g, dw, 0.1, 0.9, 1e-4, 1.0 / p, stream=s()), 20,
                      graph=True)
        if rank == 0:
            print(json.dumps({"p": p, "ctas": ctas, "allreduce_us": round(t_ar, 1),
                              "sgd_step_us": round(t_sgd, 1), "launch": list(ar_algo)}),
                  flush=True)
    comm.set_tuning(0, 0, -1)
    for x in (g, w, dw):
        x.destroy()
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
