"""Can NVLS (switch reduction) and P2P two-shot traffic run side by side and add up?

    torchrun --nproc-per-node N tools/concurrent_probe.py

Splits the ResNet-50 gradient group at fraction f: the first part lives in symmetric memory and
is reduced with NVLS on comm A / stream A, the rest with the two-shot P2P algorithm on comm B /
stream B, both launched back to back (each kernel limited to 148 CTAs so both are resident).
Prints the combined time (max over ranks) and the BASELINE bus bandwidth for each f.
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


def main():
    dist.init_process_group("gloo")
    rank, p = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    numels = W.RESNET50
    N = sum(numels)
    S = 4 * N
    ca = tc.Comm.from_process_group(device=local)
    cb = tc.Comm.from_process_group(device=local)
    sym = ca.alloc_symmetric(N)
    plain = torch.randn(N, device="cuda")
    sym.copy_(torch.randn(N, device="cuda"))
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    K = 30
    for f in [0.0, 0.5, 0.6, 0.7, 0.8, 0.9, 1.0]:
        na = int(N * f) // 4 * 4
        ga = tc.Group(ca, [sym[:na]]) if na else None
        gb = tc.Group(cb, [plain[na:]]) if na < N else None
        ca.set_algorithm(4)
        cb.set_algorithm(1)
        ctas = 148 if (ga and gb) else 0
        ca.set_tuning(ctas, 0, 0)
        cb.set_tuning(ctas, 0, 0)

        def run():
            if ga:
                tc.allreduce(ga, 1.0 / p, stream=sa)
            if gb:
                tc.allreduce(gb, 1.0 / p, stream=sb)
        for _ in range(5):
            run()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.current_stream().record_event(e0)
        sa.wait_event(e0)
        sb.wait_event(e0)
        for _ in range(K):
            run()
        ea, eb = torch.cuda.Event(), torch.cuda.Event()
        sa.record_event(ea)
        sb.record_event(eb)
        torch.cuda.current_stream().wait_event(ea)
        torch.cuda.current_stream().wait_event(eb)
        torch.cuda.current_stream().record_event(e1)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / K])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_us = float(t) * 1e3
        if rank == 0:
            print(f"f={f:.1f}  t={t_us:7.1f} us  busbw={S * 2 * (p - 1) / p / t_us / 1e3:6.1f} GB/s "
                  f"algos={ca.last_launch()[0] if ga else '-'}/{cb.last_launch()[0] if gb else '-'}",
                  flush=True)
        for g in (ga, gb):
            if g:
                g.destroy()
    ca.free_symmetric(sym)
    ca.destroy()
    cb.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
