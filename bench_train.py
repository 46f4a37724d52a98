#!/usr/bin/env python
"""NEXT row f1 on a real backward pass: data-parallel ResNet-50 training steps whose gradient
allreduce + SGD-momentum update (libtc) overlaps the backward computation bucket by bucket.

    torchrun --nproc-per-node N bench_train.py [--batch 64] [--iters 20] [--bucket-mb 25]
                                               [--graph] [--channels-last] [--split] [--ctas K]
    where f1 pays: --graph --channels-last --batch 8 --ctas 48 --priority (p = 4)

PAPER.md:59: gradients "are obtained as soon as a backward step for a layer is computed, these can
be aggregated in parallel with the backward phase".  The model is torchvision's ResNet-50 (random
init, synthetic 224x224 images and labels; bf16 autocast, fp32 master weights and gradients).
Its 161 parameters are views of one flat weight buffer and its gradients views of one flat
gradient buffer, so libtc groups wrap the model's own tensors (no copies):
  serial   -- forward + backward, then one tc_sgd_step over the whole group;
  overlap  -- tc.BucketedStep: a post-accumulate-grad hook on every parameter reports its
              gradient ready; each bucket's fused allreduce + SGD launches on a side stream as
              soon as its last gradient lands (backward order), while the backward continues;
  compute  -- forward + backward alone (no step), the floor.
With --graph each mode's iteration is captured once as a CUDA graph (the bucket launches become
side-stream nodes hanging off the gradient-producing kernels) and replayed, so host launch cost
does not decide the comparison.  Per-iteration device time (CUDA events, max over ranks); hidden
fraction = (serial - overlap) / (serial - compute) per round, median over rounds.  After the timed iterations every rank's weights are compared (bitwise hash
allgather): the fused step keeps the replicas identical.  Rank 0 prints one JSON line per mode.
"""
import argparse
import hashlib
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
import paper_1801_03855_b200 as tc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--bucket-mb", type=float, default=25.0)
    ap.add_argument("--ctas", type=int, default=0, help="CTA budget of the bucket launches")
    ap.add_argument("--split", action="store_true",
                    help="buckets run the allreduce only; the update runs once at the end")
    ap.add_argument("--graph", action="store_true",
                    help="capture each mode's whole iteration in one CUDA graph and time replays "
                         "(no host launch cost; the bucket kernels hang off the graph's edges)")
    ap.add_argument("--rounds", type=int, default=5, help="interleaved timing rounds per mode")
    ap.add_argument("--threads", type=int, default=0,
                    help="threads per CTA of the NVLS allreduce (with --switch --split: small CTAs "
                         "that can sit beside the backward pass's CTAs)")
    ap.add_argument("--priority", action="store_true",
                    help="bucket launches on a highest-priority side stream")
    ap.add_argument("--switch", action="store_true",
                    help="gradients in symmetric memory and the bucket allreduces on the switch "
                         "(NVLS, algorithm 4: link-bound on ~32 SMs; tolerance contract)")
    ap.add_argument("--channels-last", action="store_true",
                    help="NHWC activations and conv weights (the fast cuDNN layout)")
    a = ap.parse_args()
    import torchvision

    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.manual_seed(1234)  # same initial weights on every rank
    model = torchvision.models.resnet50().cuda()
    cl = a.channels_last
    if cl:
        model = model.to(memory_format=torch.channels_last)
    params = list(model.parameters())
    numels = [p.numel() for p in params]
    N = sum(numels)
    # the weights and gradients as views of flat buffers (the layout libtc and DDP buckets use)
    comm = tc.Comm.single(local) if world == 1 else tc.Comm.from_process_group(device=local)
    w_flat = torch.empty(N, device="cuda")
    if a.switch and world > 1:
        g_flat = comm.alloc_symmetric(N)
        g_flat.zero_()
        comm.set_algorithm(4)
        comm.set_tuning(0, a.threads, -1)
    else:
        g_flat = torch.zeros(N, device="cuda")
    d_flat = torch.zeros(N, device="cuda")
    def as_param(flat, p):
        # a view of the flat slice with p's shape (NHWC strides for conv weights if --channels-last)
        if cl and p.dim() == 4:
            k, c, h, w = p.shape
            return flat.view(k, h, w, c).permute(0, 3, 1, 2)
        return flat.view_as(p)

    off = 0
    for p in params:
        n = p.numel()
        as_param(w_flat[off:off + n], p).copy_(p.data)
        p.data = as_param(w_flat[off:off + n], p)
        p.grad = as_param(g_flat[off:off + n], p)
        off += n
    wv = list(torch.split(w_flat, numels))
    gv = list(torch.split(g_flat, numels))
    dv = list(torch.split(d_flat, numels))
    W, G, D = tc.Group(comm, wv), tc.Group(comm, gv), tc.Group(comm, dv)
    hp = dict(lr=0.1, momentum=0.9, wd=1e-4, rescale=1.0 / (world * a.batch))
    step = tc.BucketedStep(comm, gv, wv, dv, bucket_bytes=int(a.bucket_mb * (1 << 20)),
                           ctas=a.ctas, split=a.split,
                           stream=torch.cuda.Stream(
                               priority=torch.cuda.Stream.priority_range()[1] if a.priority else 0))
    # a hook on every parameter: the bucket launches when its last gradient is counted (hooking
    # only the lowest-index tensor of each bucket is NOT safe -- autograd may accumulate a
    # layer's weight before its bias, so a bucket could launch before its last gradient lands;
    # measured: replicas diverged)
    index = {id(p): t for t, p in enumerate(params)}
    mode = {"hooks": False}

    def hook(p):
        if mode["hooks"]:
            step.grad_ready(index[id(p)], **hp)

    for p in params:
        p.register_post_accumulate_grad_hook(hook)
    x = torch.randn(a.batch, 3, 224, 224, device="cuda")
    if cl:
        x = x.contiguous(memory_format=torch.channels_last)
    y = torch.randint(0, 1000, (a.batch,), device="cuda")
    crit = torch.nn.CrossEntropyLoss()

    def fwd_bwd():
        g_flat.zero_()
        with torch.autocast("cuda", dtype=torch.bfloat16, cache_enabled=not a.graph):
            loss = crit(model(x), y)
        loss.backward()
        # gradients must land in the flat buffer (in-place accumulation), never a fresh tensor
        assert params[0].grad.data_ptr() == g_flat.data_ptr()

    def it_compute():
        fwd_bwd()

    def it_serial():
        fwd_bwd()
        tc.sgd_step(W, G, D, **hp)

    def it_overlap():
        mode["hooks"] = True
        fwd_bwd()
        step.finish()
        mode["hooks"] = False

    def graphed(fn):
        """fn captured once as a CUDA graph (after warm-up on a side stream); returns replay."""
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(3):
                fn()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            fn()
        torch.cuda.synchronize()
        graphs.append(gr)
        return gr.replay

    graphs = []

    def timed(fn):
        for _ in range(a.warmup):
            fn()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / a.iters * 1e3], device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t)

    wrap = graphed if a.graph else (lambda f: f)
    fns = {"compute": wrap(it_compute), "serial": wrap(it_serial), "overlap": wrap(it_overlap),
           "step": wrap(lambda: tc.sgd_step(W, G, D, **hp))}
    # the modes interleaved over --rounds rounds (clock and power drift hit every mode alike);
    # per mode the median of the rounds' per-iteration means
    runs = {k: [] for k in fns}
    for _ in range(a.rounds):
        for k, fn in fns.items():
            runs[k].append(timed(fn))
    med = {k: sorted(v)[len(v) // 2] for k, v in runs.items()}
    t_compute, t_serial, t_overlap, t_step = (med[k] for k in ("compute", "serial", "overlap", "step"))
    # replicas identical after every mode (the fused step applies the same G everywhere)
    dig = hashlib.sha256(w_flat.cpu().numpy().tobytes()).digest()
    h = torch.tensor([int.from_bytes(dig[:7], "little")], device="cuda")
    same = True
    if world > 1:
        hs = [torch.zeros_like(h) for _ in range(world)]
        dist.all_gather(hs, h)
        same = all(int(v) == int(hs[0]) for v in hs)
    if rank == 0:
        print(json.dumps({
            "bench": "resnet50 training step, f1 overlap (PAPER.md:59)", "n_gpus": world,
            "batch_per_gpu": a.batch, "bucket_mb": a.bucket_mb, "buckets": step.nbuckets,
            "ctas": a.ctas or "auto", "mode": "split" if a.split else "fused",
            "graph": a.graph, "channels_last": cl, "switch": a.switch, "threads": a.threads or 512,
            "algo": comm.last_launch()[0],
            "t_compute_us": t_compute, "t_serial_us": t_serial,
            "t_overlap_us": t_overlap, "t_step_alone_us": t_step,
            # per round (the modes of one round ran back to back, so clock / power drift between
            # rounds cancels), then the median over rounds
            "hidden_fraction": sorted(
                (s - o) / max(s - c, 1e-9) for c, s, o in
                zip(runs["compute"], runs["serial"], runs["overlap"]))[len(runs["compute"]) // 2],
            "hidden_fraction_of_medians": (t_serial - t_overlap) / max(t_serial - t_compute, 1e-9),
            "rounds": {k: [round(x, 1) for x in v] for k, v in runs.items()},
            "side_stream_priority": a.priority,
            "speedup_vs_serial": t_serial / t_overlap, "replicas_identical": same,
            "data": "synthetic images/labels, random-init torchvision ResNet-50, bf16 autocast"}),
            flush=True)
    graphs.clear()
    torch.cuda.synchronize()
    step.destroy()
    for grp in (W, G, D):
        grp.destroy()
    comm.destroy()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
