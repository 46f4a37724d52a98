#!/usr/bin/env python
"""NEXT row f1: the fused SGD step overlapped with a (synthetic) backward pass, bucket by bucket.

    torchrun --nproc-per-node N bench_overlap.py [--ratio 1.0] [--bucket-mb 25]

PAPER.md:59: gradients "are obtained as soon as a backward step for a layer is computed, these
can be aggregated in parallel with the backward phase".  The backward pass is synthetic: bucket by
bucket, last layers first, a compute burst sized so the whole pass takes `ratio` x the time of one
whole-group tc_sgd_step, then the bucket's gradients are written.  The burst is either
  --compute burn: a compute-bound FMA kernel of many small CTAs (4 x 256 threads per SM, no
                  shared memory), compiled with NVRTC -- the SURVEY's "synthetic compute kernel";
  --compute gemm: cuBLAS bf16 GEMMs.  These are persistent kernels that want every SM: while the
                  collective holds some SMs the GEMM's remaining CTAs start only when it ends, so
                  the two serialise instead of overlapping (reported as measured).
Three runs:
  compute  -- the backward pass alone;
  serial   -- backward, then one tc_sgd_step over the whole group;
  overlap  -- tc.BucketedStep: each bucket's collective on a side stream once its last gradient
              is written, limited to `ctas` CTAs so the computation keeps SMs.  fused: each
              bucket runs tc_sgd_step (allreduce + update, 6S of HBM traffic through the
              collective's SMs); split: each bucket runs tc_allreduce (link-bound) and the
              update runs once at the end as a full-GPU HBM stream.
Rank 0 prints one JSON line per configuration with the fraction of the step hidden.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
import paper_1801_03855_b200 as tc  # noqa: E402
import tc_workloads as W  # noqa: E402


def timed(fn, iters, world):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / iters], device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t) * 1e3


BURN_SRC = r"""
extern "C" __global__ void burn(float* out, int iters) {
  float a = threadIdx.x * 1e-3f, b = 1.0001f, c = 0.9999f;
  for (int i = 0; i < iters; ++i) {
    a = a * b + c;
    b = b * c - a * 1e-9f;
  }
  if (a == 12345.f) out[0] = b;
}
"""


class Burn:
    """A compute-bound kernel (FMA chains) launched on torch's current stream via NVRTC."""

    def __init__(self, device):
        from cuda.bindings import driver as cu, nvrtc
        self.cu = cu
        major, minor = torch.cuda.get_device_capability(device)
        err, prog = nvrtc.nvrtcCreateProgram(BURN_SRC.encode(), b"burn.cu", 0, [], [])
        opts = [f"--gpu-architecture=sm_{major}{minor}{'a' if major >= 9 else ''}".encode()]
        (err,) = nvrtc.nvrtcCompileProgram(prog, len(opts), opts)
        if err != nvrtc.nvrtcResult.NVRTC_SUCCESS:
            _, n = nvrtc.nvrtcGetProgramLogSize(prog)
            log = b" " * n
            nvrtc.nvrtcGetProgramLog(prog, log)
            raise RuntimeError(log.decode())
        _, n = nvrtc.nvrtcGetCUBINSize(prog)
        cubin = b" " * n
        nvrtc.nvrtcGetCUBIN(prog, cubin)
        cu.cuInit(0)
        torch.cuda.synchronize()
        err, self.mod = cu.cuModuleLoadData(cubin)
        assert err == cu.CUresult.CUDA_SUCCESS, err
        err, self.fn = cu.cuModuleGetFunction(self.mod, b"burn")
        assert err == cu.CUresult.CUDA_SUCCESS, err
        self.out = torch.zeros(1, device="cuda")
        self.grid = 4 * torch.cuda.get_device_properties(device).multi_processor_count

    def __call__(self, iters):
        import ctypes
        cu = self.cu
        a0 = ctypes.c_void_p(self.out.data_ptr())
        a1 = ctypes.c_int(int(iters))
        args = (ctypes.c_void_p * 2)(ctypes.addressof(a0), ctypes.addressof(a1))
        st = torch.cuda.current_stream().cuda_stream
        (err,) = cu.cuLaunchKernel(self.fn, self.grid, 1, 1, 256, 1, 1, 0, st,
                                   ctypes.addressof(args), 0)
        assert err == cu.CUresult.CUDA_SUCCESS, err


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ratio", type=float, default=1.0)
    ap.add_argument("--compute", default="gemm", choices=["burn", "gemm"])
    ap.add_argument("--carveout", action="store_true",
                    help="GEMM mode: leave the collective's CTAs free via cuBLASLt's SM carveout")
    ap.add_argument("--bucket-mb", type=float, default=64.0)
    ap.add_argument("--algo", type=int, default=0,
                    help="collective algorithm (1: register pull, no shared memory -- its CTAs "
                         "can sit on an SM beside a GEMM CTA)")
    ap.add_argument("--threads", type=int, default=0, help="threads per CTA (register kernels)")
    ap.add_argument("--shapes", default="", help="ctas list for the overlap runs, e.g. 148,296")
    ap.add_argument("--priority", action="store_true",
                    help="the collective's side stream at the highest stream priority")
    ap.add_argument("--green", type=int, default=0,
                    help="run the backward pass in a CUDA green context of (SMs - GREEN) SMs, so "
                         "GREEN SMs stay free for the collective (budget GREEN CTAs)")
    ap.add_argument("--sym", action="store_true",
                    help="gradients in symmetric (multicast) memory, so --algo 4 (NVLS: the "
                         "switch reduces; link-bound on ~32 SMs) can run the buckets")
    ap.add_argument("--iters", type=int, default=10)
    a = ap.parse_args()
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    numels = W.RESNET50
    N = sum(numels)

    def flat(kind, role):
        f = torch.from_numpy(np.concatenate(W.group(numels, kind, W.CFG_RESNET50, 0, rank, role)))
        f = f.cuda()
        return f, list(torch.split(f, numels))

    gp_flat, gp = flat("grad", W.GRAD)
    g_flat, g = flat("grad", W.GRAD)
    w_flat, w = flat("param", W.PARAM)
    d_flat, dw = flat("dw", W.DW)
    comm = tc.Comm.single(local) if world == 1 else tc.Comm.from_process_group(device=local)
    if a.sym and world > 1:
        g_flat = comm.alloc_symmetric(N)
        g_flat.copy_(gp_flat)
        g = list(torch.split(g_flat, numels))
    hp = dict(lr=0.1, momentum=0.9, wd=1e-4, rescale=1.0 / (world * 128))
    G, Wg, D = tc.Group(comm, g), tc.Group(comm, w), tc.Group(comm, dw)

    def whole_step():
        tc.sgd_step(Wg, G, D, **hp)

    comm.set_tuning(0, a.threads, -1)
    t_step = timed(lambda: (g_flat.copy_(gp_flat), whole_step()), a.iters, world) - \
        timed(lambda: g_flat.copy_(gp_flat), a.iters, world)
    bucket_of, nb = tc.Plan(numels).buckets(int(a.bucket_mb * (1 << 20)))
    members = [[t for t in range(len(numels)) if bucket_of[t] == k] for k in range(nb)]
    offs = np.concatenate([[0], np.cumsum(numels)])
    spans = [(int(offs[m[0]]), int(offs[m[-1] + 1])) for m in members]
    if a.compute == "gemm":
        # cuBLASLt honours the SM carveout (torch._C._set_sm_carveout_experimental)
        torch.backends.cuda.preferred_blas_library("cublaslt")
        A = torch.randn(2048, 2048, device="cuda", dtype=torch.bfloat16)
        B = torch.randn(2048, 2048, device="cuda", dtype=torch.bfloat16)
        C = torch.empty_like(A)
        t_unit = timed(lambda: torch.mm(A, B, out=C), 50, world)
        total = max(1, int(round(a.ratio * t_step / t_unit)))
        per = [max(1, int(round(total * (hi - lo) / N))) for lo, hi in spans]

        def burst(k):
            for _ in range(per[k]):
                torch.mm(A, B, out=C)
        units = sum(per)
    else:
        burn = Burn(local)
        t_unit = timed(lambda: burn(10000), 20, world) / 10000  # us per iteration
        total = a.ratio * t_step / t_unit
        per = [max(100, int(round(total * (hi - lo) / N))) for lo, hi in spans]

        def burst(k):
            burn(per[k])
        units = sum(per)

    # The synthetic backward works bucket by bucket (few launches, so the host is not the
    # bottleneck): a compute burst proportional to the bucket's bytes, then one copy writing the
    # bucket's gradients (contiguous views of the flat gradient buffer), last layers first.

    gctx, gstream, cctx, cstream = None, None, None, None
    if a.green:
        # green contexts: the backward pass on (SMs - GREEN) SMs, the collective's launches on the
        # other GREEN SMs (kernels of the primary context and of a green context time-slice, so
        # both sides get one)
        from torch.cuda.green_contexts import GreenContext
        sms = torch.cuda.get_device_properties(local).multi_processor_count

        def green(n):
            ctx = GreenContext.create(n, local)
            ctx.set_context()
            s = ctx.Stream()
            ctx.pop_context()
            s = s if isinstance(s, torch.cuda.Stream) else torch.cuda.Stream(
                stream_id=s.stream_id, device_index=s.device_index, device_type=s.device_type)
            return ctx, s
        gctx, gstream = green(sms - a.green)
        cctx, cstream = green(a.green)

    def backward(after=None):
        if gstream is None:
            for k in range(nb):
                burst(k)
                lo, hi = spans[k]
                g_flat[lo:hi].copy_(gp_flat[lo:hi])
                if after:
                    for t in reversed(members[k]):
                        after(t)
            return
        # --green: the GEMMs and gradient writes on the green stream; the caller's stream waits
        cur = torch.cuda.current_stream()
        gstream.wait_stream(cur)
        gctx.set_context()
        try:
            with torch.cuda.stream(gstream):
                for k in range(nb):
                    burst(k)
                    lo, hi = spans[k]
                    g_flat[lo:hi].copy_(gp_flat[lo:hi])
                    if after:
                        for t in reversed(members[k]):
                            after(t)
        finally:
            gctx.pop_context()
            cur.wait_stream(gstream)

    t_compute = timed(backward, a.iters, world)
    t_serial = timed(lambda: (backward(), whole_step()), a.iters, world)
    rows = []
    comm.set_algorithm(a.algo)
    shapes = (((False, a.green), (True, a.green)) if a.green else
              tuple((sp, int(c)) for sp in (False, True) for c in a.shapes.split(",")) if a.shapes
              else ((False, 0), (False, 64), (False, 32), (True, 0), (True, 64), (True, 32)))
    for split, ctas in shapes:
        side = cstream
        if side is None:  # explicit either way (BucketedStep's default is the highest priority)
            lo, hi = torch.cuda.Stream.priority_range()
            side = torch.cuda.Stream(priority=hi if a.priority else lo)
        step = tc.BucketedStep(comm, g, w, dw, bucket_bytes=int(a.bucket_mb * (1 << 20)), ctas=ctas,
                               split=split, stream=side)
        # GEMM mode: cuBLAS leaves `ctas` SMs to the collective (SM carveout), as a framework
        # overlapping communication with persistent GEMMs does
        carve = ctas if (a.compute == "gemm" and ctas and a.carveout) else None
        torch._C._set_sm_carveout_experimental(carve)

        def ready(t):
            if cctx is None:
                return step.grad_ready(t, **hp)
            cs = torch.cuda.current_stream()
            cctx.set_context()  # the bucket's launch goes to the collective's green context
            try:
                step.grad_ready(t, cs, **hp)
            finally:
                cctx.pop_context()

        def overlapped():
            backward(ready)
            step.finish()

        t_comp_c = timed(backward, a.iters, world) if carve else t_compute
        t_over = timed(overlapped, a.iters, world)
        torch._C._set_sm_carveout_experimental(None)
        comm.set_tuning(0, a.threads, -1)
        rows.append({"bench": "overlap (NEXT row f1)", "n_gpus": world, "ctas": ctas or "auto",
                     "algo": step.comm.last_launch()[0], "threads": a.threads or None,
                     "mode": "split" if split else "fused",
                     "buckets": step.nbuckets, "bucket_mb": a.bucket_mb,
                     "ratio": a.ratio, "compute": a.compute, "compute_units": units,
                     "sm_carveout": carve, "green_context_sms_reserved": a.green or None,
                     "side_stream_priority": bool(a.priority), "grad_memory_symmetric": a.sym,
                     "t_step_us": t_step, "t_compute_us": t_compute,
                     "t_compute_carveout_us": t_comp_c, "t_serial_us": t_serial,
                     "t_overlap_us": t_over,
                     "hidden_fraction": (t_serial - t_over) / max(t_serial - t_compute, 1e-9),
                     "speedup_vs_serial": t_serial / t_over})
        step.destroy()
    if rank == 0:
        for r in rows:
            print(json.dumps(r), flush=True)
    for grp in (G, Wg, D):
        grp.destroy()
    comm.destroy()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
