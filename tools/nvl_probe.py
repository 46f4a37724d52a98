"""NVLink / NVSwitch data-path ceilings on 2-8 B200s (design evidence, not product code).

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tools/nvl_probe.py

Every rank holds a symmetric buffer of S bytes (torch symmetric memory: peer pointers and the
NVSwitch multicast address).  Measured per case, CUDA events, max over ranks, all ranks at once:
  * NVLS allreduce of the owner ranges (multimem.ld_reduce + multimem.st) -- per-GPU link bytes
    (1 + 1/p) S; and its two halves alone
  * copy engines, all peers at once: each rank pulls (or pushes) S/p from/to every peer with one
    cudaMemcpyAsync per peer on its own stream -- per-GPU ingress (p-1)/p S
  * TMA bulk stores into every peer, TMA bulk loads from every peer, SM 16-B stores to every peer
Prints one JSON line per case: GB/s per GPU per direction of the link bytes the case moves.
"""
import ctypes
import json
import os
import subprocess
import sys

import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "tools", "bin", "libnvl_probe.so")


def build():
    os.makedirs(os.path.dirname(SO), exist_ok=True)
    src = os.path.join(ROOT, "tools", "nvl_probe.cu")
    if not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(src):
        subprocess.check_call(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a",
                               "-shared", "-Xcompiler", "-fPIC", "-o", SO, src])


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if rank == 0:
        build()
    dist.barrier()
    lib = ctypes.CDLL(SO)
    p = world
    S = int(os.environ.get("PROBE_MB", "102")) << 20
    S -= S % (16 * p * 65536)
    n = S // 4
    try:
        symm.enable_symm_mem_for_group(dist.group.WORLD.group_name)
    except Exception:  # noqa: BLE001 -- not needed on newer torch
        pass
    buf = symm.empty(n, dtype=torch.float32, device=f"cuda:{local}")
    hdl = symm.rendezvous(buf, dist.group.WORLD.group_name)
    mc = hdl.multicast_ptr
    peers = [hdl.buffer_ptrs[q] for q in range(p) if q != rank]
    local_buf = torch.empty(n, dtype=torch.float32, device="cuda")
    buf.fill_(1.0)
    stream = torch.cuda.Stream()
    K = int(os.environ.get("PROBE_ITERS", "20"))

    def timed(fn):
        with torch.cuda.stream(stream):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(K):
                fn()
            e1.record(stream)
            torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / K / 1e3], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def report(case, link_bytes, t, **kw):
        if rank == 0:
            print(json.dumps(dict(case=case, p=p, S_MB=S / 2**20, t_us=t * 1e6,
                                  gbs_per_dir=link_bytes / t / 1e9, **kw)), flush=True)

    S4 = n // 4  # 16-B slots
    lo, hi = S4 * rank // p, S4 * (rank + 1) // p
    sp = ctypes.c_void_p
    st = lambda: sp(stream.cuda_stream)  # noqa: E731
    if mc:
        for weak in (0, 1):
            for ctas in (32, 74, 148, 296):
                for threads in (256, 512, 1024):
                    for unroll in (1, 2, 4, 8):
                        if threads == 1024 and unroll == 8:
                            continue
                        f = lambda: lib.probe_mm(0, sp(mc), sp(local_buf.data_ptr()),  # noqa
                                                 ctypes.c_long(lo), ctypes.c_long(hi), ctas,
                                                 threads, unroll, weak, st())
                        t = timed(f)
                        report("nvls_allreduce", (1 + 1 / p) * S, t, ctas=ctas, threads=threads,
                               unroll=unroll, weak=weak)
        for mode, name in ((1, "nvls_ld_reduce_only"), (2, "nvls_st_only")):
            for ctas in (74, 148, 296):
                for unroll in (2, 4, 8):
                    f = lambda: lib.probe_mm(mode, sp(mc), sp(local_buf.data_ptr()),  # noqa
                                             ctypes.c_long(lo), ctypes.c_long(hi), ctas, 512,
                                             unroll, 1, st())
                    t = timed(f)
                    # ld_reduce: the switch reads S/p from every GPU (egress S/p each) and the
                    # owner receives S/p; st: the owner sends S/p, every GPU receives S/p
                    report(name, S / p, t, ctas=ctas, threads=512, unroll=unroll,
                           note="bytes = S/p per GPU per direction")
    else:
        report("nvls", 0, 1, note="multicast unavailable")

    # copy engines: all peers at once, one stream per peer
    streams = [torch.cuda.Stream() for _ in range(p)]
    chunk = n // p
    views = {q: hdl.get_buffer(q, (n,), torch.float32) for q in range(p)}
    for mode in ("pull", "push"):
        def ce():
            cur = torch.cuda.current_stream()
            for j, q in enumerate(x for x in range(p) if x != rank):
                s = streams[j]
                s.wait_stream(cur)
                with torch.cuda.stream(s):
                    if mode == "pull":   # my chunk of q's buffer into my local buffer
                        local_buf[q * chunk:(q + 1) * chunk].copy_(
                            views[q][rank * chunk:(rank + 1) * chunk], non_blocking=True)
                    else:                # my rank's chunk into q's buffer region
                        views[q][rank * chunk:(rank + 1) * chunk].copy_(
                            local_buf[q * chunk:(q + 1) * chunk], non_blocking=True)
            for j in range(p - 1):
                cur.wait_stream(streams[j])
        t = timed(ce)
        report(f"copy_engine_allpeer_{mode}", (p - 1) / p * S, t)

    arr = (ctypes.c_void_p * 8)(*peers)
    part = (S // p) - (S // p) % (1 << 16)
    for push in (1, 0):
        for ctas in (ctypes_c for ctypes_c in (16, 32, 64, 148)):
            for tile in (4096, 16384, 32768):
                depth = 8 if push else max(2, min(16, 196608 // tile))
                f = lambda: lib.probe_tma(push, arr, p - 1, ctypes.c_long(part), tile, depth,  # noqa
                                          (ctas // (p - 1)) * (p - 1), rank, st())
                t = timed(f)
                report("tma_push_allpeer" if push else "tma_pull_allpeer", (p - 1) * part, t,
                       ctas=ctas, tile=tile, depth=depth)
    for ctas in (148, 296):
        f = lambda: lib.probe_st_push(arr, p - 1, ctypes.c_long(part),  # noqa
                                      (ctas // (p - 1)) * (p - 1), 512, rank, st())
        t = timed(f)
        report("sm_store_push_allpeer", (p - 1) * part, t, ctas=ctas)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
