"""The compute kernels f1 must share the GPU with (diagnostics): one cuBLAS bf16 GEMM as in
bench_overlap.py, and one ResNet-50 channels-last bf16 backward as in bench_train.py, for
`ncu --section LaunchStats --section Occupancy` (registers, shared memory, CTAs per SM).

    ncu --section LaunchStats --section Occupancy -c 40 python tools/gemm_launch_probe.py
"""
import torch

torch.backends.cuda.preferred_blas_library("cublaslt")
A = torch.randn(2048, 2048, device="cuda", dtype=torch.bfloat16)
B = torch.randn(2048, 2048, device="cuda", dtype=torch.bfloat16)
C = torch.mm(A, B)
try:
    import torchvision
    m = torchvision.models.resnet50().cuda().to(memory_format=torch.channels_last)
    x = torch.randn(64, 3, 224, 224, device="cuda").contiguous(memory_format=torch.channels_last)
    with torch.autocast("cuda", dtype=torch.bfloat16):
        m(x).float().sum().backward()
except ImportError:
    pass
torch.cuda.synchronize()
