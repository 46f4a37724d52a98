"""One process, p emulated ranks on one GPU: the fused SGD step on the ResNet-50 group (for ncu /
compute-sanitizer runs of the two-shot kernels; NVLink is not involved).

    python tools/emulated_step.py [p] [algo] [iters]
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1801_03855_b200 as tc  # noqa: E402
import tc_workloads as W  # noqa: E402

p = int(sys.argv[1]) if len(sys.argv) > 1 else 2
algo = int(sys.argv[2]) if len(sys.argv) > 2 else 0
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 3
numels = W.RESNET50
comm = tc.Comm.emulated(p, 0)
comm.set_algorithm(algo)


def grp(kind, role, k):
    return [torch.from_numpy(a).cuda() for a in W.group(numels, kind, 2, 0, k, role)]


G = tc.Group(comm, [grp("grad", W.GRAD, k) for k in range(p)])
Wg = tc.Group(comm, [grp("param", W.PARAM, 0) for _ in range(p)])
D = tc.Group(comm, [grp("dw", W.DW, 0) for _ in range(p)])
for _ in range(iters):
    tc.sgd_step(Wg, G, D, lr=1e-3, momentum=0.9, wd=1e-4, rescale=1.0 / p)
torch.cuda.synchronize()
assert comm.async_error() == 0
print("ok", comm.last_launch())
