"""Time the p = 1 TMA stream (fused SGD, ResNet-50 group) at several grid sizes."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1801_03855_b200 as tc  # noqa: E402
import tc_workloads as W  # noqa: E402

numels = W.GROUPS[sys.argv[1] if len(sys.argv) > 1 else "resnet50"]
S = 4 * sum(numels)


def flat(kind, role):
    f = torch.from_numpy(np.concatenate(W.group(numels, kind, 2, 0, 0, role))).cuda()
    return list(torch.split(f, numels))


g, w, dw = flat("grad", W.GRAD), flat("param", W.PARAM), flat("dw", W.DW)
comm = tc.Comm.single(0)
G, Wg, D = tc.Group(comm, g), tc.Group(comm, w), tc.Group(comm, dw)
for ctas in (0, 148, 222, 296, 444):
    comm.set_tuning(ctas, 0, -1)
    for _ in range(10):
        tc.sgd_step(Wg, G, D, lr=1e-3, momentum=0.9, wd=1e-4, rescale=1.0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(200):
        tc.sgd_step(Wg, G, D, lr=1e-3, momentum=0.9, wd=1e-4, rescale=1.0)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 200 * 1e3
    print(f"ctas={ctas:4d} launch={comm.last_launch()} {t:7.1f} us  {5 * S / t / 1e3:7.0f} GB/s")
