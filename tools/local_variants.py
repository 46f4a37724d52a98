"""Time the p = 1 fused SGD kernel (HBM stream) for each launch-shape variant (TC_VARIANT).

    python tools/local_variants.py            # spawns one process per variant
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def one():
    import numpy as np
    import torch
    sys.path.insert(0, ROOT)
    import paper_1801_03855_b200 as tc
    import tc_workloads as W
    numels = W.RESNET50
    S = 4 * sum(numels)

    def flat(kind, role):
        f = torch.from_numpy(np.concatenate(W.group(numels, kind, 2, 0, 0, role))).cuda()
        return list(torch.split(f, numels))

    g, w, dw = flat("grad", W.GRAD), flat("param", W.PARAM), flat("dw", W.DW)
    comm = tc.Comm.single(0)
    G, Wg, D = tc.Group(comm, g), tc.Group(comm, w), tc.Group(comm, dw)
    out = {}
    for op in ("sgd", "easgd"):
        for _ in range(10):
            if op == "sgd":
                tc.sgd_step(Wg, G, D, lr=1e-3, momentum=0.9, wd=1e-4, rescale=1.0)
            else:
                tc.easgd_update(Wg, D, 0.1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        K = 200
        for _ in range(K):
            if op == "sgd":
                tc.sgd_step(Wg, G, D, lr=1e-3, momentum=0.9, wd=1e-4, rescale=1.0)
            else:
                tc.easgd_update(Wg, D, 0.1)
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / K / 1e3
        out[op] = {"t_us": t * 1e6, "hbm_gbs": (5 if op == "sgd" else 4) * S / t / 1e9,
                   "launch": comm.last_launch()}
    print(json.dumps(out))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "one":
        one()
    else:
        for v in range(6):
            r = subprocess.run([sys.executable, __file__, "one"], capture_output=True, text=True,
                               env=dict(os.environ, TC_VARIANT=str(v)))
            print(f"variant {v}: {r.stdout.strip()} {r.stderr.strip()[-300:]}", flush=True)
