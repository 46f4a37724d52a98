"""Config 4 (BASELINE.json): MPI Elastic SGD on 8 ranks = 2 clients x 4 GPUs, synchronous SGD
inside each client (tc_sgd_step over the client's 4 ranks) and the elastic update across the
clients every tau = 4 steps (tc_easgd_update over the counterpart pairs (k, k+4)), 16 steps --
checked bit for bit against oracle.esgd_sequence (Fig. code-snippet-4; reading R10).

On one GPU the 8 ranks run as emulated comms (each comm = one cooperative kernel whose
blockIdx.y is the rank); test_gpu_multiproc.py covers real processes.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1801_03855_b200 as tc  # noqa: E402
import tc_workloads as W  # noqa: E402
from oracle import tc_oracle as O  # noqa: E402
from gpu_util import to_dev, to_host, assert_bitwise  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind,oneshot", [("grad", 0), ("grad", 1 << 20), ("int", 0), ("grad", "ll")])
def test_config4_esgd_sequence(kind, oneshot):
    numels = [7, 13, 1000, 4096, 65]
    C, Q, steps, tau = 2, 4, 16, 4          # clients, GPUs per client
    if kind == "int":
        hp = dict(alpha=0.25, lr=0.5, momentum=0.5, wd=0.0, rescale=1.0 / 512)
        center = W.group(numels, "int", W.CFG_EASGD, 0, 0, W.CENTER)
        x0 = [W.group(numels, "int", W.CFG_EASGD, 0, i, W.PARAM) for i in range(C)]
    else:
        hp = dict(alpha=0.1, lr=0.1, momentum=0.9, wd=1e-4, rescale=1.0 / (Q * 128))
        center = W.group(numels, "center", W.CFG_EASGD, 0, 0, W.CENTER)
        x0 = [W.client_params(numels, center, W.CFG_EASGD, 0, i) for i in range(C)]
    dw0 = [W.group(numels, "zeros", 0, 0, 0, 0) for _ in range(C)]

    def grads(t, i):
        return [W.group(numels, kind, W.CFG_EASGD, t, Q * i + k, W.GRAD) for k in range(Q)]

    # device state: every GPU holds its client's params, momentum and a center replica
    x = [to_dev(x0[g // Q]) for g in range(C * Q)]
    dw = [to_dev(dw0[g // Q]) for g in range(C * Q)]
    xc = [to_dev(center) for _ in range(C * Q)]
    g = [to_dev(W.group(numels, "zeros", 0, 0, 0, 0)) for _ in range(C * Q)]
    clients = [tc.Comm.emulated(Q, 0) for _ in range(C)]
    pairs = [tc.Comm.emulated(C, 0) for _ in range(Q)]
    for cm in clients + pairs:
        if oneshot == "ll":
            cm.set_ll_max(1 << 30)
        else:
            cm.set_ll_max(0)
            cm.set_tuning(0, 0, oneshot)
    G = [tc.Group(clients[i], [g[Q * i + k] for k in range(Q)]) for i in range(C)]
    Wt = [tc.Group(clients[i], [x[Q * i + k] for k in range(Q)]) for i in range(C)]
    D = [tc.Group(clients[i], [dw[Q * i + k] for k in range(Q)]) for i in range(C)]
    X = [tc.Group(pairs[k], [x[Q * i + k] for i in range(C)]) for k in range(Q)]
    XC = [tc.Group(pairs[k], [xc[Q * i + k] for i in range(C)]) for k in range(Q)]
    for t in range(steps):
        if t % tau == 0:
            for k in range(Q):
                tc.easgd_update(X[k], XC[k], hp["alpha"])
        for i in range(C):
            for k, gr in enumerate(grads(t, i)):
                for dst, src in zip(g[Q * i + k], gr):
                    dst.copy_(torch.from_numpy(src))
            tc.sgd_step(Wt[i], G[i], D[i], lr=hp["lr"], momentum=hp["momentum"], wd=hp["wd"],
                        rescale=hp["rescale"])
    torch.cuda.synchronize()
    wx, wc, wdw = O.esgd_sequence(x0, center, dw0, grads, steps, tau, **hp)
    for gpu in range(C * Q):
        i = gpu // Q
        assert_bitwise(to_host(x[gpu]), wx[i], f"x gpu {gpu}")
        assert_bitwise(to_host(dw[gpu]), wdw[i], f"dw gpu {gpu}")
        assert_bitwise(to_host(xc[gpu]), wc, f"center gpu {gpu}")
    for cm in clients + pairs:
        assert cm.async_error() == 0
    for grp in G + Wt + D + X + XC:
        grp.destroy()
    for cm in clients + pairs:
        cm.destroy()
