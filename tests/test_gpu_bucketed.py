"""NEXT row f1: bucketed fused SGD launched per bucket as the (synthetic) backward pass produces
gradients in reverse order, on a side stream -- bit-exact against the oracle's whole-group step
(every element's arithmetic is independent of the bucketing)."""
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


@pytest.mark.parametrize("split", [False, True])
@pytest.mark.parametrize("p,bucket_bytes", [(3, 64 << 10), (4, 1 << 20), (2, 16)])
def test_bucketed_sgd_matches_whole_group(p, bucket_bytes, split):
    """fused: tc_sgd_step per bucket; split: tc_allreduce per bucket, then one local update."""
    numels = [7, 13, 1000, 4096, 65, 30000, 3, 512, 20000]
    gs = [W.group(numels, "grad", 57, 0, k, W.GRAD) for k in range(p)]
    w = W.group(numels, "param", 57, 0, 0, W.PARAM)
    dw = W.group(numels, "dw", 57, 0, 0, W.DW)
    comm = tc.Comm.emulated(p, 0)
    dg = [to_dev([np.zeros_like(a) for a in gs[k]]) for k in range(p)]
    dwt = [to_dev(w) for _ in range(p)]
    ddw = [to_dev(dw) for _ in range(p)]
    step = tc.BucketedStep(comm, dg, dwt, ddw, bucket_bytes=bucket_bytes, split=split)
    assert step.nbuckets >= 1
    hp = dict(lr=0.1, momentum=0.9, wd=1e-4, rescale=1.0 / (p * 128))
    compute = torch.cuda.current_stream()
    for t in reversed(range(len(numels))):      # the backward pass writes gradients last-first
        for k in range(p):
            dg[k][t].copy_(torch.from_numpy(gs[k][t]))
        step.grad_ready(t, compute, **hp)
    step.finish(compute)
    torch.cuda.synchronize()
    G, Ws, Dws = O.sgd_step([w] * p, gs, [dw] * p, **hp)
    for r in range(p):
        assert_bitwise(to_host(dg[r]), G, f"g rank {r}")
        assert_bitwise(to_host(dwt[r]), Ws[r], f"w rank {r}")
        assert_bitwise(to_host(ddw[r]), Dws[r], f"dw rank {r}")
    assert comm.async_error() == 0
    step.destroy()
    comm.destroy()
