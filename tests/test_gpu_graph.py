"""Hot-path calls are CUDA-graph capturable: the call epoch lives on the device, so a captured
sequence of collectives replays correctly (launch-bound small messages, B200 guide)."""
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


@pytest.mark.parametrize("oneshot,ll", [(0, 0), (1 << 20, 0), (0, 1 << 20)])
def test_graph_capture_and_replay(oneshot, ll):
    p = 4
    numels = [7, 13, 1000, 4096]
    xs = [W.group(numels, "int", 55, 0, k, W.GRAD) for k in range(p)]
    comm = tc.Comm.emulated(p, 0)
    comm.set_tuning(0, 0, oneshot)
    comm.set_ll_max(ll)
    dev = [to_dev(x) for x in xs]
    grp = tc.Group(comm, dev)
    pristine = [[t.clone() for t in d] for d in dev]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        tc.allreduce(grp, 1.0, stream=s)  # warm-up outside the graph
        torch.cuda.synchronize()
        for d, pr in zip(dev, pristine):
            for a, b in zip(d, pr):
                a.copy_(b)
        torch.cuda.synchronize()
        with torch.cuda.graph(graph, stream=s):
            for _ in range(3):  # three dependent collectives in one graph
                tc.allreduce(grp, 0.25, stream=s)
    torch.cuda.synchronize()
    want = O.allreduce(xs, 0.25)           # integers: sum/4, then the mean is a fixed point...
    for _ in range(2):
        want = O.allreduce([want] * p, 0.25)
    for rep in range(3):                   # replay from the same inputs several times
        for d, pr in zip(dev, pristine):
            for a, b in zip(d, pr):
                a.copy_(b)
        graph.replay()
        torch.cuda.synchronize()
        for r in range(p):
            assert_bitwise(to_host(dev[r]), want, f"replay {rep} rank {r}")
    assert comm.async_error() == 0
    grp.destroy()
    comm.destroy()
