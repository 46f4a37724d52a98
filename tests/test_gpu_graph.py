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


@pytest.mark.parametrize("oneshot,ll,algo,numels", [
    (0, 0, 1, [7, 13, 1000, 4096]), (1 << 20, 0, 0, [7, 13, 1000, 4096]),
    (0, 1 << 20, 0, [7, 13, 1000, 4096]), (0, 0, 6, [7, 13, 1000, 4096, 300001])])
def test_graph_capture_and_replay(oneshot, ll, algo, numels):
    """Three dependent allreduces (scale 1/2 at p = 4) captured in one graph and replayed three
    times without resetting: every call changes the data (the first halves the rank sum, every
    later one doubles it), so each of the 9 replayed calls must have run."""
    p = 4
    xs = [W.group(numels, "int", 55, 0, k, W.GRAD) for k in range(p)]
    comm = tc.Comm.emulated(p, 0)
    comm.set_algorithm(algo)
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
                tc.allreduce(grp, 0.5, stream=s)
    torch.cuda.synchronize()
    cur = xs
    for rep in range(3):
        graph.replay()
        torch.cuda.synchronize()
        for _ in range(3):
            cur = [O.allreduce(cur, 0.5)] * p
        for r in range(p):
            assert_bitwise(to_host(dev[r]), cur[0], f"replay {rep} rank {r}")
    assert comm.async_error() == 0
    grp.destroy()
    comm.destroy()
