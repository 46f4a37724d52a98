"""T2 (real multi-GPU): one process per GPU over CUDA IPC + NVLink, launched with torchrun.

Skipped when fewer than 2 GPUs are visible.  Runs at p = 2 and, when available, at p = 3, 4 and 8
(p = 3: owner chunks of a non-power-of-two split).
"""
import os
import socket
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("p", [2, 3, 4, 8])
def test_multiprocess_parity(p):
    if NGPU < p:
        pytest.skip(f"needs {p} GPUs, have {NGPU}")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={p}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(HERE, "mp_worker.py")]
    env = dict(os.environ, TC_TIMEOUT_MS="20000")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env)
    sys.stdout.write(r.stdout[-4000:])
    sys.stderr.write(r.stderr[-4000:])
    assert r.returncode == 0
    assert f"MP_WORKER_OK p={p}" in r.stdout


@pytest.mark.parametrize("p", [2, 4])
def test_multiprocess_stress(p):
    """tools/stress_mp.py: 500 calls, every call changing the data, algorithms rotating (pull,
    TMA, NVLS, one-shot, LL) with broadcasts interleaved; every call checked on the GPU."""
    if NGPU < p:
        pytest.skip(f"needs {p} GPUs, have {NGPU}")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={p}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(os.path.dirname(HERE), "tools", "stress_mp.py"), "500"]
    env = dict(os.environ, TC_TIMEOUT_MS="20000")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    sys.stdout.write(r.stdout[-2000:])
    sys.stderr.write(r.stderr[-2000:])
    assert r.returncode == 0
    assert f"stress p={p} iters=500: mismatching calls 0, async errors 0" in r.stdout
