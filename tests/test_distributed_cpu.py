"""The multi-GPU slab path's host logic on CPU: world size 2 over gloo.

Runs tests/dist/worker_cpu.py under torch.distributed.run: the NCCL unique
id hand-off (distributed.comm_from_torch), the slab decomposition of the
3-D real FFT with the pack / all-to-all / unpack layouts of csrc/solver.cu
(tests/dist/slab_model.py) against numpy's global rfftn, and the
slab-count independence of the residual's reduction slots.
"""

import os
import socket
import subprocess
import sys

from conftest import ROOT


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_slab_model_gloo():
    env = dict(os.environ, OMP_NUM_THREADS="1", NCCL_SOCKET_IFNAME="lo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_port()}",
           os.path.join(ROOT, "tests", "dist", "worker_cpu.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=240, env=env)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert "WORKER-OK" in r.stdout
