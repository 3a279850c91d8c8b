"""One chain n-sharded over real processes through the CUDA IPC exchange
(tools/ipc_shard_check.py under torchrun).  On a one-GPU box the shards share
the device and progress by time-slicing; the check is the cross-process path
itself: IPC-mapped peer exchange words, system-scope atomics and polls."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    import socket
    with socket.socket() as sock:
        sock.bind(("127.0.0.1", 0))
        return sock.getsockname()[1]


@pytest.mark.parametrize("procs,n,trees,iters,mode", [
    (2, 3000, 6, 3, "flat"), (3, 7001, 8, 4, "flat"), (2, 3000, 6, 3, "two_level"), (3, 7001, 8, 4, "two_level"),
    # configs[3] on 8 GPUs: n = 1e7, 1.25e6 points per shard (148 CTAs, the W=8 sweep), two-level exchange
    (8, 10_000_000, 12, 2, "two_level")])
def test_sharded_chain_over_processes(procs, n, trees, iters, mode):
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={procs}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "tools", "ipc_shard_check.py"), str(n), str(trees), str(iters), mode]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    line = [l for l in out.stdout.splitlines() if "ipc shard check" in l]
    assert out.returncode == 0 and line, out.stdout[-2000:] + out.stderr[-2000:]
    assert line[0].endswith("OK"), line[0]
