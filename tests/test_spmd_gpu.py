"""The one-process-per-GPU path (spmd.py + bench.py under torchrun) on a single GPU:
three ranks share GPU 0 and exchange over gloo (NCCL refuses two ranks on one device).
Checks distributed dot / inclusive and exclusive scan / min / sample sort against numpy."""

import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_spmd_three_ranks_one_gpu():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "3",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "tools", "spmd_check.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert out.stdout.count("'dot': True, 'scan': True, 'exscan': True, 'min': True, 'sort': True, "
                            "'keysort': True") == 3


def test_spmd_nccl_one_rank():
    # the NCCL exchange itself (fill kernels -> all_gather_into_tensor on the compute stream
    # -> kernel readback) on a world of one: the only NCCL world one GPU can host
    env = dict(os.environ, SPMD_BACKEND="nccl", DRK_SPMD_COMBINE="collective")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "tools", "spmd_check.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert "'dot': True, 'scan': True, 'exscan': True, 'min': True, 'sort': True, 'keysort': True" in out.stdout


@pytest.mark.parametrize("combine", ["collective", "ipc"])
def test_bench_two_ranks_shared_gpu(combine):
    env = dict(os.environ, DRK_BENCH_SHARE_GPU="1", DRK_SPMD_COMBINE=combine)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "1", "--log2n", "24", "--no-cpu", "--no-e2e"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1 and '"n_gpus": 2' in lines[0]


def test_spmd_three_ranks_peer_memory_exchange():
    # the reduce / scan exchange forced onto the library's own kernel over CUDA-IPC-mapped
    # mailboxes (DRK_SPMD_COMBINE=ipc; "auto", the default, picks it after a trial exchange),
    # three processes on one GPU; setup over gloo, no NCCL
    env = dict(os.environ, DRK_SPMD_COMBINE="ipc")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "3",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "tools", "spmd_check.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert out.stdout.count("'dot': True, 'scan': True, 'exscan': True, 'min': True, 'sort': True, "
                            "'keysort': True") == 3
