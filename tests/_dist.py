"""Process-group bring-up shared by the torchrun helpers (tests/dist_*.py).

Two modes:

* one GPU per rank (``cuda:LOCAL_RANK``, NCCL) — the product configuration;
* ``VP_SAME_DEVICE=1``: every rank on ``cuda:0``, gloo collectives — the
  whole multi-rank data plane (IPC-mapped rings, interprocess events, the
  shm handshake, the put kernel, the DP / tie / pipeline collectives,
  dispatch and morph) on a single B200. CUDA IPC works between processes
  on one device; NCCL refuses duplicate GPUs, so collectives go over gloo
  (which stages CUDA tensors through host memory).
"""

import os
import socket
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def same_device() -> bool:
    return os.environ.get("VP_SAME_DEVICE", "0") == "1"


def init():
    """Initialise torch.distributed for this rank; returns (device, backend)."""
    import torch
    import torch.distributed as dist
    local = 0 if same_device() else int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if same_device():
        dist.init_process_group("gloo")
        return dev, "gloo"
    dist.init_process_group("nccl", device_id=dev)
    return dev, "nccl"


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def launch(script: str, nproc: int, args=(), same: bool = True, timeout: int = 900):
    """torchrun ``tests/<script>`` on ``nproc`` ranks; returns the CompletedProcess."""
    env = dict(os.environ, PYTHONPATH=ROOT, VP_SAME_DEVICE="1" if same else "0",
               OMP_NUM_THREADS=str(max(1, (os.cpu_count() or 8) // max(nproc, 1))))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={nproc}", "--master-addr=127.0.0.1", f"--master-port={free_port()}",
           os.path.join(ROOT, "tests", script)] + [str(a) for a in args]
    return subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=timeout)
