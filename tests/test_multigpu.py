"""Multi-GPU z-slab runs across real NCCL ranks (one process per GPU, torchrun), bit-identical to the
single-GPU run. Each case launches tests/multigpu_worker.py with N ranks and is
skipped when fewer than N GPUs are visible (the build pool has one GPU per call; these run on the first
multi-GPU box). Covers every storage pattern x every halo transport (zero-copy NCCL, packed NCCL, fused
NVLink peer stores through NCCL symmetric windows) and index-list boundaries."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _gpus() -> int:
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


CASES = [(w, p, h, 0) for w in (2, 4, 8) for p in ("pull", "aa", "esotwist", "push") for h in (0, 1, 2)]
CASES += [(2, p, h, 1) for p in ("pull", "aa", "esotwist", "push") for h in (0, 2)]


@pytest.mark.parametrize("world,pattern,halo,links", CASES,
                         ids=[f"n{w}-{p}-halo{h}{'-links' if k else ''}" for w, p, h, k in CASES])
def test_nccl_ranks_bit_identical_to_single_gpu(world, pattern, halo, links):
    if _gpus() < world:
        pytest.skip(f"needs {world} GPUs, {_gpus()} visible")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "tests", "multigpu_worker.py"),
           "--pattern", pattern, "--halo", str(halo), "--steps", "13", "--geometry", "obstacles" if links else "channel",
           "--links", str(links)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert r.returncode == 0 and lines, f"rc={r.returncode}\n{r.stdout[-3000:]}\n{r.stderr[-3000:]}"
    out = json.loads(lines[-1])
    assert out["ok"], out
