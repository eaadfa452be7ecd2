"""Multi-GPU tests: the NCCL-backed distributed path on >= 2 B200s (torchrun),
checked bit-exact against the oracle at the same partition (tests/mp_parity.py)."""
import os
import subprocess
import sys

import pytest

from tests.conftest import gpu_count

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


ALT = {"PAIRAMG_MP_SETUP_OVERLAP": "1"}


@pytest.mark.parametrize("world,overlap", [(2, 1), (2, 0), (2, 2), (4, 1)])
def test_distributed_parity(world, overlap):
    """overlap=0: exchange-then-compute over the whole level (one Sell with halo columns);
    overlap=2: setup exchange overlapped with R / composition (setup_overlap)."""
    if gpu_count() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + 10 * world + overlap),
           os.path.join(ROOT, "tests", "mp_parity.py")]
    env = dict(os.environ, PAIRAMG_OVERLAP=str(min(overlap, 1)))
    if overlap == 2:
        env.update(ALT)
    r = subprocess.run(["timeout", "-k", "10", "300", *cmd], capture_output=True, text=True, timeout=400, cwd=ROOT,
                       env=env)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert out.count("MP_PARITY_OK") == 5, out[-4000:]


@pytest.mark.parametrize("world", [2, 4])
def test_marching_split_launch(world):
    """27-point 192 x 192 x 384: level 0's halo sweeps run the split launch with
    marching interior blocks (tests/mp_march.py); bitwise equal to one rank."""
    if gpu_count() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29700 + world),
           os.path.join(ROOT, "tests", "mp_march.py")]
    r = subprocess.run(["timeout", "-k", "10", "400", *cmd], capture_output=True, text=True, timeout=500, cwd=ROOT)
    out = r.stdout + r.stderr
    assert r.returncode == 0 and "MP_MARCH_OK" in out, out[-4000:]
