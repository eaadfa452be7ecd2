"""Multi-GPU tests: the NCCL-backed distributed path on >= 2 B200s (torchrun),
checked bit-exact against the oracle at the same partition (tests/mp_parity.py)."""
import os
import subprocess
import sys

import pytest

from tests.conftest import gpu_count

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


@pytest.mark.parametrize("world", [2, 4])
def test_distributed_parity(world):
    if gpu_count() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + world),
           os.path.join(ROOT, "tests", "mp_parity.py")]
    r = subprocess.run(["timeout", "-k", "10", "300", *cmd], capture_output=True, text=True, timeout=400, cwd=ROOT)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert out.count("MP_PARITY_OK") == 5, out[-4000:]
