"""Multi-GPU: the real NCCL ring (ncclSend/Recv of vertex sub-parts) at
world = 2 (and 4 when present), deterministic mode against the oracle."""
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


def _ngpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("world,mode,kind", [
    (2, "det", "deepwalk"), (2, "hogwild", "deepwalk"), (4, "det", "deepwalk"), (4, "hogwild", "deepwalk"),
    (2, "det", "node2vec"), (2, "det", "line"), (4, "det", "line"), (2, "det", "bf16"), (4, "det", "bf16"),
    (4, "det", "groups2"), (2, "det", "ipc"), (4, "det", "ipc"), (4, "hogwild", "ipc"),
    (2, "det", "staged"), (4, "det", "staged"),
])
def test_nccl_ring(world, mode, kind):
    if _ngpus() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={29600 + world}",
           os.path.join(ROOT, "tools", "multi_parity.py"), mode, kind]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "MULTI" in r.stdout
