"""The copy-engine ring over CUDA IPC (NE_TRANSPORT_IPC): real multi-process
training -- processes share the available GPUs round-robin, so these run on a
single-GPU box -- compared with the oracle (tools/ipc_parity.py)."""
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world,mode,groups", [(2, "det", 1), (3, "det", 1), (2, "hogwild", 1), (4, "det", 2),
                                               (8, "det", 1), (8, "det", 4)])
def test_ipc_ring(world, mode, groups):
    """groups = 2: the NEXT-3 two-level ring (two groups of two ranks).  World 8
    (eight processes sharing the box's GPUs) covers the 8-GPU bench's default
    transport, which no 4-GPU box can run with one rank per GPU."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={29700 + world + (mode == 'hogwild') * 10 + groups * 20}",
           os.path.join(ROOT, "tools", "ipc_parity.py"), mode, str(groups)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300 if world <= 4 else 600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "IPC " in r.stdout
