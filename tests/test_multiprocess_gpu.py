"""One process per rank through the IPC communicator (cudaIpc heap mapping,
cross-process flags, peer stores / copy-engine pulls), launched with torchrun.
Also runs the chained MLP as a PyTorch autograd module (torch_ops.TPMlp).
All ranks may share the single GPU of the test box: the kernels of the two
processes time-slice, and every device wait is bounded, so a missing signal
fails as DeadlockError instead of hanging."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_two_processes_ipc_match_oracle():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29533", os.path.join(ROOT, "scripts", "mp_worker.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    print(out.stdout[-4000:], out.stderr[-4000:])
    assert out.returncode == 0
    lines = [l for l in out.stdout.splitlines() if l.startswith("RESULT")]
    assert len(lines) == 2
    for line in lines:
        res = json.loads(line.split(" ", 2)[2])
        assert len(res) == 20  # 9 operator cases, 3 torch ops, TPMlp GELU and SwiGLU (out, dx, dW_up, dW_down)
        for case, (err, tol) in res.items():
            assert err <= tol, (case, err, tol)
