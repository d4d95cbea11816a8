"""pytest wrappers of the multi-GPU parity scripts (DP cutoff exchange, TP
long rounds, DP x TP) over real NCCL / CUDA IPC, one process per GPU.  They
need 2 (4) GPUs and are skipped otherwise; tests/test_gpu_local.py runs the
same multi-rank logic on one GPU."""
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("script,marker,ngpu", [("test_gpu_dp.py", "DP PARITY PASS", 2),
                                               ("test_gpu_tp.py", "TP PARITY PASS", 2),
                                               ("test_gpu_dpxtp.py", "DPxTP PARITY PASS", 4),
                                               ("test_gpu_migrate_nccl.py", "MIGRATE NCCL PASS", 2)])
def test_multi_gpu_parity(script, marker, ngpu):
    if _ngpus() < ngpu:
        pytest.skip("needs %d GPUs" % ngpu)
    # the scripts size their KV pools from free memory: hand back what this
    # process's caching allocator still holds from earlier tests (7B engine)
    import gc
    import torch
    gc.collect()
    torch.cuda.empty_cache()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", str(ngpu),
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "tests", script)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0 and marker in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
