"""Multi-GPU parity (needs >= 2 GPUs; run with `gpurun --gpus 2`): the sync
(reduce-scatter / sharded Adam / all-gather), LocalSGD and FedAdam schemes,
through the C ABI with NCCL, against the fp64 oracle's P-rank simulation."""
import os
import signal
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _ngpu():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("nproc", [2, 4])
@pytest.mark.parametrize("mode", ["sync", "sync32", "twosided", "twosided_nccl", "twosided_peer", "async",
                                  "fedadam"])
def test_multi_gpu_parity(mode, nproc):
    if _ngpu() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--standalone", "--nnodes=1",
           f"--nproc-per-node={nproc}", str(ROOT / "tests" / "dist_worker.py"), mode]
    # own process group: on a timeout the launcher AND its workers are killed
    # (a worker left spinning in a device-side barrier would hold its GPU)
    pr = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True, cwd=ROOT,
                          start_new_session=True)
    try:
        out, err = pr.communicate(timeout=600)
    except subprocess.TimeoutExpired:
        os.killpg(pr.pid, signal.SIGKILL)
        out, err = pr.communicate()
        pytest.fail(f"{mode} at {nproc} GPUs timed out\n" + err[-1500:])
    errs = [ln for ln in (out + err).splitlines()
            if "Error" in ln or "assert" in ln or "GCP_E" in ln][:20]
    assert pr.returncode == 0, "\n".join(errs) + "\n" + err[-1500:]
    # the bounds-checked build (GCP_LIB=libgcp_bounds.so) prints device-side violations
    bounds = [ln for ln in (out + err).splitlines() if "GCP-BOUNDS" in ln]
    assert not bounds, "\n".join(bounds[:10])
    assert "DIST-OK" in out
    print([ln for ln in out.splitlines() if "DIST-OK" in ln][0])
