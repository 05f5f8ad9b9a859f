"""One process per GPU over NVLink (torchrun): every transport mode bit-exact
vs the oracle on the decode side.  Needs >= 2 GPUs (gpurun --gpus 2/4)."""
import os
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("nproc", [2, 4])
def test_modes_over_ipc(cuda, nproc):
    if cuda.cuda.device_count() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={nproc}", "--master-addr=127.0.0.1", "--master-port=29533",
           os.path.join(HERE, "mp_handoff_check.py"), "pull,pull_hostdb,pull_ldg,push,copy,nccl"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "failures=0" in r.stdout
    assert "pull bits=4: graphs=True" in r.stdout  # hand-offs replayed as CUDA graphs


@pytest.mark.parametrize("nproc", [2, 4])
def test_fullsize_pairs(cuda, nproc):
    """BASELINE configs 3 and 4 at full size over the default fused pull."""
    if cuda.cuda.device_count() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    wls = "cfg3_13b_2048x8,cfg4_70b_gqa_pair" if nproc == 2 else "cfg4_70b_gqa_pair"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={nproc}", "--master-addr=127.0.0.1", "--master-port=29534",
           os.path.join(HERE, "mp_fullsize_check.py"), wls]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "failures=0" in r.stdout and "bit-exact" in r.stdout


def test_tp_regroup(cuda):
    """Mismatched TP degrees (1->2, 2->1, 2->2, 4->2 with shared ranks) via per-overlap edges."""
    if cuda.cuda.device_count() < 4:
        pytest.skip("needs 4 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=4",
           "--master-addr=127.0.0.1", "--master-port=29535",
           os.path.join(HERE, "mp_tp_check.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "failures=0" in r.stdout
