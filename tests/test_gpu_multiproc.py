"""One process per GPU over NVLink (torchrun): every transport mode bit-exact
vs the oracle on the decode side.

The ``same_gpu`` variants run the SAME workers with every rank on cuda:0
(KVX_MP_SAME_GPU=1: two or four processes, one CUDA context each,
time-sliced on one B200, CUDA IPC between them), so the transport's whole
protocol -- IPC mapping, doorbells, queue slots, in-kernel waits, the native
pair, layer-wise streaming, host staging, kivi, TP regrouping -- is covered
on a 1-GPU box; the ``multigpu`` variants add the real NVLink links and the
NCCL baseline mode."""
import os
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ALL_MODES = "pull,pull_hostdb,pull_ldg,push,copy,nccl"


def _torchrun(nproc, port, script, *args, same_gpu=False, timeout=900):
    env = dict(os.environ)
    if same_gpu:
        env["KVX_MP_SAME_GPU"] = "1"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={nproc}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.join(HERE, script), *args]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, env=env)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    return r.stdout


@pytest.mark.gpu
def test_modes_over_ipc_same_gpu(cuda):
    """Every transport but NCCL between two processes on cuda:0."""
    out = _torchrun(2, 29543, "mp_handoff_check.py", ALL_MODES, same_gpu=True)
    assert "failures=0" in out
    assert "pull bits=4: native pair=True" in out  # the fused one-launch path ran
    assert "long/short alternation Q=2: ok" in out and "queue_depth=3" in out
    assert "recv_many: ok" in out
    assert "random lengths: 300 hand-offs" in out
    assert "latency mode: ok" in out


@pytest.mark.gpu
def test_fullsize_pairs_same_gpu(cuda):
    """BASELINE configs 3 and 4 (one pair) at full size over the fused pull,
    every byte of the decode cache checked."""
    out = _torchrun(2, 29544, "mp_fullsize_check.py", "cfg3_13b_2048x8,cfg4_70b_gqa_pair",
                    same_gpu=True)
    assert "failures=0" in out and out.count("bit-exact") == 2


@pytest.mark.gpu
def test_tp_regroup_same_gpu(cuda):
    """Mismatched TP degrees (1->2, 2->1, 2->2, 4->2 with shared ranks) via
    per-overlap edges, four processes on cuda:0."""
    out = _torchrun(4, 29545, "mp_tp_check.py", same_gpu=True)
    assert "failures=0" in out


@pytest.mark.gpu
@pytest.mark.multigpu
@pytest.mark.parametrize("nproc", [2, 4])
def test_modes_over_ipc(cuda, nproc):
    if cuda.cuda.device_count() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    out = _torchrun(nproc, 29533, "mp_handoff_check.py", ALL_MODES, timeout=600)
    assert "failures=0" in out
    assert "pull bits=4: native pair=True" in out


@pytest.mark.gpu
@pytest.mark.multigpu
@pytest.mark.parametrize("nproc", [2, 4])
def test_fullsize_pairs(cuda, nproc):
    """BASELINE configs 3 and 4 at full size over the default fused pull."""
    if cuda.cuda.device_count() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    wls = "cfg3_13b_2048x8,cfg4_70b_gqa_pair" if nproc == 2 else "cfg4_70b_gqa_pair"
    out = _torchrun(nproc, 29534, "mp_fullsize_check.py", wls)
    assert "failures=0" in out and "bit-exact" in out


@pytest.mark.gpu
@pytest.mark.multigpu
def test_tp_regroup(cuda):
    """Mismatched TP degrees (1->2, 2->1, 2->2, 4->2 with shared ranks) via per-overlap edges."""
    if cuda.cuda.device_count() < 4:
        pytest.skip("needs 4 GPUs")
    out = _torchrun(4, 29535, "mp_tp_check.py")
    assert "failures=0" in out
