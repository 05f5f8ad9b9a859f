# 1 GPU: the same-GPU multi-process transport tests (latency-mode block added)
set -x
O=gpurun_out/r2ai; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_multiproc.py -q -x -rs --timeout 1000 > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
