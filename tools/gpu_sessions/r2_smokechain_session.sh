# 1 GPU, final code: smoke (now with a chained hand-off) and the full GPU suite
set -x
O=gpurun_out/r2sc; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -rs --timeout 900 > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
echo done
