# 1 GPU, the very last build: smoke, full GPU suite, bench N=1 default
set -x
O=gpurun_out/r2z; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -rs --timeout 900 > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench_n1.log 2>&1; echo rc=$? >> $O/bench_n1.log
echo done
