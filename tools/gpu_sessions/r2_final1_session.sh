# driver-like pass on 1 GPU: smoke, the full -m gpu suite, bench default (e2e + cpu baseline), reference arm
set -x
O=gpurun_out/r2t; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x -rs --timeout 600 > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
timeout 600 python bench.py --steps 20 --warmup 3 > $O/bench_n1.log 2>&1; echo rc=$? >> $O/bench_n1.log
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > $O/ref_n1.log 2>&1; echo rc=$? >> $O/ref_n1.log
