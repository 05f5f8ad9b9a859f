# final code, 1 GPU (the driver's round-end tiers): smoke, full GPU suite, bench N=1 default + reference arm, launch list
set -x
O=gpurun_out/r2fl; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -rs --timeout 900 > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $O/ref_n1.log 2>&1; echo rc=$? >> $O/ref_n1.log
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench_n1.log 2>&1; echo rc=$? >> $O/bench_n1.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launch.log 2>&1
echo done
