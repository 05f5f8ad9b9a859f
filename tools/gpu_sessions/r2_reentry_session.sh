# re-entry validation of HEAD on 1 GPU: smoke, full GPU suite, bench N=1 + reference arm, launch list, ncu --set full of K1/K3
set -x
O=gpurun_out/r2re; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -rs --timeout 900 > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
timeout 600 python bench.py --steps 20 --warmup 3 > $O/bench_n1.log 2>&1; echo rc=$? >> $O/bench_n1.log
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $O/ref_n1.log 2>&1; echo rc=$? >> $O/ref_n1.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"quant_pack|dequant" -s 6 -c 2 -o $O/k1k3 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_full.log 2>&1
echo done
