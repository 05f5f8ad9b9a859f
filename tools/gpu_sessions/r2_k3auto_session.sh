# 1 GPU: local K3 chosen by row length (auto) -- GPU suite, smoke, bench N=1 default + shapes, launch list, ncu --set full of K1/K3
set -x
O=gpurun_out/r2ka; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -rs --timeout 900 > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
timeout 600 python bench.py --steps 20 --warmup 3 > $O/bench_n1.log 2>&1; echo rc=$? >> $O/bench_n1.log
for a in "--workload cfg3_13b_2048x8" "--workload cfg4_70b_gqa_pair" "--bits 8" "--bits 2" "--group 64" "--format kivi"; do
  echo "ARGS: $a" >> $O/shapes.log
  timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline $a >> $O/shapes.log 2>&1
done
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $O/ref_n1.log 2>&1; echo rc=$? >> $O/ref_n1.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"quant_pack|dequant" -s 6 -c 2 -o $O/k1k3 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_full.log 2>&1
echo done
