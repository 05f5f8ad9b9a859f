# N=1 final evidence: bench line (e2e + cpu baseline), GPU suite, launch list and one
# ncu --set full capture of K1 and K3 (after the same command exited 0 without ncu)
set -x
O=gpurun_out/r2k; mkdir -p $O
timeout 600 python bench.py --steps 20 --warmup 3 > $O/bench_n1.log 2>&1; echo rc=$? >> $O/bench_n1.log
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > $O/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv $CMD > $O/ncu_launches.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"quant_pack_kernel|dequant_scatter_kernel" -s 6 -c 2 -o $O/k1k3 $CMD > $O/ncu_full.log 2>&1
echo ncu_rc=$? >> $O/ncu_full.log
