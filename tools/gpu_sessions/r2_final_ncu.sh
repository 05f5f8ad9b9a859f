# final build, N=1: launch list and ncu --set full of K1-bulk and K3 (after the plain run exits 0)
set -x
O=gpurun_out/r2u; mkdir -p $O
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > $O/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv $CMD > $O/ncu_launches.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"quant_pack|dequant_scatter" -s 6 -c 2 -o $O/k1k3 $CMD > $O/ncu_full.log 2>&1
echo ncu_rc=$? >> $O/ncu_full.log
