# K3 with coalesced stores (KVX_K3_CO=1): parity tests, N=1 A/B, ncu of both K3s
set -x
O=gpurun_out/r2ah; mkdir -p $O
KVX_K3_CO=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_properties.py tests/test_gpu_handoff.py -q -x --timeout 600 > $O/tests_co.log 2>&1; echo rc=$? >> $O/tests_co.log
for pass in 1 2; do
for v in base co; do
  if [ $v = co ]; then env="KVX_K3_CO=1"; else env=""; fi
  for a in "" "--workload cfg4_70b_gqa_pair" "--bits 8" "--bits 2 --group 64"; do
    echo "ARGS: $v $a" >> $O/bench.log
    env $env timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline $a >> $O/bench.log 2>&1
  done
done
done
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
KVX_K3_CO=1 $CMD > $O/plain.log 2>&1 && \
KVX_K3_CO=1 ncu --set full --clock-control none --import-source on -k regex:"dequant_scatter" -s 3 -c 1 -o $O/k3co $CMD > $O/ncu.log 2>&1
echo ncu_rc=$? >> $O/ncu.log
