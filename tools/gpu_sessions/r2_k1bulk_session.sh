# K1-bulk (TMA-staged K1) A/B at N=1: parity tests with KVX_K1_BULK=1, bench both, ncu of both K1s
set -x
O=gpurun_out/r2m; mkdir -p $O
KVX_K1_BULK=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_properties.py tests/test_gpu_handoff.py -q -x --timeout 600 > $O/tests_bulk.log 2>&1; echo rc=$? >> $O/tests_bulk.log
KVX_K1_BULK=1 timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_bulk.log 2>&1; echo rc=$? >> $O/smoke_bulk.log
for i in 1 2; do
  timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline >> $O/bench_reg.log 2>&1
  KVX_K1_BULK=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline >> $O/bench_bulk.log 2>&1
done
for w in "--workload cfg4_70b_gqa_pair" "--bits 8" "--bits 2 --group 64"; do
  echo "ARGS: $w" >> $O/bench_reg.log; echo "ARGS: $w" >> $O/bench_bulk.log
  timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline $w >> $O/bench_reg.log 2>&1
  KVX_K1_BULK=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline $w >> $O/bench_bulk.log 2>&1
done
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
KVX_K1_BULK=1 $CMD > $O/plain.log 2>&1 && \
KVX_K1_BULK=1 ncu --set full --clock-control none --import-source on -k regex:"quant_pack" -s 3 -c 1 -o $O/k1bulk $CMD > $O/ncu.log 2>&1
echo ncu_rc=$? >> $O/ncu.log
