# K1-bulk A/B round 2 (hoisted consumer arithmetic; stage geometries), N=1 config 2 + kivi N=2 PDL A/B
set -x
O=gpurun_out/r2n; mkdir -p $O
for v in base k1b k1b32 k1b8; do
  if [ $v = base ]; then env=""; else env="KVX_LIB=paper_2502_09334_b200/_kvx_$v.so"; fi
  echo "ARGS: $v" >> $O/bench.log
  env $env timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline >> $O/bench.log 2>&1
  echo "ARGS: $v cfg4pair" >> $O/bench.log
  env $env timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --workload cfg4_70b_gqa_pair >> $O/bench.log 2>&1
done
KVX_LIB=paper_2502_09334_b200/_kvx_k1b.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_properties.py -q -x > $O/tests_k1b.log 2>&1; echo rc=$? >> $O/tests_k1b.log
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
KVX_LIB=paper_2502_09334_b200/_kvx_k1b.so $CMD > $O/plain.log 2>&1 && \
KVX_LIB=paper_2502_09334_b200/_kvx_k1b.so ncu --set full --clock-control none --import-source on -k regex:"quant_pack" -s 3 -c 1 -o $O/k1bulk $CMD > $O/ncu.log 2>&1
echo ncu_rc=$? >> $O/ncu.log
