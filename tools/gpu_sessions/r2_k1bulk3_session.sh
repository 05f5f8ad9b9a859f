# K1-bulk stage geometry A/B (N=1 config 2 and a config-4 pair shape), two passes
set -x
O=gpurun_out/r2o; mkdir -p $O
for pass in 1 2; do
for v in base k1b32 k1b24x4 k1b48x2 k1b32x4 k1b40x2; do
  if [ $v = base ]; then env=""; else env="KVX_LIB=paper_2502_09334_b200/_kvx_$v.so"; fi
  echo "ARGS: $v" >> $O/bench.log
  env $env timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline >> $O/bench.log 2>&1
  echo "ARGS: $v cfg4pair" >> $O/bench.log
  env $env timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --workload cfg4_70b_gqa_pair >> $O/bench.log 2>&1
done
done
