# N=1 K3 A/B: L2 256-B prefetch hint on the code loads, streaming stores
set -x
O=gpurun_out/r2x; mkdir -p $O
for pass in 1 2; do
for v in base k3ld k3st k3both; do
  if [ $v = base ]; then env=""; else env="KVX_LIB=paper_2502_09334_b200/_kvx_$v.so"; fi
  echo "ARGS: $v" >> $O/bench.log
  env $env timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline >> $O/bench.log 2>&1
  echo "ARGS: $v cfg4pair" >> $O/bench.log
  env $env timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --workload cfg4_70b_gqa_pair >> $O/bench.log 2>&1
done
done
