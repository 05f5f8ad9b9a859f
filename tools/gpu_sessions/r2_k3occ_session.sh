# N=1 K3 occupancy A/B (registers vs warps)
set -x
O=gpurun_out/r2ae; mkdir -p $O
for pass in 1 2; do
for v in base k3pf1 k3mb8 k3mb6; do
  if [ $v = base ]; then env=""; else env="KVX_LIB=paper_2502_09334_b200/_kvx_$v.so"; fi
  echo "ARGS: $v" >> $O/bench.log
  env $env timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline >> $O/bench.log 2>&1
  echo "ARGS: $v cfg4pair" >> $O/bench.log
  env $env timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --workload cfg4_70b_gqa_pair >> $O/bench.log 2>&1
done
done
