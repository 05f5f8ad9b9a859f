# N=1 K3 A/B: prefetch depth of the register K3, and the TMA-staged K3 (--k3 bulk) on local HBM
set -x
O=gpurun_out/r2q; mkdir -p $O
for pass in 1 2; do
for v in base k3pf3 k3pf4 k3pf6; do
  if [ $v = base ]; then env=""; else env="KVX_LIB=paper_2502_09334_b200/_kvx_$v.so"; fi
  echo "ARGS: $v" >> $O/bench.log
  env $env timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline >> $O/bench.log 2>&1
done
for v in base ps2s24 ps2s48; do
  if [ $v = base ]; then env=""; else env="KVX_LIB=paper_2502_09334_b200/_kvx_$v.so"; fi
  echo "ARGS: $v --k3 bulk" >> $O/bench.log
  env $env timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --k3 bulk >> $O/bench.log 2>&1
done
done
