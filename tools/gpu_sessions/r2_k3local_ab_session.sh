# 1 GPU, N=1 config 2: K3 LDG vs K3-bulk (the TMA pull kernel on the local payload), alternated 3x
set -x
O=gpurun_out/r2k3ab; mkdir -p $O
for pass in 1 2 3; do
for k in ldg bulk; do
  echo "ARGS: $k" >> $O/bench.log
  timeout 300 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --k3 $k >> $O/bench.log 2>&1
done
done
