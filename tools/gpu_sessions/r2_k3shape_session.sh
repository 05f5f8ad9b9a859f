# 1 GPU, N=1: per-lane K3 vs K3-bulk on the local payload across shapes and bit-widths (which local K3 to default to)
set -x
O=gpurun_out/r2k3s; mkdir -p $O
for a in "" "--group 64" "--group 32" "--workload cfg3_13b_2048x8" "--workload cfg4_70b_gqa_pair" "--bits 8" "--bits 8 --group 64" "--bits 2 --group 64" "--bits 2"; do
  for k in ldg bulk; do
    echo "ARGS: $k $a" >> $O/bench.log
    timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --k3 $k $a >> $O/bench.log 2>&1
  done
done
