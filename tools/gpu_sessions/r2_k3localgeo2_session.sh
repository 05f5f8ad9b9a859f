# 1 GPU, N=1: K3-bulk on the local payload with spans of whole consumer-warp passes -- stage bytes x CTAs per SM, vs the per-lane K3
set -x
O=gpurun_out/r2klg2; mkdir -p $O
for a in "" "--workload cfg3_13b_2048x8" "--workload cfg4_70b_gqa_pair" "--bits 8" "--bits 2"; do
  echo "ARGS: ldg $a" >> $O/bench.log
  timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --k3 ldg $a >> $O/bench.log 2>&1
  for pps in 1 2; do for st in 16384 24576 32768 49152; do
    echo "ARGS: bulk per_sm=$pps stage=$st $a" >> $O/bench.log
    KVX_LOCAL_PULL_PER_SM=$pps KVX_LOCAL_STAGE_BYTES=$st timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --k3 bulk $a >> $O/bench.log 2>&1
  done; done
done
echo done
