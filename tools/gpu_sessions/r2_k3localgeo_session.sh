# 1 GPU, N=1: K3-bulk on the local payload -- CTAs per SM x stage bytes vs the per-lane K3, across shapes and bit-widths
set -x
O=gpurun_out/r2klg; mkdir -p $O
for a in "" "--workload cfg3_13b_2048x8" "--workload cfg4_70b_gqa_pair" "--bits 8" "--bits 2"; do
  echo "ARGS: ldg $a" >> $O/bench.log
  timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --k3 ldg $a >> $O/bench.log 2>&1
  for pps in 1 2 3 4; do for st in 12288 24576; do
    echo "ARGS: bulk per_sm=$pps stage=$st $a" >> $O/bench.log
    KVX_LOCAL_PULL_PER_SM=$pps KVX_LOCAL_STAGE_BYTES=$st timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --k3 bulk $a >> $O/bench.log 2>&1
  done; done
done
echo done
