# 2 GPUs, final-build validation: full GPU suite (same-GPU + 2-GPU), N=2 lines, 2-bit pull CTAs A/B
set -x
O=gpurun_out/r2z; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29601"
timeout 1500 python -m pytest tests -m gpu -q -x -rs --timeout 900 > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
for v in base p2b3; do
  if [ $v = base ]; then env=""; else env="KVX_LIB=paper_2502_09334_b200/_kvx_$v.so"; fi
  for a in "--bits 2 --group 64 --workload cfg4_70b_gqa_pair" "--bits 2 --group 64"; do
    echo "ARGS: $v $a" >> $O/bench.log
    env $env timeout 300 $TR bench.py --gpus 2 --steps 30 --warmup 5 --no-e2e $a >> $O/bench.log 2>&1
  done
done
for a in "" "--workload cfg4_70b_gqa_pair --no-e2e" "--workload small_70b_gqa_128x1 --no-e2e" "--format kivi --group 32 --workload cfg4_70b_gqa_pair --no-e2e" "--workload trace_70b_gqa --no-e2e"; do
  echo "ARGS: base $a" >> $O/bench.log
  timeout 300 $TR bench.py --gpus 2 --steps 30 --warmup 5 $a >> $O/bench.log 2>&1
done
