# 2 GPUs: chained pulls at queue depth 4 vs 8, 16 and 128 tokens
set -x
O=gpurun_out/r2cq; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29799"
for a in "--tokens 16" "--tokens 128"; do
  for q in 4 8; do
    echo "ARGS: --chained --queue-depth $q $a" >> $O/bench.log
    timeout 300 $TR bench.py --gpus 2 --steps 400 --warmup 10 --no-e2e --workload small_70b_gqa_128x1 --chained --queue-depth $q $a >> $O/bench.log 2>&1
  done
done
echo done
