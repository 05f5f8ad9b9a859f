# 2 GPUs: chained pulls re-measured with the ring of block sets (each hand-off of a chain in its own blocks), unchained alongside
set -x
O=gpurun_out/r2cr; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29797"
for a in "--tokens 128" "--tokens 16" "--tokens 512" "--tokens 1024"; do
  for c in "" "--chained"; do
    echo "ARGS: $c $a" >> $O/bench.log
    timeout 300 $TR bench.py --gpus 2 --steps 200 --warmup 10 --no-e2e --workload small_70b_gqa_128x1 $c $a >> $O/bench.log 2>&1
  done
done
echo done
