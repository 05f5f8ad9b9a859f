# N=2 long contexts: one 70B-GQA request of 32k and 64k tokens per hand-off; kivi at 32k
set -x
O=gpurun_out/r2am; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29671"
for a in "--tokens 32768" "--tokens 65536" "--tokens 32768 --format kivi --group 32"; do
  echo "ARGS: $a" >> $O/bench.log
  timeout 600 $TR bench.py --gpus 2 --steps 10 --warmup 3 --no-e2e --workload cfg4_70b_gqa_pair --queue-depth 2 $a >> $O/bench.log 2>&1
done
