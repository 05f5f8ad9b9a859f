# N=2: recv_many correctness (multiproc test) + decode-round batching on short hand-offs
set -x
O=gpurun_out/r2h; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29561"
timeout 900 python -m pytest tests/test_gpu_multiproc.py tests/test_gpu_abort.py -q -x --timeout 600 > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
for a in "--tokens 128" "--tokens 128 --batch 2 --queue-depth 4" "--tokens 128 --batch 4 --queue-depth 4" "--tokens 128 --batch 4 --queue-depth 8" "--tokens 128 --batch 8 --queue-depth 8" "--tokens 16 --batch 8 --queue-depth 8" "--tokens 16" "--tokens 512 --batch 4 --queue-depth 8"; do
  echo "ARGS: $a" >> $O/bench.log
  timeout 300 $TR bench.py --gpus 2 --steps 50 --warmup 5 --no-e2e --workload small_70b_gqa_128x1 $a >> $O/bench.log 2>&1
done
