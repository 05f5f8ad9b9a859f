# 2 GPUs: chained pulls (KVX_PAIR_CHAINED) -- multiproc checks (same-GPU and 2-GPU), then N=2 A/B per launch: default vs --chained
set -x
O=gpurun_out/r2ch; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29791"
timeout 1200 python -m pytest tests/test_gpu_multiproc.py -q -rs --timeout 900 > $O/mp_tests.log 2>&1; echo rc=$? >> $O/mp_tests.log
for a in "--workload small_70b_gqa_128x1" "--workload small_70b_gqa_128x1 --tokens 16" "--workload small_70b_gqa_128x1 --tokens 512" "--workload small_70b_gqa_128x1 --tokens 1024" ""; do
  for c in "" "--chained"; do
    echo "ARGS: $c $a" >> $O/bench.log
    timeout 300 $TR bench.py --gpus 2 --steps 100 --warmup 10 --no-e2e $c $a >> $O/bench.log 2>&1
  done
done
echo done
