# final code, 4 GPUs: N=4 default (2P2D) + reference arm, traces, chained 128-token pairs, multigpu suite
set -x
O=gpurun_out/r2f4; mkdir -p $O
TR4="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29799"
timeout 600 $TR4 bench.py --impl reference --gpus 4 --steps 20 --warmup 5 > $O/ref_n4.log 2>&1; echo rc=$? >> $O/ref_n4.log
timeout 600 $TR4 bench.py --gpus 4 --steps 20 --warmup 5 > $O/bench_n4.log 2>&1; echo rc=$? >> $O/bench_n4.log
for a in "--workload trace_70b_gqa --no-e2e" "--workload small_70b_gqa_128x1 --no-e2e --steps 200 --warmup 10" "--workload small_70b_gqa_128x1 --no-e2e --chained --steps 200 --warmup 10"; do
  echo "ARGS: $a" >> $O/bench_n4_more.log
  timeout 400 $TR4 bench.py --gpus 4 --steps 30 --warmup 5 $a >> $O/bench_n4_more.log 2>&1
done
timeout 1200 python -m pytest tests -m multigpu -q -rs --timeout 900 > $O/multigpu_tests.log 2>&1; echo rc=$? >> $O/multigpu_tests.log
echo done
