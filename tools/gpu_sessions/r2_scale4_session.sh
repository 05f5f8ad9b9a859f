# 4 GPUs, last build: the driver's scaling sequence N=1,2,4 back to back (both arms, default flags), then the multigpu suite
set -x
O=gpurun_out/r2s4; mkdir -p $O
for n in 1 2 4; do
  if [ $n = 1 ]; then R="python"; else R="python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 --master-port=2977$n"; fi
  timeout 600 $R bench.py --impl reference --gpus $n --steps 20 --warmup 5 > $O/ref_n$n.log 2>&1; echo rc=$? >> $O/ref_n$n.log
  timeout 600 $R bench.py --gpus $n --steps 20 --warmup 5 > $O/bench_n$n.log 2>&1; echo rc=$? >> $O/bench_n$n.log
done
timeout 1200 python -m pytest tests -m multigpu -q -rs --timeout 900 > $O/multigpu_tests.log 2>&1; echo rc=$? >> $O/multigpu_tests.log
echo done
