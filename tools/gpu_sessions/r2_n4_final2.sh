# 4 GPUs, final build (K3-bulk local, kchan split, pair roofline keys): N=4 bench lines, N=2 default, TP regroup, multigpu tests, smoke
set -x
O=gpurun_out/r2n4f2; mkdir -p $O
TR4="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29751"
for a in "" "--workload trace_70b_gqa --no-e2e" "--workload trace_7b --no-e2e" "--workload small_70b_gqa_128x1 --no-e2e" "--workload small_70b_gqa_128x1 --no-e2e --batch 4 --queue-depth 8" "--format kivi --group 32 --no-e2e" "--bits 2 --group 64 --no-e2e"; do
  echo "ARGS: $a" >> $O/bench_n4.log
  timeout 400 $TR4 bench.py --gpus 4 --steps 30 --warmup 5 $a >> $O/bench_n4.log 2>&1
done
timeout 400 $TR4 bench.py --impl reference --gpus 4 --steps 3 --warmup 1 > $O/ref_n4.log 2>&1
timeout 600 $TR4 tools/tp_bench.py > $O/tp.log 2>&1
timeout 1200 python -m pytest tests -m multigpu -q -rs --timeout 900 > $O/multigpu_tests.log 2>&1; echo rc=$? >> $O/multigpu_tests.log
TR2="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29752"
timeout 400 $TR2 bench.py --gpus 2 --steps 20 --warmup 3 > $O/bench_n2.log 2>&1; echo rc=$? >> $O/bench_n2.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
