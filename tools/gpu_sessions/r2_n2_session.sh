set -x
mkdir -p gpurun_out/r2b
O=gpurun_out/r2b
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29561"
timeout 900 python -m pytest tests -m multigpu -q -x -rs --timeout 600 > $O/multigpu_tests.log 2>&1; echo rc=$? >> $O/multigpu_tests.log
for a in "" "--workload small_70b_gqa_128x1 --no-e2e" "--workload cfg4_70b_gqa_pair --no-e2e" "--workload trace_70b_gqa --no-e2e" "--workload trace_7b --no-e2e" "--format kivi --group 32 --workload cfg4_70b_gqa_pair --no-e2e"; do
  echo "ARGS: $a" >> $O/bench_n2.log
  timeout 300 $TR bench.py --gpus 2 --steps 20 --warmup 3 $a >> $O/bench_n2.log 2>&1
done
for t in 16 128 1024; do
  KVX_LIB=paper_2502_09334_b200/_kvx_trace.so timeout 300 $TR tools/handoff_trace.py --tokens $t >> $O/trace.log 2>&1
done
