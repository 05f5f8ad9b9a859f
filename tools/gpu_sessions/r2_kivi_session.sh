# GPU suite on 2 GPUs (includes same-GPU IPC + multigpu), then N=2 benches for kivi / default / small
set -x
O=gpurun_out/r2e; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29561"
timeout 1200 python -m pytest tests -m gpu -q -x -rs --timeout 600 > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
for a in "--format kivi --group 32 --workload cfg4_70b_gqa_pair" "--format kivi --group 32" "--workload cfg4_70b_gqa_pair" "" "--workload small_70b_gqa_128x1" "--workload small_70b_gqa_128x1 --queue-depth 4" "--workload trace_70b_gqa" "--workload trace_7b"; do
  echo "ARGS: $a" >> $O/bench.log
  timeout 300 $TR bench.py --gpus 2 --steps 30 --warmup 5 --no-e2e $a >> $O/bench.log 2>&1
done
KVX_LIB=paper_2502_09334_b200/_kvx_trace.so timeout 300 $TR tools/handoff_trace.py --tokens 128 >> $O/trace.log 2>&1
KVX_LIB=paper_2502_09334_b200/_kvx_trace.so timeout 300 $TR tools/handoff_trace.py --tokens 16 >> $O/trace.log 2>&1
