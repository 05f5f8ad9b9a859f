# kivi decode: caller-stream, PDL-chained K/V pulls, in-kernel slot release; host fast path
set -x
O=gpurun_out/r2l; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29561"
timeout 900 python -m pytest tests/test_gpu_kivi.py tests/test_gpu_multiproc.py tests/test_gpu_abort.py -q -x --timeout 600 > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
for a in "--format kivi --group 32 --workload cfg4_70b_gqa_pair" "--format kivi --group 32" "--format kivi --group 32 --workload trace_70b_gqa" "--workload small_70b_gqa_128x1" "--workload small_70b_gqa_128x1 --tokens 16" "--workload small_70b_gqa_128x1 --batch 4 --queue-depth 8" "--workload small_70b_gqa_128x1 --tokens 16 --batch 4 --queue-depth 8"; do
  echo "ARGS: $a" >> $O/bench.log
  timeout 300 $TR bench.py --gpus 2 --steps 50 --warmup 5 --no-e2e $a >> $O/bench.log 2>&1
done
timeout 300 $TR tools/host_overhead.py > $O/host.log 2>&1
