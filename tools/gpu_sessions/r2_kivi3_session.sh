# kivi as one pull kernel vs two: tests + N=2 lines (same box)
set -x
O=gpurun_out/r2aa; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29611"
timeout 900 python -m pytest tests/test_gpu_kivi.py tests/test_gpu_multiproc.py -q -x --timeout 800 > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
for pass in 1 2; do
for v in fused two; do
  if [ $v = two ]; then env="KVX_KIVI_TWO_KERNELS=1"; else env=""; fi
  for a in "--format kivi --group 32 --workload cfg4_70b_gqa_pair" "--format kivi --group 32" "--format kivi --group 32 --workload trace_70b_gqa"; do
    echo "ARGS: $v $a" >> $O/bench.log
    env $env timeout 300 $TR bench.py --gpus 2 --steps 30 --warmup 5 --no-e2e $a >> $O/bench.log 2>&1
  done
done
done
