# 2-bit pull: consumer-bound at one CTA per SM? A/B with 2 pull CTAs per SM; plus the random-length mp test
set -x
O=gpurun_out/r2y; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29591"
timeout 900 python -m pytest tests/test_gpu_multiproc.py -q -x -k "modes_over_ipc_same_gpu" --timeout 800 > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
for v in base ps2; do
  if [ $v = base ]; then env=""; else env="KVX_LIB=paper_2502_09334_b200/_kvx_$v.so"; fi
  for a in "--bits 2 --group 64 --workload cfg4_70b_gqa_pair" "--bits 2 --group 64" "--bits 4 --workload cfg4_70b_gqa_pair" "--bits 8 --workload cfg4_70b_gqa_pair"; do
    echo "ARGS: $v $a" >> $O/bench.log
    env $env timeout 300 $TR bench.py --gpus 2 --steps 30 --warmup 5 --no-e2e $a >> $O/bench.log 2>&1
  done
done
