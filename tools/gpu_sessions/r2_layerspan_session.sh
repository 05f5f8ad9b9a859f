# N=2: whole-layer spans for short pulls (A/B vs -DKVX_NO_LAYER_SPANS), plus the 1-GPU parity of the pull
set -x
O=gpurun_out/r2ak; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29651"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multiproc.py -q -x -k "bulk or pull or same_gpu" --timeout 800 > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
for pass in 1 2; do
for v in base nolayer; do
  if [ $v = base ]; then env=""; else env="KVX_LIB=paper_2502_09334_b200/_kvx_$v.so"; fi
  for a in "--tokens 16" "--tokens 32" "--tokens 128" "--tokens 16 --batch 4 --queue-depth 8"; do
    echo "ARGS: $v $a" >> $O/bench.log
    env $env timeout 300 $TR bench.py --gpus 2 --steps 100 --warmup 10 --no-e2e --workload small_70b_gqa_128x1 $a >> $O/bench.log 2>&1
  done
done
done
