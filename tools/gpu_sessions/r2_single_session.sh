# N=2 single short hand-off: timeline with K1-bulk (latency mode, Q=4), and what the pull's stream-order wait costs
set -x
O=gpurun_out/r2r; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29561"
for t in 128 16; do
  KVX_LIB=paper_2502_09334_b200/_kvx_trace.so timeout 300 $TR tools/handoff_trace.py --tokens $t --no-gate-send --queue-depth 4 >> $O/trace.log 2>&1
done
for v in base nowait; do
  if [ $v = base ]; then env=""; else env="KVX_LIB=paper_2502_09334_b200/_kvx_$v.so"; fi
  for a in "--tokens 128" "--tokens 16" "--tokens 1024"; do
    echo "ARGS: $v $a" >> $O/bench.log
    env $env timeout 300 $TR bench.py --gpus 2 --steps 100 --warmup 10 --no-e2e --workload small_70b_gqa_128x1 $a >> $O/bench.log 2>&1
  done
done
