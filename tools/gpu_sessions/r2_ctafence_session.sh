# K1 arrivals: one fence per CTA (bar.sync + thread 0's fence) instead of one per thread. 1 GPU K1 period, then N=2 short hand-offs and config 3
set -x
O=gpurun_out/r2cf; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29711"
for pass in 1 2; do
for v in base ctafence; do
  if [ $v = base ]; then env=""; else env="KVX_LIB=paper_2502_09334_b200/_kvx_$v.so"; fi
  for t in 16 128 1024; do
    env $env timeout 120 python tools/k1_small.py --tokens $t | sed "s/^/$v /" >> $O/period.log 2>&1
  done
done
done
for pass in 1 2; do
for v in base ctafence; do
  if [ $v = base ]; then env=""; else env="KVX_LIB=paper_2502_09334_b200/_kvx_$v.so"; fi
  for a in "--tokens 16" "--tokens 128" "--tokens 1024"; do
    echo "ARGS: $v $a" >> $O/bench.log
    env $env timeout 300 $TR bench.py --gpus 2 --steps 100 --warmup 10 --no-e2e --workload small_70b_gqa_128x1 $a >> $O/bench.log 2>&1
  done
  echo "ARGS: $v cfg3" >> $O/bench.log
  env $env timeout 300 $TR bench.py --gpus 2 --steps 20 --warmup 3 --no-e2e >> $O/bench.log 2>&1
done
done
