# N=2, 2-bit (G=64) pulls: ring depth x CTAs per SM (base = 4 stages x 3 CTAs), config 3 and a config-4 pair
set -x
O=gpurun_out/r2br; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29731"
for pass in 1 2; do
for v in base s4c4 s6c2 s6c1 s8c1; do
  if [ $v = base ]; then env=""; else env="KVX_LIB=paper_2502_09334_b200/_kvx_$v.so"; fi
  for w in cfg3_13b_2048x8 cfg4_70b_gqa_pair; do
    echo "ARGS: $v $w" >> $O/bench.log
    env $env timeout 300 $TR bench.py --gpus 2 --steps 20 --warmup 3 --no-e2e --bits 2 --group 64 --workload $w >> $O/bench.log 2>&1
  done
done
done
