# N=2: deeper pull ring for short pulls (6 stages default) vs 4 (deep0) vs 8
set -x
O=gpurun_out/r2an; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29681"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multiproc.py -q -x -k "bulk or pull or same_gpu" --timeout 800 > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
for pass in 1 2; do
for v in base deep0 deep8; do
  if [ $v = base ]; then env=""; else env="KVX_LIB=paper_2502_09334_b200/_kvx_$v.so"; fi
  for a in "--tokens 16" "--tokens 64" "--tokens 128" "--tokens 256" "--tokens 512"; do
    echo "ARGS: $v $a" >> $O/bench.log
    env $env timeout 300 $TR bench.py --gpus 2 --steps 100 --warmup 10 --no-e2e --workload small_70b_gqa_128x1 $a >> $O/bench.log 2>&1
  done
done
done
