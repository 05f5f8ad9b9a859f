# 2 GPUs: after the kchan change -- full GPU suite, kivi N=1 (G 32/64) and N=2 (config 3, config-4 pair) benches, a short soak (kivi phase included)
set -x
O=gpurun_out/r2kv; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29741"
timeout 1800 python -m pytest tests -m gpu -q -rs --timeout 900 > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
for g in 32 64; do
  echo "ARGS: N=1 kivi G=$g" >> $O/bench.log
  timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --format kivi --group $g >> $O/bench.log 2>&1
done
for w in cfg3_13b_2048x8 cfg4_70b_gqa_pair; do
  echo "ARGS: N=2 kivi G=32 $w" >> $O/bench.log
  timeout 300 $TR bench.py --gpus 2 --steps 20 --warmup 3 --no-e2e --format kivi --group 32 --workload $w >> $O/bench.log 2>&1
done
timeout 400 $TR tools/soak.py --seconds 150 > $O/soak.log 2>&1; echo rc=$? >> $O/soak.log
