# K1-bulk as the default: full GPU suite (1 GPU view + 2 GPUs), smoke, N=1 bench, geometry A/B, N=2 lines
set -x
O=gpurun_out/r2p; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29561"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x -rs --timeout 600 > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
for v in base k1b44x2 k1b56x2 k1reg; do
  if [ $v = base ]; then env=""; else env="KVX_LIB=paper_2502_09334_b200/_kvx_$v.so"; fi
  for w in "" "--workload cfg4_70b_gqa_pair" "--bits 8" "--bits 2 --group 64"; do
    echo "ARGS: $v $w" >> $O/bench_n1.log
    env $env timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline $w >> $O/bench_n1.log 2>&1
  done
done
for a in "" "--workload cfg4_70b_gqa_pair" "--workload small_70b_gqa_128x1" "--workload small_70b_gqa_128x1 --batch 4 --queue-depth 8" "--format kivi --group 32 --workload cfg4_70b_gqa_pair" "--format kivi --group 32 --workload cfg4_70b_gqa_pair --no-pdl" "--format kivi --group 32" "--format kivi --group 32 --no-pdl" "--mode nccl"; do
  echo "ARGS: $a" >> $O/bench_n2.log
  timeout 300 $TR bench.py --gpus 2 --steps 30 --warmup 5 --no-e2e $a >> $O/bench_n2.log 2>&1
done
