# N=2: kivi with concurrent K/V pulls; pull geometry A/B for small hand-offs; host enqueue cost
set -x
O=gpurun_out/r2f; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29561"
timeout 600 python -m pytest tests/test_gpu_kivi.py tests/test_gpu_multiproc.py -q -x --timeout 600 > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
for a in "--format kivi --group 32 --workload cfg4_70b_gqa_pair" "--format kivi --group 32"; do
  echo "ARGS: $a" >> $O/bench.log
  timeout 300 $TR bench.py --gpus 2 --steps 30 --warmup 5 --no-e2e $a >> $O/bench.log 2>&1
done
for wl in "--workload small_70b_gqa_128x1 --tokens 16" "--workload small_70b_gqa_128x1 --tokens 128" "--workload small_70b_gqa_128x1 --tokens 1024" "--workload cfg4_70b_gqa_pair"; do
  for v in base ps2 st8 sb6k; do
    if [ $v = base ]; then env=""; else env="KVX_LIB=paper_2502_09334_b200/_kvx_$v.so"; fi
    echo "ARGS: $v $wl" >> $O/ab.log
    env $env timeout 300 $TR bench.py --gpus 2 --steps 50 --warmup 5 --no-e2e $wl >> $O/ab.log 2>&1
  done
done
timeout 300 $TR tools/host_overhead.py > $O/host.log 2>&1
