# N=2 PDL A/B: early launch_dependents (default) vs none vs late (after the producer's last request)
set -x
O=gpurun_out/r2d; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29561"
for wl in "--workload small_70b_gqa_128x1 --tokens 128" "--workload small_70b_gqa_128x1 --tokens 512" "--workload small_70b_gqa_128x1 --tokens 1024" "--workload cfg4_70b_gqa_pair" "--workload cfg3_13b_2048x8"; do
  for v in "default|" "nopdl|--no-pdl" "late|LATE"; do
    name=${v%%|*}; flag=${v#*|}
    if [ "$flag" = "LATE" ]; then env="KVX_LIB=paper_2502_09334_b200/_kvx_pdllate.so"; flag=""; else env=""; fi
    echo "ARGS: $name $wl" >> $O/ab.log
    env $env timeout 300 $TR bench.py --gpus 2 --steps 30 --warmup 5 --no-e2e $wl $flag >> $O/ab.log 2>&1
  done
done
