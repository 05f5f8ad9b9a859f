# N=2: host enqueue cost after the lean fast path; front-end slot gate on/off
set -x
O=gpurun_out/r2g; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29561"
timeout 300 $TR tools/host_overhead.py > $O/host.log 2>&1
for wl in "--tokens 16" "--tokens 128" "--tokens 128 --queue-depth 4" "--tokens 512"; do
  for g in "" "--no-gate-send"; do
    echo "ARGS: $wl $g" >> $O/ab.log
    timeout 300 $TR bench.py --gpus 2 --steps 100 --warmup 10 --no-e2e --workload small_70b_gqa_128x1 $wl $g >> $O/ab.log 2>&1
  done
done
for a in "--workload cfg4_70b_gqa_pair" "--workload cfg4_70b_gqa_pair --no-gate-send" "--format kivi --group 32 --workload cfg4_70b_gqa_pair" "--format kivi --group 32"; do
  echo "ARGS: $a" >> $O/ab.log
  timeout 300 $TR bench.py --gpus 2 --steps 30 --warmup 5 --no-e2e $a >> $O/ab.log 2>&1
done
KVX_LIB=paper_2502_09334_b200/_kvx_trace.so timeout 300 $TR tools/handoff_trace.py --tokens 16 >> $O/trace.log 2>&1
