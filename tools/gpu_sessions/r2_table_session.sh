# N=2 with the round-2 bench defaults (latency mode, Q=4): every bit-width's
# live calibration on the 4P4D pair workload (-> HandoffTable), short-prompt
# lines, kivi, config 3, traces
set -x
O=gpurun_out/r2j; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29561"
for b in 16 8 4 2; do
  g=128; [ $b = 2 ] && g=64
  echo "ARGS: --bits $b --group $g --workload cfg4_70b_gqa_pair" >> $O/bits.log
  timeout 300 $TR bench.py --gpus 2 --steps 30 --warmup 5 --no-e2e --bits $b --group $g --workload cfg4_70b_gqa_pair >> $O/bits.log 2>&1
done
for a in "--workload small_70b_gqa_128x1" "--workload small_70b_gqa_128x1 --batch 4" "--workload small_70b_gqa_128x1 --tokens 16" "--workload small_70b_gqa_128x1 --tokens 16 --batch 4" "--workload small_70b_gqa_128x1 --tokens 16 --batch 4 --queue-depth 8" "" "--workload trace_70b_gqa" "--workload trace_7b" "--format kivi --group 32 --workload cfg4_70b_gqa_pair" "--format kivi --group 32"; do
  echo "ARGS: $a" >> $O/bench.log
  timeout 300 $TR bench.py --gpus 2 --steps 50 --warmup 5 --no-e2e $a >> $O/bench.log 2>&1
done
