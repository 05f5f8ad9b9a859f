# N=2: prefill-side latency mode (no front-end gate, K1s chained with PDL) vs gate
set -x
O=gpurun_out/r2i; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29561"
for a in "--tokens 16" "--tokens 16 --no-gate-send" "--tokens 128" "--tokens 128 --no-gate-send" "--tokens 128 --no-gate-send --queue-depth 4" "--tokens 128 --no-gate-send --queue-depth 8 --batch 4" "--tokens 512 --no-gate-send" "--tokens 1024 --no-gate-send"; do
  echo "ARGS: $a" >> $O/bench.log
  timeout 300 $TR bench.py --gpus 2 --steps 100 --warmup 10 --no-e2e --workload small_70b_gqa_128x1 $a >> $O/bench.log 2>&1
done
for a in "--workload cfg4_70b_gqa_pair" "--workload cfg4_70b_gqa_pair --no-gate-send" "" "--no-gate-send"; do
  echo "ARGS: $a" >> $O/bench.log
  timeout 300 $TR bench.py --gpus 2 --steps 30 --warmup 5 --no-e2e $a >> $O/bench.log 2>&1
done
timeout 300 $TR tools/host_overhead.py > $O/host.log 2>&1
KVX_LIB=paper_2502_09334_b200/_kvx_trace.so timeout 300 $TR tools/handoff_trace.py --tokens 128 --no-gate-send >> $O/trace.log 2>&1
KVX_LIB=paper_2502_09334_b200/_kvx_trace.so timeout 300 $TR tools/handoff_trace.py --tokens 16 --no-gate-send >> $O/trace.log 2>&1
