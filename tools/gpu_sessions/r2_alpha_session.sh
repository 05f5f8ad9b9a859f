# N=2 alpha study: small hand-offs, queue depth, PDL, token sweep, trace timelines
set -x
O=gpurun_out/r2c; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29561"
for a in "--tokens 16" "--tokens 64" "--tokens 128" "--tokens 256" "--tokens 512" "--tokens 1024" "--tokens 128 --queue-depth 4" "--tokens 128 --no-pdl" "--tokens 128 --gate-recv"; do
  echo "ARGS: $a" >> $O/sweep.log
  timeout 300 $TR bench.py --gpus 2 --steps 50 --warmup 5 --workload small_70b_gqa_128x1 --no-e2e $a >> $O/sweep.log 2>&1
done
for t in 16 128 1024; do
  KVX_LIB=paper_2502_09334_b200/_kvx_trace.so timeout 300 $TR tools/handoff_trace.py --tokens $t >> $O/trace.log 2>&1
done
KVX_LIB=paper_2502_09334_b200/_kvx_trace.so timeout 300 $TR tools/handoff_trace.py --tokens 128 --no-pdl >> $O/trace.log 2>&1
KVX_LIB=paper_2502_09334_b200/_kvx_trace.so timeout 300 $TR tools/handoff_trace.py --tokens 128 --queue-depth 4 >> $O/trace.log 2>&1
