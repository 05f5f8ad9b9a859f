# decode-round serving loop: one pull per hand-off vs draining the queue with recv_many
set -x
O=gpurun_out/r2w; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29581"
timeout 900 python -m pytest tests/test_gpu_multiproc.py -q -x -k "modes_over_ipc" --timeout 600 > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
for a in "--prompts 24 --prefill-us 3000" "--prompts 24 --prefill-us 3000 --drain" "--prompts 24 --prefill-us 500" "--prompts 24 --prefill-us 500 --drain" "--prompts 256 --tokens 128 --prefill-us 20 --queue-depth 8 --round-gb 1 --latency-mode" "--prompts 256 --tokens 128 --prefill-us 20 --queue-depth 8 --round-gb 1 --latency-mode --drain" "--prompts 256 --tokens 16 --prefill-us 5 --queue-depth 8 --round-gb 0.25 --latency-mode" "--prompts 256 --tokens 16 --prefill-us 5 --queue-depth 8 --round-gb 0.25 --latency-mode --drain"; do
  echo "ARGS: $a" >> $O/serving.log
  timeout 300 $TR tools/decode_rounds.py $a >> $O/serving.log 2>&1
done
