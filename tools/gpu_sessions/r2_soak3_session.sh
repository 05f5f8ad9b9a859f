# 2 GPUs: soak with chained recv rounds (plus recv_many and plain rounds, both prefill modes, 4 queue depths, kivi)
set -x
O=gpurun_out/r2s3; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29663"
timeout 900 $TR tools/soak.py --seconds 400 > $O/soak.log 2>&1; echo rc=$? >> $O/soak.log
echo done
