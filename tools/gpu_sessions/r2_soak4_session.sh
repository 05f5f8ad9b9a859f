# 2 GPUs, final code: a longer soak (chained, recv_many and plain rounds; 4 queue configs; kivi)
set -x
O=gpurun_out/r2s4k; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29665"
timeout 1200 $TR tools/soak.py --seconds 720 > $O/soak.log 2>&1; echo rc=$? >> $O/soak.log
echo done
