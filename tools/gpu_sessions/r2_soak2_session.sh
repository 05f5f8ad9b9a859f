set -x
O=gpurun_out/r2al; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29661"
timeout 1200 $TR tools/soak.py --seconds 500 > $O/soak.log 2>&1; echo rc=$? >> $O/soak.log
