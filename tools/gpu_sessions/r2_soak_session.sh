set -x
O=gpurun_out/r2ag; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29641"
timeout 1500 $TR tools/soak.py --seconds 900 > $O/soak.log 2>&1; echo rc=$? >> $O/soak.log
