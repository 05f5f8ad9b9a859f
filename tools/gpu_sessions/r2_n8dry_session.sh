# 4 GPUs: dry run of the N=8 rank logic (8 ranks, pairs i -> i+4 share a GPU over same-device IPC; numbers are not measurements), both arms
set -x
O=gpurun_out/r2n8; mkdir -p $O
TR8="python -m torch.distributed.run --nnodes=1 --nproc-per-node=8 --master-addr=127.0.0.1 --master-port=29781"
timeout 600 $TR8 bench.py --gpus 8 --steps 5 --warmup 3 > $O/bench_n8_dry.log 2>&1; echo rc=$? >> $O/bench_n8_dry.log
timeout 600 $TR8 bench.py --impl reference --gpus 8 --steps 3 --warmup 1 > $O/ref_n8.log 2>&1; echo rc=$? >> $O/ref_n8.log
echo done
