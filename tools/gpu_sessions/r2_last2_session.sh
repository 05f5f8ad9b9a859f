# last build, 2 GPUs: full GPU suite (same-GPU IPC + 2-GPU tests), bench N=2 default, reference arm N=2, N=1 default on a 2-GPU box
set -x
O=gpurun_out/r2l2; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29691"
timeout 1800 python -m pytest tests -m gpu -q -rs --timeout 900 > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
timeout 600 $TR bench.py --gpus 2 --steps 20 --warmup 3 > $O/bench_n2.log 2>&1; echo rc=$? >> $O/bench_n2.log
timeout 600 $TR bench.py --impl reference --gpus 2 --steps 5 --warmup 3 > $O/ref_n2.log 2>&1; echo rc=$? >> $O/ref_n2.log
timeout 600 python bench.py --steps 20 --warmup 3 > $O/bench_n1.log 2>&1; echo rc=$? >> $O/bench_n1.log
echo done
