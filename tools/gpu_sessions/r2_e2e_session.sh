# 2 GPUs: pipelined host-buffer runs (N=1 HostHandoff), e2e over all timed steps at N=1 and N=2
set -x
O=gpurun_out/r2e2e; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29691"
timeout 900 python -m pytest tests/test_gpu_handoff.py -q -rs --timeout 800 > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_n1.log 2>&1; echo rc=$? >> $O/bench_n1.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 5 > $O/bench_n1_e5.log 2>&1; echo rc=$? >> $O/bench_n1_e5.log
timeout 600 $TR bench.py --gpus 2 --steps 20 --warmup 3 > $O/bench_n2.log 2>&1; echo rc=$? >> $O/bench_n2.log
echo done
