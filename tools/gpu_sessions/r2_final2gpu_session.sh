# final code after chained pulls, 2 GPUs: smoke, full GPU suite, bench N=1 / N=2 defaults, reference arms, N=1 launch list
set -x
O=gpurun_out/r2f2g; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29795"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
timeout 1800 python -m pytest tests -m gpu -q -rs --timeout 900 > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $O/ref_n1.log 2>&1; echo rc=$? >> $O/ref_n1.log
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench_n1.log 2>&1; echo rc=$? >> $O/bench_n1.log
timeout 600 $TR bench.py --impl reference --gpus 2 --steps 20 --warmup 5 > $O/ref_n2.log 2>&1; echo rc=$? >> $O/ref_n2.log
timeout 600 $TR bench.py --gpus 2 --steps 20 --warmup 5 > $O/bench_n2.log 2>&1; echo rc=$? >> $O/bench_n2.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launch.log 2>&1
echo done
