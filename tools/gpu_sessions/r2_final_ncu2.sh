# 1 GPU, N=1 with K3-bulk as the local default: bench, GPU parity/handoff tests, launch list and ncu --set full of K1-bulk and K3-bulk
set -x
O=gpurun_out/r2f2; mkdir -p $O
timeout 600 python bench.py --steps 20 --warmup 3 > $O/bench_n1.log 2>&1; echo rc=$? >> $O/bench_n1.log
timeout 900 python -m pytest tests/test_gpu_handoff.py tests/test_gpu_parity.py -q -x --timeout 800 > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/plain.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"quant_pack_bulk|pull_dequant" -s 6 -c 2 -o $O/k1k3 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_full.log 2>&1
