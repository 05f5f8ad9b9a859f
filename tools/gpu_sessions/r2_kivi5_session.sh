# kivi pull kernel without doorbells (local payload): kivi tests, N=1 kivi A/B
set -x
O=gpurun_out/r2ad; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kivi.py -q -x --timeout 800 > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
KVX_KIVI_LOCAL_PULL=1 timeout 900 python -m pytest tests/test_gpu_kivi.py -q -x --timeout 800 > $O/tests_localpull.log 2>&1; echo rc=$? >> $O/tests_localpull.log
for pass in 1 2; do
for v in perlane pull; do
  if [ $v = pull ]; then env="KVX_KIVI_LOCAL_PULL=1"; else env=""; fi
  for a in "--format kivi --group 32" "--format kivi --group 32 --workload cfg4_70b_gqa_pair"; do
    echo "ARGS: $v $a" >> $O/bench.log
    env $env timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline $a >> $O/bench.log 2>&1
  done
done
done
