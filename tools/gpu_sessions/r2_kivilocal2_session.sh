# 1 GPU, N=1 kivi: per-lane decode kernels vs the single kivi pull on the local payload (now with the local span geometry for the V rows)
set -x
O=gpurun_out/r2kl2; mkdir -p $O
for a in "--group 32" "--group 64" "--group 32 --workload cfg4_70b_gqa_pair" "--group 32 --workload cfg3_13b_2048x8"; do
  echo "ARGS: perlane $a" >> $O/bench.log
  timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --format kivi $a >> $O/bench.log 2>&1
  echo "ARGS: pull $a" >> $O/bench.log
  KVX_KIVI_LOCAL_PULL=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --format kivi $a >> $O/bench.log 2>&1
done
echo done
