# 1 GPU: K-per-channel quantiser A/B (TMA-staged TH=8 2 CTAs/SM, TH=16 1 CTA/SM, register kernel) on kivi N=1, ncu --set full of the TH=8 kernel
set -x
O=gpurun_out/r2kb3; mkdir -p $O
for pass in 1 2; do
for v in bulk th16 reg; do
  case $v in bulk) env="";; th16) env="KVX_LIB=paper_2502_09334_b200/_kvx_kth16.so";; reg) env="KVX_KCHAN_REG=1";; esac
  for g in 32 64; do
    echo "ARGS: $v G=$g" >> $O/bench.log
    env $env timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --format kivi --group $g >> $O/bench.log 2>&1
  done
done
done
timeout 900 python -m pytest tests/test_gpu_kivi.py -q -x > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
