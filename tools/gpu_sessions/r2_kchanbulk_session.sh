# 1 GPU: TMA-staged K-per-channel quantiser (kivi prefill): parity (kivi tests incl. same-GPU IPC), N=1 kivi bench A/B vs the register kernel, ncu durations
set -x
O=gpurun_out/r2kb; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kivi.py tests/test_gpu_multiproc.py -q -x -k "kivi" --timeout 800 > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
for pass in 1 2; do
for v in bulk reg; do
  if [ $v = bulk ]; then env=""; else env="KVX_KCHAN_REG=1"; fi
  for g in 32 64; do
    echo "ARGS: $v G=$g" >> $O/bench.log
    env $env timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --format kivi --group $g >> $O/bench.log 2>&1
  done
done
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"kchan|quant_pack|dequant" -s 8 -c 4 --csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --format kivi --group 32 > $O/ncu.csv 2>&1
