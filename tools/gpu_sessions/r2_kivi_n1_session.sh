# 1 GPU, kivi N=1 (config 2, G=32): bench, then per-kernel durations and DRAM bytes of the kivi K1 kernels (K per channel, V per token) and K3
set -x
O=gpurun_out/r2kn1; mkdir -p $O
#timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --format kivi --group 32 > $O/bench.log 2>&1; echo rc=$? >> $O/bench.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,launch__block_size,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"kchan|quant_pack|dequant" -s 8 -c 8 --csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --format kivi --group 32 > $O/ncu.csv 2>&1
