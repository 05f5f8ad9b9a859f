# 1 GPU: default bench (torch-CPU variant in cpu_baseline), then 2-bit K3 local: LDG vs bulk (the pull kernel on local HBM), ncu of the bulk 2-bit kernel
set -x
O=gpurun_out/r2b2; mkdir -p $O
timeout 600 python bench.py --steps 20 --warmup 3 > $O/bench_n1.log 2>&1; echo rc=$? >> $O/bench_n1.log
for b in 2 4; do for k in ldg bulk; do
  echo "ARGS: bits $b k3 $k" >> $O/k3.log
  timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --bits $b --group 64 --k3 $k >> $O/k3.log 2>&1
done; done
timeout 600 ncu --set full --clock-control none -k regex:pull_dequant -s 3 -c 1 -o $O/k3bulk2 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --bits 2 --group 64 --k3 bulk > $O/ncu.log 2>&1
