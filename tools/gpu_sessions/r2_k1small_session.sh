# 1 GPU: K1 on short hand-offs (70B GQA, 16 / 128 tokens): period per launch and ncu kernel duration, rows-per-span and signal A/B
# (KVX_K1B_ROWS was a temporary A/B hook of this session, since removed from the library)
set -x
O=gpurun_out/r2k1s; mkdir -p $O
for t in 16 128; do
  for v in "" "KVX_K1B_ROWS=8" "KVX_K1B_ROWS=4" "KVX_K1B_ROWS=2" "KVX_K1_REG=1"; do
    env $v timeout 120 python tools/k1_small.py --tokens $t >> $O/period.log 2>&1
    env $v timeout 120 python tools/k1_small.py --tokens $t --no-signal >> $O/period.log 2>&1
    env $v timeout 120 python tools/k1_small.py --tokens $t --lpc 2 >> $O/period.log 2>&1
  done
done
for t in 16 128; do
  for v in "" "KVX_K1B_ROWS=8" "KVX_K1B_ROWS=4" "KVX_K1_REG=1"; do
    echo "ARGS: $t $v" >> $O/ncu.log
    env $v timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none -k regex:quant_pack -s 20 -c 20 --csv python tools/k1_small.py --tokens $t --iters 20 > $O/ncu_${t}_${v:-base}.csv 2>&1
  done
done
