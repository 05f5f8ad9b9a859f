# 4 GPUs: every ordered pair measured (calibrate.py, HandoffPlan pull with peer access), each bit-width
set -x
O=gpurun_out/r2aj; mkdir -p $O
for b in 16 8 4 2; do
  timeout 600 python -m paper_2502_09334_b200.calibrate --gpus 4 --bits $b --out $O/b200x4_kv$b.cluster.json > $O/calib_kv$b.log 2>&1; echo rc=$? >> $O/calib_kv$b.log
done
