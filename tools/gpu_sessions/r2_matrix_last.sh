# 2 GPUs: the full N=1 / N=2 matrix on the final code (local K3 by row length, chained pulls rows)
set -x
mkdir -p gpurun_out/r2ml
timeout 3000 python tools/bench_matrix.py --gpus 2 --out gpurun_out/r2ml/matrix_r02_last > gpurun_out/r2ml/matrix.log 2>&1
echo done
