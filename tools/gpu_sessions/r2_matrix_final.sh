# 2 GPUs: the full N=1 / N=2 matrix on the final build (K3-bulk local, kchan split)
set -x
mkdir -p gpurun_out/r2mf
timeout 3000 python tools/bench_matrix.py --gpus 2 --out gpurun_out/r2mf/matrix_r02_final > gpurun_out/r2mf/matrix.log 2>&1
