set -x
mkdir -p gpurun_out/r2v
timeout 3000 python tools/bench_matrix.py --gpus 2 --out gpurun_out/r2v/matrix_r02 > gpurun_out/r2v/matrix.log 2>&1
