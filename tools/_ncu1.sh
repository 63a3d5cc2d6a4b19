set -x
for K in chol_drop_kernel bisect_kernel tridiag_cluster_kernel; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K --launch-skip 30 --launch-count 1 -o gpurun_out/v4_$K python tools/run_config.py --config 2 --max_iters 40 > gpurun_out/v4_$K.log 2>&1
done
