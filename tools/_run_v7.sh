timeout 600 ncu --set full --clock-control none --import-source on -k regex:tridiag_packed --launch-skip 10 --launch-count 1 -o gpurun_out/v7_packed python tools/run_config.py --config 2 --max_iters 30 > gpurun_out/v7_packed.log 2>&1
for V in 1 2 3; do BK_NARROW=$V timeout 120 python tools/dense_probe.py >> gpurun_out/v7_probe.txt 2>&1; done
for V in 2 3 4; do BK_GEMM_NARROW=$V timeout 120 python tools/dense_probe.py >> gpurun_out/v7_probe.txt 2>&1; done
for W in 0 4 8; do BK_TRI_NO_PACKED=1 BK_BISECT_W=$W timeout 300 python bench.py --no-cpu-baseline > gpurun_out/v7_bench_bw$W.json 2>/dev/null; done
