timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/v9_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/v9_pytest.log
timeout 120 python tools/dense_probe.py > gpurun_out/v9_probe.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tridiag_packed --launch-skip 5 --launch-count 1 -o gpurun_out/v9_packed python tools/run_config.py --config 2 --max_iters 60 > gpurun_out/v9_packed.log 2>&1
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/v9_bench.json 2>/dev/null
