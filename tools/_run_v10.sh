timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/v10_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/v10_pytest.log
timeout 120 python tools/dense_probe.py > gpurun_out/v10_probe.txt 2>&1
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/v10_bench.json 2>/dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tridiag_packed --launch-skip 50 --launch-count 1 -o gpurun_out/v10_packed python tools/run_config.py --config 2 > gpurun_out/v10_packed.log 2>&1
