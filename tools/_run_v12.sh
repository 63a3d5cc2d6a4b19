timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/v12_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/v12_pytest.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/v12_bench.json 2>/dev/null
timeout 120 python tools/dense_probe.py > gpurun_out/v12_probe.txt 2>&1
timeout 600 python tools/timeline_gaps.py > gpurun_out/v12_gaps.txt 2>&1
