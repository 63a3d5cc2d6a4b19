timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/v6_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/v6_pytest.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/v6_bench.json 2>/dev/null
BK_TRI_NO_PACKED=1 timeout 300 python bench.py --no-cpu-baseline > gpurun_out/v6_bench_nopk.json 2>/dev/null
timeout 600 python tools/timeline_gaps.py > gpurun_out/v6_gaps.txt 2>&1
