timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/v5_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/v5_pytest.log
for T in 256 512 1024; do BK_CHOL_THREADS=$T timeout 300 python bench.py --no-cpu-baseline > gpurun_out/v5_bench_$T.json 2>/dev/null; done
