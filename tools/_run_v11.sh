timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/v11_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/v11_pytest.log
timeout 120 python tools/syev_probe.py 100 130 160 180 195 207 218 > gpurun_out/v11_syev.txt 2>&1
BK_TRI_NO_PACKED=1 timeout 120 python tools/syev_probe.py 100 130 160 180 195 207 218 >> gpurun_out/v11_syev.txt 2>&1
timeout 120 python tools/dense_probe.py > gpurun_out/v11_probe.txt 2>&1
timeout 600 python tools/timeline_gaps.py > gpurun_out/v11_gaps.txt 2>&1
