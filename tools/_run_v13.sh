P="python tools/spmm_probe.py --config 2 --k 69 96 138 26"
timeout 120 $P > gpurun_out/v13_spmm.txt 2>&1
for T in 64 128 256; do for L in 512 1024; do BK_SPMM_L1=$L BK_SPMM_TILE=$T timeout 120 $P >> gpurun_out/v13_spmm.txt 2>&1; done; done
BK_SPMM_L1=512 BK_SPMM_TILE=128 BK_SPMM_CPS=2 timeout 120 $P >> gpurun_out/v13_spmm.txt 2>&1
BK_SPMM_L1=256 BK_SPMM_TILE=64 BK_SPMM_CPS=4 timeout 120 $P >> gpurun_out/v13_spmm.txt 2>&1
BK_SPMM_L1=512 BK_SPMM_TILE=128 BK_SPMM_H=1000000 timeout 120 $P >> gpurun_out/v13_spmm.txt 2>&1
