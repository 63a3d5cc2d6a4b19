#!/bin/bash
# Tile-shape tuning of the K2/K3 DMMA kernels (BK_GRAM_VARIANT / BK_GEMM_VARIANT).
cd "$(dirname "$0")/.."
for v in 0 1 2 3 4; do
  echo "gram variant $v"
  for s in "288 288" "288 96" "192 96" "96 96" "480 480" "768 768"; do BK_GRAM_VARIANT=$v python tools/gram_probe.py $s; done
done
for v in 0 1 2 3 4; do
  echo "gemm variant $v"
  BK_GEMM_VARIANT=$v python tools/bench_kernels.py gemm | tail -1
done
