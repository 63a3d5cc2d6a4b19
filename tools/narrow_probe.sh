#!/bin/bash
# 69-wide (config 2 shrunk) shapes: Gram / update with 72- vs 96-wide tiles
cd "$(dirname "$0")/.."
for s in "69 69" "165 69" "138 69" "96 96" "192 96"; do python tools/gram_probe.py $s; done
