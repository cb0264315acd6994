#!/bin/bash
cd "$(dirname "$0")/.."
timeout 400 python -m pytest tests/ -q -m gpu -p no:cacheprovider 2>&1 | tail -3
bash tools/gpu_ab.sh "c2 c3 c4" "PHIPM_PERSIST=1" "PHIPM_PERSIST=0"
timeout 200 python tools/kclock.py c4 > gpurun_out/kclock_c4_persist2.txt 2>&1
PHIPM_PERSIST=0 timeout 200 python tools/kclock.py c4 > gpurun_out/kclock_c4_2k.txt 2>&1
