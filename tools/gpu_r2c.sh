#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import paper_0907_4631_b200 as P; P.build()"
PHIPM_EXPM_CLOCKS=1 timeout 120 python tools/cheb_clk.py 2>&1 | tail -12
timeout 900 python -m pytest tests/test_gpu_cheb.py -q -m gpu -p no:cacheprovider -rf 2>&1 | tail -8
timeout 300 python tools/cheb_bench.py 2>&1 | tail -10
