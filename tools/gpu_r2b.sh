#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import paper_0907_4631_b200 as P; P.build()"
timeout 900 python -m pytest tests/test_gpu_cheb.py tests/test_gpu_ninept.py tests/test_gpu_solve.py -q -m gpu -p no:cacheprovider -rf -x 2>&1 | tail -30 > gpurun_out/r2b_tests.txt
cat gpurun_out/r2b_tests.txt
timeout 300 python tools/cheb_bench.py > gpurun_out/r2b_cheb_bench.txt 2>&1; cat gpurun_out/r2b_cheb_bench.txt
