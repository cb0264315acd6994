#!/bin/bash
# ncu source-level capture of the c5 CSR SpMV (one launch mid-solve), summarised here.
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 300 python tools/one_solve.py --config c5 --solves 2 --profile-last > $O/p5_plain.log 2>&1 && \
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:spmv_stream -s 6 -c 1 \
    -o $O/c5s python tools/one_solve.py --config c5 --solves 2 --profile-last > $O/p5_ncu.log 2>&1
ncu -i $O/c5s.ncu-rep --page source --csv --print-source sass > $O/c5s_sass.csv 2>&1
python tools/ncu_summary.py $O/c5s.ncu-rep > $O/c5s_summary.txt 2>&1
rm -f $O/c5s.ncu-rep
