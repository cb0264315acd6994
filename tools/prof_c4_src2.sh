#!/bin/bash
# c4 TMEM Lanczos kernel: per-source-line instructions executed and stall samples (ncu source page)
cd /root/repo
O=gpurun_out
python -c "import paper_0907_4631_b200 as P; P.build()"
timeout 300 python tools/one_solve.py --config c4 --solves 2 --profile-last > $O/p4_plain.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:krylov_brick -c 1 -o $O/p4 python tools/one_solve.py --config c4 --solves 2 --profile-last > $O/p4_ncu.log 2>&1
ncu -i $O/p4.ncu-rep --page source --csv --print-source cuda > $O/p4_cuda.csv 2>&1
ncu -i $O/p4.ncu-rep --page source --csv --print-source sass > $O/p4_sass.csv 2>&1
ncu -i $O/p4.ncu-rep --page raw --csv > $O/p4_raw.csv 2>&1
rm -f $O/p4.ncu-rep
ls -la $O | grep p4
