#!/bin/bash
# ncu --set full source-level captures (SASS lines with warp-stall samples and executed instructions)
# of the c4 TMEM Lanczos kernel and the c5 x-ring SpMV; summaries only come back.
cd "$(dirname "$0")/.."
O=gpurun_out
python -c "import paper_0907_4631_b200 as P; P.build()"
cap() {  # config regex skip name
  timeout 300 python tools/one_solve.py --config $1 --solves 2 --profile-last > $O/ps_plain_$4.log 2>&1 && \
  timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 \
    -o $O/ps_$4 python tools/one_solve.py --config $1 --solves 2 --profile-last > $O/ps_ncu_$4.log 2>&1
  ncu -i $O/ps_$4.ncu-rep --page source --csv --print-source sass > $O/ps_$4_sass.csv 2>&1
  python tools/ncu_hot.py $O/ps_$4_sass.csv 40 > $O/ps_$4_hot.txt 2>&1
  rm -f $O/ps_$4.ncu-rep
}
cap c4 krylov_persist_tm 0 c4tm
cap c5 spmv_stream 6 c5spmv
gzip -f $O/ps_*_sass.csv
ls -la $O | grep ps_
