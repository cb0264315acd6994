cd /root/repo
O=gpurun_out
timeout 120 python tools/kclock.py c4 > $O/kclock_c4_f1.txt 2>&1
timeout 300 python tools/one_solve.py --config c4 --solves 2 --profile-last > $O/p_plain_c4.log 2>&1 && \
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:krylov_persist -c 1 \
    -o $O/c4p python tools/one_solve.py --config c4 --solves 2 --profile-last > $O/p_ncu_c4.log 2>&1
ncu -i $O/c4p.ncu-rep --page source --csv --print-source sass > $O/c4p_sass.csv 2>&1
ncu -i $O/c4p.ncu-rep --page raw --csv > $O/c4p_raw.csv 2>&1
python tools/ncu_summary.py $O/c4p.ncu-rep > $O/c4p_summary.txt 2>&1
rm -f $O/c4p.ncu-rep $O/*.bin $O/*.bin.p
