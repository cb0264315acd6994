cd /root/repo
O=gpurun_out
timeout 300 python tools/one_solve.py --config c4 --solves 2 --profile-last > $O/p4_plain.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:krylov_persist_tm -c 1 -o $O/p4 python tools/one_solve.py --config c4 --solves 2 --profile-last > $O/p4_ncu.log 2>&1
ncu -i $O/p4.ncu-rep --page source --csv --print-source cuda > $O/p4_cuda.csv 2>&1
ncu -i $O/p4.ncu-rep --page details --csv > $O/p4_details.csv 2>&1
ncu -i $O/p4.ncu-rep --page raw --csv > $O/p4_raw.csv 2>&1
rm -f $O/p4.ncu-rep
ls -la $O | grep p4
