python -c "import paper_0907_4631_b200 as P; P.build()"
python tools/one_solve.py --config c3 --solves 2 > gpurun_out/plain_c3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:expm -s 11 -c 1 -o gpurun_out/prof3_c3_expm python tools/one_solve.py --config c3 --solves 2 > gpurun_out/ncu3a.log 2>&1; \
ncu --set full --clock-control none --import-source on -k regex:spmv_stream -s 80 -c 1 -o gpurun_out/prof3_c3_spmv python tools/one_solve.py --config c3 --solves 2 > gpurun_out/ncu3b.log 2>&1
python tools/one_solve.py --config c5 --solves 2 > gpurun_out/plain_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:spmv_stream -s 12 -c 1 -o gpurun_out/prof3_c5_spmv python tools/one_solve.py --config c5 --solves 2 > gpurun_out/ncu3c.log 2>&1
python tools/one_solve.py --config c4 --solves 2 > gpurun_out/plain_c4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:spmv_stream -s 12 -c 1 -o gpurun_out/prof3_c4_spmv python tools/one_solve.py --config c4 --solves 2 > gpurun_out/ncu3d.log 2>&1
ls gpurun_out/prof3*
