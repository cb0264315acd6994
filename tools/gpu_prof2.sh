python -c "import paper_0907_4631_b200 as P; P.build()"
python tools/one_solve.py --config c3 --solves 2 > gpurun_out/plain_c3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:axpy_stream -s 40 -c 1 -o gpurun_out/prof2_c3_axpy python tools/one_solve.py --config c3 --solves 2 > gpurun_out/ncu2a.log 2>&1; \
ncu --set full --clock-control none --import-source on -k regex:spmv_stream -s 40 -c 1 -o gpurun_out/prof2_c3_spmv python tools/one_solve.py --config c3 --solves 2 > gpurun_out/ncu2b.log 2>&1
python tools/one_solve.py --config c5 --solves 2 > gpurun_out/plain_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:spmv_stream -s 12 -c 1 -o gpurun_out/prof2_c5_spmv python tools/one_solve.py --config c5 --solves 2 > gpurun_out/ncu2c.log 2>&1
ls -la gpurun_out/prof2*
