python -c "import paper_0907_4631_b200 as P; P.build()"
python tools/one_solve.py --config c3 --solves 2 > gpurun_out/plain_c3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:spmv_fused -s 60 -c 2 -o gpurun_out/prof_c3_spmv python tools/one_solve.py --config c3 --solves 2 > gpurun_out/ncu_c3a.log 2>&1; \
ncu --set full --clock-control none --import-source on -k regex:axpy_fused -s 60 -c 2 -o gpurun_out/prof_c3_axpy python tools/one_solve.py --config c3 --solves 2 > gpurun_out/ncu_c3b.log 2>&1; \
ncu --set full --clock-control none --import-source on -k regex:expm -s 3 -c 1 -o gpurun_out/prof_c3_expm python tools/one_solve.py --config c3 --solves 2 > gpurun_out/ncu_c3c.log 2>&1
python tools/one_solve.py --config c5 --solves 2 > gpurun_out/plain_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:spmv_fused -s 20 -c 2 -o gpurun_out/prof_c5_spmv python tools/one_solve.py --config c5 --solves 2 > gpurun_out/ncu_c5.log 2>&1
ls -la gpurun_out/
