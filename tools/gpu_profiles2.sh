python -c "import paper_0907_4631_b200 as P; P.build()"
timeout 300 python tools/one_solve.py --config c3 --solves 2 > gpurun_out/pf_plain_c3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_stream -s 75 -c 1 -o gpurun_out/pf_full_c3_spmv python tools/one_solve.py --config c3 --solves 2 > gpurun_out/pf_ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:axpy_stream -s 75 -c 1 -o gpurun_out/pf_full_c3_axpy python tools/one_solve.py --config c3 --solves 2 > gpurun_out/pf_ncu_full2.log 2>&1
ls -la gpurun_out/pf_full*
