python -c "import paper_0907_4631_b200 as P; P.build()"
python tools/one_solve.py --config c5 --solves 1 > gpurun_out/csr_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:spmv_stream -s 5 -c 1 -o gpurun_out/prof_csr_nowin python tools/one_solve.py --config c5 --solves 1 > gpurun_out/csr_ncu1.log 2>&1
PHIPM_CSR_WINDOW=1 python tools/one_solve.py --config c5 --solves 1 > gpurun_out/csr_plain2.log 2>&1 && \
PHIPM_CSR_WINDOW=1 ncu --set full --clock-control none --import-source on -k regex:spmv_stream -s 5 -c 1 -o gpurun_out/prof_csr_win python tools/one_solve.py --config c5 --solves 1 > gpurun_out/csr_ncu2.log 2>&1
ls gpurun_out/prof_csr*
