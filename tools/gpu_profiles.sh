# Round profiling evidence (run after the plain commands exit 0)
python -c "import paper_0907_4631_b200 as P; P.build()"
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/pf_plain_bench.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pf_launches_c3.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/pf_ncu_launch.log 2>&1
timeout 300 python tools/one_solve.py --config c3 --solves 2 > gpurun_out/pf_plain_c3.log 2>&1 && \
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"spmv_stream|axpy_stream|expm" -s 120 --csv --log-file gpurun_out/pf_dram_c3.csv python tools/one_solve.py --config c3 --solves 2 > gpurun_out/pf_ncu_dram.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_stream -s 100 -c 1 -o gpurun_out/pf_full_c3_spmv python tools/one_solve.py --config c3 --solves 2 > gpurun_out/pf_ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:axpy_stream -s 100 -c 1 -o gpurun_out/pf_full_c3_axpy python tools/one_solve.py --config c3 --solves 2 > gpurun_out/pf_ncu_full2.log 2>&1
ls -la gpurun_out/pf_*
