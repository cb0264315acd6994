#!/bin/bash
# Round-2 profiling evidence (each ncu command runs only after the same plain command exited 0).
cd "$(dirname "$0")/.."
O=gpurun_out
python -c "import paper_0907_4631_b200 as P; P.build()"
for c in c5 c1 c2 c3 c4; do
  timeout 400 python bench.py --config $c --steps 20 --warmup 3 > $O/pf_bench_$c.json.log 2>&1
done
timeout 200 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/pf_plain_bench.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/pf_launches_c5.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/pf_ncu_launch.log 2>&1
timeout 200 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline > $O/pf_plain_bench_c2.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/pf_launches_c2.csv \
  python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline > $O/pf_ncu_launch_c2.log 2>&1
timeout 200 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline > $O/pf_plain_bench_c4.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/pf_launches_c4.csv \
  python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline > $O/pf_ncu_launch_c4.log 2>&1
for c in c2 c3 c4 c5; do
  timeout 300 python tools/one_solve.py --config $c --solves 2 --profile-last > $O/pf_plain_$c.log 2>&1 && \
  timeout 900 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none --csv --log-file $O/pf_dram_$c.csv python tools/one_solve.py --config $c --solves 2 --profile-last \
    > $O/pf_ncu_dram_$c.log 2>&1
done
full() {  # config kernel-regex skip name [extra one_solve args]
  timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 \
    -o $O/pf_full_$4 python tools/one_solve.py --config $1 --solves 2 --profile-last $5 > $O/pf_ncu_full_$4.log 2>&1
}
full c5 spmv_stream 6 c5_spmv
full c5 axpy_stream 4 c5_axpy
full c5 csr_analyze 0 c5_analyze
full c4 krylov_persist_tm 0 c4_persist "--option brick=0"
full c4 krylov_brick 0 c4_brick
full c4 wrec_brick 0 c4_wrec_brick
full c1 phi_cheb 3 c1_cheb "--expm 2"
full c2 krylov_cluster 0 c2_cluster
full c2 expm_kernel 3 c2_expm
for c in c4 c5; do timeout 200 python tools/kclock.py $c > $O/kclock_$c.txt 2>&1; done
python tools/make_profiles.py round2 $O/round2_profiles > $O/make_profiles.log 2>&1
rm -f $O/*.ncu-rep $O/*.bin $O/*.bin.p
ls $O/round2_profiles
