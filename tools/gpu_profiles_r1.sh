#!/bin/bash
# Round-1 profiling evidence (each ncu command runs only after the same plain command exited 0).
cd "$(dirname "$0")/.."
O=gpurun_out
for c in c1 c2 c3 c4 c5; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 > $O/pf_bench_$c.json.log 2>&1
done
timeout 120 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/pf_plain_bench.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/pf_launches_c3.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/pf_ncu_launch.log 2>&1
for c in c3 c4 c5; do
  timeout 300 python tools/one_solve.py --config $c --solves 2 --profile-last > $O/pf_plain_$c.log 2>&1 && \
  timeout 900 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none --csv --log-file $O/pf_dram_$c.csv python tools/one_solve.py --config $c --solves 2 --profile-last \
    > $O/pf_ncu_dram_$c.log 2>&1
done
full() {  # config kernel-regex skip name
  timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 \
    -o $O/pf_full_$4 python tools/one_solve.py --config $1 --solves 2 --profile-last > $O/pf_ncu_full_$4.log 2>&1
}
full c3 spmv_stream 20 c3_spmv
full c3 axpy_stream 18 c3_axpy
full c5 spmv_stream 6 c5_spmv
full c3 expm_kernel 3 c3_expm
full c4 krylov_persist 0 c4_persist
full c1 krylov_small 10 c1_small
for c in c2 c3 c4 c5; do timeout 200 python tools/kclock.py $c > $O/kclock_$c.txt 2>&1; done
# summarise here and drop the raw reports: gpurun copies back at most 64 MiB of gpurun_out/
python tools/make_profiles.py round1 $O/round1_profiles > $O/make_profiles.log 2>&1
rm -f $O/*.ncu-rep $O/*.bin $O/*.bin.p
ls -la $O | tail -40
