python -c "import paper_0907_4631_b200 as P; P.build()"
timeout 120 python tools/one_solve.py --config c3_mini --solves 1 > gpurun_out/t14_first.log 2>&1; echo first rc=$? >> gpurun_out/t14_first.log
timeout 900 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider -x 2>&1 | tail -30 > gpurun_out/gpu_tests14.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench14_c3.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --config c5 --no-cpu-baseline > gpurun_out/bench14_c5.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --config c4 --no-cpu-baseline > gpurun_out/bench14_c4.log 2>&1
cat gpurun_out/t14_first.log; tail -4 gpurun_out/gpu_tests14.log
for c in c3 c5 c4; do python -c "
import json,sys
d=json.loads(open('gpurun_out/bench14_$c.log').read().strip().splitlines()[-1])
print('$c', round(d['value'],1), 'solves/s', 'roof', d['roofline']['kernel'], round(d['roofline']['achieved']), round(d['roofline']['frac'],3), 'arnoldi', round(d['arnoldi_step']['achieved_gbs']), d['profile_ms_per_solve'])
" || tail -5 gpurun_out/bench14_$c.log; done
