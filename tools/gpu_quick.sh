# quick cycle: gpu tests (fail fast) + per-launch trace of c3/c4/c5 + bench c3
python -c "import paper_0907_4631_b200 as P; P.build()"
timeout 900 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider -x 2>&1 | tail -4 > gpurun_out/q_tests.log
python tools/trace_solve.py --configs ${CONFIGS:-c3,c4,c5} > gpurun_out/q_trace.txt 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/q_bench.log 2>&1
cat gpurun_out/q_tests.log; grep -v "^    " gpurun_out/q_trace.txt
python -c "
import json
d=json.loads(open('gpurun_out/q_bench.log').read().strip().splitlines()[-1])
print('bench c3', round(d['value'],1), 'solves/s e2e', round(d['e2e']['value'],1), 'roof', d['roofline']['kernel'], round(d['roofline']['achieved']), round(d['roofline']['frac'],3), 'arnoldi', round(d['arnoldi_step']['achieved_gbs']), {k: round(v,3) for k,v in d['profile_ms_per_solve'].items()}, 'clk', d['clocks'])
" || tail -5 gpurun_out/q_bench.log
