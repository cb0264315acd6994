python -c "import paper_0907_4631_b200 as P; P.build()"
timeout 900 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider -x 2>&1 | tail -4
for c in c1 c2; do timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --config $c > gpurun_out/bs_$c.log 2>&1; python -c "
import json
d=json.loads(open('gpurun_out/bs_$c.log').read().strip().splitlines()[-1])
print('$c', round(d['value'],1), 'solves/s', round(d['ms_per_step'],3),'ms', 'prof', {k: round(v,3) for k,v in d['profile_ms_per_solve'].items()}, 'launches', d['gpu_launches'])
" || tail -3 gpurun_out/bs_$c.log; done
