python -c "import paper_0907_4631_b200 as P; P.build()"
for c in c1 c2 c3 c4 c5; do timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --config $c > gpurun_out/ball_$c.log 2>&1; done
for c in c1 c2 c3 c4 c5; do python -c "
import json
d=json.loads(open('gpurun_out/ball_$c.log').read().strip().splitlines()[-1])
print('$c', round(d['value'],1), 'solves/s', round(d['ms_per_step'],3),'ms', 'prof', {k: round(v,3) for k,v in d['profile_ms_per_solve'].items()}, 'stats', d['stats'], 'launches', d['gpu_launches'], 'e2e', round(d['e2e']['value'],1))
" || tail -3 gpurun_out/ball_$c.log; done
