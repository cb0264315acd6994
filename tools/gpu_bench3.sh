python -c "import paper_0907_4631_b200 as P; P.build()"
for c in c3 c4 c5; do timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --config $c > gpurun_out/b3_$c.log 2>&1; done
PHIPM_PDL=0 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --config c3 > gpurun_out/b3_c3_nopdl.log 2>&1
for f in gpurun_out/b3_c3.log gpurun_out/b3_c3_nopdl.log gpurun_out/b3_c4.log gpurun_out/b3_c5.log; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', round(d['value'],1), 'profiled', round(d['profiled_region']['value'],1), 'e2e', round(d['e2e']['value'],1), 'roof', d['roofline']['kernel'], round(d['roofline']['frac'],3), 'arnoldi', round(d['arnoldi_step']['achieved_gbs']), 'launches', d['gpu_launches'])
" || tail -3 $f; done
