cd /root/repo
python -c "import paper_0907_4631_b200 as P; P.build()"
timeout 600 python -m pytest tests/test_gpu_solve.py -q -m gpu -p no:cacheprovider -k "deferred or graph or trajectory or stats" 2>&1 | tail -4
for c in c5 c3; do
timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/dfr_$c.json 2>gpurun_out/dfr_$c.err
python -c "import json; d=json.loads(open('gpurun_out/dfr_$c.json').read().strip().splitlines()[-1]); print('$c', round(d['value'],1), 'frac', round(d['roofline']['frac'],4), round(d['roofline']['avg_launch_us'],2), {k: round(v,4) for k,v in d.get('profile_ms_per_solve',{}).items()})"
done
for c in c5 c3; do timeout 300 python tools/ab_opts.py --config $c defer=1 defer=0 2>&1 | tail -4; done
