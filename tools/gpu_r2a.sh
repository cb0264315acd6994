#!/bin/bash
# round-2 first GPU pass: full gpu tests, c5 bench line, c1..c4 quick lines
cd "$(dirname "$0")/.."
python -c "import paper_0907_4631_b200 as P; P.build()" 
timeout 1200 python -m pytest tests/ -q -m gpu -p no:cacheprovider -rf 2>&1 | tail -25 > gpurun_out/r2a_tests.txt
cat gpurun_out/r2a_tests.txt
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/r2a_bench_c5.json 2> gpurun_out/r2a_bench_c5.err
tail -c 3000 gpurun_out/r2a_bench_c5.json
for c in c1 c2 c3 c4; do
  timeout 200 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r2a_bench_$c.json 2>&1
  tail -1 gpurun_out/r2a_bench_$c.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['value'],1), 'frac', round(d['roofline']['frac'],3), 'solve_gbs', round(d['solve_algorithmic_gbs']))" 2>&1 | tail -1
done
