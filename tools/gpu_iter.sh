#!/bin/bash
# One GPU iteration: full gpu tests, c3 in-kernel timeline, short bench of every config.
# usage (under gpurun): bash tools/gpu_iter.sh TAG
TAG=${1:-iter}
cd "$(dirname "$0")/.."
timeout 300 python -m pytest tests/ -q -m gpu -x -p no:cacheprovider 2>&1 | tail -3
timeout 120 python tools/kclock.py c3 > gpurun_out/kclock_c3_$TAG.txt 2>&1
for c in c1 c2 c3 c4 c5; do
  timeout 180 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_$c.log 2>&1
  tail -1 gpurun_out/bench_${TAG}_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['value'],1), d['unit'], 'frac', d['roofline']['frac'], {k: round(v,3) for k,v in d.get('profile_ms_per_solve',{}).items()})" 2>&1 | tail -1
done
