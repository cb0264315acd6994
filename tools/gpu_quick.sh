#!/bin/bash
# Quick GPU iteration: gpu tests (optional), bench lines of the given configs, c4 persistent-kernel timeline.
# usage (under gpurun): bash tools/gpu_quick.sh TAG "c2 c4" [notests]
TAG=${1:-q}; CFGS=${2:-"c2 c3 c4"}
cd "$(dirname "$0")/.."
[ "$3" != "notests" ] && timeout 300 python -m pytest tests/ -q -m gpu -x -p no:cacheprovider 2>&1 | tail -3
for c in $CFGS; do
  timeout 180 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_$c.log 2>&1
  tail -1 gpurun_out/bench_${TAG}_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); m=d.get('arnoldi_microbench',{}); print('$c', round(d['value'],1), d['unit'], 'frac', round(d['roofline']['frac'],3), 'micro', round(m.get('achieved_gbs',0)), {k: round(v,3) for k,v in d.get('profile_ms_per_solve',{}).items()})" 2>&1 | tail -1
done
timeout 120 python tools/kclock.py c4 > gpurun_out/kclock_c4_$TAG.txt 2>&1; tail -8 gpurun_out/kclock_c4_$TAG.txt
