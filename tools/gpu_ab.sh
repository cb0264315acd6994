#!/bin/bash
# A/B of env settings on a few configs: bash tools/gpu_ab.sh "c4 c3" "PHIPM_RPT=8" "PHIPM_RPT=4"
cd "$(dirname "$0")/.."
CONFIGS=$1; shift
for envs in "$@"; do
  for c in $CONFIGS; do
    env $envs timeout 180 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$envs', '$c', round(d['value'],1), 'frac', round(d['roofline']['frac'],3), {k: round(v,3) for k,v in d.get('profile_ms_per_solve',{}).items()})"
  done
done
