#!/bin/bash
# A/B bench of env-var settings on one box:  tools/ab_env.sh "c2 c3" "TILECAST_CHAIN=0" "TILECAST_CHAIN=1"
cfgs=$1; shift
for rep in 1 2; do
for v in "$@"; do
  for c in $cfgs; do
    env $v timeout 300 python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', '$c', round(j['value']/1e6,1), round(j['roofline']['frac'],3), 'fused', round(j.get('rollout_fused',{}).get('value',0)/1e6,1), 'e2e', round(j['e2e']['value']/1e6,1))"
  done
done
done
