#!/bin/bash
# A/B helper: one bench line summary per (workload, env) pair.
#   tools/ab_bench.sh "config3 config2" "X=1" "DGX_NOFOLD=1" ...
cfgs=$1; shift
for cfg in $cfgs; do
  for envv in "$@"; do
    echo -n "== $cfg $envv :: "
    env $envv timeout 600 python bench.py --workload $cfg --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | \
      python -c "import json,sys
t=sys.stdin.read()
try:
  d=json.loads(t); print(round(d['value']), {k:(round(v['avg_launch_ms'],3), v['launches']) for k,v in d['roofline']['kernels'].items()}, round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])
except Exception: print('FAILED', t[-300:])"
  done
done
