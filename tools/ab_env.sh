#!/bin/bash
# A/B an engine env knob on the headline bench: tools/ab_env.sh VAR "v1 v2" [rounds] [bench args...]
var=$1; vals=$2; rounds=${3:-3}; shift 3
for i in $(seq $rounds); do
  for v in $vals; do
    env $var=$v timeout 300 python bench.py --no-cpu --no-extra --no-e2e "$@" 2>/dev/null |
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$var=$v', round(d['value']), round(d['roofline']['avg_launch_ms']*1e3,2), d['clocks']['sm_mhz'])"
  done
done
