#!/bin/bash
# A/B environment toggles on the default bench (no cpu baseline / e2e)
for e in "$@"; do
  for rep in 1 2; do
    echo "env: $e"
    env $e python bench.py --steps 1000 --warmup 20 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,2), 'M samples/s', round(d['ms_per_step']*1e3,1), 'us', d['clocks']['sm_mhz'], d['clocks']['reasons'], {k:v for k,v in d['roofline']['phases'].items() if k!='source'})"
  done
done
