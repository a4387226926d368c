#!/bin/bash
# quick A/B runs of tuning knobs (device-resident throughput only): "name:ENV=..:bench args" per line in $EXPS
mkdir -p gpurun_out
B="python bench.py --no-e2e --no-cpu --no-configs --steps 3 --warmup 3"
while IFS= read -r cfg; do
  [ -z "$cfg" ] && continue
  IFS=: read name envs args <<< "$cfg"
  env $envs $B $args > gpurun_out/exp_$name.json 2> gpurun_out/exp_$name.err
  python - <<PY
import json
try:
    d=json.load(open('gpurun_out/exp_$name.json')); print('$name', round(d['value']/1e6,1), 'M inst/s', round(d['ms_per_step'],2), 'ms', d['partition'], d['match_counts']['selected'])
except Exception as e: print('$name failed', e)
PY
done <<< "$EXPS"
[ -n "$TESTS" ] && timeout 1500 python -m pytest $TESTS -x -q -m gpu 2>&1 | tail -3
true
