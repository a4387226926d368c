#!/bin/bash
# device-resident throughput of the tile path vs the fused path per workload
mkdir -p gpurun_out
for w in mixed sm90 sm75 sm52 long; do
  for fz in 0 1; do
    CL_FUSED=$fz timeout 600 python bench.py --workload $w --insts ${1:-10e6} --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/cmp_${w}_$fz.json 2> gpurun_out/cmp_${w}_$fz.err
    python -c "
import json; d=json.load(open('gpurun_out/cmp_${w}_$fz.json')); print('$w fused=$fz', round(d['value']/1e6,1), 'M inst/s', round(d['ms_per_step'],2), 'ms', d['partition'])"
  done
done
