#!/bin/bash
# k_typeseed: resident CTAs per SM asked of ptxas (TS_MINB 4/5/6/8 = 52/46/40/32 registers), libraries built into gpurun_tmp/
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm --format=csv,noheader
timeout 600 python -m pytest tests/test_typeseed.py -x -q -m gpu 2>&1 | tail -3
for mb in 4 5 6 8; do
  CL_LIB=$PWD/gpurun_tmp/libculifter_mb$mb.so timeout 600 python bench.py --only-typeseed --no-cpu --steps 10 --warmup 3 > gpurun_out/ts_mb$mb.json 2> gpurun_out/ts_mb$mb.err
  python -c "import json; d=json.load(open('gpurun_out/ts_mb$mb.json')); print('minb $mb', round(d['ms_per_step'],3), 'ms', round(d['value']/1e9,2), 'G inst/s frac', round(d['roofline']['frac'],4), 'e2e ms', round(d['e2e']['ms_per_step'],1))"
done
