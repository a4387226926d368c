#!/bin/bash
# k_typeseed build variants (libraries built into gpurun_tmp/ as libculifter_<name>.so): bench leg of each
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm --format=csv,noheader
timeout 600 python -m pytest tests/test_typeseed.py -x -q -m gpu 2>&1 | tail -3
for lib in gpurun_tmp/libculifter_*.so; do
  name=$(basename $lib .so); name=${name#libculifter_}
  CL_LIB=$PWD/$lib timeout 600 python bench.py --only-typeseed --steps 10 --warmup 3 > gpurun_out/ts_$name.json 2> gpurun_out/ts_$name.err
  python -c "import json; d=json.load(open('gpurun_out/ts_$name.json')); print('$name', round(d['ms_per_step'],3), 'ms', round(d['value']/1e9,2), 'G inst/s frac', round(d['roofline']['frac'],4), 'e2e ms', round(d['e2e']['ms_per_step'],1), d.get('equal_to_oracle'))"
done
