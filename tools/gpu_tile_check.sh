#!/bin/bash
# tile path after a change: its parity tests, then the per-workload comparison
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_tile.py tests/test_parity_gpu.py -x -q -m gpu > gpurun_out/tile_tests.log 2>&1; echo "exit $?" >> gpurun_out/tile_tests.log
tail -4 gpurun_out/tile_tests.log
for w in mixed sm90 sm52; do
    CL_PROF=1 timeout 600 python bench.py --workload $w --insts 10e6 --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/tile_${w}.json 2> gpurun_out/tile_${w}.err
    python -c "
import json; d=json.load(open('gpurun_out/tile_${w}.json')); print('$w', round(d['value']/1e6,1), 'M inst/s', round(d['ms_per_step'],2), 'ms', d['partition']['tile_mode'])"
done
timeout 900 python bench.py --workload mixed --insts 100e6 --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/tile_mixed100M.json 2> gpurun_out/tile_mixed100M.err
python -c "
import json; d=json.load(open('gpurun_out/tile_mixed100M.json')); print('mixed100M', round(d['value']/1e6,1), 'M inst/s', round(d['ms_per_step'],2), 'ms', d['partition'])"
