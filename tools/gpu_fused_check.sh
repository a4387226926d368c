#!/bin/bash
# GPU pass of the fused path: parity tests, then short benches with the phase clock and a launch list
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
if [ "$1" != "notest" ]; then
timeout 1500 python -m pytest tests/test_fused.py -x -q -m gpu > gpurun_out/fused_tests.log 2>&1; echo "exit $?" >> gpurun_out/fused_tests.log
tail -5 gpurun_out/fused_tests.log
fi
for w in mixed sm90 sm52; do
  CL_PROF=1 timeout 600 python bench.py --workload $w --insts 10e6 --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/fused_bench_${w}_10M.json 2> gpurun_out/fused_bench_${w}_10M.err
  tail -1 gpurun_out/fused_bench_${w}_10M.err; python -c "
import json,sys; d=json.load(open('gpurun_out/fused_bench_${w}_10M.json')); print('$w', round(d['value']/1e6,1), 'M inst/s', round(d['ms_per_step'],2), 'ms', d['partition'].get('handed_back'))"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/fused_launches_mixed10M.csv python bench.py --workload mixed --insts 10e6 --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/fused_launches_mixed10M.csv')) if len(r)>10]
hdr=rows[0]; ki=hdr.index('Kernel Name'); vi=hdr.index('Metric Value')
for r in rows[1:]:
    print(r[ki][:70], r[vi])
PY
CL_PROF=1 timeout 900 python bench.py --workload mixed --insts 100e6 --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/fused_bench_mixed_100M.json 2> gpurun_out/fused_bench_mixed_100M.err
tail -1 gpurun_out/fused_bench_mixed_100M.err; python -c "
import json,sys; d=json.load(open('gpurun_out/fused_bench_mixed_100M.json')); print('mixed100M', round(d['value']/1e6,1), 'M inst/s', round(d['ms_per_step'],2), 'ms', d['partition'].get('handed_back'))"
