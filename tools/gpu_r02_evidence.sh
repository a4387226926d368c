#!/bin/bash
# round-2 evidence: GPU test suite, default bench line, ncu launch list + full capture of the dominant kernel
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
if [ "$1" != "notest" ]; then
timeout 3000 python -m pytest tests -x -q -m gpu > gpurun_out/r02_gpu_tests.log 2>&1; echo "exit $?" >> gpurun_out/r02_gpu_tests.log
tail -4 gpurun_out/r02_gpu_tests.log
fi
timeout 1500 python bench.py > gpurun_out/r02_bench_default.json 2> gpurun_out/r02_bench_default.err; echo "bench exit $?"
tail -3 gpurun_out/r02_bench_default.err
python - <<'PY'
import json
d=json.load(open('gpurun_out/r02_bench_default.json'))
print('value', round(d['value']/1e6,1), 'M inst/s', round(d['ms_per_step'],1), 'ms; e2e', round(d['e2e']['value']/1e6,1), 'M; cpu', round(d['cpu_baseline']['value']/1e6,2), 'M; frac', round(d['roofline']['frac'],5))
for c in d.get('configs') or []:
    print(' ', c['config'], round(c['value']/1e6,1), 'M inst/s', round(c['ms_per_step'],2), 'ms frac', round(c['roofline']['frac'],5), 'cpu', c.get('cpu_baseline') and round(c['cpu_baseline']['value']/1e6,2), [ (l['pass'][:12], round(l['value']/1e6,1)) for l in c.get('passes',[])])
PY
