#!/bin/bash
# last evidence of round 2 after the final k_typeseed: its tests / bench leg / captures, smoke, and the default bench line + reference arm
mkdir -p gpurun_out
T=${1:-r02k}
bash tools/gpu_typeseed.sh $T
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py --impl reference > gpurun_out/${T}_bench_reference.json 2> gpurun_out/${T}_bench_reference.err; echo "reference arm exit $?"
timeout 1500 python bench.py > gpurun_out/${T}_bench_default.json 2> gpurun_out/${T}_bench_default.err; echo "bench exit $?"
python - <<PY
import json
d=json.load(open('gpurun_out/${T}_bench_default.json'))
print('value', round(d['value']/1e6,1), 'M inst/s', round(d['ms_per_step'],1), 'ms; e2e', round(d['e2e']['value']/1e6,1), 'M; cpu', round(d['cpu_baseline']['value']/1e6,2), 'M; frac', round(d['roofline']['frac'],5), 'launches', d['gpu_launches'], d['clocks'])
t=d['typeseed']; print('typeseed', round(t['ms_per_step'],3), 'ms', round(t['value']/1e9,2), 'G inst/s frac', round(t['roofline']['frac'],4), 'traffic', t['roofline']['traffic'], 'e2e ms', round(t['e2e']['ms_per_step'],1), t['equal_to_oracle'])
PY
du -sh gpurun_out
