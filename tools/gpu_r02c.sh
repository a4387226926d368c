#!/bin/bash
# r02c evidence: default bench line (all legs), ncu launch list + full capture of the dominant kernel, phase shares
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
T=${1:-r02c}
timeout 1500 python bench.py > gpurun_out/${T}_bench_default.json 2> gpurun_out/${T}_bench_default.err; echo "bench exit $?"
tail -3 gpurun_out/${T}_bench_default.err
python - <<PY
import json
d=json.load(open('gpurun_out/${T}_bench_default.json'))
print('value', round(d['value']/1e6,1), 'M inst/s', round(d['ms_per_step'],1), 'ms; e2e', round(d['e2e']['value']/1e6,1), 'M; cpu', round(d['cpu_baseline']['value']/1e6,2), 'M; frac', round(d['roofline']['frac'],5))
o=d.get('e2e_objects'); print('objects', o and {k:(round(v) if isinstance(v,float) else v) for k,v in o.items() if k.endswith('_s') or k=='value'})
for c in d.get('configs') or []:
    print(' ', c['config'], round(c['value']/1e6,1), 'M inst/s', round(c['ms_per_step'],2), 'ms frac', round(c['roofline']['frac'],5), 'cpu', c.get('cpu_baseline') and round(c['cpu_baseline']['value']/1e6,2), [ (l['pass'][:12], round(l['value']/1e6,1)) for l in c.get('passes',[])])
PY
B="python bench.py --no-e2e --no-cpu --no-configs --no-objects --no-typeseed"
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/${T}_launches_default_mixed100M.csv $B --steps 1 --warmup 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_postssa_gtile -c 1 -o gpurun_out/${T}_ncu_gtile -f $B --steps 1 --warmup 0 > gpurun_out/${T}_ncu.log 2>&1
ncu -i gpurun_out/${T}_ncu_gtile.ncu-rep --page details > gpurun_out/${T}_ncu_full_k_postssa_gtile_details.txt
ncu -i gpurun_out/${T}_ncu_gtile.ncu-rep --page raw --csv > gpurun_out/${T}_ncu_full_k_postssa_gtile_raw.csv
grep -E "Duration|DRAM Throughput|Executed Ipc Active|No Eligible|Registers Per|Achieved Occupancy|Avg. Active Threads|L2 Hit" gpurun_out/${T}_ncu_full_k_postssa_gtile_details.txt
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/${T}_launches_long4M.csv $B --workload long --insts 4e6 --steps 1 --warmup 1 > /dev/null 2>&1
