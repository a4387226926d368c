#!/bin/bash
# per-phase cycle shares of the profile build (-DCL_PROFILE): tile path (mixed), per-function kernels on long blocks
mkdir -p gpurun_out
P=paper_2604_27486_b200/csrc/_prof/libculifter_prof.so
B="python bench.py --no-e2e --no-cpu --no-configs --no-objects --no-typeseed --steps 2 --warmup 3"
T=${1:-r02d}
CL_PROF=1 CL_LIB=$P $B --insts 30e6 > gpurun_out/${T}_prof_tile.json 2> gpurun_out/${T}_prof_tile.err
CL_PROF=1 CL_LIB=$P CL_TILE=0 $B --workload long --insts 4e6 > gpurun_out/${T}_prof_long_cta.json 2> gpurun_out/${T}_prof_long_cta.err
CL_PROF=1 CL_LIB=$P $B --workload long --insts 4e6 > gpurun_out/${T}_prof_long.json 2> gpurun_out/${T}_prof_long.err
grep -H phase gpurun_out/${T}_prof_*.err
python - <<PY
import json
for n in ('tile','long_cta','long'):
    d=json.load(open('gpurun_out/${T}_prof_%s.json'%n)); print(n, round(d['value']/1e6,1), 'M inst/s', round(d['ms_per_step'],2), 'ms', d['partition'])
PY
