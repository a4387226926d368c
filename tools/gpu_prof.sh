#!/bin/bash
# per-phase cycle shares of the profile build (-DCL_PROFILE): tile path, fused path, long-block kernels
mkdir -p gpurun_out
P=paper_2604_27486_b200/csrc/_prof/libculifter_prof.so
B="python bench.py --no-e2e --no-cpu --no-configs --steps 2 --warmup 3"
T=${1:-r02b}
CL_PROF=1 CL_LIB=$P $B --insts 30e6 > gpurun_out/${T}_prof_tile.json 2> gpurun_out/${T}_prof_tile.err
CL_PROF=1 CL_LIB=$P CL_FUSED=1 $B --insts 30e6 > gpurun_out/${T}_prof_fused.json 2> gpurun_out/${T}_prof_fused.err
CL_PROF=1 CL_LIB=$P $B --workload long --insts 4e6 > gpurun_out/${T}_prof_long.json 2> gpurun_out/${T}_prof_long.err
grep -H phase gpurun_out/${T}_prof_*.err
