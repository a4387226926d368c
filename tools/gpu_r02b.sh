#!/bin/bash
# r02b: per-phase cycle shares (profile build), launch list + full ncu capture of the dominant kernel at the bench's corpus size
mkdir -p gpurun_out
P=paper_2604_27486_b200/csrc/_prof/libculifter_prof.so
B="python bench.py --no-e2e --no-cpu --no-configs --steps 2 --warmup 3"
CL_LIB=$P $B --insts 30e6 > gpurun_out/r02b_prof_tile.json 2> gpurun_out/r02b_prof_tile.err
CL_LIB=$P CL_FUSED=1 $B --insts 30e6 > gpurun_out/r02b_prof_fused.json 2> gpurun_out/r02b_prof_fused.err
CL_LIB=$P $B --workload long --insts 4e6 > gpurun_out/r02b_prof_long.json 2> gpurun_out/r02b_prof_long.err
grep phase gpurun_out/r02b_prof_*.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r02b_launches_default_mixed100M.csv $B --steps 1 --warmup 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_postssa_gtile -c 1 -o gpurun_out/r02b_ncu_gtile -f $B --steps 1 --warmup 0 > gpurun_out/r02b_ncu.log 2>&1
ncu -i gpurun_out/r02b_ncu_gtile.ncu-rep --page details > gpurun_out/r02b_ncu_full_k_postssa_gtile_details.txt
ncu -i gpurun_out/r02b_ncu_gtile.ncu-rep --page raw --csv > gpurun_out/r02b_ncu_full_k_postssa_gtile_raw.csv
tail -3 gpurun_out/r02b_ncu.log
