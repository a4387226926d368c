#!/bin/bash
# Run under gpurun: phase-cycle profile (needs libculifter_prof.so = -DCL_PROFILE build),
# ncu launch list of the bench command, one ncu --set full capture of the top kernel.
# usage: tools/gpu_profile.sh <tag> [insts]
tag=${1:-r01b}
insts=${2:-1e7}
mkdir -p gpurun_out
if [ -f paper_2604_27486_b200/csrc/libculifter_prof.so ]; then
  CL_LIB=$PWD/paper_2604_27486_b200/csrc/libculifter_prof.so CL_PROF=1 timeout 600 python bench.py --insts 3e7 --steps 2 --warmup 1 --no-e2e --no-cpu \
    > gpurun_out/${tag}_phases.log 2>&1
fi
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches.csv \
  python bench.py --insts $insts --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/${tag}_launches.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:${KERNEL:-k_postssa_gtile} -c 1 -f -o gpurun_out/${tag}_gtile \
  python bench.py --insts $insts --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/${tag}_full.log 2>&1
ncu -i gpurun_out/${tag}_gtile.ncu-rep --page raw --csv > gpurun_out/${tag}_gtile_raw.csv 2>/dev/null
ncu -i gpurun_out/${tag}_gtile.ncu-rep --page details > gpurun_out/${tag}_gtile_details.txt 2>/dev/null
ncu -i gpurun_out/${tag}_gtile.ncu-rep --page source --csv > gpurun_out/${tag}_gtile_source.csv 2>/dev/null
gzip -f gpurun_out/${tag}_gtile_source.csv
rm -f gpurun_out/${tag}_gtile.ncu-rep
tail -2 gpurun_out/${tag}_phases.log
head -40 gpurun_out/${tag}_launches.csv | cut -c1-200
