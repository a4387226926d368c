#!/bin/bash
# Final evidence of a round, under gpurun: ncu launch list of the default bench command (small step count),
# one ncu --set full capture of the dominant kernel at the bench's own corpus size, csv/text exports only.
# usage: tools/gpu_final_profile.sh <tag> <kernel regex> [insts]
tag=$1; kern=$2; insts=${3:-1e8}
mkdir -p gpurun_out
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/${tag}_launches.csv \
  python bench.py --insts $insts --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/${tag}_launches.log 2>&1
timeout 2400 ncu --set full --clock-control none --import-source on -k regex:$kern -c 1 -f -o gpurun_out/${tag}_full \
  python bench.py --insts $insts --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/${tag}_full.log 2>&1
ncu -i gpurun_out/${tag}_full.ncu-rep --page raw --csv > gpurun_out/${tag}_full_raw.csv 2>/dev/null
ncu -i gpurun_out/${tag}_full.ncu-rep --page details > gpurun_out/${tag}_full_details.txt 2>/dev/null
ncu -i gpurun_out/${tag}_full.ncu-rep --page source --csv 2>/dev/null | gzip > gpurun_out/${tag}_full_source.csv.gz
rm -f gpurun_out/${tag}_full.ncu-rep
grep -E "Duration|DRAM Throughput|Executed Ipc Active|Achieved Occupancy|Registers Per" gpurun_out/${tag}_full_details.txt | head
