#!/bin/bash
# one full ncu capture of the fused class-S kernel (mixed 10M), details page as text
mkdir -p gpurun_out
W=${1:-mixed}; N=${2:-10e6}; K=${3:-S}; SKIP=3; [ "$K" = L ] && SKIP=4; [ "$K" = X ] && SKIP=5
timeout 1200 ncu --set full --import-source on --clock-control none -k k_fused -s $SKIP -c 1 -o gpurun_out/fused_ncu_$K -f python bench.py --workload $W --insts $N --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/fused_ncu.log 2>&1
ncu -i gpurun_out/fused_ncu_$K.ncu-rep --page details > gpurun_out/fused_ncu_${K}_details.txt 2>&1
ncu -i gpurun_out/fused_ncu_$K.ncu-rep --page raw --csv > gpurun_out/fused_ncu_${K}_raw.csv 2>&1
grep -E "Duration|Executed Ipc|No Eligible|Issue Slots Busy|One or More Eligible|Registers Per|Achieved Occupancy|Theoretical Occ|DRAM Throughput|Avg. Active Threads|L1/TEX Hit|L2 Hit|Local|Stall|stall" gpurun_out/fused_ncu_${K}_details.txt | head -40
