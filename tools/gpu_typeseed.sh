#!/bin/bash
# type seeding on the GPU: parity tests, its bench leg, ncu launch list + full capture of k_typeseed
mkdir -p gpurun_out
T=${1:-r02j}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests/test_typeseed.py -x -q -m gpu > gpurun_out/${T}_typeseed_tests.log 2>&1; echo "exit $?" >> gpurun_out/${T}_typeseed_tests.log
tail -5 gpurun_out/${T}_typeseed_tests.log
timeout 900 python bench.py --only-typeseed --steps 5 --warmup 3 > gpurun_out/${T}_bench_typeseed.json 2> gpurun_out/${T}_bench_typeseed.err; echo "bench exit $?"
tail -3 gpurun_out/${T}_bench_typeseed.err; cat gpurun_out/${T}_bench_typeseed.json
B="python bench.py --only-typeseed --no-cpu"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_typeseed -c 20 --csv --log-file gpurun_out/${T}_launches_typeseed.csv $B --steps 2 --warmup 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:^k_typeseed$ -c 1 -o gpurun_out/${T}_ncu_typeseed -f $B --steps 1 --warmup 0 > gpurun_out/${T}_ncu_typeseed.log 2>&1
ncu -i gpurun_out/${T}_ncu_typeseed.ncu-rep --page details > gpurun_out/${T}_ncu_full_k_typeseed_details.txt
ncu -i gpurun_out/${T}_ncu_typeseed.ncu-rep --page raw --csv > gpurun_out/${T}_ncu_full_k_typeseed_raw.csv
grep -E "Duration|DRAM Throughput|Memory Throughput|Executed Ipc Active|No Eligible|Registers Per|Achieved Occupancy|Avg. Active Threads|L2 Hit" gpurun_out/${T}_ncu_full_k_typeseed_details.txt

ncu -i gpurun_out/${T}_ncu_typeseed.ncu-rep --page source --csv > gpurun_out/${T}_ncu_full_k_typeseed_source.csv 2>/dev/null
rm -f gpurun_out/${T}_ncu_typeseed.ncu-rep
du -sh gpurun_out
