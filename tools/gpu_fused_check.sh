#!/bin/bash
# first GPU pass of the fused path: parity tests, then short benches with the phase clock
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests/test_fused.py -x -q -m gpu > gpurun_out/fused_tests.log 2>&1; echo "exit $?" >> gpurun_out/fused_tests.log
tail -15 gpurun_out/fused_tests.log
for w in mixed sm90 sm52 sm75; do
  CL_PROF=1 timeout 600 python bench.py --workload $w --insts 10e6 --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/fused_bench_${w}_10M.json 2> gpurun_out/fused_bench_${w}_10M.err
  tail -2 gpurun_out/fused_bench_${w}_10M.err; cut -c1-400 gpurun_out/fused_bench_${w}_10M.json
done
CL_PROF=1 timeout 900 python bench.py --workload mixed --insts 100e6 --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/fused_bench_mixed_100M.json 2> gpurun_out/fused_bench_mixed_100M.err
tail -2 gpurun_out/fused_bench_mixed_100M.err; cut -c1-600 gpurun_out/fused_bench_mixed_100M.json
