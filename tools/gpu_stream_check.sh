#!/bin/bash
# quick GPU loop for the streaming path: parity tests, then the per-phase clock on the mixed corpus
timeout 900 python -m pytest tests/test_stream.py tests/test_parity_gpu.py -m gpu -x -q 2>&1 | tail -4
for w in ${WORKLOADS:-mixed}; do
  CL_PROF=1 timeout 600 python bench.py --workload $w --insts ${INSTS:-1e7} --steps 2 --warmup 1 --no-e2e --no-cpu 2>&1 | grep -E "stream phases|value" | cut -c1-${CUT:-700}
done
