#!/bin/bash
# build the library; only when that worked, run the given command on the GPU box
set -e
python __graft_entry__.py 2>&1 | grep -v "deprecated-gpu-targets" | tail -5
test paper_2604_27486_b200/csrc/libculifter.so -nt paper_2604_27486_b200/csrc/fused.cuh || { echo "BUILD FAILED (library older than fused.cuh)"; exit 1; }
/usr/local/graft/bin/gpurun --timeout ${TIMEOUT:-2400} -- "$@"
