#!/bin/bash
# pinned H2D / D2H bandwidth of the box next to the stage times of the e2e pipeline (CL_TRACE=1)
mkdir -p gpurun_out
python - <<'PY' > gpurun_out/pcie_probe.txt 2>&1
import torch, time
n = 1 << 30
h = torch.empty(n, dtype=torch.uint8).pin_memory(); d = torch.empty(n, dtype=torch.uint8, device="cuda")
for name, src, dst in (("H2D", h, d), ("D2H", d, h)):
    for _ in range(2): dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(5): dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(name, "GB/s", 5 * n / dt / 1e9)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream(); h2 = torch.empty(n, dtype=torch.uint8).pin_memory(); d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(5):
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t
print("both directions at once, GB/s per direction", 5 * n / dt / 1e9)
PY
cat gpurun_out/pcie_probe.txt
CL_TRACE=1 python bench.py --no-cpu --no-configs --no-objects --no-typeseed --steps 3 --warmup 3 > gpurun_out/e2e_trace.json 2> gpurun_out/e2e_trace.err
grep chunk gpurun_out/e2e_trace.err | tail -16
python -c "
import json; d=json.load(open('gpurun_out/e2e_trace.json')); print(d['value']/1e6, d['e2e'])"
