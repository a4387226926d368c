"""Where the end-to-end time goes: per-call wall time of cl_upload / cl_run_postssa / cl_download
for the whole corpus and for one chunk (pinned host buffers).  usage: e2e_breakdown.py [insts] [chunks]"""
import sys, time
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch
import bench
from paper_2604_27486_b200.capi import Engine
from paper_2604_27486_b200.sharding import materialize, plan_shards

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000_000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 8
kinds, pools, kid, pick, ns, nb, shard = plan_shards("mixed", n, 100, 1)
corpus = materialize(kinds, pools, kid, pick, np.arange(len(kid)))
ranges = corpus.split(k)
for label, c in (("whole", corpus), (f"chunk 1/{k}", corpus.slice_funcs(*ranges[0]))):
    host = bench.pinned_like(c)
    eng = Engine()
    eng.upload(host); eng.run_postssa(); out = eng.download()
    holder = bench.pinned_like(out); holder.events = bench.pinned_like_array(np.zeros(len(out.events) + 16, out.events.dtype))
    del out
    for rep in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        eng.upload(host); t1 = time.perf_counter()
        eng.run_postssa(); t2 = time.perf_counter()
        eng.download(holder); t3 = time.perf_counter()
    print(f"{label}: {c.n_insts} records, in {host.nbytes()/1e9:.2f} GB; upload {1e3*(t1-t0):.1f} ms "
          f"({host.nbytes()/1e9/(t1-t0):.1f} GB/s), run {1e3*(t2-t1):.1f} ms (device {eng.last_run_ms():.1f}), "
          f"download {1e3*(t3-t2):.1f} ms ({holder.nbytes()/1e9/(t3-t2):.1f} GB/s)")
    eng.close()
