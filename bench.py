#!/usr/bin/env python
"""bench.py -- lifted SASS instructions / second of the normalisation +
pattern-aggregation path (BASELINE.json metric) on N B200s.

A "step" is one pass of the whole post-SSA stage (normalize_xmad,
normalize_reciprocal, apply_aggregations, tag_cuda_objects) over this rank's
shard of the synthetic mixed-architecture corpus (BASELINE.json configs[4]:
40 % sm90 / 40 % sm75 / 20 % sm52 kernels plus long-block kernels).  The
corpus is fixed (strong scaling): kernels are partitioned across ranks by
LPT on instruction records, no data crosses ranks, and each step ends with an
NCCL allgather of the per-pattern match counters.

  value        device-resident: input already in HBM, CUDA-event time of the
               stage INCLUDING the densification to the ABI's dense result
               (max over ranks); inputs are far larger than L2.
  e2e          through the public batch API (capi.Pipeline) with pinned HOST
               buffers: per chunk cl_upload (H2D) + cl_run_postssa (kernels +
               device densify) + cl_download (D2H); upload, run and download are
               stage threads over a few contexts, so the three overlap across chunks.
  roofline     algorithmic bytes / kernel time vs MEASURED_PEAKS.json hbm_gbs;
               `traffic` = DRAM bytes of the dominant kernel per launch from the
               committed ncu capture of this workload (profiles/r02_traffic.json).
  cpu_baseline the oracle (C port of the reference) on this box's host cores,
               bounded sample of the same corpus.
  configs      (N = 1) the other BASELINE.json configs, each with its own value,
               roofline fraction and CPU sample: bundled corpus, sm52-10M with the
               RAW stage (OpModTransform + SRSubstituteReverse via cl_run_raw, then
               XmadToImad), sm90-10M (all sequence patterns), long blocks.

`--impl reference` times that CPU port alone (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")     # before CUDA starts: see capi.py

from paper_2604_27486_b200 import synth  # noqa: E402
from paper_2604_27486_b200.soa import Corpus  # noqa: E402

METRIC = "lifted SASS instructions/sec"
UNIT = "inst/s"


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="mixed", choices=["mixed", "sm90", "sm52", "sm75", "long", "raw_x4", "raw_sr"])
    ap.add_argument("--insts", type=float, default=float(os.environ.get("CL_BENCH_INSTS", 100e6)),
                    help="SASS instructions in the whole corpus (all ranks)")
    ap.add_argument("--seed", type=int, default=100)
    ap.add_argument("--cpu-sample", type=float, default=6e6, help="SASS instructions of the CPU-baseline sample")
    ap.add_argument("--chunks", type=int, default=16, help="e2e: chunks the corpus is streamed in")
    ap.add_argument("--depth", type=int, default=4, help="e2e: contexts (chunks in flight)")
    ap.add_argument("--runners", type=int, default=2, help="e2e: run threads (kernels of two chunks back to back)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-objects", action="store_true", help="skip the objects-in / objects-out leg (e2e_objects)")
    ap.add_argument("--no-configs", action="store_true", help="skip the per-config legs (BASELINE.json configs[0..3])")
    ap.add_argument("--no-typeseed", action="store_true", help="skip the type-seeding leg (SURVEY 8 row f3)")
    ap.add_argument("--only-typeseed", action="store_true", help="run the type-seeding leg alone and print its object (ncu captures)")
    ap.add_argument("--passes", type=int, default=15, help="CL_PASS_* mask of the headline leg")
    return ap.parse_args()


from paper_2604_27486_b200.sharding import allgather_counts, materialize, plan_shards  # noqa: E402


def pinned_like_array(a: np.ndarray):
    """Copy of an array in pinned host memory (the numpy view keeps the owning tensor alive)."""
    import torch
    a = np.ascontiguousarray(a)
    t = torch.empty(max(a.nbytes, 16), dtype=torch.uint8, pin_memory=True)
    v = t.numpy()[:a.nbytes].view(a.dtype).reshape(a.shape)
    v[...] = a
    return v



def pinned_like(corpus: Corpus):
    """Copy of the corpus whose arrays live in pinned host memory."""
    import torch
    out = {}
    for name in Corpus.ARRAYS:
        a = np.ascontiguousarray(getattr(corpus, name))
        t = torch.empty(max(a.nbytes, 16), dtype=torch.uint8, pin_memory=True)
        v = t.numpy()[:a.nbytes].view(a.dtype).reshape(a.shape)
        v[...] = a
        out[name] = v
        out.setdefault("_keep", []).append(t)
    keep = out.pop("_keep")
    c = Corpus(**out)
    c._pinned = keep
    return c


# ------------------------------------------------------------- measurement
class ClockSampler:
    QUERY = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.rows, self.proc, self.index = [], None, index

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            self.t.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], 0, set()
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = max(mx, float(r[1]))
            except (ValueError, IndexError):
                continue
            for name, val in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"), r[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def algorithmic_bytes(c_in: Corpus, n_out, n_selected):
    """one read of the stage input, one write of the stage output."""
    return 64 * (c_in.n_insts + n_out) + 4 * (2 * c_in.n_blocks + 2 * c_in.n_funcs) + 16 * n_selected


def cpu_leg(corpus: Corpus, n_sass, threads, steps=1, warmup=0):
    """The oracle (C port of the reference path) on the host cores."""
    from paper_2604_27486_b200.capi import Engine
    subprocess.run(["make", "-s", "-C", str(ROOT / "oracle")], check=True)
    eng = Engine(ROOT / "oracle" / "liboracle.so")
    eng.set_threads(threads)
    eng.upload(corpus)
    times = []
    for i in range(warmup + steps):
        eng.run_postssa()
        if i >= warmup:
            times.append(eng.last_run_ms() / 1e3)
    return n_sass * len(times) / sum(times), float(np.mean(times))


def roofline_of(bytes_per_step, ms, peak, n_sass):
    achieved = bytes_per_step / (ms / 1e3) / 1e9
    return {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "algorithmic_bytes_per_launch": int(bytes_per_step), "bytes_per_sass_inst": bytes_per_step / max(n_sass, 1)}


def timed(eng, run, steps, warmup):
    """W untimed + K timed runs of `run` on an uploaded corpus: mean device ms (CUDA events inside the library)."""
    import torch
    for _ in range(warmup):
        run()
    torch.cuda.synchronize()
    ms = []
    for _ in range(steps):
        run()
        ms.append(eng.last_run_ms())
    torch.cuda.synchronize()
    return float(np.mean(ms))


def config_legs(eng, peak, threads, steps, warmup, with_cpu):
    """BASELINE.json configs[0..3] on one GPU: device-resident throughput, roofline fraction, CPU sample."""
    import gzip
    import pickle
    from paper_2604_27486_b200 import layout as L, passes as P, soa
    out = []

    def cpu_sample(kind, seed, n, passes_mask=15, raw=0):
        if not with_cpu:
            return None
        c, ns, _ = synth.build_corpus(kind, n, seed=seed)
        from paper_2604_27486_b200.capi import Engine
        o = Engine(ROOT / "oracle" / "liboracle.so")
        o.set_threads(threads)
        o.upload(c)
        if raw:
            o.run_raw(raw, P._sr_map())
        else:
            o.run_postssa(passes_mask)
        sec = o.last_run_ms() / 1e3
        o.close()
        return {"value": ns / sec, "unit": UNIT, "cores": threads, "kind": "port", "sample": f"{ns} SASS instructions of the same corpus, {sec:.2f} s"}

    def postssa_leg(name, corpus, n_sass, passes_mask, what, cpu):
        eng.upload(corpus)
        ms = timed(eng, lambda: eng.run_postssa(passes_mask), steps, warmup)
        st = eng.stats()
        b = algorithmic_bytes(corpus, int(st["n_inst_out"]), int(st["selected"].sum()))
        part = eng.debug_partition() or {}
        return {"config": name, "workload": what, "metric": METRIC, "value": n_sass / (ms / 1e3), "unit": UNIT, "ms_per_step": ms,
                "steps": steps, "warmup": warmup, "sass_insts": int(n_sass), "records": int(corpus.n_insts), "kernels": int(corpus.n_funcs),
                "roofline": roofline_of(b, ms, peak, n_sass), "cpu_baseline": cpu, "gpu_launches": int(part.get("launches", 0)) * steps,
                "match_counts": {"selected": int(st["selected"].sum()), "rewrites": int(st["rewrites"].sum()), "refused": int(st["refused"].sum())}}

    # configs[0]: the reference's bundled corpus (22 functions, 261 SASS instructions), tiled for timing only
    with gzip.open(ROOT / "tests" / "golden" / "bundled.pkl.gz", "rb") as fh:
        fns = pickle.load(fh)["functions"]
    one = soa.encode(fns)
    k = 4096
    tiled = synth.take_functions(one, np.tile(np.arange(one.n_funcs), k))
    n_bundled = 261 * k
    cpu = None
    if with_cpu:
        from paper_2604_27486_b200.capi import Engine
        o = Engine(ROOT / "oracle" / "liboracle.so"); o.set_threads(threads)
        small = synth.take_functions(one, np.tile(np.arange(one.n_funcs), 256))
        o.upload(small); o.run_postssa(); sec = o.last_run_ms() / 1e3; o.close()
        cpu = {"value": 261 * 256 / sec, "unit": UNIT, "cores": threads, "kind": "port", "sample": f"the bundled corpus x 256, {sec:.2f} s"}
    out.append(postssa_leg("bundled", tiled, n_bundled, 15, f"pkg/corpus listings (22 functions, 261 SASS instructions) x {k}, full post-SSA stage", cpu))

    # configs[1]: sm52, 10 M instructions: OpModTransform + SRSubstituteReverse (raw stage) + XmadToImad
    legs, total_ms, n_ref = [], 0.0, None
    for name, kind, raw in (("OpModTransform (cl_run_raw X4)", "raw_x4", L.RAW_X4), ("SRSubstituteReverse (cl_run_raw SR)", "raw_sr", L.RAW_SR)):
        c, ns, _ = synth.build_corpus(kind, 10_000_000, seed=52)
        eng.upload(c)
        ms = timed(eng, lambda: eng.run_raw(raw, P._sr_map()), steps, warmup)
        n_out = int(eng.stats()["n_inst_out"])
        b = 64 * (c.n_insts + n_out) + 8 * c.n_funcs
        legs.append({"pass": name, "ms_per_step": ms, "value": ns / (ms / 1e3), "sass_insts": int(ns), "records_in": int(c.n_insts), "records_out": n_out,
                     "roofline": roofline_of(b, ms, peak, ns), "cpu_baseline": cpu_sample(kind, 52, 300_000, raw=raw)})
        total_ms += ms
        n_ref = ns
    c, ns, _ = synth.build_corpus("sm52", 10_000_000, seed=52)
    xm = postssa_leg("sm52-10M/xmad", c, ns, L.PASS_XMAD, "XmadToImad (normalize_xmad only)", cpu_sample("sm52", 52, 300_000, L.PASS_XMAD))
    legs.append({"pass": "XmadToImad (cl_run_postssa XMAD)", "ms_per_step": xm["ms_per_step"], "value": xm["value"], "sass_insts": int(ns),
                 "roofline": xm["roofline"], "cpu_baseline": xm["cpu_baseline"], "match_counts": xm["match_counts"]})
    total_ms += xm["ms_per_step"]
    out.append({"config": "sm52-10M", "workload": "SM52 XMAD-heavy synthetic corpus, 10 M instructions: OpModTransform + SRSubstituteReverse + XmadToImad",
                "metric": METRIC, "value": n_ref / (total_ms / 1e3), "unit": UNIT, "ms_per_step": total_ms, "steps": steps, "warmup": warmup,
                "sass_insts": int(n_ref), "passes": legs,
                "roofline": {"bound": "hbm", "frac": sum(l["roofline"]["algorithmic_bytes_per_launch"] for l in legs) / (total_ms / 1e3) / 1e9 / peak,
                             "achieved": sum(l["roofline"]["algorithmic_bytes_per_launch"] for l in legs) / (total_ms / 1e3) / 1e9, "peak": peak, "unit": "GB/s"}})

    # configs[2]: sm90, 10 M instructions, all sequence patterns; configs[3]: long unrolled blocks
    for name, kind, n, what in (("sm90-10M", "sm90", 10_000_000, "SM90 synthetic corpus, 10 M instructions, all 8 sequence patterns, full post-SSA stage"),
                                ("long-blocks", "long", 4_000_000, "single-block kernels of 4096 / 8192 / 16384 instructions with reciprocal chains, 4 M instructions, full post-SSA stage")):
        c, ns, _ = synth.build_corpus(kind, n, seed=90 if kind == "sm90" else 4096)
        out.append(postssa_leg(name, c, ns, 15, what, cpu_sample(kind, 90, 300_000)))
    return out


def typeseed_leg(eng, peak, threads, steps, warmup, with_cpu, n_sass=20_000_000):
    """Type seeding (cl_seed_types, typerec.py:288) on the NORMALISED stream: the mixed corpus goes through the
    post-SSA stage, its result is the corpus the seeding kernel reads (device resident).  value = SASS instructions
    of that corpus per second of kernel time (CUDA events inside the call); e2e = the whole C-ABI call with the
    tables going up and the result arrays coming back to host memory."""
    from paper_2604_27486_b200 import typerec
    from paper_2604_27486_b200.capi import Engine
    c_in, ns, _ = synth.build_corpus("mixed", n_sass, seed=101)
    eng.upload(c_in)
    eng.run_postssa(15)
    corpus = eng.download()        # for the sizes, the counters below and the CPU leg; the seeding reads the result on the device
    ms, wall = [], []
    nrec, nval = corpus.n_insts, len(corpus.val_alive)
    pin = pinned_like_array if eng.backend.startswith("cuda") else (lambda a: a)
    holder = typerec.SeedArrays(pin(np.zeros(nval, np.uint32)), pin(np.zeros(nrec, np.uint8)), pin(np.zeros(nrec, np.uint16)),
                                pin(np.zeros(nrec, np.uint32)), pin(np.zeros(corpus.n_funcs, np.uint8)))
    for k in range(warmup + steps):
        t0 = time.perf_counter()
        res = typerec.seed_corpus(eng, c_in, None, upload=False, into=holder, source=typerec.SEED_RESULT)
        if k >= warmup:
            wall.append(time.perf_counter() - t0)
            ms.append(eng.last_run_ms())
    R, V, B, F = corpus.n_insts, len(corpus.val_alive), corpus.n_blocks, corpus.n_funcs
    algo = 64 * R + 7 * R + 8 * V + 16 * B + 4 * (B + 3 * F)
    t = float(np.mean(ms))
    traffic = None
    try:                       # DRAM bytes of k_typeseed per launch from the committed ncu capture of this very leg
        tr = json.loads((ROOT / "profiles" / "r02_traffic.json").read_text())["k_typeseed"]
        if abs(ns - tr["workload_sass_insts"]) < 0.01 * tr["workload_sass_insts"]:
            traffic = tr["dram_bytes_per_launch"]
    except (OSError, KeyError, ValueError):
        pass
    out = {"config": "typeseed", "workload": f"seed_types over the normalised mixed corpus: {ns} SASS instructions, {R} records, {V} values, {F} kernels",
           "metric": METRIC, "value": ns / (t / 1e3), "unit": UNIT, "ms_per_step": t, "steps": steps, "warmup": warmup,
           "gpu_launches": 4 * steps, "kernel": "k_typeseed (+ k_typeseed_prepare: mask fill, record offsets; k_typeseed_index: function of every run of 32 records; k_typeseed_check: dead values)",
           "roofline": {"bound": "hbm", "achieved": algo / (t / 1e3) / 1e9, "peak": peak, "unit": "GB/s", "frac": algo / (t / 1e3) / 1e9 / peak,
                        "traffic": traffic, "algorithmic_bytes_per_launch": int(algo),
                        "bytes_per_record": "64 read + 7 written per record, 8 per value (fill + result), 16 per block terminator, CSR offsets"},
           "e2e": {"value": ns / float(np.mean(wall)), "unit": UNIT, "ms_per_step": float(np.mean(wall)) * 1e3,
                   "h2d_bytes_per_step": 0, "d2h_bytes_per_step": int(7 * R + 4 * V + F),
                   "path": "cl_seed_types(CL_SEED_RESULT) on the dense result cl_run_postssa left on the device (no host round trip between the "
                           "stage and the seeding): tables up, kernels, result arrays back to pinned host memory"},
           "narrowed_values": int((res.val_masks != 0xFFFFFF).sum()), "transparent_records": int((res.role == 1).sum())}
    if with_cpu:
        o = Engine(ROOT / "oracle" / "liboracle.so")
        typerec.seed_corpus(o, corpus, None)
        sec = o.last_run_ms() / 1e3
        ref = typerec.seed_corpus(o, corpus, None, upload=False)
        sec = min(sec, o.last_run_ms() / 1e3)
        o.close()
        same = all(np.array_equal(getattr(res, n), getattr(ref, n)) for n in ("val_masks", "role", "link_mask", "link_def", "status"))
        out["cpu_baseline"] = {"value": ns / sec, "unit": UNIT, "cores": 1, "kind": "port",
                               "sample": f"the same corpus ({ns} SASS instructions), best of 2 passes, {sec:.2f} s on one thread"}
        out["equal_to_oracle"] = bool(same)
    return out


def objects_leg(eng, n_target=1_000_000):
    """Objects in -> objects out: what a `sasslift` user of the drop-in sees.  LiftedFunction objects
    (the synth_sm90 fixture of the reference's front half, unpickled as many times as it takes) -> soa.encode (C
    encoder) -> cl_upload / cl_run_postssa / cl_download -> soa.apply (objects mutated in place)."""
    import gzip
    import pickle
    from paper_2604_27486_b200 import soa
    from paper_2604_27486_b200 import patterns as PT
    blob = gzip.open(ROOT / "tests" / "golden" / "synth_sm90.pkl.gz", "rb").read()
    one = pickle.loads(blob)["functions"]
    lines = {id(i.raw) for fn in one for b in fn.block_order() for i in b.instructions if getattr(i, "raw", None) is not None}
    recs = sum(len(b.instructions) for fn in one for b in fn.block_order())
    n_sass_one = max(len(lines), 1)
    copies = max(1, int(round(n_target / n_sass_one)))
    fns = []
    for _ in range(copies):
        fns.extend(pickle.loads(blob)["functions"])
    t0 = time.perf_counter()
    corpus = soa.encode(fns)
    t1 = time.perf_counter()
    eng.upload(corpus)
    eng.run_postssa()
    out = eng.download()
    t2 = time.perf_counter()
    out.functions = fns
    soa.apply(out, patterns=PT.pattern_list(), c_in=corpus)
    t3 = time.perf_counter()
    n = n_sass_one * copies
    return {"value": n / (t3 - t0), "unit": UNIT, "sass_insts": n, "ssa_records": recs * copies, "functions": len(fns),
            "encode_inst_per_s": n / (t1 - t0), "device_inst_per_s": n / (t2 - t1), "decode_inst_per_s": n / (t3 - t2),
            "seconds": {"encode": t1 - t0, "upload_run_download": t2 - t1, "apply": t3 - t2},
            "path": "LiftedFunction objects -> soa.encode (csrc/codec.c) -> cl_upload + cl_run_postssa + cl_download -> soa.apply; one host thread",
            "note": "bounded by building / reading Python objects (apply creates every operand object anew): the device stage is "
                    "three orders of magnitude faster, which is why the batch API (e2e) takes encoded corpora"}


def main():
    args = parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    n_total = int(args.insts)
    threads = os.cpu_count() or 1

    if args.impl == "reference":
        if rank != 0:
            return
        sample_n = int(min(n_total, args.cpu_sample))
        kinds, pools, kid, pick, ns, nb, shard = plan_shards(args.workload, sample_n, args.seed, 1)
        corpus = materialize(kinds, pools, kid, pick, np.arange(len(kid)))
        n_sass = int(ns.sum())
        value, sec = cpu_leg(corpus, n_sass, threads, args.steps, args.warmup)
        sample = f"{n_sass} SASS instructions ({corpus.n_insts} SSA records, {corpus.n_funcs} kernels) of the {args.workload} corpus per step"
        print(json.dumps({
            "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": f"{args.workload}-{n_total / 1e6:g}M (BASELINE.json configs[4]), CPU sample", "sample": sample},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0,
        }))
        return

    import torch
    import torch.distributed as dist
    from paper_2604_27486_b200.capi import Engine

    if args.only_typeseed:
        torch.cuda.set_device(local)
        pk = 6650.0
        try:
            pk = float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text()).get("hbm_gbs", pk))
        except OSError:
            pass
        e = Engine(device=local)
        print(json.dumps(typeseed_leg(e, pk, threads, args.steps, args.warmup, not args.no_cpu)))
        e.close()
        return

    # CL_BENCH_SIM=1: dry run of the rank plumbing without a GPU (tests/test_bench_contract.py): the one-lane CPU build
    # of the device code as the engine, gloo instead of NCCL; its numbers mean nothing and the line says "sim"
    sim = os.environ.get("CL_BENCH_SIM") == "1"
    dev = "cpu" if sim else "cuda"
    if sim:
        sys.path.insert(0, str(ROOT / "tests"))
        import helpers
        sim_lib = helpers.build_sim()
        args.no_e2e = args.no_cpu = args.no_configs = args.no_objects = args.no_typeseed = True
        if world > 1:
            dist.init_process_group("gloo")
    else:
        torch.cuda.set_device(local)
        if world > 1:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    t0 = time.time()
    kinds, pools, kid, pick, ns, nb, shard = plan_shards(args.workload, n_total, args.seed, world)
    mine = np.nonzero(shard == rank)[0]
    corpus = materialize(kinds, pools, kid, pick, mine)
    n_sass_rank = int(ns[mine].sum())
    n_sass_all = int(ns.sum())
    t_gen = time.time() - t0

    eng = Engine(sim_lib) if sim else Engine(device=local)
    eng.upload(corpus)
    counts = torch.zeros(68, dtype=torch.int64, device=dev)

    class _Raw:           # device counters of the library as a CUDA array (no host copy)
        def __init__(self, ptr):
            self.__cuda_array_interface__ = {"shape": (68,), "typestr": "<i8", "data": (ptr, False), "version": 3}
    if sim:
        import ctypes
        lib_counts = torch.from_numpy(np.ctypeslib.as_array((ctypes.c_int64 * 68).from_address(eng.device_counts_ptr())))
    else:
        lib_counts = torch.as_tensor(_Raw(eng.device_counts_ptr()), device="cuda")

    gathered = [None]

    def step():
        eng.run_postssa(args.passes)
        if world > 1:                      # the only inter-GPU traffic: match counters
            counts.copy_(lib_counts)
            gathered[0] = allgather_counts(counts, world)
        return eng.last_run_ms()

    def fence():
        if world > 1:
            dist.barrier()
        if not sim:
            torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    fence()
    dev_ms = []
    with ClockSampler(local) as clocks:
        t1 = time.perf_counter()
        for _ in range(args.steps):
            dev_ms.append(step())
        fence()
        wall = time.perf_counter() - t1
    if sim:
        dev_ms = [wall / args.steps * 1e3] * args.steps         # the CPU build has no device clock
    st = eng.stats()
    part = eng.debug_partition() or {}
    if os.environ.get("CL_PROF") and rank == 0:
        prof = eng.debug_profile()
        tot = max(prof.get("total", 1), 1)
        print("phase cycles (share of group time):", {k: round(v / tot, 3) for k, v in prof.items() if v}, file=sys.stderr)
    n_out = int(st["n_inst_out"])
    n_sel = int(st["selected"].sum())
    # max over ranks of the device time of the K steps
    t_dev = torch.tensor([sum(dev_ms) / 1e3, wall], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_dev, op=dist.ReduceOp.MAX)
    t_dev_s, t_wall_s = (float(x) for x in t_dev.cpu())
    value = n_sass_all * args.steps / t_dev_s

    bytes_per_step = algorithmic_bytes(corpus, n_out, n_sel)
    peaks = {}
    try:
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except OSError:
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    # DRAM bytes of the dominant kernel per launch: from the committed ncu --set full capture of this very
    # workload (profiles/r02_traffic.json); null for any other workload or path
    traffic, kernel_name = None, "k_postssa_gtile"
    try:
        tr = json.loads((ROOT / "profiles" / "r02_traffic.json").read_text())["k_postssa_gtile"]
        if (args.workload == "mixed" and world == 1 and part.get("tile_mode") == 4 and args.passes == 15
                and abs(n_sass_all - tr["workload_sass_insts"]) < 0.01 * tr["workload_sass_insts"]):
            traffic = tr["dram_bytes_per_launch"]
    except (OSError, KeyError, ValueError):
        pass
    roofline = roofline_of(bytes_per_step, float(np.mean(dev_ms)), peak, n_sass_rank)
    roofline.update({"traffic": traffic, "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650 GB/s",
                     "kernel": ("k_fused (one function resident in shared memory per warp group) with the per-function kernels for what it hands back: the whole stage, rank 0"
                                if part.get("tile_mode") == 16 else
                                "k_postssa_gtile<TileCfgG4,32,2> (tile kernel: kernels packed into tiles of up to 32 768 records / 255 kernels, a long block a tile of its own; "
                                "two 1024-thread CTAs per SM) with the per-function kernels for what it hands back and the densify kernels: the whole stage, rank 0")})

    # end to end through the public batch API with pinned HOST buffers: the corpus flows chunk by chunk
    # (contiguous function ranges) through a few contexts, so H2D, kernels and D2H of different chunks overlap
    e2e = None
    if not args.no_e2e:
        from paper_2604_27486_b200.capi import Pipeline
        eng.close()                                             # its device buffers make room for the pipeline's contexts
        del lib_counts
        ranges = corpus.split(args.chunks)
        host_in = [pinned_like(corpus.slice_funcs(f0, f1)) for f0, f1 in ranges]
        h2d = sum(c.nbytes() for c in host_in)
        pipe = Pipeline(device=local, depth=args.depth, runners=args.runners)
        first, _, _ = pipe.run_postssa(host_in)                 # sizes the pinned result holders (and warms up)
        d2h = sum(o.nbytes() + o.events.nbytes for o in first)
        holders = []
        for o in first:
            h = pinned_like(o)
            h.events = pinned_like_array(np.zeros(len(o.events) + 16, o.events.dtype))
            holders.append(h)
        n_out_e2e = sum(o.n_insts for o in first)
        del first

        def e2e_step():
            outs, st_sum, _ = pipe.run_postssa(host_in, into=holders)
            return sum(o.n_insts for o in outs)

        for _ in range(max(1, args.warmup - 1)):
            e2e_step()
        fence()
        t2 = time.perf_counter()
        for _ in range(args.steps):
            got = e2e_step()
        fence()
        assert got == n_out_e2e == n_out, (got, n_out_e2e, n_out)     # the chunked run is the same job
        if os.environ.get("CL_TRACE") and rank == 0:
            for kk, tr in enumerate(pipe.last_trace):
                print(f"chunk {kk}: ctx {tr[0]} upload {tr[1]*1e3:7.1f}..{tr[2]*1e3:7.1f} run {tr[3]*1e3:7.1f}..{tr[4]*1e3:7.1f} download ..{tr[5]*1e3:7.1f} ms; kernels {tr[6]:6.1f} ms", file=sys.stderr)
        te = torch.tensor([time.perf_counter() - t2], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": n_sass_all * args.steps / float(te.cpu()[0]), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": float(te.cpu()[0]) / args.steps * 1e3,
               "path": f"capi.Pipeline: {len(host_in)} chunks (function ranges) through {args.depth} contexts, {args.runners} run threads; per chunk "
                       "cl_upload (pinned H2D) + cl_run_postssa + cl_download (device densify + pinned D2H); upload, run and download are "
                       "stage threads, so the three overlap across chunks"}
        pipe.close()
        del holders, host_in

    cpu = None
    if rank == 0 and not args.no_cpu and world == 1:
        sample_n = int(min(n_total, args.cpu_sample))
        k2, p2, kid2, pick2, ns2, _, _ = plan_shards(args.workload, sample_n, args.seed, 1)
        sample_c = materialize(k2, p2, kid2, pick2, np.arange(len(kid2)))
        v, sec = cpu_leg(sample_c, int(ns2.sum()), threads, steps=3, warmup=1)
        cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"{int(ns2.sum())} SASS instructions ({sample_c.n_insts} records) of the same corpus, 1 warm-up + 3 timed passes of {sec:.2f} s on {threads} threads"}

    e2e_objects = None
    if rank == 0 and world == 1 and not args.no_objects and args.workload == "mixed":
        eng3 = Engine(device=local)
        e2e_objects = objects_leg(eng3)
        eng3.close()
    configs = None
    if rank == 0 and world == 1 and not args.no_configs and args.workload == "mixed":
        eng2 = Engine(device=local)
        configs = config_legs(eng2, peak, threads, max(2, min(args.steps, 3)), max(3, args.warmup), not args.no_cpu)
        eng2.close()

    typeseed = None
    if rank == 0 and world == 1 and not args.no_typeseed and args.workload == "mixed":
        eng4 = Engine(device=local)
        typeseed = typeseed_leg(eng4, peak, threads, max(2, min(args.steps, 5)), max(3, args.warmup), not args.no_cpu)
        eng4.close()

    # whole-job match counters: this rank's at N = 1, the sum of the allgathered rows of the last step at N > 1
    whole_job = {"selected": int(n_sel), "rewrites": int(st["rewrites"].sum()), "refused": int(st["refused"].sum())}
    if world > 1 and gathered[0] is not None:
        tot = gathered[0].sum(dim=0).cpu().numpy()
        whole_job = {"selected": int(tot[16:32].sum()), "rewrites": int(tot[32:48].sum()), "refused": int(tot[48:64].sum()),
                     "per_rank_selected": [int(r[16:32].sum()) for r in gathered[0].cpu().numpy()]}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_dev_s / args.steps * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "u32", "data": "synthetic" if not sim else "synthetic (CL_BENCH_SIM dry run on the CPU build: numbers are not measurements)",
            "config": {"workload": f"{args.workload}-{n_sass_all / 1e6:.1f}M SASS instructions (BASELINE.json configs[4]: "
                                   f"40% sm90 / 40% sm75 / 20% sm52 kernels + long-block kernels), full post-SSA stage",
                       "kernels": int(len(kid)), "ssa_records_rank0": int(corpus.n_insts), "sass_rank0": n_sass_rank,
                       "sharding": f"{world} shard(s) by kernel (LPT on instruction records), no data-path collective, allgather of match counts",
                       "l2": "inputs larger than L2 (no flush needed)", "seed": args.seed,
                       "corpus": "kernels drawn with replacement from reference-front-half pools (tests/golden/pool_*.npz: 16 000 + 24 long-block kernels, each pinned to the reference by digest)",
                       "gen_seconds": round(t_gen, 1), "wall_ms_per_step": t_wall_s / args.steps * 1e3},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks.summary(),
            "gpu_launches": int(part.get("launches", 0)) * args.steps,
            "partition": part,
            "match_counts": whole_job,
            "e2e_objects": e2e_objects,
            "configs": configs,
            "typeseed": typeseed,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
