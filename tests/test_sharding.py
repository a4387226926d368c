"""Multi-GPU path on CPU.  The sharder partitions ANY encoded corpus by kernel
(LPT on instruction records; basic-block balance reported); two gloo ranks run
the stage on their shard (device code, one-lane CPU build), allgather the match
counters, and the union of their results must equal the single-process run bit
for bit -- counters AND streams.  The same partition drives
``passes.gpu_normalize(..., engines=[...])`` inside one process."""
import copy
import os
import pickle
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT / "tests"))


def _counts(st):
    return np.concatenate([st["matches"], st["selected"], st["rewrites"], st["refused"],
                           [st["n_inst_in"], st["n_inst_out"]]]).astype(np.int64)


def _worker(rank, world, port, n_sass, out_dir):
    sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import helpers
    from paper_2604_27486_b200 import sharding, synth
    corpus = synth.build_corpus("mixed", n_sass, seed=7)[0]          # every rank sees the user's whole corpus ...
    plan = sharding.shard_plan(corpus, world)
    mine = sharding.shard(corpus, world, plan)[rank]                  # ... and takes its shard of it
    eng = helpers.sim_engine()
    eng.upload(mine); eng.run_postssa()
    out = eng.download()
    allc = sharding.allgather_counts(torch.tensor(_counts(eng.stats())), world)
    out.save(Path(out_dir) / f"shard{rank}.npz")
    if rank == 0:
        with open(Path(out_dir) / "counts.pkl", "wb") as fh:
            pickle.dump((allc.numpy(), plan.balance()), fh)
    dist.barrier()
    dist.destroy_process_group()


def _single(n_sass, out_dir):
    """the single-process run, in a fresh process like the ranks: interned ids (opcodes, modifier tuples, strings) are
    process-local tables filled in load order, so results are compared between processes with the same history"""
    sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
    import helpers
    from paper_2604_27486_b200 import synth
    whole = synth.build_corpus("mixed", n_sass, seed=7)[0]
    eng = helpers.sim_engine()
    eng.upload(whole); eng.run_postssa()
    eng.download().save(Path(out_dir) / "single.npz")
    with open(Path(out_dir) / "single_counts.pkl", "wb") as fh:
        pickle.dump(_counts(eng.stats()), fh)


@pytest.mark.timeout(300)
def test_two_rank_sharding_matches_single_process(tmp_path):
    import helpers
    from paper_2604_27486_b200 import sharding, synth
    from paper_2604_27486_b200.soa import Corpus
    helpers.build_sim()
    n_sass, world, port = 60_000, 2, 29611
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_sass, str(tmp_path))) for r in range(world)]
    procs.append(ctx.Process(target=_single, args=(n_sass, str(tmp_path))))
    for p in procs:
        p.start()
    for p in procs:
        p.join(240)
        assert p.exitcode == 0
    allc, balance = pickle.load(open(tmp_path / "counts.pkl", "rb"))
    assert allc.shape[0] == world and balance["records"] < 1.02, balance
    whole = synth.build_corpus("mixed", n_sass, seed=7)[0]
    single = Corpus.load(tmp_path / "single.npz")
    assert np.array_equal(allc.sum(axis=0), pickle.load(open(tmp_path / "single_counts.pkl", "rb")))   # the allgathered counters
    plan = sharding.shard_plan(whole, world)
    union = sharding.unshard([Corpus.load(tmp_path / f"shard{r}.npz") for r in range(world)], plan)
    assert not union.equal(single)                                                # ... and every byte of the streams
    assert np.array_equal(union.events, single.events)


def test_lpt_balances_records_even_with_long_kernels():
    """a 16 384-instruction kernel has ONE basic block: balancing by block count would land it anywhere"""
    from paper_2604_27486_b200 import sharding
    rng = np.random.default_rng(1)
    cost = np.concatenate([rng.integers(20, 300, 20_000), [19_000, 19_500, 9_800, 9_700, 4_800, 4_800, 4_900]])
    for n in (2, 4, 8):
        s = sharding.assign_lpt(cost, n)
        loads = np.array([cost[s == k].sum() for k in range(n)])
        assert loads.max() / loads.mean() < 1.005, (n, loads)
        heavy = s[-7:]
        assert len(set(heavy[:2].tolist())) == 2                                  # the two longest never share a shard


def test_gpu_normalize_over_several_engines_equals_one(oracle_engine):
    """passes.gpu_normalize(engines=[a, b]): objects in, objects out, same as one engine"""
    import helpers
    from paper_2604_27486_b200 import passes
    fix = helpers.load_fixture("synth_sm75")
    one = copy.deepcopy(fix["functions"])
    two = copy.deepcopy(fix["functions"])
    passes.gpu_normalize(one, engine=helpers.sim_engine())
    out = passes.gpu_normalize(two, engines=[helpers.sim_engine(), helpers.sim_engine(), helpers.sim_engine()])
    assert [helpers.state_of(f) for f in one] == [helpers.state_of(f) for f in two]
    assert [helpers.state_of(f) for f in two] == fix["expect"]
    assert out.shard_plan.n_shards == 3 and out.shard_plan.balance()["records"] < 1.3
