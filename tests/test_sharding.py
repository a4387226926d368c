"""Multi-GPU path on CPU: two gloo ranks shard one corpus by basic-block
count, run the stage on their shard (device code, one-lane CPU build) and
allgather the match counters; the union must equal the single-process run."""
import os
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent


def _worker(rank, world, port, n_sass, q):
    sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import helpers
    from paper_2604_27486_b200 import sharding
    kinds, pools, kid, pick, ns, nb, shard = sharding.plan_shards("mixed", n_sass, 7, world)
    mine = np.nonzero(shard == rank)[0]
    corpus = sharding.materialize(kinds, pools, kid, pick, mine)
    eng = helpers.sim_engine()
    eng.upload(corpus); eng.run_postssa()
    st = eng.stats()
    counts = torch.tensor(np.concatenate([st["matches"], st["selected"], st["rewrites"], st["refused"],
                                          [st["n_inst_in"], st["n_inst_out"]]]).astype(np.int64))
    allc = sharding.allgather_counts(counts, world)
    if rank == 0:
        q.put((allc.numpy(), [int(nb[shard == r].sum()) for r in range(world)], int(len(kid)),
               sorted(np.concatenate([np.nonzero(shard == r)[0] for r in range(world)]).tolist()) == list(range(len(kid)))))
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_sharding_matches_single_process():
    sys.path.insert(0, str(ROOT / "tests"))
    import helpers
    helpers.build_sim()
    n_sass, world, port = 60_000, 2, 29611
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_sass, q)) for r in range(world)]
    for p in procs:
        p.start()
    allc, blocks, n_kernels, complete = q.get(timeout=240)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    assert complete and allc.shape[0] == world
    assert abs(blocks[0] - blocks[1]) <= max(blocks) * 0.02 + 64      # balanced by basic-block count
    from paper_2604_27486_b200 import sharding
    kinds, pools, kid, pick, ns, nb, shard = sharding.plan_shards("mixed", n_sass, 7, 1)
    assert len(kid) == n_kernels
    whole = sharding.materialize(kinds, pools, kid, pick, np.arange(len(kid)))
    eng = helpers.sim_engine()
    eng.upload(whole); eng.run_postssa()
    st = eng.stats()
    single = np.concatenate([st["matches"], st["selected"], st["rewrites"], st["refused"],
                             [st["n_inst_in"], st["n_inst_out"]]]).astype(np.int64)
    assert np.array_equal(allc.sum(axis=0), single)
