"""Corpus sharder (north-star subsystem 5).  Kernels are independent
(``ssir.py:215-235``: vids, iids, blocks, temporaries and def-use are all per
function), so a corpus is partitioned across GPUs by kernel with no data
crossing ranks; the only collective is a final allgather of the per-pattern
match counters (``allgather_counts``: NCCL on GPUs, gloo in the CPU tests).

Balance: longest-processing-time-first bin packing with the kernel's
*instruction-record count* as its cost (the better proxy; a
16 384-instruction single-block kernel has one basic block and costs as much
as two hundred small kernels).  The basic-block balance the north star words
it with is reported beside it.

    plan = shard_plan(corpus, n)              # which kernel goes where
    parts = shard(corpus, n, plan)            # list[Corpus], kernel order kept inside a shard
    whole = unshard(results, plan)            # results of the shards back in corpus order
"""
from __future__ import annotations

import heapq
from dataclasses import dataclass

import numpy as np

from . import synth
from .soa import Corpus


@dataclass
class ShardPlan:
    shard_of: np.ndarray          # [n_funcs] shard of every kernel
    members: list                 # per shard: kernel indices, ascending
    records: np.ndarray           # per shard: instruction records (the balanced cost)
    blocks: np.ndarray            # per shard: basic blocks (reported)

    @property
    def n_shards(self):
        return len(self.members)

    def balance(self):
        """{records, blocks}: max / mean over the shards (1.0 = perfect)."""
        r, b = self.records.astype(np.float64), self.blocks.astype(np.float64)
        return {"records": float(r.max() / max(r.mean(), 1.0)), "blocks": float(b.max() / max(b.mean(), 1.0))}


def assign_lpt(cost: np.ndarray, n_shards: int, head: int = 4096) -> np.ndarray:
    """Shard of every item: LPT on ``cost``.  The ``head`` heaviest items go one by one to the
    lightest shard (heap); the near-uniform rest is dealt in a snake over the shards ordered by
    load, which is LPT-equivalent for equal costs and O(n)."""
    cost = np.asarray(cost, np.int64)
    n = len(cost)
    out = np.zeros(n, np.int64)
    if n_shards <= 1 or n == 0:
        return out
    order = np.argsort(-cost, kind="stable")
    k = min(head, n)
    loads = [(0, s) for s in range(n_shards)]
    heapq.heapify(loads)
    for i in order[:k]:
        load, s = heapq.heappop(loads)
        out[i] = s
        heapq.heappush(loads, (load + int(cost[i]), s))
    if k < n:
        by_load = np.array([s for _, s in sorted(loads)], np.int64)       # lightest shard first
        pos = np.arange(n - k)
        cyc = pos % (2 * n_shards)
        out[order[k:]] = by_load[np.where(cyc < n_shards, cyc, 2 * n_shards - 1 - cyc)]
    return out


def _plan_from(shard_of, records, blocks, n_shards):
    members = [np.nonzero(shard_of == s)[0] for s in range(n_shards)]
    return ShardPlan(shard_of, members, np.array([int(records[m].sum()) for m in members]),
                     np.array([int(blocks[m].sum()) for m in members]))


def shard_plan(corpus: Corpus, n_shards: int) -> ShardPlan:
    fbo = corpus.func_blk_off.astype(np.int64)
    bo = corpus.blk_off.astype(np.int64)
    records = bo[fbo[1:]] - bo[fbo[:-1]]
    blocks = np.diff(fbo)
    return _plan_from(assign_lpt(records, n_shards), records, blocks, n_shards)


def shard(corpus: Corpus, n_shards: int, plan: ShardPlan | None = None):
    """Partition a corpus (any user's functions, encoded) into ``n_shards`` corpora."""
    plan = plan or shard_plan(corpus, n_shards)
    return [synth.take_functions(corpus, m) for m in plan.members]


def unshard(results, plan: ShardPlan) -> Corpus:
    """Results of the shards (``Engine.download()`` of each) as one corpus in the original kernel order."""
    whole = synth.concat(list(results))
    where = np.concatenate(plan.members)
    out = synth.take_functions(whole, np.argsort(where, kind="stable"))
    events = [r.events.copy() for r in results if getattr(r, "events", None) is not None]
    if len(events) == len(results):
        for ev, m in zip(events, plan.members):
            ev["func"] = m[ev["func"]]                       # shard-local kernel index -> corpus index
        allev = np.concatenate(events) if events else np.zeros(0)
        out.events = allev[np.argsort(allev["func"], kind="stable")]
    return out


# ------------------------------------------------------ synthetic corpora (bench)
def plan_shards(kind, n_sass, seed, n_shards):
    """Kernel picks of a synthetic corpus (cheap: indices into the pools only) and their partition
    (same LPT rule, cost = records): -> kinds, pools, kid, pick, ns (SASS instructions per kernel),
    nb (basic blocks per kernel), shard."""
    rng = np.random.default_rng(seed)
    shares = synth.MIXED if kind == "mixed" else ((kind, 1.0),)
    pools = {k: synth.pool(k) for k, _ in shares}
    mean = sum(sh * float(pools[k].n_sass.mean()) for k, sh in shares)
    n_kernels = max(n_shards, int(round(n_sass / mean)))
    kinds = [k for k, _ in shares]
    kid = rng.choice(len(kinds), n_kernels, p=np.array([sh for _, sh in shares]) / sum(sh for _, sh in shares))
    pick = np.zeros(n_kernels, np.int64)
    nb = np.zeros(n_kernels, np.int64)
    ns = np.zeros(n_kernels, np.int64)
    nr = np.zeros(n_kernels, np.int64)
    for i, k in enumerate(kinds):
        m = kid == i
        p = pools[k]
        pick[m] = rng.integers(0, p.corpus.n_funcs, int(m.sum()))
        fbo = p.corpus.func_blk_off.astype(np.int64)
        bo = p.corpus.blk_off.astype(np.int64)
        nb[m] = np.diff(fbo)[pick[m]]
        nr[m] = (bo[fbo[1:]] - bo[fbo[:-1]])[pick[m]]
        ns[m] = p.n_sass[pick[m]]
    shard_of = assign_lpt(nr, n_shards)
    return kinds, pools, kid, pick, ns, nb, shard_of


def materialize(kinds, pools, kid, pick, sel):
    """SoA corpus of kernels `sel` (indices into the plan), in plan order."""
    parts, where = [], []
    for i, k in enumerate(kinds):
        idx = sel[kid[sel] == i]
        if len(idx) == 0:
            continue
        parts.append(synth.take_functions(pools[k].corpus, pick[idx]))
        where.append(idx)
    if len(parts) == 1:
        return parts[0]
    corpus = synth.concat(parts)
    order = np.argsort(np.concatenate(where), kind="stable")       # back to plan order: archs interleaved
    return synth.take_functions(corpus, order)


def allgather_counts(counts, world: int):
    """counts: 1-D int64 torch tensor (device of the backend) -> [world, n] tensor."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return counts.unsqueeze(0).clone()
    out = [torch.zeros_like(counts) for _ in range(world)]
    dist.all_gather(out, counts)
    return torch.stack(out)
