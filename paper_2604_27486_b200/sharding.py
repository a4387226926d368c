"""Corpus sharder (north-star subsystem 5): kernels are independent, so a
corpus is partitioned across GPUs by basic-block count with no data crossing
ranks; the only collective is a final allgather of the per-pattern match
counters (``allgather_counts``: NCCL on GPUs, gloo in the CPU tests)."""
from __future__ import annotations

import numpy as np

from . import synth

def plan_shards(kind, n_sass, seed, n_shards):
    """Kernel picks of the whole corpus (cheap: indices only) and their
    partition by basic-block count (synth.shard_by_blocks rule)."""
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
    for i, k in enumerate(kinds):
        m = kid == i
        p = pools[k]
        pick[m] = rng.integers(0, p.corpus.n_funcs, int(m.sum()))
        nb[m] = np.diff(p.corpus.func_blk_off.astype(np.int64))[pick[m]]
        ns[m] = p.n_sass[pick[m]]
    order = np.argsort(-nb, kind="stable")
    pos = np.arange(n_kernels)
    cyc = pos % (2 * n_shards)
    shard = np.empty(n_kernels, np.int64)
    shard[order] = np.where(cyc < n_shards, cyc, 2 * n_shards - 1 - cyc)
    return kinds, pools, kid, pick, ns, nb, shard


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
