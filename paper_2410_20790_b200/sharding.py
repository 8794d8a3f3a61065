"""Chunk sharding and the per-step sparsity-statistics exchange.

Chunks are independent units -- each has its own reference frame (PAPER.md
P:113, reading R12) -- so the path shards by chunk with no data-path
collective.  The only exchange is the online threshold controller's input
(P:171-181): every step each rank all-gathers the int64 per-site
(active, pixels) counts, sums them in rank order (integers: exact and
order-free) and runs the identical controller, so every rank derives the
same thresholds for the next step (reading R15: one observation per step
over a fixed group of chunks, which makes results independent of the GPU
count).
"""
from __future__ import annotations

import numpy as np


def shard(step: int, chunks_per_step: int, rank: int, world: int):
    """Global chunk ids of `rank` in `step`: a fixed group of chunks_per_step
    chunks per step, dealt round-robin (rank r takes r, r+G, r+2G, ...)."""
    if chunks_per_step % world:
        raise ValueError("chunks_per_step must be a multiple of the world size")
    base = step * chunks_per_step
    return [base + rank + world * j for j in range(chunks_per_step // world)]


class StatsExchange:
    """All-gather of int64 [2*n_sites] per-site counts over a process group.

    With NCCL the buffers live on the rank's GPU and the gather is
    all_gather_into_tensor over NVLink; with gloo (CPU tests) the same call
    runs on host tensors."""

    def __init__(self, n_sites: int, group=None, device=None):
        import torch
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.n = n_sites
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.device = device if device is not None else torch.device("cpu")
        self.local = torch.zeros(2 * n_sites, dtype=torch.int64, device=self.device)
        self.gathered = torch.zeros(self.world * 2 * n_sites, dtype=torch.int64, device=self.device)

    def exchange(self, local_counts=None):
        """local_counts: None (self.local already filled, e.g. by
        st_copy_site_counts) or an int array [2*n_sites].  Returns
        (site_active, site_pixels) summed over ranks in rank order."""
        import torch
        if local_counts is not None:
            self.local.copy_(torch.as_tensor(np.asarray(local_counts, np.int64)))
        if self.world > 1:
            self.dist.all_gather_into_tensor(self.gathered, self.local, group=self.group)
            per_rank = self.gathered.view(self.world, 2 * self.n).cpu().numpy()
        else:
            per_rank = self.local.view(1, 2 * self.n).cpu().numpy()
        tot = np.zeros(2 * self.n, np.int64)
        for r in range(per_rank.shape[0]):   # rank order
            tot += per_rank[r]
        return tot[: self.n], tot[self.n:]


class StepLoop:
    """The step schedule of a chunk-sharded job (reading R15).

    The job is n_groups fixed groups of chunks_per_step chunks; global step s
    processes group s mod n_groups, and rank r of G takes the group's chunks
    r, r+G, r+2G, ... (``shard``).  Every step: thresholds from the
    controller -> the rank's chunks are encoded (``encode(group, chunk_ids,
    thresholds)``, which fills ``exchange.local`` with the rank's int64
    (active, pixels) site counts, e.g. via st_copy_site_counts, or returns
    them) -> one all-gather -> the identical controller update on every rank.
    One observation per step over the whole group, whatever G is, so the
    thresholds -- and with them every output -- are independent of the GPU
    count (PIN15)."""

    def __init__(self, chunks_per_step: int, n_groups: int, rank: int, world: int, controller, exchange):
        self.B, self.n_groups = chunks_per_step, n_groups
        self.rank, self.world = rank, world
        self.ctl, self.ex = controller, exchange
        self.history = []

    def group(self, step: int) -> int:
        return step % self.n_groups

    def chunks(self, step: int):
        return shard(self.group(step), self.B, self.rank, self.world)

    def run_step(self, step: int, encode, observe: bool = True):
        th = self.ctl.thresholds()
        self.history.append(np.array(th, np.float32))
        local = encode(self.group(step), self.chunks(step), th)
        if observe:
            sa, sp = self.ex.exchange(local)
            self.ctl.observe(sa, sp)
        return th
