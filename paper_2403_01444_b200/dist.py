"""View-sharded data-parallel Stage-1 (BASELINE configs 3-4).

Gaussians and NTC parameters are replicated; the B views of an iteration are
split across the W ranks (one process per GPU).  Each rank runs the whole
Stage-1 chain on its views with the image gradient scaled by 1/B, so the sum
all-reduce of the packed NTC gradient [tables | MLP] over NCCL yields the
gradient of the mean batch loss.  Every rank then applies the identical lazy
Adam step, which keeps the replicas bit-identical with no parameter broadcast.
The only collective is that one all-reduce per iteration.

Batch semantics (no reference equivalent, D6): loss = mean over views; the
oracle is the mean of per-view reference gradients followed by one Adam step.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_views(batch: list[int], rank: int, world: int) -> list[int]:
    """Contiguous split of an iteration's views across ranks (as even as possible)."""
    b = len(batch)
    lo = (b * rank) // world
    hi = (b * (rank + 1)) // world
    return batch[lo:hi]


def allreduce_sum_(flat: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """In-place sum all-reduce of the packed gradient (no-op for one rank)."""
    if world > 1:
        dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    return flat


class ViewShardedStage1:
    def __init__(self, prev_cloud, cache, views, cfg=None, rank: int = 0, world: int = 1,
                 group=None, views_per_iteration: int | None = None):
        from .stage1 import Stage1Trainer

        self.rank, self.world, self.group = rank, world, group
        self.trainer = Stage1Trainer(prev_cloud, cache, views, cfg)
        self.views_per_iteration = views_per_iteration

    def _grads_for(self, views: list[int], total: int) -> None:
        tr = self.trainer
        for v in views:
            tr.iterate(v, grad_scale=1.0 / total, adam=False)

    def step(self, batch: list[int]) -> None:
        """One iteration over `batch` (global view ids), stream-ordered with no
        host synchronisation (the all-reduce is an NCCL kernel on the stream)."""
        tr = self.trainer
        if self.world == 1 and len(batch) == 1:
            tr.iterate(batch[0])
            return
        mine = shard_views(batch, self.rank, self.world)
        self._grads_for(mine, len(batch))
        allreduce_sum_(tr.g_flat, self.world, self.group)
        tr.apply_adam()

    def step_from_host(self, batch: list[int], host_targets) -> float:
        """End-to-end iteration through host buffers (pinned target H2D, loss D2H)."""
        tr = self.trainer
        mine = shard_views(batch, self.rank, self.world)
        if self.world == 1 and len(batch) == 1:
            return tr.step_from_host(mine[0], host_targets[mine[0]])
        loss = 0.0
        for v in mine:
            tr.stage_target(v, host_targets[v])
            tr.iterate(v, grad_scale=1.0 / len(batch), adam=False, staged=True)
            loss += tr.last_loss()
        allreduce_sum_(tr.g_flat, self.world, self.group)
        tr.apply_adam()
        return loss
