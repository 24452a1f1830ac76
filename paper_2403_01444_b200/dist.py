"""View-sharded data-parallel Stage-1 (BASELINE configs 3-4).

Gaussians and NTC parameters are replicated; the B views of an iteration are
split contiguously across the W ranks (one process per GPU).  Each rank runs
the whole Stage-1 chain on its views with the image gradient scaled by 1/B, so
the sum all-reduce of the packed NTC gradient [tables | MLP | loss] yields the
gradient of the mean batch loss, and the batch-loss sum rides in the same
buffer.  Every rank then applies the identical lazy Adam step, which keeps the
replicas bit-identical with no parameter broadcast.

Per iteration the exchange is split in two so it overlaps the last kernel of
the backward: the decoder gradient (plus the loss slot) is all-reduced while
the hash-table scatter (ntc.py:278-288) still runs, then the table gradient.
View-space statistics (adaptive.py:79-97) are accumulated per view over the
last epoch's views and all-reduced once, at the end of the frame.

Batch semantics (no reference equivalent, D6): loss = mean over the views of
an iteration; the oracle is the mean of per-view reference gradients
(transform.py:99-135 -> ntc.py:250-288) followed by one Adam step
(optim.py:33-66).  The view sequence is the reference's per-epoch permutation
(pipeline.py:251-256, :263) read B views at a time.

The trainer is duck-typed (a `stage1.Stage1Trainer` on the GPU; the CPU tests
drive the same code with an oracle-backed stand-in):
  g_flat            packed fp32 gradient [tables | MLP | loss slot]
  n_table           length of the tables part
  n_views           number of training views
  batch_view(view, grad_scale=, first=, accumulate_stats=, staged=)   one view's render,
                    loss and raster backward, its transformed-cloud gradient added
                    to the batch's (first: NTC forward, gradient overwritten)
  batch_ntc_grads(defer_scatter=)   transform VJP + decoder backward + table scatter
                    (deferred: table_scatter()) of the batch gradient, once
  stage_target(view, host_tensor)   H2D copy of a view's target into the staging buffer
  table_scatter()   the deferred hash-table scatter
  apply_adam()      lazy Adam on g_flat (zeroes the table/MLP gradient)
  stats_norm, stats_count   per-Gaussian view-space statistics
  enable_loss_accum()       every iterate adds its loss to the loss slot
"""

from __future__ import annotations

import numpy as np
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


def batched_view_order(seed: int, frame_index: int, n_views: int, iterations: int,
                       views_per_iteration: int) -> list[list[int]]:
    """The reference view sequence (pipeline.py:251-256, :263, :278-279) read B
    views per iteration: iteration t trains positions [tB, tB + B)."""
    from .stage1 import view_order

    b = views_per_iteration
    seq = view_order(seed, frame_index, n_views, iterations * b)
    return [seq[t * b:(t + 1) * b] for t in range(iterations)]


class ViewShardedStage1:
    def __init__(self, prev_cloud=None, cache=None, views=None, cfg=None, rank: int = 0,
                 world: int = 1, group=None, views_per_iteration: int | None = None,
                 trainer=None):
        self.rank, self.world, self.group = rank, world, group
        if trainer is None:
            from .stage1 import Stage1Trainer

            trainer = Stage1Trainer(prev_cloud, cache, views, cfg)
        self.trainer = trainer
        self.views_per_iteration = views_per_iteration or world
        self.cfg = getattr(trainer, "cfg", cfg)
        # one view per iteration on one rank is the reference loop itself: the
        # iteration (Adam included) replays as one graph, losses in its history
        self.single = world == 1 and self.views_per_iteration == 1
        if not self.single:
            trainer.enable_loss_accum()
        self.loss_slot = trainer.g_flat[trainer.n_table + trainer.n_params:][:1]
        self._losses: list[torch.Tensor] = []

    # ------------------------------------------------------------------
    def step(self, batch: list[int], accumulate_stats=False, host_targets=None) -> None:
        """One iteration over `batch` (global view ids), stream-ordered with no
        host synchronisation.  `accumulate_stats`: one flag for the batch or
        one per view (the last-epoch window of pipeline.py:259, :276-277).
        `host_targets` (pinned host tensors by view id): each of this rank's
        targets is copied host -> device just before its view's iteration."""
        tr = self.trainer
        b = len(batch)
        flags = (list(accumulate_stats) if isinstance(accumulate_stats, (list, tuple))
                 else [bool(accumulate_stats)] * b)
        if self.single and b == 1:
            if host_targets is not None:
                tr.stage_target(batch[0], host_targets[batch[0]])
            tr.iterate(batch[0], accumulate_stats=flags[0], staged=host_targets is not None)
            self._losses.append(tr.loss_dev)
            return
        lo = (b * self.rank) // self.world
        mine = shard_views(batch, self.rank, self.world)
        split = self.world > 1
        # the views share the parameters: each adds its transformed-cloud
        # gradient, and the NTC backward (transform VJP, decoder, scatter) runs
        # once for the rank's views -- it is linear in that gradient
        for j, v in enumerate(mine):
            if host_targets is not None:
                tr.stage_target(v, host_targets[v])
            tr.batch_view(v, grad_scale=1.0 / b, first=j == 0, accumulate_stats=flags[lo + j],
                          staged=host_targets is not None)
        if mine:
            tr.batch_ntc_grads(defer_scatter=split)
        if split:  # (a rank without views contributes zeros: the collectives stay matched)
            nt = tr.n_table
            w1 = dist.all_reduce(tr.g_flat[nt:], op=dist.ReduceOp.SUM, group=self.group,
                                 async_op=True)  # decoder grads + loss, under the scatter
            if mine:
                tr.table_scatter()
            w2 = dist.all_reduce(tr.g_flat[:nt], op=dist.ReduceOp.SUM, group=self.group,
                                 async_op=True)
            w1.wait()
            w2.wait()
        self._losses.append(self.loss_slot.clone())
        self.loss_slot.zero_()
        tr.apply_adam()

    def step_from_host(self, batch: list[int], host_targets, accumulate_stats=False) -> float:
        """End-to-end iteration through host buffers: each view's target is
        copied from pinned host memory, the iteration runs, and the batch loss
        is read back (device -> host)."""
        self.step(batch, accumulate_stats, host_targets)
        return float(self._losses[-1].item()) / (1 if self.single else len(batch))

    def run(self, iterations: int | None = None, frame_index: int = 1) -> np.ndarray:
        """The batched Stage-1 loop: reference view sequence B views at a time,
        statistics over the last epoch's views, then the statistics all-reduce.
        Returns the batch loss per iteration (mean over the batch's views)."""
        it = iterations if iterations is not None else self.cfg.stage1_iterations
        b = self.views_per_iteration
        n_views = self.trainer.n_views
        seed = getattr(self.cfg, "seed", 0)
        stats_from = it * b - n_views
        self._losses = []
        for t, batch in enumerate(batched_view_order(seed, frame_index, n_views, it, b)):
            self.step(batch, [t * b + j >= stats_from for j in range(b)])
            if self.single:
                self._losses[-1] = self._losses[-1].clone()
        self.reduce_stats()
        return self.batch_losses()

    def reduce_stats(self) -> None:
        """Sum the per-rank view-space statistics (once per frame)."""
        if self.world > 1:
            tr = self.trainer
            dist.all_reduce(tr.stats_norm, op=dist.ReduceOp.SUM, group=self.group)
            dist.all_reduce(tr.stats_count, op=dist.ReduceOp.SUM, group=self.group)

    def batch_losses(self) -> np.ndarray:
        """Mean loss over the views of each iteration stepped so far."""
        if not self._losses:
            return np.zeros(0)
        b = 1 if self.single else self.views_per_iteration
        return torch.cat([x.reshape(1) for x in self._losses]).double().cpu().numpy() / b
