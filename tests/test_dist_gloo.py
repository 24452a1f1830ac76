"""View-sharded data parallelism (paper_2403_01444_b200/dist.py) on CPU with gloo.

`ViewShardedStage1` is driven at world size 2 exactly as on the GPU, with an
oracle-backed stand-in for the device trainer: each rank computes the float64
oracle's per-view NTC gradients for its shard of the batch (image gradient
scaled by 1/B, as the CUDA path does), the packed [tables | MLP | loss] buffer
is all-reduced in the two overlapped pieces, and every rank applies the same
lazy Adam step.  Checked against an independent single-process loop that
averages the per-view reference gradients and takes one Adam step per batch
(SURVEY.md section 8(e3)): parameters, batch losses, replica lock-step and the
view-space statistics window (adaptive.py:79-97, pipeline.py:259, :276-277).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2403_01444_b200.dist import ViewShardedStage1, batched_view_order, shard_views


def test_shard_views_partition():
    for b in range(1, 17):
        for w in (1, 2, 3, 4, 8):
            parts = [shard_views(list(range(b)), r, w) for r in range(w)]
            assert sum(parts, []) == list(range(b))
            assert max(map(len, parts)) - min(map(len, parts)) <= 1


def test_batched_view_order_is_the_reference_sequence():
    from oracle import stage1 as O

    seq = O.stage1_view_order(0, 3, 5, 12)
    got = batched_view_order(0, 3, 5, 4, 3)
    assert sum(got, []) == seq


def _problem():
    from oracle import stage1 as O
    from paper_2403_01444_b200 import scenes

    sc = scenes.small_scene(seed=5, n=300, width=40, height=32, sh_degree=1, n_views=4)
    tables, mlp = O.init_ntc(sc.grid, output_init="random", seed=3)
    tables = scenes.f32(np.random.default_rng(2).uniform(-0.05, 0.05, size=tables.shape))
    moved = scenes.moved_cloud(sc.cloud, np.random.default_rng(4))
    targets = [O.render(moved, c)[0]["image"] for c in sc.cameras]
    return sc, tables, mlp, targets


def _flat(g_tab, g_w, g_b):
    parts = [g_tab.ravel()]
    for w, b in zip(g_w, g_b):
        parts += [w.ravel(), b.ravel()]
    return np.concatenate(parts)


class OracleTrainer:
    """The trainer interface dist.py drives, backed by the float64 oracle."""

    def __init__(self, sc, tables, mlp, targets):
        from oracle import stage1 as O

        self.O, self.sc, self.targets = O, sc, targets
        self.n_views = len(sc.cameras)
        self.state = dict(grid=sc.grid, tables=tables.copy(),
                          mlp=dict(weights=[w.copy() for w in mlp["weights"]],
                                   biases=[b.copy() for b in mlp["biases"]]),
                          inside=O.inside_mask(sc.grid, sc.cloud["means"]), enc=None)
        self.n_table = tables.size
        self.n_params = sum(w.size + b.size for w, b in zip(mlp["weights"], mlp["biases"]))
        self.g_flat = torch.zeros(self.n_table + self.n_params + 4, dtype=torch.float64)
        n = len(sc.cloud["means"])
        self.stats_norm = torch.zeros(n, dtype=torch.float64)
        self.stats_count = torch.zeros(n, dtype=torch.int64)
        self.loss_accum = False
        self._pending = None

    def enable_loss_accum(self):
        self.loss_accum = True

    def iterate(self, view, grad_scale=1.0, adam=False, defer_scatter=False,
                accumulate_stats=False, staged=False):
        assert not adam
        r = self.O.stage1_iteration(self.state, self.sc.cloud, self.sc.cameras[view],
                                    self.targets[view], apply_adam=False)
        g = grad_scale * _flat(r["g_tables"], r["g_w"], r["g_b"])
        nt = self.n_table
        self.g_flat[nt:nt + self.n_params] += torch.from_numpy(g[nt:])
        if defer_scatter:
            self._pending = g[:nt]
        else:
            self.g_flat[:nt] += torch.from_numpy(g[:nt])
        if self.loss_accum:
            self.g_flat[nt + self.n_params] += r["loss"]
        if accumulate_stats:
            self.stats_norm += torch.from_numpy(r["render_grads"]["viewspace"])
            self.stats_count += torch.from_numpy(r["render_grads"]["contributed"].astype(np.int64))

    def batch_view(self, view, grad_scale=1.0, first=False, accumulate_stats=False,
                   staged=False):
        """One view of a batch: the oracle's gradient of this view, pending
        until batch_ntc_grads (the device runs the NTC backward once)."""
        if first:
            self._batch = None
        r = self.O.stage1_iteration(self.state, self.sc.cloud, self.sc.cameras[view],
                                    self.targets[view], apply_adam=False)
        g = grad_scale * _flat(r["g_tables"], r["g_w"], r["g_b"])
        self._batch = g if self._batch is None else self._batch + g
        if self.loss_accum:
            self.g_flat[self.n_table + self.n_params] += r["loss"]
        if accumulate_stats:
            self.stats_norm += torch.from_numpy(r["render_grads"]["viewspace"])
            self.stats_count += torch.from_numpy(r["render_grads"]["contributed"].astype(np.int64))

    def batch_ntc_grads(self, defer_scatter=False):
        g, nt = self._batch, self.n_table
        self.g_flat[nt:nt + self.n_params] += torch.from_numpy(g[nt:])
        if defer_scatter:
            self._pending = g[:nt]
        else:
            self.g_flat[:nt] += torch.from_numpy(g[:nt])

    def table_scatter(self):
        self.g_flat[:self.n_table] += torch.from_numpy(self._pending)
        self._pending = None

    def apply_adam(self):
        g = self.g_flat.numpy()
        st = self.state
        g_tab = g[:self.n_table].reshape(st["tables"].shape).copy()
        off, gw, gb = self.n_table, [], []
        for w, b in zip(st["mlp"]["weights"], st["mlp"]["biases"]):
            gw.append(g[off:off + w.size].reshape(w.shape).copy())
            off += w.size
            gb.append(g[off:off + b.size].reshape(b.shape).copy())
            off += b.size
        self.O.adam_apply(st, g_tab, gw, gb, 0.002)
        self.g_flat[:self.n_table + self.n_params] = 0.0

    def params(self):
        st = self.state
        return np.concatenate([st["tables"].ravel()] + [a.ravel() for wb in zip(
            st["mlp"]["weights"], st["mlp"]["biases"]) for a in wb])


ITERS, B = 3, 3


def _reference():
    """Independent loop: mean of per-view reference gradients, one Adam step."""
    from oracle import stage1 as O

    sc, tables, mlp, targets = _problem()
    tr = OracleTrainer(sc, tables, mlp, targets)
    batches = batched_view_order(0, 1, tr.n_views, ITERS, B)
    stats_from = ITERS * B - tr.n_views
    losses = []
    n = len(sc.cloud["means"])
    norm, count = np.zeros(n), np.zeros(n, dtype=np.int64)
    for t, batch in enumerate(batches):
        acc, lsum = 0.0, 0.0
        for j, v in enumerate(batch):
            r = O.stage1_iteration(tr.state, sc.cloud, sc.cameras[v], targets[v], apply_adam=False)
            acc = acc + _flat(r["g_tables"], r["g_w"], r["g_b"]) / len(batch)
            lsum += r["loss"]
            if t * B + j >= stats_from:
                norm += r["render_grads"]["viewspace"]
                count += r["render_grads"]["contributed"]
        tr.g_flat[:tr.n_table + tr.n_params] = torch.from_numpy(acc)
        tr.apply_adam()
        losses.append(lsum / len(batch))
    return tr.params(), np.array(losses), norm, count


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sc, tables, mlp, targets = _problem()
    tr = OracleTrainer(sc, tables, mlp, targets)

    class Cfg:
        stage1_iterations, seed = ITERS, 0

    vs = ViewShardedStage1(trainer=tr, cfg=Cfg(), rank=rank, world=world, views_per_iteration=B)
    vs.cfg = Cfg()
    losses = vs.run()
    out[rank] = (tr.params(), losses, tr.stats_norm.numpy().copy(), tr.stats_count.numpy().copy())
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_two_rank_view_sharded_loop_equals_mean_of_views():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    p_ref, l_ref, n_ref, c_ref = _reference()
    p0, l0, n0, c0 = out[0]
    p1, l1, n1, c1 = out[1]
    np.testing.assert_array_equal(p0, p1)  # replicas stay in lock-step (no broadcast)
    np.testing.assert_array_equal(l0, l1)
    np.testing.assert_allclose(p0, p_ref, rtol=1e-9, atol=1e-15)
    np.testing.assert_allclose(l0, l_ref, rtol=1e-12)
    # statistics: every view of the last epoch once, summed over the ranks
    np.testing.assert_allclose(n0, n_ref, rtol=1e-12, atol=1e-18)
    np.testing.assert_array_equal(c0, c_ref)
    np.testing.assert_array_equal(n0, n1)
    assert c_ref.max() > 0


def test_one_rank_batched_loop_equals_mean_of_views():
    sc, tables, mlp, targets = _problem()
    tr = OracleTrainer(sc, tables, mlp, targets)

    class Cfg:
        stage1_iterations, seed = ITERS, 0

    vs = ViewShardedStage1(trainer=tr, cfg=Cfg(), views_per_iteration=B)
    vs.cfg = Cfg()
    losses = vs.run()
    p_ref, l_ref, n_ref, c_ref = _reference()
    np.testing.assert_allclose(tr.params(), p_ref, rtol=1e-9, atol=1e-15)
    np.testing.assert_allclose(losses, l_ref, rtol=1e-12)
    np.testing.assert_allclose(tr.stats_norm.numpy(), n_ref, rtol=1e-12, atol=1e-18)
