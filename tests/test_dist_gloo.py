"""View-sharded data parallelism (paper_2403_01444_b200/dist.py) on CPU with gloo.

World size 2: each rank computes the oracle's per-view NTC gradients for its
shard of the batch (image gradient scaled by 1/B, as the CUDA path does),
packs them like the device buffer [tables | MLP], sum-all-reduces, and applies
the same Adam step.  The result must equal the single-process mean-of-views
gradient, and the replicas must stay identical.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2403_01444_b200.dist import allreduce_sum_, shard_views


def test_shard_views_partition():
    for b in range(1, 17):
        for w in (1, 2, 3, 4, 8):
            parts = [shard_views(list(range(b)), r, w) for r in range(w)]
            assert sum(parts, []) == list(range(b))
            assert max(map(len, parts)) - min(map(len, parts)) <= 1


def _problem():
    from oracle import stage1 as O
    from paper_2403_01444_b200 import scenes

    sc = scenes.small_scene(seed=5, n=300, width=40, height=32, sh_degree=1, n_views=4)
    tables, mlp = O.init_ntc(sc.grid, output_init="random", seed=3)
    tables = scenes.f32(np.random.default_rng(2).uniform(-0.05, 0.05, size=tables.shape))
    moved = scenes.moved_cloud(sc.cloud, np.random.default_rng(4))
    targets = [O.render(moved, c)[0]["image"] for c in sc.cameras]
    return sc, tables, mlp, targets


def _view_grad(sc, tables, mlp, target, cam, scale):
    """Flat [tables | w,b ...] NTC gradient of one view's loss times `scale`."""
    from oracle import stage1 as O

    state = dict(grid=sc.grid, tables=tables.copy(),
                 mlp=dict(weights=[w.copy() for w in mlp["weights"]],
                          biases=[b.copy() for b in mlp["biases"]]),
                 inside=O.inside_mask(sc.grid, sc.cloud["means"]), enc=None)
    r = O.stage1_iteration(state, sc.cloud, cam, target, apply_adam=False)
    parts = [r["g_tables"].ravel()]
    for w, b in zip(r["g_w"], r["g_b"]):
        parts += [w.ravel(), b.ravel()]
    return scale * np.concatenate(parts)


def _worker(rank, world, port, batch, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sc, tables, mlp, targets = _problem()
    flat = np.zeros(0)
    for v in shard_views(batch, rank, world):
        g = _view_grad(sc, tables, mlp, targets[v], sc.cameras[v], 1.0 / len(batch))
        flat = g if flat.size == 0 else flat + g
    t = torch.from_numpy(flat)
    allreduce_sum_(t, world)
    # identical Adam step on every rank (optim.py:33-66, first step)
    from oracle import stage1 as O

    p = np.zeros_like(flat)
    m, v = np.zeros_like(flat), np.zeros_like(flat)
    O.adam_update(p, t.numpy(), m, v, 1, 0.002)
    out[rank] = (t.numpy().copy(), p.copy())
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("batch", [[0, 1], [3, 0, 2]])
def test_two_rank_allreduce_equals_mean_of_views(batch):
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), batch, out), nprocs=world, join=True)
    sc, tables, mlp, targets = _problem()
    ref = sum(_view_grad(sc, tables, mlp, targets[v], sc.cameras[v], 1.0 / len(batch))
              for v in batch)
    g0, p0 = out[0]
    g1, p1 = out[1]
    np.testing.assert_array_equal(g0, g1)  # replicas see the identical reduced gradient
    np.testing.assert_array_equal(p0, p1)  # ... and stay in lock-step after Adam
    np.testing.assert_allclose(g0, ref, rtol=1e-12, atol=1e-18)
