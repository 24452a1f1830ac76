"""All-core CPU Stage-1 iteration -- TEST / BASELINE INFRASTRUCTURE ONLY.

The same float64 oracle (`oracle/stage1.py`, itself a restatement of the
reference functions it cites) split over forked worker processes, so the
reference arm and `cpu_baseline` of bench.py can time one FULL-HEIGHT Stage-1
iteration on every host core instead of extrapolating a band.  Nothing here
changes the arithmetic: every piece of work is an oracle call on a slice of
the data (rows of the cloud, bands of tile rows, survivor chunks), and the
partial sums are added in the parent.  `tests/test_oracle_parallel.py` checks
the result against `stage1.stage1_iteration`.

Partition (pipeline.py:263-277):
  NTC forward + transform      inside rows       ntc.py:205-248, transform.py:53-96
  projection                   Gaussian rows     rasterizer.py:227-240 (+ global lexsort)
  blend forward / backward     tile rows (interleaved) rasterizer.py:107-211, :264-349
  loss                         colour channels   losses.py:84-148
  per-Gaussian backward        survivor chunks   rasterizer.py:351-402
  transform/MLP bwd + scatter  inside rows       transform.py:99-135, ntc.py:250-288
  Adam                         parent            optim.py:33-66

Workers are plain os.fork() children writing into MAP_SHARED anonymous
arrays allocated by the parent (no pickling); each child runs BLAS with one
thread.
"""

from __future__ import annotations

import mmap
import os
import traceback

import numpy as np

from . import stage1 as O


def shared(shape, dtype=np.float64) -> np.ndarray:
    """Zero-initialised array in anonymous shared memory (visible to forked children)."""
    shape = tuple(int(s) for s in np.atleast_1d(shape))
    count = int(np.prod(shape)) if shape else 1
    nbytes = max(count * np.dtype(dtype).itemsize, 1)
    buf = mmap.mmap(-1, nbytes, flags=mmap.MAP_SHARED)
    return np.frombuffer(buf, dtype=dtype, count=count).reshape(shape)


def _single_thread_blas():
    try:
        from threadpoolctl import threadpool_limits

        threadpool_limits(1)
    except Exception:  # pragma: no cover
        pass


def fork_map(nproc: int, fn) -> None:
    """Run fn(worker_id) in nproc forked children; raise if any failed."""
    pids = []
    for w in range(nproc):
        pid = os.fork()
        if pid == 0:  # child
            code = 0
            try:
                _single_thread_blas()
                fn(w)
            except BaseException:
                traceback.print_exc()
                code = 1
            os._exit(code)
        pids.append(pid)
    bad = 0
    for p in pids:
        _, st = os.waitpid(p, 0)
        bad += st != 0
    if bad:
        raise RuntimeError(f"{bad} oracle worker(s) failed")


def _chunks(n: int, parts: int):
    b = np.linspace(0, n, parts + 1).astype(np.int64)
    return [(int(b[i]), int(b[i + 1])) for i in range(parts)]


_PROJ_COLS = (("indices", 1), ("p_cam", 3), ("mean2d", 2), ("cov3d", 9), ("cov2d", 4),
              ("conic", 4), ("dirs", 3), ("dist", 1), ("colors", 3), ("raw", 3), ("opacity", 1))


def _band_tiles(rect, vis, ty0, ty1, ntx, ts, width, height):
    """tile_lists (rasterizer.py:107-175, oracle tile_lists) restricted to the
    tile rows [ty0, ty1): [(y0, y1, x0, x1, members)] in (ty, tx) order."""
    sel = np.flatnonzero(vis & (rect[:, 3] >= ty0) & (rect[:, 2] < ty1))
    if len(sel) == 0:
        return []
    x0, x1 = rect[sel, 0], rect[sel, 1]
    y0, y1 = np.maximum(rect[sel, 2], ty0), np.minimum(rect[sel, 3], ty1 - 1)
    wx = x1 - x0 + 1
    cnt = wx * (y1 - y0 + 1)
    ranks = np.repeat(sel, cnt)
    local = np.arange(cnt.sum()) - np.repeat(np.cumsum(cnt) - cnt, cnt)
    wxr = np.repeat(wx, cnt)
    tids = (np.repeat(y0, cnt) + local // wxr) * ntx + np.repeat(x0, cnt) + local % wxr
    order = np.lexsort((ranks, tids))
    tids, ranks = tids[order], ranks[order]
    starts = np.flatnonzero(np.r_[True, tids[1:] != tids[:-1]])
    ends = np.r_[starts[1:], len(tids)]
    out = []
    for s, e in zip(starts, ends):
        ty, tx = divmod(int(tids[s]), ntx)
        out.append((ty * ts, min(ty * ts + ts, height), tx * ts, min(tx * ts + ts, width),
                    ranks[s:e]))
    return out


class ParallelStage1:
    """One Stage-1 iteration (oracle stage1_iteration semantics) on nproc cores."""

    def __init__(self, nproc: int | None = None):
        self.nproc = int(nproc or os.cpu_count() or 1)

    # ------------------------------------------------------------------
    def render(self, cloud, cam) -> np.ndarray:
        """rasterize_forward's image (rasterizer.py:214-281), black background."""
        return np.array(self._render(cloud, cam)[4])

    def _render(self, cloud, cam):
        """Projection over Gaussian rows, the global stable depth order, then the
        forward blend over interleaved tile rows.  Returns the projected
        survivors, tile rectangles, a per-worker tile-list function and the image."""
        P = self.nproc
        n = len(cloud["means"])
        ncol = sum(c for _, c in _PROJ_COLS)
        pbuf = shared((n, ncol))
        pcount = shared(P, np.int64)
        gch = _chunks(n, P)

        def proj(wid):
            a, b = gch[wid]
            if a == b:
                return
            pj = O.project({k: v[a:b] for k, v in cloud.items()}, cam)
            m = len(pj["indices"])
            col = 0
            for name, c in _PROJ_COLS:
                v = pj[name] + (a if name == "indices" else 0)
                pbuf[a:a + m, col:col + c] = v.reshape(m, c)
                col += c
            pcount[wid] = m

        fork_map(P, proj)
        parts = np.concatenate([pbuf[a:a + int(pcount[i])] for i, (a, _) in enumerate(gch)])
        keep = parts[:, 0].astype(np.int64)
        order = np.lexsort((keep, parts[:, 3]))  # (depth, index): rasterizer.py:228-230
        parts = parts[order]
        pj, col = {}, 0
        for name, c in _PROJ_COLS:
            v = parts[:, col:col + c]
            shape = {"cov3d": (3, 3), "cov2d": (2, 2), "conic": (2, 2)}.get(name)
            pj[name] = v.reshape(-1, *shape) if shape else (v[:, 0] if c == 1 else v)
            col += c
        pj["indices"] = pj["indices"].astype(np.int64)
        s = dict(O.DEFAULT_SETTINGS)
        h, wd, ts = cam["height"], cam["width"], s["tile_size"]
        rect, vis = O.tile_rects(pj["mean2d"], pj["cov2d"], pj["opacity"], wd, h, ts,
                                 s["skip_alpha"])
        ntx, nty = (wd + ts - 1) // ts, (h + ts - 1) // ts
        # tile rows interleaved over the workers (the centre rows carry most pairs)
        bands = [[(r, r + 1) for r in range(wk, nty, P)] for wk in range(min(P, nty))]
        self._bands = bands

        def band_tiles(wid):
            return [t for band in bands[wid] for t in _band_tiles(rect, vis, *band, ntx, ts, wd, h)]

        image = shared((h, wd, 3))

        def blend(wid):
            if wid >= len(bands):
                return
            for tile in band_tiles(wid):
                y0, y1, x0, x1, mem = tile
                _, _, _, _, al, tb, alive, tf = O._tile_pairs(pj, tile, s)
                wgt = al * tb * alive
                image[y0:y1, x0:x1] = (wgt @ pj["colors"][mem]).reshape(y1 - y0, x1 - x0, 3)

        fork_map(P, blend)
        return pj, rect, vis, band_tiles, image

    # ------------------------------------------------------------------
    def _ntc_transform(self, state, cloud, rotate_sh=True):
        """NTC forward + transform of the inside rows (ntc.py:205-248,
        transform.py:53-96): the moved cloud (shared arrays) and out7."""
        P = self.nproc
        grid, mlp, tables = state["grid"], state["mlp"], state["tables"]
        inside = state["inside"]
        if state.get("enc") is None:
            state["enc"] = O.encode(grid, cloud["means"][inside])
        idx, w, _ = state["enc"]
        n_in = len(inside)
        out7 = shared((n_in, 7))
        moved = {k: shared(v.shape) for k, v in cloud.items()}
        for k in cloud:
            moved[k][...] = cloud[k]
        rows = _chunks(n_in, P)

        def fwd(wid):
            a, b = rows[wid]
            if a == b:
                return
            o7, _ = O.mlp_forward(mlp, O.gather(tables, idx[a:b], w[a:b]))
            out7[a:b] = o7
            sub = {k: v[inside[a:b]] for k, v in cloud.items()}
            mv, _ = O.transform_forward(sub, np.arange(b - a), o7, rotate_sh)
            for k in ("means", "rotations", "sh"):
                moved[k][inside[a:b]] = mv[k]

        fork_map(P, fwd)
        return moved, out7

    def transform_render(self, state, cloud, cam, rotate_sh=True) -> np.ndarray:
        """apply_ntc + rasterize_forward (pipeline.py:471-480, render-only: the
        config-2 frame), black background: the image."""
        moved, _ = self._ntc_transform(state, cloud, rotate_sh)
        return np.array(self._render(moved, cam)[4])

    # ------------------------------------------------------------------
    def iteration(self, state, cloud, cam, target, lam=0.2, lr=0.002, apply_adam=True,
                  rotate_sh=True):
        """Same contract as oracle.stage1.stage1_iteration with its defaults
        (RasterSettings(), black background, as Stage 1 renders); returns
        dict(loss, image, d_image, render_grads, g_tables, g_w, g_b)."""
        P = self.nproc
        grid, mlp, tables = state["grid"], state["mlp"], state["tables"]
        inside = state["inside"]
        n_in, n = len(inside), len(cloud["means"])
        K = cloud["sh"].shape[1]
        moved, out7 = self._ntc_transform(state, cloud, rotate_sh)
        idx, w, _ = state["enc"]
        rows = _chunks(n_in, P)
        pj, rect, vis, band_tiles, image = self._render(moved, cam)
        m = len(pj["indices"])
        s = dict(O.DEFAULT_SETTINGS)
        h, wd = cam["height"], cam["width"]
        bands = self._bands
        # ---- loss (colour channels): the 3-channel loss is the mean of the
        # per-channel losses and its gradient a third of theirs (losses.py:84-148)
        lbuf = shared(3)
        gbuf = shared((h, wd, 3))

        def loss(wid):
            if wid >= 3:
                return
            lc, gc = O.render_loss(image[..., wid], target[..., wid], lam)
            lbuf[wid] = lc
            gbuf[..., wid] = gc / 3.0

        fork_map(3, loss)
        loss_v = float(np.mean(lbuf))
        if not np.isfinite(loss_v):
            raise O.OracleNumericalError("non-finite values detected in 'stage1 loss'")
        d_img = np.array(gbuf)
        # ---- blend backward (bands), per-worker partial accumulators
        acc = shared((len(bands), m, 12))
        live = shared((len(bands), m), np.uint8)

        def blend_bwd(wid):
            if wid >= len(bands):
                return
            ac = acc[wid]
            for tile in band_tiles(wid):
                y0, y1, x0, x1, mem = tile
                dx, dy, g, og, al, tb, alive, tf = O._tile_pairs(pj, tile, s)
                gp = d_img[y0:y1, x0:x1].reshape(-1, 3)
                wgt = al * tb * alive
                np.add.at(ac[:, 0:3], mem, wgt.T @ gp)
                u = gp @ pj["colors"][mem].T
                lv = wgt > 0
                term = u * al * tb * lv
                rev = np.cumsum(term[:, ::-1], axis=1)[:, ::-1]
                suffix = np.concatenate([rev[:, 1:], np.zeros((len(gp), 1))], 1)  # bg = 0
                da = (u * tb - suffix / np.maximum(1.0 - al, 1e-12)) * alive
                da = np.where((al > 0) & (og < s["alpha_clamp"]), da, 0.0)
                np.add.at(ac[:, 3], mem, (da * g).sum(0))
                dm = -0.5 * g * da * pj["opacity"][mem][None, :]
                con = pj["conic"][mem]
                cdx = con[:, 0, 0] * dx + con[:, 0, 1] * dy
                cdy = con[:, 1, 0] * dx + con[:, 1, 1] * dy
                np.add.at(ac[:, 4:6], mem, -np.stack([(2 * cdx * dm).sum(0),
                                                      (2 * cdy * dm).sum(0)], 1))
                dxy = (dm * dx * dy).sum(0)
                np.add.at(ac[:, 6:10], mem, np.stack([(dm * dx * dx).sum(0), dxy, dxy,
                                                      (dm * dy * dy).sum(0)], 1))
                live[wid][mem] |= lv.any(0)

        fork_map(P, blend_bwd)
        tot = acc.sum(axis=0)
        ctx = dict(cloud=moved, cam=cam, settings=s, bg=np.zeros(3), proj=pj)
        out = dict(d_means=shared((n, 3)), d_rotations=shared((n, 4)), d_log_scales=shared((n, 3)),
                   d_opacity_logits=shared(n), d_sh=shared((n, K, 3)), viewspace=shared(n),
                   contributed=shared(n, np.bool_))
        live_any = live.any(axis=0)
        sch = _chunks(m, P)

        def gbwd(wid):
            a, b = sch[wid]
            if a == b:
                return
            sub = dict(ctx, proj={k: v[a:b] for k, v in pj.items()})
            O._gaussian_backward(sub, tot[a:b, 0:3], tot[a:b, 3], tot[a:b, 4:6],
                                 tot[a:b, 6:10].reshape(-1, 2, 2), live_any[a:b], out)

        fork_map(P, gbwd)
        # ---- transform / MLP backward and table scatter (inside rows)
        nw = len(mlp["weights"])
        sizes = [wi.size + bi.size for wi, bi in zip(mlp["weights"], mlp["biases"])]
        g_tab = shared((P,) + tables.shape)
        g_mlp = shared((P, sum(sizes)))

        def nbwd(wid):
            a, b = rows[wid]
            if a == b:
                return
            o7 = out7[a:b]
            ins = inside[a:b]
            tctx = dict(inside=np.arange(b - a), d_q=o7[:, 3:], u=O.qnormalize(o7[:, 3:]),
                        q_src=cloud["rotations"][ins], sh_in=cloud["sh"][ins],
                        rotate_sh=rotate_sh)
            g7 = O.transform_backward(tctx, out["d_means"][ins], out["d_rotations"][ins],
                                      out["d_sh"][ins])
            feats = O.gather(tables, idx[a:b], w[a:b])
            _, hidden = O.mlp_forward(mlp, feats)
            gw, gb, g_feats = O.mlp_backward(mlp, feats, hidden, g7)
            g_tab[wid] = O.table_scatter(tables.shape, idx[a:b], w[a:b], g_feats)
            g_mlp[wid] = np.concatenate([x.ravel() for wb in zip(gw, gb) for x in wb])

        fork_map(P, nbwd)
        gt = g_tab.sum(axis=0)
        flat = g_mlp.sum(axis=0)
        gw, gb, off = [], [], 0
        for i in range(nw):
            wi, bi = mlp["weights"][i], mlp["biases"][i]
            gw.append(flat[off:off + wi.size].reshape(wi.shape))
            off += wi.size
            gb.append(flat[off:off + bi.size].reshape(bi.shape))
            off += bi.size
        if apply_adam:
            O.adam_apply(state, gt, gw, gb, lr)
        return dict(loss=loss_v, image=np.array(image), g_tables=gt, g_w=gw, g_b=gb,
                    d_image=d_img, render_grads={k: np.array(v) for k, v in out.items()})
