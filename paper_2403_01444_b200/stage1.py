"""Device-resident Stage-1 trainer: the hot loop of `process_frame`
(pipeline.py:238-283) with every tensor in HBM and one library call per half
iteration.

    trainer = Stage1Trainer(prev_cloud, warm_cache, views)
    losses = trainer.run()            # 150 iterations, reference view order
    trainer.export_to(cache)          # parameters back into the reference-shaped cache

Per iteration (pipeline.py:263-277): apply_ntc -> rasterize_forward ->
render_loss -> rasterize_backward -> apply_ntc_backward -> lazy Adam, plus the
view-space statistics of the last epoch.  The only host synchronisation is
the tile-pair count that sizes the binning sort.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .device import (DeviceCloud, camera_struct, empty_bytes, grid_struct, mlp_layout, mlp_struct,
                     pack_params, pinned, ptr, require_cuda, settings_struct, stream, to_dev,
                     unpack_params)
from .errors import DataError
from .types import Camera, GaussianCloud, HashGridConfig, LossConfig, RasterSettings


@dataclass
class Stage1Config:
    """The Stage-1 slice of PipelineConfig (pipeline.py:40-86)."""

    stage1_iterations: int = 150
    ntc_lr: float = 0.002
    seed: int = 0
    raster: RasterSettings = field(default_factory=RasterSettings)
    loss: LossConfig = field(default_factory=LossConfig)
    rotate_sh: bool = True
    # decoder arithmetic: None = the cache's own mlp_dtype ("f32" for reference
    # caches), "f16" = fp16 weights / activations with fp32 accumulation
    mlp_dtype: str | None = None


def inside_rows(grid: HashGridConfig, means: np.ndarray) -> np.ndarray:
    """Rows the cache moves: all(lo <= mu <= hi) (transform.py:64-68); means
    are frozen for a frame so this is per-frame setup, not per-iteration work."""
    lo = np.asarray(grid.aabb_min, dtype=np.float64)
    hi = np.asarray(grid.aabb_max, dtype=np.float64)
    return np.flatnonzero(np.all((means >= lo) & (means <= hi), axis=1)).astype(np.int32)


def _spread10(v: np.ndarray) -> np.ndarray:
    v = v.astype(np.uint64) & np.uint64(0x3FF)
    v = (v | (v << np.uint64(16))) & np.uint64(0x030000FF)
    v = (v | (v << np.uint64(8))) & np.uint64(0x0300F00F)
    v = (v | (v << np.uint64(4))) & np.uint64(0x030C30C3)
    v = (v | (v << np.uint64(2))) & np.uint64(0x09249249)
    return v


def morton_rows(grid: HashGridConfig, means: np.ndarray, rows: np.ndarray) -> np.ndarray:
    """Inside rows ordered along a 30-bit Morton curve of their AABB-normalised
    position (stable for ties).  The NTC kernels run a thread per row, so this
    puts rows that share hash-grid cells in the same warp: coalesced gathers
    and warp-aggregated table scatters.  Frame setup; the order of the rows
    does not change any result."""
    if len(rows) == 0:
        return rows
    lo = np.asarray(grid.aabb_min, dtype=np.float64)
    hi = np.asarray(grid.aabb_max, dtype=np.float64)
    q = np.clip((means[rows].astype(np.float64) - lo) / (hi - lo), 0.0, 1.0)
    c = np.minimum((q * 1024.0).astype(np.int64), 1023)
    code = _spread10(c[:, 0]) | (_spread10(c[:, 1]) << np.uint64(1)) | (_spread10(c[:, 2]) << np.uint64(2))
    return rows[np.argsort(code, kind="stable")].astype(np.int32)


def view_order(seed: int, frame_index: int, n_views: int, iterations: int) -> list[int]:
    """pipeline.py:251-256, :263, :278-279."""
    rng = np.random.default_rng([seed, frame_index])
    order = rng.permutation(n_views)
    seq = []
    for t in range(iterations):
        seq.append(int(order[t % n_views]))
        if (t + 1) % n_views == 0:
            order = rng.permutation(n_views)
    return seq


class Stage1Trainer:
    def __init__(self, prev_cloud, cache, views, cfg: Stage1Config | None = None,
                 background=None, accumulate_stats: bool = True, history: int = 0):
        dev = require_cuda()
        self.lib = _lib.load()
        self.cfg = cfg or Stage1Config()
        self.dev = dev
        grid = HashGridConfig.from_any(cache.grid)
        self.grid_cfg = grid
        cloud = prev_cloud if isinstance(prev_cloud, dict) else GaussianCloud.from_any(prev_cloud)
        means_np = cloud["means"] if isinstance(cloud, dict) else cloud.means
        self.cloud = DeviceCloud(cloud, dev)
        n, K = self.cloud.n, self.cloud.sh_coeffs
        if n == 0:
            raise DataError("previous cloud is empty")
        if len(views) == 0:
            raise DataError("no training views")
        # ---- views: cameras on the host, targets resident in HBM
        self.cameras = [Camera.from_any(c) for c, _ in views]
        self.n_views = len(self.cameras)
        self.cam_structs = [camera_struct(c) for c in self.cameras]
        self.targets = [to_dev(t, dev=dev) for _, t in views]
        self.settings = settings_struct(self.cfg.raster, background)
        # ---- NTC parameters in the padded device layout
        weights = [np.asarray(w) for w in cache.weights]
        biases = [np.asarray(b) for b in cache.biases]
        self.w_shapes = [w.shape for w in weights]
        self.mlp_dtype = self.cfg.mlp_dtype or getattr(cache, "mlp_dtype", "f32")
        self.mlp = mlp_struct(weights[0].shape[0], weights[0].shape[1], len(weights) - 1,
                              self.mlp_dtype)
        self.layout = mlp_layout(self.mlp)
        self.tables = to_dev(np.asarray(cache.tables), dev=dev)
        self.params = to_dev(pack_params(weights, biases, self.layout), dev=dev)
        nt, npar = self.tables.numel(), self.params.numel()
        f32, f64 = dict(dtype=torch.float32, device=dev), dict(dtype=torch.float64, device=dev)
        # one packed gradient buffer [tables | MLP] so data parallelism needs a
        # single all-reduce (nt is a multiple of 4: the MLP part stays 16B-aligned)
        # (+ 4 floats: the batch-loss slot of view-sharded training, reduced with it)
        self.g_flat = torch.zeros(nt + npar + 4, **f32)
        self.g_tables = self.g_flat[:nt]
        self.g_params = self.g_flat[nt:nt + npar]
        self.n_table, self.n_params = nt, npar
        self.m_tables = torch.zeros(nt, **f64)
        self.v_tables = torch.zeros(nt, **f64)
        self.m_params = torch.zeros(npar, **f64)
        self.v_params = torch.zeros(npar, **f64)
        self.row_mask = torch.zeros(grid.n_levels * grid.table_size, dtype=torch.uint8, device=dev)
        self.step_dev = torch.zeros(1, dtype=torch.int32, device=dev)
        rows_idx = inside_rows(grid, means_np)
        rows_sorted = morton_rows(grid, means_np, rows_idx)
        pos = np.empty(len(rows_idx), dtype=np.int32)  # slot of rows_idx[j] in rows_sorted
        pos[np.searchsorted(rows_idx, rows_sorted)] = np.arange(len(rows_idx), dtype=np.int32)
        self.rows = to_dev(rows_sorted, dtype=torch.int32, dev=dev)
        self.rows_index = to_dev(rows_idx, dtype=torch.int32, dev=dev)
        self.rows_pos = to_dev(pos, dtype=torch.int32, dev=dev)
        # ---- transformed cloud and per-view buffers
        self.t_means = torch.empty(n, 3, **f32)
        self.t_rot = torch.empty(n, 4, **f32)
        self.t_sh = torch.empty(n, K, 3, **f32)
        H = max(c.height for c in self.cameras)
        W = max(c.width for c in self.cameras)
        self.image = torch.empty(H * W * 3, **f32)
        self.alpha = torch.empty(H * W, **f32)
        self.d_image = torch.empty(H * W * 3, **f32)
        self.d_means = torch.empty(n, 3, **f32)
        self.d_rot = torch.empty(n, 4, **f32)
        self.d_sh = torch.empty(n, K, 3, **f32)
        self.viewspace = torch.empty(n, **f32)
        self.contributed = torch.empty(n, dtype=torch.uint8, device=dev)
        self.stats_norm = torch.zeros(n, **f32)
        self.stats_count = torch.zeros(n, dtype=torch.int32, device=dev)
        self.loss_dev = torch.zeros(1, **f64)
        hist = max(1, history or self.cfg.stage1_iterations)
        self.loss_hist = torch.zeros(hist, **f64)
        self.pair_hist = torch.zeros(hist, dtype=torch.int64, device=dev)
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        self.iter_dev = torch.zeros(1, dtype=torch.int32, device=dev)
        geom = max(self.lib.ss_raster_geom_bytes(n, C.byref(cs), C.byref(self.settings))
                   for cs in self.cam_structs)
        lossb = max(self.lib.ss_loss_bytes(c.height, c.width, 3) for c in self.cameras)
        self.geom = empty_bytes(geom, dev)
        self.loss_scratch = empty_bytes(lossb, dev)
        self.bins = None
        self.bin_capacity = 0
        self.counts = pinned(2)
        self.flags = pinned(1, torch.int32)
        # ---- the ABI struct
        s = _lib.Stage1()
        s.grid = grid_struct(grid)
        s.mlp = self.mlp
        s.settings = self.settings
        s.lr, s.beta1, s.beta2, s.eps = self.cfg.ntc_lr, 0.9, 0.999, 1e-15  # optim.py:22-24
        loss = self.cfg.loss  # may be the reference's LossConfig: re-validated here
        loss = LossConfig(lambda_dssim=loss.lambda_dssim, ssim_window=loss.ssim_window,
                          ssim_sigma=loss.ssim_sigma, ssim_c1=loss.ssim_c1, ssim_c2=loss.ssim_c2)
        s.lambda_dssim = loss.lambda_dssim
        s.ssim_c1, s.ssim_c2 = loss.ssim_c1, loss.ssim_c2
        s.rotate_sh = int(self.cfg.rotate_sh)
        s.accumulate_stats = int(accumulate_stats)
        s.src = self.cloud.struct()
        s.n_in = int(self.rows.numel())
        s.rows = ptr(self.rows)
        s.rows_index = ptr(self.rows_index)
        s.rows_pos = ptr(self.rows_pos)
        for name, t in (("tables", self.tables), ("params", self.params),
                        ("g_tables", self.g_tables), ("g_params", self.g_params),
                        ("m_tables", self.m_tables), ("v_tables", self.v_tables),
                        ("m_params", self.m_params), ("v_params", self.v_params),
                        ("row_mask", self.row_mask), ("step_dev", self.step_dev),
                        ("t_means", self.t_means), ("t_rotations", self.t_rot),
                        ("t_sh", self.t_sh), ("image", self.image), ("alpha_map", self.alpha),
                        ("d_image", self.d_image), ("d_means", self.d_means),
                        ("d_rotations", self.d_rot), ("d_sh", self.d_sh),
                        ("viewspace", self.viewspace), ("contributed", self.contributed),
                        ("stats_norm", self.stats_norm), ("stats_count", self.stats_count),
                        ("loss_dev", self.loss_dev), ("loss_history", self.loss_hist),
                        ("pair_history", self.pair_hist), ("iter_dev", self.iter_dev),
                        ("status", self.status), ("geom", self.geom),
                        ("loss_scratch", self.loss_scratch)):
            setattr(s, name, ptr(t))
        s.history_len = hist
        self.ntc_scratch = empty_bytes(self.lib.ss_apply_ntc_backward_bytes(s.n_in), dev)
        s.ntc_scratch = ptr(self.ntc_scratch)
        self.s = s
        self.capacity_margin = 1.3
        self.banded = False
        self.use_graphs = True
        self._graphs = {}
        self._frame_start = (self.tables.clone(), self.params.clone())
        self.graph_launches = 0  # kernel launches issued through graph replays
        self.frame_begin()

    # ------------------------------------------------------------------
    def _call(self, fn, *args, what=""):
        _lib.check(fn(*args), what or fn.__name__)

    def reset_frame(self):
        """Back to the start of the frame: the parameters the trainer was built
        with, fresh Adam state and statistics (captured graphs stay valid)."""
        self.tables.copy_(self._frame_start[0])
        self.params.copy_(self._frame_start[1])
        self.status.zero_()
        self.frame_begin()

    def frame_begin(self):
        """clone_cache + reset_adam (pipeline.py:213-219): fresh moments, step 0."""
        self._call(self.lib.ss_stage1_frame_begin, C.byref(self.s), stream())

    def _ensure_bins(self, pairs: int, cam, exact: bool = False):
        from .rasterizer import BIN_PAIR_LIMIT

        if self.bins is not None and (pairs <= self.bin_capacity or
                                      self.bin_capacity >= BIN_PAIR_LIMIT):
            return
        cap = max(pairs if exact else int(pairs * 1.25) + 1024, 1 << 16)
        cap = min(cap, BIN_PAIR_LIMIT)  # more pairs: binned in bands of tile rows
        self._graphs = {}  # captured iterations point at the old workspace
        nbytes = self.lib.ss_raster_bin_bytes(cap, self.cloud.n, C.byref(cam),
                                              C.byref(self.settings))
        self.bins = empty_bytes(nbytes, self.dev)
        self.bin_capacity = cap
        self.s.bins = ptr(self.bins)
        self.s.bin_capacity = cap

    def begin(self, view: int) -> int:
        """apply_ntc + projection/depth sort/tile counts; returns the pair count."""
        cam = self.cam_structs[view]
        self._call(self.lib.ss_stage1_iter_begin, C.byref(self.s), C.byref(cam),
                   ptr(self.counts), stream())
        self.flags.copy_(self.status, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        _lib.check_flags(int(self.flags.item()), "stage1 loss")
        return int(self.counts[1].item())

    def stage_target(self, view: int, target_host: torch.Tensor):
        """Asynchronous H2D copy of a view's target from pinned host memory."""
        if getattr(self, "_staging", None) is None:
            self._staging = torch.empty_like(self.targets[0])
        self._staging.view(-1)[: target_host.numel()].copy_(target_host.view(-1),
                                                            non_blocking=True)

    def finish(self, view: int, pairs: int, adam: bool = True, grad_scale: float = 1.0,
               staged: bool = False, target: torch.Tensor | None = None):
        """Iteration part B with the host-known pair count (views above the bin
        workspace are binned in bands of tile rows)."""
        cam = self.cam_structs[view]
        self._ensure_bins(pairs, cam)
        tgt = ptr(target if target is not None else (self._staging if staged else self.targets[view]))
        if adam and grad_scale == 1.0:
            self._call(self.lib.ss_stage1_iter_finish, C.byref(self.s), C.byref(cam), tgt, pairs,
                       stream())
        else:
            self._call(self.lib.ss_stage1_iter_grads, C.byref(self.s), C.byref(cam), tgt, pairs,
                       C.c_float(grad_scale), stream())
            if adam:
                self.apply_adam()

    def apply_adam(self):
        self._call(self.lib.ss_stage1_apply_adam, C.byref(self.s), stream())

    def table_scatter(self):
        """The hash-table scatter deferred by iterate(..., defer_scatter=True)."""
        self._call(self.lib.ss_stage1_table_scatter, C.byref(self.s), stream())

    def enable_loss_accum(self):
        """Every iteration adds its loss to g_flat's loss slot (batch-loss sum)."""
        self.s.loss_accum = ptr(self.g_flat[self.n_table + self.n_params:])
        self._graphs = {}

    def render_async(self, view: int) -> None:
        """Forward only with no host synchronisation (ss_stage1_render), one
        CUDA-graph replay per call when graphs are on."""
        if self.bins is None:
            self.plan_capacity()

        def launch():
            self._call(self.lib.ss_stage1_render, C.byref(self.s),
                       C.byref(self.cam_structs[view]), stream())

        if not self.use_graphs:
            launch()
            return
        self._replay(("render", view), launch)

    def render(self, view: int) -> int:
        """Forward only (render-only config 2 / playback, pipeline.py:471-480):
        NTC transform + rasterize_forward of the current cache into self.image."""
        pairs = self.begin(view)
        cam = self.cam_structs[view]
        self._ensure_bins(pairs, cam)
        tc = self.cloud.struct(self.t_means, self.t_rot, self.t_sh)
        self._call(self.lib.ss_raster_forward_finish_banded, C.byref(tc), C.byref(cam),
                   C.byref(self.settings), ptr(self.geom), ptr(self.bins), self.bin_capacity,
                   pairs, ptr(self.image), ptr(self.alpha), None, stream())
        return pairs

    def plan_capacity(self, margin: float | None = None) -> int:
        """Size the tile-pair workspace for the no-sync iteration: the pair
        count of every view under the current parameters (one host read per
        view, once), times a margin for the motion Stage 1 applies."""
        from .rasterizer import BIN_PAIR_LIMIT

        m = self.capacity_margin if margin is None else margin
        peak = max(self.begin(v) for v in range(len(self.cameras)))
        cap = int(peak * m) + 65536
        # views beyond one bin workspace: every iteration reads its pair count
        # and bins in bands of tile rows (synchronous, no graphs)
        self.banded = cap > BIN_PAIR_LIMIT
        cap = min(cap, BIN_PAIR_LIMIT)
        if cap > self.bin_capacity:
            self._ensure_bins(cap, self.cam_structs[0], exact=True)
        return self.bin_capacity

    def step_from_host(self, view: int, target_host: torch.Tensor) -> float:
        """End-to-end step through host buffers: H2D copy of the view's target
        from pinned memory, the iteration, D2H read of the loss."""
        self.stage_target(view, target_host)
        self.iterate(view, staged=True)
        return float(self.loss_dev.item())

    def iterate(self, view: int, grad_scale: float = 1.0, adam: bool = True,
                staged: bool = False, target: torch.Tensor | None = None,
                graph: bool | None = None, defer_scatter: bool = False,
                accumulate_stats: bool | None = None) -> None:
        """One Stage-1 iteration with no host synchronisation (ss_stage1_iter):
        the pair count stays on the device, bounded by the planned capacity.
        `target` overrides the view's resident target (a device buffer).

        With graphs on (default), the iteration's ~40 launches are captured
        once per (view, target buffer, flags) into a CUDA graph and replayed
        as one launch; everything an iteration reads from the host (camera,
        buffers, flags) is fixed per key and the iteration index lives on the
        device, so replays are exact."""
        if self.bins is None:
            self.plan_capacity()
        if accumulate_stats is not None:
            self.s.accumulate_stats = int(accumulate_stats)
        self.s.defer_scatter = int(defer_scatter)
        if self.banded:
            pairs = self.begin(view)
            self.finish(view, pairs, adam=adam, grad_scale=grad_scale, staged=staged,
                        target=target)
            return
        use = self.use_graphs if graph is None else graph
        if not use:
            self._iterate_eager(view, grad_scale, adam, staged, target)
            return
        buf = target if target is not None else (self._staging if staged else None)
        key = (view, None if buf is None else buf.data_ptr(), int(self.s.accumulate_stats),
               bool(adam), float(grad_scale), bool(defer_scatter),
               int(self.lib.ss_profile_enabled()))  # profiled graphs hold event nodes
        self._replay(key, lambda: self._iterate_eager(view, grad_scale, adam, staged, target))

    def batch_view(self, view: int, grad_scale: float, first: bool, staged: bool = False,
                   accumulate_stats: bool | None = None) -> None:
        """One view of a batch that shares the parameter state (ss_stage1_batch_view):
        render, loss and raster backward, its transformed-cloud gradient added
        to the batch's (first: NTC forward + transform, gradient overwritten).
        The NTC backward runs once per batch in batch_ntc_grads()."""
        if self.bins is None:
            self.plan_capacity()
        if self.banded:
            raise DataError("views above the bin workspace train one view per iteration")
        if accumulate_stats is not None:
            self.s.accumulate_stats = int(accumulate_stats)
        cam = self.cam_structs[view]

        def launch():
            tgt = ptr(self._staging if staged else self.targets[view])
            self._call(self.lib.ss_stage1_batch_view, C.byref(self.s), C.byref(cam), tgt,
                       C.c_float(grad_scale), int(bool(first)), stream())

        if not self.use_graphs:
            launch()
            return
        key = ("batch", view, bool(first), float(grad_scale), int(self.s.accumulate_stats),
               self._staging.data_ptr() if staged else None,
               int(self.lib.ss_profile_enabled()))
        self._replay(key, launch)

    def batch_ntc_grads(self, defer_scatter: bool = False) -> None:
        """Transform VJP + decoder backward (+ table scatter unless deferred) of
        the accumulated batch gradient (ss_stage1_batch_ntc_grads)."""
        self.s.defer_scatter = int(defer_scatter)

        def launch():
            self._call(self.lib.ss_stage1_batch_ntc_grads, C.byref(self.s), stream())

        if not self.use_graphs:
            launch()
            return
        self._replay(("batch_ntc", bool(defer_scatter), int(self.lib.ss_profile_enabled())), launch)

    def _replay(self, key, launch) -> None:
        """Capture `launch` into a CUDA graph on first use of `key`, then replay.
        Kernel nodes per graph are counted (graph_launches) for telemetry."""
        ent = self._graphs.get(key)
        if ent is None:
            g = torch.cuda.CUDAGraph()
            torch.cuda.synchronize()
            l0 = self.lib.ss_launch_count()
            with torch.cuda.graph(g):
                launch()
            ent = (g, self.lib.ss_launch_count() - l0)
            self._graphs[key] = ent
        ent[0].replay()
        self.graph_launches += ent[1]

    def _iterate_eager(self, view, grad_scale, adam, staged, target):
        cam = self.cam_structs[view]
        if target is not None:
            tgt = ptr(target)
        else:
            tgt = ptr(self._staging if staged else self.targets[view])
        self._call(self.lib.ss_stage1_iter, C.byref(self.s), C.byref(cam), tgt,
                   C.c_float(grad_scale), int(adam), stream())

    def step(self, view: int) -> None:
        self.iterate(view)

    def run_from_host(self, order: list[int], host_targets, before_step=None,
                      after_step=None, flags=None) -> np.ndarray:
        """Stage-1 iterations whose targets live in pinned HOST memory: each
        iteration's target is copied host->device on a copy stream while the
        previous iteration computes (two staging buffers), and each
        iteration's loss is read device->host into pinned memory.  One
        synchronisation at the end; returns the per-iteration losses.

        before_step(k) / after_step(k) run on the host around step k's work;
        everything step k puts on the device -- its own target copy if not
        already prefetched, the prefetch of step k+1's target, the iteration,
        the loss read-back -- is stream-ordered between them (a timer can
        record CUDA events there).  flags: per-step accumulate_stats."""
        dev = self.dev
        main = torch.cuda.current_stream(dev)
        copy = getattr(self, "_copy_stream", None) or torch.cuda.Stream(dev)
        self._copy_stream = copy
        if getattr(self, "_stage2", None) is None:
            self._stage2 = [torch.empty_like(self.targets[0]) for _ in range(2)]
        ready = [torch.cuda.Event() for _ in range(2)]
        losses = torch.empty(len(order), dtype=torch.float64, pin_memory=True)

        def h2d(k):
            b = k & 1
            copy.wait_stream(main)  # buffer b is free, and the copy starts inside step k-1
            with torch.cuda.stream(copy):
                t = host_targets[order[k]]
                self._stage2[b].view(-1)[: t.numel()].copy_(t.view(-1), non_blocking=True)
                ready[b].record(copy)

        for k, v in enumerate(order):
            if before_step is not None:
                before_step(k)
            if k == 0:
                h2d(0)
            if k + 1 < len(order):
                h2d(k + 1)
            main.wait_event(ready[k & 1])
            self.iterate(v, target=self._stage2[k & 1],
                         accumulate_stats=None if flags is None else flags[k])
            losses[k:k + 1].copy_(self.loss_dev, non_blocking=True)
            if k + 1 < len(order):
                main.wait_event(ready[(k + 1) & 1])  # the prefetch counts in this step
            if after_step is not None:
                after_step(k)
        main.synchronize()
        return losses.numpy().copy()

    def pairs_of_last(self, k: int) -> np.ndarray:
        """Tile-pair counts of the last k iterations (device history; syncs)."""
        h, it = self.pair_hist.numel(), int(self.iter_dev.item())
        idx = [(it - k + j) % h for j in range(k)]
        return self.pair_hist.cpu().numpy()[idx]

    def check_status(self, what: str = "stage1 loss") -> int:
        self.flags.copy_(self.status, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return int(self.flags.item())

    def run(self, iterations: int | None = None, frame_index: int = 1) -> np.ndarray:
        """The Stage-1 loop (pipeline.py:262-279); returns the loss history.
        Iterations queue back to back without host synchronisation; if the
        pair capacity overflowed, the frame is replayed from its starting
        parameters with a larger workspace."""
        iters = self.cfg.stage1_iterations if iterations is None else iterations
        if iters > self.loss_hist.numel():
            self.loss_hist = torch.zeros(iters, dtype=torch.float64, device=self.dev)
            self.pair_hist = torch.zeros(iters, dtype=torch.int64, device=self.dev)
            self.s.loss_history = ptr(self.loss_hist)
            self.s.pair_history = ptr(self.pair_hist)
            self.s.history_len = iters
            self._graphs = {}
        order = view_order(self.cfg.seed, frame_index, len(self.cameras), iters)
        stats_from = max(0, iters - len(self.cameras))
        if self.bins is None:
            self.plan_capacity()
        start = (self.tables.clone(), self.params.clone())
        for attempt in range(4):
            for t, v in enumerate(order):
                self.s.accumulate_stats = int(t >= stats_from)
                self.iterate(v)
            flags = self.check_status()
            if not flags & _lib.FLAG_OVERFLOW:
                break
            # replay the frame from its start with a larger pair workspace
            peak = int(self.pair_hist[:iters].max().item())
            self.tables.copy_(start[0])
            self.params.copy_(start[1])
            self.status.zero_()
            self._ensure_bins(int(max(peak, self.bin_capacity) * 1.5), self.cam_structs[0],
                              exact=True)
            self.frame_begin()
        _lib.check_flags(flags, "stage1 loss")
        return self.loss_hist[:iters].cpu().numpy()

    # ------------------------------------------------------------------
    def last_loss(self) -> float:
        return float(self.loss_dev.item())

    def rendered_image(self, view: int) -> np.ndarray:
        c = self.cameras[view]
        return self.image[: c.height * c.width * 3].view(c.height, c.width, 3).cpu().numpy()

    def transformed_cloud(self) -> GaussianCloud:
        return GaussianCloud(self.t_means.cpu().numpy(), self.t_rot.cpu().numpy(),
                             self.cloud.log_scales.cpu().numpy(),
                             self.cloud.opacity_logits.cpu().numpy(), self.t_sh.cpu().numpy())

    def ntc_grads(self):
        """Current (un-stepped) NTC gradients in the reference layout."""
        g = self.g_params.cpu().numpy()
        ws, bs = unpack_params(g, self.w_shapes, self.layout)
        tab = self.g_tables.view(self.tables.shape).cpu().numpy().astype(np.float64)
        return tab, ws, bs

    def export_to(self, cache) -> None:
        """Write the device parameters back into a reference-shaped cache."""
        cache.tables[:] = self.tables.cpu().numpy()
        ws, bs = unpack_params(self.params.cpu().numpy(), self.w_shapes, self.layout)
        for i in range(len(ws)):
            cache.weights[i][:] = ws[i]
            cache.biases[i][:] = bs[i]

    def viewspace_stats(self):
        """(norm_accum, view_count) of ViewspaceStats (adaptive.py:79-97)."""
        return (self.stats_norm.cpu().numpy().astype(np.float64),
                self.stats_count.cpu().numpy().astype(np.int64))
