"""Stage-1 benchmark (BASELINE.json metric): NTC train iterations/s at 1352x1014
with 250k SH-3 Gaussians (config 1), render FPS (config 2), the view-sharded
16-view batch (config 3), per-kernel rooflines and the CPU baseline, as one
JSON line.

    python bench.py [--gpus N --steps K --warmup W]           # B200 path
    python bench.py --impl reference [--steps K --warmup W]   # CPU reference arm

A "step" is one Stage-1 iteration (pipeline.py:263-277).  With N GPUs (one
process per GPU; the script re-launches itself under torch.distributed.run when
started without WORLD_SIZE) each iteration of the headline config trains N
views, one per rank, and all-reduces the NTC gradient over NCCL (view-sharded
data parallelism, weak scaling); config 3 keeps its 16 views per iteration and
splits them over the N ranks (strong scaling).
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "stage1_ntc_train_iters_per_s"
UNIT = "iter/s"
L2_FLUSH_BYTES = 256 << 20  # > 126 MB L2
FRAME = 150  # Stage-1 iterations per frame (pipeline.py:262)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip render / cfg3 / F1-F2 lines")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


# ---------------------------------------------------------------- helpers
class Clocks:
    """Samples SM clocks and throttle reasons (NVML) while the timed region runs."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x2: "applications_clocks_setting", 0x1: "gpu_idle"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.stop = [], set(), threading.Event()
        self.max_mhz = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # pragma: no cover - NVML missing
            self.nv = None

    def _run(self):
        while not self.stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        if self.nv is not None:
            self.t.join()

    def summary(self):
        s = sorted(self.samples)
        return {"sm_mhz": float(np.median(s)) if s else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(s)}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return (d["hbm_gbs"], d.get("bf16_tflops_sustained", d["bf16_tflops"]),
                "MEASURED_PEAKS.json (hbm_gbs; bf16_tflops_sustained)")
    return 6650.0, 1400.0, "fallback (B200_PROFILING.md)"


def headline_config(sc, world):
    cam = sc.cameras[0]
    return {"workload": sc.name, "gaussians": int(len(sc.cloud["means"])),
            "sh_degree": sc.sh_degree, "resolution": [cam["width"], cam["height"]],
            "views": len(sc.cameras), "views_per_iteration": world,
            "parallelism": f"view-sharded dp{world}" if world > 1 else "single",
            "ntc": "16 levels x 2 features, 2^15 rows, MLP 32-64-64-7",
            "frame": f"{FRAME} Stage-1 iterations, reference view order (pipeline.py:251-263)",
            "l2": "flushed between timed steps (256 MB write, outside the timed events)"}


def sample_positions(k: int) -> list[int]:
    """Timeline positions of the K timed iterations: K evenly spaced samples of
    the 150-iteration frame (K >= 150: every iteration, frame after frame)."""
    if k >= FRAME:
        return list(range(k))
    return [int(i * FRAME / k) for i in range(k)]


def build_problem(cfg_idx):
    """Scene, an identity-initialised NTC (ntc.py:100-128) and targets rendered on
    the device from the seeded rigid + sinusoidal motion field (synthetic data)."""
    from paper_2403_01444_b200 import scenes
    from paper_2403_01444_b200.device import DeviceCloud
    from paper_2403_01444_b200.ntc import NeuralTransformationCache
    from paper_2403_01444_b200.rasterizer import render_device
    from paper_2403_01444_b200.types import HashGridConfig

    sc = scenes.config(cfg_idx)
    # BASELINE.json configs[1] (and 3, 4 "NTC as config 1"): fp16 MLP weights
    # with fp32 accumulation; cfg0 / cfg2 fp32
    cache = NeuralTransformationCache(HashGridConfig.from_any(sc.grid), output_init="identity",
                                      mlp_dtype=sc.mlp_dtype)
    moved = scenes.moved_cloud(sc.cloud, np.random.default_rng(7), axis=(0.3, 1.0, 0.2),
                               deg=1.5, shift=(0.01, -0.005, 0.008))
    dm = DeviceCloud(moved)
    targets = [render_device(dm, cam, None, want_touch=False)[0] for cam in sc.cameras]
    return sc, cache, targets


def survivors(sc):
    """Per view, the Gaussians in front of the near plane (rasterizer.py:228), on
    the frame's source cloud (the NTC moves means by ~1e-2)."""
    m = sc.cloud["means"]
    return [int(((m @ c["w2c"][:3, :3].T + c["w2c"][:3, 3])[:, 2] > c["near"]).sum())
            for c in sc.cameras]


# algorithmic bytes (or FLOPs) per launch of each
# kernel.  N = Gaussians, n_in = inside rows, V = survivors, D = tile pairs,
# P = pixels, S = 3 K SH floats per Gaussian, LTF = table floats.
def kernel_model(name, u):
    n, n_in, V, D, P, S, ltf, npar, I = (u[k] for k in ("n", "n_in", "V", "D", "P", "S", "ltf",
                                                       "npar", "I"))
    flops_fwd = 2.0 * (I * 64 + 64 * 64 + 64 * 7)
    table = {
        "gather": ("hbm", 40 * n_in + 4 * ltf, "K1f 40N + 4LTF"),
        "decoder_forward": ("tensor", flops_fwd * n_in, "K2f 2(I*64+64*64+64*7) FLOP/row"),
        "transform": ("hbm", 156 * n_in, "K3f 156N"),
        "project": ("hbm", (44 + 4 * S + 60) * n, "K4a (44+4S)+60 per G"),
        "depth_sort": ("hbm", 24 * V, "K4b 24V"),
        "rank_scan": ("hbm", 32 * n, "K4c 32N (tile counts + prefix)"),
        "duplicate": ("hbm", 12 * D, "K4c 12D"),
        "tile_sort": ("hbm", 24 * D, "K4d 24D"),
        "ranges": ("hbm", 8 * D, "K4d 8D"),
        "blend_forward": ("hbm", 40 * D + 20 * P, "K4e 40D + 20P"),
        "ssim_map": ("hbm", 24 * P, "KL 24P of 36P (both images)"),
        "ssim_grad": ("hbm", 12 * P, "KL 12P of 36P (the gradient)"),
        "blend_backward": ("hbm", 20 * P + 40 * D + 36 * V, "K5a 20P + 40D + 36V"),
        "gaussian_backward": ("hbm", (80 + 4 * S + 72) * n, "K5b (80+4S)+72 per G"),
        "transform_vjp": ("hbm", 160 * n_in, "K3b 160N"),
        "decoder_backward": ("tensor", 2 * flops_fwd * n_in, "K2b 2x forward FLOP/row"),
        "scatter": ("hbm", 40 * n_in + 8 * ltf, "K1b 40N + 8LTF"),
        "adam": ("hbm", 28 * ltf + 28 * npar, "KA 7 LTF 4 (+7x MLP)"),
    }
    return table.get(name)


SINGLE_KERNEL = {"gather", "decoder_forward", "transform", "project", "duplicate", "ranges",
                 "blend_forward", "ssim_map", "ssim_grad", "blend_backward",
                 "gaussian_backward", "transform_vjp", "decoder_backward", "scatter", "adam"}


# ---------------------------------------------------------------- CPU arms
def _cpu_problem(cfg_idx):
    from oracle import stage1 as O
    from paper_2403_01444_b200 import scenes

    sc = scenes.config(cfg_idx)
    tables, mlp = O.init_ntc(sc.grid, output_init="identity", seed=0)
    state = dict(grid=sc.grid, tables=tables, mlp=mlp,
                 inside=O.inside_mask(sc.grid, sc.cloud["means"]), enc=None)
    state["enc"] = O.encode(sc.grid, sc.cloud["means"][state["inside"]])  # once per frame
    moved = scenes.moved_cloud(sc.cloud, np.random.default_rng(7), axis=(0.3, 1.0, 0.2),
                               deg=1.5, shift=(0.01, -0.005, 0.008))
    return sc, state, moved


def cpu_baseline_sample(cfg_idx=1):
    """One FULL-HEIGHT Stage-1 iteration of the headline workload on every host
    core: the float64 oracle port split over forked workers (oracle/parallel.py)."""
    from threadpoolctl import threadpool_limits

    from oracle import parallel
    from oracle import stage1 as O

    sc, state, moved = _cpu_problem(cfg_idx)
    cam = sc.cameras[0]
    cores = os.cpu_count() or 1
    ps = parallel.ParallelStage1(cores)
    with threadpool_limits(1):
        target = ps.render(moved, cam)  # outside the timed region
        t0 = time.perf_counter()
        ps.iteration(state, sc.cloud, cam, target)
        dt = time.perf_counter() - t0
    return {"value": 1.0 / dt, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"one full-height Stage-1 iteration of {sc.name} view 0 "
                      f"({cam['width']}x{cam['height']}, {len(sc.cloud['means'])} SH-3 Gaussians), "
                      f"float64 oracle port on {cores} forked workers (oracle/parallel.py): "
                      f"{dt:.1f} s"}


REF_VIEWS = 4


def run_reference(a):
    """The reference's CPU path (its float64 numpy algorithm, restated in
    oracle/ and pinned to it by the golden tests) on every host core, over the
    same frame schedule as the B200 arm: each step is one full-height Stage-1
    iteration (pipeline.py:263-277) of the same workload."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from threadpoolctl import threadpool_limits

    from oracle import parallel
    from paper_2403_01444_b200.stage1 import view_order

    sc, state, moved = _cpu_problem(a.config)
    cores = os.cpu_count() or 1
    ps = parallel.ParallelStage1(cores)
    world = a.gpus
    # the steps cycle over the first REF_VIEWS views of the frame's order: each
    # target is a full oracle render (~3 s on 16 cores), made once per view
    # outside the timed steps, so the wall clock stays bounded for any K
    order = view_order(0, 1, len(sc.cameras), FRAME)[:REF_VIEWS]
    targets = {}
    steps = []
    with threadpool_limits(1):
        for k in range(a.warmup + a.steps):
            v = order[k % len(order)]
            if v not in targets:  # rendered once per view, outside the timed steps
                targets[v] = ps.render(moved, sc.cameras[v])
            t0 = time.perf_counter()
            ps.iteration(state, sc.cloud, sc.cameras[v], targets[v])
            if k >= a.warmup:
                steps.append(time.perf_counter() - t0)
    ms = 1000.0 * float(np.mean(steps))
    v = 1000.0 / ms
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": headline_config(sc, 1),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": f"each step = one full-height Stage-1 iteration of "
                                       f"{sc.name} (the first {REF_VIEWS} views of the reference "
                                       f"view order, cycled), float64 oracle port on {cores} "
                                       f"forked workers; target renders outside the timed steps"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- B200 arm
def relaunch(a) -> int:
    """--gpus N without a launcher: one process per GPU via torch.distributed.run."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={a.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


class Timeline:
    """The frame schedule of a ViewShardedStage1: iteration t of the timeline is
    iteration t % 150 of a frame; frames restart from their parameters."""

    def __init__(self, vs, n_views, batch):
        from paper_2403_01444_b200.dist import batched_view_order

        self.vs, self.b = vs, batch
        self.batches = batched_view_order(0, 1, n_views, FRAME, batch)
        self.stats_from = FRAME * batch - n_views
        self.cur = 0

    def flags(self, t):
        return [t * self.b + j >= self.stats_from for j in range(self.b)]

    def run(self, t, host_targets=None):
        """Iteration t of the timeline (frame reset when a new frame starts)."""
        f = t % FRAME
        if f == 0 and t > 0:
            self.vs.trainer.reset_frame()
        self.vs.step(self.batches[f], self.flags(f), host_targets)

    def advance_to(self, p, host_targets=None):
        while self.cur < p:
            self.run(self.cur, host_targets)
            self.cur += 1


def time_positions(torch, tl, positions, flush, host_targets=None, on_step=None):
    """CUDA-event time of the iterations at `positions` of the timeline; the
    iterations in between run untimed, the L2 flush runs before each timed one
    (outside the events).  Returns per-step ms."""
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in positions]
    for k, p in enumerate(positions):
        tl.advance_to(p, host_targets)
        flush.fill_(k & 0xFF)
        ev[k][0].record()
        tl.run(p, host_targets)
        if on_step is not None:
            on_step(k)
        ev[k][1].record()
        tl.cur = p + 1
    torch.cuda.synchronize()
    return [e0.elapsed_time(e1) for e0, e1 in ev]


def max_over_ranks(torch, dist, world, x):
    if world > 1:
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())
    return x


def main():
    a = parse()
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(a))
    if a.impl == "reference":
        run_reference(a)
        return
    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    backend = os.environ.get("SS_DIST_BACKEND", "nccl")  # gloo: functional tests only
    if backend == "gloo":  # (ranks may then share a GPU; never a measurement)
        local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group(backend, device_id=torch.device("cuda", local)
                                if backend == "nccl" else None)
    from paper_2403_01444_b200 import _lib
    from paper_2403_01444_b200.dist import ViewShardedStage1
    from paper_2403_01444_b200.stage1 import Stage1Config

    lib = _lib.load()
    if "SS_MLP_MODE" in os.environ:  # decoder arithmetic (0 FFMA, 1 3xTF32, 2 tf32)
        lib.ss_set_mlp_mode(int(os.environ["SS_MLP_MODE"]))
    sc, cache, targets = build_problem(a.config)
    views = list(zip(sc.cameras, targets))
    n_views = len(views)
    vs = ViewShardedStage1(sc.cloud, cache, views, Stage1Config(), rank=rank, world=world,
                           views_per_iteration=world)
    tr = vs.trainer
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device="cuda")
    tl = Timeline(vs, n_views, world)
    # ---- warm-up: W iterations from the frame start, then one untimed pass over
    # the whole frame so every (view, statistics flag) iteration graph is
    # captured before timing; back to the frame start
    for t in range(a.warmup):
        tl.run(t)
    tl.cur = a.warmup
    tl.advance_to(FRAME)
    tr.reset_frame()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    positions = sample_positions(a.steps)
    tl.cur = 0
    l0, g0 = lib.ss_launch_count(), tr.graph_launches
    with Clocks(local) as clk:
        step_ms = time_positions(torch, tl, positions, flush)
    total_launches = lib.ss_launch_count() - l0 + tr.graph_launches - g0
    per_iter_launches = total_launches / max(1, tl.cur)
    if int(tr.check_status()) & _lib.FLAG_OVERFLOW:
        raise RuntimeError("tile-pair capacity overflow in the timed region")
    ms = max_over_ranks(torch, dist, world, float(np.mean(step_ms)))
    value = world * 1000.0 / ms  # view-iterations per second over the whole job
    # ---- per-kernel breakdown: the same timed positions replayed again from
    # the frame start, from graphs captured with event-record nodes around every
    # phase (ss_profile_enable), the L2 flushed before each timed iteration
    tr.reset_frame()
    lib.ss_profile_enable(1)
    tl.cur = 0
    tl.advance_to(FRAME)  # capture the profiled graphs
    tr.reset_frame()
    torch.cuda.synchronize()
    tl.cur = 0
    nph = lib.ss_profile_count()
    names = [lib.ss_profile_name(i).decode() for i in range(nph)]
    phase_ms = {n: [] for n in names}
    pairs = []
    buf = (np.ctypeslib.ctypes.c_double * nph)()
    for k, p in enumerate(positions):
        tl.advance_to(p)
        flush.fill_(k & 0xFF)
        tl.run(p)
        tl.cur = p + 1
        torch.cuda.synchronize()
        lib.ss_profile_read(buf, nph)
        for i, n in enumerate(names):
            if buf[i] >= 0:
                phase_ms[n].append(buf[i])
        pairs.append(int(tr.pairs_of_last(1)[0]))
    lib.ss_profile_enable(0)
    hbm, tc, peak_src = peaks()
    surv = survivors(sc)
    units = dict(n=len(sc.cloud["means"]), n_in=int(tr.rows.numel()),
                 V=float(np.mean([surv[tl.batches[p % FRAME][rank]] for p in positions])),
                 D=float(np.mean(pairs)), P=sc.cameras[0]["width"] * sc.cameras[0]["height"],
                 S=3 * sc.cloud["sh"].shape[1], ltf=int(tr.tables.numel()),
                 npar=int(tr.params.numel()), I=32)
    traffic_db = {}
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        traffic_db = json.load(open(tp)).get("per_launch_bytes", {})
    kernels = {}
    for nm, v in phase_ms.items():
        if not v:
            continue
        m = float(np.mean(v))
        model = kernel_model(nm, units)
        ent = {"ms": m, "share": m / ms, "single_kernel": nm in SINGLE_KERNEL}
        if model:
            bound, amount, formula = model
            if bound == "hbm":
                ach = amount / (m * 1e-3) / 1e9
                ent.update(bound="hbm", bytes=amount, achieved_gbs=ach, frac=ach / hbm)
            else:
                ach = amount / (m * 1e-3) / 1e12
                ent.update(bound="tensor", flops=amount, achieved_tflops=ach, frac=ach / tc)
            ent["model"] = formula
        kernels[nm] = ent
    singles = [k for k in kernels if kernels[k]["single_kernel"]]
    dom = max(singles, key=lambda k: kernels[k]["ms"])
    d = kernels[dom]
    if d["bound"] == "hbm":
        roof = {"bound": "hbm", "kernel": dom, "achieved": d["achieved_gbs"], "peak": hbm,
                "unit": "GB/s", "frac": d["frac"], "algorithmic_bytes": d["bytes"],
                "model": d["model"], "traffic": traffic_db.get(dom), "peak_source": peak_src}
    else:
        roof = {"bound": "tensor", "kernel": dom, "achieved": d["achieved_tflops"], "peak": tc,
                "unit": "TFLOP/s", "frac": d["frac"], "model": d["model"],
                "traffic": traffic_db.get(dom), "peak_source": peak_src}
    dec = kernels.get("decoder_forward")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": dict(headline_config(sc, world),
                           timed=f"{a.steps} iterations sampled evenly over the {FRAME}-iteration "
                                 f"frame (positions {positions[:3]}...{positions[-1]}); the "
                                 f"iterations between them run untimed",
                           graph_capture="every (view, statistics flag) iteration graph captured "
                                         "in one untimed pass over the frame after the warm-up",
                           kernel_times="CUDA events recorded inside the replayed iteration "
                                        "graphs (a second pass over the same positions)",
                           mean_tile_pairs=units["D"],
                           decoder=("tcgen05 kind::f16: fp16 weights and activations, fp32 "
                                    "accumulation (BASELINE configs[1])"
                                    if sc.mlp_dtype == "f16" else
                                    ["fp32 FFMA", "tcgen05 3xTF32",
                                     "tcgen05 tf32"][lib.ss_get_mlp_mode()])),
            "gpu_launches": int(round(per_iter_launches * len(positions))),
            "roofline": roof,
            "roofline_tensor": ({"kernel": "decoder_forward", "achieved": dec["achieved_tflops"],
                                 "peak": tc, "unit": "TFLOP/s", "frac": dec["frac"],
                                 "model": dec["model"]} if dec else None),
            "kernels": kernels}
    # ---- end to end through the public API with host buffers, same positions
    # and L2 policy: per step the pinned target(s) H2D, the iteration and the
    # loss D2H, all inside the step's events
    if not a.no_e2e:
        host_t = [t.cpu().pin_memory() for t in targets]
        tr.reset_frame()
        torch.cuda.synchronize()
        tl.cur = 0
        if world == 1:
            e2e_ms = _e2e_single(torch, tr, tl, positions, host_t, flush)
            path = ("Stage1Trainer.run_from_host: pinned target H2D on a copy stream (the next "
                    "step's prefetch inside the step), iteration, loss D2H every step")
        else:
            loss_host = torch.empty(len(positions), dtype=torch.float32, pin_memory=True)

            def readback(k):
                loss_host[k:k + 1].copy_(vs._losses[-1].float(), non_blocking=True)

            tl.advance_to(FRAME, host_t)  # capture the staged-target graphs
            tr.reset_frame()
            torch.cuda.synchronize()
            tl.cur = 0
            e2e_ms = time_positions(torch, tl, positions, flush, host_t, readback)
            path = "ViewShardedStage1.step(host_targets=...): pinned target H2D + iteration + loss D2H"
        e = max_over_ranks(torch, dist, world, float(np.mean(e2e_ms)))
        line["e2e"] = {"value": world * 1000.0 / e, "unit": UNIT,
                       "h2d_bytes_per_step": int(world * targets[0].numel() * 4),
                       "d2h_bytes_per_step": 8 if world == 1 else 4 * world, "path": path,
                       "ms_per_step": e}
    line["clocks"] = clk.summary()
    # ---- config 3 (16 views per iteration split over the ranks) at every N
    if not a.no_extras:
        line["cfg3"] = cfg3_rate(a, torch, dist, rank, world, flush)
    if rank == 0 and world == 1 and not a.no_extras:
        line["cfg4"] = cfg4_rate(a)
        line["render"] = render_fps(a)
        line["ntc_warmup"] = warmup_rate(sc, cache)
        line["stage2"] = stage2_rate(sc, targets)
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_sample(a.config)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def _e2e_single(torch, tr, tl, positions, host_t, flush):
    """run_from_host over the timeline up to the last timed position, events
    around the timed steps only, L2 flush before each of them.  A first untimed
    pass over the whole frame captures the staged-target iteration graphs."""
    views = [tl.batches[t][0] for t in range(FRAME)]
    flags = [tl.flags(t)[0] for t in range(FRAME)]
    tr.run_from_host(views, host_t, flags=flags)
    tr.reset_frame()
    torch.cuda.synchronize()
    n = positions[-1] + 1
    timed = {p: k for k, p in enumerate(positions)}
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in positions]

    def before(k):
        if k in timed:
            flush.fill_(timed[k] & 0xFF)
            ev[timed[k]][0].record()

    def after(k):
        if k in timed:
            ev[timed[k]][1].record()

    tr.run_from_host(views[:n], host_t, before, after, flags=flags[:n])
    torch.cuda.synchronize()
    return [e0.elapsed_time(e1) for e0, e1 in ev]


def cfg3_rate(a, torch, dist, rank, world, flush):
    """BASELINE config 3: 1M SH-3 Gaussians, 48 hemisphere cameras, 16 views per
    iteration split contiguously over the ranks, NTC gradients all-reduced per
    iteration; timed over the first iterations of the frame."""
    from paper_2403_01444_b200.dist import ViewShardedStage1
    from paper_2403_01444_b200.stage1 import Stage1Config

    sc, cache, targets = build_problem(3)
    b = sc.views_per_iteration
    vs = ViewShardedStage1(sc.cloud, cache, list(zip(sc.cameras, targets)), Stage1Config(),
                           rank=rank, world=world, views_per_iteration=b)
    tl = Timeline(vs, len(sc.cameras), b)
    # one pass over all 48 views (3 iterations) captures every graph; back to the start
    w = max(3, a.warmup)
    for t in range(w):
        tl.run(t)
    vs.trainer.reset_frame()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    k = max(3, min(a.steps, 10))
    tl.cur = 0
    ms = time_positions(torch, tl, list(range(k)), flush)
    m = max_over_ranks(torch, dist, world, float(np.mean(ms)))
    out = {"metric": "cfg3_views_per_s", "value": b * 1000.0 / m, "unit": "views/s",
           "iters_per_s": 1000.0 / m, "ms_per_iteration": m, "n_gpus": world,
           "views_per_iteration": b, "scaling": "strong", "steps": k,
           "workload": f"cfg3: {len(sc.cloud['means'])} SH-3 Gaussians, {len(sc.cameras)} "
                       f"hemisphere cameras 1352x1014, {b} views per iteration split over "
                       f"{world} rank(s), NTC gradient all-reduced per iteration "
                       f"(iterations 0..{k - 1} of the frame, L2 flushed between them)"}
    del vs
    torch.cuda.empty_cache()
    return out


def cfg4_rate(a):
    """BASELINE config 4: 3M SH-3 Gaussians at 3840x2160 (T = 2^19 NTC), one
    Stage-1 iteration per view (forward, loss, backward, NTC gradients, Adam)
    through the banded path: the view's pair count is read on the host and the
    view is binned and blended in bands of tile rows (bin workspace of
    rasterizer.BIN_PAIR_LIMIT pairs)."""
    import torch

    from paper_2403_01444_b200 import rasterizer
    from paper_2403_01444_b200.stage1 import Stage1Config, Stage1Trainer

    sc, cache, targets = build_problem(4)
    tr = Stage1Trainer(sc.cloud, cache, list(zip(sc.cameras, targets)), Stage1Config())
    pairs = tr.begin(0)
    tr.finish(0, pairs)  # warm-up (workspace, first launches)
    torch.cuda.synchronize()
    ms, counts = [], []
    for v in range(min(len(sc.cameras), max(2, a.steps // 10))):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        p = tr.begin(v)  # (reads the pair count: a host synchronisation inside the window)
        tr.finish(v, p)
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
        counts.append(p)
    m = float(np.mean(ms))
    out = {"metric": "cfg4_stage1_iters_per_s", "value": 1000.0 / m, "unit": "iter/s",
           "ms_per_iteration": m, "tile_pairs_per_view": [int(c) for c in counts],
           "bin_workspace_pairs": int(tr.bin_capacity),
           "bands": [int(-(-c // rasterizer.BIN_PAIR_LIMIT)) for c in counts],
           "workload": f"cfg4: {len(sc.cloud['means'])} SH-3 Gaussians (16 clusters, "
                       f"anisotropy <= 10:1), 3840x2160, NTC 2^19 rows; one view per iteration "
                       f"on 1 GPU (the 8-views-over-8-GPUs batch is the view-sharded path)"}
    del tr
    torch.cuda.empty_cache()
    return out


def warmup_rate(sc, cache):
    """NTC warm-up iterations/s (ntc.py:296-333) on the cfg1
    initial means, 65536-point batches, host sampling included."""
    import copy

    from paper_2403_01444_b200.warmup import warmup_train

    means = sc.cloud["means"]
    warmup_train(copy.deepcopy(cache), means, 0.05, 3)
    t0 = time.perf_counter()
    n = 20
    _, hist = warmup_train(copy.deepcopy(cache), means, 0.05, n)
    dt = time.perf_counter() - t0
    return {"metric": "ntc_warmup_iters_per_s", "value": n / dt, "unit": "iter/s",
            "batch": 65536, "loss_first_last": [hist[0], hist[-1]],
            "workload": "warmup_train on the 250k cfg1 means, noise 0.05, wall clock incl. "
                        "numpy batch sampling (Generator.choice without replacement), H2D, "
                        "device step and the final D2H"}


def stage2_rate(sc, targets):
    """Stage-2 iterations/s (adaptive.py:218-288) at cfg1 scale:
    the 250k cloud frozen, 5000 spawned additional Gaussians, 100 iterations
    (the paper's per-frame count) over the 20 device-resident views with
    quantity control at every epoch."""
    from paper_2403_01444_b200.stage2 import AdditionConfig, spawn_gaussians, stage2_optimize

    rng = np.random.default_rng(0)
    cfg = AdditionConfig()
    sel = np.sort(rng.choice(len(sc.cloud["means"]), 5000, replace=False))
    add = spawn_gaussians(sc.cloud, sel, cfg, rng)
    views = list(zip(sc.cameras, targets))
    stage2_optimize(sc.cloud, add, views[:2], cfg, 2, np.random.default_rng(1))
    n = 100
    t0 = time.perf_counter()
    out, losses = stage2_optimize(sc.cloud, add, views, cfg, n, np.random.default_rng(1))
    dt = time.perf_counter() - t0
    return {"metric": "stage2_iters_per_s", "value": n / dt, "unit": "iter/s",
            "additional": [5000, len(out.means)], "loss_first_last": [losses[0], losses[-1]],
            "workload": "stage2_optimize: 250k frozen + 5000 spawned Gaussians at 1352x1014, "
                        "100 iterations (5 epochs with split/prune), wall clock incl. per-frame "
                        "setup, the per-iteration pair-count read and the host split/prune"}


def render_fps(a):
    """Config 2: NTC transform + rasterize_forward of 300k SH-3 Gaussians per view."""
    import torch

    from paper_2403_01444_b200.stage1 import Stage1Config, Stage1Trainer

    sc, cache, targets = build_problem(2)
    tr = Stage1Trainer(sc.cloud, cache, list(zip(sc.cameras, targets)), Stage1Config())
    for v in range(len(sc.cameras)):  # one warm-up frame per view (graph capture)
        tr.render_async(v)
    torch.cuda.synchronize()
    nv = len(sc.cameras)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device="cuda")
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(2 * nv)]
    for i in range(2 * nv):
        flush.fill_(i & 0xFF)  # L2 flush between frames (outside the events)
        ev[i][0].record()
        tr.render_async(i % nv)
        ev[i][1].record()
    torch.cuda.synchronize()
    if tr.check_status() & 8:
        raise RuntimeError("tile-pair capacity overflow while rendering")
    times = [e0.elapsed_time(e1) for e0, e1 in ev]
    ms = float(np.mean(times))
    out = {"metric": "render_fps", "value": 1000.0 / ms, "unit": "frames/s", "ms_per_frame": ms,
           "workload": "cfg2: 300k SH-3 Gaussians, 1352x1014, NTC transform + forward, "
                       "20 views x 2, L2 flushed between frames"}
    if not a.no_cpu_baseline:
        out["cpu_baseline"] = cpu_render_sample()
    return out


def cpu_render_sample():
    """SURVEY 8(d8) cfg2 CPU baseline: one full frame (apply_ntc +
    rasterize_forward of view 0) of the float64 oracle port on every host core
    (oracle/parallel.py; the views are independent, so frames/s per core set)."""
    from threadpoolctl import threadpool_limits

    from oracle import parallel

    sc, state, _ = _cpu_problem(2)
    cam = sc.cameras[0]
    cores = os.cpu_count() or 1
    ps = parallel.ParallelStage1(cores)
    with threadpool_limits(1):
        t0 = time.perf_counter()
        ps.transform_render(state, sc.cloud, cam)
        dt = time.perf_counter() - t0
    return {"value": 1.0 / dt, "unit": "frames/s", "cores": cores, "kind": "port",
            "sample": f"one cfg2 frame (NTC transform + forward of {len(sc.cloud['means'])} SH-3 "
                      f"Gaussians at {cam['width']}x{cam['height']}), float64 oracle port on "
                      f"{cores} forked workers: {dt:.1f} s"}


if __name__ == "__main__":
    main()
