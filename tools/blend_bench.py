"""Deterministic A/B timing of the raster kernels (no training trajectory):
the cfg1 cloud with its means displaced by a fixed seeded field (|d| ~ the
late-frame drift of bench.py's frame), four views, forward + backward through
the Stage-1 trainer's device path, per-phase CUDA events (graph replay).

python tools/blend_bench.py [sigma]   -> one JSON line
python tools/blend_bench.py late[:K]  -> the same on the frame's own late state:
    the cloud as transformed after K (default 144) trained iterations, saved to
    $BB_CLOUD (default /tmp/bb_late.npz) by the first run and reused by later
    ones, so A/B runs of different libraries time the same cloud"""
import os
import json
import sys

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
import bench  # noqa: E402
from paper_2403_01444_b200 import _lib, scenes  # noqa: E402
from paper_2403_01444_b200.stage1 import Stage1Config, Stage1Trainer  # noqa: E402

arg = sys.argv[1] if len(sys.argv) > 1 else "0.5"
lib = _lib.load()
sc, cache, targets = bench.build_problem(1)
cloud = dict(sc.cloud)
if arg.startswith("late"):
    from paper_2403_01444_b200.stage1 import view_order

    path = os.environ.get("BB_CLOUD", "/tmp/bb_late.npz")
    if not os.path.exists(path):
        K = int(arg.split(":")[1]) if ":" in arg else 144
        warm = bench.build_problem(1)[1]
        tr0 = Stage1Trainer(sc.cloud, warm, list(zip(sc.cameras, targets)), Stage1Config())
        order = view_order(0, 1, len(sc.cameras), 150)
        for t in range(K):
            tr0.iterate(order[t])
        torch.cuda.synchronize()
        cl = tr0.transformed_cloud()
        np.savez(path, means=cl.means, rotations=cl.rotations, log_scales=cl.log_scales,
                 opacity_logits=cl.opacity_logits, sh=cl.sh)
        del tr0
    z = np.load(path)
    cloud = {k: scenes.f32(z[k]) for k in z.files}
    sigma = arg
else:
    sigma = float(arg)
    cloud["means"] = scenes.f32(cloud["means"] + np.random.default_rng(3).normal(
        scale=sigma, size=cloud["means"].shape))
tr = Stage1Trainer(cloud, cache, list(zip(sc.cameras, targets)), Stage1Config())
views = [0, 5, 10, 15]
lib.ss_profile_enable(1)
for v in views:  # capture
    tr.iterate(v, adam=False)
torch.cuda.synchronize()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
nph = lib.ss_profile_count()
names = [lib.ss_profile_name(i).decode() for i in range(nph)]
acc = {n: [] for n in names}
buf = (np.ctypeslib.ctypes.c_double * nph)()
for rep in range(3):
    for v in views:
        flush.fill_(rep)
        tr.iterate(v, adam=False)
        torch.cuda.synchronize()
        lib.ss_profile_read(buf, nph)
        for i, n in enumerate(names):
            acc[n].append(buf[i])
out = {n: round(1000 * float(np.mean(x)), 1) for n, x in acc.items() if x}
# the same iterations from graphs without event nodes, timed whole
lib.ss_profile_enable(0)
for v in views:
    tr.iterate(v, adam=False)
torch.cuda.synchronize()
tot = []
for rep in range(3):
    for v in views:
        flush.fill_(rep)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        tr.iterate(v, adam=False)
        e1.record()
        torch.cuda.synchronize()
        tot.append(e0.elapsed_time(e1))
out["iteration_us"] = round(1000 * float(np.mean(tot)), 1)
out["sum_of_kernels_us"] = round(sum(v for k, v in out.items() if k != "iteration_us" and v > 0), 1)
out["pairs"] = int(np.mean(tr.pairs_of_last(len(views))))
out["sigma"] = sigma
print(json.dumps(out))
