"""Which Gaussians carry the banded gradient error at cfg1/cfg2 scale (diagnostic)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import stage1 as O
from paper_2403_01444_b200 import _lib, rasterizer as R, scenes, types as T

_lib.load()
for cfg, y0 in ((2, 240), (1, 496)):
    sc = scenes.config(cfg)
    cloud = T.GaussianCloud(**sc.cloud)
    counts = [R.rasterize_forward(cloud, T.Camera.from_any(c))[1].n_pairs for c in sc.cameras]
    v = int(np.argmax(counts))
    cam = dict(sc.cameras[v], height=32, cy=sc.cameras[v]["cy"] - y0)
    bg = np.array([0.05, 0.1, 0.15])
    ref, rctx = O.render(sc.cloud, cam, bg)
    out, ctx = R.rasterize_forward(cloud, T.Camera.from_any(cam), bg)
    d_img = np.random.default_rng(cfg).normal(size=out.image.shape)
    g = R.rasterize_backward(ctx, d_img)
    rg = O.render_backward(rctx, d_img)
    pj = rctx["proj"]
    rect, vis = O.tile_rects(pj["mean2d"], pj["cov2d"], pj["opacity"], cam["width"], 32, 16, 1 / 255)
    area = np.zeros(len(sc.cloud["means"]), dtype=np.int64)
    area[pj["indices"]] = (rect[:, 1] - rect[:, 0] + 1) * (rect[:, 3] - rect[:, 2] + 1) * vis
    for k in ("d_means", "d_rotations", "d_log_scales", "d_opacity_logits", "d_sh", "viewspace"):
        a = getattr(g, k if k != "viewspace" else "viewspace_grad_norm").reshape(len(area), -1)
        b = rg[k].reshape(len(area), -1)
        e = np.linalg.norm(a - b, axis=1)
        tot = np.linalg.norm(b)
        print(f"cfg{cfg} {k}: norm_rel {np.linalg.norm(a-b)/tot:.3e}")
        for i in np.argsort(-e)[:4]:
            print(f"   g{i}: err {e[i]:.3e} ref {np.linalg.norm(b[i]):.3e} got {np.linalg.norm(a[i]):.3e} "
                  f"tiles {area[i]} depth {pj['p_cam'][np.searchsorted(pj['indices'], i) if False else 0, 2]:.3f}")
    # the big ones
    big = np.argsort(-area)[:5]
    print("biggest:", [(int(i), int(area[i])) for i in big])
