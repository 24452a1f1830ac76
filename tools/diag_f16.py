"""Diagnostic: f16 decoder gradients vs the oracle's f16 / f32 restatements."""
import sys
import numpy as np
sys.path.insert(0, "/root/repo")
sys.path.insert(0, "/root/repo/tests")
import golden_io as G
from oracle import stage1 as O
from paper_2403_01444_b200 import ntc, scenes, transform, types

levels, hidden = int(sys.argv[1]), int(sys.argv[2])
dt = sys.argv[3] if len(sys.argv) > 3 else "f16"
sc = scenes.small_scene(seed=60 + levels, n=5000, sh_degree=1, levels=levels, log2_table=12)
cache = ntc.NeuralTransformationCache(types.HashGridConfig.from_any(sc.grid), hidden_layers=hidden,
                                      output_init="random", seed=levels, mlp_dtype=dt)
cache.tables[:] = scenes.f32(np.random.default_rng(7).uniform(-0.3, 0.3, size=cache.tables.shape))
cloud = types.GaussianCloud(**sc.cloud)
out, ctx = transform.apply_ntc(cloud, cache)
inside = O.inside_mask(sc.grid, sc.cloud["means"])
idx, w, _ = O.encode(sc.grid, sc.cloud["means"][inside])
feats = O.gather(cache.tables, idx, w)
rng = np.random.default_rng(5)
gm, gr = rng.normal(size=out.means.shape), rng.normal(size=(len(out.means), 4))
gs = rng.normal(size=out.sh.shape)
grads, _ = transform.apply_ntc_backward(ctx, gm, gr, gs)
for name, mlp in (("f16", dict(weights=cache.weights, biases=cache.biases, dtype="f16")),
                  ("f32", dict(weights=cache.weights, biases=cache.biases))):
    out7, hid = O.mlp_forward(mlp, feats)
    moved, octx = O.transform_forward(sc.cloud, inside, out7)
    g7 = O.transform_backward(octx, gm, gr, gs)
    gw, gb, gf = O.mlp_backward(mlp, feats, hid, g7)
    print(name, "out7 |g7|", np.abs(g7).max(axis=0))
    for i in range(hidden + 1):
        e = grads[f"w_{i}"] - gw[i]
        print(name, f"w_{i}", G.norm_rel(grads[f"w_{i}"], gw[i]), "b", G.norm_rel(grads[f"b_{i}"], gb[i]),
              "worst col", np.argmax(np.abs(e).max(axis=0)), "worst row", np.argmax(np.abs(e).max(axis=1)))
    pre = feats.astype(np.float16).astype(np.float64) @ np.asarray(cache.weights[0]).astype(np.float16).astype(np.float64)
    print(name, "pre-activation |x| < 1e-6 count", int((np.abs(pre) < 1e-6).sum()))
mlp = dict(weights=cache.weights, biases=cache.biases, dtype="f16")
out7, hid = O.mlp_forward(mlp, feats)
moved, octx = O.transform_forward(sc.cloud, inside, out7)
g7 = O.transform_backward(octx, gm, gr, gs)
gw, gb, gf = O.mlp_backward(mlp, feats, hid, g7)
e = grads["w_0"] - gw[0]
coln = np.linalg.norm(e, axis=0)
print("w_0 error by unit (top 5):", [(int(j), float(coln[j])) for j in np.argsort(-coln)[:5]],
      "total", float(np.linalg.norm(e)), "ref norm", float(np.linalg.norm(gw[0])))
pre = feats.astype(np.float16).astype(np.float64) @ np.asarray(cache.weights[0]).astype(np.float16).astype(np.float64) \
    + np.asarray(cache.biases[0]).astype(np.float16).astype(np.float64)
r, c = np.nonzero(np.abs(pre) < 1e-6)
print("near-zero pre-activations (row, unit, pre):", list(zip(r.tolist(), c.tolist(), pre[r, c].tolist())))
