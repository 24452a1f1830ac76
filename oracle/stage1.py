"""Float64 numpy restatement of the reference Stage-1 hot path (CPU oracle).

TEST INFRASTRUCTURE ONLY -- see `oracle/__init__.py`.  Every function cites
the reference lines it restates (paths relative to
`/root/reference/pkg/src/splatstream/`).  The code is organised around flat
arrays and dicts rather than the reference's classes so the same routines
serve the parity tests, the golden-vector generator and the CPU baseline.

Containers used here (all float64 numpy unless noted):
  cloud  = dict(means (N,3), rotations (N,4) wxyz, log_scales (N,3),
                opacity_logits (N,), sh (N,K,3) with K=(deg+1)^2)
  camera = dict(w2c (4,4), fx, fy, cx, cy, width, height, near)
  grid   = dict(levels, features, log2_table, base, growth, lo (3,), hi (3,))
  mlp    = dict(weights [W_i (fan_in, fan_out)], biases [b_i], optional dtype "f16")
"""

from __future__ import annotations

import math

import numpy as np

# ---------------------------------------------------------------------------
# constants
# ---------------------------------------------------------------------------
HASH_PRIMES = (1, 2654435761, 805459861)  # ntc.py:23
LOWPASS = 0.3  # cameras.py:27
SH_C0 = 0.28209479177387814  # sh.py:26
SH_C1 = 0.4886025119029199  # sh.py:27
# degree 2/3: orthonormal real SH *without* the Condon-Shortley phase, which is
# the convention the reference's degree-1 basis (+y, +z, +x) follows.
# (extension; parity unpinned)
SH_C2 = (1.0925484305920792, 0.31539156525252005, 0.5462742152960396)
SH_C3 = (0.5900435899266435, 2.890611442640554, 0.4570457994644658,
         0.3731763325901154, 1.445305721320277)


class OracleDataError(ValueError):
    """Mirror of splatstream.errors.DataError (errors.py:12-13)."""


class OracleNumericalError(ArithmeticError):
    """Mirror of splatstream.errors.NumericalError (errors.py:20-21)."""


# ---------------------------------------------------------------------------
# hash grid (ntc.py)
# ---------------------------------------------------------------------------
def level_resolutions(base: int, growth: float, levels: int) -> list[int]:
    """floor(base * growth**l) in float64, ntc.py:54-55 (host-side, D9)."""
    return [int(np.floor(base * growth ** l)) for l in range(levels)]


def growth_for(base: int, finest: int, levels: int) -> float:
    """ntc.py:57-61."""
    if levels <= 1:
        return 1.0
    return float((finest / base) ** (1.0 / (levels - 1)))


def encode(grid: dict, x: np.ndarray):
    """Corner rows and trilinear weights, ntc.py:161-203.

    Returns idx (B, L, 8) int64, w (B, L, 8) float64, touched [unique rows per
    level].  Corner k has offsets (k&1, k>>1&1, k>>2&1): x fastest (ntc.py:25-27).
    """
    x = np.asarray(x, dtype=np.float64).reshape(-1, 3)
    lo = np.asarray(grid["lo"], dtype=np.float64)
    hi = np.asarray(grid["hi"], dtype=np.float64)
    xn = (x - lo) / (hi - lo)
    if xn.size and (xn.min() < -1e-9 or xn.max() > 1.0 + 1e-9):
        raise OracleDataError("point outside the hash grid bounding box")
    xn = np.clip(xn, 0.0, 1.0)
    levels = grid["levels"]
    table = 1 << grid["log2_table"]
    res_list = level_resolutions(grid["base"], grid["growth"], levels)
    b = len(x)
    idx = np.empty((b, levels, 8), dtype=np.int64)
    w = np.empty((b, levels, 8))
    touched = []
    for l, res in enumerate(res_list):
        pos = xn * res
        c0 = np.minimum(np.floor(pos), res - 1).astype(np.int64)
        frac = pos - c0
        dense = (res + 1) ** 3 <= table
        for k in range(8):
            off = np.array([k & 1, (k >> 1) & 1, (k >> 2) & 1])
            c = c0 + off
            t = np.where(off.astype(bool), frac, 1.0 - frac)
            w[:, l, k] = t[:, 0] * t[:, 1] * t[:, 2]
            if dense:
                s = res + 1
                idx[:, l, k] = c[:, 0] + s * (c[:, 1] + s * c[:, 2])
            else:
                h = (c[:, 0] * HASH_PRIMES[0]) ^ (c[:, 1] * HASH_PRIMES[1]) ^ (
                    c[:, 2] * HASH_PRIMES[2])
                idx[:, l, k] = h % table
        touched.append(np.unique(idx[:, l]))
    return idx, w, touched


def gather(tables: np.ndarray, idx: np.ndarray, w: np.ndarray) -> np.ndarray:
    """feats[b, l*F + f] = sum_k w[b,l,k] tables[l, idx[b,l,k], f]; ntc.py:205-216."""
    b, levels, _ = idx.shape
    feats = np.empty((b, levels, tables.shape[2]))
    for l in range(levels):
        feats[:, l] = np.einsum("bk,bkf->bf", w[:, l], tables[l][idx[:, l]])
    return feats.reshape(b, -1)


def _f16(a):
    return np.asarray(a).astype(np.float16).astype(np.float64)


def _mlp_operands(mlp: dict):
    """The decoder's operands.  mlp["dtype"] == "f16" (BASELINE config 1's
    fp16 MLP weights, fp32 accumulation -- not a reference mode: the reference
    is float64, ntc.py:241-276) rounds weights, biases, the input features and
    every hidden activation to float16 (round to nearest even) and accumulates
    exactly, as the tensor-core kernel does up to fp32 summation order."""
    if mlp.get("dtype", "f32") == "f16":
        return [_f16(w) for w in mlp["weights"]], [_f16(b) for b in mlp["biases"]], _f16
    return mlp["weights"], mlp["biases"], lambda a: a


def mlp_forward(mlp: dict, feats: np.ndarray):
    """ReLU hidden layers, linear output; ntc.py:241-248."""
    ws, bs, rnd = _mlp_operands(mlp)
    z = rnd(feats)
    hidden = []
    for wi, bi in zip(ws[:-1], bs[:-1]):
        z = rnd(np.maximum(z @ wi + bi, 0.0))
        hidden.append(z)
    out = z @ ws[-1] + bs[-1]
    return out, hidden


def mlp_backward(mlp: dict, feats, hidden, g_out):
    """dW, db and dL/dfeats; ntc.py:258-276 (f16: the straight-through
    gradient of the rounded forward, see _mlp_operands)."""
    ws, _, rnd = _mlp_operands(mlp)
    ins = [rnd(feats)] + hidden
    delta = g_out
    gw, gb = [None] * len(ws), [None] * len(ws)
    for i in range(len(ws) - 1, -1, -1):
        gw[i] = ins[i].T @ delta
        gb[i] = delta.sum(axis=0)
        delta = delta @ ws[i].T
        if i > 0:
            delta = delta * (hidden[i - 1] > 0)
    return gw, gb, delta


def table_scatter(shape, idx, w, g_feats):
    """Dense per-level table gradients via unbuffered add; ntc.py:278-288."""
    levels, t, f = shape
    b = idx.shape[0]
    g = np.zeros(shape)
    gf = g_feats.reshape(b, levels, f)
    for l in range(levels):
        contrib = w[:, l, :, None] * gf[:, l, None, :]
        np.add.at(g[l], idx[:, l].ravel(), contrib.reshape(-1, f))
    return g


def init_ntc(grid: dict, hidden_dim=64, hidden_layers=2, output_init="identity", seed=0):
    """Parameter init and float32 quantisation; ntc.py:100-128."""
    rng = np.random.default_rng(seed)
    levels, f = grid["levels"], grid["features"]
    tables = rng.uniform(-1e-4, 1e-4, size=(levels, 1 << grid["log2_table"], f))
    dims = [levels * f] + [hidden_dim] * hidden_layers
    weights, biases = [], []
    for a, b in zip(dims[:-1], dims[1:]):
        bound = np.sqrt(6.0 / (a + b))
        weights.append(rng.uniform(-bound, bound, size=(a, b)))
        biases.append(np.zeros(b))
    if output_init == "identity":
        weights.append(np.zeros((dims[-1], 7)))
        ob = np.zeros(7)
        ob[3] = 1.0
        biases.append(ob)
    else:
        bound = np.sqrt(6.0 / (dims[-1] + 7))
        weights.append(rng.uniform(-bound, bound, size=(dims[-1], 7)))
        biases.append(rng.normal(scale=0.1, size=7))
    q = lambda a: a.astype(np.float32).astype(np.float64)  # noqa: E731
    return q(tables), {"weights": [q(a) for a in weights], "biases": [q(a) for a in biases]}


def adam_update(p, g, m, v, step, lr, rows=None, b1=0.9, b2=0.999, eps=1e-15):
    """One Adam update in place (step already incremented); optim.py:33-66.

    `rows` restricts the update to those first-axis rows (lazy branch :60-66).
    """
    bc1 = 1.0 - b1 ** step
    bc2 = 1.0 - b2 ** step
    if rows is None:
        m *= b1
        m += (1.0 - b1) * g
        v *= b2
        v += (1.0 - b2) * (g * g)
        p -= lr * (m / bc1) / (np.sqrt(v / bc2) + eps)
    else:
        gr = g[rows]
        m[rows] = b1 * m[rows] + (1.0 - b1) * gr
        v[rows] = b2 * v[rows] + (1.0 - b2) * (gr * gr)
        p[rows] -= lr * (m[rows] / bc1) / (np.sqrt(v[rows] / bc2) + eps)


# ---------------------------------------------------------------------------
# quaternions (gaussians.py)
# ---------------------------------------------------------------------------
def qnormalize(q, eps=1e-12):
    """gaussians.py:42-48 (raises NumericalError on |q| < eps)."""
    n = np.linalg.norm(q, axis=-1, keepdims=True)
    if np.any(n < eps):
        raise OracleNumericalError("cannot normalize near-zero quaternion")
    return q / n


def qmul(a, b):
    """Hamilton product, wxyz; gaussians.py:51-65."""
    aw, ax, ay, az = np.moveaxis(a, -1, 0)
    bw, bx, by, bz = np.moveaxis(b, -1, 0)
    return np.stack([aw * bw - ax * bx - ay * by - az * bz,
                     aw * bx + ax * bw + ay * bz - az * by,
                     aw * by - ax * bz + ay * bw + az * bx,
                     aw * bz + ax * by - ay * bx + az * bw], axis=-1)


def qrot(q):
    """Polynomial rotation matrix of a unit quaternion; gaussians.py:68-85."""
    w, x, y, z = np.moveaxis(q, -1, 0)
    r = np.empty(q.shape[:-1] + (3, 3))
    r[..., 0, 0] = 1 - 2 * (y * y + z * z)
    r[..., 0, 1] = 2 * (x * y - w * z)
    r[..., 0, 2] = 2 * (x * z + w * y)
    r[..., 1, 0] = 2 * (x * y + w * z)
    r[..., 1, 1] = 1 - 2 * (x * x + z * z)
    r[..., 1, 2] = 2 * (y * z - w * x)
    r[..., 2, 0] = 2 * (x * z - w * y)
    r[..., 2, 1] = 2 * (y * z + w * x)
    r[..., 2, 2] = 1 - 2 * (x * x + y * y)
    return r


def qrot_vjp(q, g_r):
    """sum_ij g_r[ij] dR_ij/dq_k for the polynomial map; gaussians.py:88-106."""
    w, x, y, z = np.moveaxis(q, -1, 0)
    g = g_r
    gw = 2 * (-z * g[..., 0, 1] + y * g[..., 0, 2] + z * g[..., 1, 0]
              - x * g[..., 1, 2] - y * g[..., 2, 0] + x * g[..., 2, 1])
    gx = 2 * (y * g[..., 0, 1] + z * g[..., 0, 2] + y * g[..., 1, 0] - 2 * x * g[..., 1, 1]
              - w * g[..., 1, 2] + z * g[..., 2, 0] + w * g[..., 2, 1] - 2 * x * g[..., 2, 2])
    gy = 2 * (-2 * y * g[..., 0, 0] + x * g[..., 0, 1] + w * g[..., 0, 2] + x * g[..., 1, 0]
              + z * g[..., 1, 2] - w * g[..., 2, 0] + z * g[..., 2, 1] - 2 * y * g[..., 2, 2])
    gz = 2 * (-2 * z * g[..., 0, 0] - w * g[..., 0, 1] + x * g[..., 0, 2] + w * g[..., 1, 0]
              - 2 * z * g[..., 1, 1] + y * g[..., 1, 2] + x * g[..., 2, 0] + y * g[..., 2, 1])
    return np.stack([gw, gx, gy, gz], axis=-1)


def qnormalize_vjp(q, g_u):
    """g_u (I - u u^T)/|q|; gaussians.py:109-117."""
    n = np.linalg.norm(q, axis=-1, keepdims=True)
    if np.any(n < 1e-12):
        raise OracleNumericalError("cannot normalize near-zero quaternion")
    u = q / n
    return (g_u - u * np.sum(u * g_u, axis=-1, keepdims=True)) / n


def quat_right_matrix(q):
    """A(q) with A(q) p = p (x) q; transform.py:43-50."""
    w, x, y, z = np.moveaxis(q, -1, 0)
    return np.stack([np.stack([w, -x, -y, -z], -1), np.stack([x, w, z, -y], -1),
                     np.stack([y, -z, w, x], -1), np.stack([z, y, -x, w], -1)], -2)


# ---------------------------------------------------------------------------
# spherical harmonics (sh.py, degree 0-1; 2-3 = unpinned extension)
# ---------------------------------------------------------------------------
def sh_degree_of(k: int) -> int:
    d = int(round(math.sqrt(k))) - 1
    if (d + 1) ** 2 != k or d > 3:
        raise OracleDataError(f"unsupported SH coefficient count {k}")
    return d


def sh_basis(d, deg):
    """(..., K) basis at directions d (..., 3); sh.py:35-42 for deg <= 1."""
    x, y, z = d[..., 0], d[..., 1], d[..., 2]
    out = [np.full(x.shape, SH_C0)]
    if deg >= 1:
        out += [SH_C1 * y, SH_C1 * z, SH_C1 * x]
    if deg >= 2:
        a, b, c = SH_C2
        out += [a * x * y, a * y * z, b * (2 * z * z - x * x - y * y), a * x * z,
                c * (x * x - y * y)]
    if deg >= 3:
        c3, c2, c1, c0, c2h = SH_C3
        out += [c3 * y * (3 * x * x - y * y), c2 * x * y * z,
                c1 * y * (4 * z * z - x * x - y * y),
                c0 * z * (2 * z * z - 3 * x * x - 3 * y * y),
                c1 * x * (4 * z * z - x * x - y * y), c2h * z * (x * x - y * y),
                c3 * x * (x * x - 3 * y * y)]
    return np.stack(out, axis=-1)


def sh_basis_jac(d, deg):
    """(..., K, 3) d basis_k / d d_j of the polynomial forms in sh_basis."""
    x, y, z = d[..., 0], d[..., 1], d[..., 2]
    zero = np.zeros_like(x)
    rows = [(zero, zero, zero)]
    if deg >= 1:
        c = SH_C1
        rows += [(zero, c + zero, zero), (zero, zero, c + zero), (c + zero, zero, zero)]
    if deg >= 2:
        a, b, c = SH_C2
        rows += [(a * y, a * x, zero), (zero, a * z, a * y),
                 (-2 * b * x, -2 * b * y, 4 * b * z), (a * z, zero, a * x),
                 (2 * c * x, -2 * c * y, zero)]
    if deg >= 3:
        c3, c2, c1, c0, c2h = SH_C3
        rows += [(6 * c3 * x * y, c3 * (3 * x * x - 3 * y * y), zero),
                 (c2 * y * z, c2 * x * z, c2 * x * y),
                 (-2 * c1 * x * y, c1 * (4 * z * z - x * x - 3 * y * y), 8 * c1 * y * z),
                 (-6 * c0 * x * z, -6 * c0 * y * z, c0 * (6 * z * z - 3 * x * x - 3 * y * y)),
                 (c1 * (4 * z * z - 3 * x * x - y * y), -2 * c1 * x * y, 8 * c1 * x * z),
                 (2 * c2h * x * z, -2 * c2h * y * z, c2h * (x * x - y * y)),
                 (c3 * (3 * x * x - 3 * y * y), -6 * c3 * x * y, zero)]
    return np.stack([np.stack(r, axis=-1) for r in rows], axis=-2)


_PERM = np.array([[0.0, 1.0, 0.0], [0.0, 0.0, 1.0], [1.0, 0.0, 0.0]])  # sh.py:30-32

# sample directions for band rotations of degree 2-3 (oracle-only; independent
# of the CUDA library's own set -- M does not depend on the choice)
_LS_DIRS = {}


def _ls_dirs(l):
    if l not in _LS_DIRS:
        r = np.random.default_rng(20240302 + l).normal(size=(2 * l + 1, 3))
        d = r / np.linalg.norm(r, axis=1, keepdims=True)
        assert np.linalg.cond(sh_basis(d, l)[:, _band(l)]) < 1e3
        _LS_DIRS[l] = d
    return _LS_DIRS[l]


def _band(l):
    return slice(l * l, (l + 1) * (l + 1))


def sh_band_rotation(rot, l):
    """(..., 2l+1, 2l+1) M with f'(d) = f(R^T d) coefficient-wise.

    l = 1 is the reference's P R P^T (sh.py:84-109).  l = 2, 3 solve the same
    identity exactly on 2l+1 fixed directions (extension).
    """
    if l == 1:
        return _PERM @ rot @ _PERM.T
    s = _ls_dirs(l)
    ys = sh_basis(s, l)[:, _band(l)]  # (n, 2l+1)
    pinv = np.linalg.pinv(ys)
    e = np.einsum("...ji,kj->...ki", rot, s)  # R^T s_k
    ye = sh_basis(e, l)[..., _band(l)]  # (..., n, 2l+1)
    return np.einsum("ak,...kb->...ab", pinv, ye)


def sh_band_rotation_vjp(rot, l, g_m):
    """dL/dR from dL/dM for sh_band_rotation; sh.py:103-109 for l = 1."""
    if l == 1:
        return _PERM.T @ g_m @ _PERM
    s = _ls_dirs(l)
    pinv = np.linalg.pinv(sh_basis(s, l)[:, _band(l)])
    e = np.einsum("...ji,kj->...ki", rot, s)
    jac = sh_basis_jac(e, l)[..., _band(l), :]  # (..., n, 2l+1, 3)
    g_y = np.einsum("ak,...ab->...kb", pinv, g_m)  # (..., n, 2l+1)
    g_e = np.einsum("...kb,...kbj->...kj", g_y, jac)  # (..., n, 3)
    # e_k,i = sum_j R_ji s_kj  ->  dL/dR_ji = sum_k s_kj g_e_ki
    return np.einsum("kj,...ki->...ji", s, g_e)


def colors_forward(sh, dirs):
    """clip(0.5 + basis . sh, 0, 1) and raw values; sh.py:51-59."""
    deg = sh_degree_of(sh.shape[1])
    raw = 0.5 + np.einsum("nk,nkc->nc", sh_basis(dirs, deg), sh)
    return np.clip(raw, 0.0, 1.0), raw


def colors_vjp(sh, dirs, raw, g_col):
    """(g_sh, g_dirs) with saturated channels masked; sh.py:62-81."""
    deg = sh_degree_of(sh.shape[1])
    g = g_col * ((raw > 0.0) & (raw < 1.0))
    basis = sh_basis(dirs, deg)
    g_sh = basis[:, :, None] * g[:, None, :]
    g_basis = np.einsum("nkc,nc->nk", sh, g)
    g_dirs = np.einsum("nk,nkj->nj", g_basis, sh_basis_jac(dirs, deg))
    return g_sh, g_dirs


# ---------------------------------------------------------------------------
# NTC transform (transform.py)
# ---------------------------------------------------------------------------
def inside_mask(grid, means):
    """transform.py:64-68."""
    lo = np.asarray(grid["lo"], dtype=np.float64)
    hi = np.asarray(grid["hi"], dtype=np.float64)
    return np.flatnonzero(np.all((means >= lo) & (means <= hi), axis=1))


def transform_forward(cloud, inside, out7, rotate_sh=True):
    """Apply d_mu / d_q (and rotate SH bands >= 1); transform.py:53-96."""
    d_mu, d_q = out7[:, :3], out7[:, 3:]
    u = qnormalize(d_q) if len(inside) else d_q.copy()
    q_src = cloud["rotations"][inside]
    out = {k: v.copy() for k, v in cloud.items()}
    out["means"][inside] += d_mu
    out["rotations"][inside] = qmul(u, q_src)
    deg = sh_degree_of(cloud["sh"].shape[1])
    if rotate_sh and len(inside) and deg >= 1:
        rot = qrot(u)
        for l in range(1, deg + 1):
            m = sh_band_rotation(rot, l)
            out["sh"][inside, _band(l)] = m @ cloud["sh"][inside, _band(l)]
    ctx = dict(inside=inside, d_q=d_q, u=u, q_src=q_src,
               sh_in=cloud["sh"][inside].copy(), rotate_sh=rotate_sh)
    return out, ctx


def transform_backward(ctx, d_means, d_rot, d_sh):
    """dL/d(out7) of the inside rows; transform.py:99-134."""
    inside = ctx["inside"]
    g_mu = d_means[inside]
    g_u = np.einsum("nij,ni->nj", quat_right_matrix(ctx["q_src"]), d_rot[inside])
    deg = sh_degree_of(ctx["sh_in"].shape[1])
    if ctx["rotate_sh"] and len(inside) and deg >= 1:
        rot = qrot(ctx["u"])
        g_r = np.zeros_like(rot)
        for l in range(1, deg + 1):
            g_m = np.einsum("nic,njc->nij", d_sh[inside, _band(l)], ctx["sh_in"][:, _band(l)])
            g_r += sh_band_rotation_vjp(rot, l, g_m)
        g_u = g_u + qrot_vjp(ctx["u"], g_r)
    g_q = qnormalize_vjp(ctx["d_q"], g_u) if len(inside) else np.zeros((0, 4))
    return np.concatenate([g_mu, g_q], axis=1)


# ---------------------------------------------------------------------------
# camera + projection (cameras.py)
# ---------------------------------------------------------------------------
def look_at(eye, target, up, fx, fy, cx, cy, width, height, near=0.01):
    """cameras.py:83-129."""
    eye = np.asarray(eye, dtype=np.float64)
    zc = np.asarray(target, dtype=np.float64) - eye
    zc = zc / np.linalg.norm(zc)
    xc = np.cross(zc, np.asarray(up, dtype=np.float64))
    xc = xc / np.linalg.norm(xc)
    yc = np.cross(zc, xc)
    rot = np.stack([xc, yc, zc])
    w2c = np.eye(4)
    w2c[:3, :3] = rot
    w2c[:3, 3] = -rot @ eye
    return dict(w2c=w2c, fx=float(fx), fy=float(fy), cx=float(cx), cy=float(cy),
                width=int(width), height=int(height), near=float(near))


def _jacobian(cam, p):
    """cameras.py:148-160 -> (M, 2, 3)."""
    x, y, z = p[:, 0], p[:, 1], p[:, 2]
    z = np.where(np.abs(z) < 1e-12, 1e-12, z)
    j = np.zeros((len(p), 2, 3))
    j[:, 0, 0] = cam["fx"] / z
    j[:, 0, 2] = -cam["fx"] * x / (z * z)
    j[:, 1, 1] = cam["fy"] / z
    j[:, 1, 2] = -cam["fy"] * y / (z * z)
    return j


def covariance(q_raw, log_scales):
    """Sigma = R diag(e^{2s}) R^T with q normalised; gaussians.py:120-124, :231-235."""
    r = qrot(qnormalize(q_raw))
    var = np.exp(2.0 * log_scales)
    return np.einsum("nij,nj,nkj->nik", r, var, r)


def covariance_vjp(q_raw, log_scales, g_cov):
    """(g_q_raw, g_log_scales); gaussians.py:127-154."""
    u = qnormalize(q_raw)
    r = qrot(u)
    var = np.exp(2.0 * log_scales)
    g_sym = g_cov + np.swapaxes(g_cov, -1, -2)
    g_r = np.einsum("nij,njk,nk->nik", g_sym, r, var)
    diag = np.einsum("nji,njk,nki->ni", r, g_cov, r)
    g_s = diag * 2.0 * var
    return qnormalize_vjp(q_raw, qrot_vjp(u, g_r)), g_s


# ---------------------------------------------------------------------------
# rasterizer (rasterizer.py)
# ---------------------------------------------------------------------------
def project(cloud, cam):
    """Survivor order and per-survivor projected records; rasterizer.py:227-240."""
    rot = cam["w2c"][:3, :3]
    t = cam["w2c"][:3, 3]
    means = cloud["means"]
    pc_all = means @ rot.T + t
    z_all = pc_all[:, 2]
    keep = np.flatnonzero(z_all > cam["near"])
    keep = keep[np.lexsort((keep, z_all[keep]))]
    pc = pc_all[keep]
    z = np.where(np.abs(pc[:, 2]) < 1e-12, 1e-12, pc[:, 2])
    mean2d = np.stack([cam["fx"] * pc[:, 0] / z + cam["cx"],
                       cam["fy"] * pc[:, 1] / z + cam["cy"]], axis=1)
    cov3d = covariance(cloud["rotations"][keep], cloud["log_scales"][keep])
    mmat = _jacobian(cam, pc) @ rot
    cov2d = np.einsum("nij,njk,nlk->nil", mmat, cov3d, mmat)
    cov2d[:, 0, 0] += LOWPASS
    cov2d[:, 1, 1] += LOWPASS
    a, b, c, d = cov2d[:, 0, 0], cov2d[:, 0, 1], cov2d[:, 1, 0], cov2d[:, 1, 1]
    det = a * d - b * c
    conic = np.stack([np.stack([d, -b], -1), np.stack([-c, a], -1)], -2) / det[:, None, None]
    cam_pos = -rot.T @ t
    delta = means[keep] - cam_pos
    dist = np.linalg.norm(delta, axis=1)
    dirs = delta / np.maximum(dist, 1e-12)[:, None]
    colors, raw = colors_forward(cloud["sh"][keep], dirs)
    opacity = 1.0 / (1.0 + np.exp(-cloud["opacity_logits"][keep]))
    return dict(indices=keep, p_cam=pc, mean2d=mean2d, cov3d=cov3d, cov2d=cov2d,
                conic=conic, dirs=dirs, dist=dist, colors=colors, raw=raw,
                opacity=opacity)


def tile_rects(mean2d, cov2d, opacity, width, height, ts, skip):
    """Per-survivor inclusive tile rectangle and visibility; rasterizer.py:132-154."""
    n = len(mean2d)
    ntx = (width + ts - 1) // ts
    nty = (height + ts - 1) // ts
    if skip > 0.0:
        r = np.sqrt(np.maximum(9.0, 2.0 * np.log(np.maximum(opacity / skip, 1.0))))
        hx = r * np.sqrt(np.maximum(cov2d[:, 0, 0], 0.0))
        hy = r * np.sqrt(np.maximum(cov2d[:, 1, 1], 0.0))
        xl, xh = mean2d[:, 0] - hx, mean2d[:, 0] + hx
        yl, yh = mean2d[:, 1] - hy, mean2d[:, 1] + hy
        cl = lambda v, m: np.clip(np.floor(v).astype(np.int64) // ts, 0, m - 1)  # noqa: E731
        rect = np.stack([cl(xl, ntx), cl(xh, ntx), cl(yl, nty), cl(yh, nty)], 1)
        vis = ~((xh < 0) | (xl > width - 1) | (yh < 0) | (yl > height - 1))
    else:
        rect = np.tile(np.array([0, ntx - 1, 0, nty - 1], dtype=np.int64), (n, 1))
        vis = np.ones(n, dtype=bool)
    return rect, vis


def tile_lists(mean2d, cov2d, opacity, width, height, ts, skip):
    """[(y0, y1, x0, x1, members)] for non-empty tiles in (ty, tx) order, members
    in depth-rank order; rasterizer.py:107-175 (vectorised binning)."""
    rect, vis = tile_rects(mean2d, cov2d, opacity, width, height, ts, skip)
    ntx = (width + ts - 1) // ts
    idx = np.flatnonzero(vis)
    if len(idx) == 0:
        return []
    x0, x1, y0, y1 = rect[idx].T
    wx = x1 - x0 + 1
    cnt = wx * (y1 - y0 + 1)
    ranks = np.repeat(idx, cnt)  # emitted in rank order, tiles row-major per splat
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
                    ranks[s:e].astype(np.intp)))
    return out


def _tile_pairs(proj, tile, s):
    """Dense (pixel x member) alpha / transmittance of one tile; rasterizer.py:178-211."""
    y0, y1, x0, x1, mem = tile
    ys, xs = np.mgrid[y0:y1, x0:x1]
    dx = xs.ravel()[:, None].astype(np.float64) - proj["mean2d"][mem, 0][None, :]
    dy = ys.ravel()[:, None].astype(np.float64) - proj["mean2d"][mem, 1][None, :]
    con = proj["conic"][mem]
    maha = (con[:, 0, 0] * dx * dx + (con[:, 0, 1] + con[:, 1, 0]) * dx * dy
            + con[:, 1, 1] * dy * dy)
    g = np.exp(-0.5 * maha)
    og = proj["opacity"][mem][None, :] * g
    alpha = np.minimum(s["alpha_clamp"], og)
    alpha = np.where(alpha < s["skip_alpha"], 0.0, alpha)
    t_all = np.concatenate([np.ones((len(dx), 1)), np.cumprod(1.0 - alpha, axis=1)], 1)
    t_before = t_all[:, :-1]
    alive = t_before >= s["stop_transmittance"]
    t_final = t_all[np.arange(len(dx)), alive.sum(axis=1)]
    return dx, dy, g, og, alpha, t_before, alive, t_final


DEFAULT_SETTINGS = dict(tile_size=16, alpha_clamp=0.99, skip_alpha=1.0 / 255.0,
                        stop_transmittance=1e-4)


def render(cloud, cam, background=None, settings=None):
    """Forward render; rasterizer.py:214-281.  Returns (out, ctx)."""
    s = dict(DEFAULT_SETTINGS, **(settings or {}))
    bg = np.zeros(3) if background is None else np.asarray(background, dtype=np.float64)
    h, w = cam["height"], cam["width"]
    proj = project(cloud, cam)
    tiles = tile_lists(proj["mean2d"], proj["cov2d"], proj["opacity"], w, h,
                       s["tile_size"], s["skip_alpha"])
    image = np.empty((h, w, 3))
    image[:] = bg
    alpha_map = np.zeros((h, w))
    touch = np.zeros(len(cloud["means"]), dtype=np.int64)
    for tile in tiles:
        y0, y1, x0, x1, mem = tile
        _, _, _, _, alpha, tb, alive, tf = _tile_pairs(proj, tile, s)
        wgt = alpha * tb * alive
        img = wgt @ proj["colors"][mem] + tf[:, None] * bg
        image[y0:y1, x0:x1] = img.reshape(y1 - y0, x1 - x0, 3)
        alpha_map[y0:y1, x0:x1] = (1.0 - tf).reshape(y1 - y0, x1 - x0)
        np.add.at(touch, proj["indices"][mem], (wgt > 0).sum(axis=0))
    ctx = dict(cloud=cloud, cam=cam, settings=s, bg=bg, proj=proj, tiles=tiles)
    return dict(image=image, alpha_map=alpha_map, touch=touch), ctx


def render_backward(ctx, d_image):
    """Gradients for every raw cloud parameter; rasterizer.py:284-402."""
    cloud, cam, s, bg, pj = ctx["cloud"], ctx["cam"], ctx["settings"], ctx["bg"], ctx["proj"]
    n = len(cloud["means"])
    k = cloud["sh"].shape[1]
    out = dict(d_means=np.zeros((n, 3)), d_rotations=np.zeros((n, 4)),
               d_log_scales=np.zeros((n, 3)), d_opacity_logits=np.zeros(n),
               d_sh=np.zeros((n, k, 3)), viewspace=np.zeros(n),
               contributed=np.zeros(n, dtype=bool))
    m = len(pj["indices"])
    if m == 0:
        return out
    acc_col = np.zeros((m, 3))
    acc_op = np.zeros(m)
    acc_m2 = np.zeros((m, 2))
    acc_con = np.zeros((m, 2, 2))
    live_any = np.zeros(m, dtype=bool)
    gb_dot = d_image @ bg
    for tile in ctx["tiles"]:
        y0, y1, x0, x1, mem = tile
        dx, dy, g, og, alpha, tb, alive, tf = _tile_pairs(pj, tile, s)
        gp = d_image[y0:y1, x0:x1].reshape(-1, 3)
        gb = gb_dot[y0:y1, x0:x1].ravel()
        wgt = alpha * tb * alive
        np.add.at(acc_col, mem, wgt.T @ gp)
        u = gp @ pj["colors"][mem].T
        live = wgt > 0
        term = u * alpha * tb * live
        rev = np.cumsum(term[:, ::-1], axis=1)[:, ::-1]
        suffix = np.concatenate([rev[:, 1:], np.zeros((len(gp), 1))], 1) + (gb * tf)[:, None]
        da = (u * tb - suffix / np.maximum(1.0 - alpha, 1e-12)) * alive
        da = np.where((alpha > 0) & (og < s["alpha_clamp"]), da, 0.0)
        np.add.at(acc_op, mem, (da * g).sum(0))
        dm = -0.5 * g * da * pj["opacity"][mem][None, :]
        con = pj["conic"][mem]
        cdx = con[:, 0, 0] * dx + con[:, 0, 1] * dy
        cdy = con[:, 1, 0] * dx + con[:, 1, 1] * dy
        np.add.at(acc_m2, mem, -np.stack([(2 * cdx * dm).sum(0), (2 * cdy * dm).sum(0)], 1))
        dc = np.empty((len(mem), 2, 2))
        dc[:, 0, 0] = (dm * dx * dx).sum(0)
        dc[:, 0, 1] = dc[:, 1, 0] = (dm * dx * dy).sum(0)
        dc[:, 1, 1] = (dm * dy * dy).sum(0)
        np.add.at(acc_con, mem, dc)
        np.logical_or.at(live_any, mem, live.any(0))
    return _gaussian_backward(ctx, acc_col, acc_op, acc_m2, acc_con, live_any, out)


def _gaussian_backward(ctx, acc_col, acc_op, acc_m2, acc_con, live_any, out):
    """Per-survivor chain to raw parameters; rasterizer.py:351-402."""
    cloud, cam, pj = ctx["cloud"], ctx["cam"], ctx["proj"]
    idx = pj["indices"]
    rot = cam["w2c"][:3, :3]
    out["viewspace"][idx] = np.linalg.norm(acc_m2, axis=1)
    out["contributed"][idx] = live_any
    g_sh, g_dirs = colors_vjp(cloud["sh"][idx], pj["dirs"], pj["raw"], acc_col)
    out["d_sh"][idx] = g_sh
    dirs = pj["dirs"]
    g_world = (g_dirs - dirs * np.sum(dirs * g_dirs, 1, keepdims=True)) / np.maximum(
        pj["dist"], 1e-12)[:, None]
    con = pj["conic"]
    g_cov2d = -np.einsum("nij,njk,nkl->nil", con, acc_con, con)
    jac = _jacobian(cam, pj["p_cam"])
    mm = jac @ rot
    g_cov3d = np.einsum("nji,njk,nkl->nil", mm, g_cov2d, mm)
    g_mm = np.einsum("nij,njk,nkl->nil", g_cov2d + np.swapaxes(g_cov2d, 1, 2), mm, pj["cov3d"])
    g_j = g_mm @ rot.T
    x, y, z = pj["p_cam"][:, 0], pj["p_cam"][:, 1], pj["p_cam"][:, 2]
    fx, fy = cam["fx"], cam["fy"]
    g_pc = np.zeros_like(pj["p_cam"])
    g_pc[:, 0] = g_j[:, 0, 2] * (-fx / z ** 2)
    g_pc[:, 1] = g_j[:, 1, 2] * (-fy / z ** 2)
    g_pc[:, 2] = (g_j[:, 0, 0] * (-fx / z ** 2) + g_j[:, 1, 1] * (-fy / z ** 2)
                  + g_j[:, 0, 2] * (2 * fx * x / z ** 3) + g_j[:, 1, 2] * (2 * fy * y / z ** 3))
    g_pc += np.einsum("nji,nj->ni", jac, acc_m2)
    g_world = g_world + g_pc @ rot
    g_q, g_s = covariance_vjp(cloud["rotations"][idx], cloud["log_scales"][idx], g_cov3d)
    out["d_means"][idx] = g_world
    out["d_rotations"][idx] = g_q
    out["d_log_scales"][idx] = g_s
    op = pj["opacity"]
    out["d_opacity_logits"][idx] = acc_op * op * (1.0 - op)
    return out


# ---------------------------------------------------------------------------
# loss (losses.py)
# ---------------------------------------------------------------------------
def _gauss1d(window, sigma):
    ax = np.arange(window, dtype=np.float64) - window // 2
    g = np.exp(-(ax ** 2) / (2.0 * sigma ** 2))
    return g / g.sum()


def _valid_sep(img, g):
    """Valid 2-D correlation with the separable kernel g g^T (losses.py:43-44)."""
    win = len(g)
    h, w = img.shape
    rows = sum(g[i] * img[:, i:w - win + 1 + i] for i in range(win))
    return sum(g[i] * rows[i:h - win + 1 + i, :] for i in range(win))


def _full_sep(img, g):
    """Full 2-D convolution with g g^T (adjoint of _valid_sep, losses.py:139-141)."""
    win = len(g)
    pad = np.pad(img, win - 1)
    return _valid_sep(pad, g[::-1])


def render_loss(rendered, target, lam=0.2, window=11, sigma=1.5, c1=0.01 ** 2, c2=0.03 ** 2):
    """(1-lam) L1 + lam (1 - mean SSIM)/2 over valid windows and its image
    gradient; losses.py:84-148."""
    x_all = np.asarray(rendered, dtype=np.float64)
    y_all = np.asarray(target, dtype=np.float64)
    if x_all.shape != y_all.shape:
        raise OracleDataError("render_loss shape mismatch")
    squeeze = x_all.ndim == 2
    if squeeze:
        x_all, y_all = x_all[..., None], y_all[..., None]
    h, w, ch = x_all.shape
    if h < window or w < window:
        raise OracleDataError("image smaller than the SSIM window")
    diff = x_all - y_all
    l1 = float(np.mean(np.abs(diff)))
    grad = (1.0 - lam) * np.sign(diff) / diff.size
    g = _gauss1d(window, sigma)
    nwin = (h - window + 1) * (w - window + 1) * ch
    up = -lam / (2.0 * nwin)
    ssum = 0.0
    for c in range(ch):
        x, y = x_all[..., c], y_all[..., c]
        mx, my = _valid_sep(x, g), _valid_sep(y, g)
        sxx = _valid_sep(x * x, g) - mx * mx
        syy = _valid_sep(y * y, g) - my * my
        sxy = _valid_sep(x * y, g) - mx * my
        a1, a2 = 2 * mx * my + c1, 2 * sxy + c2
        b1, b2 = mx * mx + my * my + c1, sxx + syy + c2
        smap = (a1 * a2) / (b1 * b2)
        ssum += float(smap.sum())
        if lam == 0.0:
            continue
        inv = 1.0 / (b1 * b2)
        g_a1, g_a2 = a2 * inv, a1 * inv
        g_b1, g_b2 = -smap / b1, -smap / b2
        g_mx = 2 * my * g_a1 + 2 * mx * g_b1 - 2 * my * g_a2 - 2 * mx * g_b2
        back = (_full_sep(g_mx, g) + _full_sep(g_b2, g) * (2.0 * x)
                + _full_sep(2.0 * g_a2, g) * y)
        grad[..., c] += up * back
    loss = (1.0 - lam) * l1 + lam * (1.0 - ssum / nwin) / 2.0
    return float(loss), (grad[..., 0] if squeeze else grad)


# ---------------------------------------------------------------------------
# one Stage-1 iteration (pipeline.py:262-277) and the loop around it
# ---------------------------------------------------------------------------
def stage1_iteration(state, cloud, cam, target, background=None, settings=None,
                     rotate_sh=True, lam=0.2, lr=0.002, apply_adam=True):
    """One Stage-1 step on `state` (dict: grid, tables, mlp, m/v moments, step,
    inside, enc=(idx, w, touched)) in place; pipeline.py:263-277.

    Returns a dict with loss, image, render grads and the NTC grads."""
    grid = state["grid"]
    inside = state["inside"]
    if state.get("enc") is None:
        state["enc"] = encode(grid, cloud["means"][inside])
    idx, w, touched = state["enc"]
    mlp = state["mlp"]
    feats = gather(state["tables"], idx, w)
    out7, hidden = mlp_forward(mlp, feats)
    moved, tctx = transform_forward(cloud, inside, out7, rotate_sh)
    rout, rctx = render(moved, cam, background, settings)
    loss, d_img = render_loss(rout["image"], target, lam)
    if not np.isfinite(loss):
        raise OracleNumericalError("non-finite values detected in 'stage1 loss'")
    rg = render_backward(rctx, d_img)
    g7 = transform_backward(tctx, rg["d_means"], rg["d_rotations"], rg["d_sh"])
    gw, gb, g_feats = mlp_backward(mlp, feats, hidden, g7)
    g_tab = table_scatter(state["tables"].shape, idx, w, g_feats)
    if apply_adam:
        adam_apply(state, g_tab, gw, gb, lr)
    return dict(loss=loss, image=rout["image"], d_image=d_img, render_grads=rg,
                g7=g7, g_tables=g_tab, g_w=gw, g_b=gb, out7=out7, moved=moved)


def adam_apply(state, g_tab, gw, gb, lr):
    """cache.adam_step: lazy rows for tables, dense for the MLP; ntc.py:290-293."""
    if "m" not in state:
        state["m"] = dict(t=np.zeros_like(state["tables"]),
                          w=[np.zeros_like(a) for a in state["mlp"]["weights"]],
                          b=[np.zeros_like(a) for a in state["mlp"]["biases"]])
        state["v"] = dict(t=np.zeros_like(state["tables"]),
                          w=[np.zeros_like(a) for a in state["mlp"]["weights"]],
                          b=[np.zeros_like(a) for a in state["mlp"]["biases"]])
        state["step"] = 0
    state["step"] += 1
    t = state["step"]
    touched = state["enc"][2]
    for l in range(state["tables"].shape[0]):
        adam_update(state["tables"][l], g_tab[l], state["m"]["t"][l], state["v"]["t"][l],
                    t, lr, rows=touched[l])
    for i in range(len(gw)):
        adam_update(state["mlp"]["weights"][i], gw[i], state["m"]["w"][i], state["v"]["w"][i],
                    t, lr)
        adam_update(state["mlp"]["biases"][i], gb[i], state["m"]["b"][i], state["v"]["b"][i],
                    t, lr)


def fit_grid(grid, means, margin=1.5):
    """fit_grid_to_cloud, pipeline.py:348-360."""
    lo = means.min(axis=0)
    hi = means.max(axis=0)
    c = 0.5 * (lo + hi)
    half = np.maximum(0.5 * (hi - lo) * margin, 0.25)
    return dict(grid, lo=tuple(c - half), hi=tuple(c + half))


def stage1_view_order(seed, frame_index, n_views, iterations):
    """View sequence of the Stage-1 loop: default_rng([seed, frame]) permutations
    re-drawn every n_views iterations; pipeline.py:251-256, :263, :278-279."""
    rng = np.random.default_rng([seed, frame_index])
    order = rng.permutation(n_views)
    seq = []
    for t in range(iterations):
        seq.append(int(order[t % n_views]))
        if (t + 1) % n_views == 0:
            order = rng.permutation(n_views)
    return seq


# ---------------------------------------------------------------- NTC warm-up (F2)
def warmup_loss(d_mu, d_q):
    """Identity-pull loss, mean over the batch; losses.py:151-180.
    Per row |d_mu|_1 - cos^2(angle(norm(d_q), identity)); returns (loss, g_mu, g_q)."""
    d_mu = np.asarray(d_mu, dtype=np.float64)
    d_q = np.asarray(d_q, dtype=np.float64)
    b = d_mu.shape[0]
    n2 = np.sum(d_q * d_q, axis=1)
    if np.any(n2 < 1e-24):
        raise OracleNumericalError("zero-norm d_q in warmup_loss")
    w = d_q[:, 0]
    loss = float(np.mean(np.sum(np.abs(d_mu), axis=1) - w * w / n2))
    g_mu = np.sign(d_mu) / b
    g_q = (-2.0 * (w * w)[:, None] * d_q) / (n2 ** 2)[:, None]
    g_q[:, 0] = 2.0 * w * (n2 - w * w) / n2 ** 2
    return loss, g_mu, -g_q / b


def warmup_train(grid, tables, mlp, initial_means, noise_sigma, iterations, lr=0.002,
                 batch_size=65536, seed=0):
    """ntc.py:296-333: Adam on batches of the initial means plus Gaussian jitter
    (clamped to the AABB), touched rows = the batch's corners; returns the
    float32-quantised (tables, mlp) and the loss history."""
    means = np.asarray(initial_means, dtype=np.float64).reshape(-1, 3)
    rng = np.random.default_rng(seed)
    lo, hi = np.asarray(grid["lo"]), np.asarray(grid["hi"])
    state = dict(grid=grid, tables=np.array(tables, dtype=np.float64),
                 mlp=dict(weights=[np.array(w, dtype=np.float64) for w in mlp["weights"]],
                          biases=[np.array(b, dtype=np.float64) for b in mlp["biases"]]))
    hist = []
    for _ in range(iterations):
        take = min(batch_size, len(means))
        sel = rng.choice(len(means), size=take, replace=False)
        batch = np.clip(means[sel] + rng.normal(scale=noise_sigma, size=(take, 3)), lo, hi)
        idx, w, touched = encode(grid, batch)
        feats = gather(state["tables"], idx, w)
        out7, hidden = mlp_forward(state["mlp"], feats)
        loss, g_mu, g_q = warmup_loss(out7[:, :3], out7[:, 3:])
        hist.append(loss)
        gw, gb, gf = mlp_backward(state["mlp"], feats, hidden, np.concatenate([g_mu, g_q], 1))
        state["enc"] = (idx, w, touched)
        adam_apply(state, table_scatter(state["tables"].shape, idx, w, gf), gw, gb, lr)
    q = lambda a: a.astype(np.float32).astype(np.float64)  # noqa: E731
    return (q(state["tables"]), dict(weights=[q(a) for a in state["mlp"]["weights"]],
                                     biases=[q(a) for a in state["mlp"]["biases"]]), hist)
