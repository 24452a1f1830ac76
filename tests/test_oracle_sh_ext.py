"""Property checks of the SH degree 2-3 extension (no reference exists: parity
unpinned).  The band rotation must be a representation of SO(3) consistent
with the reference's degree-1 convention, and every analytic gradient must
match central differences."""

import numpy as np
import pytest

from oracle import stage1 as O


def _rot(rng):
    q = rng.normal(size=4)
    return O.qrot(q / np.linalg.norm(q))


@pytest.mark.parametrize("l", [1, 2, 3])
def test_band_rotation_is_orthogonal_group_homomorphism(l, rng):
    r1, r2 = _rot(rng), _rot(rng)
    m1, m2, m12 = (O.sh_band_rotation(r, l) for r in (r1, r2, r1 @ r2))
    np.testing.assert_allclose(m1 @ m1.T, np.eye(2 * l + 1), atol=1e-12)
    np.testing.assert_allclose(m12, m1 @ m2, atol=1e-12)


def test_band1_matches_reference_permutation_form(rng):
    r = _rot(rng)
    np.testing.assert_allclose(O.sh_band_rotation(r, 1), O._PERM @ r @ O._PERM.T, atol=1e-15)


@pytest.mark.parametrize("deg", [1, 2, 3])
def test_colour_equivariance(deg, rng):
    """Rotating the coefficients by M(R) and the view direction by R leaves the colour unchanged."""
    k = (deg + 1) ** 2
    sh = rng.normal(scale=0.2, size=(1, k, 3))
    d = rng.normal(size=3)
    d /= np.linalg.norm(d)
    r = _rot(rng)
    rot_sh = sh.copy()
    for l in range(1, deg + 1):
        rot_sh[0, O._band(l)] = O.sh_band_rotation(r, l) @ sh[0, O._band(l)]
    c0, _ = O.colors_forward(sh, d[None])
    c1, _ = O.colors_forward(rot_sh, (r @ d)[None])
    np.testing.assert_allclose(c0, c1, atol=1e-12)


def test_basis_jacobian_fd(rng):
    d = rng.normal(size=(5, 3))
    jac = O.sh_basis_jac(d, 3)
    eps = 1e-6
    for j in range(3):
        dp, dm = d.copy(), d.copy()
        dp[:, j] += eps
        dm[:, j] -= eps
        fd = (O.sh_basis(dp, 3) - O.sh_basis(dm, 3)) / (2 * eps)
        np.testing.assert_allclose(jac[..., j], fd, atol=1e-7)


@pytest.mark.parametrize("deg", [2, 3])
def test_transform_backward_fd_sh3(deg, rng):
    """d(sum w . transformed cloud)/d(out7) vs central differences, bands 1..deg rotated."""
    n = 3
    k = (deg + 1) ** 2
    cloud = dict(means=rng.normal(size=(n, 3)), rotations=rng.normal(size=(n, 4)),
                 log_scales=rng.normal(size=(n, 3)), opacity_logits=rng.normal(size=n),
                 sh=rng.normal(scale=0.3, size=(n, k, 3)))
    inside = np.arange(n)
    out7 = rng.normal(size=(n, 7))
    out7[:, 3] += 2.0
    wm, wr, ws = rng.normal(size=(n, 3)), rng.normal(size=(n, 4)), rng.normal(size=(n, k, 3))

    def f(o7):
        moved, _ = O.transform_forward(cloud, inside, o7)
        return (wm * moved["means"]).sum() + (wr * moved["rotations"]).sum() + (ws * moved["sh"]).sum()

    _, ctx = O.transform_forward(cloud, inside, out7)
    g = O.transform_backward(ctx, wm, wr, ws)
    eps = 1e-6
    fd = np.zeros_like(out7)
    for i in range(n):
        for j in range(7):
            p, m = out7.copy(), out7.copy()
            p[i, j] += eps
            m[i, j] -= eps
            fd[i, j] = (f(p) - f(m)) / (2 * eps)
    np.testing.assert_allclose(g, fd, rtol=1e-5, atol=1e-7)


def test_render_backward_fd_sh3(rng):
    """Full raster backward with SH3 colours against central differences
    (threshold-free settings, as the reference's SMOOTH FD test)."""
    from paper_2403_01444_b200 import scenes

    sc = scenes.small_scene(seed=9, n=6, width=24, height=20, sh_degree=3, n_views=1)
    cloud = {k: v.astype(np.float64) for k, v in sc.cloud.items()}
    cloud["log_scales"] = np.full((6, 3), np.log(0.25))
    cloud["sh"][:, 1:] *= 4.0
    cam = sc.cameras[0]
    s = dict(tile_size=64, skip_alpha=0.0, stop_transmittance=0.0)
    w = rng.normal(size=(20, 24, 3))
    bg = np.array([0.2, 0.3, 0.1])

    def loss(c):
        return float((w * O.render(c, cam, bg, s)[0]["image"]).sum())

    _, ctx = O.render(cloud, cam, bg, s)
    g = O.render_backward(ctx, w)
    eps = 1e-5
    for key, gk in (("sh", "d_sh"), ("means", "d_means"), ("rotations", "d_rotations")):
        arr = cloud[key]
        flat = arr.reshape(-1)
        idx = np.random.default_rng(1).choice(flat.size, size=min(12, flat.size), replace=False)
        for i in idx:
            o = flat[i]
            flat[i] = o + eps
            lp = loss(cloud)
            flat[i] = o - eps
            lm = loss(cloud)
            flat[i] = o
            num = (lp - lm) / (2 * eps)
            ana = g[gk].reshape(-1)[i]
            assert abs(ana - num) <= 2e-3 * max(abs(num), abs(ana)) + 1e-6, (key, i, ana, num)
