"""Pins for the oracle's 4D (space x time) ray, hyperplane and box labellers
(Suppl. Tab. 4/5 "4D Ray, Plane, Box" P:844, P:865;
records per P:777; reading R48).  Each is pinned against an
independent brute force on small grids, against the already-pinned 3D
labellers in the special cases that reduce to one frame (d_t = 0, a box
inside one frame, a hyperplane with n_t = 0), a sampling lower bound
(Alg. 1's SampleRegion/Any) and containment / monotonicity."""
import numpy as np
import pytest

import nbgen
import oracle


def rand_grid4(R, F, p, seed):
    rng = np.random.default_rng(seed)
    return (rng.random((F, R, R, R)) < p).astype(np.uint8)


def rand_dirs4(rng, n):
    d = rng.normal(size=(n, 4))
    return d / np.linalg.norm(d, axis=1, keepdims=True)


@pytest.mark.parametrize("R,F,p,seed", [(4, 3, 0.05, 1), (5, 4, 0.02, 2), (4, 2, 0.2, 3)])
def test_ray4_dda_equals_brute_force(R, F, p, seed):
    g = rand_grid4(R, F, p, seed)
    rng = np.random.default_rng(seed)
    n = 6000
    o = rng.random((n, 4)) * 1.4 - 0.2
    d = rand_dirs4(rng, n)
    # axis-aligned and zero-component directions, origins on cell faces
    d[:500] = np.eye(4)[rng.integers(0, 4, 500)] * rng.choice([-1, 1], (500, 1))
    d[500:1000, rng.integers(0, 4)] = 0.0
    d[500:1000] /= np.linalg.norm(d[500:1000], axis=1, keepdims=True)
    res = np.array([R, R, R, F])
    o[1000:1500] = np.round(rng.random((500, 4)) * res) / res
    q = np.concatenate([o, d], 1).astype(np.float32)
    y = oracle.label(g, 4, "ray", q, frames=F)
    yb = oracle.label(g, 4, "ray", q, brute=True, frames=F)
    assert np.array_equal(y, yb), int((y != yb).sum())
    assert 0 < y.mean() < 1


def test_ray4_constant_time_equals_3d_dda_on_the_frame():
    """A ray with d_t = 0 stays in one frame: its 4D label is the 3D DDA label
    of (o_xyz, d_xyz) on that frame's grid (R16 in 3D, pinned separately)."""
    cfg = nbgen.EXTRA_CONFIGS["c4ray"]
    g = nbgen.make_grid(cfg).numpy()
    F = g.shape[0]
    rng = np.random.default_rng(5)
    n = 4000
    d3 = rand_dirs4(rng, n)[:, :3]
    d3 /= np.linalg.norm(d3, axis=1, keepdims=True)
    o3 = rng.random((n, 3))
    t = rng.random(n)
    q4 = np.concatenate([o3, t[:, None], d3, np.zeros((n, 1))], 1).astype(np.float32)
    y4 = oracle.label(g, 4, "ray", q4, frames=F)
    q3 = np.concatenate([o3, d3], 1).astype(np.float32)
    fr = np.minimum(F - 1, np.floor(q4[:, 3].astype(np.float64) * F).astype(int))
    y3 = np.array([oracle.label(g[fr[i]], 3, "ray", q3[i:i + 1])[0] for i in range(n)])
    assert np.array_equal(y4, y3)
    assert y4.mean() > 0.02


def test_ray4_sampling_lower_bound():
    """Alg. 1's SampleRegion/Any: points sampled strictly inside the clipped
    segment that fall in an occupied cell imply a positive exact label."""
    cfg = nbgen.EXTRA_CONFIGS["c4ray"]
    g = nbgen.make_grid(cfg).numpy()
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, 3000).numpy()
    y = oracle.label(g, 4, "ray", q, frames=32)
    o, d = q[:, :4].astype(np.float64), q[:, 4:].astype(np.float64)
    s = np.linspace(0.0, 2.0, 1025)[1:-1]
    hits = np.zeros(len(q), bool)
    for k in range(0, len(s), 64):
        pts = o[:, None, :] + s[None, k:k + 64, None] * d[:, None, :]
        inside = np.all((pts > 1e-9) & (pts < 1 - 1e-9), axis=2)
        lab = oracle.label(g, 4, "point", pts.reshape(-1, 4).astype(np.float32), frames=32).reshape(inside.shape)
        hits |= np.any(inside & (lab == 1), axis=1)
    assert np.all(y[hits] == 1)
    assert hits.sum() > 0.8 * y.sum()  # dense sampling finds most positives


@pytest.mark.parametrize("R,F,p,seed", [(4, 3, 0.05, 1), (6, 5, 0.02, 2), (5, 4, 0.3, 3)])
def test_box4_sat_equals_scan(R, F, p, seed):
    g = rand_grid4(R, F, p, seed)
    rng = np.random.default_rng(seed)
    n = 8000
    lo = rng.random((n, 4)) * 1.2 - 0.1
    hi = lo + rng.random((n, 4)) * 0.6 - 0.05
    q = np.concatenate([lo, hi], 1).astype(np.float32)
    y = oracle.label(g, 4, "box", q, frames=F)
    yb = oracle.label(g, 4, "box", q, brute=True, frames=F)
    assert np.array_equal(y, yb)
    assert 0 < y.mean() < 1


def test_box4_containment_monotonicity_and_one_frame():
    cfg = nbgen.EXTRA_CONFIGS["c4box"]
    g = nbgen.make_grid(cfg).numpy()
    F, R = g.shape[0], g.shape[1]
    rng = np.random.default_rng(7)
    # a box containing an occupied cell (with margin) is positive (BJ north star)
    occ = np.argwhere(g)
    pick = occ[rng.choice(len(occ), 2000)]
    res = np.array([R, R, R, F], np.float64)
    cells = np.stack([pick[:, 1], pick[:, 2], pick[:, 3], pick[:, 0]], 1).astype(np.float64)
    lo = (cells - rng.random((2000, 4)) * 0.5) / res
    hi = (cells + 1 + rng.random((2000, 4)) * 0.5) / res
    q = np.clip(np.concatenate([lo, hi], 1), 0, 1).astype(np.float32)
    assert oracle.label(g, 4, "box", q, frames=F).all()
    # monotone under inclusion
    qs = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, 4000).numpy().astype(np.float64)
    big = qs.copy()
    big[:, :4] -= 0.02
    big[:, 4:] += 0.02
    y, yb = (oracle.label(g, 4, "box", x.astype(np.float32), frames=F) for x in (qs, np.clip(big, 0, 1)))
    assert np.all(yb >= y)
    # a box whose time extent lies inside one frame is the 3D box label of that frame
    f = rng.integers(0, F, 3000)
    t0 = (f + 0.2) / F
    t1 = (f + 0.7) / F
    q3 = qs[:3000].copy()
    q4 = np.concatenate([q3[:, :3], t0[:, None], q3[:, 4:7], t1[:, None]], 1).astype(np.float32)
    y4 = oracle.label(g, 4, "box", q4, frames=F)
    b3 = np.concatenate([q3[:, :3], q3[:, 4:7]], 1).astype(np.float32)
    y3 = np.array([oracle.label(g[f[i]], 3, "box", b3[i:i + 1])[0] for i in range(3000)])
    assert np.array_equal(y4, y3)


@pytest.mark.parametrize("R,F,p,seed", [(3, 2, 0.1, 1), (4, 3, 0.03, 2)])
def test_plane4_scan_equals_subdivision(R, F, p, seed):
    g = rand_grid4(R, F, p, seed)
    rng = np.random.default_rng(seed)
    n = 1500
    p0 = rng.random((n, 4))
    nrm = rand_dirs4(rng, n)
    nrm[:200] = np.eye(4)[rng.integers(0, 4, 200)]               # axis-aligned hyperplanes ...
    res = np.array([R, R, R, F])
    p0[:200] = np.round(p0[:200] * res) / res                     # ... through cell faces
    q = np.concatenate([p0, nrm], 1).astype(np.float32)
    y = oracle.label(g, 4, "plane", q, frames=F)
    yb = oracle.label(g, 4, "plane", q, brute=True, frames=F)
    assert np.array_equal(y, yb)
    assert 0 < y.mean() < 1


def test_plane4_special_cases():
    R, F = 4, 3
    full = np.ones((F, R, R, R), np.uint8)
    empty = np.zeros_like(full)
    rng = np.random.default_rng(3)
    q = np.concatenate([rng.random((500, 4)), rand_dirs4(rng, 500)], 1).astype(np.float32)
    assert oracle.label(full, 4, "plane", q, frames=F).all()      # through the cube: cuts an occupied cell
    assert not oracle.label(empty, 4, "plane", q, frames=F).any()
    # n_t = 0: the hyperplane cuts cell (c, f) iff the 3D plane cuts c, for every frame
    g = rand_grid4(R, F, 0.08, 9)
    n3 = rand_dirs4(rng, 500)[:, :3]
    n3 /= np.linalg.norm(n3, axis=1, keepdims=True)
    p3 = rng.random((500, 3))
    q4 = np.concatenate([p3, rng.random((500, 1)), n3, np.zeros((500, 1))], 1).astype(np.float32)
    y4 = oracle.label(g, 4, "plane", q4, frames=F)
    q3 = np.concatenate([p3, n3], 1).astype(np.float32)
    y3 = np.zeros(500, np.uint8)
    for f in range(F):
        y3 |= oracle.label(g[f], 3, "plane", q3)
    assert np.array_equal(y4, y3)


def test_4d_samplers():
    for k in ("ray", "box", "plane"):
        cfg = nbgen.EXTRA_CONFIGS["c4" + k]
        q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, 20000).double().numpy()
        assert q.shape == (20000, 8)
        assert np.array_equal(q, nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, 20000).double().numpy())
        if k in ("ray", "plane"):
            assert np.allclose(np.linalg.norm(q[:, 4:], axis=1), 1.0, atol=1e-6)
            assert np.abs(q[:, 4:].mean(0)).max() < 0.02      # isotropic on S^3
        if k == "ray":
            assert np.all(((q[:, :4] == 0) | (q[:, :4] == 1)).sum(1) >= 1)   # on the hypercube boundary
        if k == "box":
            assert np.all(q[:, :4] <= q[:, 4:]) and np.all(q[:, 4:] <= 1.0)
