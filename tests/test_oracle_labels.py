"""Pins for the oracle's indicator and exact labellers (oracle/nb_oracle.c;
PAPER.md P:134-142 §3.1, readings R15-R19).  Each labeller is pinned
against an independent brute force, a sampling lower bound (Alg. 1's
SampleRegion/Any), and closed-form special cases."""
import numpy as np
import pytest
import torch

import nbgen
import oracle


def rand_grid(R, p, seed):
    rng = np.random.default_rng(seed)
    return (rng.random((R, R, R)) < p).astype(np.uint8)


def test_indicator_floor_example():
    # SPEC-style example: on R=4, x=0.3 falls in cell floor(0.3*4) = 1.
    g = np.zeros((4, 4), np.uint8)
    g[1, 0] = 1
    assert oracle.indicator(g, 2, [0.3, 0.1]) == 1
    assert oracle.indicator(g, 2, [0.2, 0.1]) == 0
    # x = 1 belongs to the last cell; outside the unit cube f = 0 (R15)
    g[3, 3] = 1
    assert oracle.indicator(g, 2, [1.0, 1.0]) == 1
    assert oracle.indicator(g, 2, [1.0 + 1e-12, 1.0]) == 0
    assert oracle.indicator(g, 2, [-1e-12, 0.1]) == 0


def test_point_labels_disc_geometry():
    # A single disc of radius r rasterised at voxel centres: points deeper than
    # one voxel diagonal inside are labelled 1, farther than that outside are 0.
    R, cx, cy, r = 128, 0.5, 0.45, 0.2
    c = (np.arange(R) + 0.5) / R
    X, Y = np.meshgrid(c, c, indexing="ij")
    g = ((X - cx) ** 2 + (Y - cy) ** 2 <= r * r).astype(np.uint8)
    q = np.random.default_rng(0).random((20000, 2)).astype(np.float32)
    y = oracle.label(g, 2, "point", q)
    dist = np.hypot(q[:, 0] - cx, q[:, 1] - cy)
    diag = np.sqrt(2) / R
    assert (y[dist < r - diag] == 1).all()
    assert (y[dist > r + diag] == 0).all()


def test_point_labels_4d_frame_select():
    g = np.zeros((32, 8, 8, 8), np.uint8)
    g[5, 2, 3, 4] = 1
    x = np.array([[2.5 / 8, 3.5 / 8, 4.5 / 8, 5.5 / 32], [2.5 / 8, 3.5 / 8, 4.5 / 8, 6.5 / 32]],
                 np.float32)
    assert oracle.label(g, 4, "point", x, frames=32).tolist() == [1, 0]


@pytest.mark.parametrize("R,p,seed", [(4, 0.05, 1), (8, 0.02, 2), (8, 0.2, 3), (6, 0.01, 4)])
def test_ray_dda_equals_brute_force(R, p, seed):
    g = rand_grid(R, p, seed)
    rng = np.random.default_rng(seed)
    n = 20000
    o = rng.random((n, 3)) * 1.4 - 0.2
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    # also axis-aligned and grid-aligned rays (ties on voxel faces/edges)
    o[:2000] = np.round(o[:2000] * R) / R
    d[:1000] = np.eye(3)[rng.integers(0, 3, 1000)] * rng.choice([-1, 1], (1000, 1))
    q = np.concatenate([o, d], 1).astype(np.float32)
    a = oracle.label(g, 3, "ray", q)
    b = oracle.label(g, 3, "ray", q, brute=True)
    assert (a == b).all(), np.nonzero(a != b)[0][:10]


def test_ray_c3_vs_brute_and_sampling_lower_bound():
    cfg = nbgen.CONFIGS["c3"]
    g = nbgen.make_grid(cfg).numpy()
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, 3000).numpy()
    a = oracle.label(g, 3, "ray", q)
    b = oracle.label(g, 3, "ray", q, brute=True)
    assert (a == b).all()
    # Alg. 1 SampleRegion + Any: sampled hits are a lower bound of the exact label
    o, d = q[:, :3].astype(np.float64), q[:, 3:].astype(np.float64)
    s = np.linspace(1e-4, np.sqrt(3), 4096)
    hit = np.zeros(len(q), bool)
    R = g.shape[0]
    for chunk in np.array_split(s, 16):
        pts = o[:, None, :] + chunk[None, :, None] * d[:, None, :]
        inside = ((pts >= 0) & (pts <= 1)).all(-1)
        idx = np.minimum(np.floor(np.clip(pts, 0, 1) * R).astype(int), R - 1)
        occ = g[idx[..., 0], idx[..., 1], idx[..., 2]] == 1
        hit |= (inside & occ).any(1)
    assert (a[hit] == 1).all()
    assert 0.02 < a.mean() < 0.5


def test_ray_full_and_empty_grid():
    R = 8
    rng = np.random.default_rng(5)
    o = rng.random((2000, 3))
    d = rng.normal(size=(2000, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    q = np.concatenate([o, d], 1).astype(np.float32)
    assert oracle.label(np.zeros((R, R, R), np.uint8), 3, "ray", q).sum() == 0
    # origins strictly inside the cube: every ray has positive length inside
    assert oracle.label(np.ones((R, R, R), np.uint8), 3, "ray", q).all()
    # a ray on a face pointing outwards has zero length inside: negative (R16)
    out = np.array([[0.0, 0.5, 0.5, -1.0, 0.0, 0.0]], np.float32)
    assert oracle.label(np.ones((R, R, R), np.uint8), 3, "ray", out)[0] == 0


@pytest.mark.parametrize("R,p,seed", [(8, 0.01, 1), (16, 0.002, 2), (16, 0.05, 3)])
def test_box_sat_equals_scan(R, p, seed):
    g = rand_grid(R, p, seed)
    rng = np.random.default_rng(seed)
    lo = rng.random((20000, 3))
    hi = np.minimum(1.0, lo + rng.random((20000, 3)) * 0.4)
    lo[:3000] = np.round(lo[:3000] * R) / R          # faces exactly on voxel boundaries
    hi[:3000] = np.maximum(lo[:3000], np.round(hi[:3000] * R) / R)
    q = np.concatenate([lo, hi], 1).astype(np.float32)
    assert (oracle.label(g, 3, "box", q) == oracle.label(g, 3, "box", q, brute=True)).all()


def test_sat_definition():
    g = rand_grid(6, 0.3, 9)
    S = oracle.sat(g)
    rng = np.random.default_rng(0)
    for _ in range(50):
        i, j, k = rng.integers(0, 7, 3)
        assert S[i, j, k] == g[:i, :j, :k].sum()


def test_box_invariants_c5():
    cfg = nbgen.CONFIGS["c5"]
    g = nbgen.make_grid(cfg).numpy()
    R = g.shape[0]
    # a box containing an occupied voxel is positive (BASELINE.json north_star)
    occ = np.argwhere(g == 1)[:: 997][:300]
    pad = np.random.default_rng(1).random((len(occ), 6)) * 0.01
    lo = np.maximum(0, occ / R - pad[:, :3])
    hi = np.minimum(1, (occ + 1) / R + pad[:, 3:])
    q = np.concatenate([lo, hi], 1).astype(np.float32)
    assert oracle.label(g, 3, "box", q).all()
    # monotone under inclusion and lower-bounded by corner sampling
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, 20000).numpy()
    y = oracle.label(g, 3, "box", q)
    big = q.copy()
    big[:, :3] = np.maximum(0, q[:, :3] - 0.01)
    big[:, 3:] = np.minimum(1, q[:, 3:] + 0.01)
    yb = oracle.label(g, 3, "box", big.astype(np.float32))
    assert (yb >= y).all()
    rng = np.random.default_rng(2)
    t = rng.random((20000, 64, 3))
    pts = q[:, None, :3] + t * (q[:, None, 3:] - q[:, None, :3])
    idx = np.minimum(np.floor(pts * R).astype(int), R - 1)
    hit = (g[idx[..., 0], idx[..., 1], idx[..., 2]] == 1).any(1)
    assert (y[hit] == 1).all()
    assert 0.1 < y.mean() < 0.7


def test_plane_scan_equals_subdivision():
    R = 8
    g = rand_grid(R, 0.03, 11)
    rng = np.random.default_rng(3)
    p0 = rng.random((3000, 3))
    nrm = rng.normal(size=(3000, 3))
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    nrm[:300] = np.eye(3)[rng.integers(0, 3, 300)]
    p0[:300] = np.round(p0[:300] * R) / R
    q = np.concatenate([p0, nrm], 1).astype(np.float32)
    a = oracle.label(g, 3, "plane", q)
    b = oracle.label(g, 3, "plane", q, brute=True)
    assert (a == b).all()
    assert 0 < a.mean() < 1


# ---------------------------------------------------------------- 2D rays, boxes, lines (NEXT-3)
def _cfg2(kind):
    import dataclasses
    return dataclasses.replace(nbgen.CONFIGS["c1"], kind=kind)


def rand_grid2(R, p, seed):
    rng = np.random.default_rng(seed)
    return (rng.random((R, R)) < p).astype(np.uint8)


@pytest.mark.parametrize("R,p,seed", [(4, 0.2, 0), (8, 0.1, 1), (8, 0.4, 2), (16, 0.05, 3)])
def test_ray2_dda_equals_brute_force(R, p, seed):
    """2D DDA (R16 with pixels) == slab test of every occupied pixel, on
    random rays plus rays along pixel edges and through pixel corners."""
    g = rand_grid2(R, p, seed)
    q = nbgen.make_queries(_cfg2("ray"), nbgen.TAG_EVAL, seed * 1000, 3000).numpy()
    edge = []
    for k in range(R + 1):
        edge.append([k / R, 0.0, 0.0, 1.0])
        edge.append([0.0, k / R, 1.0, 0.0])
        edge.append([0.0, k / R, 0.70710678, 0.70710678])
        edge.append([1.0, k / R, -1.0, 0.0])
    q = np.concatenate([q, np.array(edge, np.float32)])
    assert np.array_equal(oracle.label(g, 2, "ray", q), oracle.label(g, 2, "ray", q, brute=True))


def test_ray2_full_and_empty_grid():
    q = nbgen.make_queries(_cfg2("ray"), nbgen.TAG_EVAL, 0, 2000).numpy()
    assert oracle.label(np.zeros((8, 8), np.uint8), 2, "ray", q).sum() == 0
    # a ray entering through the left edge crosses a pixel with positive length
    rng = np.random.default_rng(3)
    th = rng.uniform(-1.3, 1.3, 500)
    inward = np.stack([np.zeros(500), rng.random(500), np.cos(th), np.sin(th)], 1).astype(np.float32)
    assert oracle.label(np.ones((8, 8), np.uint8), 2, "ray", inward).all()
    # and one leaving it (pointing away from the square) crosses none
    assert oracle.label(np.ones((8, 8), np.uint8), 2, "ray", inward * np.array([1, 1, -1, 1], np.float32)).sum() == 0


@pytest.mark.parametrize("R,p,seed", [(8, 0.05, 0), (16, 0.02, 1), (32, 0.01, 2)])
def test_box2_sat_equals_scan_and_contains_pixel(R, p, seed):
    g = rand_grid2(R, p, seed)
    q = nbgen.make_queries(_cfg2("box"), nbgen.TAG_EVAL, seed, 5000).numpy()
    y = oracle.label(g, 2, "box", q)
    assert np.array_equal(y, oracle.label(g, 2, "box", q, brute=True))
    # a box containing the centre of an occupied pixel is positive (R17)
    occ = np.argwhere(g)
    c = (occ + 0.5) / R
    boxes = np.concatenate([c - 1e-3, c + 1e-3], 1).astype(np.float32)
    assert oracle.label(g, 2, "box", boxes).all()


@pytest.mark.parametrize("R,p,seed", [(8, 0.1, 0), (16, 0.03, 1)])
def test_line2_scan_equals_subdivision(R, p, seed):
    """2D lines (R19 with pixels): the corner test on occupied pixels equals
    the same test on their 2x2 children (a convex square is cut iff a child is)."""
    g = rand_grid2(R, p, seed)
    q = nbgen.make_queries(_cfg2("plane"), nbgen.TAG_EVAL, seed, 3000).numpy()
    edge = np.array([[k / R, 0.5, 1.0, 0.0] for k in range(R + 1)] +
                    [[0.5, k / R, 0.0, 1.0] for k in range(R + 1)], np.float32)
    q = np.concatenate([q, edge])
    y = oracle.label(g, 2, "plane", q)
    assert np.array_equal(y, oracle.label(g, 2, "plane", q, brute=True))
    assert 0 < y.mean() < 1
