"""Seeded generator pins: SplitMix64 known answers, determinism,
random access, sampler invariants and moments."""
import math

import numpy as np
import torch

import nbgen


def test_splitmix64_kat():
    # Published SplitMix64 outputs for state 0 (Steele, Lea, Flood 2014 reference code).
    assert nbgen.splitmix64_sequence(0, 3) == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4,
                                               0x06C45D188009454F]
    d = nbgen.u64d(nbgen.draws(0, 0, 3)).tolist()
    assert d == [0.8833108082136426, 0.43152799704850997, 0.026433771592597743]


def test_mix64_matches_python_ints():
    xs = [0, 1, 2**63, 2**64 - 1, 0x1234567890ABCDEF]
    t = torch.tensor([nbgen._s64(x) for x in xs], dtype=torch.int64)
    got = [nbgen._u64(int(v)) for v in nbgen.mix64(t).tolist()]
    assert got == [nbgen.mix64_int(x) for x in xs]


def test_random_access_and_determinism():
    cfg = nbgen.CONFIGS["c5"]
    a = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, 1000)
    b = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 400, 100)
    assert torch.equal(a[400:500], b)
    assert torch.equal(a, nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, 1000))


def test_u32f_exact_and_range():
    u = nbgen.u32f(nbgen.draws(7, 0, 100000))
    assert u.dtype == torch.float32
    assert float(u.min()) >= 0.0 and float(u.max()) < 1.0
    # 24-bit grid: u * 2^24 is an integer
    assert torch.equal(u * 2**24, (u * 2**24).floor())
    m = float(u.double().mean())
    assert abs(m - 0.5) < 3 * math.sqrt(1 / 12 / 1e5)


def test_ray_sampler_invariants():
    cfg = nbgen.CONFIGS["c3"]
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, 20000).double()
    o, d = q[:, :3], q[:, 3:]
    on_face = ((o == 0) | (o == 1)).sum(1)
    assert bool((on_face >= 1).all())
    assert bool(((o >= 0) & (o <= 1)).all())
    assert torch.allclose(d.norm(dim=1), torch.ones(len(d), dtype=torch.float64), atol=1e-6)
    assert float(d.mean(0).abs().max()) < 0.03  # isotropic directions


def test_box_sampler_invariants():
    cfg = nbgen.CONFIGS["c5"]
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, 20000)
    lo, hi = q[:, :3], q[:, 3:]
    assert bool((lo <= hi).all()) and bool((hi <= 1).all()) and bool((lo >= 0).all())
    e = (hi - lo).double()
    assert float(e.max()) <= 0.1 + 1e-6


def test_param_counts():
    # 3 -> 50 -> 50 -> 1 has 2,801 parameters (§5 "Storage")
    cfg = nbgen.Config("paper3d", 3, "point", 50, 2)
    assert nbgen.num_params(cfg) == 2801
    assert [nbgen.num_params(c) for c in nbgen.CONFIGS.values()] == [1185, 12801, 50561, 83587, 199425]


def test_xavier_bounds():
    cfg = nbgen.CONFIGS["c2"]
    p = nbgen.init_params(cfg)
    w1 = p[: 3 * 64]
    a = math.sqrt(6 / (3 + 64))
    assert float(w1.abs().max()) <= a
    assert float(p[3 * 64: 3 * 64 + 64].abs().max()) == 0.0  # b1 = 0


def test_grids_nontrivial():
    for name in ["c1", "c2", "c5"]:
        g = nbgen.make_grid(nbgen.CONFIGS[name])
        frac = float(g.float().mean())
        assert 0.01 < frac < 0.5, (name, frac)


# ---------------------------------------------------------------- O2 grid pins (R11, R12)
def _lattice_centroid(o):
    R = o.shape[-1]
    c = (torch.arange(R, dtype=torch.float64) + 0.5) / R
    n = o.sum()
    return [float((o.sum(dim=tuple(d for d in range(3) if d != a)) * c).sum() / n) for a in range(3)]


def test_sphere_rasterisation_closed_forms():
    """R11 (voxel occupied iff its centre is in the closed shape), closed
    forms on a 4^3 grid with the sphere at the cube centre: the 8 central
    centres lie at sqrt(3)/8 = 0.2165 from it, the next 24 at
    sqrt(0.375^2 + 2 * 0.125^2) = 0.4146."""
    for r, want in [(0.21, 0), (0.22, 8), (0.41, 8), (0.42, 32)]:
        occ = torch.zeros(4, 4, 4, dtype=torch.bool)
        nbgen._sphere_into(occ, 4, [0.5, 0.5, 0.5], r)
        assert int(occ.sum()) == want, (r, int(occ.sum()))
    # axis-aligned ellipsoid, semi-axes (0.42, 0.22, 0.22): the central 8 have
    # (0.125/0.42)^2 + 2 (0.125/0.22)^2 = 0.73 <= 1; the x-outer neighbours
    # (0.375/0.42)^2 + 2 (0.125/0.22)^2 = 1.44 and the y/z-outer ones 2.1 are out
    occ = torch.zeros(4, 4, 4, dtype=torch.bool)
    nbgen._ellipsoid_into(occ, 4, [0.5, 0.5, 0.5], [0.42, 0.22, 0.22])
    assert int(occ.sum()) == 8


def test_centred_sphere_has_cube_symmetry():
    """A sphere centred in the cube rasterises to a set invariant under every
    axis flip and permutation (a half-voxel centre offset would break the flips)."""
    occ = torch.zeros(64, 64, 64, dtype=torch.bool)
    nbgen._sphere_into(occ, 64, [0.5, 0.5, 0.5], 0.3)
    for d in range(3):
        assert torch.equal(occ, occ.flip(d))
    assert torch.equal(occ, occ.permute(1, 0, 2)) and torch.equal(occ, occ.permute(0, 2, 1))


def test_ellipsoid_and_sphere_volume_within_shell_bound():
    """The voxels whose centres lie in a closed ellipsoid cover its volume up to
    the voxels meeting the surface: every such voxel lies within
    delta = sqrt(3) / (2R) of the surface, where the ellipsoidal radius is
    1 +- delta / a_min, so |N / R^3 - V| <= V ((1 + delta/a_min)^3 - (1 - delta/a_min)^3)."""
    R = 128
    for cen, ax in [([0.4, 0.55, 0.5], [0.13, 0.07, 0.1]), ([0.3, 0.3, 0.7], [0.05, 0.05, 0.05]),
                    ([0.62, 0.41, 0.33], [0.02, 0.15, 0.09])]:
        occ = torch.zeros(R, R, R, dtype=torch.bool)
        nbgen._ellipsoid_into(occ, R, cen, ax)
        V = 4.0 / 3.0 * math.pi * ax[0] * ax[1] * ax[2]
        e = math.sqrt(3) / (2 * R) / min(ax)
        bound = V * ((1 + e) ** 3 - (1 - e) ** 3)
        assert abs(float(occ.sum()) / R ** 3 - V) <= bound, (cen, ax)
        # the lattice centroid sits at the centre (symmetric shape)
        assert max(abs(a - b) for a, b in zip(_lattice_centroid(occ), cen)) < 1.0 / R
    occ = torch.zeros(R, R, R, dtype=torch.bool)
    nbgen._sphere_into(occ, R, [0.45, 0.5, 0.58], 0.08)
    V = 4.0 / 3.0 * math.pi * 0.08 ** 3
    e = math.sqrt(3) / (2 * R) / 0.08
    assert abs(float(occ.sum()) / R ** 3 - V) <= V * ((1 + e) ** 3 - (1 - e) ** 3)


def test_c4_frame_times_and_clamp():
    """R12: frame k shows each sphere at time t_k = (k + 1/2) / 32 with its
    centre clamped per axis to [r, 1 - r].  Single-sphere grids (the c4 recipe
    with count = 1; seed 1 has a sphere whose z path leaves the cube) are
    compared frame by frame with the path drawn from the GRID stream in the
    documented order (c0, r, v): the voxel centroid follows the clamped
    centre to 1.5e-3, which the readings t_k = k / 31 or an unclamped centre
    miss by more."""
    import dataclasses
    for seed in (0, 1):
        cfg = dataclasses.replace(nbgen.CONFIGS["c4"], seed=seed,
                                  grid=dict(nbgen.CONFIGS["c4"].grid, count=1))
        occ = nbgen.make_grid(cfg)
        F = occ.shape[0]
        u = nbgen.u64d(nbgen.draws(nbgen.stream_key(seed, nbgen.TAG_GRID), 0, 7)).tolist()
        r = 0.04 + 0.06 * u[3]
        c0 = [0.15 + 0.7 * u[j] for j in range(3)]
        v = [-0.3 + 0.6 * u[4 + j] for j in range(3)]
        worst_alt, worst_unclamped = 0.0, 0.0
        for f in range(F):
            cen = _lattice_centroid(occ[f])
            t = (f + 0.5) / F
            want = [min(max(c0[j] + v[j] * t, r), 1 - r) for j in range(3)]
            assert max(abs(a - b) for a, b in zip(cen, want)) < 1.5e-3, (seed, f)
            alt = [min(max(c0[j] + v[j] * f / (F - 1), r), 1 - r) for j in range(3)]
            worst_alt = max(worst_alt, max(abs(a - b) for a, b in zip(cen, alt)))
            worst_unclamped = max(worst_unclamped, max(abs(a - (c0[j] + v[j] * t)) for j, a in enumerate(cen)))
        assert worst_alt > 2.5e-3
        if seed == 1:
            assert worst_unclamped > 0.05
