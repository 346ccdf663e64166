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
