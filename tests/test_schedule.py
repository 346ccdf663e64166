"""The paper's training control: FN-gated weight
schedule, early stop, L1/L2 (Suppl. §2.1-2.2; readings
DESIGN.md R37-R39).  The oracle is pinned to the paper's printed decrements,
to the early-stop rule and to a finite-difference derivative of the
regulariser; the product's host-only nb_schedule_* then matches it step by
step on random FN sequences."""
import numpy as np
import pytest

import oracle
import paper_2310_06822_b200 as nb


def run(sched, fns):
    for fn in fns:
        sched.after_step(fn)
    return sched


@pytest.mark.parametrize("dim,first", [(2, 20.0), (3, 100.0), (4, 200.0)])
def test_oracle_decrements_are_the_papers(dim, first):
    """2D decreases by 1/20, 1/40, 1/60 ...; 3D 1/100, 1/200, 1/300;
    4D 1/200, 1/400, 1/600; the other weight rises by 0.2 each time."""
    s = oracle.PaperSchedule(dim, step_every=4)
    printed = {2: [1 / 20, 1 / 40, 1 / 60], 3: [1 / 100, 1 / 200, 1 / 300],
               4: [1 / 200, 1 / 400, 1 / 600]}[dim]
    beta, alpha = 1.0, 1.0
    for k in range(3):
        run(s, [0, 5, 0, 0])              # one window with FN > 0
        beta -= printed[k]
        alpha += 0.2
        assert s.triggers == k + 1
        assert s.beta == pytest.approx(beta, abs=1e-15)
        assert s.alpha == pytest.approx(alpha, abs=1e-15)
    run(s, [0, 0, 0, 0])                  # FN-free window: weights unchanged
    assert s.beta == pytest.approx(beta, abs=1e-15) and s.triggers == 3


def test_oracle_weights_change_only_at_window_ends():
    """'every 10,000 iterations': nothing moves inside a window."""
    s = oracle.PaperSchedule(2, step_every=10)
    run(s, [7] * 9)
    assert (s.alpha, s.beta, s.triggers) == (1.0, 1.0, 0)
    s.after_step(0)
    assert s.triggers == 1 and s.beta == pytest.approx(0.95)


def test_oracle_early_stop_after_six_stable_windows():
    """stop once FN = 0 has been stable for the past six scheduling
    iterations; an FN window in between restarts the count."""
    s = oracle.PaperSchedule(3, step_every=2)
    run(s, [1, 0] + [0, 0] * 5)
    assert not s.stop and s.stable == 5
    run(s, [0, 3])
    assert not s.stop and s.stable == 0
    run(s, [0, 0] * 5)
    assert not s.stop
    run(s, [0, 0])
    assert s.stop and s.stable == 6


def test_oracle_long_run_closed_form_and_cap():
    """After k FN windows the decrements sum to base * H_k (harmonic number,
    H_k = digamma(k + 1) + Euler-gamma) and the other weight is 1 + 0.2 k."""
    from scipy.special import digamma
    s = oracle.PaperSchedule(2, step_every=1, max_steps=10 ** 9)
    run(s, [1] * 5000)
    hk = digamma(5001.0) + np.euler_gamma
    assert s.beta == pytest.approx(1 - hk / 20, abs=1e-12)
    assert s.alpha == pytest.approx(1 + 0.2 * 5000, abs=1e-9)
    s = oracle.PaperSchedule(2, step_every=1, max_steps=3)
    run(s, [1, 1, 1])
    assert s.stop


def test_oracle_lambda_linear_to_5e7():
    """Suppl. §2.2: lambda ranges from 0 to 5e-7, linear schedule."""
    s = oracle.PaperSchedule(4, step_every=100, max_steps=1000)
    assert s.lam == 0.0
    run(s, [1] * 250)
    assert s.lam == pytest.approx(5e-7 * 0.25)
    run(s, [1] * 750)
    assert s.lam == pytest.approx(5e-7)


def test_oracle_reg_grad_is_the_regulariser_derivative():
    """Central finite difference of R(theta) = l1 sum|theta| + l2 sum theta^2,
    away from the kink at 0."""
    rng = np.random.default_rng(5)
    th = rng.uniform(0.05, 1.0, 64) * rng.choice([-1.0, 1.0], 64)
    l1, l2 = 0.3, 1.7

    def R(t):
        return l1 * np.abs(t).sum() + l2 * (t * t).sum()

    h = 1e-6
    fd = np.array([(R(th + h * e) - R(th - h * e)) / (2 * h) for e in np.eye(64)])
    assert np.allclose(oracle.reg_grad(th, l1, l2), fd, atol=1e-7)
    assert oracle.reg_grad(np.zeros(3), l1, l2).tolist() == [0.0, 0.0, 0.0]


@pytest.mark.parametrize("dim", [2, 3, 4])
def test_product_schedule_matches_oracle(dim):
    """libnb.so's host-only nb_schedule_* against the oracle, step by step,
    on FN sequences with long FN-free stretches (so early stop is reached)."""
    rng = np.random.default_rng(dim)
    for trial in range(4):
        every = int(rng.integers(1, 6))
        cap = int(rng.integers(200, 2000))
        p = nb.PaperSchedule(dim, step_every=every, max_steps=cap)
        o = oracle.PaperSchedule(dim, step_every=every, max_steps=cap)
        p_fn = np.where(rng.random(cap) < np.linspace(0.6, 0.0, cap),
                        rng.integers(1, 1 << 40, cap), 0)
        for fn in p_fn:
            p.after_step(int(fn))
            o.after_step(int(fn))
            assert p.triggers == o.triggers
            assert p.alpha == pytest.approx(o.alpha, rel=1e-12)
            assert p.beta == pytest.approx(o.beta, rel=1e-12, abs=1e-15)
            assert p.lam == pytest.approx(o.lam, rel=1e-12, abs=1e-25)
            assert p.stop == o.stop
            if o.stop:
                break


def test_product_schedule_rejects_bad_arguments():
    with pytest.raises(nb.NBError):
        nb.PaperSchedule(5)
    with pytest.raises(nb.NBError):
        nb.PaperSchedule(3, step_every=0)
