"""Pins for the oracle's MLP forward, asymmetric loss, backward, Adam,
calibration and scoring (oracle/nb_oracle.c).  Pins are known answers
(SPEC-derived KATs, P:631's parameter count), closed forms, central finite
differences, independent library routines (torch fp64 nn.functional /
autograd / optim.Adam), and invariants."""
import math

import numpy as np
import pytest
import torch

import nbgen
import oracle



@pytest.fixture(autouse=True)
def _float64_default():
    """fp64 torch references inside this module only: a module-level
    set_default_dtype leaked into every later test of the session (a GPU
    test's torch.full output buffers became float64)."""
    prev = torch.get_default_dtype()
    torch.set_default_dtype(torch.float64)
    yield
    torch.set_default_dtype(prev)


def torch_forward(arch, theta, q, emulate_bf16=False):
    """Independent fp64 torch chain (library routine), optionally with bf16
    rounding where the kernel rounds (weights, hi/lo inputs, activations)."""
    th = torch.as_tensor(theta, dtype=torch.float64)
    x = torch.as_tensor(q, dtype=torch.float32)
    if emulate_bf16:
        hi = x.to(torch.bfloat16).float()
        lo = (x - hi).to(torch.bfloat16).float()
        h = hi.double() + lo.double()
    else:
        h = x.double()
    p = 0
    d_in = arch.d0
    heads = {arch.head_after[k]: k for k in range(arch.n_heads)}
    out_heads = [None] * arch.n_heads
    for l in range(arch.layers):
        W = th[p:p + d_in * arch.width].view(arch.width, d_in); p += d_in * arch.width
        b = th[p:p + arch.width]; p += arch.width
        if emulate_bf16:
            W = W.float().to(torch.bfloat16).double()
            z = (torch.nn.functional.linear(h, W).float() + b.float())
            r = torch.relu(z)
            hn = r.to(torch.bfloat16).double() if l < arch.layers - 1 else r.double()
            r = r.double()
        else:
            r = torch.relu(torch.nn.functional.linear(h, W, b))
            hn = r
        if (l + 1) in heads:
            out_heads[heads[l + 1]] = r
        h = hn
        d_in = arch.width
    wo = th[p:p + arch.width]; p += arch.width
    bo = th[p]; p += 1
    outs = [h @ wo + bo]
    for k in range(arch.n_heads):
        u = th[p:p + arch.width]; p += arch.width
        c = th[p]; p += 1
        outs.append(out_heads[k] @ u + c)
    z = torch.stack(outs, 1)
    if emulate_bf16:
        z = z.float().double()
    return z


def rand_theta(arch, seed, scale=1.0):
    rng = np.random.default_rng(seed)
    return rng.normal(size=oracle.num_params(arch)) * scale / math.sqrt(arch.width)


def test_param_count_paper():
    assert oracle.num_params(oracle.make_arch(3, 50, 2)) == 2801
    for c, n in zip(nbgen.CONFIGS.values(), [1185, 12801, 50561, 83587, 199425]):
        assert oracle.num_params(oracle.arch_of(c)) == n


def test_forward_zero_weights_kat():
    a = oracle.make_arch(3, 8, 2)
    th = np.zeros(oracle.num_params(a))
    th[-1] = 3.0  # b_out
    z = oracle.forward(a, th, np.random.rand(5, 3).astype(np.float32))
    sig = 1 / (1 + np.exp(-z[:, 0]))
    assert np.allclose(sig, 0.9525741268224334, atol=1e-12)  # sigma(3)
    th[-1] = 0.0
    z = oracle.forward(a, th, np.random.rand(5, 3).astype(np.float32))
    assert np.all(z == 0.0)  # sigma = 0.5


@pytest.mark.parametrize("head_after", [(), (2, 4)])
def test_forward_equals_torch_fp64(head_after):
    a = oracle.make_arch(4, 32, 6 if head_after else 3, head_after)
    th = rand_theta(a, 1)
    q = np.random.default_rng(2).random((500, 4)).astype(np.float32)
    z = oracle.forward(a, th, q)
    ref = torch_forward(a, th, q).numpy()
    assert np.allclose(z, ref, rtol=1e-12, atol=1e-12)


def test_forward_bf16_emulation_equals_torch_bf16_chain():
    a = oracle.make_arch(6, 64, 4)
    th = rand_theta(a, 3).astype(np.float32).astype(np.float64)
    q = np.random.default_rng(4).random((400, 6)).astype(np.float32)
    z = oracle.forward(a, th, q, oracle.BF16_EMU)
    ref = torch_forward(a, th, q, emulate_bf16=True).numpy()
    # both round the same quantities; only fp64 summation order differs,
    # which can flip a rare bf16 rounding of an activation.
    close = np.abs(z - ref) <= 1e-5 * np.maximum(1, np.abs(ref))
    assert close.mean() > 0.97
    assert np.median(np.abs(z - ref)) == 0.0
    # emulation differs from the fp64 definition by bf16-level error only
    zf = oracle.forward(a, th, q)
    assert np.max(np.abs(z - zf)) < 0.05 * np.max(np.abs(zf)) + 1e-3


def test_encode_bf16_matches_torch_rne():
    q = (np.random.default_rng(5).random((1000, 6)) * 2 - 0.5).astype(np.float32)
    q[0, :] = [0.0, 1.0, 1 / 3, 0.999999, 2.0 ** -20, 0.5 + 2 ** -9]
    e = oracle.encode_bf16(q)
    x = torch.from_numpy(q)
    hi = x.to(torch.bfloat16)
    lo = (x - hi.float()).to(torch.bfloat16)
    assert np.array_equal(e[:, :6], hi.view(torch.int16).numpy().view(np.uint16))
    assert np.array_equal(e[:, 6:12], lo.view(torch.int16).numpy().view(np.uint16))
    assert np.all(e[:, 12:] == 0)
    rec = hi.double() + lo.double()
    assert torch.all((rec - x.double()).abs() <= 2.0 ** -16 * x.double().abs() + 1e-30)


def test_weighted_bce_kats():
    # SPEC loss KATs: ln 2, 2 ln 2, ln 2
    assert oracle.weighted_bce(0.0, 1, 1.0, 1.0) == pytest.approx(0.693147, abs=1e-6)
    assert oracle.weighted_bce(0.0, 1, 2.0, 1.0) == pytest.approx(1.386294, abs=1e-6)
    assert oracle.weighted_bce(0.0, 0, 1.0, 1.0) == pytest.approx(0.693147, abs=1e-6)
    # Eq. (1) with log(sigmoid) written directly, away from saturation
    for z in [-5.0, -0.3, 0.7, 4.0]:
        s = 1 / (1 + math.exp(-z))
        assert oracle.weighted_bce(z, 1, 7.0, 1.0) == pytest.approx(-7 * math.log(s), rel=1e-12)
        assert oracle.weighted_bce(z, 0, 1.0, 0.5) == pytest.approx(-0.5 * math.log(1 - s), rel=1e-12)


@pytest.mark.parametrize("head_after", [(), (2, 4)])
def test_loss_and_grad_equal_torch_autograd(head_after):
    a = oracle.make_arch(3, 16, 5 if head_after else 3, head_after)
    th = rand_theta(a, 7)
    rng = np.random.default_rng(8)
    q = rng.random((300, 3)).astype(np.float32)
    y = (rng.random(300) < 0.3).astype(np.uint8)
    alpha, beta, B = 37.0, 1.0, 1000
    loss, g, st = oracle.loss_grad(a, th, q, y, alpha, beta, n_global=B)
    t = torch.tensor(th, requires_grad=True)
    z = torch_forward(a, t, q)
    w = torch.where(torch.from_numpy(y).bool(), alpha, beta).double()
    yt = torch.from_numpy(y).double()
    L = 0
    for k in range(z.shape[1]):  # L_Late + sum of head losses
        L = L + torch.nn.functional.binary_cross_entropy_with_logits(
            z[:, k], yt, weight=w, reduction="sum") / B
    L.backward()
    assert loss == pytest.approx(L.item(), rel=1e-12)
    assert np.allclose(g, t.grad.numpy(), rtol=1e-9, atol=1e-14)
    zz = z[:, 0].detach().numpy()
    assert st["tp"] == int(((zz >= 0) & (y == 1)).sum()) and st["fn"] == int(((zz < 0) & (y == 1)).sum())


def test_grad_central_finite_differences():
    # FD protocol: central differences, h = 1e-4, fp64, relative error <= 1e-4
    a = oracle.make_arch(2, 8, 2)
    th = rand_theta(a, 11)
    rng = np.random.default_rng(12)
    q = rng.random((64, 2)).astype(np.float32)
    y = (rng.random(64) < 0.5).astype(np.uint8)
    _, g, _ = oracle.loss_grad(a, th, q, y, 5.0, 1.0)
    h = 1e-4
    fd = np.zeros_like(g)
    for i in range(len(th)):
        tp, tm = th.copy(), th.copy()
        tp[i] += h
        tm[i] -= h
        fd[i] = (oracle.loss_grad(a, tp, q, y, 5.0, 1.0)[0] - oracle.loss_grad(a, tm, q, y, 5.0, 1.0)[0]) / (2 * h)
    err = np.abs(fd - g) / np.maximum(np.abs(g), 1e-3 * np.abs(g).max())
    # skip parameters whose FD window crosses a ReLU kink
    assert np.median(err) < 1e-6
    assert (err < 1e-4).mean() > 0.95


def test_symmetric_loss_is_plain_bce():
    # alpha = beta = 1 reduces Eq. (1) to the ordinary (OccNet) BCE
    a = oracle.make_arch(3, 8, 2)
    th = rand_theta(a, 5)
    q = np.random.default_rng(1).random((100, 3)).astype(np.float32)
    y = (np.random.default_rng(2).random(100) < 0.5).astype(np.uint8)
    loss, _, _ = oracle.loss_grad(a, th, q, y, 1.0, 1.0)
    z = oracle.forward(a, th, q)[:, 0]
    ref = torch.nn.functional.binary_cross_entropy_with_logits(torch.tensor(z), torch.tensor(y, dtype=torch.float64))
    assert loss == pytest.approx(ref.item(), rel=1e-12)


def test_adam_equals_torch_optim():
    rng = np.random.default_rng(3)
    th = rng.normal(size=50)
    m, v = np.zeros(50), np.zeros(50)
    p = torch.tensor(th.copy(), requires_grad=True)
    opt = torch.optim.Adam([p], lr=1e-3, betas=(0.9, 0.999), eps=1e-8)
    for t in range(1, 11):
        g = rng.normal(size=50)
        oracle.adam(th, m, v, t, g)
        p.grad = torch.tensor(g)
        opt.step()
        if t == 1:  # closed form: first step is -lr * sign(g) up to eps
            assert np.allclose(th - p.detach().numpy(), 0, atol=1e-15)
        assert np.allclose(th, p.detach().numpy(), rtol=0, atol=1e-14)


def test_adam_first_step_closed_form():
    th = np.array([1.0, 2.0, -3.0])
    m, v = np.zeros(3), np.zeros(3)
    g = np.array([0.5, -2.0, 1e-3])
    oracle.adam(th, m, v, 1, g)
    assert np.allclose(th, np.array([1.0, 2.0, -3.0]) - 1e-3 * np.sign(g), atol=1e-10)


def test_alpha_schedule():
    assert oracle.alpha(0, 200) == 1.0
    assert oracle.alpha(199, 200) == 1000.0
    assert oracle.alpha(100, 201) == pytest.approx(500.5)


def test_calibrate_minimality_and_fn_zero():
    rng = np.random.default_rng(4)
    z = rng.normal(size=(5000, 3))
    y = (rng.random(5000) < 0.2).astype(np.uint8)
    tau, rc = oracle.calibrate(z, y)
    assert rc == 0
    for k in range(3):
        pos = z[y == 1, k]
        assert tau[k] in pos                       # tau is a positive's logit
        assert np.all(pos >= tau[k])               # FN = 0 for this head
        nxt = np.sort(np.unique(pos))[1]           # the next larger positive logit
        assert (pos < nxt).sum() >= 1              # would give FN >= 1
    c = oracle.score(z, y, tau)
    assert c["fn"] == 0
    assert c["tp"] + c["fn"] == int(y.sum()) and c["fp"] + c["tn"] == int((y == 0).sum())
    assert sum(c["exit_hist"]) == 5000
    # exits only skip work: the early-exit predictor is the dense conjunction
    pred = (z[:, 1] >= tau[1]) & (z[:, 2] >= tau[2]) & (z[:, 0] >= tau[0])
    assert c["tp"] + c["fp"] == int(pred.sum())
    assert c["exit_hist"][0] == int((z[:, 1] < tau[1]).sum())
    # exits happen only on negatives of the calibration set
    exited = (z[:, 1] < tau[1]) | ((z[:, 1] >= tau[1]) & (z[:, 2] < tau[2]))
    assert np.all(y[exited] == 0)


def test_calibrate_no_positives():
    tau, rc = oracle.calibrate(np.zeros((10, 1)), np.zeros(10, np.uint8))
    assert rc == 1 and np.isinf(tau[0])


def test_score_always_one_predictor():
    rng = np.random.default_rng(1)
    z = rng.normal(size=1000)
    y = (rng.random(1000) < 0.4).astype(np.uint8)
    c = oracle.score(z, y, [-np.inf])
    assert c["fn"] == 0 and c["fp"] == int((y == 0).sum()) and c["tn"] == 0
    z[3] = np.nan  # NaN never satisfies >= tau (R26) and is counted
    c = oracle.score(z, y, [-np.inf])
    assert c["nonfinite"] == 1 and c["tp"] + c["fp"] == 999


def test_c1_training_reduces_fp_and_stays_conservative():
    """Invariant pin of the whole loop (trajectory itself: parity unpinned)."""
    cfg = nbgen.CONFIGS["c1"]
    g = nbgen.make_grid(cfg)
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, cfg.n_eval).numpy()
    y = oracle.label(g, 2, "point", q)
    a = oracle.arch_of(cfg)
    th0 = nbgen.init_params(cfg).double().numpy()
    steps = 60
    batches = ((q[(t % 16) * 4096:(t % 16 + 1) * 4096], y[(t % 16) * 4096:(t % 16 + 1) * 4096])
               for t in range(steps))
    th, hist = oracle.train(cfg, th0, batches, T=steps)
    fp = []
    for theta in (th0, th):
        z = oracle.forward(a, theta, q)
        tau, _ = oracle.calibrate(z, y)
        c = oracle.score(z, y, tau)
        assert c["fn"] == 0
        fp.append(c["fp"])
    assert fp[1] < fp[0]


def test_bf16_emulated_gradient_equals_torch_straight_through():
    """ORA_BF16_EMU gradient = the exact gradient of the bf16-precision forward
    (R33/R34), pinned against torch autograd through an independent bf16 chain
    whose roundings are straight-through (library routine)."""
    a = oracle.make_arch(4, 32, 6, (2, 4))
    th = rand_theta(a, 21, scale=1.5).astype(np.float32).astype(np.float64)
    rng = np.random.default_rng(22)
    q = rng.random((200, 4)).astype(np.float32)
    y = (rng.random(200) < 0.4).astype(np.uint8)
    loss, g, _ = oracle.loss_grad(a, th, q, y, 20.0, 1.0, mode=oracle.BF16_EMU)

    def st(x, f):  # straight-through rounding
        return x + (f(x) - x).detach()

    bfr = lambda x: x.float().to(torch.bfloat16).double()   # noqa: E731
    f32 = lambda x: x.float().double()                        # noqa: E731
    t = torch.tensor(th, requires_grad=True)
    x = torch.from_numpy(q)
    hi = x.to(torch.bfloat16).float()
    h = hi.double() + (x - hi).to(torch.bfloat16).double()
    p, d_in, rl = 0, a.d0, {}
    for l in range(a.layers):
        W = t[p:p + d_in * a.width].view(a.width, d_in); p += d_in * a.width
        b = t[p:p + a.width]; p += a.width
        z = st(st(h @ st(W, bfr).T, f32) + b, f32)
        r = torch.relu(z)
        rl[l + 1] = r
        h = st(r, bfr) if l < a.layers - 1 else r
        d_in = a.width
    wo = t[p:p + a.width]; p += a.width
    bo = t[p]; p += 1
    outs = [h @ wo + bo]
    for k in range(a.n_heads):
        u = t[p:p + a.width]; p += a.width
        c = t[p]; p += 1
        outs.append(rl[a.head_after[k]] @ u + c)  # heads read the fp32 ReLU output (R33)
    yt = torch.from_numpy(y).double()
    w = torch.where(yt > 0, 20.0, 1.0)
    L = sum(torch.nn.functional.binary_cross_entropy_with_logits(st(o, f32), yt, weight=w,
                                                                 reduction="sum") / 200 for o in outs)
    L.backward()
    assert loss == pytest.approx(L.item(), rel=1e-6)
    rel = np.linalg.norm(g - t.grad.numpy()) / np.linalg.norm(t.grad.numpy())
    assert rel < 2e-3, rel
