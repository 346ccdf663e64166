"""Pins for the oracle's sine activation (R41) and NeRF
positional encoding (Suppl. §3, R42) — SURVEY §8(f) NEXT-1.
Pins: the paper's 18-input arithmetic, feature values written out for
points where sin / cos are exact, a hand-computed sine KAT, an independent
torch fp64 chain (library sin / cos / linear / autograd), and central finite
differences (a sine net has no kinks, so the FD check is tight)."""
import math

import numpy as np
import pytest
import torch

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


def torch_features(x, pe):
    """gamma(x): x, then per k < pe/2: sin(2^k pi x), cos(2^k pi x) (library sin/cos)."""
    x = torch.as_tensor(x, dtype=torch.float32).double()
    parts = [x]
    for k in range(pe // 2):
        parts += [torch.sin((2.0 ** k) * math.pi * x), torch.cos((2.0 ** k) * math.pi * x)]
    return torch.cat(parts, 1)


def torch_forward(arch, theta, q, act, pe, emulate_bf16=False):
    th = torch.as_tensor(theta, dtype=torch.float64)
    h = torch_features(q, pe)
    if emulate_bf16:
        f = h.float()
        hi = f.to(torch.bfloat16).float()
        lo = (f - hi).to(torch.bfloat16).float()
        h = hi.double() + lo.double()
    sig = torch.sin if act == "sine" else torch.relu
    p, d_in = 0, h.shape[1]
    for l in range(arch.layers):
        W = th[p:p + d_in * arch.width].view(arch.width, d_in); p += d_in * arch.width
        b = th[p:p + arch.width]; p += arch.width
        if emulate_bf16:
            W = W.float().to(torch.bfloat16).double()
            z = torch.nn.functional.linear(h, W).float() + b.float()
            r = sig(z.double()).float()
            h = r.to(torch.bfloat16).double() if l < arch.layers - 1 else r.double()
        else:
            h = sig(torch.nn.functional.linear(h, W, b))
        d_in = arch.width
    wo = th[p:p + arch.width]
    z = h @ wo + th[p + arch.width]
    return z.float().double() if emulate_bf16 else z


def test_pe_gives_the_papers_18_inputs():
    """depth 8 on a 2D point -> 18-dimensional input; Suppl. Tab. 3's
    PE net 2 -> 128 x 3 -> 1 (Main Fig. 11 d) therefore has 19*128 + 2*129*128 + 129 params."""
    a = oracle.make_arch(2, 128, 3, pe=8)
    assert oracle.num_params(a) == 19 * 128 + 2 * 129 * 128 + 129
    assert oracle.num_params(oracle.make_arch(3, 10, 1, pe=4)) == (15 + 1) * 10 + 11


def _feature(x, j, pe):
    """f_j(x) through the oracle: relu(f_j) - relu(-f_j) with a 2-unit ReLU net."""
    a = oracle.make_arch(2, 2, 1, pe=pe)
    din = 2 * (1 + pe)
    th = np.zeros(oracle.num_params(a))
    th[j] = 1.0                 # W_1[0][j]
    th[din + j] = -1.0          # W_1[1][j]
    th[2 * din + 2] = 1.0       # w_out[0]   (after b_1[0..1])
    th[2 * din + 3] = -1.0      # w_out[1]
    return float(oracle.forward(a, th, np.array([x], np.float32))[0, 0])


def test_pe_feature_values_written_out():
    # x = (0, 0): x, then (sin, sin), (cos, cos) per frequency
    want0 = [0, 0] + [0, 0, 1, 1] * 4
    # x = (0.25, 0.5): frequencies pi, 2 pi, 4 pi, 8 pi
    r = math.sqrt(0.5)
    want1 = [0.25, 0.5,
             r, 1.0, r, 0.0,       # sin(pi/4), sin(pi/2), cos(pi/4), cos(pi/2)
             1.0, 0.0, 0.0, -1.0,  # sin(pi/2), sin(pi), cos(pi/2), cos(pi)
             0.0, 0.0, -1.0, 1.0,  # sin(pi), sin(2 pi), cos(pi), cos(2 pi)
             0.0, 0.0, 1.0, 1.0]   # sin(2 pi), sin(4 pi), cos(2 pi), cos(4 pi)
    for x, want in (((0.0, 0.0), want0), ((0.25, 0.5), want1)):
        got = [_feature(x, j, 8) for j in range(18)]
        assert np.allclose(got, want, atol=1e-14), (x, got)


def test_sine_kat():
    """One sine unit: W = 0, b = pi/6 -> h = sin(pi/6) = 1/2; w_out = 2,
    b_out = 0.25 -> z = 1.25.  All-zero parameters give z = 0 (yhat = 1/2)."""
    a = oracle.make_arch(2, 1, 1, act="sine")
    th = np.array([0.0, 0.0, math.pi / 6, 2.0, 0.25])
    q = np.array([[0.3, 0.9], [0.0, 1.0]], np.float32)
    assert np.allclose(oracle.forward(a, th, q), 1.25, atol=1e-15)
    assert np.all(oracle.forward(a, np.zeros(5), q) == 0.0)


@pytest.mark.parametrize("pe", [0, 8])
def test_sine_forward_equals_torch_fp64(pe):
    a = oracle.make_arch(2, 24, 3, act="sine", pe=pe)
    th = np.random.default_rng(1).normal(size=oracle.num_params(a)) * 0.7
    q = np.random.default_rng(2).random((257, 2)).astype(np.float32)
    z = oracle.forward(a, th, q)[:, 0]
    zt = torch_forward(a, th, q, "sine", pe).numpy()
    assert np.allclose(z, zt, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("act,pe", [("sine", 0), ("sine", 4), ("relu", 4)])
def test_sine_pe_bf16_emulation_equals_torch_bf16_chain(act, pe):
    a = oracle.make_arch(3, 32, 3, act=act, pe=pe)
    th = np.random.default_rng(3).normal(size=oracle.num_params(a)) * 0.5
    q = np.random.default_rng(4).random((200, 3)).astype(np.float32)
    z = oracle.forward(a, th, q, oracle.BF16_EMU)[:, 0]
    zt = torch_forward(a, th, q, act, pe, emulate_bf16=True).numpy()
    assert np.allclose(z, zt, rtol=1e-6, atol=1e-6)


@pytest.mark.parametrize("pe", [0, 4])
def test_sine_loss_and_grad_equal_torch_autograd(pe):
    a = oracle.make_arch(3, 16, 3, act="sine", pe=pe)
    th = np.random.default_rng(7).normal(size=oracle.num_params(a)) * 0.5
    rng = np.random.default_rng(8)
    q = rng.random((300, 3)).astype(np.float32)
    y = (rng.random(300) < 0.3).astype(np.uint8)
    alpha, beta, B = 37.0, 0.6, 1000
    loss, g, _ = oracle.loss_grad(a, th, q, y, alpha, beta, n_global=B)
    t = torch.tensor(th, requires_grad=True)
    z = torch_forward(a, t, q, "sine", pe)
    w = torch.where(torch.from_numpy(y).bool(), alpha, beta).double()
    L = torch.nn.functional.binary_cross_entropy_with_logits(z, torch.from_numpy(y).double(), weight=w,
                                                             reduction="sum") / B
    L.backward()
    assert loss == pytest.approx(L.item(), rel=1e-12)
    assert np.allclose(g, t.grad.numpy(), rtol=1e-9, atol=1e-14)


def test_sine_grad_central_finite_differences():
    a = oracle.make_arch(2, 6, 2, act="sine", pe=2)
    th = np.random.default_rng(11).normal(size=oracle.num_params(a)) * 0.8
    rng = np.random.default_rng(12)
    q = rng.random((64, 2)).astype(np.float32)
    y = (rng.random(64) < 0.5).astype(np.uint8)
    _, g, _ = oracle.loss_grad(a, th, q, y, 5.0, 1.0)
    h = 1e-5
    fd = np.zeros_like(g)
    for i in range(len(th)):
        tp, tm = th.copy(), th.copy()
        tp[i] += h
        tm[i] -= h
        fd[i] = (oracle.loss_grad(a, tp, q, y, 5.0, 1.0)[0] - oracle.loss_grad(a, tm, q, y, 5.0, 1.0)[0]) / (2 * h)
    assert np.allclose(fd, g, rtol=1e-6, atol=1e-9 * np.abs(g).max())


def test_encode_pe_operand_layout_and_values():
    """oracle.encode_pe (the K = 64 bf16 PE operand, R42/R20): hi at
    [0, d_in), lo at [32, 32 + d_in), zeros elsewhere; hi + lo reproduces the
    written-out features gamma(x) (x, then sin / cos of 2^k pi x per
    frequency) to the fp32 rounding, and hi is the RNE bf16 of that fp32."""
    import torch
    q = np.random.default_rng(1).random((200, 2)).astype(np.float32)
    e = oracle.encode_pe(q, 8)
    assert e.shape == (200, 64) and not e[:, 18:32].any() and not e[:, 50:].any()
    tof = lambda u: torch.from_numpy(u.view(np.int16).astype(np.int32) << 16).view(torch.float32).numpy()  # noqa: E731
    v = tof(e[:, :18].copy()).astype(np.float64) + tof(e[:, 32:50].copy())
    x = q.astype(np.float64)
    feats = [x[:, 0], x[:, 1]]
    for k in range(4):
        feats += [np.sin(2 ** k * np.pi * x[:, 0]), np.sin(2 ** k * np.pi * x[:, 1]),
                  np.cos(2 ** k * np.pi * x[:, 0]), np.cos(2 ** k * np.pi * x[:, 1])]
    ref = np.stack(feats, 1)
    assert np.all(np.abs(v - ref) <= 2.0 ** -16 * np.abs(ref) + 1e-12)
    hi = torch.from_numpy(ref.astype(np.float32)).bfloat16().view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(e[:, :18], hi)
