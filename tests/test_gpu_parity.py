"""GPU parity tests: the CUDA path through the C ABI against the oracle on the
same seeded inputs (protocol P1-P6; tolerances from
BASELINE.json north_star).  All marked gpu."""
import ctypes

import numpy as np
import pytest
import torch

import nbgen
import oracle
import paper_2310_06822_b200 as nb
from gpu_helpers import (BAND, band_mask, desc_of, grid_of, labels_oracle, scaled_params,
                         sigmoid)

pytestmark = pytest.mark.gpu
DEV = 0


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    cc = nb.C.c_int32()
    assert nb.lib().nb_device_check(DEV, nb.C.byref(cc)) == 0, "libnb needs sm_100"


def cuda(t):
    return torch.as_tensor(t).to(f"cuda:{DEV}").contiguous()


# ---------------------------------------------------------------- labeller (P6)
@pytest.mark.parametrize("name,n", [("c1", 1 << 16), ("c2", 1 << 18), ("c3", 1 << 16),
                                    ("c4", 1 << 18), ("c5", 1 << 18)])
def test_labeller_bit_exact(name, n):
    cfg = nbgen.CONFIGS[name]
    q = nbgen.make_queries(cfg, nbgen.TAG_HOLDOUT, 0, n)
    y_ref = labels_oracle(cfg, q.numpy())
    g = nb.Grid(torch.from_numpy(grid_of(cfg)), cfg.space_dim, DEV)
    y = g.label(cfg.kind, cuda(q)).cpu().numpy()
    assert np.array_equal(y, y_ref), int((y != y_ref).sum())
    assert 0 < y.mean() < 1


def test_labeller_ray_edge_cases():
    cfg = nbgen.CONFIGS["c3"]
    R = 64
    rng = np.random.default_rng(0)
    o = np.round(rng.random((20000, 3)) * R) / R
    d = np.eye(3)[rng.integers(0, 3, 20000)] * rng.choice([-1, 1], (20000, 1))
    d[10000:] = rng.normal(size=(10000, 3))
    d[10000:] /= np.linalg.norm(d[10000:], axis=1, keepdims=True)
    q = np.concatenate([o, d], 1).astype(np.float32)
    y_ref = oracle.label(grid_of(cfg), 3, "ray", q)
    g = nb.Grid(torch.from_numpy(grid_of(cfg)), 3, DEV)
    assert np.array_equal(g.label("ray", cuda(q)).cpu().numpy(), y_ref)


# ---------------------------------------------------------------- encoder (a1)
@pytest.mark.parametrize("name", ["c2", "c3", "c4", "c5"])
def test_encode_bit_exact(name):
    cfg = nbgen.CONFIGS[name]
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, 5000)
    m = nb.Model(desc_of(cfg), DEV)
    x = m.encode(cuda(q)).cpu().numpy().view(np.uint16)
    assert np.array_equal(x, oracle.encode_bf16(q.numpy()))


# ---------------------------------------------------------------- fp32 path (c1)
def test_c1_fp32_forward_within_1e5():
    cfg = nbgen.CONFIGS["c1"]
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, cfg.n_eval)
    m = nb.Model(desc_of(cfg), DEV)
    for th in (nbgen.init_params(cfg), scaled_params(cfg, 1)):
        m.set_params(th)
        z, p = m.forward(cuda(q), prob=True)
        z = z.cpu().double().numpy()
        zr = oracle.forward(oracle.arch_of(cfg), th.double().numpy(), q.numpy())
        err = np.abs(z - zr) / np.maximum(1.0, np.abs(zr))
        assert err.max() <= 1e-5, err.max()
        assert np.allclose(p.cpu().numpy(), sigmoid(zr[:, 0]), atol=1e-6)


def test_c1_calibrate_score_counts():
    cfg = nbgen.CONFIGS["c1"]
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, cfg.n_eval)
    y = labels_oracle(cfg, q.numpy())
    th = scaled_params(cfg, 2)
    m = nb.Model(desc_of(cfg), DEV)
    m.set_params(th)
    qd, yd = cuda(q), cuda(y)
    tau = m.calibrate(qd, yd).numpy()
    c = m.score(qd, yd)
    zr = oracle.forward(oracle.arch_of(cfg), th.double().numpy(), q.numpy())
    tr, _ = oracle.calibrate(zr, y)
    cr = oracle.score(zr, y, tr)
    assert c["fn"] == 0 and cr["fn"] == 0                     # P5
    assert c["tp"] + c["fn"] == int(y.sum())
    zg = m.forward(qd).cpu().double().numpy()
    keep = ~band_mask(zg, tau, zr, tr)
    cg = m.score(cuda(q.numpy()[keep]), cuda(y[keep]))
    co = oracle.score(zr[keep], y[keep], tr)
    for k in ("tp", "fp", "fn", "tn"):
        assert cg[k] == co[k], (k, cg, co)                     # P4


def test_c1_train_step_gradient_parity():
    cfg = nbgen.CONFIGS["c1"]
    q = nbgen.train_batch(cfg, 0)
    y = labels_oracle(cfg, q.numpy())
    th = scaled_params(cfg, 3)
    m = nb.Model(desc_of(cfg), DEV)
    m.set_params(th)
    st = m.train_step(cuda(q), cuda(y), alpha=37.0, beta=1.0, lr=1e-3, stats=True)
    g = m.get_grad().double().numpy()
    loss, gr, sr = oracle.loss_grad(oracle.arch_of(cfg), th.double().numpy(), q.numpy(), y, 37.0, 1.0)
    assert abs(st["loss"] - loss) <= 1e-4 * abs(loss)
    assert np.linalg.norm(g - gr) <= 1e-4 * np.linalg.norm(gr)
    assert (st["tp"], st["fn"]) == (sr["tp"], sr["fn"])
    # Adam step applied to the fp32 master weights
    th1 = m.get_params().double().numpy()
    mm, vv = np.zeros_like(gr), np.zeros_like(gr)
    ref = th.double().numpy().copy()
    oracle.adam(ref, mm, vv, 1, g)
    assert np.allclose(th1, ref, atol=2e-6)


def test_c1_training_run_conservative():
    """200 Adam steps (BASELINE.json configs[0]); whole trajectory: parity
    unpinned (chaotic), checked by invariants: FN = 0 after calibration and
    FP below the initial network's."""
    cfg = nbgen.CONFIGS["c1"]
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, cfg.n_eval)
    y = labels_oracle(cfg, q.numpy())
    qd, yd = cuda(q), cuda(y)
    m = nb.Model(desc_of(cfg), DEV)
    th0 = nbgen.init_params(cfg)
    m.set_params(th0)
    m.calibrate(qd, yd)
    fp0 = m.score(qd, yd)["fp"]
    T = cfg.train_steps
    for t in range(T):
        sl = slice((t % 16) * 4096, (t % 16 + 1) * 4096)
        m.train_step(qd[sl], yd[sl], alpha=nb.alpha(t, T))
    m.calibrate(qd, yd)
    c = m.score(qd, yd)
    assert c["fn"] == 0 and c["fp"] < fp0


# ---------------------------------------------------------------- bf16 tensor-core path
BF16_CASES = [("c2", (1 << 16) + 77), ("c3", (1 << 15) + 5), ("c4", (1 << 15) + 129),
              ("c5", (1 << 15) + 200)]


@pytest.mark.parametrize("name,n", BF16_CASES)
def test_bf16_forward_sigmoid_within_2e2(name, n):
    cfg = nbgen.CONFIGS[name]
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, n)
    th = scaled_params(cfg, 4)
    m = nb.Model(desc_of(cfg), DEV)
    m.set_params(th)
    z, p = m.forward(cuda(q), prob=True)
    z = z.cpu().double().numpy()
    a = oracle.arch_of(cfg)
    zr = oracle.forward(a, th.double().numpy(), q.numpy())           # plain fp64 (P2)
    assert np.abs(sigmoid(z) - sigmoid(zr)).max() <= 2e-2
    assert np.abs(p.cpu().numpy() - sigmoid(zr[:, 0])).max() <= 2e-2
    ze = oracle.forward(a, th.double().numpy(), q.numpy(), oracle.BF16_EMU)  # kernel precision
    close = np.abs(z - ze) < BAND
    assert close.mean() > 0.99, close.mean()


@pytest.mark.parametrize("name,n", BF16_CASES)
def test_bf16_calibrate_score_counts(name, n):
    cfg = nbgen.CONFIGS[name]
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, n)
    y = labels_oracle(cfg, q.numpy())
    th = scaled_params(cfg, 5)
    m = nb.Model(desc_of(cfg), DEV)
    m.set_params(th)
    qd, yd = cuda(q), cuda(y)
    tau = m.calibrate(qd, yd).numpy()
    c = m.score(qd, yd)
    assert c["fn"] == 0                                               # P5 GPU
    assert sum(c[k] for k in ("tp", "fp", "fn", "tn")) == n
    assert sum(c["exit_hist"]) == n
    zg = m.forward(qd).cpu().double().numpy()
    # the fused score kernel and the forward kernel produce identical logits
    cf = oracle.score(zg, y, tau)
    for k in ("tp", "fp", "fn", "tn"):
        assert cf[k] == c[k]
    assert cf["exit_hist"] == c["exit_hist"]
    ze = oracle.forward(oracle.arch_of(cfg), th.double().numpy(), q.numpy(), oracle.BF16_EMU)
    te, _ = oracle.calibrate(ze, y)
    ce = oracle.score(ze, y, te)
    assert ce["fn"] == 0                                              # P5 oracle
    keep = ~band_mask(zg, tau, ze, te)
    assert keep.mean() > 0.95
    cg = m.score(cuda(q.numpy()[keep]), cuda(y[keep]))
    co = oracle.score(ze[keep], y[keep], te)
    for k in ("tp", "fp", "fn", "tn"):
        assert cg[k] == co[k], (k, cg, co)                            # P4


@pytest.mark.parametrize("n", [0, 1, 127, 128, 129, 255, 257, 128 * 148 * 2 + 1])
def test_bf16_edge_sizes(n):
    cfg = nbgen.CONFIGS["c2"]
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, max(n, 1))[:n]
    th = scaled_params(cfg, 6)
    m = nb.Model(desc_of(cfg), DEV)
    m.set_params(th)
    z = m.forward(cuda(q)).cpu().double().numpy()
    assert z.shape == (n, 1)
    if n:
        zr = oracle.forward(oracle.arch_of(cfg), th.double().numpy(), q.numpy())
        assert np.abs(sigmoid(z) - sigmoid(zr)).max() <= 2e-2
    c = m.score(cuda(q), cuda(np.zeros(n, np.uint8)))
    assert c["tp"] + c["fp"] + c["fn"] + c["tn"] == n


def test_score_host_equals_score():
    cfg = nbgen.CONFIGS["c2"]
    n = (1 << 21) + 333
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, n)
    g = nb.Grid(torch.from_numpy(grid_of(cfg)), 3, DEV)
    qd = cuda(q)
    yd = g.label("point", qd)
    m = nb.Model(desc_of(cfg), DEV)
    m.set_params(scaled_params(cfg, 7))
    m.calibrate(qd, yd)
    c1 = m.score(qd, yd)
    c2 = m.score_host(q, yd.cpu())
    assert c1 == c2 and c1["fn"] == 0


def test_no_positives_and_bad_labels():
    cfg = nbgen.CONFIGS["c2"]
    q = cuda(nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, 1000))
    m = nb.Model(desc_of(cfg), DEV)
    m.set_params(scaled_params(cfg, 8))
    tau = m.calibrate(q, cuda(np.zeros(1000, np.uint8)), allow_no_positives=True)
    assert np.isinf(tau[0].item())
    with pytest.raises(nb.NBError) as e:
        m.score(q, cuda(np.full(1000, 2, np.uint8)))
    assert e.value.status == 4  # NB_E_LABEL


# ---------------------------------------------------------------- bf16 training (a7-a9)
def param_tensors(cfg):
    """(name, slice) of every parameter tensor in the canonical blob (R32)."""
    out, p, d_in = [], 0, cfg.record_floats
    for l in range(cfg.hidden_layers):
        out.append((f"W{l + 1}", slice(p, p + d_in * cfg.width))); p += d_in * cfg.width
        out.append((f"b{l + 1}", slice(p, p + cfg.width))); p += cfg.width
        d_in = cfg.width
    out.append(("w_out", slice(p, p + cfg.width))); p += cfg.width
    out.append(("b_out", slice(p, p + 1))); p += 1
    for k in range(cfg.n_heads):
        out.append((f"u{k + 1}", slice(p, p + cfg.width))); p += cfg.width
        out.append((f"c{k + 1}", slice(p, p + 1))); p += 1
    return out


@pytest.mark.parametrize("name,n", [("c2", (1 << 13) + 77), ("c3", (1 << 12) + 5), ("c4", (1 << 12) + 33),
                                    ("c5", (1 << 12) + 300)])
def test_bf16_train_step_gradient_parity(name, n):
    """P3: one step from identical state, per parameter tensor
    ||g_gpu - g_oracle|| <= 2e-2 ||g_oracle|| (BASELINE.json north_star)."""
    cfg = nbgen.CONFIGS[name]
    q = nbgen.make_queries(cfg, nbgen.TAG_TRAIN, 0, n)
    y = labels_oracle(cfg, q.numpy())
    th = scaled_params(cfg, 9)
    m = nb.Model(desc_of(cfg), DEV)
    m.set_params(th)
    alpha = 50.0
    st = m.train_step(cuda(q), cuda(y), alpha=alpha, beta=1.0, lr=1e-3, stats=True)
    g = m.get_grad().double().numpy()
    a = oracle.arch_of(cfg)
    # the gradient of the bf16-precision network (R33/R34): kernels vs oracle
    le, ge_, _ = oracle.loss_grad(a, th.double().numpy(), q.numpy(), y, alpha, 1.0,
                                  mode=oracle.BF16_EMU)
    assert abs(st["loss"] - le) <= 1e-3 * abs(le)
    rel_emu = {nm: np.linalg.norm(g[sl] - ge_[sl]) / np.linalg.norm(ge_[sl])
               for nm, sl in param_tensors(cfg) if np.linalg.norm(ge_[sl]) > 0}
    assert max(rel_emu.values()) <= 2e-2, rel_emu
    # against the plain fp64 definition (BASELINE.json 2e-2): holds for the
    # shallow nets; the 6-layer c4 net differs from fp64 by the bf16 forward
    # itself (the oracle's own bf16-precision gradient shows the same gap):
    # the kernel is held to that gap + 2e-2 (R47)
    loss, gr, sr = oracle.loss_grad(a, th.double().numpy(), q.numpy(), y, alpha, 1.0)
    rel64 = {nm: np.linalg.norm(g[sl] - gr[sl]) / np.linalg.norm(gr[sl])
             for nm, sl in param_tensors(cfg) if np.linalg.norm(gr[sl]) > 0}
    if name != "c4":
        assert abs(st["loss"] - loss) <= 2e-2 * abs(loss)
        assert max(rel64.values()) <= 2e-2, rel64
    else:
        gap = {nm: np.linalg.norm(ge_[sl] - gr[sl]) / np.linalg.norm(gr[sl])
               for nm, sl in param_tensors(cfg) if np.linalg.norm(gr[sl]) > 0}
        assert all(rel64[k] <= gap[k] + 2e-2 for k in rel64), (rel64, gap)
    assert st["tp"] + st["fp"] + st["fn"] + st["tn"] == n


def test_bf16_training_run_conservative():
    """c2 architecture, 150 Adam steps at batch 2^14 (reduced from 5,000 x 2^16):
    invariants FN = 0 after calibration and FP below the initial network's."""
    cfg = nbgen.CONFIGS["c2"]
    g = nb.Grid(torch.from_numpy(grid_of(cfg)), 3, DEV)
    m = nb.Model(desc_of(cfg), DEV)
    m.set_params(nbgen.init_params(cfg))
    qe = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, 1 << 18, device=f"cuda:{DEV}")
    ye = g.label("point", qe)
    m.calibrate(qe, ye)
    fp0 = m.score(qe, ye)["fp"]
    T, B = 150, 1 << 14
    for t in range(T):
        qt = nbgen.make_queries(cfg, nbgen.TAG_TRAIN, t * B, B, device=f"cuda:{DEV}")
        m.train_step(qt, g.label("point", qt), alpha=nb.alpha(t, T))
    m.calibrate(qe, ye)
    c = m.score(qe, ye)
    assert c["fn"] == 0 and c["fp"] < fp0, (c, fp0)


# ---------------------------------------------------------------- full BASELINE.json sizes
@pytest.mark.parametrize("name", ["c2", "c3", "c4", "c5"])
def test_full_size_sampled_parity(name):
    """At the config's full N (c2 2^22, c3 2^24, c4 2^26, c5 2^28) in the launch
    configuration bench.py uses: properties that hold at any size (FN = 0 after
    calibration, count identities, fused score == forward + threshold) plus
    sampled rows checked one by one against the oracle (labels bit-exact,
    sigmoid within 2e-2 of fp64, logit vs bf16-precision oracle)."""
    cfg = nbgen.CONFIGS[name]
    N = cfg.n_eval
    dev = f"cuda:{DEV}"
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, N, device=dev)
    g = nb.Grid(torch.from_numpy(grid_of(cfg)), cfg.space_dim, DEV)
    y = g.label(cfg.kind, q)
    th = scaled_params(cfg, 10)
    m = nb.Model(desc_of(cfg), DEV)
    m.set_params(th)
    tau = m.calibrate(q, y).numpy()
    c = m.score(q, y)
    npos = int(y.sum().item())
    assert c["fn"] == 0
    assert c["tp"] == npos and c["tp"] + c["fp"] + c["fn"] + c["tn"] == N
    assert sum(c["exit_hist"]) == N and c["nonfinite"] == 0
    z = m.forward(q)
    zt = torch.tensor(tau, device=dev)
    pred = (z >= zt).all(dim=1)
    assert int((pred & (y == 0)).sum().item()) == c["fp"]
    # sampled rows, one by one against the oracle
    rng = np.random.default_rng(11)
    idx = np.sort(rng.choice(N, 3000, replace=False))
    it = torch.from_numpy(idx).to(dev)
    qs = q[it].cpu().numpy()
    assert np.array_equal(y[it].cpu().numpy(), labels_oracle(cfg, qs))
    zs = z[it].cpu().double().numpy()
    a = oracle.arch_of(cfg)
    zr = oracle.forward(a, th.double().numpy(), qs)
    assert np.abs(sigmoid(zs) - sigmoid(zr)).max() <= 2e-2
    ze = oracle.forward(a, th.double().numpy(), qs, oracle.BF16_EMU)
    assert (np.abs(zs - ze) < BAND).mean() > 0.99


@pytest.mark.gpu
def test_score_async_matches_score():
    """nb_score_async (pinned host and device destinations) gives nb_score's counts."""
    import torch

    cfg = nbgen.CONFIGS["c2"]
    n = 128 * 300 + 5
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, n, device="cuda:0")
    g = nb.Grid(nbgen.make_grid(cfg), cfg.space_dim, 0)
    y = g.label(cfg.kind, q)
    m = nb.Model(nb.Desc(cfg.kind, cfg.space_dim, cfg.width, cfg.hidden_layers, (), "bf16"), 0)
    m.set_params(nbgen.init_params(cfg) * 2.5)
    m.calibrate(q, y)
    ref = m.score(q, y)
    h = torch.zeros(9, dtype=torch.int64).pin_memory()
    d = torch.zeros(9, dtype=torch.int64, device="cuda:0")
    m.score_async(q, y, h)
    m.score_async(q, y, d)
    torch.cuda.synchronize()
    assert m.counts_dict(h) == ref and m.counts_dict(d) == ref
    assert ref["fn"] == 0
    # repeated launches re-arm the in-kernel finalisation (counters start at 0)
    for _ in range(3):
        m.score_async(q, y, h)
    torch.cuda.synchronize()
    assert m.counts_dict(h) == ref and m.score(q, y) == ref
    # n = 0 writes zeros; pageable host memory is rejected
    m.score_async(q[:0], y[:0], h)
    torch.cuda.synchronize()
    assert all(v == 0 for v in h.tolist())
    with pytest.raises(ValueError):
        m.score_async(q, y, torch.zeros(9, dtype=torch.int64))


@pytest.mark.parametrize("name", ["c2", "c3", "c4", "c5"])
def test_fused_adam_repack_matches_full_pack(name):
    """The training step's fused Adam + bf16 re-pack leaves exactly the image a
    full pack of the updated fp32 master builds: logits after 3 steps equal the
    logits of a fresh model given the same parameters (bit for bit)."""
    cfg = nbgen.CONFIGS[name]
    B = 1 << 12
    m = nb.Model(desc_of(cfg), DEV)
    m.set_params(scaled_params(cfg, 9))
    g = nb.Grid(torch.from_numpy(grid_of(cfg)), cfg.space_dim, DEV)
    for t in range(3):
        qt = nbgen.make_queries(cfg, nbgen.TAG_TRAIN, t * B, B, device=f"cuda:{DEV}")
        m.train_step(qt, g.label(cfg.kind, qt), alpha=10.0 * (t + 1))
    th = m.get_params()
    m2 = nb.Model(desc_of(cfg), DEV)
    m2.set_params(th)
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, 128 * 40 + 3, device=f"cuda:{DEV}")
    assert torch.equal(m.forward(q), m2.forward(q))


@pytest.mark.parametrize("name", ["c2", "c5"])
def test_train_micro_batches_equal_one_batch(name, monkeypatch):
    """A step split into micro-batches (dW partials accumulated in a fixed order)
    gives the single-batch gradient up to fp32 summation order, and the same
    loss and batch counts."""
    cfg = nbgen.CONFIGS[name]
    n = 5 * 1024 + 77
    q = nbgen.make_queries(cfg, nbgen.TAG_TRAIN, 0, n)
    y = labels_oracle(cfg, q.numpy())
    th = scaled_params(cfg, 9)
    out = []
    for chunk in (None, "1024"):
        if chunk:
            monkeypatch.setenv("NB_TRAIN_CHUNK", chunk)
        m = nb.Model(desc_of(cfg), DEV)
        m.set_params(th)
        st = m.train_step(cuda(q), cuda(y), alpha=20.0, beta=1.0, lr=1e-3, stats=True)
        out.append((st, m.get_grad().double().numpy()))
        monkeypatch.delenv("NB_TRAIN_CHUNK", raising=False)
    (s1, g1), (s2, g2) = out
    assert all(s1[k] == s2[k] for k in ("tp", "fp", "fn", "tn"))
    assert abs(s1["loss"] - s2["loss"]) <= 1e-5 * abs(s1["loss"])
    assert np.linalg.norm(g1 - g2) <= 1e-5 * np.linalg.norm(g1)


@pytest.mark.parametrize("name,fused", [("c2", False), ("c3", True), ("c4", True), ("c5", True)])
def test_relu_bit_masks_equal_h_images(name, fused, monkeypatch):
    """The backward's ReLU' (R25: [h_l > 0]) read from the forward's bit masks
    equals the one read from the h_l images: bit-identical gradient, loss and
    counts (NB_NO_MASKS=1 selects the h-image read; c2 runs the unfused
    kernels with NB_NO_FUSED=1)."""
    cfg = nbgen.CONFIGS[name]
    n = 7 * 1024 + 77
    q = nbgen.make_queries(cfg, nbgen.TAG_TRAIN, 0, n)
    y = labels_oracle(cfg, q.numpy())
    th = scaled_params(cfg, 13)
    if not fused:
        monkeypatch.setenv("NB_NO_FUSED", "1")
    out = []
    for no_masks in (False, True):
        if no_masks:
            monkeypatch.setenv("NB_NO_MASKS", "1")
        m = nb.Model(desc_of(cfg), DEV)
        m.set_params(th)
        st = m.train_step(cuda(q), cuda(y), alpha=20.0, beta=1.0, lr=1e-3, stats=True)
        out.append((st, m.get_grad()))
    (s1, g1), (s2, g2) = out
    assert all(s1[k] == s2[k] for k in ("tp", "fp", "fn", "tn")), (s1, s2)
    assert abs(s1["loss"] - s2["loss"]) <= 1e-12 * abs(s1["loss"])   # fp64 atomic sum order
    assert torch.equal(g1, g2), float((g1 - g2).abs().max())


@pytest.mark.parametrize("name", ["c1", "c2", "c5"])
def test_nonfinite_records(name):
    """Non-finite input ("non-finite input -> error"; R26):
    nb_score counts the rows whose logit is not finite, never predicts them
    positive when NaN, and returns the warning-class NB_E_NONFINITE with the
    counts written; nb_forward's NaN logits surface as NB_E_NONFINITE on the
    next synchronising call."""
    cfg = nbgen.CONFIGS[name]
    n = 128 * 3 + 9
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, n)
    y = labels_oracle(cfg, q.numpy())
    m = nb.Model(desc_of(cfg), DEV)
    m.set_params(scaled_params(cfg, 9))
    qd, yd = cuda(q), cuda(y)
    m.calibrate(qd, yd, allow_no_positives=True)
    ref = m.score(qd, yd)
    bad = q.clone()
    rows = [0, 130, n - 1]
    for r in rows:
        bad[r, 0] = float("nan")
    with pytest.raises(nb.NBError) as ei:
        m.score(cuda(bad), yd)
    assert "NONFINITE" in str(ei.value)
    c = m.score(cuda(bad), yd, allow_nonfinite=True)
    assert c["nonfinite"] == len(rows)
    assert c["tp"] + c["fp"] + c["fn"] + c["tn"] == n
    # a non-finite record's logit is NaN, which never passes z >= tau: those rows
    # move to the predicted-negative side, every other row is unchanged
    z0 = m.forward(qd)
    predpos = (z0[rows, 0].cpu() >= m.get_thresholds()[0]).numpy()
    pos_bad = [r for r, pp in zip(rows, predpos) if pp]
    assert c["tp"] + c["fp"] == ref["tp"] + ref["fp"] - len(pos_bad)
    z = m.forward(cuda(bad))
    assert torch.isnan(z[rows, 0]).all() and torch.isfinite(z[[1, 2, 129], 0]).all()
    with pytest.raises(nb.NBError):
        m.calibrate(qd, yd, allow_no_positives=True)  # reports the forward's flag


def test_nccl_communicator_world1():
    """The NCCL path of nb_comm_init / the in-library allreduces on a real GPU
    (world size 1 on the one-GPU box; the multi-rank host logic is covered by
    the gloo tests): calibrate, score, score_async and a training step with a
    communicator give the results of the same model without one."""
    import os
    import socket

    import torch.distributed as dist

    from paper_2310_06822_b200.dist import comm_init

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", DEV))
    try:
        cfg = nbgen.CONFIGS["c2"]
        n = 128 * 50 + 3
        q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, n)
        y = labels_oracle(cfg, q.numpy())
        qd, yd = cuda(q), cuda(y)
        th = scaled_params(cfg, 9)
        out = []
        for with_comm in (False, True):
            m = nb.Model(desc_of(cfg), DEV)
            if with_comm:
                comm_init(m)
            m.set_params(th)
            tau = m.calibrate(qd, yd)
            c = m.score(qd, yd)
            h = torch.zeros(9, dtype=torch.int64).pin_memory()
            m.score_async(qd, yd, h)
            torch.cuda.synchronize()
            st = m.train_step(qd, yd, alpha=5.0, stats=True)
            out.append((tau, c, m.counts_dict(h), st, m.get_grad()))
        (t0, c0, a0, s0, g0), (t1, c1, a1, s1, g1) = out
        assert torch.equal(t0, t1) and c0 == c1 and a0 == a1 == c0
        assert all(s0[k] == s1[k] for k in ("tp", "fp", "fn", "tn"))
        assert torch.equal(g0, g1)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["c1", "c2", "c5"])
def test_regularized_adam_step(name):
    """NEXT-2 (Suppl. §2.2, R38): with L1/L2 set, the step's Adam update uses
    g + l1 sign(theta) + 2 l2 theta over every parameter (fp32 SIMT, fused w=64
    and CTA-pair paths); get_grad stays the pure Eq. (1) gradient."""
    cfg = nbgen.CONFIGS[name]
    B = 3 * 1024 + 5
    q = nbgen.make_queries(cfg, nbgen.TAG_TRAIN, 0, B)
    y = labels_oracle(cfg, q.numpy())
    th = scaled_params(cfg, 4).double().numpy()
    th[::7] = 0.0                                   # sign(0) = 0 on both sides
    l1, l2 = 3e-3, 0.4
    m = nb.Model(desc_of(cfg), DEV)
    m.set_params(torch.from_numpy(th).float())
    m.set_regularization(l1, l2)
    m.train_step(cuda(q), cuda(y), alpha=5.0, beta=0.8, lr=1e-3)
    g = m.get_grad().double().numpy()
    th32 = torch.from_numpy(th).float().double().numpy()
    ref = th32.copy()
    mm, vv = np.zeros_like(ref), np.zeros_like(ref)
    oracle.adam(ref, mm, vv, 1, g + oracle.reg_grad(th32, l1, l2))
    noreg = th32.copy()
    oracle.adam(noreg, np.zeros_like(ref), np.zeros_like(ref), 1, g)
    th1 = m.get_params().double().numpy()
    assert np.allclose(th1, ref, atol=2e-6)
    assert not np.allclose(th1, noreg, atol=2e-6)   # the terms did act
    # the gradient itself is not regularised
    _, gr, _ = oracle.loss_grad(oracle.arch_of(cfg), th32, q.numpy(), y, 5.0, 0.8,
                                mode=oracle.FP64 if cfg.precision == "fp32" else oracle.BF16_EMU)
    assert np.linalg.norm(g - gr) <= 2e-2 * np.linalg.norm(gr)


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_paper_training_control_run(name):
    """NEXT-2 end to end: training driven by the paper's control (R37-R39):
    the batch FN the kernels report feed nb_schedule_after_step, its alpha,
    beta and lambda drive the next step.  The schedule equals the oracle's on
    the same FN sequence, and the calibrated network keeps FN = 0."""
    cfg = nbgen.CONFIGS[name]
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, 1 << 16)
    y = labels_oracle(cfg, q.numpy())
    qd, yd = cuda(q), cuda(y)
    m = nb.Model(desc_of(cfg), DEV)
    m.set_params(nbgen.init_params(cfg))
    s = nb.PaperSchedule(cfg.space_dim, step_every=5, max_steps=120)
    o = oracle.PaperSchedule(cfg.space_dim, step_every=5, max_steps=120)
    fns = []
    while not s.stop:
        t = s.step
        m.set_regularization(s.lam, s.lam)
        sl = slice((t % 16) * 4096, (t % 16 + 1) * 4096)
        st = m.train_step(qd[sl], yd[sl], alpha=s.alpha, beta=s.beta, lr=1e-3, stats=True)
        fns.append(st["fn"])
        s.after_step(st["fn"])
        o.after_step(st["fn"])
        assert (s.alpha, s.beta, s.triggers, s.stop) == \
            (pytest.approx(o.alpha), pytest.approx(o.beta), o.triggers, o.stop)
        assert s.lam == pytest.approx(o.lam, abs=1e-20)
    assert len(fns) <= 120 and sum(fns) > 0 and s.triggers > 0
    m.calibrate(qd, yd)
    assert m.score(qd, yd)["fn"] == 0


# ---------------------------------------------------------------- early-exit compaction (K9)
def _exit_model(n, seed=0):
    cfg = nbgen.CONFIGS["c4"]
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, seed, n)
    y = labels_oracle(cfg, q.numpy())
    m = nb.Model(desc_of(cfg), DEV)
    m.set_params(scaled_params(cfg, 3))
    return cfg, q, y, m


def _score_both(m, qd, yd):
    L = nb.lib()
    try:
        c = m.score(qd, yd, allow_nonfinite=True)
        L.nb_debug_set_dense_exits(1)
        d = m.score(qd, yd, allow_nonfinite=True)
    finally:
        L.nb_debug_set_dense_exits(0)
    return c, d


class _ExitRecords:
    """Select the record hand-off between the exit segments (survivors' fp32
    records, later segments recompute the earlier layers) for a block."""

    def __init__(self, on):
        self.on = on

    def __enter__(self):
        nb.lib().nb_debug_set_exit_records(1 if self.on else 0)

    def __exit__(self, *a):
        nb.lib().nb_debug_set_exit_records(0)


@pytest.mark.parametrize("handoff", ["images", "records"])
@pytest.mark.parametrize("n", [1, 127, 128, 129, 2 * 148 * 128 + 77, (1 << 20) + 5])
def test_exit_compaction_counts_equal_dense(n, handoff):
    """the compacted three-segment score (survivors of each head
    packed into full tiles) gives exactly the dense kernel's counts and exit
    histogram, with either hand-off between the segments (activation images
    or records + recompute); thresholds are set at logit quantiles so both
    heads exit a sizeable share of rows."""
    cfg, q, y, m = _exit_model(n)
    qd, yd = cuda(q), cuda(y)
    z = m.forward(qd).cpu()
    m.set_thresholds([float(z[:, 0].median()), float(z[:, 1].quantile(0.4)) if n > 1 else 0.0,
                      float(z[:, 2].quantile(0.3)) if n > 1 else 0.0])
    with _ExitRecords(handoff == "records"):
        c, d = _score_both(m, qd, yd)
    assert c == d, (c, d)
    assert sum(c["exit_hist"]) == n
    if n > 1000:
        assert c["exit_hist"][0] > 0.2 * n and c["exit_hist"][1] > 0.05 * n


def test_exit_compaction_vs_oracle_and_chunks():
    """Compaction in chunks (2^20 rows here, so four chunks plus a ragged
    tail; 2^24 by default): counts equal the dense kernel's and the
    bf16-emulating oracle's outside the 1e-3 band of every threshold
    (R28)."""
    n = (1 << 22) + 3 * 128 + 11
    cfg, q, y, m = _exit_model(n, seed=1)
    qd, yd = cuda(q), cuda(y)
    z = m.forward(qd).cpu()
    tau = [float(z[:, 0].median()), float(z[:, 1].quantile(0.5)), float(z[:, 2].quantile(0.2))]
    m.set_thresholds(tau)
    L = nb.lib()
    L.nb_debug_set_exit_chunk.argtypes = [ctypes.c_int64]
    try:
        L.nb_debug_set_exit_chunk(1 << 20)
        c, d = _score_both(m, qd, yd)
        with _ExitRecords(True):
            cr, _ = _score_both(m, qd, yd)
        L.nb_debug_set_exit_chunk(0)
        c1, _ = _score_both(m, qd, yd)
        with _ExitRecords(True):
            cr1, _ = _score_both(m, qd, yd)
    finally:
        L.nb_debug_set_exit_chunk(0)
    assert c == d and c1 == d and cr == d and cr1 == d
    # oracle on a sample of rows away from every threshold
    rng = np.random.default_rng(0)
    idx = np.sort(rng.choice(n, 40000, replace=False))
    zs = z[idx].double().numpy()
    keep = np.all(np.abs(zs - np.array(tau)) >= 1e-3, axis=1)
    idx = idx[keep]
    th = m.get_params().double().numpy()
    zo = oracle.forward(oracle.arch_of(cfg), th, q.numpy()[idx], oracle.BF16_EMU)
    zo = zo.reshape(len(idx), -1)
    keep2 = np.all(np.abs(zo - np.array(tau)) >= 1e-3, axis=1)
    idx, zo = idx[keep2], zo[keep2]
    sub = m.score(cuda(q.numpy()[idx]), cuda(y[idx]))
    co = oracle.score(zo, y[idx], np.array(tau, dtype=np.float64))
    for k in ("tp", "fp", "fn", "tn", "exit_hist"):
        assert sub[k] == co[k], (k, sub, co)
    assert co["exit_hist"][0] > 0.3 * len(idx) and co["exit_hist"][1] > 0.05 * len(idx)


def test_exit_compaction_nonfinite_and_async_paths():
    """NaN records exit at head 1 and are counted once as non-finite; the
    async (device destination) and host-buffer entry points take the same
    compacted path and agree with nb_score."""
    n = 3 * 128 * 148 + 19
    cfg, q, y, m = _exit_model(n, seed=2)
    z = m.forward(cuda(q)).cpu()
    m.set_thresholds([float(z[:, 0].median()), float(z[:, 1].quantile(0.4)), float(z[:, 2].quantile(0.4))])
    bad = q.clone()
    rows = [0, 200, 9000, n - 1]
    for r in rows:
        bad[r, 1] = float("nan")
    c, d = _score_both(m, cuda(bad), cuda(y))
    assert c == d and c["nonfinite"] == len(rows)
    out = torch.zeros(9, dtype=torch.int64, device=f"cuda:{DEV}")
    m.score_async(cuda(bad), cuda(y), out)
    assert nb.Model.counts_dict(out.cpu()) == c
    clean = m.score(cuda(q), cuda(y))
    h = m.score_host(q.contiguous(), torch.from_numpy(y).contiguous())
    assert h == clean


# ---------------------------------------------------------------- NEXT-1: sine + positional encoding
def _sine_case(name, width, layers, pe, precision, n, seed=0, scale=0.9):
    cfg = nbgen.CONFIGS[name]
    desc = nb.Desc(cfg.kind, cfg.space_dim, width, layers, (), precision, activation="sine",
                   pe_depth=pe)
    a = oracle.make_arch(cfg.record_floats, width, layers, act="sine", pe=pe)
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, seed, n)
    y = labels_oracle(cfg, q.numpy())
    rng = np.random.default_rng(seed + 5)
    th = rng.uniform(-1, 1, oracle.num_params(a)) * scale * np.sqrt(6.0 / (width + width))
    return cfg, desc, a, q, y, th


@pytest.mark.parametrize("pe", [0, 8])
def test_fp32_sine_pe_forward_and_gradient(pe):
    """fp32 path (P1 / P3 tolerances) with the paper's sine activation
    and the NeRF encoding (Suppl. §3; 2D points, depth 8 -> 18 inputs)."""
    cfg, desc, a, q, y, th = _sine_case("c1", 32, 2, pe, "fp32", 4096 + 77)
    m = nb.Model(desc, DEV)
    m.set_params(torch.from_numpy(th).float())
    th32 = torch.from_numpy(th).float().double().numpy()
    z = m.forward(cuda(q)).cpu().double().numpy()[:, 0]
    zr = oracle.forward(a, th32, q.numpy())[:, 0]
    assert np.all(np.abs(z - zr) <= 1e-5 * np.maximum(1.0, np.abs(zr)))
    st = m.train_step(cuda(q), cuda(y), alpha=9.0, beta=0.7, lr=1e-3, stats=True)
    g = m.get_grad().double().numpy()
    loss, gr, sr = oracle.loss_grad(a, th32, q.numpy(), y, 9.0, 0.7)
    assert abs(st["loss"] - loss) <= 1e-4 * abs(loss)
    assert np.linalg.norm(g - gr) <= 1e-4 * np.linalg.norm(gr)


@pytest.mark.parametrize("name,width,layers,pe,n", [("c2", 64, 3, 0, (1 << 15) + 77),
                                                    ("c1", 128, 3, 8, (1 << 15) + 5),
                                                    ("c2", 128, 2, 4, (1 << 14) + 3)])
def test_bf16_sine_pe_forward_and_counts(name, width, layers, pe, n):
    """bf16 tensor-core path with sine epilogues (range-reduced SFU sine) and
    the in-kernel positional encoding (layer-1 K up to 64): sigmoid within
    2e-2 of the fp64 definition, counts equal to the bf16-emulating oracle's
    outside the threshold band, FN = 0 on the calibration set."""
    cfg, desc, a, q, y, th = _sine_case(name, width, layers, pe, "bf16", n)
    m = nb.Model(desc, DEV)
    m.set_params(torch.from_numpy(th).float())
    th32 = torch.from_numpy(th).float().double().numpy()
    qd, yd = cuda(q), cuda(y)
    z, p = m.forward(qd, prob=True)
    zr = oracle.forward(a, th32, q.numpy())[:, 0]
    assert np.max(np.abs(p.cpu().double().numpy() - 1 / (1 + np.exp(-zr)))) <= 2e-2
    tau = m.calibrate(qd, yd).numpy()
    c = m.score(qd, yd)
    assert c["fn"] == 0
    ze = oracle.forward(a, th32, q.numpy(), oracle.BF16_EMU)
    te, _ = oracle.calibrate(ze, y)
    zg = z.cpu().double().numpy()
    keep = ~band_mask(zg, tau, ze, te)
    assert keep.mean() > 0.95
    cg = m.score(cuda(q.numpy()[keep]), cuda(y[keep]))
    co = oracle.score(ze[keep], y[keep], te)
    for k in ("tp", "fp", "fn", "tn"):
        assert cg[k] == co[k], (k, cg, co)


def test_sine_pe_unsupported_paths_fail_loudly():
    """Paths not built fail loudly (NB_E_UNSUPPORTED, never a silent
    fallback): nb_encode of an fp32 PE net (it encodes in place), training of
    sine / PE nets on CTA pairs (w = 256), sine pair nets with exit heads."""
    cfg, desc, a, q, y, th = _sine_case("c2", 64, 3, 2, "fp32", 1024)
    m = nb.Model(nb.Desc("point", 3, 32, 2, (), "fp32", activation="sine", pe_depth=2), DEV)
    with pytest.raises(nb.NBError) as ei:
        m.encode(cuda(q))
    assert "UNSUPPORTED" in str(ei.value)
    m2 = nb.Model(nb.Desc("point", 3, 256, 3, (), "bf16", activation="sine"), DEV)
    with pytest.raises(nb.NBError) as ei:
        m2.train_step(cuda(q), cuda(y), alpha=2.0)
    assert "UNSUPPORTED" in str(ei.value)
    with pytest.raises(nb.NBError):
        nb.Model(nb.Desc("point", 3, 256, 4, (2,), "bf16", activation="sine"), DEV)
    with pytest.raises(nb.NBError) as ei:   # a 4-layer PE pair image exceeds shared memory
        nb.Model(nb.Desc("point", 3, 256, 4, (), "bf16", activation="sine", pe_depth=4), DEV)
    assert "UNSUPPORTED" in str(ei.value)


@pytest.mark.parametrize("name,layers,pe,n", [("c2", 3, 0, 256 * 74 * 2 + 77), ("c1", 3, 8, 256 * 74 * 2 + 5),
                                              ("c2", 3, 4, 256 * 74 + 3), ("c2", 4, 0, 256 * 74 * 3 + 11)])
def test_bf16_sine_pe_on_cta_pairs(name, layers, pe, n):
    """The paper's architecture at w = 256 (sine hidden layers; NeRF
    encoding) on the pipelined CTA-pair kernel: sigmoid within
    2e-2 of fp64, counts equal to the bf16-emulating oracle outside the band,
    FN = 0 after calibration."""
    cfg, desc, a, q, y, th = _sine_case(name, 256, layers, pe, "bf16", n, scale=0.7)
    m = nb.Model(desc, DEV)
    m.set_params(torch.from_numpy(th).float())
    th32 = torch.from_numpy(th).float().double().numpy()
    qd, yd = cuda(q), cuda(y)
    z, p = m.forward(qd, prob=True)
    zr = oracle.forward(a, th32, q.numpy())[:, 0]
    assert np.max(np.abs(p.cpu().double().numpy() - 1 / (1 + np.exp(-zr)))) <= 2e-2
    tau = m.calibrate(qd, yd).numpy()
    assert m.score(qd, yd)["fn"] == 0
    ze = oracle.forward(a, th32, q.numpy(), oracle.BF16_EMU)
    te, _ = oracle.calibrate(ze, y)
    zg = z.cpu().double().numpy()
    keep = ~band_mask(zg, tau, ze, te)
    assert keep.mean() > 0.9
    cg = m.score(cuda(q.numpy()[keep]), cuda(y[keep]))
    co = oracle.score(ze[keep], y[keep], te)
    assert all(cg[k] == co[k] for k in ("tp", "fp", "fn", "tn")), (cg, co)


def _tensor_slices(din, width, layers):
    out, p, d_in = [], 0, din
    for l in range(layers):
        out.append((f"W{l + 1}", slice(p, p + d_in * width))); p += d_in * width
        out.append((f"b{l + 1}", slice(p, p + width))); p += width
        d_in = width
    out.append(("w_out", slice(p, p + width))); p += width
    out.append(("b_out", slice(p, p + 1)))
    return out


@pytest.mark.parametrize("name,width,layers,pe,n", [("c2", 64, 3, 0, (1 << 13) + 77),
                                                    ("c2", 128, 3, 0, (1 << 12) + 5),
                                                    ("c1", 128, 3, 8, (1 << 12) + 33),
                                                    ("c2", 64, 2, 4, (1 << 12) + 9)])
def test_bf16_sine_pe_train_step_gradient_parity(name, width, layers, pe, n):
    """NEXT-1 training on tensor cores: the forward keeps cos(z_l) images for
    the backward chain (delta = g cos z, R41) and the PE layer-1 image (K =
    64); per-tensor gradient within 2e-2 of the oracle's bf16-precision
    gradient, then the fused Adam + re-pack leaves exactly the image a full
    pack builds (logits bit-identical)."""
    cfg, desc, a, q, y, th = _sine_case(name, width, layers, pe, "bf16", n, seed=3)
    m = nb.Model(desc, DEV)
    m.set_params(torch.from_numpy(th).float())
    th32 = torch.from_numpy(th).float().double().numpy()
    alpha = 20.0
    st = m.train_step(cuda(q), cuda(y), alpha=alpha, beta=1.0, lr=1e-3, stats=True)
    g = m.get_grad().double().numpy()
    le, ge_, _ = oracle.loss_grad(a, th32, q.numpy(), y, alpha, 1.0, mode=oracle.BF16_EMU)
    assert abs(st["loss"] - le) <= 1e-3 * abs(le)
    rel = {nm: np.linalg.norm(g[sl] - ge_[sl]) / np.linalg.norm(ge_[sl])
           for nm, sl in _tensor_slices(cfg.record_floats * (1 + pe), width, layers)
           if np.linalg.norm(ge_[sl]) > 0}
    assert max(rel.values()) <= 2e-2, rel
    m2 = nb.Model(desc, DEV)
    m2.set_params(m.get_params())
    qq = cuda(q[:1000])
    assert torch.equal(m.forward(qq), m2.forward(qq))


# ---------------------------------------------------------------- NEXT-3: planes, OccNet ablation
def _plane_cfg():
    import dataclasses
    return dataclasses.replace(nbgen.CONFIGS["c3"], name="c3plane", kind="plane")


def test_gpu_plane_labeller_bit_exact():
    """Plane queries (R19): the GPU labeller (block-pruned fp64 corner
    test) equals the oracle's voxel scan, including planes through voxel
    faces and edges (closed-side ties)."""
    cfg = _plane_cfg()
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, 6000).numpy()
    R = nbgen.CONFIGS["c3"].grid["R"]
    edge = []
    for k in (0, 1, 17, 32, 63, 64):   # axis-aligned planes on grid faces
        for ax in range(3):
            p0 = [0.5, 0.5, 0.5]
            p0[ax] = k / R
            nrm = [0.0, 0.0, 0.0]
            nrm[ax] = 1.0
            edge.append(p0 + nrm)
    edge.append([0.25, 0.25, 0.25, 0.70710678, 0.70710678, 0.0])
    q = np.concatenate([q, np.array(edge, np.float32)], 0)
    grid = grid_of(nbgen.CONFIGS["c3"])
    y_ora = oracle.label(grid, 3, "plane", q)
    g = nb.Grid(torch.from_numpy(grid), 3, DEV)
    y_gpu = g.label("plane", cuda(torch.from_numpy(q))).cpu().numpy()
    assert np.array_equal(y_gpu, y_ora)
    assert 0.05 < y_ora.mean() < 0.99


def test_bf16_plane_queries_forward_and_counts():
    """Plane records (p0, unit normal) through the fused kernels (the encoder
    is kind-agnostic: 6 floats like a ray): sigmoid within 2e-2 of fp64 and
    counts equal to the bf16-emulating oracle outside the band."""
    cfg = _plane_cfg()
    n = (1 << 14) + 21
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, n)
    grid = grid_of(nbgen.CONFIGS["c3"])
    y = oracle.label(grid, 3, "plane", q.numpy())
    th = scaled_params(nbgen.CONFIGS["c3"], 4)
    m = nb.Model(nb.Desc("plane", 3, 128, 4, (), "bf16"), DEV)
    m.set_params(th)
    qd, yd = cuda(q), cuda(y)
    z, p = m.forward(qd, prob=True)
    a = oracle.make_arch(6, 128, 4)
    zr = oracle.forward(a, th.double().numpy(), q.numpy())[:, 0]
    assert np.max(np.abs(p.cpu().double().numpy() - 1 / (1 + np.exp(-zr)))) <= 2e-2
    tau = m.calibrate(qd, yd).numpy()
    ze = oracle.forward(a, th.double().numpy(), q.numpy(), oracle.BF16_EMU)
    te, _ = oracle.calibrate(ze, y)
    keep = ~band_mask(z.cpu().double().numpy(), tau, ze, te)
    cg = m.score(cuda(q.numpy()[keep]), cuda(y[keep]))
    co = oracle.score(ze[keep], y[keep], te)
    assert all(cg[k] == co[k] for k in ("tp", "fp", "fn", "tn")), (cg, co)
    assert m.score(qd, yd)["fn"] == 0


def test_symmetric_loss_ablation_leaves_false_negatives():
    """The OccNet-style symmetric loss (alpha = beta = 1) trained
    like c1 misses positives at the rounding rule z >= 0; the
    asymmetric ramp of Eq. (1) leaves fewer, and calibration (R21) removes
    them for both."""
    cfg = nbgen.CONFIGS["c1"]
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, cfg.n_eval)
    y = labels_oracle(cfg, q.numpy())
    qd, yd = cuda(q), cuda(y)
    fn = {}
    for mode in ("symmetric", "asymmetric"):
        m = nb.Model(desc_of(cfg), DEV)
        m.set_params(nbgen.init_params(cfg))
        T = cfg.train_steps
        for t in range(T):
            sl = slice((t % 16) * 4096, (t % 16 + 1) * 4096)
            m.train_step(qd[sl], yd[sl], alpha=1.0 if mode == "symmetric" else nb.alpha(t, T), beta=1.0)
        m.set_thresholds([0.0])
        fn[mode] = m.score(qd, yd)["fn"]
        m.calibrate(qd, yd)
        assert m.score(qd, yd)["fn"] == 0
    assert fn["symmetric"] > 0 and fn["asymmetric"] < fn["symmetric"], fn


@pytest.mark.parametrize("name", ["c1", "c2", "c5"])
def test_inverted_certainly_hit_bounding(name):
    """Inverted bounding (R43): trained with the asymmetry flipped
    (FP weight ramped, FN weight 1), nb_calibrate_inverted's threshold is the
    next float above the largest negative logit: FP = 0 on the set, equal to
    the oracle's (bf16-emulating for bf16 nets) max over negatives outside
    the band."""
    cfg = nbgen.CONFIGS[name]
    n = 1 << 14
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, n)
    y = labels_oracle(cfg, q.numpy())
    qd, yd = cuda(q), cuda(y)
    m = nb.Model(desc_of(cfg), DEV)
    m.set_params(nbgen.init_params(cfg))
    B = 4096
    for t in range(30):
        sl = slice((t % 4) * B, (t % 4 + 1) * B)
        m.train_step(qd[sl], yd[sl], alpha=1.0, beta=nb.alpha(t, 30), lr=1e-3)
    tau = float(m.calibrate_inverted(qd, yd)[0])
    c = m.score(qd, yd)
    assert c["fp"] == 0 and c["tp"] + c["fn"] == int(y.sum())
    z = m.forward(qd).cpu().double().numpy()[:, 0]
    zmax = z[y == 0].max()
    assert tau == np.nextafter(np.float32(zmax), np.float32(np.inf))
    mode = oracle.FP64 if cfg.precision == "fp32" else oracle.BF16_EMU
    zo = oracle.forward(oracle.arch_of(cfg), m.get_params().double().numpy(), q.numpy(), mode)[:, 0]
    tol = 1e-5 * max(1.0, abs(zmax)) if cfg.precision == "fp32" else 1e-3 + 2e-2 * abs(zmax)
    assert abs(zo[y == 0].max() - zmax) <= tol


@pytest.mark.parametrize("kind", ["ray", "box", "plane"])
def test_gpu_2d_labellers_bit_exact_and_kernels(kind):
    """2D rays, boxes and lines (4-float records, NEXT-3) on the c1 grid: the
    GPU labeller equals the oracle (pixel readings of R15-R19), and a bf16
    4 -> 64 x 3 net scores them with counts equal to the bf16-emulating
    oracle outside the band and FN = 0 after calibration."""
    import dataclasses
    cfg = dataclasses.replace(nbgen.CONFIGS["c1"], kind=kind)
    n = (1 << 14) + 3
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, n)
    grid = grid_of(nbgen.CONFIGS["c1"])
    y = oracle.label(grid, 2, kind, q.numpy())
    g = nb.Grid(torch.from_numpy(grid), 2, DEV)
    assert np.array_equal(g.label(kind, cuda(q)).cpu().numpy(), y)
    assert 0.02 < y.mean() < 0.98
    a = oracle.make_arch(4, 64, 3)
    th = torch.from_numpy(np.random.default_rng(2).normal(size=oracle.num_params(a)) * 0.15).float()
    m = nb.Model(nb.Desc(kind, 2, 64, 3, (), "bf16"), DEV)
    m.set_params(th)
    qd, yd = cuda(q), cuda(y)
    tau = m.calibrate(qd, yd).numpy()
    assert m.score(qd, yd)["fn"] == 0
    zg = m.forward(qd).cpu().double().numpy()
    ze = oracle.forward(a, th.double().numpy(), q.numpy(), oracle.BF16_EMU)
    te, _ = oracle.calibrate(ze, y)
    keep = ~band_mask(zg, tau, ze, te)
    cg = m.score(cuda(q.numpy()[keep]), cuda(y[keep]))
    co = oracle.score(ze[keep], y[keep], te)
    assert all(cg[k] == co[k] for k in ("tp", "fp", "fn", "tn")), (cg, co)


@pytest.mark.parametrize("width,pe", [(64, 0), (128, 8)])
def test_sine_pe_train_micro_batches_equal_one_batch(width, pe, monkeypatch):
    """Sine / PE training split into micro-batches (the cos images and the
    K = 64 layer-1 image per chunk) gives the single-batch gradient up to
    fp32 summation order."""
    cfg, desc, a, q, y, th = _sine_case("c1", width, 3, pe, "bf16", 5 * 1024 + 77, seed=4)
    out = []
    for chunk in (None, "1024"):
        if chunk:
            monkeypatch.setenv("NB_TRAIN_CHUNK", chunk)
        m = nb.Model(desc, DEV)
        m.set_params(torch.from_numpy(th).float())
        st = m.train_step(cuda(q), cuda(y), alpha=20.0, beta=1.0, lr=1e-3, stats=True)
        out.append((st, m.get_grad().double().numpy()))
        monkeypatch.delenv("NB_TRAIN_CHUNK", raising=False)
    (s1, g1), (s2, g2) = out
    assert all(s1[k] == s2[k] for k in ("tp", "fp", "fn", "tn"))
    assert np.linalg.norm(g1 - g2) <= 1e-5 * np.linalg.norm(g1)


def test_bf16_sine_with_exit_heads():
    """Sine nets with early-exit heads (heads read sin(z_l), R41/R22) take the
    dense EXT kernels (compaction is ReLU-only): every head's logit within the
    bf16 tolerance of fp64, counts and exit histogram equal to the
    bf16-emulating oracle outside the band."""
    cfg = nbgen.CONFIGS["c4"]
    n = (1 << 14) + 9
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, n)
    y = labels_oracle(cfg, q.numpy())
    a = oracle.make_arch(4, 128, 6, (2, 4), act="sine")
    th = np.random.default_rng(6).uniform(-1, 1, oracle.num_params(a)) * 0.9 * np.sqrt(6.0 / 256)
    m = nb.Model(nb.Desc("point", 4, 128, 6, (2, 4), "bf16", activation="sine"), DEV)
    m.set_params(torch.from_numpy(th).float())
    th32 = torch.from_numpy(th).float().double().numpy()
    qd, yd = cuda(q), cuda(y)
    zg = m.forward(qd).cpu().double().numpy()
    zr = oracle.forward(a, th32, q.numpy())
    assert np.max(np.abs(1 / (1 + np.exp(-zg)) - 1 / (1 + np.exp(-zr)))) <= 2e-2
    tau = m.calibrate(qd, yd).numpy()
    assert m.score(qd, yd)["fn"] == 0
    ze = oracle.forward(a, th32, q.numpy(), oracle.BF16_EMU)
    te, _ = oracle.calibrate(ze, y)
    keep = ~band_mask(zg, tau, ze, te)
    assert keep.mean() > 0.9
    cg = m.score(cuda(q.numpy()[keep]), cuda(y[keep]))
    co = oracle.score(ze[keep], y[keep], te)
    for k in ("tp", "fp", "fn", "tn", "exit_hist"):
        assert cg[k] == co[k], (k, cg, co)


# ---------------------------------------------------------------- data-parallel semantics (§8(e))
@pytest.mark.parametrize("name", ["c2", "c5"])
def test_two_shards_equal_one_call(name):
    """libnb's data-parallel semantics on one GPU: two models
    holding the same parameters each take one contiguous shard (dist.shard,
    tile-aligned) and the host combines what NCCL would: tau = min of the
    shard minima, counts = sum, gradient = sum of the shard gradients with
    each shard normalised by n_global.  Thresholds and counts equal the one
    full call bit for bit; the summed gradient equals the full-batch gradient
    up to fp32 summation order, the loss and batch counts likewise."""
    from paper_2310_06822_b200.dist import shard
    cfg = nbgen.CONFIGS[name]
    n = 128 * 148 * 2 + 333
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, n)
    y = labels_oracle(cfg, q.numpy())
    qd, yd = cuda(q), cuda(y)
    th = scaled_params(cfg, 12)
    full = nb.Model(desc_of(cfg), DEV)
    full.set_params(th)
    tau = full.calibrate(qd, yd)
    c = full.score(qd, yd)
    parts = [shard(n, r, 2) for r in range(2)]
    ms = []
    for s0, cnt in parts:
        m = nb.Model(desc_of(cfg), DEV)
        m.set_params(th)
        ms.append(m)
    taus = [m.calibrate(qd[s0:s0 + cnt], yd[s0:s0 + cnt]) for m, (s0, cnt) in zip(ms, parts)]
    tg = torch.minimum(taus[0], taus[1])
    assert torch.equal(tg, tau)
    tot = dict(tp=0, fp=0, fn=0, tn=0)
    for m, (s0, cnt) in zip(ms, parts):
        m.set_thresholds(tg)
        cs = m.score(qd[s0:s0 + cnt], yd[s0:s0 + cnt])
        for k in tot:
            tot[k] += cs[k]
    assert tot == {k: c[k] for k in tot} and tot["fn"] == 0
    # one data-parallel training step: shard gradients normalised by n_global
    B = 128 * 40 + 77
    qt = nbgen.make_queries(cfg, nbgen.TAG_TRAIN, 0, B)
    yt = labels_oracle(cfg, qt.numpy())
    qtd, ytd = cuda(qt), cuda(yt)
    full.set_params(th)
    sf = full.train_step(qtd, ytd, alpha=30.0, stats=True)
    gf = full.get_grad().double().numpy()
    gs, ss = np.zeros_like(gf), dict(loss=0.0, tp=0, fp=0, fn=0, tn=0)
    for m, (s0, cnt) in zip(ms, [shard(B, r, 2) for r in range(2)]):
        m.set_params(th)
        st = m.train_step(qtd[s0:s0 + cnt], ytd[s0:s0 + cnt], alpha=30.0, n_global=B, stats=True)
        gs += m.get_grad().double().numpy()
        for k in ss:
            ss[k] += st[k]
    assert all(ss[k] == sf[k] for k in ("tp", "fp", "fn", "tn"))
    assert abs(ss["loss"] - sf["loss"]) <= 1e-5 * abs(sf["loss"])
    assert np.linalg.norm(gs - gf) <= 1e-5 * np.linalg.norm(gf)


def test_misaligned_views_rejected_aligned_offsets_work():
    """nb.h "Alignment": a q/y view that is not 16-byte aligned (row 1 of a
    contiguous tensor) is rejected with NB_E_ARG before any launch (no
    misaligned bulk copy can fault the context); a 16-row offset works and
    equals the same rows copied to a fresh allocation."""
    cfg = nbgen.CONFIGS["c2"]
    n = 128 * 30 + 5
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, n)
    y = labels_oracle(cfg, q.numpy())
    qd, yd = cuda(q), cuda(y)
    m = nb.Model(desc_of(cfg), DEV)
    m.set_params(scaled_params(cfg, 2))
    m.calibrate(qd, yd)
    for call in (lambda: m.forward(qd[1:]), lambda: m.score(qd[1:], yd[1:]),
                 lambda: m.score(qd[:n - 1], yd[1:]), lambda: m.calibrate(qd[3:], yd[3:]),
                 lambda: m.train_step(qd[1:], yd[1:], alpha=2.0)):
        with pytest.raises(nb.NBError) as ei:
            call()
        assert ei.value.status == 1  # NB_E_ARG
    assert m.score(qd[16:], yd[16:]) == m.score(qd[16:].clone(), yd[16:].clone())
    assert torch.equal(m.forward(qd[16:]), m.forward(qd[16:].clone()))
    torch.cuda.synchronize()   # the context is healthy


# ---------------------------------------------------------------- NEXT-3: 4D rays, hyperplanes, boxes (R48)
@pytest.mark.parametrize("kind,n", [("ray", (1 << 15) + 77), ("box", (1 << 15) + 5), ("plane", (1 << 13) + 3)])
def test_4d_queries_bf16_forward_counts_and_gradient(kind, n):
    """8-float records through the tensor-core kernels (layer 1 K = 32: hi, lo
    and the bias ones in a second K step): encoder bytes bit-exact, sigmoid
    within 2e-2 of fp64, counts equal to the bf16-emulating oracle outside
    the band, FN = 0 after calibration on both sides, and one training
    step's per-tensor gradient within 2e-2 of the kernel-precision oracle."""
    cfg = nbgen.EXTRA_CONFIGS["c4" + kind]
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, n)
    y = labels_oracle(cfg, q.numpy())
    assert 0.01 < y.mean() < 0.99
    a = oracle.arch_of(cfg)
    th = scaled_params(cfg, 13, scale=1.8)
    m = nb.Model(desc_of(cfg), DEV)
    m.set_params(th)
    qd, yd = cuda(q), cuda(y)
    assert np.array_equal(m.encode(qd).cpu().numpy().view(np.uint16), oracle.encode_bf16(q.numpy()))
    z = m.forward(qd).cpu().double().numpy()
    zr = oracle.forward(a, th.double().numpy(), q.numpy())
    assert np.abs(sigmoid(z) - sigmoid(zr)).max() <= 2e-2
    tau = m.calibrate(qd, yd).numpy()
    c = m.score(qd, yd)
    assert c["fn"] == 0 and c["tp"] == int(y.sum())
    ze = oracle.forward(a, th.double().numpy(), q.numpy(), oracle.BF16_EMU)
    te, _ = oracle.calibrate(ze, y)
    assert oracle.score(ze, y, te)["fn"] == 0
    keep = ~band_mask(z, tau, ze, te)
    assert keep.mean() > 0.95
    cg = m.score(cuda(q.numpy()[keep]), cuda(y[keep]))
    co = oracle.score(ze[keep], y[keep], te)
    assert all(cg[k] == co[k] for k in ("tp", "fp", "fn", "tn")), (cg, co)
    nt = 4096 + 33
    st = m.train_step(qd[:nt], yd[:nt], alpha=40.0, stats=True)
    g = m.get_grad().double().numpy()
    le, ge, _ = oracle.loss_grad(a, th.double().numpy(), q.numpy()[:nt], y[:nt], 40.0, 1.0, mode=oracle.BF16_EMU)
    assert abs(st["loss"] - le) <= 1e-3 * abs(le)
    rel = {nm: np.linalg.norm(g[sl] - ge[sl]) / np.linalg.norm(ge[sl]) for nm, sl in param_tensors(cfg)
           if np.linalg.norm(ge[sl]) > 0}
    assert max(rel.values()) <= 2e-2, rel


@pytest.mark.parametrize("kind", ["ray", "box", "plane"])
def test_4d_queries_fp32_path(kind):
    """fp32 CUDA-core path with 8-float records: forward within 1e-5 of fp64
    (P1) and the gradient within 1e-4."""
    cfg = nbgen.EXTRA_CONFIGS["c4" + kind]
    n = 4096 + 17
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, n)
    y = labels_oracle(cfg, q.numpy())
    a = oracle.make_arch(8, 32, 2)
    th = torch.from_numpy(np.random.default_rng(3).normal(size=oracle.num_params(a)) * 0.3).float()
    m = nb.Model(nb.Desc(kind, 4, 32, 2, (), "fp32"), DEV)
    m.set_params(th)
    z = m.forward(cuda(q)).cpu().double().numpy()
    zr = oracle.forward(a, th.double().numpy(), q.numpy())
    assert np.all(np.abs(z - zr) <= 1e-5 * np.maximum(1.0, np.abs(zr)))
    m.train_step(cuda(q), cuda(y), alpha=9.0)
    g = m.get_grad().double().numpy()
    _, gr, _ = oracle.loss_grad(a, th.double().numpy(), q.numpy(), y, 9.0, 1.0)
    assert np.linalg.norm(g - gr) <= 1e-4 * np.linalg.norm(gr)


def test_4d_training_run_conservative():
    """A short training run on 4D boxes (the c4 scene, 300 steps x 2^14,
    alpha 1 -> 1000): FN = 0 after calibration and FP below the initial
    network's."""
    cfg = nbgen.EXTRA_CONFIGS["c4box"]
    m = nb.Model(desc_of(cfg), DEV)
    m.set_params(nbgen.init_params(cfg))
    qe = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, 1 << 16)
    ye = labels_oracle(cfg, qe.numpy())
    qd, yd = cuda(qe), cuda(ye)
    m.calibrate(qd, yd)
    fp0 = m.score(qd, yd)["fp"]
    T, B = 300, 1 << 14
    qt = nbgen.make_queries(cfg, nbgen.TAG_TRAIN, 0, 4 * B)
    yt = labels_oracle(cfg, qt.numpy())
    qtd, ytd = cuda(qt), cuda(yt)
    for t in range(T):
        sl = slice((t % 4) * B, (t % 4 + 1) * B)
        m.train_step(qtd[sl], ytd[sl], alpha=nb.alpha(t, T))
    m.calibrate(qd, yd)
    c = m.score(qd, yd)
    assert c["fn"] == 0 and c["fp"] < fp0, (c, fp0)


@pytest.mark.parametrize("name,pe", [("c1", 8), ("c2", 4), ("c2", 2)])
def test_encode_pe_operand(name, pe):
    """nb_encode of a bf16 PE net returns the K = 64 operand the kernels
    build (R42): equal to the oracle's (fp64 features rounded to fp32, bf16
    hi / lo split) except where the kernel's fp32 sincospif differs from the
    correctly rounded value by an ulp — hi bit-exact on >= 99.9 % of the
    features, hi + lo within 2^-16 relative everywhere, layout zeros exact."""
    cfg = nbgen.CONFIGS[name]
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, 40000)
    m = nb.Model(nb.Desc(cfg.kind, cfg.space_dim, 128, 3, (), "bf16", activation="sine", pe_depth=pe), DEV)
    e = m.encode(cuda(q)).cpu().numpy().view(np.uint16)
    o = oracle.encode_pe(q.numpy(), pe)
    din = cfg.record_floats * (1 + pe)
    assert e.shape == (40000, 64)
    assert not e[:, din:32].any() and not e[:, 32 + din:].any()
    assert (e[:, :din] == o[:, :din]).mean() >= 0.999
    tof = lambda u: torch.from_numpy(u.view(np.int16).astype(np.int32) << 16).view(torch.float32).numpy()  # noqa: E731
    vg = tof(e[:, :din].copy()).astype(np.float64) + tof(e[:, 32:32 + din].copy())
    vo = tof(o[:, :din].copy()).astype(np.float64) + tof(o[:, 32:32 + din].copy())
    # a 1-ulp fp32 feature difference can flip lo's bf16 rounding: 2^-16 relative
    assert np.all(np.abs(vg - vo) <= 2.0 ** -16 * np.maximum(np.abs(vo), 2.0 ** -10))


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c5"])
def test_train_steps_graph_equals_step_loop(name):
    """nb_train_steps (the step sequence captured in one CUDA graph) leaves
    exactly the parameters, Adam state and gradient of the same number of
    nb_train_step calls with the same batches and alpha ramp; two
    consecutive calls (re-capture, bias corrections of later steps) too."""
    cfg = nbgen.CONFIGS[name]
    T, B = 6, 2048
    q = nbgen.make_queries(cfg, nbgen.TAG_TRAIN, 0, 2 * T * B)
    y = labels_oracle(cfg, q.numpy())
    qd, yd = cuda(q), cuda(y)
    th = scaled_params(cfg, 17)
    a = nb.Model(desc_of(cfg), DEV)
    b = nb.Model(desc_of(cfg), DEV)
    a.set_params(th)
    b.set_params(th)
    for c in range(2):
        for t in range(T):
            r = (c * T + t) * B
            a.train_step(qd[r:r + B], yd[r:r + B], alpha=2.0 + 98.0 * t / (T - 1), beta=0.9, lr=2e-3)
        b.train_steps(qd[c * T * B:(c + 1) * T * B], yd[c * T * B:(c + 1) * T * B], T, 2.0, 100.0, beta=0.9, lr=2e-3)
    torch.cuda.synchronize()
    assert torch.equal(a.get_params(), b.get_params())
    assert torch.equal(a.get_grad(), b.get_grad())
    ma, va, sa = a.get_adam()
    mb, vb, sb = b.get_adam()
    assert sa == sb == 2 * T and torch.equal(ma, mb) and torch.equal(va, vb)


@pytest.mark.parametrize("kind,n", [("ray", 1 << 16), ("box", 1 << 16), ("plane", 1 << 13)])
def test_labeller_4d_bit_exact(kind, n):
    """P6 for 4D rays / hyperplanes / boxes (R48): the GPU labeller (4-axis
    fp64 DDA, 4D summed-area table, block-pruned 16-corner cut test) equals
    the oracle on the c4 scene, with axis-aligned rays / hyperplanes through
    cell faces added."""
    cfg = nbgen.EXTRA_CONFIGS["c4" + kind]
    q = nbgen.make_queries(cfg, nbgen.TAG_HOLDOUT, 0, n).numpy()
    rng = np.random.default_rng(4)
    extra = np.zeros((512, 8), np.float32)
    res = np.array([64, 64, 64, 32])
    extra[:, :4] = np.round(rng.random((512, 4)) * res) / res
    extra[:, 4:] = np.eye(4)[rng.integers(0, 4, 512)] * rng.choice([-1, 1], (512, 1))
    if kind == "box":
        extra[:, 4:] = np.minimum(1.0, extra[:, :4] + rng.random((512, 4)) * 0.1)
    q = np.concatenate([q, extra], 0)
    y_ref = labels_oracle(cfg, q)
    g = nb.Grid(torch.from_numpy(grid_of(cfg)), 4, DEV)
    y = g.label(kind, cuda(torch.from_numpy(q))).cpu().numpy()
    assert np.array_equal(y, y_ref), int((y != y_ref).sum())
    assert 0 < y.mean() < 1
