"""GPU parity at full pipeline depth.

Every row, not a sample, is compared with the oracle at sizes where each of
the persistent kernels' tile slots runs many tiles (148 CTAs x 5 slots for
c2, x 2 slots for c3/c4, 74 CTA pairs for c5: 11-14 tiles per slot), so the
double-buffered record staging, the mbarrier phase flips and the
next-tile/epilogue overlap all run in the compared launches.  Two weight
sets per config: the scaled random weights of the other tests (R46) and a
model trained through nb_train_step (the P2 case "trained weights").

Per config and weight set:
  P2  |sigmoid(z_gpu) - sigmoid(z_emu)| <= 2e-2 against the network the
      kernel evaluates (bf16 weights and activations, ORA_BF16_EMU, R33) on
      >= 99.99 % of rows (the rest: bf16 rounding flips from the fp32
      summation order, R47), so against the plain fp64 network the kernel
      adds at most 2e-2 to the bf16 network's own gap (printed); for the
      scaled weights the plain 2e-2 against fp64 holds on every row;
      the logit against ORA_BF16_EMU: >= 99 % of all rows and >= 90 % of
      every 128-row tile within the 1e-3 band (a tile staged from the wrong
      rows or a stale buffer fails the per-tile bound);
  P4  counts of the calibrated predictor bit-exact against the oracle's
      outside the band (R28), and the fused score's counts equal to the
      forward logits thresholded row by row (score and forward agree at
      depth, R23);
  P5  FN = 0 on the calibration set for both sides.
"""
import numpy as np
import pytest
import torch

import nbgen
import oracle
import paper_2310_06822_b200 as nb
from gpu_helpers import BAND, band_mask, desc_of, labels_oracle, scaled_params, sigmoid

pytestmark = pytest.mark.gpu
DEV = 0
DEPTH = [("c2", 1 << 20), ("c3", 1 << 19), ("c4", 1 << 19), ("c5", 1 << 18)]
TRAIN_STEPS = 1000
_TRAINED = {}


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")


def trained_params(cfg) -> torch.Tensor:
    """Xavier init + TRAIN_STEPS Adam steps of Eq. (1) through nb_train_step
    on fresh TRAIN batches of the config's batch (alpha 1 -> 1000)."""
    if cfg.name not in _TRAINED:
        m = nb.Model(desc_of(cfg), DEV)
        m.set_params(nbgen.init_params(cfg))
        g = nb.Grid(nbgen.make_grid(cfg), cfg.space_dim, DEV)
        for t in range(TRAIN_STEPS):
            qt = nbgen.train_batch(cfg, t, device=f"cuda:{DEV}")
            m.train_step(qt, g.label(cfg.kind, qt), alpha=nb.alpha(t, TRAIN_STEPS))
        _TRAINED[cfg.name] = m.get_params()
    return _TRAINED[cfg.name]


@pytest.mark.parametrize("weights", ["scaled", "trained"])
@pytest.mark.parametrize("name,n", DEPTH)
def test_every_row_at_depth(name, n, weights):
    cfg = nbgen.CONFIGS[name]
    th = scaled_params(cfg, 21) if weights == "scaled" else trained_params(cfg)
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, n)
    y = labels_oracle(cfg, q.numpy())
    qd, yd = q.to(f"cuda:{DEV}"), torch.from_numpy(y).to(f"cuda:{DEV}")
    m = nb.Model(desc_of(cfg), DEV)
    m.set_params(th)
    z = m.forward(qd).cpu().double().numpy()
    a = oracle.arch_of(cfg)
    th64 = th.double().numpy()
    # P2 every row against the network the kernel evaluates and against fp64 (R47)
    zr = oracle.forward(a, th64, q.numpy())
    ze = oracle.forward(a, th64, q.numpy(), oracle.BF16_EMU)
    err_emu = np.abs(sigmoid(z) - sigmoid(ze))
    # a flipped bf16 rounding (fp32 summation order, R35) can move one row of a
    # deep trained net by more; such rows are rare (R47)
    assert (err_emu.max(1) <= 2e-2).mean() >= 0.9999, int((err_emu.max(1) > 2e-2).sum())
    gap = np.abs(sigmoid(ze) - sigmoid(zr))          # the bf16 network vs the fp64 network (oracle only)
    err = np.abs(sigmoid(z) - sigmoid(zr))            # (<= gap + err_emu by the triangle inequality)
    if weights == "scaled":
        assert err.max() <= 2e-2, (err.max(), int(np.argmax(err.max(1))))
    print(name, weights, "max |dsig| vs emu %.2e, vs fp64 %.2e (bf16-network gap %.2e, rows > 2e-2: %d)"
          % (err_emu.max(), err.max(), gap.max(), int((err.max(1) > 2e-2).sum())))
    # every row against the kernel-precision oracle; per-tile bound catches pipeline faults
    close = np.all(np.abs(z - ze) < BAND, axis=1)
    assert close.mean() >= 0.99, close.mean()
    nt = n // 128
    per_tile = close[: nt * 128].reshape(nt, 128).mean(1)
    assert per_tile.min() >= 0.9, (per_tile.min(), int(per_tile.argmin()))
    # P5 + P4
    tau = m.calibrate(qd, yd).numpy()
    c = m.score(qd, yd)
    assert c["fn"] == 0 and c["tp"] == int(y.sum()) and c["tp"] + c["fp"] + c["fn"] + c["tn"] == n
    cf = oracle.score(z, y, tau)            # fused score == forward logits thresholded
    for k in ("tp", "fp", "fn", "tn", "exit_hist"):
        assert cf[k] == c[k], (k, cf, c)
    te, _ = oracle.calibrate(ze, y)
    ce = oracle.score(ze, y, te)
    assert ce["fn"] == 0
    # P4 outside the 1e-3 band of either threshold, on the rows where the kernel
    # and the emulation agree to the band: at trained weights a rare row's
    # logit moves by more when the fp32 summation order flips one bf16
    # rounding (R47); those rows are bounded by the checks above
    keep = ~band_mask(z, tau, ze, te) & close
    assert keep.mean() > 0.95
    kd = torch.from_numpy(keep).to(f"cuda:{DEV}")
    cg = m.score(qd[kd].contiguous(), yd[kd].contiguous())
    co = oracle.score(ze[keep], y[keep], te)
    for k in ("tp", "fp", "fn", "tn", "exit_hist"):
        assert cg[k] == co[k], (k, cg, co)


def _tensors(cfg):
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


@pytest.mark.parametrize("name", ["c2", "c3", "c4", "c5"])
def test_trained_gradient_parity_vs_fp64(name):
    """P3 at trained weights, over a batch spanning many tiles: one step's
    per-tensor gradient within 2e-2 of the gradient of the network the
    kernels evaluate (ORA_BF16_EMU, R34), and within 2e-2 + that network's
    own gap to the fp64 gradient of the plain definition (R47)."""
    cfg = nbgen.CONFIGS[name]
    th = trained_params(cfg)
    n = (1 << 14) + 77
    q = nbgen.make_queries(cfg, nbgen.TAG_HOLDOUT, 0, n)
    y = labels_oracle(cfg, q.numpy())
    m = nb.Model(desc_of(cfg), DEV)
    m.set_params(th)
    alpha = 500.0
    st = m.train_step(q.to(f"cuda:{DEV}"), torch.from_numpy(y).to(f"cuda:{DEV}"), alpha=alpha, stats=True)
    g = m.get_grad().double().numpy()
    a = oracle.arch_of(cfg)
    th64 = th.double().numpy()
    loss, gr, _ = oracle.loss_grad(a, th64, q.numpy(), y, alpha, 1.0)
    le, ge, _ = oracle.loss_grad(a, th64, q.numpy(), y, alpha, 1.0, mode=oracle.BF16_EMU)
    rel64 = {k: np.linalg.norm(g[s] - gr[s]) / np.linalg.norm(gr[s]) for k, s in _tensors(cfg)
             if np.linalg.norm(gr[s]) > 0}
    relem = {k: np.linalg.norm(g[s] - ge[s]) / np.linalg.norm(ge[s]) for k, s in _tensors(cfg)
             if np.linalg.norm(ge[s]) > 0}
    print(name, "rel64", {k: round(v, 4) for k, v in rel64.items()})
    print(name, "relemu", {k: round(v, 4) for k, v in relem.items()})
    gap = {k: np.linalg.norm(ge[s] - gr[s]) / np.linalg.norm(gr[s]) for k, s in _tensors(cfg)
           if np.linalg.norm(gr[s]) > 0}
    print(name, "bf16-network gap", {k: round(v, 4) for k, v in gap.items()})
    assert max(relem.values()) <= 2e-2, relem
    assert all(rel64[k] <= gap[k] + 2e-2 for k in rel64), (rel64, gap)
    assert abs(st["loss"] - le) <= 1e-3 * abs(le)
    assert abs(st["loss"] - loss) <= abs(le - loss) + 2e-2 * abs(loss)
