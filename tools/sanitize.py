"""Small invocations of the hand-rolled pipelines (SURVEY §5 race/sync
checking).  compute-sanitizer is closed on this pool, so the stand-in is the
NB_CHECKS build (libnb_checked.so: bounded mbarrier waits that trap with the
barrier and phase, alignment / bounds / TMEM-base checks) run on these cases
and compared bit for bit with the release build (tests/test_gpu_checked.py).

    python tools/sanitize.py [--lib checked] [part ...]     (prints one JSON line)

Parts: the fused forward (k_fwd_tc: forward, calibrate, score), the CTA-pair
kernels (k_fwd_tc2p, and k_fwd_tc2 for heads), the early-exit compaction
segments (k_score_exit), the fused w = 64 training kernel (k_train_fused),
the w = 128 and w = 256 training chains, 4D box records (K = 32 layer 1).
Sizes give every tile slot >= 2 tiles plus a ragged tail so the
double-buffered staging and mbarrier phase flips run.
"""
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import nbgen  # noqa: E402
import paper_2310_06822_b200 as nb  # noqa: E402


def digest(t: torch.Tensor) -> str:
    return hashlib.sha256(t.detach().cpu().contiguous().numpy().tobytes()).hexdigest()[:16]


def model(cfg, heads=None):
    m = nb.Model(nb.Desc(cfg.kind, cfg.space_dim, cfg.width, cfg.hidden_layers,
                         tuple(cfg.head_after) if heads is None else heads, cfg.precision), 0)
    m.set_params(nbgen.init_params(cfg) * 2.0 if heads is None else
                 torch.cat([nbgen.init_params(cfg) * 2.0, torch.full((len(heads) * (cfg.width + 1),), 0.01)]))
    return m


def grid(cfg):
    return nb.Grid(nbgen.make_grid(cfg), cfg.space_dim, 0)


def fwd(name, n, cfg=None):
    cfg = cfg or nbgen.CONFIGS[name]
    m, g = model(cfg), grid(cfg)
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, n, device="cuda:0")
    y = g.label(cfg.kind, q) if cfg.space_dim < 4 or cfg.kind == "point" else (q[:, 0] < 0.3).to(torch.uint8)
    z = m.forward(q)
    tau = m.calibrate(q, y)
    if cfg.n_heads:   # thresholds at logit quantiles so every segment has survivors and exits
        zc = z.cpu()
        m.set_thresholds([float(zc[:, 0].median()), float(zc[:, 1].quantile(0.4)), float(zc[:, 2].quantile(0.3))])
    c = m.score(q, y)
    return {"logits": digest(z), "tau": tau.tolist(), "counts": c}


def train(name, n, steps=2, cfg=None):
    cfg = cfg or nbgen.CONFIGS[name]
    m, g = model(cfg), grid(cfg)
    st = None
    for t in range(steps):
        q = nbgen.make_queries(cfg, nbgen.TAG_TRAIN, t * n, n, device="cuda:0")
        st = m.train_step(q, g.label(cfg.kind, q), alpha=10.0, stats=True)
    return {"grad": digest(m.get_grad()), "params": digest(m.get_params()),
            "stats": {k: st[k] for k in ("tp", "fp", "fn", "tn")}}


PARTS = {
    "fwd_c2": lambda: fwd("c2", 128 * 148 * 5 * 2 + 77),   # k_fwd_tc<64>: 5 slots x 2 tiles + tail
    "fwd_c3": lambda: fwd("c3", 128 * 148 * 2 * 2 + 5),
    "fwd_c5": lambda: fwd("c5", 256 * 74 * 2 + 200),       # k_fwd_tc2p (pipelined CTA pairs)
    "exit_c4": lambda: fwd("c4", 128 * 148 * 2 * 3 + 19),  # k_score_exit segments
    "fwd_4dbox": lambda: fwd("c4box", 128 * 148 * 2 * 2 + 9, nbgen.EXTRA_CONFIGS["c4box"]),
    "train_c2": lambda: train("c2", 128 * 148 * 2 + 77),   # k_train_fused
    "train_c3": lambda: train("c3", 128 * 148 + 5),        # kTrain forward, k_bwd_tc, k_dw_tc
    "train_c5": lambda: train("c5", 256 * 74 + 33),        # pipelined kTrain forward, k_bwd_tc2
}

if __name__ == "__main__":
    args = sys.argv[1:]
    if args[:1] == ["--lib"]:
        nb.LIB_PATH = os.path.join(os.path.dirname(nb.LIB_PATH), f"libnb_{args[1]}.so")
        args = args[2:]
    out = {}
    for p in (args or list(PARTS)):
        out[p] = PARTS[p]()
    torch.cuda.synchronize()
    print(json.dumps(out), flush=True)
