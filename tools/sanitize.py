"""Small invocations of the hand-rolled pipelines for compute-sanitizer
(SURVEY §5): memcheck / racecheck / synccheck over the fused forward
(k_fwd_tc: forward, calibrate, score), the CTA-pair kernel (k_fwd_tc2), the
early-exit compaction segments (k_score_exit), the fused w=64 training kernel
(k_train_fused) and the w=128 training chain (k_fwd_tc kTrain, k_bwd_tc,
k_dw_tc, k_dw_reduce, k_adam_pack).  Sizes give every tile slot >= 2 tiles
plus a ragged tail so the double-buffered staging and mbarrier phase flips run.

    compute-sanitizer --tool racecheck python tools/sanitize.py [part ...]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import nbgen  # noqa: E402
import paper_2310_06822_b200 as nb  # noqa: E402


def model(name):
    cfg = nbgen.CONFIGS[name]
    m = nb.Model(nb.Desc(cfg.kind, cfg.space_dim, cfg.width, cfg.hidden_layers, tuple(cfg.head_after),
                         cfg.precision), 0)
    m.set_params(nbgen.init_params(cfg) * 2.0)
    g = nb.Grid(nbgen.make_grid(cfg), cfg.space_dim, 0)
    return cfg, m, g


def fwd(name, n):
    cfg, m, g = model(name)
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, n, device="cuda:0")
    y = g.label(cfg.kind, q)
    m.forward(q)
    m.calibrate(q, y)
    if cfg.n_heads:   # thresholds at logit quantiles so every segment has survivors and exits
        z = m.forward(q).cpu()
        m.set_thresholds([float(z[:, 0].median()), float(z[:, 1].quantile(0.4)), float(z[:, 2].quantile(0.3))])
    c = m.score(q, y)
    print(name, "score", c, flush=True)


def train(name, n, steps=2):
    cfg, m, g = model(name)
    for t in range(steps):
        q = nbgen.make_queries(cfg, nbgen.TAG_TRAIN, t * n, n, device="cuda:0")
        st = m.train_step(q, g.label(cfg.kind, q), alpha=10.0, stats=True)
    print(name, "train", st, flush=True)


PARTS = {
    "fwd_c2": lambda: fwd("c2", 128 * 148 * 5 * 2 + 77),   # k_fwd_tc<64>: 5 slots x 2 tiles + tail
    "fwd_c3": lambda: fwd("c3", 128 * 148 * 2 * 2 + 5),
    "fwd_c5": lambda: fwd("c5", 256 * 74 * 2 + 200),       # k_fwd_tc2 (CTA pairs)
    "exit_c4": lambda: fwd("c4", 128 * 148 * 2 * 3 + 19),  # k_score_exit segments
    "train_c2": lambda: train("c2", 128 * 148 * 2 + 77),   # k_train_fused
    "train_c3": lambda: train("c3", 128 * 148 + 5),        # kTrain forward, k_bwd_tc, k_dw_tc
    "train_c5": lambda: train("c5", 256 * 74 + 33),        # CTA-pair training
}

if __name__ == "__main__":
    for p in (sys.argv[1:] or list(PARTS)):
        PARTS[p]()
    torch.cuda.synchronize()
    print("sanitize parts done", flush=True)
