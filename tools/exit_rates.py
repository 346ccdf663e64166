"""Exit-rate probe for c4 (early-exit heads): train the 4->128x6->1 net with
its two heads under the paper's schedule for a few thousand steps, calibrate
all three thresholds to FN = 0, and print the exit histogram on fresh queries.
Measures how much work early-exit compaction can skip.  GPU only."""
import sys
import time

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import nbgen  # noqa: E402
import paper_2310_06822_b200 as nb  # noqa: E402


def main(steps=3000, batch=1 << 16, n_eval=1 << 22):
    cfg = nbgen.CONFIGS["c4"]
    dev = 0
    m = nb.Model(nb.Desc(cfg.kind, cfg.space_dim, cfg.width, cfg.hidden_layers, tuple(cfg.head_after),
                         "bf16"), dev)
    m.set_params(nbgen.init_params(cfg))
    g = nb.Grid(nbgen.make_grid(cfg), cfg.space_dim, dev)
    qe = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, n_eval, device=f"cuda:{dev}")
    ye = g.label(cfg.kind, qe)
    t0 = time.time()
    for t in range(steps):
        q = nbgen.make_queries(cfg, nbgen.TAG_TRAIN, t * batch, batch, device=f"cuda:{dev}")
        m.train_step(q, g.label(cfg.kind, q), alpha=nb.alpha(t, steps))
        if t % 500 == 499 or t == steps - 1:
            m.calibrate(qe, ye)
            c = m.score(qe, ye)
            h = c["exit_hist"]
            print(f"step {t + 1}: fp {c['fp']} tp {c['tp']} fn {c['fn']} exits {h} "
                  f"exit@1 {h[0] / n_eval:.3f} exit@2 {h[1] / n_eval:.3f} ({time.time() - t0:.1f}s)",
                  flush=True)


if __name__ == "__main__":
    main(*(int(a) for a in sys.argv[1:]))
