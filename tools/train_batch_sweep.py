"""Train-step device time vs batch size (dev tool): the per-step chain latency of
the training kernels against their throughput at larger batches.

    python tools/train_batch_sweep.py [config] [log2 batch ...]
"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import nbgen
import paper_2310_06822_b200 as nb

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
logs = [int(a) for a in sys.argv[2:]] or [16, 17, 18, 20]
cfg = nbgen.CONFIGS[name]
g = nb.Grid(nbgen.make_grid(cfg), cfg.space_dim, 0)
flop = 2 * (cfg.record_floats * cfg.width + (cfg.hidden_layers - 1) * cfg.width ** 2 + cfg.width * (1 + cfg.n_heads))
for lb in logs:
    B = 1 << lb
    m = nb.Model(nb.Desc(cfg.kind, cfg.space_dim, cfg.width, cfg.hidden_layers, tuple(cfg.head_after), cfg.precision), 0)
    m.set_params(nbgen.init_params(cfg))
    qs = [nbgen.make_queries(cfg, nbgen.TAG_TRAIN, t * B, B, device="cuda") for t in range(4)]
    ys = [g.label(cfg.kind, q) for q in qs]
    for t in range(3):
        m.train_step(qs[t % 4], ys[t % 4], alpha=1.0)
    torch.cuda.synchronize()
    steps = 50
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for t in range(steps):
        m.train_step(qs[t % 4], ys[t % 4], alpha=nb.alpha(t, steps))
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / steps
    # forward + backward (dX and dW) = 3x the forward flops (dX of layer 1 is not needed: slightly less)
    print(f"{name} train B=2^{lb}: {ms*1e3:.1f} us/step  {B/ms*1e3:.3e} samples/s  "
          f"{3*flop*B/ms/1e9:.1f} TFLOP/s (3 x forward flops)", flush=True)
    del m, qs, ys
