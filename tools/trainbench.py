"""Train-step timing of one config (dev tool): device time per nb_train_step
over pre-generated, pre-labelled batches.

    python tools/trainbench.py [config] [steps]
"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import nbgen
import paper_2310_06822_b200 as nb

if os.environ.get("NB_LIB", ""):  # measurement variant (build.py name=...)
    nb.LIB_PATH = os.path.join(os.path.dirname(nb.LIB_PATH), f"libnb_{os.environ['NB_LIB']}.so")

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
cfg = nbgen.CONFIGS[name]
m = nb.Model(nb.Desc(cfg.kind, cfg.space_dim, cfg.width, cfg.hidden_layers, tuple(cfg.head_after), cfg.precision), 0)
m.set_params(nbgen.init_params(cfg))
g = nb.Grid(nbgen.make_grid(cfg), cfg.space_dim, 0)
B = cfg.train_batch
qs = [nbgen.train_batch(cfg, t, 0, 1, device="cuda") for t in range(4)]
ys = [g.label(cfg.kind, q) for q in qs]
for t in range(3):
    m.train_step(qs[t % 4], ys[t % 4], alpha=1.0)
torch.cuda.synchronize()
m.set_timing(True)
m.kernel_time()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for t in range(steps):
    m.train_step(qs[t % 4], ys[t % 4], alpha=nb.alpha(t, steps))
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / steps
print(f"{name} train B={B}: {ms*1e3:.1f} us/step  {B/ms*1e3:.3e} samples/s")
