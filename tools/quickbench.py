"""Quick device-time measurement of the fused score kernel (dev tool)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time

import torch

import nbgen
import paper_2310_06822_b200 as nb

if os.environ.get("NB_NO_FOLD"):
    nb.lib().nb_debug_set_no_fold(1)
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
logn = int(sys.argv[2]) if len(sys.argv) > 2 else 22
cfg = nbgen.CONFIGS[name]
n = 1 << logn
q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, n, device="cuda")
g = nb.Grid(nbgen.make_grid(cfg), cfg.space_dim, 0)
y = g.label(cfg.kind, q)
m = nb.Model(nb.Desc(cfg.kind, cfg.space_dim, cfg.width, cfg.hidden_layers, tuple(cfg.head_after), cfg.precision), 0)
m.set_params(nbgen.init_params(cfg) * 2.5)
m.calibrate(q, y)
flop = 2 * (cfg.record_floats * cfg.width + (cfg.hidden_layers - 1) * cfg.width ** 2 + cfg.width * (1 + cfg.n_heads))
logits = torch.empty(n, 1 + cfg.n_heads, device="cuda")
for mode in ["forward", "score"]:
    ts = []
    for it in range(8):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        if mode == "forward":
            nb.lib().nb_forward(m._h, q.data_ptr(), n, logits.data_ptr(), None, torch.cuda.current_stream().cuda_stream)
        else:
            m.score(q, y)
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    t = sorted(ts)[len(ts) // 2] * 1e-3
    print(f"{name} {mode} n=2^{logn}: {t*1e3:.3f} ms  {n/t:.3e} q/s  {flop*n/t/1e12:.1f} TFLOP/s ({flop*n/t/1.599e15*100:.1f}% of 1599)")
