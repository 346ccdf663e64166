"""Device time of the score kernel for sine / positional-encoding nets (dev tool):
the BJ c2 / c3 shapes with sine activations, and the paper's PE net (Suppl.
Tab. 3, Main Fig. 11 d: 2D points, PE depth 8 -> 18 inputs, 2 -> 128 x 3 -> 1, sine).

    python tools/sinebench.py [log2 n]
"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import nbgen
import paper_2310_06822_b200 as nb

if os.environ.get("NB_LIB", ""):  # measurement variant (build.py --name=...)
    nb.LIB_PATH = os.path.join(os.path.dirname(nb.LIB_PATH), f"libnb_{os.environ['NB_LIB']}.so")

logn = int(sys.argv[1]) if len(sys.argv) > 1 else 22
n = 1 << logn
cases = [("c2", 64, 4, "relu", 0), ("c2", 64, 4, "sine", 0), ("c3", 128, 4, "relu", 0),
         ("c3", 128, 4, "sine", 0), ("c1", 128, 3, "sine", 8), ("c1", 128, 3, "relu", 8)]
if os.environ.get("NB_SINE_ONLY"):
    cases = [c for c in cases if c[3] == "sine"]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for name, W, L, act, pe in cases:
    cfg = nbgen.CONFIGS[name]
    d = nb.Desc(cfg.kind, cfg.space_dim, W, L, (), "bf16", activation=act, pe_depth=pe)
    m = nb.Model(d, 0)
    m.set_params(torch.randn(d.num_params) * 0.1)
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, n, device="cuda")
    y = nb.Grid(nbgen.make_grid(cfg), cfg.space_dim, 0).label(cfg.kind, q)
    m.calibrate(q, y)
    out = torch.zeros(9, dtype=torch.int64, device="cuda")
    for _ in range(3):
        m.score_async(q, y, out)
    ts = []
    for it in range(10):
        flush.fill_(it)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        m.score_async(q, y, out)
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1e-3)
    t = sorted(ts)[len(ts) // 2]
    din = cfg.record_floats * (1 + pe)
    flop = 2 * (din * W + (L - 1) * W * W + W)
    print(f"{name} {din}->{W}x{L} {act:4s} pe={pe}: {t*1e3:.3f} ms  {n/t:.3e} q/s  "
          f"{flop*n/t/1e12:.0f} TFLOP/s ({flop*n/t/1.6878e15*100:.1f}%)", flush=True)
