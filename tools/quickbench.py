"""Quick device-time measurement of the fused kernels (dev tool).

    python tools/quickbench.py [config] [log2 n]
    NB_LIB=<name>   use the measurement variant libnb_<name>.so (build.py --name=)
    NB_NO_FOLD=1    epilogue-bias kernels instead of bias-folded ones

Prints, per mode, the median device time of the library's own kernel events
(forward, score) and of one nb_score_async step (kernel + count finalisation,
events on the stream, L2 flushed in between like bench.py).
"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import nbgen
import paper_2310_06822_b200 as nb

if os.environ.get("NB_LIB", ""):  # measurement variant (build.py --name=...)
    nb.LIB_PATH = os.path.join(os.path.dirname(nb.LIB_PATH), f"libnb_{os.environ['NB_LIB']}.so")
if os.environ.get("NB_NO_FOLD"):
    nb.lib().nb_debug_set_no_fold(1)
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
logn = int(sys.argv[2]) if len(sys.argv) > 2 else 22
cfg = nbgen.CONFIGS[name]
n = 1 << logn
if len(sys.argv) > 3:  # explicit row count (e.g. an exact multiple of 148 CTAs x slots x 128)
    n = int(sys.argv[3])
q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, n, device="cuda")
g = nb.Grid(nbgen.make_grid(cfg), cfg.space_dim, 0)
y = g.label(cfg.kind, q)
m = nb.Model(nb.Desc(cfg.kind, cfg.space_dim, cfg.width, cfg.hidden_layers, tuple(cfg.head_after), cfg.precision), 0)
m.set_params(nbgen.init_params(cfg) * 2.5)
m.calibrate(q, y, allow_no_positives=bool(os.environ.get('NB_LIB', '')))
flop = 2 * (cfg.record_floats * cfg.width + (cfg.hidden_layers - 1) * cfg.width ** 2 + cfg.width * (1 + cfg.n_heads))
logits = torch.empty(n, 1 + cfg.n_heads, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
out = torch.zeros(9, dtype=torch.int64).pin_memory()
st = torch.cuda.current_stream().cuda_stream


def run(mode):
    if mode == "forward":
        nb.lib().nb_forward(m._h, q.data_ptr(), n, logits.data_ptr(), None, st)
    else:
        m.score_async(q, y, out)


for mode in (os.environ.get("NB_QB_MODES", "forward,score").split(",")):
    for _ in range(3):
        run(mode)
    ks, ss = [], []
    for it in range(10):
        flush.fill_(it)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        m.set_timing(True)
        m.kernel_time()
        s.record()
        run(mode)
        e.record()
        torch.cuda.synchronize()
        ks.append(m.kernel_time()[0])
        m.set_timing(False)
        ss.append(s.elapsed_time(e))
    k = sorted(ks)[len(ks) // 2] * 1e-3
    t = sorted(ss)[len(ss) // 2] * 1e-3
    print(f"{name} {mode:7s} n=2^{logn}: kernel {k*1e3:.4f} ms {flop*n/k/1e12:7.1f} TFLOP/s "
          f"({flop*n/k/1.6878e15*100:.1f}% of 1687.8) | step {t*1e3:.4f} ms {n/t:.3e} q/s")
