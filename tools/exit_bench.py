"""Early-exit compaction timing (dev tool): a c4 model trained for `steps`
Adam steps (exit heads learn to reject empty space), calibrated to FN = 0 on
the 2^22 labelled set, then nb_score over 2^logn queries timed with CUDA
events (L2 flushed in between), compacted vs dense.

    python tools/exit_bench.py [steps] [log2 n]       NB_EXIT_CHUNK=<rows>
"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import nbgen
import paper_2310_06822_b200 as nb

if os.environ.get("NB_LIB", ""):  # measurement variant (build.py --name=...)
    nb.LIB_PATH = os.path.join(os.path.dirname(nb.LIB_PATH), f"libnb_{os.environ['NB_LIB']}.so")

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
logn = int(sys.argv[2]) if len(sys.argv) > 2 else 26
cfg = nbgen.CONFIGS["c4"]
n = 1 << logn
g = nb.Grid(nbgen.make_grid(cfg), cfg.space_dim, 0)
m = nb.Model(nb.Desc(cfg.kind, cfg.space_dim, cfg.width, cfg.hidden_layers, tuple(cfg.head_after), "bf16"), 0)
m.set_params(nbgen.init_params(cfg))
for t in range(steps):
    qt = nbgen.make_queries(cfg, nbgen.TAG_TRAIN, t << 16, 1 << 16, device="cuda")
    m.train_step(qt, g.label(cfg.kind, qt), alpha=nb.alpha(t, steps))
qc = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, 1 << 22, device="cuda")
m.calibrate(qc, g.label(cfg.kind, qc))
q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, n, device="cuda")
y = g.label(cfg.kind, q)
W = cfg.width
lay = 2 * (2 * cfg.space_dim * W)  # layer-1 flops use the record (unpadded)
per_layer = 2 * W * W
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
out = torch.zeros(9, dtype=torch.int64).pin_memory()
L = nb.lib()
for dense in (0, 1):
    L.nb_debug_set_dense_exits(dense)
    for _ in range(3):
        m.score_async(q, y, out)
    ts = []
    for it in range(8):
        flush.fill_(it)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        m.score_async(q, y, out)
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1e-3)
    t = sorted(ts)[len(ts) // 2]
    c = nb.Model.counts_dict(out)
    h = c["exit_hist"]
    s1 = (n - h[0]) / n
    s2 = (n - h[0] - h[1]) / n
    dense_flop = n * (cfg.record_floats * W * 2 + 5 * per_layer + 2 * W * 3)
    exec_flop = n * (cfg.record_floats * W * 2 + per_layer + 2 * W) + n * s1 * (2 * per_layer + 2 * W) \
        + n * s2 * (2 * per_layer + 2 * W)
    print(f"{'dense' if dense else 'compact'}: {t*1e3:.3f} ms  {n/t:.3e} q/s  exits {h} "
          f"survive {s1:.3f}/{s2:.3f}  executed {exec_flop/t/1e12:.0f} TFLOP/s "
          f"(dense-equiv {dense_flop/t/1e12:.0f})  fn {c['fn']}", flush=True)
L.nb_debug_set_dense_exits(0)
