"""Neural bounding hierarchy evaluation time (dev tool): a binary tree of
depth D of c2-shape bf16 nets (3 -> 64 x 4 -> 1) over 2^22 points, nodes
calibrated on the scene labels (every node passes every positive), against
one c2 score of the root alone.

    python tools/hier_bench.py [depth]
"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import nbgen
import paper_2310_06822_b200 as nb

depth = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = nbgen.CONFIGS["c2"]
n = 1 << 22
q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, n, device="cuda")
y = nb.Grid(nbgen.make_grid(cfg), 3, 0).label("point", q)
parent = [-1]
for i in range(1, 2 ** (depth + 1) - 1):
    parent.append((i - 1) // 2)
models = []
for i in range(len(parent)):
    m = nb.Model(nb.Desc("point", 3, 64, 4, (), "bf16"), 0)
    m.set_params(nbgen.init_params(cfg) * (2.0 + 0.1 * i))
    m.calibrate(q, y)
    models.append(m)
for _ in range(2):
    nb.hier_score(models, parent, q, y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    c = nb.hier_score(models, parent, q, y)
e1.record()
torch.cuda.synchronize()
t = e0.elapsed_time(e1) / 5
e0.record()
for _ in range(5):
    r = models[0].score(q, y)
e1.record()
torch.cuda.synchronize()
tr = e0.elapsed_time(e1) / 5
print(f"depth {depth} ({len(parent)} nodes): {t:.3f} ms  {n / t * 1e3:.3e} q/s  "
      f"(root score alone {tr:.3f} ms); tree positives {c['tp'] + c['fp']} vs root {r['tp'] + r['fp']}, fn {c['fn']}")
