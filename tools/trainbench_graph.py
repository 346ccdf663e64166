"""Train-step timing with the step loop captured in a CUDA graph (dev tool):
the same nb_train_step calls (fixed device batches, per-step alpha baked
into the capture), replayed; vs the eager loop.

    python tools/trainbench_graph.py [config] [steps]
"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import nbgen
import paper_2310_06822_b200 as nb

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
cfg = nbgen.CONFIGS[name]
m = nb.Model(nb.Desc(cfg.kind, cfg.space_dim, cfg.width, cfg.hidden_layers, tuple(cfg.head_after), cfg.precision), 0)
m.set_params(nbgen.init_params(cfg))
g = nb.Grid(nbgen.make_grid(cfg), cfg.space_dim, 0)
qs = [nbgen.train_batch(cfg, t, 0, 1, device="cuda") for t in range(4)]
ys = [g.label(cfg.kind, q) for q in qs]
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for t in range(3):
        m.train_step(qs[t % 4], ys[t % 4], alpha=1.0)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(s):
    e0.record(s)
    for t in range(steps):
        m.train_step(qs[t % 4], ys[t % 4], alpha=nb.alpha(t, steps))
    e1.record(s)
torch.cuda.synchronize()
eager = e0.elapsed_time(e1) / steps
graph = torch.cuda.CUDAGraph()
with torch.cuda.graph(graph, stream=s):
    for t in range(steps):
        m.train_step(qs[t % 4], ys[t % 4], alpha=nb.alpha(t, steps))
torch.cuda.synchronize()
graph.replay()
torch.cuda.synchronize()
with torch.cuda.stream(s):
    e0.record(s)
    graph.replay()
    e1.record(s)
torch.cuda.synchronize()
gr = e0.elapsed_time(e1) / steps
print(f"{name} train B={cfg.train_batch}: eager {eager*1e3:.1f} us/step, graph {gr*1e3:.1f} us/step")
