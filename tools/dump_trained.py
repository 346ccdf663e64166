"""Train each config's model for T steps through nb_train_step (the same
recipe as tests/test_gpu_depth.py) and save the fp32 parameters, so the
precision gap of the trained bf16 networks can be studied on the CPU."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import nbgen  # noqa: E402
import paper_2310_06822_b200 as nb  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
os.makedirs("gpurun_out", exist_ok=True)
for name in ["c2", "c3", "c4", "c5"]:
    cfg = nbgen.CONFIGS[name]
    m = nb.Model(nb.Desc(cfg.kind, cfg.space_dim, cfg.width, cfg.hidden_layers, tuple(cfg.head_after),
                         cfg.precision), 0)
    m.set_params(nbgen.init_params(cfg))
    g = nb.Grid(nbgen.make_grid(cfg), cfg.space_dim, 0)
    for t in range(T):
        qt = nbgen.train_batch(cfg, t, device="cuda:0")
        m.train_step(qt, g.label(cfg.kind, qt), alpha=nb.alpha(t, T))
    torch.save(m.get_params(), f"gpurun_out/trained_{name}_{T}.pt")
    print(name, "saved", flush=True)
