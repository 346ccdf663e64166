"""Timeline of CTA 0 (the pair leader) of the pipelined CTA-pair kernel
k_fwd_tc2p (dev tool; NB_TRACE build, see tools/trace_fwd.py).

Regions: 0 issuer warp 16 (0 a_done seen, 1 early K issued, 2 b_done seen,
3 rest issued); epilogue warps 0, 8, 15 (4/8 acc_a/acc_b wake, 5/9 epilogue
done, 6/10 signalled).
"""
import ctypes as C
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402

import nbgen  # noqa: E402
import paper_2310_06822_b200 as nb  # noqa: E402
import trace_fwd  # noqa: E402


def main():
    logn = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    if not os.path.exists(trace_fwd.TRACE_LIB) or "--rebuild" in sys.argv:
        trace_fwd.build_trace()
    nb.LIB_PATH = trace_fwd.TRACE_LIB
    L = nb.lib()
    L.nb_debug_set_trace.argtypes = [C.c_void_p]
    cfg = nbgen.CONFIGS["c5"]
    n = 1 << logn
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, n, device="cuda")
    g = nb.Grid(nbgen.make_grid(cfg), cfg.space_dim, 0)
    y = g.label(cfg.kind, q)
    m = nb.Model(nb.Desc("box", 3, 256, 4, (), "bf16"), 0)
    m.set_params(nbgen.init_params(cfg) * 2.0)
    m.calibrate(q, y)
    buf = torch.zeros(4 * 2000 * 2, dtype=torch.int64, device="cuda")
    m.score(q, y)
    L.nb_debug_set_trace(buf.data_ptr())
    m.score(q, y)
    L.nb_debug_set_trace(None)
    torch.cuda.synchronize()
    b = buf.view(4, 2000, 2).cpu().tolist()
    ev = []
    for r in range(4):
        for t, c in b[r]:
            if t:
                ev.append((t, r, c & 255, c >> 8))
    ev.sort()
    t0 = ev[0][0]
    names = {0: "a_done seen", 1: "early issued", 2: "b_done seen", 3: "rest issued", 4: "a wake",
             5: "a epi done", 6: "a signalled", 8: "b wake", 9: "b epi done", 10: "b signalled"}
    for t, r, typ, l in ev[:120]:
        print(f"{t - t0:8d}  r{r} L{l} {names[typ]}")
    # steady-state latencies
    lat = defaultdict(list)
    per = defaultdict(list)
    for t, r, typ, l in ev:
        per[r].append((t, typ, l))
    for r, lst in per.items():
        for (ta, a, la), (tb, bb, lb) in zip(lst, lst[1:]):
            lat[(r, a, bb)].append(tb - ta)
    for k, v in sorted(lat.items()):
        v.sort()
        print(f"r{k[0]} {names[k[1]]:>13s} -> {names[k[2]]:<13s} n={len(v):5d} median={v[len(v)//2]:6d} p90={v[int(len(v)*.9)]:6d}")
    iss = [t for t, r, typ, l in ev if r == 0 and typ == 3]
    d = sorted(b_ - a_ for a_, b_ in zip(iss, iss[1:]))
    print("stage period (rest issued -> next rest issued) median", d[len(d) // 2], "p90", d[int(len(d) * .9)])


if __name__ == "__main__":
    main()
