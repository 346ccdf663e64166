"""Per-CTA timeline of the two-slot fused training kernel k_train_fused2
(dev tool; libnb_ftrace.so = nb_train_fused.cu + nb_fwd_tc.cu with -DNB_TRACE).

    python tools/trace_fused.py [config] [--build-only]

Events (globaltimer ns): 0 entry, 1 weights resident, 10+s / 20+s / 30+s
slot s tile start / loss done / tile done, 2 all tiles done, 3 partials written.
"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2310_06822_b200 import build as B  # noqa: E402

LIB = os.path.join(ROOT, "paper_2310_06822_b200", "libnb_ftrace.so")


def main():
    if "--build-only" in sys.argv or not os.path.exists(LIB):
        B.build(defines=("NB_TRACE",), name="ftrace", only=("nb_train_fused.cu", "nb_fwd_tc.cu"))
        if "--build-only" in sys.argv:
            return
    import torch

    import nbgen
    import paper_2310_06822_b200 as nb
    nb.LIB_PATH = LIB
    lib = nb.lib()
    lib.nb_debug_set_trace.argtypes = [C.c_void_p]
    name = next((a for a in sys.argv[1:] if not a.startswith("-")), "c2")
    cfg = nbgen.CONFIGS[name]
    m = nb.Model(nb.Desc(cfg.kind, cfg.space_dim, cfg.width, cfg.hidden_layers, tuple(cfg.head_after),
                         cfg.precision), 0)
    m.set_params(nbgen.init_params(cfg))
    g = nb.Grid(nbgen.make_grid(cfg), cfg.space_dim, 0)
    q = nbgen.train_batch(cfg, 0, 0, 1, device="cuda")
    y = g.label(cfg.kind, q)
    buf = torch.zeros(148 * 64 * 2 + 3 * 512 * 2, dtype=torch.int64, device="cuda")
    for _ in range(5):
        m.train_step(q, y, alpha=1.0)
    lib.nb_debug_set_trace(C.c_void_p(buf.data_ptr()))
    torch.cuda.synchronize()
    m.train_step(q, y, alpha=1.0)
    torch.cuda.synchronize()
    lib.nb_debug_set_trace(C.c_void_p(0))
    fine = buf[148 * 64 * 2:].view(3, 512, 2).cpu().numpy()
    t = buf[:148 * 64 * 2].view(148, 64, 2).cpu().numpy()
    t0 = t[:, 0, 0][t[:, 0, 0] > 0].min()
    ev = lambda c, i: (t[c, i, 0] - t0) / 1e3 if t[c, i, 0] else float("nan")
    rows = []
    for c in range(148):
        if not t[c, 0, 0]:
            continue
        r = {"cta": c, "entry": ev(c, 0), "setup": ev(c, 1), "tiles_done": ev(c, 2), "end": ev(c, 3)}
        for s in range(2):
            tiles = []
            for i in range(16 + 24 * s, 40 + 24 * s):
                if t[c, i, 0]:
                    tiles.append((int(t[c, i, 1]), (t[c, i, 0] - t0) / 1e3))
            r[f"slot{s}"] = tiles
        rows.append(r)
    ent = np.array([r["entry"] for r in rows])
    st = np.array([r["setup"] - r["entry"] for r in rows])
    td = np.array([r["tiles_done"] for r in rows])
    en = np.array([r["end"] for r in rows])
    print(f"CTAs {len(rows)}  entry spread {ent.min():.2f}..{ent.max():.2f} us  setup {st.mean():.2f} us (max {st.max():.2f})")
    print(f"tiles done {td.min():.2f}..{td.max():.2f} us  partials {np.nanmean(en - td):.2f} us  end max {np.nanmax(en):.2f} us")
    for c in (0, 1, 70, 100, 147):
        r = next((x for x in rows if x["cta"] == c), None)
        if r is None:
            continue
        print(f"cta {c}: entry {r['entry']:.2f} setup {r['setup']:.2f} tiles_done {r['tiles_done']:.2f} end {r['end']:.2f}")
        for s in range(2):
            print("   slot", s, " ".join(f"{code}@{x:.2f}" for code, x in r[f"slot{s}"]))
    fine_timeline(fine)


def fine_timeline(fine):
    """CTA 0: issuer (code 100 s + step: ready seen) and slot leads (1 acc wait
    start, 2 acc seen, 4 ld done, 3 arriving), cycles from the first event."""
    ev = []
    for r in range(3):
        for i in range(512):
            if fine[r, i, 0]:
                ev.append((int(fine[r, i, 0]), r, int(fine[r, i, 1])))
    ev.sort()
    c0 = ev[0][0]
    names = {1: "wait", 2: "acc", 4: "ld", 3: "arrive"}
    for c, r, code in ev[:400]:
        who = "issuer" if r == 0 else f"slot{r - 1}"
        what = f"ready s{code // 100} step {code % 100}" if r == 0 else names.get(code, code)
        print(f"{c - c0:8d} {who:7s} {what}")


if __name__ == "__main__":
    main()
