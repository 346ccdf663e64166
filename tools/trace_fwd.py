"""Timeline of one CTA of the fused forward kernel (dev tool).

Builds libnb_trace.so (nb_fwd_tc.cu with -DNB_TRACE) next to libnb.so, runs a
score pass of a config and prints per-event-type latency statistics:
  0 MMA thread: a_full wait satisfied      1 MMA thread: MMAs issued + committed
  2 epilogue: acc_full wait satisfied      3 epilogue: tcgen05.ld complete
  4 epilogue: next A stored, arriving      5 epilogue: encoded input stored
"""
import ctypes as C
import os
import shutil
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import nbgen  # noqa: E402
import paper_2310_06822_b200 as nb  # noqa: E402
from paper_2310_06822_b200 import build as B  # noqa: E402

TRACE_LIB = os.path.join(ROOT, "paper_2310_06822_b200", "libnb_trace.so")


def build_trace():
    import concurrent.futures as cf

    tdir = os.path.join(B.OBJ, "trace")
    os.makedirs(tdir, exist_ok=True)

    def one(item):
        src, extra = item
        obj = os.path.join(tdir, src + ".o")
        lang = ["-x", "cu"] if src.endswith(".cu") else ["-x", "c++"]
        cmd = [B.NVCC] + lang + B.ARCH + B.COMMON + extra + ["-DNB_TRACE", "-c",
                                                              os.path.join(B.CSRC, src), "-o", obj]
        subprocess.check_call(cmd, stderr=subprocess.DEVNULL)
        return obj

    with cf.ThreadPoolExecutor(max_workers=len(B.SOURCES)) as ex:
        objs = list(ex.map(one, B.SOURCES.items()))
    subprocess.check_call([B.NVCC] + B.ARCH + ["-shared", "-o", TRACE_LIB] + objs + ["-ldl"])


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    logn = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    if not os.path.exists(TRACE_LIB) or "--rebuild" in sys.argv:
        build_trace()
        if "--build-only" in sys.argv:
            return
    nb.LIB_PATH = TRACE_LIB
    L = nb.lib()
    L.nb_debug_set_trace.argtypes = [C.c_void_p]
    cfg = nbgen.CONFIGS[name]
    n = 1 << logn
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, n, device="cuda")
    g = nb.Grid(nbgen.make_grid(cfg), cfg.space_dim, 0)
    y = g.label(cfg.kind, q)
    m = nb.Model(nb.Desc(cfg.kind, cfg.space_dim, cfg.width, cfg.hidden_layers,
                         tuple(cfg.head_after), cfg.precision), 0)
    m.set_params(nbgen.init_params(cfg) * 2.0)
    m.calibrate(q, y)
    buf = torch.zeros(9 * 2000 * 2, dtype=torch.int64, device="cuda")
    m.score(q, y)
    L.nb_debug_set_trace(buf.data_ptr())
    m.score(q, y)
    L.nb_debug_set_trace(None)
    torch.cuda.synchronize()
    ev = [row for row in buf.view(-1, 2).cpu().tolist() if row[0] != 0]
    cnt = len(ev)
    import json
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(ev, open(os.path.join(ROOT, "gpurun_out", f"trace_{name}_{logn}.json"), "w"))
    ev.sort()
    t0 = ev[0][0]
    # per (slot, layer-sequence) latencies
    last = {}
    lat = defaultdict(list)
    prev_type = {(1, 2): "MMA committed -> acc ready (wake)", (2, 3): "wake -> ld done",
                 (3, 4): "ld done -> st done", (4, 0): "st done -> slot barrier passed",
                 (5, 0): "encode -> slot barrier passed", (0, 1): "MMA issue (elect) -> committed"}
    seq = defaultdict(list)
    for t, code in ev:
        typ, s, l = code & 15, (code >> 4) & 15, (code >> 8) & 15
        seq[s].append((t, typ, l))
    for s, lst in seq.items():
        for (ta, a, la), (tb, b, lb) in zip(lst, lst[1:]):
            if (a, b) in prev_type:
                lat[prev_type[(a, b)]].append(tb - ta)
    for k, v in lat.items():
        v.sort()
        print(f"{k:34s} n={len(v):5d} median={v[len(v)//2]:6d} p90={v[int(len(v)*0.9)]:6d}")
    mma = [t for t, c in ev if c & 15 == 1]
    print("span cycles", ev[-1][0] - t0, "events", cnt)
    # MMA thread idle: gaps between commit and next wait-done
    ts = [(t, c & 15) for t, c in ev if (c & 15) in (0, 1)]
    idle = [b[0] - a[0] for a, b in zip(ts, ts[1:]) if a[1] == 1 and b[1] == 0]
    idle.sort()
    print("MMA thread: commit -> next wait done median", idle[len(idle) // 2], "p90", idle[int(len(idle) * .9)])
    for row in ev[:60]:
        print(row[0] - t0, row[1] & 15, (row[1] >> 4) & 15, (row[1] >> 8) & 15)


if __name__ == "__main__":
    main()
