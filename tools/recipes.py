"""BASELINE.json configs[0..4] trained to their recipes end to end, then
calibrated and scored (VERDICT r1 "BJ recipes end to end").

    python tools/recipes.py [--configs c1,c2,c3,c4,c5] [--out profiles/r2_recipes.json]
    torchrun --nproc-per-node N tools/recipes.py --configs c5    (data parallel)
    python tools/recipes.py --configs c4ray,c4box,c4plane    (NEXT-3 4D records, R48)

Per config: Xavier init (nbgen), the recipe's Adam steps of Eq. (1) through
nb_train_step (c1: 200 x 4096 slices of the 65,536 labelled points, R9; c2,
c3, c4: 5,000 x 2^16 fresh TRAIN batches, R7/R10; c5: 20,000 x 2^18 global,
split over the ranks with the NCCL gradient allreduce), FN weight ramped
alpha_t = 1 + 999 t / (T - 1) (R6), then:
  * calibration on the config's labelled evaluation set (R29) and the
    calibrated predictor's FP/FN/TP/TN there (FN = 0 by construction; the
    north star's "zero FN on every config"), c4's exit histogram;
  * the paper's uncalibrated rule sigma(z) + 1e-5 >= 0.5 (Suppl. §3.1;
    z >= logit(0.49999)) on the same set, for comparison;
  * generalisation: the calibrated predictor on a HOLDOUT set never seen in
    training or calibration (same distribution, min(N, 2^24) rows; R29 and
    P:338 "fewer than 1 FN in 100 million queries").
Labels come from the library's GPU labeller (bit-exact against the oracle,
tests P6).  Training time is device time around the step loop.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import nbgen  # noqa: E402
import paper_2310_06822_b200 as nb  # noqa: E402
from bench import ClockSampler  # noqa: E402
from paper_2310_06822_b200.dist import comm_init, shard  # noqa: E402

EPS_TAU = math.log(0.49999 / 0.50001)   # sigma(z) + 1e-5 >= 0.5  <=>  z >= logit(0.49999)


def rates(c, n):
    neg = c["fp"] + c["tn"]
    return {"fp_rate_of_negatives": c["fp"] / neg if neg else None, "fp_per_query": c["fp"] / n,
            "positives": c["tp"] + c["fn"], "negatives": neg}


def score_in_chunks(m, cfg, grid, tag, n, rank, world, dev, chunk=1 << 26):
    """Counts of the model's current predictor over rows [0, n) of stream
    `tag` (this rank's tile-aligned shard), generated and labelled on the
    device chunk by chunk; summed over the ranks by nb_score's allreduce."""
    s0, cnt = shard(n, rank, world)
    tot = None
    # every rank issues the same number of collective calls
    steps = -(-max(shard(n, r, world)[1] for r in range(world)) // chunk)
    for i in range(steps):
        a = s0 + min(cnt, i * chunk)
        b = s0 + min(cnt, (i + 1) * chunk)
        q = nbgen.make_queries(cfg, tag, a, b - a, device=dev)
        c = m.score(q, grid.label(cfg.kind, q))
        if tot is None:
            tot = c
        else:
            for k in ("tp", "fp", "fn", "tn", "nonfinite"):
                tot[k] += c[k]
            tot["exit_hist"] = [x + y for x, y in zip(tot["exit_hist"], c["exit_hist"])]
    return tot


def run(name, rank, world, local, log_every, steps=0):
    cfg = nbgen.CONFIGS[name] if name in nbgen.CONFIGS else nbgen.EXTRA_CONFIGS[name]
    if steps:
        import dataclasses

        cfg = dataclasses.replace(cfg, train_steps=steps)
    dev = f"cuda:{local}"
    m = nb.Model(nb.Desc(cfg.kind, cfg.space_dim, cfg.width, cfg.hidden_layers, tuple(cfg.head_after),
                         cfg.precision), local)
    if world > 1:
        comm_init(m)
    m.set_params(nbgen.init_params(cfg))
    grid = nb.Grid(nbgen.make_grid(cfg), cfg.space_dim, local)
    T, B = cfg.train_steps, cfg.train_batch
    # ---------------- training (the recipe) ----------------
    if name == "c1":   # R9: sequential 4096-row slices of the labelled set
        q_all = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, cfg.n_eval, device=dev)
        y_all = grid.label(cfg.kind, q_all)
    curve = []
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    gen_ms = 0.0
    t_wall = time.perf_counter()
    e0.record()
    for t in range(T):
        if name == "c1":
            b = B // world
            base = (t % (cfg.n_eval // B)) * B + rank * b
            qt, yt = q_all[base:base + b], y_all[base:base + b]
        else:
            qt = nbgen.train_batch(cfg, t, rank, world, device=dev)
            yt = grid.label(cfg.kind, qt)
        want = log_every and (t % log_every == 0 or t == T - 1)
        st = m.train_step(qt, yt, alpha=nb.alpha(t, T), n_global=B, stats=want)
        if want:
            curve.append({"step": t, "alpha": nb.alpha(t, T), "loss": st["loss"], "batch_fn_at_0": st["fn"],
                          "batch_fp_at_0": st["fp"]})
    e1.record()
    torch.cuda.synchronize()
    train_ms = e0.elapsed_time(e1)
    wall = time.perf_counter() - t_wall
    # ---------------- calibrate on the labelled evaluation set ----------------
    N = cfg.n_eval
    s0, cnt = shard(N, rank, world)
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, s0, cnt, device=dev)
    y = grid.label(cfg.kind, q)
    tau = m.calibrate(q, y).tolist()
    cal = m.score(q, y)
    m.set_thresholds([EPS_TAU] * (1 + cfg.n_heads))
    eps = m.score(q, y)
    m.set_thresholds(tau)
    del q, y
    hold_n = min(N, 1 << 24)
    hold = score_in_chunks(m, cfg, grid, nbgen.TAG_HOLDOUT, hold_n, rank, world, dev)
    out = {
        "config": name, "recipe": f"{T} Adam steps x global batch {B} (lr 1e-3, alpha 1 -> 1000 linear, beta 1)",
        "arch": f"{cfg.record_floats}->{cfg.width}x{cfg.hidden_layers}->1 {cfg.precision}"
                + (f", exit heads after {list(cfg.head_after)}" if cfg.head_after else ""),
        "ranks": world, "train_device_ms": train_ms, "train_wall_s": wall,
        "train_samples_per_s_incl_batch_generation": B * T / (train_ms * 1e-3),
        "calibration_set": {"n": N, "tau": tau, "counts": cal, **rates(cal, N)},
        "eps_rule_uncalibrated": {"rule": "sigma(z) + 1e-5 >= 0.5 (P:772) i.e. z >= logit(0.49999) on every head",
                                  "tau": EPS_TAU, "counts": eps, **rates(eps, N)},
        "holdout": {"n": hold_n, "stream": "HOLDOUT (tag 5), never trained or calibrated on", "counts": hold,
                    **rates(hold, hold_n)},
        "curve": curve,
    }
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c2,c3,c4,c5")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r2_recipes.json"))
    ap.add_argument("--log-every", type=int, default=500)
    ap.add_argument("--steps", type=int, default=0, help="override the recipe's step count (0: the recipe's)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    res = {"gpu": torch.cuda.get_device_name(local), "ranks": world, "results": []}
    with ClockSampler(local) as clk:
        for name in args.configs.split(","):
            r = run(name, rank, world, local, args.log_every, args.steps)
            res["results"].append(r)
            if rank == 0:
                print(json.dumps({k: r[k] for k in ("config", "train_device_ms", "calibration_set", "holdout")}),
                      flush=True)
    res["clocks"] = clk.summary()
    if rank == 0:
        os.makedirs(os.path.dirname(args.out), exist_ok=True)
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
