"""bench.py — the driver's benchmark contract for the Neural Bounding hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step is one pass of the fused hot path (encode -> MLP on tcgen05 -> classify
with the calibrated threshold -> FP/FN/TP/TN counts -> NCCL allreduce of the
counts across ranks) over one batch of the workload BASELINE.json's metric
("bounding queries/s (1/2/4/8 B200)") is quoted on: configs[4] ("c5": 3D box
bounding, 6 -> 256x4 -> 1 bf16, "2^28 box queries sharded over 1/2/4/8
GPUs").  Inputs are seeded synthetic (nbgen), labels come from the library's
GPU labeller, the model is trained through nb_train_step and calibrated with
nb_calibrate; the timed region is nb_score_async (kernel + count allreduce +
the step's count readback into pinned memory).

Strong scaling (c5): the 2^28 queries of a step are split into tile-aligned
contiguous shards (dist.shard), one per rank; value = 2^28 x steps / the
max-over-ranks device time.  --config c2|c3|c4 time the other BASELINE
configs (weak scaling: each rank its own full batch).  --gpus N without
torchrun re-launches this script under torch.distributed.run with N ranks.
L2 (126 MB) is flushed by writing a 256 MiB buffer between timed steps,
outside the timed events.

--impl reference times the oracle (oracle/, plain C fp64) on the host cores on
a bounded sample of the same workload; under torchrun only rank
0 runs it.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG = "c5"  # --config: c5 (default: the metric's "1/2/4/8 B200" workload, BASELINE.json configs[4]) or c2..c4
# Queries per step (BASELINE.json): c2 2^22, c3 2^24, c4 2^26 per rank (weak
# scaling); c5 2^28 in total, sharded over the ranks (strong scaling, BJ.c5).
N_STEP = {"c2": 1 << 22, "c3": 1 << 24, "c4": 1 << 26, "c5": 1 << 28}
STRONG = {"c5"}
WORKLOAD = {
    "c2": "BASELINE.json configs[1], 3D point bounding, 3->64x4->1 ReLU bf16 (fp32 accumulate), "
          "2^22 uniform points per rank per step",
    "c3": "BASELINE.json configs[2], 3D ray bounding, 6->128x4->1 ReLU bf16, 2^24 rays per rank per step",
    "c4": "BASELINE.json configs[3], 4D animated point bounding, 4->128x6->1 ReLU bf16 with exit heads "
          "after hidden 2 and 4, 2^26 queries per rank per step",
    "c5": "BASELINE.json configs[4], 3D box bounding, 6->256x4->1 ReLU bf16 on CTA pairs, 2^28 boxes "
          "per step sharded over the ranks",
}
KERNEL = {"c2": "k_fwd_tc<64,4,0,0,kScore,d0=3,BF>", "c3": "k_fwd_tc<128,4,0,0,kScore,d0=6,BF>",
          "c4": "k_score_exit<2,{records,image,image},{head1,head2,output}> (early-exit compaction, "
                "3 segment kernels per 2^24-row chunk)",
          "c5": "k_fwd_tc2p<4,kScore,d0=6> (pipelined CTA pairs)"}
# launched by torch.distributed.run (WORLD_SIZE set): process group + the
# model's NCCL communicator at every world size, N = 1 included (the same
# data-parallel path, a one-rank allreduce per call)
DIST = "WORLD_SIZE" in os.environ
METRIC = "bounding queries/s"
UNIT = "queries/s"
# bounded oracle samples (about 10 s of host work per step at 16 cores)
CPU_SAMPLE = {"c2": 1 << 23, "c3": 1 << 21, "c4": 1 << 21, "c5": 1 << 20}
REF_SAMPLE = {"c2": 1 << 20, "c3": 1 << 18, "c4": 1 << 18, "c5": 1 << 17}


def flop_per_query(cfg) -> int:
    """Algorithmic flops of one forward: 2 * MACs of all layers
    + output head (+ exit heads), unpadded."""
    macs = cfg.record_floats * cfg.width + (cfg.hidden_layers - 1) * cfg.width ** 2
    macs += cfg.width * (1 + cfg.n_heads)
    return 2 * macs


def executed_flop_per_query(cfg, hist, n) -> float:
    """Algorithmic flops per query actually computed with early exits (c4):
    layers 1..h1 and head 1 for every row, layers h1+1..h2 and head 2 for the
    rows that passed head 1, the rest and the output head for rows that passed
    both."""
    W = cfg.width
    h1, h2 = cfg.head_after
    s1 = (n - hist[0]) / n
    s2 = (n - hist[0] - hist[1]) / n
    f0 = cfg.record_floats * W + (h1 - 1) * W * W + W
    f1 = (h2 - h1) * W * W + W
    f2 = (cfg.hidden_layers - h2) * W * W + W
    return 2 * (f0 + s1 * f1 + s2 * f2)


def train_model(nb, nbgen, m, grid, cfg, steps, rank, world):
    """The bench scores a trained bounding model (c4's exit heads only skip
    work once trained): `steps` Adam steps of Eq. (1) through nb_train_step
    on fresh TRAIN batches (the config's global batch split over the ranks,
    gradient allreduce under a communicator, alpha ramp 1 -> 1000), then
    calibration."""
    dev = f"cuda:{m.device}"
    B = cfg.train_batch
    for t in range(steps):
        qt = nbgen.train_batch(cfg, t, rank, world, device=dev)
        m.train_step(qt, grid.label(cfg.kind, qt), alpha=nb.alpha(t, steps), n_global=B)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("bf16_tflops", 1590.0), "measured (MEASURED_PEAKS.json bf16_tflops, burst)"
    return 1590.0, "fallback (B200_PROFILING.md)"


def load_sustained_peak():
    """the driver's sustained bf16 figure (cuBLAS back to back for 4 s): context
    for a kernel timed over seconds under the board power cap; the line's
    `frac` stays against the burst peak (the conservative denominator)."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        return json.load(open(p)).get("bf16_tflops_sustained")
    return None


def load_traffic():
    """dram bytes per launch of the score kernel from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(p):
        d = json.load(open(p))
        k = d.get(CONFIG, {}).get("score_kernel", {})  # (only for the captured config)
        if "dram_bytes_per_launch" in k:
            return k["dram_bytes_per_launch"], k.get("tensor_pipe_pct")
    return None, None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        try:  # NVML: microsecond queries, sampled every 2 ms
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            get_r = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
            bits = (0x8, 0x40, 0x20, 0x4)  # hw_slowdown, hw_thermal, sw_thermal, sw_power_cap
            while not self._stop.is_set():
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                r = get_r(h)
                self.samples.append([str(sm), str(mx)] +
                                    ["Active" if r & b else "Not Active" for b in bits])
                self._stop.wait(0.002)
            return
        except Exception:
            pass
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                parts = [x.strip() for x in out.stdout.strip().split(",")]
                if len(parts) == 6:
                    self.samples.append(parts)
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = sorted(float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit())
        mx = max(float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i] == "Active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.samples)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def run_reference(args):
    """Oracle (plain C, fp64) on host cores: forward + calibrated score."""
    import torch

    import nbgen
    import oracle

    rank, world, _ = dist_env()
    if rank != 0:
        return
    cfg = nbgen.CONFIGS[CONFIG]
    oracle.build()
    a = oracle.arch_of(cfg)
    grid = nbgen.make_grid(cfg).numpy()
    th = (nbgen.init_params(cfg) * 2.5).double().numpy()
    n = args.ref_sample or REF_SAMPLE[CONFIG]
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, n).numpy()
    frames = grid.shape[0] if cfg.space_dim == 4 else 1
    y = oracle.label(grid, cfg.space_dim, cfg.kind, q, frames=frames)
    z = oracle.forward(a, th, q)  # warm, and the calibration pass
    tau, _ = oracle.calibrate(z, y)
    for _ in range(args.warmup if args.warmup < 2 else 1):
        oracle.score(oracle.forward(a, th, q[:4096]), y[:4096], tau)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        c = oracle.score(oracle.forward(a, th, q), y, tau)
        times.append(time.perf_counter() - t0)
    t = sum(times) / len(times)
    v = n / t
    cores = oracle.num_threads()
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "strong" if CONFIG in STRONG else "weak", "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"{CONFIG}: {WORKLOAD[CONFIG]}; oracle sample of {n} queries per step",
                   "global_batch": n},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu": cpu_model(),
                         "precision": "fp64",
                         "sample": f"{n} {CONFIG} EVAL queries, fp64 forward + calibrated score"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0, "counts_sample": {k: c[k] for k in ("tp", "fp", "fn", "tn")},
    }
    print(json.dumps(line), flush=True)


def cpu_model() -> str:
    """The host CPU model (BASELINE.md §3 asks for it beside the core count)."""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def cpu_baseline_sample(n=1 << 18):
    """The oracle as it stands on this host's cores (bounded sample)."""
    import nbgen
    import oracle

    cfg = nbgen.CONFIGS[CONFIG]
    oracle.build()
    a = oracle.arch_of(cfg)
    th = (nbgen.init_params(cfg) * 2.5).double().numpy()
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, n).numpy()
    grid = nbgen.make_grid(cfg).numpy()
    frames = grid.shape[0] if cfg.space_dim == 4 else 1
    y = oracle.label(grid, cfg.space_dim, cfg.kind, q, frames=frames)
    t0 = time.perf_counter()
    z = oracle.forward(a, th, q)
    tau, _ = oracle.calibrate(z, y)
    oracle.score(z, y, tau)
    t = time.perf_counter() - t0
    return {"value": n / t, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle", "cpu": cpu_model(),
            "precision": "fp64",
            "sample": f"{n} {CONFIG} EVAL queries: fp64 forward + calibrate + score ({t:.1f} s)"}


def run_ours(args):
    import torch
    import torch.distributed as dist

    import nbgen
    import paper_2310_06822_b200 as nb

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if DIST:
        dist.init_process_group("nccl", device_id=dev)
    cfg = nbgen.CONFIGS[CONFIG]
    desc = nb.Desc(cfg.kind, cfg.space_dim, cfg.width, cfg.hidden_layers, tuple(cfg.head_after),
                   cfg.precision)
    m = nb.Model(desc, local)
    if DIST:
        from paper_2310_06822_b200.dist import comm_init

        comm_init(m)
    from paper_2310_06822_b200.dist import shard

    strong = CONFIG in STRONG
    if strong:   # the step's 2^28 queries, tile-aligned contiguous shards
        s0, n = shard(N_STEP[CONFIG], rank, world)
    else:        # weak scaling: every rank its own full batch
        s0, n = rank * N_STEP[CONFIG], N_STEP[CONFIG]
    grid = nb.Grid(nbgen.make_grid(cfg), cfg.space_dim, local)
    m.set_params(nbgen.init_params(cfg))
    if args.model_train_steps > 0:
        train_model(nb, nbgen, m, grid, cfg, args.model_train_steps, rank, world)
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, s0, n, device=dev)
    y = grid.label(cfg.kind, q)
    tau = m.calibrate(q, y)                       # global tau (allreduce min across ranks)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > the 126 MB L2
    stream = torch.cuda.current_stream(dev)

    # one step = nb_score_async: fused encode/MLP/classify/count kernel, NCCL
    # allreduce of the counts (N > 1), async copy of the step's counts into its
    # own pinned host row; the host synchronises once after the timed loop.
    out = torch.zeros(max(args.steps, args.warmup), 9, dtype=torch.int64).pin_memory()

    def step(i):
        m.score_async(q, y, out[i])

    c = m.score(q, y)
    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    assert all(m.counts_dict(out[i]) == c for i in range(args.warmup)), (c, out)
    assert c["fn"] == 0, c
    # ---------------- timed region (device time, per-step events) ----------------
    m.set_timing(True)
    m.kernel_time()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    if DIST:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.fill_(i & 0xFF)                 # evict the inputs from L2 (untimed)
            evs[i][0].record(stream)
            step(i)
            evs[i][1].record(stream)
        torch.cuda.synchronize()
    assert all(m.counts_dict(out[i]) == c for i in range(args.steps)), "per-step counts differ"
    if DIST:
        dist.barrier()
    kernel_ms, launches = m.kernel_time()
    m.set_timing(False)
    dev_ms = sum(a.elapsed_time(b) for a, b in evs)
    t = torch.tensor([dev_ms, kernel_ms], dtype=torch.float64, device=dev)
    if DIST:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dev_ms, kernel_ms = t.tolist()
    n_total = N_STEP[CONFIG] if strong else n * world
    total_q = n_total * args.steps
    value = total_q / (dev_ms * 1e-3)
    # ---------------- roofline of the dominant kernel ----------------
    fq = flop_per_query(cfg)
    peak, peak_src = load_peaks()
    calls = args.steps
    per_launch_ms = kernel_ms / max(1, calls)
    exit_info = None
    if cfg.n_heads > 0:
        fq_exec = executed_flop_per_query(cfg, c["exit_hist"], n_total)
        achieved = fq_exec * n / (per_launch_ms * 1e-3) / 1e12
        # the dense kernel (every head on every row) on the same model, same protocol
        nb.lib().nb_debug_set_dense_exits(1)
        for i in range(3):
            step(i)
        torch.cuda.synchronize()
        dts = []
        for i in range(min(args.steps, 10)):
            flush.fill_(i & 0xFF)
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            step(i)
            a1.record(stream)
            torch.cuda.synchronize()
            dts.append(a0.elapsed_time(a1))
        nb.lib().nb_debug_set_dense_exits(0)
        assert m.counts_dict(out[0]) == c
        dense_ms = sorted(dts)[len(dts) // 2]
        # the record hand-off between the segments (8x less DRAM, recomputes)
        nb.lib().nb_debug_set_exit_records(1)
        for i in range(3):
            step(i)
        torch.cuda.synchronize()
        rts = []
        for i in range(min(args.steps, 10)):
            flush.fill_(i & 0xFF)
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            step(i)
            a1.record(stream)
            torch.cuda.synchronize()
            rts.append(a0.elapsed_time(a1))
        nb.lib().nb_debug_set_exit_records(0)
        assert m.counts_dict(out[0]) == c
        rec_ms = sorted(rts)[len(rts) // 2]
        exit_info = {"exit_hist": c["exit_hist"], "bins": "exit@1, exit@2, final-negative, final-positive",
                     "survive_head1": (n_total - c["exit_hist"][0]) / n_total,
                     "survive_head2": (n_total - c["exit_hist"][0] - c["exit_hist"][1]) / n_total,
                     "executed_flop_per_query": fq_exec, "dense_flop_per_query": fq,
                     "dense_kernel_q_per_s": n_total / (dense_ms * 1e-3),
                     "dense_kernel_ms_per_step": dense_ms,
                     "records_handoff_q_per_s": n_total / (rec_ms * 1e-3),
                     "records_handoff_ms_per_step": rec_ms,
                     "model": f"trained {args.model_train_steps} Adam steps (Eq. 1, alpha 1->1000) "
                              "from Xavier init, calibrated to FN = 0 on the step's queries"}
    else:
        achieved = fq * n / (per_launch_ms * 1e-3) / 1e12
    traffic, tensor_pct = load_traffic()
    # ---------------- end to end: host buffers through the C ABI ----------------
    q_h = q.cpu().pin_memory()
    y_h = y.cpu().pin_memory()
    for _ in range(2):
        m.score_host(q_h, y_h)
    if DIST:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(args.steps):
        ce = m.score_host(q_h, y_h)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if DIST:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_value = total_q / (e2e_ms.item() * 1e-3)
    assert ce == c, (ce, c)
    # ---------------- train samples/s (BASELINE.json metric part 2) ----------------
    train = None
    if args.train_steps > 0:
        train = train_rate(nb, nbgen, cfg, local, rank, world, args.train_steps)
    if rank == 0:
        clocks = clk.summary()
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic",
            "config": {"workload": f"{CONFIG}: {WORKLOAD[CONFIG]}, fused forward+calibrated score+counts",
                       "global_batch": n_total, "per_rank_batch": n,
                       "model": f"Xavier init + {args.model_train_steps} Adam steps of Eq. (1) "
                                f"(batch {cfg.train_batch}, alpha 1->1000) via nb_train_step, then nb_calibrate",
                       "parallelism": f"dp{world} (query shards, NCCL allreduce of counts)",
                       "l2": "flushed between timed steps (256 MiB write, untimed)"},
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "kernel": KERNEL[CONFIG],
                         "flop_per_query": exit_info["executed_flop_per_query"] if exit_info else fq,
                         "kernel_ms_per_launch": per_launch_ms,
                         "ncu_tensor_pipe_pct": tensor_pct,
                         "peak_sustained": load_sustained_peak(),
                         "frac_vs_sustained": (achieved / load_sustained_peak()) if load_sustained_peak() else None},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": n * (4 * cfg.record_floats + 1),
                    "d2h_bytes_per_step": 9 * 8, "api": "nb_score_host (pinned host q/y)",
                    "bytes": "per rank"},
            "gpu_launches": launches,
            "clocks": clocks,
            "counts": {k: c[k] for k in ("tp", "fp", "fn", "tn")},
            "tau": float(tau[0]),
        }
        if train is not None:
            line["train"] = train
        if exit_info is not None:
            line["early_exit"] = exit_info
        if not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline_sample(args.cpu_sample or CPU_SAMPLE[CONFIG])
        print(json.dumps(line), flush=True)
    if DIST:
        dist.barrier()
        dist.destroy_process_group()


def train_rate(nb, nbgen, cfg, local, rank, world, steps):
    """Train samples/s (BASELINE.json metric part 2) of the bench config: one
    step = bf16 forward (train mode) + Eq. (1) gradient + backward + dW GEMMs
    + (NCCL gradient allreduce) + Adam + bf16 re-pack, global batch split
    over the ranks; `steps` distinct fresh batches pre-generated and labelled
    on the device.  Measured two ways through the C ABI: a Python loop of
    nb_train_step calls (the reported value) and nb_train_steps (the step
    loop in one call, captured into a CUDA graph per call; three back-to-back
    calls so each capture overlaps the previous call's execution)."""
    import torch
    import torch.distributed as dist

    desc = nb.Desc(cfg.kind, cfg.space_dim, cfg.width, cfg.hidden_layers, tuple(cfg.head_after),
                   cfg.precision)
    m = nb.Model(desc, local)
    if DIST:
        from paper_2310_06822_b200.dist import comm_init

        comm_init(m)
    m.set_params(nbgen.init_params(cfg))
    g = nb.Grid(nbgen.make_grid(cfg), cfg.space_dim, local)
    B = cfg.train_batch
    b = B // world
    dev = f"cuda:{local}"
    q_all = torch.cat([nbgen.train_batch(cfg, t, rank, world, device=dev) for t in range(steps)])
    y_all = g.label(cfg.kind, q_all)
    m.train_steps(q_all[:3 * b], y_all[:3 * b], 3, 1.0, 1.0, n_global=B)   # warm-up (scratch, capture)
    for t in range(3):
        m.train_step(q_all[t * b:(t + 1) * b], y_all[t * b:(t + 1) * b], alpha=1.0, n_global=B)

    def timed(fn):
        if DIST:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if DIST:
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        return ms.item()

    def graph_loop():
        for _ in range(3):
            m.train_steps(q_all, y_all, steps, 1.0, 1000.0, n_global=B)

    def eager_loop():
        for t in range(steps):
            m.train_step(q_all[t * b:(t + 1) * b], y_all[t * b:(t + 1) * b], alpha=nb.alpha(t, steps), n_global=B)

    ms_graph = timed(graph_loop) / 3
    ms_eager = timed(eager_loop)
    flop = 3 * flop_per_query(cfg)  # forward + delta back-propagation + dW (algorithmic)
    return {"metric": "train samples/s", "value": B * steps / (ms_eager * 1e-3), "unit": "samples/s",
            "config": f"{CONFIG} bf16 {cfg.record_floats}->{cfg.width}x{cfg.hidden_layers}->1, global batch {B}, "
                      "Adam lr 1e-3, alpha ramp 1 -> 1000",
            "api": "nb_train_step per step (Python loop)",
            "steps": steps, "ms_per_step": ms_eager / steps,
            "tflops_algorithmic": flop * B * steps / (ms_eager * 1e-3) / 1e12,
            "graph": {"api": "nb_train_steps (the call captures its step loop in a CUDA graph, launched once; "
                             "the capture is host time inside the call)",
                      "value": B * steps / (ms_graph * 1e-3), "ms_per_step": ms_graph / steps}}


def free_port() -> int:
    import socket

    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    return port


def spawn(args) -> int:
    """--gpus N without torchrun: re-launch this script with N ranks under
    torch.distributed.run (the driver's own launch line), one rank per GPU."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, cwd=ROOT)


def run_dry(args):
    """CPU rehearsal of the multi-rank launch (no GPU work): every rank joins a
    gloo process group, computes its shard of the step, and rank 0 prints the
    world it saw (tests/test_bench_contract.py)."""
    import torch
    import torch.distributed as dist

    from paper_2310_06822_b200.dist import shard

    rank, world, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    strong = CONFIG in STRONG
    part = shard(N_STEP[CONFIG], rank, world) if strong else (rank * N_STEP[CONFIG], N_STEP[CONFIG])
    t = torch.tensor([rank, world, part[0], part[1]], dtype=torch.int64)
    parts = [torch.zeros_like(t) for _ in range(world)]
    if world > 1:
        dist.all_gather(parts, t)
    else:
        parts = [t]
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "ranks": [int(p[0]) for p in parts],
                          "shards": [[int(p[2]), int(p[3])] for p in parts], "config": CONFIG,
                          "scaling": "strong" if strong else "weak"}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c5", choices=["c2", "c3", "c4", "c5"])
    ap.add_argument("--ref-sample", type=int, default=0, help="oracle rows per reference step (0: per config)")
    ap.add_argument("--cpu-sample", type=int, default=0, help="oracle rows of cpu_baseline (0: per config)")
    ap.add_argument("--train-steps", type=int, default=100)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--model-train-steps", type=int, default=2000,
                    help="Adam steps on the bench model before calibration (c4: exit heads reject empty space)")
    ap.add_argument("--dry-run", action="store_true", help="CPU launch rehearsal (no GPU work)")
    args = ap.parse_args()
    global CONFIG
    CONFIG = args.config
    if args.warmup < 3:
        args.warmup = 3
    launched = "WORLD_SIZE" in os.environ
    if not launched and args.gpus > 1 and args.impl == "ours":
        sys.exit(spawn(args))
    if launched and args.impl == "ours" and int(os.environ["WORLD_SIZE"]) != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={os.environ['WORLD_SIZE']}")
    if args.dry_run:
        run_dry(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
