"""World-size-2 CPU (gloo) tests of the data-parallel host logic:
shard ranges, the unique-id broadcast, and that the per-shard reductions the
library performs with NCCL (counts: sum, calibration keys: min, gradient: sum)
reproduce the single-process results (oracle compute on each shard)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import nbgen
import oracle
from paper_2310_06822_b200.dist import float_key, key_float, shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = nbgen.CONFIGS["c2"]
        n = 10007
        a = oracle.arch_of(cfg)
        th = (nbgen.init_params(cfg) * 2.5).double().numpy()
        grid = nbgen.make_grid(cfg).numpy()
        s0, cnt = shard(n, rank, world)
        q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, s0, cnt).numpy()
        y = oracle.label(grid, 3, "point", q)
        # unique-id broadcast (what comm_init does before nb_comm_init)
        uid = [os.urandom(128) if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        # C2: tau = min over ranks of the local min positive logit (as keys)
        z = oracle.forward(a, th, q)
        tau_loc, _ = oracle.calibrate(z, y)
        k = torch.tensor(float_key(np.float32(tau_loc[0])).astype(np.int64).reshape(1))
        dist.all_reduce(k, op=dist.ReduceOp.MIN)
        tau = float(key_float(np.array([k.item()], np.uint32))[0])
        # C1: counts summed over ranks
        c = oracle.score(z.astype(np.float32).astype(np.float64), y, [tau])
        ct = torch.tensor([c["tp"], c["fp"], c["fn"], c["tn"]], dtype=torch.int64)
        dist.all_reduce(ct)
        # C3: gradient of the global-batch loss = sum of shard gradients (n_global normalisation)
        _, g, _ = oracle.loss_grad(a, th, q, y, 17.0, 1.0, n_global=n)
        gt = torch.from_numpy(g)
        dist.all_reduce(gt)
        if rank == 0:
            out.put((uid[0], tau, ct.tolist(), gt.numpy()))
        else:
            out.put((uid[0], None, None, None))
    finally:
        dist.destroy_process_group()


def test_shard_partition():
    for n in [0, 1, 7, 10007, 1 << 22]:
        for world in [1, 2, 3, 8]:
            parts = [shard(n, r, world) for r in range(world)]
            assert parts[0][0] == 0
            assert sum(c for _, c in parts) == n
            for (s, c), (s2, _) in zip(parts, parts[1:]):
                assert s + c == s2
            assert all(s % 128 == 0 or c == 0 for s, c in parts)   # tile-aligned starts
            tiles = [-(-c // 128) for _, c in parts]
            assert max(tiles) - min(tiles) <= 1                       # balanced in tiles


def test_float_key_order_preserving():
    x = np.array([-np.inf, -3.5, -1e-30, -0.0, 0.0, 1e-30, 2.0, np.inf], np.float32)
    k = float_key(x)
    assert np.all(np.diff(k.astype(np.int64)) >= 0)
    assert np.array_equal(key_float(k).view(np.uint32), x.view(np.uint32))


def test_world2_reductions_equal_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    uids = {r[0] for r in res}
    assert len(uids) == 1  # every rank received rank 0's id
    tau, counts, grad = next((r[1], r[2], r[3]) for r in res if r[1] is not None)
    # single process on the whole set
    cfg = nbgen.CONFIGS["c2"]
    n = 10007
    a = oracle.arch_of(cfg)
    th = (nbgen.init_params(cfg) * 2.5).double().numpy()
    qq = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, n).numpy()
    y = oracle.label(nbgen.make_grid(cfg).numpy(), 3, "point", qq)
    z = oracle.forward(a, th, qq)
    t1, _ = oracle.calibrate(z, y)
    assert tau == np.float32(t1[0])
    c1 = oracle.score(z.astype(np.float32).astype(np.float64), y, [tau])
    assert counts == [c1["tp"], c1["fp"], c1["fn"], c1["tn"]] and c1["fn"] == 0
    _, g1, _ = oracle.loss_grad(a, th, qq, y, 17.0, 1.0)
    assert np.allclose(grad, g1, rtol=1e-10, atol=1e-15)
