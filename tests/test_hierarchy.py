"""Neural bounding hierarchies (§3.2, DESIGN.md
R45).  The oracle's combination is pinned against an independent recursive
traversal on random pass tables and against closed-form special cases; the
GPU evaluation (pruned: gather -> node kernel -> compaction) is compared with
the oracle on a three-node tree over the c1 scene."""
import numpy as np
import pytest
import torch

import nbgen
import oracle


def dfs(parent, passes, r):
    """Independent formulation: depth-first search from the root."""
    children = {}
    for i, p in enumerate(parent):
        children.setdefault(p, []).append(i)

    def visit(i):
        if not passes[i][r]:
            return False
        kids = children.get(i, [])
        return True if not kids else any(visit(c) for c in kids)

    return visit(0)


@pytest.mark.parametrize("seed", range(5))
def test_combine_equals_recursive_traversal(seed):
    rng = np.random.default_rng(seed)
    N = int(rng.integers(1, 9))
    parent = [-1] + [int(rng.integers(0, i)) for i in range(1, N)]
    passes = rng.random((N, 300)) < rng.uniform(0.3, 0.9)
    got = oracle.hier_combine(parent, passes)
    want = np.array([dfs(parent, passes, r) for r in range(300)])
    assert np.array_equal(got, want)


def test_combine_special_cases():
    rng = np.random.default_rng(9)
    leaves = rng.random((3, 100)) < 0.4
    # a single node is its own predictor
    assert np.array_equal(oracle.hier_combine([-1], leaves[:1]), leaves[0])
    # inner nodes that always pass: the OR of the leaves
    parent = [-1, 0, 0, 1, 1, 2]
    passes = np.concatenate([np.ones((3, 100), bool), leaves], 0)
    assert np.array_equal(oracle.hier_combine(parent, passes), leaves.any(0))
    # a root that rejects everything prunes the whole tree
    passes[0] = False
    assert not oracle.hier_combine(parent, passes).any()


@pytest.mark.gpu
def test_gpu_hierarchy_matches_oracle_and_is_conservative():
    import paper_2310_06822_b200 as nb
    from gpu_helpers import BAND, grid_of
    cfg = nbgen.CONFIGS["c1"]
    grid = grid_of(cfg)
    R = grid.shape[0]
    left = grid.copy(); left[R // 2:] = 0
    right = grid.copy(); right[:R // 2] = 0
    n = (1 << 16) + 7
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, n)
    ys = [oracle.label(g_, 2, "point", q.numpy()) for g_ in (grid, left, right)]
    qd = q.cuda()
    a = oracle.make_arch(2, 64, 3)
    models, thetas, taus = [], [], []
    for i in range(3):
        th = torch.from_numpy(np.random.default_rng(i).normal(size=oracle.num_params(a)) * 0.25).float()
        m = nb.Model(nb.Desc("point", 2, 64, 3, (), "bf16"), 0)
        m.set_params(th)
        taus.append(m.calibrate(qd, torch.from_numpy(ys[i]).cuda()).double().numpy())
        models.append(m)
        thetas.append(th.double().numpy())
    parent = [-1, 0, 0]
    c = nb.hier_score(models, parent, qd, torch.from_numpy(ys[0]).cuda())
    assert c["fn"] == 0 and c["tp"] == int(ys[0].sum())          # conservative nodes -> conservative tree
    assert c["tp"] + c["fp"] + c["fn"] + c["tn"] == n
    # against the oracle's definition on the bf16-emulated logits, away from every threshold
    ze = [oracle.forward(a, th, q.numpy(), oracle.BF16_EMU)[:, 0] for th in thetas]
    zg = [m.forward(qd).cpu().double().numpy()[:, 0] for m in models]
    keep = np.ones(n, bool)
    for i in range(3):
        keep &= (np.abs(ze[i] - taus[i][0]) >= BAND) & (np.abs(zg[i] - taus[i][0]) >= BAND)
    assert keep.mean() > 0.95
    pred = oracle.hier_combine(parent, [z >= t[0] for z, t in zip(ze, taus)])
    sub = nb.hier_score(models, parent, qd[torch.from_numpy(keep).cuda()],
                        torch.from_numpy(ys[0][keep]).cuda())
    y = ys[0][keep].astype(bool)
    p = pred[keep]
    assert (sub["tp"], sub["fp"], sub["fn"], sub["tn"]) == (int((p & y).sum()), int((p & ~y).sum()),
                                                            int((~p & y).sum()), int((~p & ~y).sum()))
    # the hierarchy prunes: it never predicts more than the root alone
    assert c["tp"] + c["fp"] <= models[0].score(qd, torch.from_numpy(ys[0]).cuda())["tp"] + \
        models[0].score(qd, torch.from_numpy(ys[0]).cuda())["fp"]


@pytest.mark.gpu
def test_gpu_hierarchy_argument_checks_and_fp32_nodes():
    """Malformed trees are rejected; fp32 (CUDA-core) node models take the
    same path (forward -> compaction) and agree with the oracle exactly."""
    import paper_2310_06822_b200 as nb
    from gpu_helpers import grid_of
    cfg = nbgen.CONFIGS["c1"]
    grid = grid_of(cfg)
    n = 20000
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, n)
    y = oracle.label(grid, 2, "point", q.numpy())
    qd, yd = q.cuda(), torch.from_numpy(y).cuda()
    a = oracle.make_arch(2, 32, 2)
    models, thetas, taus = [], [], []
    for i in range(3):
        th = torch.from_numpy(np.random.default_rng(10 + i).normal(size=oracle.num_params(a)) * 0.6).float()
        m = nb.Model(nb.Desc("point", 2, 32, 2, (), "fp32"), 0)
        m.set_params(th)
        m.set_thresholds([0.1 * i - 0.05])
        models.append(m)
        thetas.append(th.double().numpy())
        taus.append(np.array([0.1 * i - 0.05]))
    for bad in ([0, 0, 0], [-1, 2, 0], [-1, 0, 5]):
        with pytest.raises(nb.NBError):
            nb.hier_score(models, bad, qd, yd)
    parent = [-1, 0, 0]
    c = nb.hier_score(models, parent, qd, yd)
    z = [oracle.forward(a, th, q.numpy())[:, 0] for th in thetas]
    keep = np.all([np.abs(zi - t[0]) > 1e-4 for zi, t in zip(z, taus)], axis=0)
    pred = oracle.hier_combine(parent, [zi >= np.float32(t[0]) for zi, t in zip(z, taus)])
    sub = nb.hier_score(models, parent, qd[torch.from_numpy(keep).cuda()], yd[torch.from_numpy(keep).cuda()])
    yy = y[keep].astype(bool)
    p = pred[keep]
    assert (sub["tp"], sub["fp"], sub["fn"], sub["tn"]) == (int((p & yy).sum()), int((p & ~yy).sum()),
                                                            int((~p & yy).sum()), int((~p & ~yy).sum()))
    assert c["tp"] + c["fp"] + c["fn"] + c["tn"] == n


@pytest.mark.gpu
def test_gpu_hierarchy_nonfinite_and_scratch_reuse():
    """Non-finite records fail the node that sees them and are reported
    (warning-class NB_E_NONFINITE with the counts written); repeated calls
    reuse the root's scratch and give identical counts."""
    import paper_2310_06822_b200 as nb
    from gpu_helpers import grid_of
    cfg = nbgen.CONFIGS["c1"]
    n = 5000
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, n)
    y = oracle.label(grid_of(cfg), 2, "point", q.numpy())
    a = oracle.make_arch(2, 64, 3)
    models = []
    for i in range(3):
        m = nb.Model(nb.Desc("point", 2, 64, 3, (), "bf16"), 0)
        m.set_params(torch.from_numpy(np.random.default_rng(20 + i).normal(size=oracle.num_params(a)) * 0.25).float())
        m.set_thresholds([-1e9])   # every finite row passes every node
        models.append(m)
    yd = torch.from_numpy(y).cuda()
    ref = nb.hier_score(models, [-1, 0, 0], q.cuda(), yd)
    assert ref == nb.hier_score(models, [-1, 0, 0], q.cuda(), yd)
    assert ref["tp"] + ref["fp"] == n and ref["nonfinite"] == 0
    bad = q.clone()
    rows = [0, 777, n - 1]
    bad[rows, 1] = float("nan")
    with pytest.raises(nb.NBError) as ei:
        nb.hier_score(models, [-1, 0, 0], bad.cuda(), yd)
    assert "NONFINITE" in str(ei.value)
    c = nb.hier_score(models, [-1, 0, 0], bad.cuda(), yd, allow_nonfinite=True)
    assert c["nonfinite"] == len(rows)
    assert c["tp"] + c["fp"] == n - len(rows) and c["tp"] + c["fp"] + c["fn"] + c["tn"] == n


@pytest.mark.gpu
@pytest.mark.parametrize("parent", [[-1, 0, 1, 1, 0, 4, 4], [-1, 0, 0, 1, 2, 1, 2]])
def test_gpu_hierarchy_depth2_interleaved_siblings(parent):
    """Seven fp32 nodes, depth 2, in depth-first order (siblings 2/3 and 5/6
    consecutive, 1 and 4 not) and in an order where no two consecutive nodes
    share a parent: every node's gather (shared by consecutive siblings) must
    see its own parent's survivors.  Counts equal the oracle's combination
    exactly away from the thresholds."""
    import paper_2310_06822_b200 as nb
    from gpu_helpers import grid_of
    cfg = nbgen.CONFIGS["c1"]
    n = 3 * 4096 + 11
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 1, n)
    y = oracle.label(grid_of(cfg), 2, "point", q.numpy())
    qd, yd = q.cuda(), torch.from_numpy(y).cuda()
    a = oracle.make_arch(2, 32, 2)
    models, thetas, taus = [], [], []
    for i in range(len(parent)):
        th = torch.from_numpy(np.random.default_rng(40 + i).normal(size=oracle.num_params(a)) * 0.6).float()
        m = nb.Model(nb.Desc("point", 2, 32, 2, (), "fp32"), 0)
        m.set_params(th)
        t = float(np.quantile(oracle.forward(a, th.double().numpy(), q.numpy()[:2000])[:, 0], 0.3))
        m.set_thresholds([t])
        models.append(m)
        thetas.append(th.double().numpy())
        taus.append(t)
    z = [oracle.forward(a, th, q.numpy())[:, 0] for th in thetas]
    keep = np.all([np.abs(zi - t) > 1e-4 for zi, t in zip(z, taus)], axis=0)
    pred = oracle.hier_combine(parent, [zi >= np.float32(t) for zi, t in zip(z, taus)])
    c = nb.hier_score(models, parent, qd[torch.from_numpy(keep).cuda()], yd[torch.from_numpy(keep).cuda()])
    yy = y[keep].astype(bool)
    p = pred[keep]
    assert 0.05 < p.mean() < 0.95  # pruning happens at every level
    assert (c["tp"], c["fp"], c["fn"], c["tn"]) == (int((p & yy).sum()), int((p & ~yy).sum()),
                                                    int((~p & yy).sum()), int((~p & ~yy).sum()))
