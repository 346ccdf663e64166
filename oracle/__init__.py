"""oracle — plain CPU oracle for the Neural Bounding hot path (ctypes binding).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py, never by the product package
(paper_2310_06822_b200).  It shares no code with the CUDA path; see
oracle/nb_oracle.h for the per-function citations into PAPER.md.  The training
control (PaperSchedule, reg_grad; NEXT-2) is plain Python/numpy in this file.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libnb_oracle.so")
SRC = os.path.join(HERE, "nb_oracle.c")

POINT, RAY, PLANE, BOX = 0, 1, 2, 3
KIND = {"point": POINT, "ray": RAY, "plane": PLANE, "box": BOX}
FP64, BF16_EMU = 0, 1


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no fast-math, no FMA contraction)."""
    if force or not os.path.exists(LIB_PATH) or \
            os.path.getmtime(LIB_PATH) < os.path.getmtime(SRC) or \
            os.path.getmtime(LIB_PATH) < os.path.getmtime(os.path.join(HERE, "nb_oracle.h")):
        cmd = ["gcc", "-O2", "-fno-fast-math", "-ffp-contract=off", "-fopenmp", "-std=c11",
               "-shared", "-fPIC", "-o", LIB_PATH, SRC, "-lm"]
        subprocess.check_call(cmd)
    return LIB_PATH


class Arch(C.Structure):
    _fields_ = [("d0", C.c_int32), ("width", C.c_int32), ("layers", C.c_int32),
                ("n_heads", C.c_int32), ("head_after", C.c_int32 * 2),
                ("act", C.c_int32), ("pe", C.c_int32)]


class Counts(C.Structure):
    _fields_ = [("tp", C.c_uint64), ("fp", C.c_uint64), ("fn", C.c_uint64), ("tn", C.c_uint64),
                ("exit_hist", C.c_uint64 * 4), ("nonfinite", C.c_uint64)]

    def as_dict(self):
        return dict(tp=self.tp, fp=self.fp, fn=self.fn, tn=self.tn,
                    exit_hist=list(self.exit_hist), nonfinite=self.nonfinite)


class Stats(C.Structure):
    _fields_ = [("loss", C.c_double), ("tp", C.c_uint64), ("fp", C.c_uint64),
                ("fn", C.c_uint64), ("tn", C.c_uint64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P, I64, I32, D = C.c_void_p, C.c_int64, C.c_int32, C.c_double
        sig = {
            "ora_indicator": (C.c_int, [P, I32, I32, I32, P]),
            "ora_label": (C.c_int, [P, I32, I32, I32, I32, P, I64, P]),
            "ora_label_brute": (C.c_int, [P, I32, I32, I32, I32, P, I64, P]),
            "ora_sat_build": (None, [P, I32, P]),
            "ora_encode_bf16": (None, [P, I64, I32, P]),
            "ora_encode_pe": (None, [P, I64, I32, I32, P]),
            "ora_bf16_rne": (C.c_uint16, [C.c_float]),
            "ora_num_params": (I64, [P]),
            "ora_forward": (None, [P, P, P, I64, I32, P]),
            "ora_loss_grad": (D, [P, P, P, P, I64, I64, D, D, P, P]),
            "ora_loss_grad_mode": (D, [P, P, P, P, I64, I64, D, D, P, P, I32]),
            "ora_weighted_bce": (D, [D, I32, D, D]),
            "ora_adam": (None, [I64, P, P, P, I64, D, D, D, D, P]),
            "ora_alpha": (D, [I64, I64]),
            "ora_calibrate": (C.c_int, [I32, P, P, I64, P]),
            "ora_score": (None, [I32, P, P, I64, P, P]),
            "ora_num_threads": (C.c_int, []),
        }
        for name, (res, args) in sig.items():
            f = getattr(_lib, name)
            f.restype = res
            f.argtypes = args
    return _lib


def _ptr(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.c_void_p)


def _np(x, dtype):
    if isinstance(x, torch.Tensor):
        x = x.detach().cpu().numpy()
    return np.ascontiguousarray(x, dtype=dtype)


ACT = {"relu": 0, "sine": 1}


def arch_of(cfg) -> Arch:
    a = Arch()
    a.d0, a.width, a.layers, a.n_heads = cfg.record_floats, cfg.width, cfg.hidden_layers, cfg.n_heads
    for k, l in enumerate(cfg.head_after):
        a.head_after[k] = l
    a.act = ACT[getattr(cfg, "activation", "relu")]
    a.pe = getattr(cfg, "pe_depth", 0)
    return a


def make_arch(d0, width, layers, head_after=(), act="relu", pe=0) -> Arch:
    """d0 = record floats; act "relu" | "sine" (R1, R41); pe = positional
    encoding depth (R42), layer 1 then reads d0 (1 + pe) inputs."""
    a = Arch()
    a.d0, a.width, a.layers, a.n_heads = d0, width, layers, len(head_after)
    for k, l in enumerate(head_after):
        a.head_after[k] = l
    a.act = ACT[act]
    a.pe = pe
    return a


def num_params(a: Arch) -> int:
    return int(lib().ora_num_params(C.byref(a)))


def label(grid, space_dim, kind, q, brute=False, frames=1) -> np.ndarray:
    g = _np(grid, np.uint8)
    q = _np(q, np.float32)
    R = g.shape[-1]
    n = q.shape[0]
    y = np.zeros(n, np.uint8)
    f = lib().ora_label_brute if brute else lib().ora_label
    rc = f(_ptr(g), space_dim, R, frames, KIND[kind] if isinstance(kind, str) else kind,
           _ptr(q), n, _ptr(y))
    assert rc == 0
    return y


def indicator(grid, space_dim, x, frames=1) -> int:
    g = _np(grid, np.uint8)
    xx = np.ascontiguousarray(x, np.float64)
    return int(lib().ora_indicator(_ptr(g), space_dim, g.shape[-1], frames, _ptr(xx)))


def sat(grid) -> np.ndarray:
    g = _np(grid, np.uint8)
    R = g.shape[0]
    S = np.zeros((R + 1,) * 3, np.int32)
    lib().ora_sat_build(_ptr(g), R, _ptr(S))
    return S


def encode_bf16(q) -> np.ndarray:
    q = _np(q, np.float32)
    n, d0 = q.shape
    out = np.zeros((n, 16), np.uint16)
    lib().ora_encode_bf16(_ptr(q), n, d0, _ptr(out))
    return out


def encode_pe(q, pe) -> np.ndarray:
    """bf16 PE operand [n][64] (R42): hi at [0, d_in), lo at [32, 32 + d_in)."""
    q = _np(q, np.float32)
    n, d0 = q.shape
    out = np.zeros((n, 64), np.uint16)
    lib().ora_encode_pe(_ptr(q), n, d0, pe, _ptr(out))
    return out


def forward(a: Arch, theta, q, mode=FP64) -> np.ndarray:
    th = _np(theta, np.float64)
    q = _np(q, np.float32)
    n = q.shape[0]
    out = np.zeros((n, 1 + a.n_heads), np.float64)
    lib().ora_forward(C.byref(a), _ptr(th), _ptr(q), n, mode, _ptr(out))
    return out


def loss_grad(a: Arch, theta, q, y, alpha, beta, n_global=None, mode=FP64):
    th = _np(theta, np.float64)
    q = _np(q, np.float32)
    yy = _np(y, np.uint8)
    n = q.shape[0]
    g = np.zeros(num_params(a), np.float64)
    st = Stats()
    loss = lib().ora_loss_grad_mode(C.byref(a), _ptr(th), _ptr(q), _ptr(yy), n,
                                    n if n_global is None else n_global, alpha, beta, _ptr(g),
                                    C.byref(st), mode)
    return loss, g, dict(loss=st.loss, tp=st.tp, fp=st.fp, fn=st.fn, tn=st.tn)


def weighted_bce(z, y, alpha, beta) -> float:
    return float(lib().ora_weighted_bce(z, y, alpha, beta))


def adam(theta, m, v, t, g, lr=1e-3, b1=0.9, b2=0.999, eps=1e-8):
    """In-place Adam on float64 numpy arrays."""
    lib().ora_adam(theta.size, _ptr(theta), _ptr(m), _ptr(v), t, lr, b1, b2, eps,
                   _ptr(_np(g, np.float64)))


def reg_grad(theta, l1, l2) -> np.ndarray:
    """Gradient of l1 sum|theta| + l2 sum theta^2 (Suppl. Sec. 2.2 "L1 and L2
    regularizations"; R38: every parameter)."""
    th = _np(theta, np.float64)
    return l1 * np.sign(th) + 2.0 * l2 * th


class PaperSchedule:
    """Suppl. Sec. 2.1 FN-gated weight schedule and the early stop
    of P:297, step by step in the paper's terms (R37-R39): every
    `step_every` iterations, if the window saw FNs, the k-th such step moves
    the weights by the dimension's harmonic decrement (1/20, 1/40, ... in 2D;
    1/100, 1/200, ... in 3D; 1/200, 1/400, ... in 4D) on the FP side (beta,
    floor 1e-3) and by 0.2 on the FN side (alpha); lambda ramps linearly from
    0 to 5e-7 (Suppl. Sec. 2.2); training stops after six FN-free windows."""

    def __init__(self, space_dim, step_every=10000, max_steps=1 << 40):
        self.space_dim, self.step_every, self.max_steps = space_dim, step_every, max_steps
        self.alpha, self.beta, self.lam = 1.0, 1.0, 0.0
        self.step = self.triggers = self.window_fn = self.stable = 0
        self.stop = False

    def decrement(self, k):
        first = {2: 20.0, 3: 100.0, 4: 200.0}[self.space_dim]
        return 1.0 / (first * k)  # 1/20, 1/40, 1/60 ... (2D)

    def after_step(self, batch_fn):
        self.window_fn += int(batch_fn)
        self.step += 1
        if self.step % self.step_every == 0:
            if self.window_fn > 0:
                self.triggers += 1
                self.beta = max(1e-3, self.beta - self.decrement(self.triggers))
                self.alpha = self.alpha + 0.2
                self.stable = 0
            else:
                self.stable += 1
            self.window_fn = 0
        self.lam = 5e-7 * min(1.0, self.step / self.max_steps)
        self.stop = self.stable >= 6 or self.step >= self.max_steps


def hier_combine(parent, passes) -> np.ndarray:
    """Neural bounding hierarchy (§3.2; R45): a record is
    positive iff some root-to-leaf path has every node passing.  parent[0] =
    -1, parent[i] < i; passes: bool [nodes][n].  Forward propagation of
    "every node on the path so far passes", then OR over the leaves."""
    passes = np.asarray(passes, bool)
    ok = np.zeros_like(passes)
    leaf = np.ones(len(parent), bool)
    for i, p in enumerate(parent):
        ok[i] = passes[i] if p < 0 else (ok[p] & passes[i])
        if p >= 0:
            leaf[p] = False
    return np.any(ok[leaf], axis=0)


def hier_predict(archs, thetas, taus, parent, q, mode=FP64) -> np.ndarray:
    """Each node's calibrated predictor [e_k >= tau_k][z >= tau] on every
    record (no pruning: the definition), combined by hier_combine."""
    passes = []
    for a, th, tau in zip(archs, thetas, taus):
        z = forward(a, th, q, mode)
        ok = z[:, 0] >= tau[0]
        for k in range(a.n_heads):
            ok &= z[:, 1 + k] >= tau[1 + k]
        passes.append(ok)
    return hier_combine(parent, passes)


def alpha(t, T) -> float:
    return float(lib().ora_alpha(t, T))


def calibrate(logits, y):
    z = _np(logits, np.float64)
    if z.ndim == 1:
        z = z[:, None]
    yy = _np(y, np.uint8)
    tau = np.zeros(z.shape[1], np.float64)
    rc = lib().ora_calibrate(z.shape[1] - 1, _ptr(z), _ptr(yy), z.shape[0], _ptr(tau))
    return tau, rc


def score(logits, y, tau) -> dict:
    z = _np(logits, np.float64)
    if z.ndim == 1:
        z = z[:, None]
    yy = _np(y, np.uint8)
    t = _np(tau, np.float64)
    c = Counts()
    lib().ora_score(z.shape[1] - 1, _ptr(z), _ptr(yy), z.shape[0], _ptr(t), C.byref(c))
    return c.as_dict()


def num_threads() -> int:
    return int(lib().ora_num_threads())


def train(cfg, theta0, batches, T=None, lr=1e-3):
    """Plain training loop (Alg. 1 + Adam): batches yields (q, y) per step."""
    a = arch_of(cfg)
    th = _np(theta0, np.float64).copy()
    m = np.zeros_like(th)
    v = np.zeros_like(th)
    hist = []
    for t, (q, y) in enumerate(batches):
        al = alpha(t, T)
        loss, g, st = loss_grad(a, th, q, y, al, 1.0)
        adam(th, m, v, t + 1, g, lr=lr)
        hist.append(st)
    return th, hist
