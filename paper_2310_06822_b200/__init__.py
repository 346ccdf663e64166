"""paper_2310_06822_b200 — B200-native Neural Bounding hot path (Python binding).

Thin ctypes marshalling over libnb.so (include/nb.h).  Every step of the path
runs in the library's CUDA kernels; PyTorch only provides device memory,
streams and process groups.  There is no CPU fallback: if libnb.so is missing
or the device is not sm_100, calls raise.

    import paper_2310_06822_b200 as nb
    m = nb.Model(nb.Desc(kind="point", space_dim=3, width=64, hidden_layers=4,
                         precision="bf16"), device=0)
    m.set_params(theta)                      # canonical fp32 blob (CPU tensor)
    tau = m.calibrate(q, y)                  # q fp32 [n][d0], y uint8 [n] on cuda
    counts = m.score(q, y)                   # FP/FN/TP/TN of the calibrated predictor
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libnb.so")

POINT, RAY, PLANE, BOX = 0, 1, 2, 3
KINDS = {"point": POINT, "ray": RAY, "plane": PLANE, "box": BOX}
FP32, BF16 = 0, 1
PRECISIONS = {"fp32": FP32, "bf16": BF16}
ACTIVATIONS = {"relu": 0, "sine": 1}  # nb_activation (R1, R41)
STATUS = ["NB_OK", "NB_E_ARG", "NB_E_SHAPE", "NB_E_NONFINITE", "NB_E_LABEL",
          "NB_E_NO_POSITIVES", "NB_E_CUDA", "NB_E_NCCL", "NB_E_UNSUPPORTED", "NB_E_OOM"]
NB_OK, NB_E_NONFINITE, NB_E_NO_POSITIVES = 0, 3, 5


class NBError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        self.status = status
        name = STATUS[status] if 0 <= status < len(STATUS) else str(status)
        super().__init__(f"{where}: {name}: {detail}")


class _Desc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("space_dim", C.c_int32), ("width", C.c_int32),
                ("hidden_layers", C.c_int32), ("n_heads", C.c_int32),
                ("head_after", C.c_int32 * 2), ("precision", C.c_int32),
                ("activation", C.c_int32), ("pe_depth", C.c_int32)]


class _Counts(C.Structure):
    _fields_ = [("tp", C.c_uint64), ("fp", C.c_uint64), ("fn", C.c_uint64), ("tn", C.c_uint64),
                ("exit_hist", C.c_uint64 * 4), ("nonfinite", C.c_uint64)]

    def as_dict(self):
        return dict(tp=self.tp, fp=self.fp, fn=self.fn, tn=self.tn,
                    exit_hist=list(self.exit_hist), nonfinite=self.nonfinite)


class _Schedule(C.Structure):
    _fields_ = [("space_dim", C.c_int32), ("patience", C.c_int32), ("step_every", C.c_int64),
                ("max_steps", C.c_int64), ("alpha", C.c_double), ("beta", C.c_double),
                ("lam", C.c_double), ("step", C.c_int64), ("triggers", C.c_int64),
                ("window_fn", C.c_uint64), ("stable", C.c_int32), ("stop", C.c_int32)]


class PaperSchedule:
    """The paper's FN-gated training control (nb_schedule_*, nb.h): alpha, beta
    and the L1/L2 weight for the next step; report each step's batch FN."""

    def __init__(self, space_dim: int, step_every: int = 10000, max_steps: int = 1 << 40):
        self._s = _Schedule()
        _check(lib().nb_schedule_init(C.byref(self._s), space_dim, step_every, max_steps),
               "nb_schedule_init")

    def after_step(self, batch_fn: int) -> None:
        _check(lib().nb_schedule_after_step(C.byref(self._s), int(batch_fn)), "nb_schedule_after_step")

    alpha = property(lambda self: self._s.alpha)
    beta = property(lambda self: self._s.beta)
    lam = property(lambda self: self._s.lam)
    triggers = property(lambda self: self._s.triggers)
    step = property(lambda self: self._s.step)
    stop = property(lambda self: bool(self._s.stop))


class _Stats(C.Structure):
    _fields_ = [("loss", C.c_double), ("tp", C.c_uint64), ("fp", C.c_uint64),
                ("fn", C.c_uint64), ("tn", C.c_uint64)]


# name -> (restype, argtypes); must cover every function declared in include/nb.h
_P, _I32, _I64, _F, _D = C.c_void_p, C.c_int32, C.c_int64, C.c_float, C.c_double
SIGNATURES = {
    "nb_record_floats": (_I64, [_I32, _I32]),
    "nb_num_params": (_I64, [_P]),
    "nb_status_string": (C.c_char_p, [C.c_int]),
    "nb_last_error": (C.c_char_p, []),
    "nb_device_check": (C.c_int, [_I32, _P]),
    "nb_model_create": (C.c_int, [_P, _I32, _P]),
    "nb_model_destroy": (None, [_P]),
    "nb_model_set_params": (C.c_int, [_P, _P, _I64]),
    "nb_model_get_params": (C.c_int, [_P, _P, _I64]),
    "nb_model_set_thresholds": (C.c_int, [_P, _P, _I32]),
    "nb_model_get_thresholds": (C.c_int, [_P, _P, _I32]),
    "nb_model_get_grad": (C.c_int, [_P, _P, _I64]),
    "nb_model_get_adam": (C.c_int, [_P, _P, _P, _P]),
    "nb_model_set_adam": (C.c_int, [_P, _P, _P, _I64]),
    "nb_model_set_timing": (C.c_int, [_P, _I32]),
    "nb_model_kernel_time": (C.c_int, [_P, _P, _P]),
    "nb_comm_unique_id": (C.c_int, [_P]),
    "nb_comm_init": (C.c_int, [_P, _P, _I32, _I32]),
    "nb_comm_version": (C.c_int, [_P]),
    "nb_encode": (C.c_int, [_P, _P, _I64, _P, _P]),
    "nb_forward": (C.c_int, [_P, _P, _I64, _P, _P, _P]),
    "nb_calibrate": (C.c_int, [_P, _P, _P, _I64, _P, _P]),
    "nb_score": (C.c_int, [_P, _P, _P, _I64, _P, _P]),
    "nb_calibrate_inverted": (C.c_int, [_P, _P, _P, _I64, _P, _P]),
    "nb_hier_score": (C.c_int, [_P, _I32, _P, _P, _P, _I64, _P, _P]),
    "nb_score_host": (C.c_int, [_P, _P, _P, _I64, _P, _P]),
    "nb_score_async": (C.c_int, [_P, _P, _P, _I64, _P, _P]),
    "nb_train_step": (C.c_int, [_P, _P, _P, _I64, _I64, _F, _F, _F, _P, _P]),
    "nb_train_steps": (C.c_int, [_P, _P, _P, _I64, _I64, _I32, _F, _F, _F, _F, _P]),
    "nb_alpha": (_D, [_I64, _I64]),
    "nb_model_set_regularization": (C.c_int, [_P, _F, _F]),
    "nb_schedule_init": (C.c_int, [_P, _I32, _I64, _I64]),
    "nb_schedule_after_step": (C.c_int, [_P, C.c_uint64]),
    "nb_grid_create": (C.c_int, [_I32, _I32, _I32, _P, _I32, _P]),
    "nb_grid_destroy": (None, [_P]),
    "nb_label": (C.c_int, [_P, _I32, _P, _I64, _P, _P]),
}

_lib = None


def lib():
    """Load libnb.so (built in-tree by __graft_entry__.build()); raise if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run python -m paper_2310_06822_b200.build")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(status: int, where: str, ok=(NB_OK,)):
    if status not in ok:
        raise NBError(status, where, lib().nb_last_error().decode())
    return status


def _stream(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _dev_ptr(t: torch.Tensor, dtype, device, name):
    if not isinstance(t, torch.Tensor) or t.device.type != "cuda" or t.device.index != device:
        raise ValueError(f"{name} must be a CUDA tensor on cuda:{device}")
    if t.dtype != dtype or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous {dtype} tensor")
    return t.data_ptr()


@dataclass(frozen=True)
class Desc:
    kind: str = "point"
    space_dim: int = 3
    width: int = 64
    hidden_layers: int = 4
    head_after: tuple = ()
    precision: str = "bf16"
    activation: str = "relu"   # or "sine" (R41)
    pe_depth: int = 0          # positional encoding depth L (Suppl. §3, R42)

    def to_c(self) -> _Desc:
        d = _Desc()
        d.kind = KINDS[self.kind]
        d.space_dim = self.space_dim
        d.width = self.width
        d.hidden_layers = self.hidden_layers
        d.n_heads = len(self.head_after)
        for k, l in enumerate(self.head_after):
            d.head_after[k] = l
        d.precision = PRECISIONS[self.precision]
        d.activation = ACTIVATIONS[self.activation]
        d.pe_depth = self.pe_depth
        return d

    @property
    def record_floats(self) -> int:
        return int(lib().nb_record_floats(KINDS[self.kind], self.space_dim))

    @property
    def n_heads(self) -> int:
        return len(self.head_after)

    @property
    def num_params(self) -> int:
        d = self.to_c()
        return int(lib().nb_num_params(C.byref(d)))


def alpha(t: int, T: int) -> float:
    """FN weight of step t of T (row a10; R6). beta = 1."""
    return float(lib().nb_alpha(t, T))


def comm_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(lib().nb_comm_unique_id(buf), "nb_comm_unique_id")
    return bytes(buf)


def comm_version() -> int:
    v = C.c_int32()
    _check(lib().nb_comm_version(C.byref(v)), "nb_comm_version")
    return v.value


class Model:
    """A bounding MLP resident on one GPU (owning weights, Adam state, tau)."""

    def __init__(self, desc: Desc, device: int = 0):
        self.desc = desc
        self.device = device
        self._d = desc.to_c()
        h = C.c_void_p()
        _check(lib().nb_model_create(C.byref(self._d), device, C.byref(h)), "nb_model_create")
        self._h = h
        self.P = desc.num_params
        self.d0 = desc.record_floats
        self.nl = 1 + desc.n_heads

    def close(self):
        if getattr(self, "_h", None):
            lib().nb_model_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- state ---------------------------------------------------------
    def set_params(self, theta: torch.Tensor):
        t = theta.detach().to("cpu", torch.float32).contiguous()
        _check(lib().nb_model_set_params(self._h, t.data_ptr(), t.numel()), "nb_model_set_params")

    def get_params(self) -> torch.Tensor:
        t = torch.empty(self.P, dtype=torch.float32)
        _check(lib().nb_model_get_params(self._h, t.data_ptr(), self.P), "nb_model_get_params")
        return t

    def get_grad(self) -> torch.Tensor:
        t = torch.empty(self.P, dtype=torch.float32)
        _check(lib().nb_model_get_grad(self._h, t.data_ptr(), self.P), "nb_model_get_grad")
        return t

    def set_thresholds(self, tau):
        t = torch.as_tensor(tau, dtype=torch.float32).contiguous()
        _check(lib().nb_model_set_thresholds(self._h, t.data_ptr(), t.numel()), "set_thresholds")

    def get_thresholds(self) -> torch.Tensor:
        t = torch.empty(self.nl, dtype=torch.float32)
        _check(lib().nb_model_get_thresholds(self._h, t.data_ptr(), self.nl), "get_thresholds")
        return t

    def get_adam(self):
        m = torch.empty(self.P, dtype=torch.float32)
        v = torch.empty(self.P, dtype=torch.float32)
        step = C.c_int64()
        _check(lib().nb_model_get_adam(self._h, m.data_ptr(), v.data_ptr(), C.byref(step)), "get_adam")
        return m, v, step.value

    def set_adam(self, m, v, step):
        m = m.to("cpu", torch.float32).contiguous()
        v = v.to("cpu", torch.float32).contiguous()
        _check(lib().nb_model_set_adam(self._h, m.data_ptr(), v.data_ptr(), step), "set_adam")

    def set_timing(self, enable: bool):
        _check(lib().nb_model_set_timing(self._h, 1 if enable else 0), "nb_model_set_timing")

    def kernel_time(self):
        """(device ms, launches) of the bracketed hot-path kernels since last call."""
        ms = C.c_double()
        k = C.c_int64()
        _check(lib().nb_model_kernel_time(self._h, C.byref(ms), C.byref(k)), "nb_model_kernel_time")
        return ms.value, k.value

    def comm_init(self, uid: bytes, rank: int, world: int):
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        _check(lib().nb_comm_init(self._h, buf, rank, world), "nb_comm_init")

    # ---- hot path ------------------------------------------------------
    def _q(self, q):
        if q.dim() != 2 or q.shape[1] != self.d0:
            raise ValueError(f"q must be [n][{self.d0}]")
        return _dev_ptr(q, torch.float32, self.device, "q")

    def encode(self, q: torch.Tensor) -> torch.Tensor:
        n = q.shape[0]
        if self.desc.precision == "bf16":
            out = torch.empty(n, 64 if self.desc.pe_depth else 16, dtype=torch.int16, device=q.device)
        else:
            out = torch.empty(n, self.d0, dtype=torch.float32, device=q.device)
        _check(lib().nb_encode(self._h, self._q(q), n, out.data_ptr(), _stream(self.device)), "nb_encode")
        return out

    def forward(self, q: torch.Tensor, prob: bool = False):
        n = q.shape[0]
        logits = torch.empty(n, self.nl, dtype=torch.float32, device=q.device)
        p = torch.empty(n, dtype=torch.float32, device=q.device) if prob else None
        _check(lib().nb_forward(self._h, self._q(q), n, logits.data_ptr(),
                                p.data_ptr() if p is not None else None, _stream(self.device)),
               "nb_forward")
        return (logits, p) if prob else logits

    def calibrate(self, q: torch.Tensor, y: torch.Tensor, allow_no_positives=False) -> torch.Tensor:
        n = q.shape[0]
        tau = torch.empty(self.nl, dtype=torch.float32)
        ok = (NB_OK, NB_E_NO_POSITIVES) if allow_no_positives else (NB_OK,)
        _check(lib().nb_calibrate(self._h, self._q(q), _dev_ptr(y, torch.uint8, self.device, "y"),
                                  n, tau.data_ptr(), _stream(self.device)), "nb_calibrate", ok)
        return tau

    def calibrate_inverted(self, q: torch.Tensor, y: torch.Tensor) -> torch.Tensor:
        """Certainly-hit threshold (R43): FP = 0 on (q, y)."""
        n = q.shape[0]
        tau = torch.empty(self.nl, dtype=torch.float32)
        _check(lib().nb_calibrate_inverted(self._h, self._q(q), _dev_ptr(y, torch.uint8, self.device, "y"),
                                           n, tau.data_ptr(), _stream(self.device)), "nb_calibrate_inverted")
        return tau

    def score(self, q: torch.Tensor, y: torch.Tensor, allow_nonfinite: bool = False) -> dict:
        c = _Counts()
        ok = (NB_OK, NB_E_NONFINITE) if allow_nonfinite else (NB_OK,)
        _check(lib().nb_score(self._h, self._q(q), _dev_ptr(y, torch.uint8, self.device, "y"),
                              q.shape[0], C.byref(c), _stream(self.device)), "nb_score", ok)
        return c.as_dict()

    def score_async(self, q: torch.Tensor, y: torch.Tensor, out: torch.Tensor) -> None:
        """nb_score_async: counts land in `out` (uint64/int64 [9], pinned host or
        on this device) when the current stream gets there; no synchronisation."""
        if out.dtype not in (torch.int64, torch.uint64) or out.numel() != 9 or not out.is_contiguous():
            raise ValueError("out must be a contiguous 9-element 64-bit tensor")
        if out.device.type == "cpu" and not out.is_pinned():
            raise ValueError("host out must be pinned")
        _check(lib().nb_score_async(self._h, self._q(q), _dev_ptr(y, torch.uint8, self.device, "y"),
                                    q.shape[0], out.data_ptr(), _stream(self.device)),
               "nb_score_async")

    @staticmethod
    def counts_dict(out: torch.Tensor) -> dict:
        v = [int(x) for x in out.cpu().view(torch.int64).tolist()]
        return dict(tp=v[0], fp=v[1], fn=v[2], tn=v[3], exit_hist=v[4:8], nonfinite=v[8])

    def score_host(self, q: torch.Tensor, y: torch.Tensor) -> dict:
        if q.device.type != "cpu" or y.device.type != "cpu":
            raise ValueError("score_host takes host tensors")
        q = q.contiguous()
        y = y.contiguous()
        if q.dtype != torch.float32 or y.dtype != torch.uint8 or q.shape[1] != self.d0:
            raise ValueError("q fp32 [n][d0], y uint8 [n]")
        c = _Counts()
        _check(lib().nb_score_host(self._h, q.data_ptr(), y.data_ptr(), q.shape[0], C.byref(c),
                                   _stream(self.device)), "nb_score_host")
        return c.as_dict()

    def set_regularization(self, l1: float, l2: float) -> None:
        _check(lib().nb_model_set_regularization(self._h, l1, l2), "nb_model_set_regularization")

    def train_steps(self, q, y, steps: int, alpha0: float, alpha1: float, beta: float = 1.0,
                    lr: float = 1e-3, n_global: int | None = None):
        """nb_train_steps: `steps` consecutive batches of q.shape[0] // steps
        rows (one CUDA graph without a communicator); asynchronous."""
        n = q.shape[0] // steps
        if n * steps != q.shape[0] or y.shape[0] != q.shape[0]:
            raise ValueError("q / y must hold steps equal batches")
        _check(lib().nb_train_steps(self._h, self._q(q), _dev_ptr(y, torch.uint8, self.device, "y"), n,
                                    n if n_global is None else n_global, steps, alpha0, alpha1, beta, lr,
                                    _stream(self.device)), "nb_train_steps")

    def train_step(self, q, y, alpha: float, beta: float = 1.0, lr: float = 1e-3,
                   n_global: int | None = None, stats: bool = False):
        n = q.shape[0]
        st = _Stats() if stats else None
        _check(lib().nb_train_step(self._h, self._q(q), _dev_ptr(y, torch.uint8, self.device, "y"),
                                   n, n if n_global is None else n_global, alpha, beta, lr,
                                   C.byref(st) if st is not None else None, _stream(self.device)),
               "nb_train_step")
        if st is not None:
            return dict(loss=st.loss, tp=st.tp, fp=st.fp, fn=st.fn, tn=st.tn)
        return None


def set_exit_handoff(mode: str) -> None:
    """Hand-off between the early-exit segments of nb_score (models with exit
    heads): "images" (the survivors' bf16 activations, default, faster) or
    "records" (their fp32 records; the later segments recompute the earlier
    layers: 8x less DRAM traffic).  Process-wide; counts are identical."""
    if mode not in ("images", "records"):
        raise ValueError("mode must be 'images' or 'records'")
    lib().nb_debug_set_exit_records(1 if mode == "records" else 0)


def hier_score(nodes, parent, q: torch.Tensor, y: torch.Tensor, allow_nonfinite: bool = False) -> dict:
    """Neural bounding hierarchy (nb_hier_score): counts of the
    predictor "some root-to-leaf path passes every node"."""
    dev = nodes[0].device
    arr = (C.c_void_p * len(nodes))(*[m._h.value if isinstance(m._h, C.c_void_p) else m._h for m in nodes])
    par = (C.c_int32 * len(parent))(*parent)
    c = _Counts()
    _check(lib().nb_hier_score(arr, len(nodes), par, nodes[0]._q(q), _dev_ptr(y, torch.uint8, dev, "y"),
                               q.shape[0], C.byref(c), _stream(dev)), "nb_hier_score",
           (NB_OK, NB_E_NONFINITE) if allow_nonfinite else (NB_OK,))
    return c.as_dict()


class Grid:
    """Occupancy grid resident on the GPU for the ground-truth labeller."""

    def __init__(self, occ: torch.Tensor, space_dim: int, device: int = 0):
        g = occ.detach().to("cpu", torch.uint8).contiguous()
        frames = g.shape[0] if space_dim == 4 else 1
        R = g.shape[-1]
        h = C.c_void_p()
        _check(lib().nb_grid_create(space_dim, R, frames, g.data_ptr(), device, C.byref(h)),
               "nb_grid_create")
        self._h = h
        self.device = device
        self.space_dim = space_dim

    def label(self, kind: str, q: torch.Tensor) -> torch.Tensor:
        n = q.shape[0]
        y = torch.empty(n, dtype=torch.uint8, device=q.device)
        _check(lib().nb_label(self._h, KINDS[kind], _dev_ptr(q, torch.float32, self.device, "q"),
                              n, y.data_ptr(), _stream(self.device)), "nb_label")
        return y

    def close(self):
        if getattr(self, "_h", None):
            lib().nb_grid_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
