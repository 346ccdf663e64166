"""nbgen — seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NONE of the method's arithmetic (no encoding, no MLP, no loss,
no labelling): it only draws numbers and rasterises the synthetic indicator
grids that stand in for the paper's datasets (§4.2 "Indicators",
P:354-361; the datasets themselves are not in this container).  Every config is
the one BASELINE.json names (configs[0..4], called c1..c5 here); the recipe is
restated in DESIGN.md §3.

Random numbers come from counter-based SplitMix64 streams:
output i of the stream keyed k is mix64(k + (i+1)*GAMMA), so any row of any
query set can be regenerated on its own.  The implementation is torch integer
arithmetic on int64 (wrapping, logical shifts by masking) so the same bytes are
produced on CPU and on a CUDA device.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import torch

GAMMA = 0x9E3779B97F4A7C15
C1 = 0xBF58476D1CE4E5B9
C2 = 0x94D049BB133111EB
TAG_GRID, TAG_INIT, TAG_TRAIN, TAG_EVAL, TAG_HOLDOUT = 1, 2, 3, 4, 5
M64 = (1 << 64) - 1


def _s64(x: int) -> int:
    """Python int (mod 2^64) -> the int64 with the same bits."""
    x &= M64
    return x - (1 << 64) if x >> 63 else x


def _u64(x: int) -> int:
    return x & M64


def mix64_int(z: int) -> int:
    """Scalar SplitMix64 finaliser on Python ints (used for stream keys)."""
    z &= M64
    z = ((z ^ (z >> 30)) * C1) & M64
    z = ((z ^ (z >> 27)) * C2) & M64
    return z ^ (z >> 31)


def _lsr(z: torch.Tensor, k: int) -> torch.Tensor:
    """Logical right shift of int64 bit patterns."""
    return (z >> k) & ((1 << (64 - k)) - 1)


def mix64(z: torch.Tensor) -> torch.Tensor:
    z = (z ^ _lsr(z, 30)) * _s64(C1)
    z = (z ^ _lsr(z, 27)) * _s64(C2)
    return z ^ _lsr(z, 31)


def stream_key(seed: int, tag: int) -> int:
    return mix64_int(seed ^ tag)


def draws(key: int, start: int, count: int, device="cpu") -> torch.Tensor:
    """int64 bit patterns of outputs [start, start+count) of stream `key`."""
    i = torch.arange(start + 1, start + 1 + count, dtype=torch.int64, device=device)
    return mix64(i * _s64(GAMMA) + _s64(key))


def u32f(x: torch.Tensor) -> torch.Tensor:
    """Top 24 bits -> float32 in [0, 1), exact."""
    return _lsr(x, 40).to(torch.float32) * (2.0 ** -24)


def u64d(x: torch.Tensor) -> torch.Tensor:
    """Top 53 bits -> float64 in [0, 1), exact."""
    return _lsr(x, 11).to(torch.float64) * (2.0 ** -53)


def splitmix64_sequence(seed: int, count: int) -> list[int]:
    """The plain SplitMix64 generator state=seed, for the known-answer test."""
    d = draws(seed, 0, count)
    return [_u64(int(v)) for v in d.tolist()]


# --------------------------------------------------------------------------
# Configs (BASELINE.json configs[0..4])
# --------------------------------------------------------------------------
@dataclass(frozen=True)
class Config:
    name: str
    space_dim: int          # 2, 3, or 4 (= 3D + time)
    kind: str               # "point" | "ray" | "box" | "plane"
    width: int
    hidden_layers: int
    head_after: tuple = ()  # hidden-layer indices (1-based) after which exit heads sit
    precision: str = "bf16"
    n_eval: int = 0
    train_batch: int = 0
    train_steps: int = 0
    seed: int = 0
    grid: dict = field(default_factory=dict)

    @property
    def record_floats(self) -> int:
        if self.kind == "point":
            return self.space_dim
        return 2 * self.space_dim

    @property
    def n_heads(self) -> int:
        return len(self.head_after)


CONFIGS = {
    "c1": Config("c1", 2, "point", 32, 2, (), "fp32", 65536, 4096, 200,
                 grid=dict(kind="discs", R=128, count=8)),
    "c2": Config("c2", 3, "point", 64, 4, (), "bf16", 1 << 22, 1 << 16, 5000,
                 grid=dict(kind="ellipsoids", R=64, count=16)),
    "c3": Config("c3", 3, "ray", 128, 4, (), "bf16", 1 << 24, 1 << 16, 5000,
                 grid=dict(kind="ellipsoids", R=64, count=16)),
    "c4": Config("c4", 4, "point", 128, 6, (2, 4), "bf16", 1 << 26, 1 << 16, 5000,
                 grid=dict(kind="moving_spheres", R=64, frames=32, count=12)),
    "c5": Config("c5", 3, "box", 256, 4, (), "bf16", 1 << 28, 1 << 18, 20000,
                 grid=dict(kind="ellipsoids", R=128, count=64)),
}


# NEXT-3: 4D rays, boxes and hyperplanes over c4's animated
# scene (8-float records, Suppl. Tab. 4/5 "4D Ray, Plane, Box"; R48).  Test and
# measurement configs beside BASELINE.json's five; net 8 -> 128 x 4 -> 1 bf16.
EXTRA_CONFIGS = {
    f"c4{k}": Config(f"c4{k}", 4, k, 128, 4, (), "bf16", 1 << 20, 1 << 16, 5000,
                     grid=dict(kind="moving_spheres", R=64, frames=32, count=12))
    for k in ("ray", "box", "plane")
}


def grid_shape(cfg: Config) -> tuple:
    g = cfg.grid
    if g["kind"] == "discs":
        return (g["R"], g["R"])
    if g["kind"] == "moving_spheres":
        return (g["frames"], g["R"], g["R"], g["R"])
    return (g["R"], g["R"], g["R"])


# --------------------------------------------------------------------------
# Occupancy grids: voxel occupied iff its centre lies in the closed shape
# (reading R11; "1 inside and on the surface").
# --------------------------------------------------------------------------
def _centres(R: int) -> torch.Tensor:
    return (torch.arange(R, dtype=torch.float64) + 0.5) / R


def _span(R: int, lo: float, hi: float) -> slice:
    """Index range whose voxel centres may lie in [lo, hi] (conservative)."""
    a = max(0, int(math.floor(lo * R - 0.5)) - 1)
    b = min(R, int(math.ceil(hi * R - 0.5)) + 2)
    return slice(a, max(a, b))


def _ellipsoid_into(occ: torch.Tensor, R: int, cen, axes) -> None:
    """occ[i,j,k] |= sum(((centre - cen)/axes)^2) <= 1 over the bounding block."""
    c = _centres(R)
    sl = [_span(R, cen[j] - axes[j], cen[j] + axes[j]) for j in range(3)]
    X, Y, Z = torch.meshgrid(c[sl[0]], c[sl[1]], c[sl[2]], indexing="ij")
    inside = ((X - cen[0]) / axes[0]) ** 2 + ((Y - cen[1]) / axes[1]) ** 2 \
        + ((Z - cen[2]) / axes[2]) ** 2 <= 1.0
    occ[sl[0], sl[1], sl[2]] |= inside


def _sphere_into(occ: torch.Tensor, R: int, cen, r: float) -> None:
    c = _centres(R)
    sl = [_span(R, cen[j] - r, cen[j] + r) for j in range(3)]
    X, Y, Z = torch.meshgrid(c[sl[0]], c[sl[1]], c[sl[2]], indexing="ij")
    inside = (X - cen[0]) ** 2 + (Y - cen[1]) ** 2 + (Z - cen[2]) ** 2 <= r * r
    occ[sl[0], sl[1], sl[2]] |= inside


def make_grid(cfg: Config) -> torch.Tensor:
    """uint8 occupancy, row-major, axis 0 slowest (time first for 4D)."""
    g = cfg.grid
    key = stream_key(cfg.seed, TAG_GRID)
    R = g["R"]
    if g["kind"] == "discs":
        c = _centres(R)
        u = u64d(draws(key, 0, 3 * g["count"])).view(g["count"], 3).tolist()
        occ = torch.zeros(R, R, dtype=torch.bool)
        X, Y = torch.meshgrid(c, c, indexing="ij")
        for k in range(g["count"]):
            cx = 0.2 + 0.6 * u[k][0]
            cy = 0.2 + 0.6 * u[k][1]
            r = 0.03 + 0.09 * u[k][2]
            occ |= (X - cx) ** 2 + (Y - cy) ** 2 <= r * r
        return occ.to(torch.uint8).contiguous()
    if g["kind"] == "ellipsoids":
        u = u64d(draws(key, 0, 6 * g["count"])).view(g["count"], 6).tolist()
        occ = torch.zeros(R, R, R, dtype=torch.bool)
        for k in range(g["count"]):
            cc = [0.15 + 0.7 * u[k][j] for j in range(3)]
            aa = [0.02 + 0.13 * u[k][3 + j] for j in range(3)]
            _ellipsoid_into(occ, R, cc, aa)
        return occ.to(torch.uint8).contiguous()
    if g["kind"] == "moving_spheres":
        F = g["frames"]
        u = u64d(draws(key, 0, 7 * g["count"])).view(g["count"], 7).tolist()
        occ = torch.zeros(F, R, R, R, dtype=torch.bool)
        for f in range(F):
            t = (f + 0.5) / F
            for k in range(g["count"]):
                r = 0.04 + 0.06 * u[k][3]
                cen = []
                for j in range(3):
                    c0 = 0.15 + 0.7 * u[k][j]
                    v = -0.3 + 0.6 * u[k][4 + j]
                    cen.append(min(max(c0 + v * t, r), 1.0 - r))
                _sphere_into(occ[f], R, cen, r)
        return occ.to(torch.uint8).contiguous()
    raise ValueError(g["kind"])


# --------------------------------------------------------------------------
# Query samplers ("r = Uniform()", Alg. 1 line 2; parameterisations
# per Suppl. §3.2).  Records are fp32 rows of record_floats values.
# --------------------------------------------------------------------------
DRAWS_PER_ROW = {"point": None, "ray": 5, "box": 6, "plane": 5}
DRAWS_PER_ROW_2D = {"ray": 3, "box": 4, "plane": 3}  # 2D rays / boxes / lines
DRAWS_PER_ROW_4D = {"ray": 7, "box": 8, "plane": 7}  # 4D rays / boxes / hyperplanes (NEXT-3, R48)


def _draws_per_row(cfg: Config) -> int:
    if cfg.kind == "point":
        return cfg.space_dim
    if cfg.space_dim == 4:
        return DRAWS_PER_ROW_4D[cfg.kind]
    return DRAWS_PER_ROW_2D[cfg.kind] if cfg.space_dim == 2 else DRAWS_PER_ROW[cfg.kind]


def _unit_dirs_2d(u_phi: torch.Tensor) -> torch.Tensor:
    """Uniform directions on the unit circle."""
    phi = 2.0 * math.pi * u_phi.double()
    return torch.stack([torch.cos(phi), torch.sin(phi)], dim=1)


def _unit_dirs(u_z: torch.Tensor, u_phi: torch.Tensor) -> torch.Tensor:
    """Uniform directions on S^2 (Archimedes: z uniform in [-1,1])."""
    z = 2.0 * u_z.double() - 1.0
    phi = 2.0 * math.pi * u_phi.double()
    r = torch.sqrt(torch.clamp(1.0 - z * z, min=0.0))
    return torch.stack([r * torch.cos(phi), r * torch.sin(phi), z], dim=1)


def _unit_dirs_4d(u1: torch.Tensor, u2: torch.Tensor, u3: torch.Tensor) -> torch.Tensor:
    """Uniform directions on S^3 (Shoemake's uniform unit quaternions)."""
    a = torch.sqrt(1.0 - u1.double())
    b = torch.sqrt(u1.double())
    t1 = 2.0 * math.pi * u2.double()
    t2 = 2.0 * math.pi * u3.double()
    return torch.stack([a * torch.sin(t1), a * torch.cos(t1), b * torch.sin(t2), b * torch.cos(t2)], dim=1)


def make_queries(cfg: Config, tag: int, row0: int, n: int, device="cpu") -> torch.Tensor:
    """fp32 [n][record_floats] for rows [row0, row0+n) of stream `tag`."""
    D = _draws_per_row(cfg)
    key = stream_key(cfg.seed, tag)
    u = u32f(draws(key, row0 * D, n * D, device)).view(n, D)
    if cfg.kind == "point":
        return u.contiguous()
    if cfg.space_dim == 4:  # 8-float records over (x, y, z, t) (R48)
        if cfg.kind == "ray":  # origin on the boundary of [0,1]^4, direction uniform on S^3
            facet = torch.clamp((u[:, 0].double() * 8.0).floor().long(), max=7)
            axis, side = facet % 4, (facet // 4).double()
            o = torch.empty(n, 4, dtype=torch.float64, device=device)
            free = [u[:, 1].double(), u[:, 2].double(), u[:, 3].double()]
            for a in range(4):
                others = [b for b in range(4) if b != a]
                m = axis == a
                o[m, a] = side[m]
                for j, b in enumerate(others):
                    o[m, b] = free[j][m]
            d = _unit_dirs_4d(u[:, 4], u[:, 5], u[:, 6])
            return torch.cat([o, d], 1).to(torch.float32).contiguous()
        if cfg.kind == "box":  # c5's box recipe with 4 axes
            lo = u[:, 0:4]
            e = 0.005 + 0.095 * u[:, 4:8].double()
            hi = torch.clamp(lo.double() + e, max=1.0).to(torch.float32)
            return torch.cat([lo, hi], 1).contiguous()
        if cfg.kind == "plane":  # a point of [0,1]^4 and a unit normal on S^3
            nrm = _unit_dirs_4d(u[:, 4], u[:, 5], u[:, 6])
            return torch.cat([u[:, 0:4].double(), nrm], 1).to(torch.float32).contiguous()
    if cfg.space_dim == 2:  # 4-float records: origin on the square's boundary + direction,
        if cfg.kind == "ray":  # lo/hi corners, or a line's point + unit normal
            edge = torch.clamp((u[:, 0].double() * 4.0).floor().long(), max=3)
            axis, side = edge % 2, (edge // 2).double()
            o = torch.empty(n, 2, dtype=torch.float64, device=device)
            for a in range(2):
                m = axis == a
                o[m, a] = side[m]
                o[m, 1 - a] = u[:, 1].double()[m]
            return torch.cat([o, _unit_dirs_2d(u[:, 2])], 1).to(torch.float32).contiguous()
        if cfg.kind == "box":
            lo = u[:, 0:2]
            e = 0.005 + 0.095 * u[:, 2:4].double()
            hi = torch.clamp(lo.double() + e, max=1.0).to(torch.float32)
            return torch.cat([lo, hi], 1).contiguous()
        if cfg.kind == "plane":
            return torch.cat([u[:, 0:2].double(), _unit_dirs_2d(u[:, 2])], 1).to(torch.float32).contiguous()
    if cfg.kind == "ray":
        assert cfg.space_dim == 3
        face = torch.clamp((u[:, 0].double() * 6.0).floor().long(), max=5)
        axis, side = face % 3, (face // 3).double()
        o = torch.empty(n, 3, dtype=torch.float64, device=device)
        free = [u[:, 1].double(), u[:, 2].double()]
        for a in range(3):
            others = [b for b in range(3) if b != a]
            m = axis == a
            o[m, a] = side[m]
            o[m, others[0]] = free[0][m]
            o[m, others[1]] = free[1][m]
        d = _unit_dirs(u[:, 3], u[:, 4])
        return torch.cat([o, d], 1).to(torch.float32).contiguous()
    if cfg.kind == "box":
        assert cfg.space_dim == 3
        lo = u[:, 0:3]
        e = 0.005 + 0.095 * u[:, 3:6].double()
        hi = torch.clamp(lo.double() + e, max=1.0).to(torch.float32)
        return torch.cat([lo, hi], 1).contiguous()
    if cfg.kind == "plane":
        assert cfg.space_dim == 3
        p0 = u[:, 0:3].double()
        nrm = _unit_dirs(u[:, 3], u[:, 4])
        return torch.cat([p0, nrm], 1).to(torch.float32).contiguous()
    raise ValueError(cfg.kind)


def train_batch(cfg: Config, step: int, rank: int = 0, world: int = 1,
                device="cpu") -> torch.Tensor:
    """Queries of training step `step` for `rank` (readings R9/R10).

    c1: rows [(step mod 16)*4096, +4096) of the EVAL set (sequential slices).
    others: fresh rows of the TRAIN stream at counter step*B_global.
    The global batch is split into contiguous, equal rank shards.
    """
    B = cfg.train_batch
    assert B % world == 0
    b = B // world
    if cfg.name == "c1":
        base = (step % (cfg.n_eval // B)) * B
        return make_queries(cfg, TAG_EVAL, base + rank * b, b, device)
    return make_queries(cfg, TAG_TRAIN, step * B + rank * b, b, device)


# --------------------------------------------------------------------------
# Parameters: canonical flat fp32 blob
#   for each hidden layer l: W_l [out][in] row-major, then b_l
#   then w_out [w], b_out; then each exit head (u_k [w], c_k)
# Xavier-uniform weights drawn in blob order from INIT, biases 0.
# --------------------------------------------------------------------------
def layer_dims(cfg: Config) -> list:
    dims = [cfg.record_floats] + [cfg.width] * cfg.hidden_layers
    return list(zip(dims[:-1], dims[1:]))


def num_params(cfg: Config) -> int:
    n = sum((i + 1) * o for i, o in layer_dims(cfg))
    n += cfg.width + 1
    n += cfg.n_heads * (cfg.width + 1)
    return n


def init_params(cfg: Config) -> torch.Tensor:
    key = stream_key(cfg.seed, TAG_INIT)
    out = []
    cursor = 0

    def xavier(fan_in, fan_out, count):
        nonlocal cursor
        a = math.sqrt(6.0 / (fan_in + fan_out))
        u = u64d(draws(key, cursor, count))
        cursor += count
        return ((2.0 * u - 1.0) * a).to(torch.float32)

    for i, o in layer_dims(cfg):
        out.append(xavier(i, o, i * o))
        out.append(torch.zeros(o, dtype=torch.float32))
    out.append(xavier(cfg.width, 1, cfg.width))
    out.append(torch.zeros(1, dtype=torch.float32))
    for _ in range(cfg.n_heads):
        out.append(xavier(cfg.width, 1, cfg.width))
        out.append(torch.zeros(1, dtype=torch.float32))
    p = torch.cat(out).contiguous()
    assert p.numel() == num_params(cfg)
    return p
