"""Host-side plumbing of the data-parallel path.

One process per GPU.  Queries shard into contiguous, balanced row ranges; the
library's NCCL communicator (nb_comm_init) is created from a unique id that
rank 0 draws and the torch process group broadcasts.  Inside libnb the only
exchanges are one allreduce per call: counts (sum), calibration keys (min),
training gradient (sum).
"""
from __future__ import annotations

import numpy as np


TILE = 128  # rows per MMA tile; shard starts are tile multiples


def shard(n: int, rank: int, world: int, align: int = TILE) -> tuple[int, int]:
    """Contiguous shard [start, start+count) of n rows for `rank`.

    Starts are multiples of `align` rows (whole 128-row tiles, so every rank's
    q and y views stay 16-byte aligned for the kernels' bulk copies, nb.h
    "Alignment"); the tiles are balanced (counts differ by at most one tile)
    and the last rank takes the ragged tail."""
    if world < 1 or not 0 <= rank < world or n < 0 or align < 1:
        raise ValueError("bad shard arguments")
    tiles = -(-n // align)
    base, extra = divmod(tiles, world)
    t0 = rank * base + min(rank, extra)
    t1 = t0 + base + (1 if rank < extra else 0)
    start, end = min(n, t0 * align), min(n, t1 * align)
    return start, end - start


def comm_init(model, group=None) -> None:
    """Create the model's NCCL communicator across the torch process group."""
    import torch.distributed as dist

    from . import comm_unique_id

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    uid = [comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0, group=group)
    model.comm_init(uid[0], rank, world)


# Order-preserving map between fp32 and uint32 used for the calibration
# minimum (min over keys == key of the min), the same bijection nb_calibrate
# applies on the device before its allreduce(min).
def float_key(x: np.ndarray) -> np.ndarray:
    b = np.ascontiguousarray(x, np.float32).view(np.uint32)
    return np.where(b & 0x80000000, ~b, b | 0x80000000).astype(np.uint32)


def key_float(k: np.ndarray) -> np.ndarray:
    k = np.ascontiguousarray(k, np.uint32)
    b = np.where(k & 0x80000000, k & 0x7FFFFFFF, ~k).astype(np.uint32)
    return b.view(np.float32)
