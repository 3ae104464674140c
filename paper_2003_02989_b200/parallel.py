"""Multi-GPU batch sharding (one process per GPU, torch.distributed).

The north-star workloads' rows are independent: rank r evaluates the
contiguous row block ``shard_rows(B, r, world)`` on its own GPU and the only
collective is the gather of the per-row outputs -- there is no data-path
exchange.  ``run_sharded`` is backend-agnostic (NCCL on the GPU box, gloo in the
CPU tests).
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def shard_rows(rows: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [start, stop) block of ``rows`` for ``rank``."""
    base, extra = divmod(rows, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def run_sharded(fn, values: np.ndarray, out_cols: int, device=None) -> np.ndarray:
    """Evaluate ``fn(values[start:stop]) -> [rows_local, out_cols]`` on every rank and
    all-gather the row blocks (float64).  Works with world_size 1 without a process group."""
    values = np.asarray(values)
    if not (dist.is_available() and dist.is_initialized()):
        return np.asarray(fn(values), dtype=np.float64).reshape(len(values), out_cols)
    world, rank = dist.get_world_size(), dist.get_rank()
    start, stop = shard_rows(len(values), rank, world)
    local = np.asarray(fn(values[start:stop]), dtype=np.float64).reshape(stop - start, out_cols)
    dev = device if device is not None else torch.device("cpu")
    maxr = -(-len(values) // world)
    buf = torch.zeros((maxr, out_cols), dtype=torch.float64, device=dev)
    buf[: stop - start] = torch.from_numpy(local).to(dev)
    parts = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf)
    out = np.empty((len(values), out_cols))
    for r in range(world):
        s, e = shard_rows(len(values), r, world)
        out[s:e] = parts[r][: e - s].cpu().numpy()
    return out
