"""Host logic of the slab decomposition along x.

Rank r owns x-cells [X_r, X_{r+1}) (R21: positions [X_r Delta, X_{r+1} Delta),
a tie goes to the right).  Uniform slabs for C1-C3; count-balanced slabs from
a per-x-plane particle histogram for the magnetosphere configs (H10).
"""
from __future__ import annotations

from typing import List, Optional, Sequence

import torch


def uniform_bounds(ncell_x: int, nranks: int) -> List[int]:
    if ncell_x < nranks:
        raise ValueError("fewer x cells than ranks")
    return [ncell_x * r // nranks for r in range(nranks + 1)]


def balanced_bounds(plane_counts: Sequence[float], nranks: int, min_width: int = 3) -> List[int]:
    """Cut the x-planes so every rank gets ~1/nranks of the particles, each slab
    at least min_width cells wide (needed for ghost reach)."""
    n = len(plane_counts)
    if n < nranks * min_width:
        raise ValueError("domain too narrow for the requested slabs")
    c = torch.tensor(plane_counts, dtype=torch.float64).cumsum(0)
    total = float(c[-1]) if n else 0.0
    b = [0]
    for r in range(1, nranks):
        target = total * r / nranks
        k = int(torch.searchsorted(c, torch.tensor(target, dtype=torch.float64)).item()) + 1
        k = max(k, b[-1] + min_width)
        k = min(k, n - (nranks - r) * min_width)
        b.append(k)
    b.append(n)
    return b


def owner_of_cells(cx: torch.Tensor, bounds: Sequence[int]) -> torch.Tensor:
    """Rank owning each global x-cell index."""
    bt = torch.tensor(bounds[1:-1], dtype=cx.dtype, device=cx.device)
    return torch.bucketize(cx, bt, right=True)


def broadcast_nccl_id(make_id, group=None) -> bytes:
    """Rank 0 creates the NCCL unique id (pic_nccl_id); every rank returns it."""
    import torch.distributed as dist
    obj = [make_id() if dist.get_rank() == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]
