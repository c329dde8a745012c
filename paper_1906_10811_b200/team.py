"""Multi-process slab teams: bootstrap plumbing over torch.distributed.

Each rank creates ``Grid(..., rank=r, world=N)`` on its own GPU; this module
exchanges the ranks' export records (cudaIpc handles of the wavefield buffers
and flag words, via ``aw_team_export``) with an all-gather and hands the
concatenation to ``aw_team_connect``.  After that the halo exchange happens
inside the stencil kernels as peer-memory stores (no collective on the data
path).  torch.distributed is plumbing only (works with nccl or gloo).
"""
from __future__ import annotations

from . import _binding


def gather_records(record: bytes, group=None) -> bytes:
    """All-gather equal-size byte records in rank order."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    backend = dist.get_backend(group)
    device = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.frombuffer(bytearray(record), dtype=torch.uint8).to(device)
    out = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    return b"".join(bytes(x.cpu().numpy().tobytes()) for x in out)


def connect(grid: "_binding.Grid", group=None) -> None:
    """Collective: connect `grid` (rank r of a world-N team) to its slab neighbours."""
    import torch.distributed as dist

    if grid.world != dist.get_world_size(group) or grid.rank != dist.get_rank(group):
        raise ValueError("grid rank/world must match the process group")
    grid.team_connect(gather_records(grid.team_export(), group))
    dist.barrier(group)
