"""NEXT-4: many shots -- independent sources over the same model.

Seismic surveys fire many shots (sources) into one velocity model; each shot
is an independent forward problem, and the FWI gradient of the survey is the
sum of the per-shot gradients ("seismic inversion problems";
SURVEY §8(f) NEXT-4 reading: replicas, no exchange during propagation).  On
B200 the shots are sharded across GPUs, one process per GPU: every rank runs
its shots through its own grid handle (the C ABI, no peer exchange), and the
only collective is one all-reduce (sum) of the rank-local gradient and misfit
at the end -- over NCCL/NVLink with the nccl backend.

Canonical order (DESIGN.md §3 Q27): on each rank the gradients of its shots
are summed in the rank's shot order inside the library (AW_OPT_FWI_ACCUMULATE,
fp32 adds of the finalised per-shot gradients); ranks are then summed by the
all-reduce (fp32, NCCL's order), so a multi-rank sum agrees with the
single-rank sum to fp32 rounding, not bit for bit.

This module is host-side plumbing only (shot assignment, the per-shot calls,
the all-reduce); every numerical step runs in libaw's kernels.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

from . import _binding


@dataclass
class Shot:
    """One shot: source positions [ns][ndim] (fp64) and their wavelet [nt][ns] (fp32, host or device)."""
    src_coords: np.ndarray
    wavelet: object
    d_obs: object = None  # observed traces [nt][nr] for FWI (host or device), or None


def assign(nshots: int, world: int, rank: int) -> List[int]:
    """Round-robin shot ids of `rank` (shots of similar cost interleave across ranks)."""
    if world < 1 or not 0 <= rank < world or nshots < 0:
        raise ValueError("bad shot assignment arguments")
    return list(range(rank, nshots, world))


def forward(grid: "_binding.Grid", shots: Sequence[Shot], ids: Sequence[int], nt: int, dt: float,
            traces_out: Optional[list] = None) -> list:
    """Run the shots `ids` one after another on `grid` (reset + sources + nt steps each); returns the
    traces [nt][nr] of each shot (numpy arrays, or the caller's buffers in traces_out)."""
    out = []
    for k, i in enumerate(ids):
        grid.reset()
        grid.add_sources(shots[i].src_coords, shots[i].wavelet)
        grid.run(nt, dt)
        buf = traces_out[k] if traces_out is not None else None
        out.append(grid.read_receivers(out=buf))
    return out


def fwi_gradient(grid: "_binding.Grid", shots: Sequence[Shot], ids: Sequence[int], nt: int, dt: float,
                 grad=None, group=None):
    """Sum over the shots `ids` of the FWI gradients (aw_fwi_gradient) accumulated in the library, then
    (if torch.distributed is initialised) all-reduced over `group`.  Returns (grad, J) with J the
    summed misfit.  `grad` may be a torch tensor on the grid's device (kept there, all-reduced in
    place over NCCL) or None (a host numpy array is returned)."""
    grid.set_option(_binding.AW_OPT_FWI_ACCUMULATE, 1)  # (re)arms and clears the accumulator
    J = 0.0
    if grad is None:
        grad = np.zeros(grid.shape, np.float32)
    for i in ids:
        grid.add_sources(shots[i].src_coords, shots[i].wavelet)
        _, _, j = grid.fwi_gradient(nt, dt, shots[i].d_obs, grad=grad, want_residual=False)
        J += j
    grid.set_option(_binding.AW_OPT_FWI_ACCUMULATE, 0)
    if not ids:  # a rank without shots contributes zeros
        if hasattr(grad, "zero_"):
            grad.zero_()
        else:
            grad[...] = 0.0
    return _allreduce(grad, J, group)


def _allreduce(grad, J: float, group=None):
    try:
        import torch.distributed as dist
    except ImportError:  # pragma: no cover
        return grad, J
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return grad, J
    import torch
    backend = dist.get_backend(group)
    # NCCL reduces device tensors only; gloo host tensors only: stage through the right side
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    src = grad if hasattr(grad, "data_ptr") else torch.from_numpy(grad)
    t = src if src.device == dev else src.to(dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    if t is not src:
        src.copy_(t)  # numpy grad: src shares its memory
    jt = torch.tensor([J], dtype=torch.float64, device=t.device)
    dist.all_reduce(jt, op=dist.ReduceOp.SUM, group=group)
    return grad, float(jt.item())
