"""Multi-GPU sharding of the KRP rounding path (one process per GPU,
torch.distributed over NCCL/NVLink as plumbing).

* Independent tensors (config 5a) need no collective: each rank rounds its own
  slice of the batch (`round_fixed_krp_batched` on a local TTBatch).
* One large tensor (config 5b): KRP sketch columns are independent
  (W_{k-1}(:, c) depends only on W_k(:, c) and Omega_k(:, c), sketch.cpp:19-23),
  so rank p contracts the global columns [c_p, c_{p+1}) on its replica of the
  input (ttr_krp_sketch_into; Philox draws keyed by the global column make the
  slice bitwise equal to those columns of a single-GPU contraction), the slices
  of every W_k are all-gathered over NCCL, and the left-to-right Rand-Orth sweep
  runs from the gathered sketch (ttr_round_fixed_krp_from_sketch). The sweep is
  replicated in this version (each rank ends with the full result).
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence, Tuple

from . import TTTensor, _check, _i64, lib


def column_bounds(width: int, world: int) -> List[int]:
    """Contiguous, as-equal-as-possible column slices: slice p = [b[p], b[p+1])."""
    return [width * p // world for p in range(world + 1)]


def gather_columns(local, bounds: Sequence[int], rank: int, world: int, group=None):
    """All-gather row blocks [bounds[p], bounds[p+1]) of a (width, ld) tensor.

    `local` is the full-size (width, ld) tensor whose rows of this rank's slice
    are filled; returns the tensor with every rank's rows filled. Works on any
    torch.distributed backend (gloo tests on CPU, NCCL on GPU)."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return local
    chunk = max(bounds[p + 1] - bounds[p] for p in range(world))
    ld = local.shape[1]
    mine = torch.zeros((chunk, ld), dtype=local.dtype, device=local.device)
    n_mine = bounds[rank + 1] - bounds[rank]
    mine[:n_mine] = local[bounds[rank]:bounds[rank + 1]]
    allv = torch.empty((world * chunk, ld), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(allv, mine, group=group)
    for p in range(world):
        n_p = bounds[p + 1] - bounds[p]
        local[bounds[p]:bounds[p + 1]] = allv[p * chunk:p * chunk + n_p]
    return local


def sketch_buffers(tt: TTTensor, width: int):
    """Device buffers for W_2..W_d as torch tensors of shape (width, ld_k):
    row c of buffer k is column c of W_k (column-major r_{k-1} x width)."""
    import torch
    _, r, _ = tt.shape()
    d = len(r) - 1
    bufs, lds = [], []
    for k in range(2, d + 1):
        ld = r[k - 1] + (r[k - 1] & 1)
        bufs.append(torch.zeros((width, ld), dtype=torch.float64, device="cuda"))
        lds.append(ld)
    return bufs, lds


def sketch_slice_into(tt: TTTensor, bufs, lds, col0: int, ncols: int, seed: int):
    ptrs = (C.c_void_p * len(bufs))(*[b.data_ptr() for b in bufs])
    _check(lib().ttr_krp_sketch_into(tt.ctx._h, tt._h, C.c_int64(col0), C.c_int64(ncols), C.c_uint64(seed), ptrs,
                                     _i64(lds)))


def round_from_sketch(tt: TTTensor, target_ranks: Sequence[int], bufs, lds, width: int) -> TTTensor:
    ptrs = (C.c_void_p * len(bufs))(*[b.data_ptr() for b in bufs])
    out = C.c_void_p()
    _check(lib().ttr_round_fixed_krp_from_sketch(tt.ctx._h, tt._h, _i64(target_ranks), C.c_int64(len(target_ranks)),
                                                 ptrs, _i64(lds), C.c_int64(width), C.byref(out)))
    return TTTensor(out, tt.ctx)


def round_fixed_krp_column_sharded(tt: TTTensor, target_ranks: Sequence[int], seed: int, group=None,
                                   rank: Optional[int] = None, world: Optional[int] = None
                                   ) -> Tuple[TTTensor, dict]:
    """Config-5b multi-GPU rounding: column-sharded KRP sketch + NCCL all-gather
    of the W slices + Rand-Orth sweep. Every rank passes its replica of the same
    input; returns (result, timings-free info)."""
    import torch.distributed as dist
    if world is None:
        world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    if rank is None:
        rank = dist.get_rank(group) if world > 1 else 0
    width = max(target_ranks)
    bounds = column_bounds(width, world)
    bufs, lds = sketch_buffers(tt, width)
    c0, c1 = bounds[rank], bounds[rank + 1]
    if c1 > c0:
        sketch_slice_into(tt, bufs, lds, c0, c1 - c0, seed)
    for b in bufs:
        gather_columns(b, bounds, rank, world, group)
    out = round_from_sketch(tt, target_ranks, bufs, lds, width)
    return out, {"bounds": bounds, "width": width}
