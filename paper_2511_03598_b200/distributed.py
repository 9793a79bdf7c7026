"""Multi-GPU sharding of the KRP rounding path (one process per GPU).

* Independent tensors (config 5a) need no collective: each rank rounds its own
  slice of the batch (`round_fixed_krp_batched` on a local TTBatch).
* One large tensor (config 5b): `round_fixed_krp_sharded` runs the library's
  sharded driver (csrc/sharded.cu) over a `Communicator`: the KRP sketch is
  column-sharded (Philox draws keyed by the global column, so every slice is
  bitwise the matching columns of a one-GPU contraction) with an NCCL
  all-gather of the W slices, and the Rand-Orth sweep is row-sharded by the
  mode index with a TSQR per mode (all-gather of the l x l R factors, a
  redundant QR of the stack, M = sum_p Q_p^T V_p by all-gather and a
  fixed-order sum). The whole driver — collectives included — is C++ on one
  stream; torch.distributed only broadcasts the NCCL unique id.
  `Communicator.local(ctx, P)` runs P ranks inside this process on one GPU
  with the same code and kernels (the sharded algorithm on one device).
* `rand_orth_row_sharded` below is the same sweep written against a generic
  `ops` backend: the CPU tests run it with numpy/oracle arithmetic over gloo at
  world sizes 2 and 3 (tests/test_distributed.py) as the host-side model of
  the device driver.
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


# ---------------------------------------------------------------------------
# Row-sharded Rand-Orth sweep with an NVLink TSQR (SURVEY §8e, config 5b at
# P GPUs). The rows of V(Y_k) are sharded by the mode index j: rank p owns the
# slices J_p (contiguous rows j*l_{k-1} .. of V(Y_k)). Per mode:
#   S_p = V_p W_{k+1}(:, 1:l)             local GEMM
#   S_p = Q_p R_p                         local Householder QR
#   [R_0; ...; R_{P-1}] = Q_s R           all-gather of the l x l R_p (NCCL),
#                                         redundant QR on every rank (TSQR)
#   Q_k(rows J_p) = Q_p Q_s(p-block)      local GEMM: this rank's rows of core k
#   M = sum_p Q_k(J_p)^T V_p              local GEMM + all-reduce (l x r_k)
#   V_{p}(Y_{k+1}) = M X_{k+1}(:, j, :)   for j in J_p (strided batch): local
# Modes whose local blocks would be shorter than l (mode 1: n rows) run
# replicated. The same orchestration as the device driver (csrc/sharded.cu),
# over a generic `ops` backend: the CPU tests run it with numpy GEMMs, the
# oracle's Householder QR and gloo collectives.

class View:
    """Column-major matrix view: element (i, j) at base[off + i + j*ld]."""
    __slots__ = ("base", "off", "ld", "rows", "cols")

    def __init__(self, base, off, ld, rows, cols):
        self.base, self.off, self.ld, self.rows, self.cols = base, off, ld, rows, cols

    def sub(self, r0: int, nr: int, c0: int, nc: int) -> "View":
        return View(self.base, self.off + r0 + c0 * self.ld, self.ld, nr, nc)


def slice_bounds(n: int, world: int) -> List[int]:
    """Contiguous slices of the mode index: rank p owns j in [b[p], b[p+1])."""
    return [n * p // world for p in range(world + 1)]


def rand_orth_row_sharded(ops, n: Sequence[int], r_in: Sequence[int], r_out: Sequence[int], W, core, rank: int,
                          world: int):
    """Left-to-right Rand-Orth sweep (round_rand.cpp:26-44) with rows sharded
    by the mode index. n: mode sizes (d); r_in: input ranks (d+1); r_out:
    output ranks (the l_eff caps, d+1); W[k]: View of the gathered W_k
    (r_{k-1} x width), k = 2..d; core(k): View of input core k (0-based,
    V-unfolding r_k n_k x r_{k+1}). Returns the full output cores (Views,
    identical on every rank)."""
    d = len(n)
    out = [None] * d
    V = None          # local rows of V(Y_k) (mode k >= 2), or None -> mode 1 uses core 0
    V_rows = None     # slice bounds the local V refers to
    for k in range(1, d):
        l_prev, l, cols = r_out[k - 1], r_out[k], r_in[k]
        nk = n[k - 1]
        sb = slice_bounds(nk, world)
        counts = [(sb[p + 1] - sb[p]) * l_prev for p in range(world)]
        sharded = world > 1 and min(counts) >= l
        Wk = W[k + 1].sub(0, cols, 0, l)
        # ---- this mode's V (full if replicated, local rows if sharded) ----
        if k == 1:
            Vfull = core(0)  # replicated input: (n_0 x r_1), l_prev = 1
            Vp = Vfull.sub(sb[rank], counts[rank], 0, cols) if sharded else Vfull
        else:
            Vp = V if sharded else ops.gather_rows(V, V_rows, world)
        rows_p = Vp.rows
        S = ops.alloc(rows_p, l)
        ops.gemm(False, 1.0, Vp, Wk, 0.0, S)
        if sharded:
            Qp, Rp = ops.qr(S)
            Rs = ops.all_gather_blocks(Rp, world)           # (world*l x l), rank order
            Qs, _ = ops.qr(Rs)
            Qk = ops.alloc(rows_p, l)
            ops.gemm(False, 1.0, Qp, Qs.sub(rank * l, l, 0, l), 0.0, Qk)
        else:
            Qk, _ = ops.qr(S)
        M = ops.alloc(l, cols)
        ops.gemm(True, 1.0, Qk, Vp, 0.0, M)
        if sharded:  # M = sum_p parts in rank order (all-gather + fixed-order sum, as the device driver)
            parts = ops.all_gather_blocks(M, world)  # (world*l x cols)
            ops.sum_blocks(parts, world, M)
            out[k - 1] = ops.gather_rows(Qk, counts, world)
        else:
            out[k - 1] = Qk
        # ---- next: local rows of V(Y_{k+1}) = M X_{k+1}(:, j, :), j in this rank's slices ----
        n1, r1 = n[k], r_in[k + 1]
        sb1 = slice_bounds(n1, world)
        j0, j1 = sb1[rank], sb1[rank + 1]
        nj = j1 - j0
        X = core(k)  # (cols*n1 x r1): element (i, j, g) at i + j*cols + g*cols*n1
        if k < d - 1:
            Vn = ops.alloc(nj * l, r1)
            if nj:
                ops.gemm_batched(1.0, M, 0, View(X.base, X.off + j0 * cols, cols * n1, cols, r1), cols, 0.0,
                                 View(Vn.base, Vn.off, nj * l, l, r1), l, nj)
            V = Vn
            V_rows = [(sb1[p + 1] - sb1[p]) * l for p in range(world)]
        else:
            last = ops.alloc(l, nj)
            if nj:
                ops.gemm(False, 1.0, M, View(X.base, X.off + j0 * cols, cols, cols, nj), 0.0, last)
            # local rows of the last core's V-unfolding (l x n_d): columns j0..j1
            out[d - 1] = ops.gather_rows(View(last.base, last.off, l * max(nj, 1), l * nj, 1),
                                         [(sb1[p + 1] - sb1[p]) * l for p in range(world)], world)
    return out


def fixed_krp_output_ranks(n: Sequence[int], r_in: Sequence[int], targets: Sequence[int]) -> List[int]:
    """l_eff = min(l_k, rows, cols) of V(Y_k) (round_rand.cpp:34-35)."""
    d = len(n)
    r = [1] * (d + 1)
    for k in range(1, d):
        r[k] = min(targets[k - 1], r[k - 1] * n[k - 1], r_in[k])
    return r


class Communicator:
    """ttr_comm: an NCCL communicator over the torch.distributed group (rank 0
    makes the unique id, torch broadcasts it), or `Communicator.local(ctx, P)`:
    P ranks simulated in this process on one device."""

    def __init__(self, handle, ctx, world: int, rank: int, nlocal: int):
        self._h, self.ctx, self.world, self.rank, self.nlocal = handle, ctx, world, rank, nlocal

    @staticmethod
    def from_torch(ctx, group=None) -> "Communicator":
        import torch.distributed as dist
        world = dist.get_world_size(group)
        rank = dist.get_rank(group)
        idbuf = (C.c_uint8 * 128)()
        if rank == 0:
            _check(lib().ttr_comm_unique_id(idbuf))
        obj = [bytes(idbuf)]
        dist.broadcast_object_list(obj, src=0, group=group)
        idbuf = (C.c_uint8 * 128).from_buffer_copy(obj[0])
        h = C.c_void_p()
        _check(lib().ttr_comm_init(ctx._h, C.c_int(world), C.c_int(rank), idbuf, C.byref(h)))
        return Communicator(h, ctx, world, rank, 1)

    @staticmethod
    def local(ctx, world: int) -> "Communicator":
        h = C.c_void_p()
        _check(lib().ttr_comm_init_local(ctx._h, C.c_int(world), C.byref(h)))
        return Communicator(h, ctx, world, 0, world)

    def close(self):
        if getattr(self, "_h", None) and self._h.value and lib() is not None:
            lib().ttr_comm_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        self.close()


def round_fixed_krp_sharded(tt: TTTensor, target_ranks: Sequence[int], seed: int, comm: Communicator,
                            gather: bool = True):
    """Config-5b rounding of ONE tensor over comm.world GPUs (ttr_round_fixed_krp_sharded).
    Every rank passes its replica of the same input. Returns (local, full): local =
    this process's rank slices Y_k(:, J_p, :) of every core (a list, one per local
    rank; entries may be None), full = the all-gathered result (gather=True) or None."""
    n = comm.nlocal
    loc = (C.c_void_p * n)()
    full = C.c_void_p()
    _check(lib().ttr_round_fixed_krp_sharded(tt.ctx._h, comm._h, tt._h, _i64(target_ranks),
                                             C.c_int64(len(target_ranks)), C.c_uint64(seed), C.c_int(int(gather)),
                                             loc, C.byref(full) if gather else None))
    local = [TTTensor(C.c_void_p(loc[q]), tt.ctx) if loc[q] else None for q in range(n)]
    return local, (TTTensor(full, tt.ctx) if gather else None)
