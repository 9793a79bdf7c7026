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
# replicated. The same orchestration runs over any `ops` backend: DeviceOps
# (the library's DMMA GEMM / Householder QR through the C ABI on torch CUDA
# buffers, NCCL collectives) here, a numpy backend in the CPU tests.

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


class DeviceOps:
    """Device backend: torch CUDA buffers as storage, the library's kernels for
    the arithmetic (ttr_dev_gemm / ttr_dev_gemm_batched / ttr_dev_thin_qr on
    the context stream = torch's current stream), torch.distributed (NCCL) for
    the collectives."""

    def __init__(self, ctx, group=None):
        import torch
        self.ctx, self.group, self.torch = ctx, group, torch
        self.L = lib()

    def alloc(self, rows: int, cols: int) -> View:
        t = self.torch.zeros(max(1, rows * cols), dtype=self.torch.float64, device="cuda")
        return View(t, 0, max(1, rows), rows, cols)

    def ptr(self, v: View) -> int:
        base = v.base if isinstance(v.base, int) else v.base.data_ptr()
        return base + 8 * v.off

    def gemm(self, ta: bool, alpha: float, A: View, B: View, beta: float, Cm: View):
        k = A.rows if ta else A.cols
        _check(self.L.ttr_dev_gemm(self.ctx._h, C.c_int(int(ta)), C_i64(Cm.rows), C_i64(Cm.cols), C_i64(k),
                                   C_dbl(alpha), C_vp(self.ptr(A)), C_i64(A.ld), C_vp(self.ptr(B)), C_i64(B.ld),
                                   C_dbl(beta), C_vp(self.ptr(Cm)), C_i64(Cm.ld)))

    def gemm_batched(self, alpha, A, sA, B, sB, beta, Cv, sC, batch):
        _check(self.L.ttr_dev_gemm_batched(self.ctx._h, C.c_int(0), C_i64(Cv.rows), C_i64(Cv.cols), C_i64(A.cols), C_dbl(alpha),
                                           C_vp(self.ptr(A)), C_i64(A.ld), C_i64(sA), C_vp(self.ptr(B)), C_i64(B.ld),
                                           C_i64(sB), C_dbl(beta), C_vp(self.ptr(Cv)), C_i64(Cv.ld), C_i64(sC),
                                           C_i64(batch)))

    def qr(self, A: View):
        m, n = A.rows, A.cols
        k = min(m, n)
        Q, R = self.alloc(m, k), self.alloc(k, n)
        _check(self.L.ttr_dev_thin_qr(self.ctx._h, C_i64(m), C_i64(n), C_vp(self.ptr(A)), C_i64(A.ld),
                                      C_vp(self.ptr(Q)), C_i64(Q.ld), C_vp(self.ptr(R)), C_i64(R.ld)))
        return Q, R

    def all_gather_blocks(self, block: View, world: int) -> View:
        """Stack the ranks' (b x c) blocks row-wise: (world*b x c)."""
        torch = self.torch
        b, c = block.rows, block.cols
        mine = self.contiguous(block)
        if world == 1:
            return mine
        out = torch.empty(world * b * c, dtype=torch.float64, device="cuda")
        import torch.distributed as dist
        dist.all_gather_into_tensor(out, mine.base[:b * c], group=self.group)
        st = out.view(world, c, b).permute(1, 0, 2).contiguous().view(-1)  # column j: block 0 rows, block 1 rows...
        return View(st, 0, world * b, world * b, c)

    def all_reduce(self, v: View, world: int):
        if world == 1:
            return
        import torch.distributed as dist
        assert v.off == 0 and v.ld == v.rows
        dist.all_reduce(v.base[:v.rows * v.cols], group=self.group)

    def contiguous(self, v: View) -> View:
        if not isinstance(v.base, int) and v.off == 0 and v.ld == v.rows:
            return v
        out = self.alloc(v.rows, v.cols)
        self.copy(v, out)
        return out

    def copy(self, src: View, dst: View):
        # 2-D strided copy through torch views of the underlying storage (plumbing)
        s = self._tview(src)
        d = self._tview(dst)
        d.copy_(s)

    def _tview(self, v: View):
        if isinstance(v.base, int):
            raise TypeError("raw pointer views are read through the library only")
        return self.torch.as_strided(v.base, (v.cols, v.rows), (v.ld, 1), v.off)

    def gather_rows(self, local: View, counts: List[int], world: int) -> View:
        """All-gather row blocks of different heights (counts[p] rows each, same
        column count) into the full matrix, in rank order."""
        torch = self.torch
        c = local.cols
        full_rows = sum(counts)
        if world == 1:
            return self.contiguous(local)
        import torch.distributed as dist
        mx = max(counts)
        pad = self.alloc(mx, c)
        if local.rows:
            self.copy(local, pad.sub(0, local.rows, 0, c))
        out = torch.empty(world * mx * c, dtype=torch.float64, device="cuda")
        dist.all_gather_into_tensor(out, pad.base[:mx * c], group=self.group)
        full = self.alloc(full_rows, c)
        r0 = 0
        for p in range(world):
            blk = View(out, p * mx * c, mx, counts[p], c)
            if counts[p]:
                self.copy(blk, full.sub(r0, counts[p], 0, c))
            r0 += counts[p]
        return full


def C_i64(v):
    return C.c_int64(int(v))


def C_dbl(v):
    return C.c_double(float(v))


def C_vp(v):
    return C.c_void_p(int(v))


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
        if sharded:
            ops.all_reduce(M, world)
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


def round_fixed_krp_row_sharded(tt: TTTensor, target_ranks: Sequence[int], seed: int, group=None,
                                rank: Optional[int] = None, world: Optional[int] = None) -> TTTensor:
    """Config-5b multi-GPU rounding with BOTH phases sharded: column-sharded KRP
    sketch + NCCL all-gather of the W slices, then the row-sharded Rand-Orth
    sweep with the NVLink TSQR (rand_orth_row_sharded). Every rank passes its
    replica of the same input and receives the full result."""
    import torch
    import torch.distributed as dist
    if world is None:
        world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    if rank is None:
        rank = dist.get_rank(group) if world > 1 else 0
    n, r_in, _ = tt.shape()
    d = len(n)
    width = max(target_ranks)
    r_out = fixed_krp_output_ranks(n, r_in, target_ranks)

    def core(k):
        rows = r_in[k] * n[k]
        return View(tt.core_ptr(k), 0, rows, rows, r_in[k + 1])

    # the library and torch (buffers, NCCL) must share one stream
    cur = torch.cuda.current_stream().cuda_stream
    prev = tt.ctx.stream
    if prev != cur:
        tt.ctx.set_stream(cur)
    try:
        bounds = column_bounds(width, world)
        bufs, lds = sketch_buffers(tt, width)
        c0, c1 = bounds[rank], bounds[rank + 1]
        if c1 > c0:
            sketch_slice_into(tt, bufs, lds, c0, c1 - c0, seed)
        for b in bufs:
            gather_columns(b, bounds, rank, world, group)
        W = {k: View(bufs[k - 2].view(-1), 0, lds[k - 2], r_in[k - 1], width) for k in range(2, d + 1)}
        ops = DeviceOps(tt.ctx, group)
        cores = rand_orth_row_sharded(ops, n, r_in, r_out, W, core, rank, world)
        flat = torch.cat([ops.contiguous(v).base[:v.rows * v.cols] for v in cores])
        out = C.c_void_p()
        _check(lib().ttr_tt_from_device(tt.ctx._h, C.c_int64(d), _i64(n), _i64(r_out), C.c_void_p(flat.data_ptr()),
                                        C.byref(out)))
        tt.ctx.synchronize()
    finally:
        if prev != cur:
            tt.ctx.set_stream(prev)
    return TTTensor(out, tt.ctx)
