"""Multi-GPU sharding logic. The column-sharded sketch of config 5b is checked
(a) on CPU with the gloo backend at world size 2 — every rank computes its KRP
column slice with the oracle and the slices are all-gathered by the same
`gather_columns` the GPU path uses — and (b) on one GPU, where slices computed
separately through the C ABI and swept must reproduce round_fixed_krp bitwise."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, result_q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import py_oracle as O
    from paper_2511_03598_b200.distributed import column_bounds, gather_columns
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    x = O.random_gaussian_tt([6, 5, 7, 4], [1, 3, 5, 2, 1], 21)
    n, r, _ = x.shape()
    width, seed = 11, 9
    bounds = column_bounds(width, world)
    c0, c1 = bounds[rank], bounds[rank + 1]
    # this rank's slice: Philox factors for the GLOBAL columns c0..c1
    fac = [O.philox_factor(seed, k, n[k - 1], c1 - c0, c0) for k in range(2, len(n) + 1)]
    w_slice = O.krp_contractions(x, fac)
    full = []
    for k, wk in zip(range(2, len(n) + 1), w_slice):
        buf = torch.zeros((width, r[k - 1]), dtype=torch.float64)
        buf[c0:c1] = torch.from_numpy(wk.T.copy())
        full.append(gather_columns(buf, bounds, rank, world).numpy().T.copy())
    if rank == 0:
        fac_all = [O.philox_factor(seed, k, n[k - 1], width, 0) for k in range(2, len(n) + 1)]
        ref = O.krp_contractions(x, fac_all)
        result_q.put(all(np.array_equal(a, b) for a, b in zip(full, ref)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_column_sharded_sketch_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    ok = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert ok, "gathered column slices differ from the one-shot contraction"
    assert all(p.exitcode == 0 for p in procs)


def test_column_bounds_cover_width():
    from paper_2511_03598_b200.distributed import column_bounds
    for width in (1, 7, 320):
        for world in (1, 2, 3, 8):
            b = column_bounds(width, world)
            assert b[0] == 0 and b[-1] == width and all(b[i] <= b[i + 1] for i in range(world))


@pytest.mark.gpu
def test_column_sharded_path_matches_single_gpu_bitwise():
    import sys
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import py_oracle as O
    import paper_2511_03598_b200 as P
    from paper_2511_03598_b200.distributed import column_bounds, round_from_sketch, sketch_buffers, sketch_slice_into
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = P.Context(0, stream.cuda_stream)
    x = O.two_part_tt(6, 32, 20, 40, 1e-6, 1005)
    n, r, _ = x.shape()
    y = P.TTTensor.from_flat(n, r, x.flat(), ctx)
    ranks, width, seed = [24] * 5, 24, 7
    bufs, lds = sketch_buffers(y, width)
    b = column_bounds(width, 3)  # three "ranks" without a collective
    for p in range(3):
        sketch_slice_into(y, bufs, lds, b[p], b[p + 1] - b[p], seed)
    sharded = round_from_sketch(y, ranks, bufs, lds, width)
    single = P.round_fixed_krp(y, ranks, seed)
    torch.cuda.synchronize()
    assert sharded.ranks() == single.ranks()
    assert np.array_equal(sharded.flat(), single.flat())


# ---- row-sharded Rand-Orth sweep (NVLink TSQR), CPU stand-in backend -----------------

class NumpyOps:
    """CPU backend for rand_orth_row_sharded: numpy GEMMs, the oracle's
    Householder QR, gloo collectives — the same orchestration the GPU runs."""

    def __init__(self, O, group=None):
        self.O, self.group = O, group

    def alloc(self, rows, cols):
        from paper_2511_03598_b200.distributed import View
        return View(np.zeros(max(1, rows * cols)), 0, max(1, rows), rows, cols)

    @staticmethod
    def mat(v):
        return np.lib.stride_tricks.as_strided(v.base[v.off:], shape=(v.rows, v.cols), strides=(8, 8 * v.ld))

    def gemm(self, ta, alpha, A, B, beta, Cm):
        a = self.mat(A).T if ta else self.mat(A)
        c = self.mat(Cm)
        c[...] = alpha * (a @ self.mat(B)) + (beta * c if beta != 0.0 else 0.0)

    def gemm_batched(self, alpha, A, sA, B, sB, beta, Cv, sC, batch):
        from paper_2511_03598_b200.distributed import View
        for b in range(batch):
            self.gemm(False, alpha, View(A.base, A.off + b * sA, A.ld, A.rows, A.cols),
                      View(B.base, B.off + b * sB, B.ld, B.rows, B.cols), beta,
                      View(Cv.base, Cv.off + b * sC, Cv.ld, Cv.rows, Cv.cols))

    def qr(self, A):
        q, r = self.O.thin_qr(np.array(self.mat(A)))
        Q, R = self.alloc(*q.shape), self.alloc(*r.shape)
        self.mat(Q)[...] = q
        self.mat(R)[...] = r
        return Q, R

    def contiguous(self, v):
        out = self.alloc(v.rows, v.cols)
        self.mat(out)[...] = self.mat(v)
        return out

    def all_gather_blocks(self, block, world):
        from paper_2511_03598_b200.distributed import View
        b, c = block.rows, block.cols
        mine = torch.from_numpy(np.ascontiguousarray(self.mat(block).T).reshape(-1))  # column-major
        parts = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(parts, mine, group=self.group)
        st = np.concatenate([p.numpy().reshape(c, b) for p in parts], axis=1).reshape(-1)  # (c, world*b)
        return View(st, 0, world * b, world * b, c)

    def sum_blocks(self, stacked, world, out):
        """out = sum_p stacked[p*b:(p+1)*b, :] in rank order (the device driver's fixed-order sum)."""
        b = out.rows
        m = self.mat(stacked)
        acc = m[0:b].copy()
        for p in range(1, world):
            acc = acc + m[p * b:(p + 1) * b]
        self.mat(out)[...] = acc

    def gather_rows(self, local, counts, world):
        from paper_2511_03598_b200.distributed import View
        c = local.cols
        mx = max(counts)
        pad = np.zeros((c, mx))
        pad[:, :local.rows] = self.mat(local).T
        parts = [torch.empty(c * mx, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(pad.reshape(-1)), group=self.group)
        full = np.concatenate([p.numpy().reshape(c, mx)[:, :counts[q]] for q, p in enumerate(parts)], axis=1)
        return View(np.ascontiguousarray(full).reshape(-1), 0, sum(counts), sum(counts), c)


def _row_worker(rank, world, port, result_q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import py_oracle as O
    from paper_2511_03598_b200.distributed import View, fixed_krp_output_ranks, rand_orth_row_sharded
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    x = O.two_part_tt(5, 8, 6, 10, 1e-6, 31)
    n, r_in, _ = x.shape()
    targets, seed = [12] * 4, 7
    width = max(targets)
    fac = [O.philox_factor(seed, k, n[k - 1], width, 0) for k in range(2, len(n) + 1)]
    w = O.krp_contractions(x, fac)
    W = {k: View(np.asfortranarray(wk).reshape(-1, order="F"), 0, wk.shape[0], wk.shape[0], width)
         for k, wk in zip(range(2, len(n) + 1), w)}
    flat = x.flat()
    offs = np.cumsum([0] + [r_in[k] * n[k] * r_in[k + 1] for k in range(len(n))])

    def core(k):
        rows = r_in[k] * n[k]
        return View(flat, int(offs[k]), rows, rows, r_in[k + 1])

    r_out = fixed_krp_output_ranks(n, r_in, targets)
    cores = rand_orth_row_sharded(NumpyOps(O), n, r_in, r_out, W, core, rank, world)
    y_flat = np.concatenate([NumpyOps.mat(v).reshape(-1, order="F") for v in cores])
    y = O.TT.from_flat(len(n), n, r_out, y_flat)
    ref = O.round_fixed_krp(x, targets, seed, rng=O.PHILOX)
    err = O.relative_error(ref, y)
    gathered = [None] * world
    dist.all_gather_object(gathered, y_flat.tobytes())
    if rank == 0:
        result_q.put((err, r_out == ref.ranks, all(g == gathered[0] for g in gathered)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_row_sharded_sweep_gloo(world):
    """The TSQR row-sharded sweep (mode 1 replicated, modes >= 2 sharded) on 2 and
    3 CPU ranks (3 does not divide n = 8: uneven slice ownership) reproduces the
    oracle's round_fixed_krp to 1e-10 with identical ranks, and every rank ends
    with the same tensor."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_row_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    err, ranks_ok, same = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert ranks_ok
    assert same
    assert err <= 1e-10, err
    assert all(p.exitcode == 0 for p in procs)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 2, 3])
def test_sharded_library_path_local_ranks(world):
    """The library's sharded driver (csrc/sharded.cu) with `world` ranks simulated on
    one GPU (ttr_comm_init_local: the same code, kernels and fixed-order sums as the
    NCCL run): column-sharded sketch, TSQR row-sharded sweep. The gathered result
    equals the oracle's round_fixed_krp to 1e-10 with identical ranks (world 3 does
    not divide n = 16: uneven slices); world 1 is bitwise round_fixed_krp; the local
    shards are the index slices Y(J_p, ..., J_p) of the gathered tensor; two runs
    are bitwise equal."""
    import sys
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import py_oracle as O
    from helpers import rel_err_vs_ref, to_device
    import paper_2511_03598_b200 as P
    from paper_2511_03598_b200.distributed import Communicator, round_fixed_krp_sharded, slice_bounds
    x = O.two_part_tt(6, 16, 10, 30, 1e-6, 41)
    xd = to_device(x)
    comm = Communicator.local(xd.ctx, world)
    local, full = round_fixed_krp_sharded(xd, [24] * 5, 7, comm)
    ref = O.round_fixed_krp(x, [24] * 5, 7, rng=O.PHILOX)
    assert full.ranks() == ref.ranks
    assert rel_err_vs_ref(ref, full) <= 1e-10
    _, again = round_fixed_krp_sharded(xd, [24] * 5, 7, comm)
    assert np.array_equal(again.flat(), full.flat())
    if world == 1:
        assert np.array_equal(full.flat(), P.round_fixed_krp(xd, [24] * 5, 7).flat())
    cores = full.cores()
    for p, lt in enumerate(local):
        for k, c in enumerate(lt.cores()):
            sb = slice_bounds(cores[k].shape[1], world)
            assert np.array_equal(c, cores[k][:, sb[p]:sb[p + 1], :])
    comm.close()


@pytest.mark.gpu
def test_nccl_communicator_world1():
    """The NCCL communicator loads and runs (world size 1 on this one-GPU box): its
    all-gather copies, and the sharded driver over it is bitwise round_fixed_krp."""
    import sys
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import ctypes as C
    import py_oracle as O
    from helpers import to_device
    import paper_2511_03598_b200 as P
    from paper_2511_03598_b200.distributed import Communicator, round_fixed_krp_sharded
    if not dist.is_initialized():
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1)
    x = O.two_part_tt(5, 12, 8, 20, 1e-6, 43)
    xd = to_device(x)
    comm = Communicator.from_torch(xd.ctx)
    src = torch.arange(10, dtype=torch.float64, device="cuda")
    dst = torch.zeros(10, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    ptrs = (C.c_void_p * 1)(src.data_ptr())
    P._check(P.lib().ttr_comm_all_gather(xd.ctx._h, comm._h, ptrs, C.c_int64(10), C.c_void_p(dst.data_ptr())))
    xd.ctx.synchronize()
    assert torch.equal(src, dst)
    _, full = round_fixed_krp_sharded(xd, [16] * 4, 7, comm)
    assert np.array_equal(full.flat(), P.round_fixed_krp(xd, [16] * 4, 7).flat())
    comm.close()
    dist.destroy_process_group()
