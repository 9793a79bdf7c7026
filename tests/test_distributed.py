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


def test_column_sharded_sketch_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
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
