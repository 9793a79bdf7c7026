"""Shared helpers: move tensors between the oracle (CPU checker) and the
device library, and compare them in TT arithmetic (tensor.cpp:264-268)."""
import numpy as np


def to_device(ott, ctx=None):
    import paper_2511_03598_b200 as P
    n, r, _ = ott.shape()
    return P.TTTensor.from_flat(n, r, ott.flat(), ctx)


def to_oracle(dtt):
    import py_oracle as O
    n, r, _ = dtt.shape()
    return O.TT.from_flat(len(n), n, r, dtt.flat())


def rel_err_vs_ref(y_ref, y_gpu):
    """||Y_gpu - Y_ref|| / ||Y_ref|| via the oracle's stable formal difference."""
    import py_oracle as O
    return O.relative_error(y_ref, to_oracle(y_gpu))


def left_orth_defect(cores):
    worst = 0.0
    for c in cores[:-1]:
        rl, n, rr = c.shape
        v = c.reshape(rl * n, rr, order="F")  # V(j*rl + i, g) = X(i, j, g)
        g = v.T @ v - np.eye(rr)
        worst = max(worst, np.linalg.norm(g))
    return worst
