"""ctypes binding of the CPU oracle (oracle/_build/libttr_oracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs — never by the product
package paper_2511_03598_b200/.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libttr_oracle.so")

XOSHIRO = 0
PHILOX = 1

ERRC_NAMES = [
    "RankChainMismatch", "BoundaryRankNotOne", "EmptyCoreList", "IndexOutOfRange",
    "DenseTooLarge", "ModeSizeMismatch", "EmptyTermList", "InvalidRankChain", "SVDFailure",
    "InvalidRanks", "NotLeftOrthogonal", "InvalidGrid", "Breakdown", "InvalidArgument", "IoError",
]


class OracleError(RuntimeError):
    def __init__(self, status: int, msg: str):
        self.status = status
        self.errc = ERRC_NAMES[status - 1] if 1 <= status <= 15 else "Internal"
        super().__init__(msg)


def build() -> str:
    """Compile the oracle with its Makefile (g++, no GPU needed)."""
    import subprocess
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = C.CDLL(_LIB_PATH)
        _lib.ttro_last_error.restype = C.c_char_p
        _lib.ttro_tt_destroy.argtypes = [C.c_void_p]
        _lib.ttro_tt_destroy.restype = None
        _lib.ttro_flops_reset.restype = None
        _lib.ttro_flops_get.restype = None
    return _lib


def _check(status: int):
    if status != 0:
        raise OracleError(status, lib().ttro_last_error().decode())


def _i64(seq) -> C.Array:
    arr = (C.c_int64 * len(seq))(*[int(x) for x in seq])
    return arr


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


class TT:
    """Oracle-side TT tensor (owns a C++ ttr_oracle::TT)."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle) if not isinstance(handle, C.c_void_p) else handle

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value and _lib is not None:
            _lib.ttro_tt_destroy(self._h)
            self._h = None

    @staticmethod
    def _new(fn, *args) -> "TT":
        out = C.c_void_p()
        _check(fn(*args, C.byref(out)))
        return TT(out)

    @staticmethod
    def from_cores(cores: Sequence[np.ndarray]) -> "TT":
        """cores[k] has shape (r_{k-1}, n_k, r_k); stored in the reference layout."""
        d = len(cores)
        n = [c.shape[1] for c in cores]
        rl = [c.shape[0] for c in cores]
        rr = [c.shape[2] for c in cores]
        flat = (np.concatenate([np.asarray(c, dtype=np.float64).transpose(2, 1, 0).reshape(-1) for c in cores])
                if d else np.zeros(1))
        flat = np.ascontiguousarray(flat)
        return TT._new(lib().ttro_tt_create_chain, C.c_int64(d), _i64(n), _i64(rl), _i64(rr), _dptr(flat))

    @staticmethod
    def from_flat(d, n, r, flat) -> "TT":
        flat = np.ascontiguousarray(flat, dtype=np.float64)
        return TT._new(lib().ttro_tt_create, C.c_int64(d), _i64(n), _i64(r), _dptr(flat))

    # -- shape / data --------------------------------------------------------
    @property
    def order(self) -> int:
        return lib().ttro_tt_order(self._h)

    def shape(self):
        d = self.order
        n = (C.c_int64 * d)()
        r = (C.c_int64 * (d + 1))()
        dd = C.c_int64()
        tot = C.c_int64()
        _check(lib().ttro_tt_shape(self._h, C.byref(dd), n, r, C.byref(tot)))
        return list(n), list(r), tot.value

    @property
    def ranks(self) -> List[int]:
        return self.shape()[1]

    @property
    def mode_sizes(self) -> List[int]:
        return self.shape()[0]

    def flat(self) -> np.ndarray:
        _, _, tot = self.shape()
        out = np.empty(tot, dtype=np.float64)
        _check(lib().ttro_tt_data(self._h, _dptr(out)))
        return out

    def cores(self) -> List[np.ndarray]:
        n, r, _ = self.shape()
        flat = self.flat()
        out, off = [], 0
        for k in range(len(n)):
            cnt = r[k] * n[k] * r[k + 1]
            out.append(flat[off:off + cnt].reshape(r[k + 1], n[k], r[k]).transpose(2, 1, 0).copy())
            off += cnt
        return out

    def entry(self, idx_one_based: Sequence[int]) -> float:
        v = C.c_double()
        _check(lib().ttro_entry(self._h, _i64(idx_one_based), C.byref(v)))
        return v.value

    def dense(self, max_entries: int = 10_000_000) -> np.ndarray:
        sz = C.c_int64()
        _check(lib().ttro_dense_size(self._h, C.byref(sz)))
        if sz.value > max_entries:
            out = np.empty(1)
        else:
            out = np.empty(sz.value, dtype=np.float64)
        _check(lib().ttro_contract_to_dense(self._h, C.c_int64(max_entries), _dptr(out)))
        return out


# -- constructors ---------------------------------------------------------------

def random_gaussian_tt(modes, ranks, seed) -> TT:
    return TT._new(lib().ttro_random_gaussian_tt, C.c_int64(len(modes)), _i64(modes), _i64(ranks), C.c_uint64(seed))


def synthetic_perturbed_tt(d, n, r, eps, seed) -> TT:
    return TT._new(lib().ttro_synthetic, C.c_int64(d), C.c_int64(n), C.c_int64(r), C.c_double(eps), C.c_uint64(seed))


def two_part_tt(d, n, rx, rz, eps, seed) -> TT:
    return TT._new(lib().ttro_two_part, C.c_int64(d), C.c_int64(n), C.c_int64(rx), C.c_int64(rz),
                   C.c_double(eps), C.c_uint64(seed))


def kernel_sum_tt(d, n, r, terms, ell, seed) -> TT:
    return TT._new(lib().ttro_kernel_sum, C.c_int64(d), C.c_int64(n), C.c_int64(r), C.c_int64(terms),
                   C.c_double(ell), C.c_uint64(seed))


def formal_sum(terms: Sequence[TT]) -> TT:
    arr = (C.c_void_p * len(terms))(*[t._h.value for t in terms])
    return TT._new(lib().ttro_formal_sum, arr, C.c_int(len(terms)))


def scaled(t: TT, alpha: float) -> TT:
    return TT._new(lib().ttro_scaled, t._h, C.c_double(alpha))


def _scalar(fn, *args) -> float:
    v = C.c_double()
    _check(fn(*args, C.byref(v)))
    return v.value


def norm_exact(t: TT) -> float:
    return _scalar(lib().ttro_norm_exact, t._h)


def dot(a: TT, b: TT) -> float:
    return _scalar(lib().ttro_dot, a._h, b._h)


def relative_error(a: TT, b: TT) -> float:
    return _scalar(lib().ttro_relative_error, a._h, b._h)


def orthogonalize(t: TT, right_to_left: bool = True) -> TT:
    return TT._new(lib().ttro_orthogonalize, t._h, C.c_int(1 if right_to_left else 0))


def round_deterministic(t: TT, eps=None, ranks=None) -> TT:
    if ranks is not None:
        return TT._new(lib().ttro_round_det_ranks, t._h, _i64(ranks), C.c_int64(len(ranks)))
    return TT._new(lib().ttro_round_det_tol, t._h, C.c_double(eps))


def round_fixed_krp(t: TT, ranks, seed, rng=XOSHIRO) -> TT:
    return TT._new(lib().ttro_round_fixed_krp, t._h, _i64(ranks), C.c_int64(len(ranks)), C.c_uint64(seed), C.c_int(rng))


def round_adaptive_krp(t: TT, tolerance=1e-6, f_init=0.1, f_inc=0.05, seed=0, rng=XOSHIRO,
                       known_norm: Optional[float] = None, max_rank_cap=None, trace: Optional[dict] = None) -> TT:
    out = C.c_void_p()
    cap = _i64(max_rank_cap) if max_rank_cap is not None else None
    est = (C.c_double * 4096)()
    n_est = C.c_int64()
    tau = C.c_double()
    _check(lib().ttro_round_adaptive_krp(
        t._h, C.c_double(tolerance), C.c_double(f_init), C.c_double(f_inc), C.c_uint64(seed), C.c_int(rng),
        C.c_double(math.nan if known_norm is None else known_norm), cap, C.byref(out), est, C.c_int64(4096),
        C.byref(n_est), C.byref(tau)))
    if trace is not None:
        trace["estimates"] = list(est[: min(4096, n_est.value)])
        trace["tau"] = tau.value
    return TT(out)


def round_rand_orth_tt(t: TT, target_ranks: Sequence[int], seed: int, rng=XOSHIRO) -> TT:
    """round_rand.cpp:66-78 — Rand-Orth with a Gaussian TT sketch (xoshiro: the reference stream)."""
    return TT._new(lib().ttro_round_rand_orth_tt, t._h, _i64(target_ranks), C.c_int64(len(target_ranks)),
                   C.c_uint64(seed), C.c_int(rng))


def tt_partial_contractions(x: TT, r: TT) -> List[np.ndarray]:
    """sketch.cpp:94-109: [W_1 .. W_{d-1}] with W_{k-1} = H(X_k x_3 W_k) H(R_k)^T."""
    _, rx, _ = x.shape()
    _, rr, _ = r.shape()
    d = len(rx) - 1
    shapes = [(rx[k], rr[k]) for k in range(1, d)]
    out = np.empty(sum(a * b for a, b in shapes), dtype=np.float64)
    _check(lib().ttro_tt_partial_contractions(x._h, r._h, _dptr(out)))
    res, o = [], 0
    for a, b in shapes:
        res.append(out[o:o + a * b].reshape(b, a).T.copy())
        o += a * b
    return res


def round_sum_adaptive_krp(terms: Sequence[TT], eps: float, f_inc: float, seed: int, rng=XOSHIRO) -> TT:
    """sum_round.cpp:52-173 — adaptive rounding of sum(terms) without the formal sum."""
    arr = (C.c_void_p * max(1, len(terms)))(*[t._h.value for t in terms])
    return TT._new(lib().ttro_round_sum_adaptive_krp, arr, C.c_int(len(terms)), C.c_double(eps), C.c_double(f_inc),
                   C.c_uint64(seed), C.c_int(rng))


def compression_pass(t: TT, tau: float) -> TT:
    return TT._new(lib().ttro_compression_pass, t._h, C.c_double(tau))


def estimate_norm_krp(t: TT, width, seed, rng=XOSHIRO) -> float:
    return _scalar(lib().ttro_estimate_norm_krp, t._h, C.c_int64(width), C.c_uint64(seed), C.c_int(rng))


def draw_factors(t: TT, start_mode, cols, seed, rng=XOSHIRO, col0=0) -> List[np.ndarray]:
    n, _, _ = t.shape()
    tot = sum(n[k - 1] * cols for k in range(start_mode, len(n) + 1))
    out = np.empty(tot, dtype=np.float64)
    _check(lib().ttro_draw_factors(t._h, C.c_int64(start_mode), C.c_int64(cols), C.c_uint64(seed), C.c_int(rng),
                                   C.c_int64(col0), _dptr(out)))
    res, off = [], 0
    for k in range(start_mode, len(n) + 1):
        cnt = n[k - 1] * cols
        res.append(out[off:off + cnt].reshape(cols, n[k - 1]).T.copy())
        off += cnt
    return res


def krp_contractions(t: TT, factors: Sequence[np.ndarray], start_mode=2) -> List[np.ndarray]:
    n, r, _ = t.shape()
    cols = factors[0].shape[1]
    flat = np.concatenate([np.asarray(f, dtype=np.float64).T.reshape(-1) for f in factors])
    tot = sum(r[k - 1] * cols for k in range(start_mode, len(n) + 1))
    out = np.empty(tot, dtype=np.float64)
    _check(lib().ttro_krp_contractions(t._h, C.c_int64(start_mode), C.c_int64(cols), _dptr(flat), _dptr(out)))
    res, off = [], 0
    for k in range(start_mode, len(n) + 1):
        cnt = r[k - 1] * cols
        res.append(out[off:off + cnt].reshape(cols, r[k - 1]).T.copy())
        off += cnt
    return res


def residual_sketch(t: TT, w0: int, seed: int, rng: int, z: np.ndarray, q: np.ndarray, k: int, b: int):
    """generate_residual_sketch (round_rand.cpp:80-94) after an initial width-w0
    contraction from mode 2: returns (S, widths of W_2..W_d afterwards)."""
    z = np.asfortranarray(z, dtype=np.float64)
    q = np.asfortranarray(q, dtype=np.float64)
    s = np.empty((z.shape[0], b), dtype=np.float64, order="F")
    widths = (C.c_int64 * t.order)()
    _check(lib().ttro_residual_sketch(t._h, C.c_int64(w0), C.c_uint64(seed), C.c_int(rng), C.c_int64(z.shape[0]),
                                      C.c_int64(z.shape[1]), _dptr(z), C.c_int64(q.shape[1]),
                                      _dptr(q) if q.size else None, C.c_int64(k), C.c_int64(b), _dptr(s), widths))
    return s, list(widths)[:t.order - 1]


def residual_norm_estimate(s: np.ndarray, block: int) -> float:
    s = np.asfortranarray(s, dtype=np.float64)
    return _scalar(lib().ttro_residual_norm_estimate, C.c_int64(s.shape[0]), C.c_int64(s.shape[1]),
                   _dptr(s) if s.size else None, C.c_int64(block))


def set_backend(backend: str = "port", threads: int = 0) -> None:
    """Dense-kernel backend of the oracle: "port" (plain-loop restatement, the
    pinned default) or "blas" (the same algorithms on OpenBLAS/LAPACK: dgemm,
    dgeqrf + dorgqr, dgesvd). threads > 0 sizes both the OpenMP and OpenBLAS pools."""
    _check(lib().ttro_set_backend(C.c_int({"port": 0, "blas": 1}[backend]), C.c_int(threads)))


def backend() -> str:
    return ["port", "blas"][lib().ttro_backend()]


def blas_available() -> bool:
    return bool(lib().ttro_blas_available())


class backend_scope:
    """with backend_scope("blas", threads): ... — restores the previous backend."""

    def __init__(self, name: str, threads: int = 0):
        self.name, self.threads = name, threads

    def __enter__(self):
        self.prev = backend()
        set_backend(self.name, self.threads)
        return self

    def __exit__(self, *a):
        set_backend(self.prev, 0)


def random_philox_tt(modes, ranks, seed) -> TT:
    """Bitwise the device generator ttr_tt_random_philox (Philox tags 1000 + k)."""
    return TT._new(lib().ttro_random_philox_tt, C.c_int64(len(modes)), _i64(modes), _i64(ranks), C.c_uint64(seed))


def gaussian_matrix(rows, cols, seed) -> np.ndarray:
    out = np.empty(rows * cols, dtype=np.float64)
    _check(lib().ttro_gaussian_matrix(C.c_int64(rows), C.c_int64(cols), C.c_uint64(seed), _dptr(out)))
    return out.reshape(cols, rows).T.copy()


def derive_seed(seed, tag) -> int:
    v = C.c_uint64()
    lib().ttro_derive_seed(C.c_uint64(seed), C.c_uint64(tag), C.byref(v))
    return v.value


def philox_factor(seed, mode, rows, cols, col0=0) -> np.ndarray:
    out = np.empty(rows * cols, dtype=np.float64)
    _check(lib().ttro_philox_factor(C.c_uint64(seed), C.c_int64(mode), C.c_int64(rows), C.c_int64(cols),
                                    C.c_int64(col0), _dptr(out)))
    return out.reshape(cols, rows).T.copy()


def thin_qr(a: np.ndarray):
    a = np.asfortranarray(a, dtype=np.float64)
    m, n = a.shape
    k = min(m, n)
    q = np.empty((k, m), dtype=np.float64)
    r = np.empty((n, k), dtype=np.float64)
    flat = np.ascontiguousarray(a.T).reshape(-1)
    _check(lib().ttro_thin_qr(C.c_int64(m), C.c_int64(n), _dptr(flat), _dptr(q), _dptr(r)))
    return q.T.copy(), r.T.copy()


def truncated_svd(a: np.ndarray, tau=None, rank=None):
    m, n = a.shape
    k = min(m, n)
    flat = np.ascontiguousarray(np.asarray(a, dtype=np.float64).T).reshape(-1)
    u = np.empty(m * k)
    s = np.empty(k)
    v = np.empty(n * k)
    rk = C.c_int64()
    _check(lib().ttro_truncated_svd(C.c_int64(m), C.c_int64(n), _dptr(flat), C.c_int(1 if tau is not None else 0),
                                    C.c_double(tau or 0.0), C.c_int64(rank or 0), C.byref(rk), _dptr(u), _dptr(s), _dptr(v)))
    kk = rk.value
    return u[: m * kk].reshape(kk, m).T.copy(), s[:kk].copy(), v[: n * kk].reshape(kk, n).T.copy(), kk


def flops_reset():
    lib().ttro_flops_reset()


def flops_get() -> dict:
    arr = (C.c_uint64 * 5)()
    lib().ttro_flops_get(arr)
    return dict(gemm=arr[0], qr=arr[1], svd=arr[2], sketch=arr[3], rng=arr[4], total=arr[0] + arr[1] + arr[2])


# -- TT-GMRES cookie harness (solver.cpp; ttr_oracle_solver.cpp) ------------------

DETERMINISTIC, RAND_ORTH_TT, ADAPTIVE_KRP_SUM = 0, 1, 2


def cookie_problem(p: int, grid: int, samples: int, rho_min: float, rho_max: float):
    """build_cookie_problem (solver.cpp:81-135): (factors[term][mode] as arrays, rhs TT)."""
    modes = [grid * grid] + [samples] * p
    nterms = p + 1
    tot = nterms * sum(m * m for m in modes)
    buf = np.empty(tot, dtype=np.float64)
    h = C.c_void_p()
    _check(lib().ttro_cookie_problem(C.c_int64(p), C.c_int64(grid), C.c_int64(samples), C.c_double(rho_min),
                                     C.c_double(rho_max), _dptr(buf), C.byref(h)))
    terms, off = [], 0
    for _ in range(nterms):
        term = []
        for m in modes:
            term.append(buf[off:off + m * m].reshape(m, m).T.copy())
            off += m * m
        terms.append(term)
    return terms, TT(h)


def apply_operator(terms, t: TT) -> List[TT]:
    """apply_operator (solver.cpp:137-151) of explicit factors terms[i][k]."""
    flat = np.concatenate([np.asarray(a, dtype=np.float64).T.reshape(-1) for term in terms for a in term])
    outs = (C.c_void_p * len(terms))()
    _check(lib().ttro_apply_operator(C.c_int64(len(terms)), _dptr(flat), t._h, outs))
    return [TT(C.c_void_p(outs[i])) for i in range(len(terms))]


def tt_gmres_cookie(p, grid, samples, rho_min, rho_max, rel_tolerance=1e-8, max_iterations=200,
                    strategy=DETERMINISTIC, rounding_tolerance=0.0, seed=0, track_true_residual=True,
                    mean_field_preconditioner=True, rng=XOSHIRO):
    """tt_gmres on build_cookie_problem(p, grid, samples, rho_min, rho_max) -> dict."""
    it = C.c_int64()
    conv = C.c_int()
    rh = np.zeros(max_iterations)
    th = np.zeros(max_iterations)
    kh = np.zeros(max_iterations, dtype=np.int64)
    h = C.c_void_p()
    _check(lib().ttro_gmres_cookie(C.c_int64(p), C.c_int64(grid), C.c_int64(samples), C.c_double(rho_min),
                                   C.c_double(rho_max), C.c_double(rel_tolerance), C.c_int64(max_iterations),
                                   C.c_int(strategy), C.c_double(rounding_tolerance), C.c_uint64(seed),
                                   C.c_int(1 if track_true_residual else 0),
                                   C.c_int(1 if mean_field_preconditioner else 0), C.c_int(rng), C.byref(it),
                                   C.byref(conv), _dptr(rh), _dptr(th), kh.ctypes.data_as(C.c_void_p), C.byref(h)))
    n = it.value
    return {"iterations": n, "converged": bool(conv.value), "residual_history": rh[:n].tolist(),
            "true_residual_history": th[:n].tolist() if track_true_residual else [],
            "max_rank_history": kh[:n].tolist(), "solution": TT(h)}
