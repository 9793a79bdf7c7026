"""paper_2511_03598_b200 — B200-native randomized TT-rounding with KRP sketches.

Python mirror of the reference `ttround` core/ API for the hot path
(proj/core/include/ttround/{tensor,sketch,round_rand,orthogonalize}.hpp),
bound with ctypes to the C ABI in include/ttround_b200.h
(paper_2511_03598_b200/lib/libttround_b200.so). Every computation runs in the
CUDA library on the device; there is no CPU fallback — importing works
without a GPU (so the build can be checked on a CPU host), but creating a
Context raises TTRoundError(NoDevice) when no CUDA device exists.

Names, argument meaning and error kinds follow the reference:

    TTTensor            <- ttround::TTTensor (tensor.hpp:56-84), device resident
    round_fixed_krp     <- round_rand.hpp:14-15
    round_adaptive_krp  <- round_rand.hpp:31  (AdaptiveConfig :18-25)
    round_deterministic <- orthogonalize.hpp:50,54
    estimate_norm_krp   <- sketch.hpp:63
    krp_partial_contractions_rl <- sketch.hpp:47-48
    norm_exact, relative_error, formal_sum, scaled <- tensor.hpp:172-191
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libttround_b200.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "ttround_b200.h")

RNG_XOSHIRO = 0
RNG_PHILOX = 1

ERRC_NAMES = [
    "RankChainMismatch", "BoundaryRankNotOne", "EmptyCoreList", "IndexOutOfRange",
    "DenseTooLarge", "ModeSizeMismatch", "EmptyTermList", "InvalidRankChain", "SVDFailure",
    "InvalidRanks", "NotLeftOrthogonal", "InvalidGrid", "Breakdown", "InvalidArgument", "IoError",
]
_EXTRA = {100: "Cuda", 101: "OutOfMemory", 102: "Nccl", 103: "Internal", 104: "NoDevice"}


class TTRoundError(RuntimeError):
    """Mirrors ttround::Error: `.code` is the Errc name (types.hpp:15-31)."""

    def __init__(self, status: int, message: str):
        self.status = status
        self.code = ERRC_NAMES[status - 1] if 1 <= status <= 15 else _EXTRA.get(status, "Unknown")
        super().__init__(message)


_lib = None


def build(verbose: bool = False) -> str:
    """Compile libttround_b200.so for sm_100a (nvcc; no GPU needed)."""
    import subprocess
    cmd = ["make", "-C", os.path.join(_HERE, "csrc"), "-j8"]
    subprocess.run(cmd, check=True, stdout=None if verbose else subprocess.DEVNULL)
    return LIB_PATH


def lib():
    """Load the CUDA library (fails loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run paper_2511_03598_b200.build() "
                              "(the product has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        L.ttr_last_error.restype = C.c_char_p
        L.ttr_version.restype = C.c_char_p
        _lib = L
    return _lib


def _check(status: int):
    if status != 0:
        raise TTRoundError(status, lib().ttr_last_error().decode())


def _i64(seq):
    return (C.c_int64 * max(1, len(seq)))(*[int(x) for x in seq])


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


class Counts(C.Structure):
    """flops::Counts (flops.hpp:12-20)."""
    _fields_ = [("gemm", C.c_uint64), ("qr", C.c_uint64), ("svd", C.c_uint64),
                ("sketch", C.c_uint64), ("rng", C.c_uint64)]

    def total(self) -> int:
        return self.gemm + self.qr + self.svd


class _AdaptiveCfg(C.Structure):
    _fields_ = [("tolerance", C.c_double), ("f_init", C.c_double), ("f_inc", C.c_double),
                ("seed", C.c_uint64), ("has_known_norm", C.c_int), ("known_norm", C.c_double),
                ("max_rank_cap", C.POINTER(C.c_int64)), ("max_rank_cap_len", C.c_int64),
                ("rng_mode", C.c_int)]


def _ctx_alive(obj) -> bool:
    ctx = getattr(obj, "ctx", None)
    h = getattr(ctx, "_h", None)
    return bool(h is not None and h.value)


class Context:
    """One CUDA device + stream (ttr_ctx). Pass `stream` (an int handle, e.g.
    torch.cuda.current_stream().cuda_stream) to order work on a caller stream."""

    def __init__(self, device: int = 0, stream: Optional[int] = None):
        self._h = C.c_void_p()
        _check(lib().ttr_ctx_create(C.c_int(device), C.c_void_p(stream) if stream else None, C.byref(self._h)))
        self.device = device
        self.stream = stream  # caller stream handle, or None (library-owned stream)

    def close(self):
        if getattr(self, "_h", None) and self._h.value and _lib is not None:
            _lib.ttr_ctx_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        self.close()

    def set_stream(self, stream: Optional[int]):
        _check(lib().ttr_ctx_set_stream(self._h, C.c_void_p(stream) if stream else None))
        self.stream = stream

    def synchronize(self):
        _check(lib().ttr_ctx_synchronize(self._h))

    def kernel_launches(self) -> int:
        v = C.c_uint64()
        _check(lib().ttr_ctx_kernel_launches(self._h, C.byref(v)))
        return v.value

    def counters(self) -> Counts:
        c = Counts()
        _check(lib().ttr_counters(self._h, C.byref(c)))
        return c

    def reset_counters(self):
        _check(lib().ttr_counters_reset(self._h))


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


class TTTensor:
    """Device-resident TT tensor (ttr_tt). Cores keep the reference layout."""

    def __init__(self, handle: C.c_void_p, ctx: Context):
        self._h = handle
        self.ctx = ctx

    def __del__(self):
        # a tensor outliving its context (garbage-collection order at teardown)
        # is not destroyed: its device memory went with the context
        if getattr(self, "_h", None) and self._h.value and _lib is not None and _ctx_alive(self):
            _lib.ttr_tt_destroy(self._h)
            self._h = C.c_void_p()

    @staticmethod
    def _new(ctx: Context, fn, *args) -> "TTTensor":
        out = C.c_void_p()
        _check(fn(*args, C.byref(out)))
        return TTTensor(out, ctx)

    # -- construction ---------------------------------------------------
    @staticmethod
    def from_flat(mode_sizes: Sequence[int], ranks: Sequence[int], flat: np.ndarray,
                  ctx: Optional[Context] = None) -> "TTTensor":
        """Upload cores given as one flat buffer (core k = its column-major
        vertical unfolding, concatenated)."""
        ctx = ctx or default_context()
        flat = np.ascontiguousarray(flat, dtype=np.float64)
        return TTTensor._new(ctx, lib().ttr_tt_upload, ctx._h, C.c_int64(len(mode_sizes)), _i64(mode_sizes),
                             _i64(ranks), _dptr(flat))

    @staticmethod
    def from_cores(cores: Sequence[np.ndarray], ctx: Optional[Context] = None) -> "TTTensor":
        """TTTensor(std::vector<Core>) (tensor.hpp:63): cores[k] of shape
        (r_{k-1}, n_k, r_k); the constructor's checks (tensor.cpp:66-79, incl. the
        finiteness scan) run in the library (ttr_tt_upload_cores)."""
        ctx = ctx or default_context()
        d = len(cores)
        bufs = [np.ascontiguousarray(np.asarray(c, dtype=np.float64).transpose(2, 1, 0).reshape(-1)) for c in cores]
        ptrs = (C.POINTER(C.c_double) * max(1, d))(*[_dptr(b) for b in bufs])
        rl = [c.shape[0] for c in cores]
        n = [c.shape[1] for c in cores]
        rr = [c.shape[2] for c in cores]
        return TTTensor._new(ctx, lib().ttr_tt_upload_cores, ctx._h, C.c_int64(d), _i64(rl), _i64(n), _i64(rr), ptrs)

    @staticmethod
    def random_gaussian(mode_sizes: Sequence[int], ranks: Sequence[int], seed: int,
                        ctx: Optional[Context] = None) -> "TTTensor":
        """random_gaussian_tt (tensor.cpp:217-242): the reference's xoshiro stream, bitwise."""
        ctx = ctx or default_context()
        return TTTensor._new(ctx, lib().ttr_tt_random_gaussian, ctx._h, C.c_int64(len(mode_sizes)),
                             _i64(mode_sizes), _i64(ranks), C.c_uint64(seed))

    @staticmethod
    def random_philox(mode_sizes: Sequence[int], ranks: Sequence[int], seed: int,
                      ctx: Optional[Context] = None) -> "TTTensor":
        """Gaussian cores N(0, 1/(r n r)) drawn on the device (Philox)."""
        ctx = ctx or default_context()
        return TTTensor._new(ctx, lib().ttr_tt_random_philox, ctx._h, C.c_int64(len(mode_sizes)), _i64(mode_sizes),
                             _i64(ranks), C.c_uint64(seed))

    @staticmethod
    def kernel_sum(d, n, r, terms, ell, seed, ctx: Optional[Context] = None) -> "TTTensor":
        """BASELINE config 4 input (smooth exp(-|t - c_ab|/ell) cores, weights 2^-t), built on the device."""
        ctx = ctx or default_context()
        return TTTensor._new(ctx, lib().ttr_tt_kernel_sum, ctx._h, C.c_int64(d), C.c_int64(n), C.c_int64(r),
                             C.c_int64(terms), C.c_double(ell), C.c_uint64(seed))

    @staticmethod
    def kernel_term(d, n, r, term, ell, seed, ctx: Optional[Context] = None) -> "TTTensor":
        """Term `term` of kernel_sum alone (weight 2^-term): config 4 kept as a TT sum."""
        ctx = ctx or default_context()
        return TTTensor._new(ctx, lib().ttr_tt_kernel_term, ctx._h, C.c_int64(d), C.c_int64(n), C.c_int64(r),
                             C.c_int64(term), C.c_double(ell), C.c_uint64(seed))

    @staticmethod
    def two_part_philox(d, n, rx, rz, eps, seed, ctx: Optional[Context] = None) -> "TTTensor":
        """X/||X|| + eps Z/||Z|| with Gaussian X (ranks rx) and Z (ranks rz) drawn on the device
        from derive_seed(seed, 1) and derive_seed(seed, 2) (BASELINE configs 1, 2, 3, 5b)."""
        from .seeds import derive_seed
        ctx = ctx or default_context()
        kx = [1] + [rx] * (d - 1) + [1]
        kz = [1] + [rz] * (d - 1) + [1]
        x = TTTensor.random_philox([n] * d, kx, derive_seed(seed, 1), ctx)
        z = TTTensor.random_philox([n] * d, kz, derive_seed(seed, 2), ctx)
        x = scaled(x, 1.0 / norm_exact(x))
        z = scaled(z, eps / norm_exact(z))
        return formal_sum([x, z])

    # -- shape / data ---------------------------------------------------
    def shape(self):
        d = C.c_int64()
        _check(lib().ttr_tt_shape(self._h, C.byref(d), None, None, None))
        n = (C.c_int64 * d.value)()
        r = (C.c_int64 * (d.value + 1))()
        tot = C.c_int64()
        _check(lib().ttr_tt_shape(self._h, C.byref(d), n, r, C.byref(tot)))
        return list(n), list(r), tot.value

    @property
    def order(self) -> int:
        return len(self.shape()[0])

    def mode_sizes(self) -> List[int]:
        return self.shape()[0]

    def ranks(self) -> List[int]:
        return self.shape()[1]

    def max_rank(self) -> int:
        return max(self.ranks())

    def flat(self) -> np.ndarray:
        _, _, tot = self.shape()
        out = np.empty(tot, dtype=np.float64)
        _check(lib().ttr_tt_download(self.ctx._h, self._h, _dptr(out)))
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

    @staticmethod
    def read_ttf1(path: str, ctx: Optional[Context] = None) -> "TTTensor":
        """Read a reference TTF1 file (io.cpp:45-76) into a device tensor."""
        ctx = ctx or default_context()
        return TTTensor._new(ctx, lib().ttr_tt_read_ttf1, ctx._h, C.c_char_p(os.fsencode(path)))

    def write_ttf1(self, path: str):
        """Write the tensor as a reference TTF1 file (io.cpp:27-43)."""
        _check(lib().ttr_tt_write_ttf1(self.ctx._h, self._h, C.c_char_p(os.fsencode(path))))

    def core_ptr(self, k: int) -> int:
        p = C.c_void_p()
        _check(lib().ttr_tt_core_ptr(self._h, C.c_int64(k), C.byref(p)))
        return p.value


# ---- TT arithmetic (tensor.hpp:172-191) ----------------------------------------

def formal_sum(terms: Sequence[TTTensor]) -> TTTensor:
    if len(terms) == 0:
        raise TTRoundError(7, "EmptyTermList: formal sum of no terms")
    ctx = terms[0].ctx
    arr = (C.c_void_p * len(terms))(*[t._h.value for t in terms])
    return TTTensor._new(ctx, lib().ttr_tt_formal_sum, ctx._h, arr, C.c_int(len(terms)))


def scaled(tt: TTTensor, alpha: float) -> TTTensor:
    out = formal_sum([tt])
    _check(lib().ttr_tt_scale(out.ctx._h, out._h, C.c_double(alpha)))
    return out


def norm_exact(tt: TTTensor) -> float:
    v = C.c_double()
    _check(lib().ttr_norm_exact(tt.ctx._h, tt._h, C.byref(v)))
    return v.value


def relative_error(a: TTTensor, b: TTTensor) -> float:
    v = C.c_double()
    _check(lib().ttr_relative_error(a.ctx._h, a._h, b._h, C.byref(v)))
    return v.value


# ---- rounding (the hot path) -----------------------------------------------------

def round_fixed_krp(tt: TTTensor, target_ranks: Sequence[int], seed: int, rng: int = RNG_PHILOX) -> TTTensor:
    return TTTensor._new(tt.ctx, lib().ttr_round_fixed_krp, tt.ctx._h, tt._h, _i64(target_ranks),
                         C.c_int64(len(target_ranks)), C.c_uint64(seed), C.c_int(rng))


def _host_ptr(buf) -> int:
    if hasattr(buf, "data_ptr"):
        return buf.data_ptr()
    if isinstance(buf, np.ndarray):
        return buf.ctypes.data
    raise TypeError("host buffer must be a torch tensor or numpy array")


class FixedKrpPlan:
    """CUDA-graph plan of round_fixed_krp for one input buffer (ttr_plan):
    `execute()` replays the captured sweep; `output` is the plan-owned result
    (valid until the plan is closed)."""

    def __init__(self, tt: TTTensor, target_ranks: Sequence[int], seed: int, rng: int = RNG_PHILOX,
                 host_in=None, host_out=None):
        """host_in/host_out (pinned host buffers with the flat input cores / room for
        the flat result; e.g. torch tensors with pin_memory()): the plan also
        streams the input in and the result out, overlapped with the sweep
        (ttr_plan_fixed_krp_host)."""
        self.ctx = tt.ctx
        self.input = tt
        self._h = C.c_void_p()
        self._host = (host_in, host_out)  # keep alive
        if host_in is not None or host_out is not None:
            if host_in is None or host_out is None or rng != RNG_PHILOX:
                raise ValueError("host streaming needs both host buffers and the Philox generator")
            _check(lib().ttr_plan_fixed_krp_host(tt.ctx._h, tt._h, _i64(target_ranks), C.c_int64(len(target_ranks)),
                                                 C.c_uint64(seed), C.c_void_p(_host_ptr(host_in)),
                                                 C.c_void_p(_host_ptr(host_out)), C.byref(self._h)))
        else:
            _check(lib().ttr_plan_fixed_krp(tt.ctx._h, tt._h, _i64(target_ranks), C.c_int64(len(target_ranks)),
                                            C.c_uint64(seed), C.c_int(rng), C.byref(self._h)))
        out = C.c_void_p()
        _check(lib().ttr_plan_output(self._h, C.byref(out)))
        self.output = _BorrowedTT(out, tt.ctx, self)

    def execute(self):
        _check(lib().ttr_plan_execute(self._h))

    def close(self):
        if getattr(self, "_h", None) and self._h.value and _lib is not None and _ctx_alive(self):
            _lib.ttr_plan_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        self.close()


class _BorrowedTT(TTTensor):
    """A TTTensor view owned by someone else (not destroyed on GC)."""

    def __init__(self, handle, ctx, owner):
        super().__init__(handle, ctx)
        self._owner = owner

    def __del__(self):
        pass


def copy_from_host(tt: TTTensor, flat: np.ndarray):
    """Overwrite the cores of `tt` from a host buffer (same shape, reference layout)."""
    flat = np.ascontiguousarray(flat, dtype=np.float64)
    _check(lib().ttr_tt_copy_from_host(tt.ctx._h, tt._h, _dptr(flat)))


class TTBatch:
    """Batch of identically shaped device TT tensors (ttr_batch, config 5a)."""

    def __init__(self, handle, ctx: Context):
        self._h = handle
        self.ctx = ctx

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value and _lib is not None and _ctx_alive(self):
            _lib.ttr_batch_destroy(self._h)
            self._h = C.c_void_p()

    @staticmethod
    def from_flats(mode_sizes, ranks, flats: Sequence[np.ndarray], ctx: Optional[Context] = None) -> "TTBatch":
        ctx = ctx or default_context()
        host = np.ascontiguousarray(np.concatenate([np.asarray(f, dtype=np.float64) for f in flats]))
        out = C.c_void_p()
        _check(lib().ttr_batch_upload(ctx._h, C.c_int64(len(flats)), C.c_int64(len(mode_sizes)), _i64(mode_sizes),
                                      _i64(ranks), _dptr(host), C.byref(out)))
        return TTBatch(out, ctx)

    @staticmethod
    def two_part_philox(batch, d, n, rx, rz, eps, seed, ctx: Optional[Context] = None) -> "TTBatch":
        ctx = ctx or default_context()
        out = C.c_void_p()
        _check(lib().ttr_batch_two_part_philox(ctx._h, C.c_int64(batch), C.c_int64(d), C.c_int64(n), C.c_int64(rx),
                                               C.c_int64(rz), C.c_double(eps), C.c_uint64(seed), C.byref(out)))
        return TTBatch(out, ctx)

    def shape(self):
        b, d = C.c_int64(), C.c_int64()
        _check(lib().ttr_batch_shape(self._h, C.byref(b), C.byref(d), None, None, None))
        n = (C.c_int64 * d.value)()
        r = (C.c_int64 * (d.value + 1))()
        tot = C.c_int64()
        _check(lib().ttr_batch_shape(self._h, C.byref(b), C.byref(d), n, r, C.byref(tot)))
        return b.value, list(n), list(r), tot.value

    def flats(self, first=0, count=None) -> List[np.ndarray]:
        b, _, _, tot = self.shape()
        count = b - first if count is None else count
        out = np.empty(max(1, count * tot), dtype=np.float64)
        _check(lib().ttr_batch_download(self.ctx._h, self._h, C.c_int64(first), C.c_int64(count), _dptr(out)))
        return [out[q * tot:(q + 1) * tot].copy() for q in range(count)]


def round_fixed_krp_batched(batch: TTBatch, target_ranks: Sequence[int], seed: int) -> TTBatch:
    """Tensor b rounded as round_fixed_krp(Y_b, target_ranks, derive_seed(seed, b)) (Philox)."""
    out = C.c_void_p()
    _check(lib().ttr_round_fixed_krp_batched(batch.ctx._h, batch._h, _i64(target_ranks), C.c_int64(len(target_ranks)),
                                             C.c_uint64(seed), C.byref(out)))
    return TTBatch(out, batch.ctx)


@dataclass
class AdaptiveConfig:
    """ttround::AdaptiveConfig (round_rand.hpp:18-25)."""
    tolerance: float = 1e-6
    f_init: float = 0.1
    f_inc: float = 0.05
    seed: int = 0
    known_norm: Optional[float] = None
    max_rank_cap: Optional[Sequence[int]] = None
    rng: int = RNG_PHILOX


def _adaptive_cfg(cfg: AdaptiveConfig):
    c = _AdaptiveCfg()
    c.tolerance, c.f_init, c.f_inc, c.seed = cfg.tolerance, cfg.f_init, cfg.f_inc, cfg.seed
    c.has_known_norm = 1 if cfg.known_norm is not None else 0
    c.known_norm = cfg.known_norm or 0.0
    cap = _i64(cfg.max_rank_cap) if cfg.max_rank_cap is not None else None
    c.max_rank_cap = C.cast(cap, C.POINTER(C.c_int64)) if cap is not None else None
    c.max_rank_cap_len = len(cfg.max_rank_cap) if cfg.max_rank_cap is not None else 0
    c.rng_mode = cfg.rng
    return c, cap


class AdaptiveKrpPlan:
    """CUDA-graph plan of round_adaptive_krp (ttr_plan_adaptive_krp): the growth
    decisions of an eager run are replayed by the graph and re-checked on the
    device; `execute()` re-records when the input's contents decide otherwise.
    `output` re-reads the plan-owned result (its shape may change then)."""

    def __init__(self, tt: TTTensor, cfg: AdaptiveConfig):
        self.ctx = tt.ctx
        self.input = tt
        c, self._cap = _adaptive_cfg(cfg)
        self._h = C.c_void_p()
        _check(lib().ttr_plan_adaptive_krp(tt.ctx._h, tt._h, C.byref(c), C.byref(self._h)))

    @property
    def output(self) -> TTTensor:
        out = C.c_void_p()
        _check(lib().ttr_plan_output(self._h, C.byref(out)))
        return _BorrowedTT(out, self.ctx, self)

    def execute(self):
        _check(lib().ttr_plan_execute(self._h))

    def rerecords(self) -> int:
        v = C.c_int64()
        _check(lib().ttr_plan_rerecords(self._h, C.byref(v)))
        return v.value

    def close(self):
        if getattr(self, "_h", None) and self._h.value and _lib is not None and _ctx_alive(self):
            _lib.ttr_plan_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        self.close()


def round_adaptive_krp(tt: TTTensor, cfg: AdaptiveConfig) -> TTTensor:
    c = _AdaptiveCfg()
    c.tolerance, c.f_init, c.f_inc, c.seed = cfg.tolerance, cfg.f_init, cfg.f_inc, cfg.seed
    c.has_known_norm = 1 if cfg.known_norm is not None else 0
    c.known_norm = cfg.known_norm or 0.0
    cap = _i64(cfg.max_rank_cap) if cfg.max_rank_cap is not None else None
    c.max_rank_cap = C.cast(cap, C.POINTER(C.c_int64)) if cap is not None else None
    c.max_rank_cap_len = len(cfg.max_rank_cap) if cfg.max_rank_cap is not None else 0
    c.rng_mode = cfg.rng
    return TTTensor._new(tt.ctx, lib().ttr_round_adaptive_krp, tt.ctx._h, tt._h, C.byref(c))


def round_rand_orth_tt(tt: TTTensor, target_ranks: Sequence[int], seed: int, rng: int = RNG_PHILOX) -> TTTensor:
    """Rand-Orth with a Gaussian TT sketch (ttr_round_rand_orth_tt; round_rand.cpp:66-78)."""
    return TTTensor._new(tt.ctx, lib().ttr_round_rand_orth_tt, tt.ctx._h, tt._h, _i64(target_ranks),
                         C.c_int64(len(target_ranks)), C.c_uint64(seed), C.c_int(rng))


def compression_pass(tt: TTTensor, tau: float) -> TTTensor:
    """Right-to-left QR + truncated-SVD pass over a left-orthogonal tensor
    (ttr_compression_pass; round_rand.cpp:155-179, the second pass of Adap-R)."""
    return TTTensor._new(tt.ctx, lib().ttr_compression_pass, tt.ctx._h, tt._h, C.c_double(tau))


def round_sum_adaptive_krp(terms: Sequence[TTTensor], eps: float, f_inc: float = 0.05, seed: int = 0,
                           rng: int = RNG_PHILOX) -> TTTensor:
    """Adaptive rounding of sum(terms) without forming the formal sum
    (ttr_round_sum_adaptive_krp; sum_round.cpp:52-173)."""
    if len(terms) == 0:
        raise TTRoundError(7, "EmptyTermList: sum of no TT terms")
    ctx = terms[0].ctx
    arr = (C.c_void_p * len(terms))(*[t._h.value for t in terms])
    return TTTensor._new(ctx, lib().ttr_round_sum_adaptive_krp, ctx._h, arr, C.c_int64(len(terms)), C.c_double(eps),
                         C.c_double(f_inc), C.c_uint64(seed), C.c_int(rng))


def round_deterministic(tt: TTTensor, eps: Optional[float] = None,
                        target_ranks: Optional[Sequence[int]] = None) -> TTTensor:
    if target_ranks is not None:
        return TTTensor._new(tt.ctx, lib().ttr_round_deterministic_ranks, tt.ctx._h, tt._h, _i64(target_ranks),
                             C.c_int64(len(target_ranks)))
    return TTTensor._new(tt.ctx, lib().ttr_round_deterministic_tol, tt.ctx._h, tt._h, C.c_double(eps))


def estimate_norm_krp(tt: TTTensor, width: int, seed: int, rng: int = RNG_PHILOX) -> float:
    v = C.c_double()
    _check(lib().ttr_estimate_norm_krp(tt.ctx._h, tt._h, C.c_int64(width), C.c_uint64(seed), C.c_int(rng),
                                       C.byref(v)))
    return v.value


def dot(a: TTTensor, b: TTTensor) -> float:
    """dot (tensor.cpp:244-256) on the device."""
    v = C.c_double()
    _check(lib().ttr_dot(a.ctx._h, a._h, b._h, C.byref(v)))
    return v.value


class GaussianStream:
    """GaussianStream (rng.hpp:12-35): RNG_XOSHIRO = the reference's sequential
    stream (bitwise); RNG_PHILOX = the device generator (state: next global column)."""

    def __init__(self, seed: int, rng: int = RNG_XOSHIRO):
        self._h = C.c_void_p()
        _check(lib().ttr_stream_create(C.c_uint64(seed), C.c_int(rng), C.byref(self._h)))

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value and _lib is not None:
            _lib.ttr_stream_destroy(self._h)
            self._h = C.c_void_p()


class GaussianFactorSet:
    """GaussianFactorSet (sketch.hpp:13-22): device-resident Omega_start..Omega_d."""

    def __init__(self, handle, ctx: Context, mode_sizes: Sequence[int]):
        self._h, self.ctx, self._n = handle, ctx, list(mode_sizes)

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value and _lib is not None and _ctx_alive(self):
            _lib.ttr_factors_destroy(self._h)
            self._h = C.c_void_p()

    def _shape(self):
        a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
        _check(lib().ttr_factors_shape(self._h, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    @property
    def start_mode(self) -> int:
        return self._shape()[0]

    def cols(self) -> int:
        return self._shape()[2]

    def at_mode(self, k: int) -> np.ndarray:
        rows = self._n[k - 1]
        out = np.empty(rows * self.cols(), dtype=np.float64)
        _check(lib().ttr_factors_download(self.ctx._h, self._h, C.c_int64(k), _dptr(out)))
        return out.reshape(self.cols(), rows).T.copy()


def draw_gaussian_factors(tt: TTTensor, start_mode: int, cols: int, stream: GaussianStream) -> GaussianFactorSet:
    out = C.c_void_p()
    _check(lib().ttr_draw_gaussian_factors(tt.ctx._h, tt._h, C.c_int64(start_mode), C.c_int64(cols), stream._h,
                                           C.byref(out)))
    return GaussianFactorSet(out, tt.ctx, tt.mode_sizes())


def append_gaussian_columns(factors: GaussianFactorSet, extra: int, stream: GaussianStream) -> None:
    _check(lib().ttr_append_gaussian_columns(factors.ctx._h, factors._h, C.c_int64(extra), stream._h))


class PartialContractionSet:
    """PartialContractionSet (sketch.hpp:35-44): device-resident W_start..W_d."""

    def __init__(self, handle, ctx: Context):
        self._h, self.ctx = handle, ctx

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value and _lib is not None and _ctx_alive(self):
            _lib.ttr_contractions_destroy(self._h)
            self._h = C.c_void_p()

    @property
    def start_mode(self) -> int:
        s = C.c_int64()
        _check(lib().ttr_contractions_shape(self._h, C.c_int64(0), C.byref(s), None, None, None))
        return s.value

    def at_mode(self, k: int) -> np.ndarray:
        rows, cols = C.c_int64(), C.c_int64()
        _check(lib().ttr_contractions_shape(self._h, C.c_int64(k), None, None, C.byref(rows), C.byref(cols)))
        out = np.empty(max(1, rows.value * cols.value), dtype=np.float64)
        _check(lib().ttr_contractions_download(self.ctx._h, self._h, C.c_int64(k), _dptr(out)))
        return out[:rows.value * cols.value].reshape(cols.value, rows.value).T.copy()


def append_krp_contractions(w: PartialContractionSet, tt: TTTensor, fresh: GaussianFactorSet) -> None:
    _check(lib().ttr_append_krp_contractions(tt.ctx._h, w._h, tt._h, fresh._h))


def generate_residual_sketch(tt: TTTensor, z: np.ndarray, q: np.ndarray, w: PartialContractionSet, k: int, b: int,
                             stream: GaussianStream) -> np.ndarray:
    """generate_residual_sketch (round_rand.cpp:80-94) on the device; z, q host matrices."""
    z = np.asfortranarray(z, dtype=np.float64)
    q = np.asfortranarray(q, dtype=np.float64)
    rows = z.shape[0]
    out = np.empty((rows, max(b, 0)), dtype=np.float64, order="F")
    _check(lib().ttr_generate_residual_sketch(tt.ctx._h, tt._h, C.c_int64(rows), C.c_int64(z.shape[1]), _dptr(z),
                                              C.c_int64(q.shape[1]), _dptr(q) if q.size else None, w._h,
                                              C.c_int64(k), C.c_int64(b), stream._h, _dptr(out)))
    return out


def residual_norm_estimate(s: np.ndarray, block: int, ctx: Optional[Context] = None) -> float:
    """residual_norm_estimate (sketch.cpp:121-124): ||S||_F / sqrt(block), on the device."""
    ctx = ctx or default_context()
    s = np.asfortranarray(s, dtype=np.float64)
    v = C.c_double()
    _check(lib().ttr_residual_norm_estimate(ctx._h, C.c_int64(s.shape[0]), C.c_int64(s.shape[1]),
                                            _dptr(s) if s.size else None, C.c_int64(block), C.byref(v)))
    return v.value


def krp_partial_contractions_rl(tt: TTTensor, cols, factors: Optional[Sequence[np.ndarray]] = None,
                                seed: int = 0, start_mode: int = 2, col0: int = 0):
    """krp_partial_contractions_rl (sketch.cpp:67-78). With a GaussianFactorSet as the
    second argument: the reference call, returning a device PartialContractionSet.
    Otherwise the flat helper: W_start..W_d (r_{k-1} x cols) as host arrays, with
    `factors` = Omega_start..Omega_d (n_k x cols) or None for device Philox factors of
    global columns col0..col0+cols."""
    if isinstance(cols, GaussianFactorSet):
        out = C.c_void_p()
        _check(lib().ttr_krp_partial_contractions_rl(tt.ctx._h, tt._h, cols._h, C.byref(out)))
        return PartialContractionSet(out, tt.ctx)
    n, r, _ = tt.shape()
    d = len(n)
    if factors is not None:
        flat = np.concatenate([np.asarray(f, dtype=np.float64).T.reshape(-1) for f in factors])
        fptr = _dptr(flat)
    else:
        flat, fptr = None, None
    tot = sum(r[k - 1] * cols for k in range(start_mode, d + 1))
    out = np.empty(max(tot, 1), dtype=np.float64)
    _check(lib().ttr_krp_partial_contractions(tt.ctx._h, tt._h, C.c_int64(start_mode), C.c_int64(cols), fptr,
                                              C.c_uint64(seed), C.c_int64(col0), _dptr(out)))
    res, off = [], 0
    for k in range(start_mode, d + 1):
        cnt = r[k - 1] * cols
        res.append(out[off:off + cnt].reshape(cols, r[k - 1]).T.copy())
        off += cnt
    return res


def philox_factor(seed: int, mode: int, rows: int, cols: int, col0: int = 0,
                  ctx: Optional[Context] = None) -> np.ndarray:
    ctx = ctx or default_context()
    out = np.empty(rows * cols, dtype=np.float64)
    _check(lib().ttr_philox_factor(ctx._h, C.c_uint64(seed), C.c_int64(mode), C.c_int64(rows), C.c_int64(cols),
                                   C.c_int64(col0), _dptr(out)))
    return out.reshape(cols, rows).T.copy()


def thin_qr(a: np.ndarray, ctx: Optional[Context] = None):
    ctx = ctx or default_context()
    m, n = a.shape
    k = min(m, n)
    flat = np.ascontiguousarray(np.asarray(a, dtype=np.float64).T).reshape(-1)
    q = np.empty(m * k)
    r = np.empty(k * n)
    _check(lib().ttr_thin_qr(ctx._h, C.c_int64(m), C.c_int64(n), _dptr(flat), _dptr(q), _dptr(r)))
    return q.reshape(k, m).T.copy(), r.reshape(n, k).T.copy()


def thin_qr_speculative(a: np.ndarray, ctx: Optional[Context] = None):
    """thin_qr with the sweep's speculation tag set: the blocked Householder QR may
    take the Cholesky-QR panels (qr_chol.cu K4d/K4f). Returns (q, r, breakdown);
    on breakdown q and r are unspecified (the sweep reruns on the Householder panels)."""
    ctx = ctx or default_context()
    m, n = a.shape
    k = min(m, n)
    flat = np.ascontiguousarray(np.asarray(a, dtype=np.float64).T).reshape(-1)
    q = np.empty(m * k)
    r = np.empty(k * n)
    bd = C.c_int(0)
    _check(lib().ttr_thin_qr_speculative(ctx._h, C.c_int64(m), C.c_int64(n), _dptr(flat), _dptr(q), _dptr(r),
                                         C.byref(bd)))
    return q.reshape(k, m).T.copy(), r.reshape(n, k).T.copy(), bool(bd.value)


def thin_qr_cholesky(a: np.ndarray, ctx: Optional[Context] = None):
    """sCQR3 on the device (qr_chol.cu): (q, r, breakdown)."""
    ctx = ctx or default_context()
    m, n = a.shape
    flat = np.ascontiguousarray(np.asarray(a, dtype=np.float64).T).reshape(-1)
    q = np.empty(m * n)
    r = np.empty(n * n)
    bd = C.c_int(0)
    _check(lib().ttr_thin_qr_cholesky(ctx._h, C.c_int64(m), C.c_int64(n), _dptr(flat), _dptr(q), _dptr(r),
                                      C.byref(bd)))
    return q.reshape(n, m).T.copy(), r.reshape(n, n).T.copy(), bool(bd.value)


def thin_qr_cholesky_batched(a: np.ndarray, ctx: Optional[Context] = None):
    """Batched sCQR3 on the device (qr_chol.cu K4e) of a (batch, m, n) array:
    (q of the same shape, per-matrix breakdown flags)."""
    ctx = ctx or default_context()
    bsz, m, n = a.shape
    flat = np.ascontiguousarray(np.swapaxes(np.asarray(a, dtype=np.float64), 1, 2)).reshape(-1)
    q = np.empty(bsz * m * n)
    flags = np.zeros(bsz, dtype=np.int32)
    _check(lib().ttr_thin_qr_cholesky_batched(ctx._h, C.c_int64(m), C.c_int64(n), C.c_int64(bsz), _dptr(flat),
                                              _dptr(q), flags.ctypes.data_as(C.POINTER(C.c_int))))
    return np.swapaxes(q.reshape(bsz, n, m), 1, 2).copy(), flags.astype(bool)


def gemm(a: np.ndarray, b: np.ndarray, trans_a: bool = False, ctx: Optional[Context] = None) -> np.ndarray:
    ctx = ctx or default_context()
    if trans_a:
        k, m = a.shape
    else:
        m, k = a.shape
    n = b.shape[1]
    fa = np.ascontiguousarray(np.asarray(a, dtype=np.float64).T).reshape(-1)
    fb = np.ascontiguousarray(np.asarray(b, dtype=np.float64).T).reshape(-1)
    out = np.empty(m * n)
    _check(lib().ttr_gemm(ctx._h, C.c_int(1 if trans_a else 0), C.c_int64(m), C.c_int64(n), C.c_int64(k),
                          _dptr(fa), _dptr(fb), _dptr(out)))
    return out.reshape(n, m).T.copy()


# ---- TT-GMRES cookie harness (solver.hpp; csrc/tt_gmres.cu) -------------------------

GMRES_DETERMINISTIC, GMRES_RAND_ORTH_TT, GMRES_ADAPTIVE_KRP_SUM = 0, 1, 2


class _GmresCfg(C.Structure):
    _fields_ = [("rel_tolerance", C.c_double), ("max_iterations", C.c_int64), ("strategy", C.c_int),
                ("rounding_tolerance", C.c_double), ("seed", C.c_uint64), ("track_true_residual", C.c_int),
                ("mean_field_preconditioner", C.c_int), ("rng_mode", C.c_int)]


class _GmresResult(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("converged", C.c_int), ("rounding_seconds", C.c_double),
                ("residual_history", C.POINTER(C.c_double)), ("true_residual_history", C.POINTER(C.c_double)),
                ("max_rank_history", C.POINTER(C.c_int64)), ("rounding_seconds_history", C.POINTER(C.c_double))]


class KronOp:
    """KroneckerSumOperator on the device (solver.hpp:12-21): terms[i][k] = A_{i,k}."""

    def __init__(self, handle: C.c_void_p, ctx: Context, nterms: int, modes: Sequence[int]):
        self._h = handle
        self.ctx = ctx
        self.nterms = nterms
        self.modes = list(modes)

    @staticmethod
    def of(terms, ctx: Optional[Context] = None) -> "KronOp":
        ctx = ctx or default_context()
        modes = [np.asarray(a).shape[0] for a in terms[0]]
        flat = np.concatenate([np.asarray(a, dtype=np.float64).T.reshape(-1) for term in terms for a in term])
        h = C.c_void_p()
        _check(lib().ttr_kron_op_create(ctx._h, C.c_int64(len(terms)), C.c_int64(len(modes)), _i64(modes),
                                        _dptr(flat), C.byref(h)))
        return KronOp(h, ctx, len(terms), modes)

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            lib().ttr_kron_op_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        self.close()


def cookie_problem(num_param_modes: int, grid_size: int, num_param_samples: int, rho_min: float, rho_max: float,
                   ctx: Optional[Context] = None):
    """build_cookie_problem (solver.hpp:32-40): (KronOp, rhs TTTensor)."""
    ctx = ctx or default_context()
    ho, ht = C.c_void_p(), C.c_void_p()
    _check(lib().ttr_cookie_problem(ctx._h, C.c_int64(num_param_modes), C.c_int64(grid_size),
                                    C.c_int64(num_param_samples), C.c_double(rho_min), C.c_double(rho_max),
                                    C.byref(ho), C.byref(ht)))
    modes = [grid_size * grid_size] + [num_param_samples] * num_param_modes
    return KronOp(ho, ctx, num_param_modes + 1, modes), TTTensor(ht, ctx)


def apply_operator(op: KronOp, x: TTTensor) -> List[TTTensor]:
    """apply_operator (solver.hpp:42-44): the terms of the TTSum A x."""
    outs = (C.c_void_p * op.nterms)()
    _check(lib().ttr_apply_operator(op.ctx._h, op._h, x._h, outs))
    return [TTTensor(C.c_void_p(outs[i]), op.ctx) for i in range(op.nterms)]


def tt_gmres(op: KronOp, rhs: TTTensor, rel_tolerance: float = 1e-8, max_iterations: int = 200,
             strategy: int = GMRES_DETERMINISTIC, rounding_tolerance: float = 0.0, seed: int = 0,
             track_true_residual: bool = True, mean_field_preconditioner: bool = True, rng: int = RNG_XOSHIRO):
    """tt_gmres (solver.hpp:80-82) on the device -> dict like GMRESResult."""
    cfg = _GmresCfg(rel_tolerance, max_iterations, strategy, rounding_tolerance, seed, 1 if track_true_residual else 0,
                    1 if mean_field_preconditioner else 0, rng)
    rh = np.zeros(max_iterations)
    th = np.zeros(max_iterations)
    kh = np.zeros(max_iterations, dtype=np.int64)
    sh = np.zeros(max_iterations)
    res = _GmresResult(0, 0, 0.0, rh.ctypes.data_as(C.POINTER(C.c_double)), th.ctypes.data_as(C.POINTER(C.c_double)),
                       kh.ctypes.data_as(C.POINTER(C.c_int64)), sh.ctypes.data_as(C.POINTER(C.c_double)))
    h = C.c_void_p()
    _check(lib().ttr_tt_gmres(op.ctx._h, op._h, rhs._h, C.byref(cfg), C.byref(res), C.byref(h)))
    n = res.iterations
    return {"iterations": n, "converged": bool(res.converged), "residual_history": rh[:n].tolist(),
            "true_residual_history": th[:n].tolist() if track_true_residual else [],
            "max_rank_history": kh[:n].tolist(), "rounding_seconds": res.rounding_seconds,
            "rounding_seconds_history": sh[:n].tolist(),
            "solution": TTTensor(h, op.ctx)}
