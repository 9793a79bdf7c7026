"""GPU parity tests: the CUDA library (through its C ABI) against the CPU
oracle on identical inputs. Tolerances are the reference's own
(tests/test_sketch.cpp, test_round_rand.cpp, test_orthogonalize.cpp) or the
north-star bar (||Y_gpu - Y_ref|| / ||Y_ref|| <= 1e-10, identical ranks)."""
import numpy as np
import pytest

from helpers import left_orth_defect, rel_err_vs_ref, to_device, to_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2511_03598_b200 as P
    return P


@pytest.fixture(scope="module")
def O():
    import py_oracle as O
    return O


# ---- dense kernels ---------------------------------------------------------------

@pytest.mark.parametrize("m,n,k,ta", [(7, 5, 3, False), (130, 70, 33, False), (1000, 320, 1000, False),
                                      (33, 65, 4001, True), (320, 1000, 40960, True), (257, 129, 16, True),
                                      (64, 1, 640, False)])
def test_gemm_matches_numpy(P, m, n, k, ta):
    rng = np.random.default_rng(m * 7 + n)
    a = rng.standard_normal((k, m) if ta else (m, k))
    b = rng.standard_normal((k, n))
    c = P.gemm(a, b, trans_a=ta)
    ref = (a.T if ta else a) @ b
    assert np.linalg.norm(c - ref) <= 1e-13 * np.sqrt(k) * np.linalg.norm(np.abs(a)) * np.linalg.norm(np.abs(b)) + 1e-300


@pytest.mark.parametrize("m,n", [(6, 3), (64, 64), (320, 20), (300, 15), (7040, 110), (2000, 70), (40, 60),
                                 (80000, 8), (160000, 40),  # these two exceed one panel grid: TSQR split
                                 (40960, 32), (5000, 20), (2049, 33), (4097, 5), (40960, 320), (9000, 45)])
def test_thin_qr(P, m, n):
    rng = np.random.default_rng(m + 13 * n)
    a = rng.standard_normal((m, n))
    q, r = P.thin_qr(a)
    k = min(m, n)
    assert q.shape == (m, k) and r.shape == (k, n)
    assert np.linalg.norm(q.T @ q - np.eye(k)) <= 1e-12 * np.sqrt(k)
    assert np.linalg.norm(q @ r - a) <= 1e-13 * np.sqrt(m * n) * np.linalg.norm(a)
    assert np.allclose(np.tril(r, -1), 0.0)


@pytest.mark.parametrize("m,n,rank", [(320, 60, 16), (5000, 96, 40), (50, 20, 0), (40960, 32, 10), (9000, 70, 0),
                                      (7040, 110, 64), (3000, 20, 19)])
def test_thin_qr_rank_deficient_is_orthonormal(P, m, n, rank):
    """linalg.hpp:22 — Q is orthonormal even for rank-deficient input."""
    rng = np.random.default_rng(5)
    a = rng.standard_normal((m, rank)) @ rng.standard_normal((rank, n)) if rank else np.zeros((m, n))
    q, r = P.thin_qr(a)
    assert np.all(np.isfinite(q))
    assert np.linalg.norm(q.T @ q - np.eye(n)) <= 1e-10
    assert np.linalg.norm(q @ r - a) <= 1e-12 * max(1.0, np.linalg.norm(a))


@pytest.mark.parametrize("m,n", [(40960, 64), (7040, 110), (4000, 20)])
def test_thin_qr_graded_columns(P, m, n):
    """Sketch-like conditioning (singular values 1 .. 1e-12): Q stays orthonormal
    to working precision and A = QR holds (tall panels take the TSQR route)."""
    rng = np.random.default_rng(m + n)
    u, _ = np.linalg.qr(rng.standard_normal((m, n)))
    v, _ = np.linalg.qr(rng.standard_normal((n, n)))
    a = (u * np.logspace(0, -12, n)) @ v.T
    q, r = P.thin_qr(a)
    assert np.linalg.norm(q.T @ q - np.eye(n)) <= 1e-12 * np.sqrt(n)
    assert np.linalg.norm(q @ r - a) <= 1e-13 * np.sqrt(m * n) * np.linalg.norm(a)


# ---- K4c: shifted Cholesky QR (the sweep's speculative QR) ---------------------------

@pytest.mark.parametrize("m,n", [(7040, 110), (40960, 320), (25600, 400), (2000, 70), (16384, 320), (300, 33),
                                 (5000, 144), (5000, 145), (100, 100), (6400, 416)])
@pytest.mark.parametrize("graded", [False, True])
def test_thin_qr_cholesky(P, m, n, graded):
    """sCQR3: orthonormal Q, A = QR, R upper, no breakdown for kappa up to 1e12,
    and the same basis as the Householder QR up to column signs."""
    rng = np.random.default_rng(m + 7 * n + graded)
    if graded:
        u, _ = np.linalg.qr(rng.standard_normal((m, n)))
        v, _ = np.linalg.qr(rng.standard_normal((n, n)))
        a = (u * np.logspace(0, -12, n)) @ v.T
    else:
        a = rng.standard_normal((m, n))
    q, r, breakdown = P.thin_qr_cholesky(a)
    assert not breakdown
    assert np.linalg.norm(q.T @ q - np.eye(n)) <= 1e-12 * np.sqrt(n)
    assert np.linalg.norm(q @ r - a) <= 1e-13 * np.sqrt(m * n) * np.linalg.norm(a)
    assert np.allclose(np.tril(r, -1), 0.0)
    if not graded:
        qh, _ = P.thin_qr(a)
        signs = np.sign(np.sum(q * qh, axis=0))
        assert np.all(np.abs(signs) == 1)
        assert np.linalg.norm(q - qh * signs) <= 1e-11 * np.sqrt(n)


@pytest.mark.parametrize("m,n,rank", [(7040, 110, 64), (40960, 320, 128), (500, 40, 0), (3000, 60, 59)])
def test_thin_qr_cholesky_rank_deficient(P, m, n, rank):
    """Exactly rank-deficient input: either the breakdown flag is raised (the
    caller redoes the call with Householder) or the result is still a valid
    thin QR — orthonormal Q (any completion of the range) and A = QR."""
    rng = np.random.default_rng(3)
    a = rng.standard_normal((m, rank)) @ rng.standard_normal((rank, n)) if rank else np.zeros((m, n))
    q, r, breakdown = P.thin_qr_cholesky(a)
    if rank == 0:
        assert breakdown
    if not breakdown:
        assert np.linalg.norm(q.T @ q - np.eye(n)) <= 1e-12 * np.sqrt(n)
        assert np.linalg.norm(q @ r - a) <= 1e-13 * np.sqrt(m * n) * max(1.0, np.linalg.norm(a))


@pytest.mark.parametrize("m,n", [(320, 20), (256, 20), (64, 8), (101, 13), (512, 32), (40, 20), (1024, 17), (16, 16), (21, 20)])
def test_thin_qr_cholesky_batched(P, m, n):
    """Batched CholeskyQR2 / sCQR3 (K4e): per matrix orthonormal Q with A = Q Q^T A
    for well-conditioned, graded (kappa 1e6: CQR2) and ill-conditioned (kappa
    1e11: CQR2 breaks down, the kernel redoes the matrix as sCQR3) members; exactly
    rank-deficient and zero members raise their flag or still give a valid basis."""
    rng = np.random.default_rng(m * 31 + n)
    mats = []
    for kind in ("gauss", "graded", "ill", "gauss", "rankdef", "zero", "ill", "gauss"):
        if kind == "gauss":
            a = rng.standard_normal((m, n))
        elif kind in ("graded", "ill"):
            u, _ = np.linalg.qr(rng.standard_normal((m, n)))
            v, _ = np.linalg.qr(rng.standard_normal((n, n)))
            a = (u * np.logspace(0, -6 if kind == "graded" else -11, n)) @ v.T
        elif kind == "rankdef":
            a = rng.standard_normal((m, n // 2)) @ rng.standard_normal((n // 2, n))
        else:
            a = np.zeros((m, n))
        mats.append((kind, a))
    q, flags = P.thin_qr_cholesky_batched(np.stack([a for _, a in mats]))
    for b, (kind, a) in enumerate(mats):
        if kind == "zero":
            assert flags[b]
        if kind in ("gauss", "graded", "ill"):
            assert not flags[b], (b, kind)
        if not flags[b]:
            assert np.linalg.norm(q[b].T @ q[b] - np.eye(n)) <= 1e-12 * np.sqrt(n), (b, kind)
            assert np.linalg.norm(q[b] @ (q[b].T @ a) - a) <= 1e-13 * np.sqrt(m * n) * np.linalg.norm(a), (b, kind)
    # the same basis as Householder up to column signs (well-conditioned member)
    qh, _ = P.thin_qr(mats[0][1])
    signs = np.sign(np.sum(q[0] * qh, axis=0))
    assert np.all(np.abs(signs) == 1)
    assert np.linalg.norm(q[0] - qh * signs) <= 1e-11 * np.sqrt(n)


def _padded_low_rank(O, modes, true_r, pad_r, seed):
    x = O.random_gaussian_tt(modes, true_r, seed)
    out = []
    for k, c in enumerate(x.cores()):
        z = np.zeros((pad_r[k], c.shape[1], pad_r[k + 1]))
        z[:c.shape[0], :, :c.shape[2]] = c
        out.append(z)
    return O.TT.from_cores(out)


_CHOL_SWEEP_SCRIPT = r"""
import sys, numpy as np
sys.path[:0] = [sys.argv[1], sys.argv[2], sys.argv[3]]
import paper_2511_03598_b200 as P, py_oracle as O
from helpers import left_orth_defect, rel_err_vs_ref, to_device
from test_gpu_parity import _padded_low_rank
# exactly rank-deficient padded input (true ranks 20 stored as 60, l = 40):
# the speculative Cholesky QR of mode 1.. breaks down or yields a valid basis
xp = _padded_low_rank(O, [16] * 5, [1, 20, 20, 20, 20, 1], [1, 60, 60, 60, 60, 1], 17)
y = P.round_fixed_krp(to_device(xp), [40] * 4, 3, rng=P.RNG_PHILOX)
assert np.all(np.isfinite(y.flat()))
assert rel_err_vs_ref(xp, y) <= 1e-10
assert left_orth_defect(y.cores()) <= 1e-12
t = to_device(xp)
plan = P.FixedKrpPlan(t, [40] * 4, 3)
plan.execute()
assert np.array_equal(plan.output.flat(), y.flat())
# full-rank input of the same shape through the same plan, against the oracle
x2 = O.two_part_tt(5, 16, 20, 40, 1e-8, 2203)
P.copy_from_host(t, x2.flat())
plan.execute()
y2 = P.round_fixed_krp(to_device(x2), [40] * 4, 3, rng=P.RNG_PHILOX)
assert np.array_equal(plan.output.flat(), y2.flat())
assert rel_err_vs_ref(O.round_fixed_krp(x2, [40] * 4, 3, rng=O.PHILOX), y2) <= 1e-10
# config-3 shapes (7040 x 110 sketches) at reduced order
x3 = O.two_part_tt(6, 64, 100, 300, 1e-8, 1003)
y3 = P.round_fixed_krp(to_device(x3), [110] * 5, 7, rng=P.RNG_PHILOX)
assert rel_err_vs_ref(O.round_fixed_krp(x3, [110] * 5, 7, rng=O.PHILOX), y3) <= 1e-10
plan.close()
print("ok")
"""


_CQR_PANEL_SCRIPT = r"""
import sys, numpy as np
sys.path[:0] = [sys.argv[1], sys.argv[2], sys.argv[3]]
import paper_2511_03598_b200 as P, py_oracle as O
from helpers import rel_err_vs_ref, to_device
# mode-2 sketch 7,680 x 120 (> one cluster of rows: the grid-panel blocked QR)
x = O.two_part_tt(4, 64, 100, 140, 1e-8, 3101)
y = P.round_fixed_krp(to_device(x), [120] * 3, 7, rng=P.RNG_PHILOX)
ref = O.round_fixed_krp(x, [120] * 3, 7, rng=O.PHILOX)
assert y.ranks() == ref.ranks, (y.ranks(), ref.ranks)
assert rel_err_vs_ref(ref, y) <= 1e-10
t = to_device(x)
plan = P.FixedKrpPlan(t, [120] * 3, 7)
plan.execute()
assert np.array_equal(plan.output.flat(), y.flat())
plan.close()
print("ok")
"""


def test_fixed_krp_straddling_panel_runs_once(P, O):
    """Config-5b structure at reduced size (rank 40 + 1e-8 x rank 88, l = 64: the
    second 32-column panel of every sketch holds 8 dominant directions and 24 at
    1e-8, kappa ~ 1e8-1e9): the Cholesky-QR panel takes its shifted passes instead
    of breaking down, so the eager call runs ONCE (about as many kernel launches as
    one replay of its plan), charges the reference's flops once, and matches the
    oracle; the last bond (n_d < l, rank-deficient by construction) does not
    speculate."""
    x = O.two_part_tt(6, 48, 40, 88, 1e-8, 4101)
    ranks = [64] * 5
    y = to_device(x)
    ctx = y.ctx
    P.round_fixed_krp(y, ranks, 7, rng=P.RNG_PHILOX)  # warm-up: pools, kernel attributes
    ctx.reset_counters()
    O.flops_reset()
    l0 = ctx.kernel_launches()
    out = P.round_fixed_krp(y, ranks, 7, rng=P.RNG_PHILOX)
    eager_launches = ctx.kernel_launches() - l0
    ref = O.round_fixed_krp(x, ranks, 7, rng=O.PHILOX)
    dev, rf = ctx.counters(), O.flops_get()
    assert (dev.gemm, dev.qr, dev.svd, dev.sketch) == (rf["gemm"], rf["qr"], rf["svd"], rf["sketch"])
    assert out.ranks() == ref.ranks
    assert rel_err_vs_ref(ref, out) <= 1e-10
    plan = P.FixedKrpPlan(y, ranks, 7)
    l1 = ctx.kernel_launches()
    plan.execute()
    plan_launches = ctx.kernel_launches() - l1
    assert np.array_equal(plan.output.flat(), out.flat())
    plan.close()
    assert eager_launches <= 1.2 * plan_launches, (eager_launches, plan_launches)


@pytest.mark.parametrize("knobs", [{"TTR_QR_CQR": "1"}, {"TTR_QR_CQR": "1", "TTR_QR_CQR_FUSED": "0"},
                                   {"TTR_QR_CQR": "0"}],
                         ids=["fused-K4f", "launches-K4d", "householder-panels"])
def test_fixed_krp_cholesky_qr_panels(P, O, knobs):
    """The sweep's blocked grid QR with its three panel kernels — the Cholesky-QR
    panels with Householder reconstruction as one cooperative kernel (K4f, the
    default), as separate launches (K4d), and the Householder panels: oracle
    parity, plan == eager (the knobs are read once per process: subprocess)."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    root = os.path.dirname(here)
    env = dict(os.environ, **knobs)
    r = subprocess.run([sys.executable, "-c", _CQR_PANEL_SCRIPT, root, os.path.join(root, "oracle"), here],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr


def test_fused_cholesky_qr_panel_kernel(P):
    """K4f (one cooperative kernel per Cholesky-QR panel): A = QR, Q^T Q = I and an
    upper R on Gaussian, graded, nearly dependent and 5b-like matrices (panels of 32
    and fewer columns, two- and three-pass panels); a rank-deficient matrix flags
    a breakdown or yields a valid factorisation (tools/qr_fused_check.py)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, TTR_QR_CQR="1")
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "qr_fused_check.py")], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr


def test_fixed_krp_cholesky_sweep_and_fallback(P, O):
    """The opt-in Cholesky-QR sweep (TTR_QR_CHOL=1, read once per process, so
    in a subprocess): oracle parity, and exactly rank-deficient sketches either
    get a valid basis or are redone on the Householder path — eager and plan."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    root = os.path.dirname(here)
    env = dict(os.environ, TTR_QR_CHOL="1")
    r = subprocess.run([sys.executable, "-c", _CHOL_SWEEP_SCRIPT, root, os.path.join(root, "oracle"), here],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr


# ---- K1: Philox factors are bit-identical on host and device ---------------------

@pytest.mark.parametrize("seed,mode,rows,cols,col0", [(7, 2, 20, 15, 0), (7, 30, 64, 110, 0), (2**40 + 3, 5, 33, 9, 17),
                                                      (0, 12, 128, 40, 400)])
def test_philox_factor_bitwise(P, O, seed, mode, rows, cols, col0):
    dev = P.philox_factor(seed, mode, rows, cols, col0)
    host = O.philox_factor(seed, mode, rows, cols, col0)
    assert np.array_equal(dev, host)


# ---- K2: KRP partial contractions ----------------------------------------------------

def test_krp_hand_example(P):
    """tests/test_sketch.cpp:34-43: cores (1,2)/(3,4), Omega = ones -> W_2 = 7."""
    tt = P.TTTensor.from_cores([np.array([[[1.0], [2.0]]]), np.array([[[3.0], [4.0]]])])
    w = P.krp_partial_contractions_rl(tt, 1, factors=[np.ones((2, 1))])
    assert w[0].shape == (1, 1) and abs(w[0][0, 0] - 7.0) < 1e-14


def test_krp_zero_factors(P, O):
    ott = O.random_gaussian_tt([3, 4, 3], [1, 2, 2, 1], 5)
    w = P.krp_partial_contractions_rl(to_device(ott), 2, factors=[np.zeros((4, 2)), np.zeros((3, 2))])
    assert all(np.linalg.norm(x) == 0.0 for x in w)


@pytest.mark.parametrize("seed", range(8))
def test_krp_matches_oracle_random_shapes(P, O, seed):
    """tests/test_sketch.cpp:54-77 shapes (d<=5, small n, r) plus the reference tolerance."""
    rng = np.random.default_rng(seed)
    d = 3 + seed % 3
    modes = [int(rng.integers(2, 7)) for _ in range(d)]
    ranks = [1] + [int(rng.integers(1, 5)) for _ in range(d - 1)] + [1]
    ott = O.random_gaussian_tt(modes, ranks, 900 + seed)
    cols = 1 + seed % 4
    f = O.draw_factors(ott, 2, cols, O.derive_seed(seed, 4))
    w_ref = O.krp_contractions(ott, f)
    w_gpu = P.krp_partial_contractions_rl(to_device(ott), cols, factors=f)
    for a, b in zip(w_ref, w_gpu):
        assert np.linalg.norm(a - b) <= 1e-12 * (1.0 + np.linalg.norm(a))


@pytest.mark.parametrize("d,n,r,cols", [(6, 16, 24, 20), (5, 64, 130, 110), (4, 20, 50, 15), (4, 32, 200, 40)])
def test_krp_matches_oracle_config_shapes(P, O, d, n, r, cols):
    ranks = [1] + [r] * (d - 1) + [1]
    ott = O.random_gaussian_tt([n] * d, ranks, 11)
    f = O.draw_factors(ott, 2, cols, 3, rng=O.PHILOX)
    w_ref = O.krp_contractions(ott, f)
    w_gpu = P.krp_partial_contractions_rl(to_device(ott), cols, seed=3)  # device Philox draw
    for a, b in zip(w_ref, w_gpu):
        assert np.linalg.norm(a - b) <= 1e-12 * (1.0 + np.linalg.norm(a))


def test_krp_append_equals_one_shot_bitwise(P, O):
    """tests/test_sketch.cpp:78-98 on the device: columns are contraction-batch independent."""
    ott = O.random_gaussian_tt([4, 32, 16, 4], [1, 3, 40, 2, 1], 77)
    dtt = to_device(ott)
    once = P.krp_partial_contractions_rl(dtt, 5, seed=500)
    first = P.krp_partial_contractions_rl(dtt, 3, seed=500, col0=0)
    rest = P.krp_partial_contractions_rl(dtt, 2, seed=500, col0=3)
    for a, b, c in zip(once, first, rest):
        assert np.array_equal(a, np.hstack([b, c]))


# ---- TT arithmetic -------------------------------------------------------------------

def test_norm_exact_and_relative_error(P, O):
    ott = O.random_gaussian_tt([6, 6, 6, 6, 6], [1, 4, 4, 4, 4, 1], 21)
    dtt = to_device(ott)
    assert abs(P.norm_exact(dtt) - O.norm_exact(ott)) <= 1e-12 * O.norm_exact(ott)
    other = O.random_gaussian_tt([6, 6, 6, 6, 6], [1, 3, 5, 2, 4, 1], 22)
    ref = O.relative_error(ott, other)
    assert abs(P.relative_error(dtt, to_device(other)) - ref) <= 1e-12 * ref
    assert P.relative_error(dtt, dtt) <= 1e-14


def test_formal_sum_matches_oracle(P, O):
    ts = [O.random_gaussian_tt([3, 2, 4, 3], [1, 2, 3, 2, 1], 100 + i) for i in range(3)]
    ref = O.formal_sum(ts)
    got = P.formal_sum([to_device(t) for t in ts])
    assert np.array_equal(got.flat(), ref.flat())


# ---- fixed-rank KRP rounding -------------------------------------------------------------

@pytest.mark.parametrize("rng_mode", [0, 1])
def test_fixed_krp_config1_parity(P, O, rng_mode):
    """BASELINE config 1 (d=10, n=20, rank 10 + 1e-4 rank 40, l = 15)."""
    x = O.two_part_tt(10, 20, 10, 40, 1e-4, 1001)
    y_ref = O.round_fixed_krp(x, [15] * 9, 7, rng=rng_mode)
    y_gpu = P.round_fixed_krp(to_device(x), [15] * 9, 7, rng=rng_mode)
    assert y_gpu.ranks() == y_ref.ranks == [1] + [15] * 9 + [1]
    assert rel_err_vs_ref(y_ref, y_gpu) <= 1e-10
    assert left_orth_defect(y_gpu.cores()) <= 1e-12


def test_fixed_krp_exact_recovery(P, O):
    """tests/test_round_rand.cpp:35-42: padded exact-rank tensor, true ranks."""
    base = O.random_gaussian_tt([6, 5, 6, 5], [1, 3, 4, 3, 1], 88)
    cores = base.cores()
    pad = [1, 7, 8, 7, 1]
    pc = []
    for k, c in enumerate(cores):
        z = np.zeros((pad[k], c.shape[1], pad[k + 1]))
        z[: c.shape[0], :, : c.shape[2]] = c
        pc.append(z)
    padded = O.TT.from_cores(pc)
    y = P.round_fixed_krp(to_device(padded), [3, 4, 3], 5)
    assert y.ranks() == [1, 3, 4, 3, 1]
    assert rel_err_vs_ref(padded, y) <= 1e-10
    assert left_orth_defect(y.cores()) <= 1e-12


def test_fixed_krp_invalid_ranks(P, O):
    t = to_device(O.random_gaussian_tt([4, 4], [1, 2, 1], 0))
    with pytest.raises(P.TTRoundError) as e:
        P.round_fixed_krp(t, [2, 2], 0)
    assert e.value.code == "InvalidRanks"
    with pytest.raises(P.TTRoundError) as e:
        P.round_fixed_krp(t, [0], 0)
    assert e.value.code == "InvalidRanks"


def test_fixed_krp_config3_shape_parity(P, O):
    """Config 3 shapes at reduced order (d=6 instead of 30): n=64, formal rank 400, l=110."""
    x = O.two_part_tt(6, 64, 100, 300, 1e-8, 1003)
    y_ref = O.round_fixed_krp(x, [110] * 5, 7, rng=O.PHILOX)
    y_gpu = P.round_fixed_krp(to_device(x), [110] * 5, 7, rng=P.RNG_PHILOX)
    assert y_gpu.ranks() == y_ref.ranks == [1, 64, 110, 110, 110, 110, 1]
    assert rel_err_vs_ref(y_ref, y_gpu) <= 1e-10


def test_plan_replays_bitwise(P, O):
    """The CUDA-graph plan reproduces the eager call bit for bit, also after the
    input buffer is refilled with other data."""
    x1 = O.two_part_tt(5, 24, 12, 36, 1e-6, 2001)
    x2 = O.two_part_tt(5, 24, 12, 36, 1e-6, 2002)
    t = to_device(x1)
    plan = P.FixedKrpPlan(t, [20] * 4, 7)
    plan.execute()
    assert np.array_equal(plan.output.flat(), P.round_fixed_krp(to_device(x1), [20] * 4, 7).flat())
    P.copy_from_host(t, x2.flat())
    plan.execute()
    y2 = P.round_fixed_krp(to_device(x2), [20] * 4, 7)
    assert np.array_equal(plan.output.flat(), y2.flat())
    assert rel_err_vs_ref(O.round_fixed_krp(x2, [20] * 4, 7, rng=O.PHILOX), y2) <= 1e-10
    plan.close()


def test_random_philox_tt_bitwise(P, O):
    """The bench inputs are reproducible on the host: the oracle's
    random_philox_tt equals the device generator bit for bit (so the CPU
    reference arm rounds the same config input as the GPU arm)."""
    modes, ranks = [7, 16, 5, 9], [1, 13, 30, 4, 1]
    dev = P.TTTensor.random_philox(modes, ranks, 123456789, P.Context(0))
    host = O.random_philox_tt(modes, ranks, 123456789)
    assert np.array_equal(dev.flat(), host.flat())


def test_rank_cap_length_checked(P, O):
    """max_rank_cap crosses the C ABI with its length: anything but d-1 caps >= 1
    is InvalidRanks (the reference would index the vector out of bounds)."""
    x = to_device(O.two_part_tt(4, 8, 3, 5, 1e-6, 2005))
    for cap in ([3, 3], [3, 3, 3, 3], [3, 0, 3]):
        with pytest.raises(P.TTRoundError) as e:
            P.round_adaptive_krp(x, P.AdaptiveConfig(tolerance=1e-6, seed=1, max_rank_cap=cap))
        assert e.value.code == "InvalidRanks"


def test_plan_survives_scratch_growth(P, O):
    """A plan keeps the split-K scratch it captured: a later call on the same
    context that needs a larger scratch (a bigger tensor) must not free the
    buffer under the graph — the replay still equals the eager result bitwise."""
    ctx = P.Context(0)
    x = O.two_part_tt(5, 24, 12, 36, 1e-6, 2001)
    t = to_device(x, ctx)
    plan = P.FixedKrpPlan(t, [20] * 4, 7)
    plan.execute()
    first = plan.output.flat()
    big = P.TTTensor.two_part_philox(4, 128, 300, 700, 1e-8, 1005, ctx)  # split-K scratch of 1000 x 320 slices
    big_out = P.round_fixed_krp(big, [320] * 3, 7)
    del big, big_out
    for _ in range(2):
        plan.execute()
        assert np.array_equal(plan.output.flat(), first)
    plan.close()


def test_host_streaming_plan(P, O):
    """ttr_plan_fixed_krp_host: H2D of the input and D2H of the result inside the
    graph (copy stream, per-core events) give the eager result bitwise."""
    import torch
    x = O.two_part_tt(6, 32, 20, 60, 1e-6, 2003)
    y_eager = P.round_fixed_krp(to_device(x), [25] * 5, 7)
    t = to_device(O.two_part_tt(6, 32, 20, 60, 1e-6, 2004))  # staging buffer, other contents
    host_in = torch.from_numpy(np.ascontiguousarray(x.flat())).pin_memory()
    y_flat = y_eager.flat()
    out_len = y_flat.size
    host_out = torch.zeros(out_len, dtype=torch.float64).pin_memory()
    plan = P.FixedKrpPlan(t, [25] * 5, 7, host_in=host_in, host_out=host_out)
    for _ in range(2):
        host_out.zero_()
        plan.execute()
        t.ctx.synchronize()
        assert np.array_equal(host_out.numpy(), y_flat)
    plan.close()


# ---- Rand-Orth with a Gaussian TT sketch (round_rand.cpp:66-78) --------------------------------

def test_rand_orth_tt_parity(P, O):
    """Same R (reference xoshiro stream) on both sides: identical ranks, <= 1e-10;
    full width is exact (test_round_rand.cpp:274-277)."""
    x = O.two_part_tt(6, 16, 10, 30, 1e-6, 88)
    for seed, rng in ((0, 0), (5, 0), (5, 1)):
        ref = O.round_rand_orth_tt(x, [14] * 5, seed, rng=rng)
        y = P.round_rand_orth_tt(to_device(x), [14] * 5, seed, rng=rng)
        assert y.ranks() == ref.ranks
        assert rel_err_vs_ref(ref, y) <= 1e-10
    t = O.random_gaussian_tt([5, 4, 5], [1, 4, 3, 1], 77)
    assert rel_err_vs_ref(t, P.round_rand_orth_tt(to_device(t), [4, 3], 5)) <= 1e-10


# ---- compression_pass / Adap-R (round_rand.cpp:155-179) ----------------------------------------

def test_compression_pass_parity(P, O):
    """Adap-R: adaptive rounding then the right-to-left truncation pass, same ranks
    and <= 1e-10 against the oracle; non-left-orthogonal input is rejected."""
    x = O.two_part_tt(6, 16, 12, 36, 1e-6, 77)
    a_ref = O.round_adaptive_krp(x, tolerance=1e-4, f_init=0.1, f_inc=0.05, seed=3, rng=O.PHILOX)
    a_gpu = P.round_adaptive_krp(to_device(x), P.AdaptiveConfig(tolerance=1e-4, seed=3))
    assert a_gpu.ranks() == a_ref.ranks
    nrm = O.norm_exact(a_ref)
    for tau in (1e-6 * nrm, 1e-3 * nrm):
        c_ref = O.compression_pass(a_ref, tau)
        c_gpu = P.compression_pass(to_device(a_ref), tau)
        assert c_gpu.ranks() == c_ref.ranks
        assert rel_err_vs_ref(c_ref, c_gpu) <= 1e-10
    with pytest.raises(P.TTRoundError) as e:
        P.compression_pass(to_device(x), 1e-6)
    assert e.value.code == "NotLeftOrthogonal"


# ---- sum of TT tensors without the formal sum (sum_round.cpp) ----------------------------------

@pytest.mark.parametrize("rng_mode", [0, 1])
def test_sum_round_parity(P, O, rng_mode):
    """Eight random terms (test_sum_round.cpp:100-126 shapes): identical ranks and
    <= 1e-10 against the oracle's round_sum_adaptive_krp, both generators."""
    terms = [O.random_gaussian_tt([8] * 4, [1, 3, 3, 3, 1], O.derive_seed(99, i)) for i in range(8)]
    for seed in (0, 3):
        ref = O.round_sum_adaptive_krp(terms, 1e-6, 0.05, seed, rng=rng_mode)
        y = P.round_sum_adaptive_krp([to_device(t) for t in terms], 1e-6, 0.05, seed, rng=rng_mode)
        assert y.ranks() == ref.ranks
        assert rel_err_vs_ref(ref, y) <= 1e-10


def test_sum_round_two_part_parity(P, O):
    """The structure of every config input (X + eps Z) rounded as a 2-term sum:
    ranks and values match the oracle; the sum sketch never touches the formal
    sum's zero blocks."""
    x = O.random_gaussian_tt([16] * 6, [1] + [20] * 5 + [1], 5)
    z = O.random_gaussian_tt([16] * 6, [1] + [40] * 5 + [1], 6)
    x = O.scaled(x, 1.0 / O.norm_exact(x))
    z = O.scaled(z, 1e-6 / O.norm_exact(z))
    ref = O.round_sum_adaptive_krp([x, z], 1e-4, 0.05, 7, rng=O.PHILOX)
    y = P.round_sum_adaptive_krp([to_device(x), to_device(z)], 1e-4, 0.05, 7)
    assert y.ranks() == ref.ranks
    assert rel_err_vs_ref(ref, y) <= 1e-10


def test_sum_round_edge_cases(P, O):
    x = O.random_gaussian_tt([5, 4, 5], [1, 3, 3, 1], 37)
    y = P.round_sum_adaptive_krp([to_device(x), to_device(O.scaled(x, -1.0))], 1e-6, 0.05, 4)
    assert max(y.ranks()) == 1 and P.norm_exact(y) <= 1e-10 * O.norm_exact(x)
    x = O.random_gaussian_tt([6, 5, 6], [1, 4, 4, 1], 52)
    y = P.round_sum_adaptive_krp([to_device(x)], 1e-10, 0.05, 8)
    assert rel_err_vs_ref(x, y) <= 1e-9
    with pytest.raises(P.TTRoundError) as e:
        P.round_sum_adaptive_krp([to_device(O.random_gaussian_tt([4, 4], [1, 2, 1], 3)),
                                  to_device(O.random_gaussian_tt([4, 5], [1, 2, 1], 3))], 1e-6, 0.05, 1)
    assert e.value.code == "ModeSizeMismatch"
    with pytest.raises(P.TTRoundError) as e:
        P.round_sum_adaptive_krp([to_device(x)], 0.0, 0.05, 1)
    assert e.value.code == "InvalidArgument"


# ---- adaptive KRP rounding -------------------------------------------------------------------

@pytest.mark.parametrize("rng_mode", [0, 1])
def test_adaptive_config2_small_parity(P, O, rng_mode):
    """Config 2 structure at reduced order: identical ranks and <= 1e-10 difference."""
    x = O.two_part_tt(6, 32, 30, 170, 1e-6, 1002)
    y_ref = O.round_adaptive_krp(x, tolerance=1e-4, f_init=0.1, f_inc=0.05, seed=7, rng=rng_mode)
    y_gpu = P.round_adaptive_krp(to_device(x), P.AdaptiveConfig(tolerance=1e-4, seed=7, rng=rng_mode))
    assert y_gpu.ranks() == y_ref.ranks
    assert rel_err_vs_ref(y_ref, y_gpu) <= 1e-10


def test_adaptive_rank_caps(P, O):
    x = O.synthetic_perturbed_tt(4, 10, 6, 1e-5, 23)
    y = P.round_adaptive_krp(to_device(x), P.AdaptiveConfig(tolerance=1e-8, seed=2, max_rank_cap=[3, 3, 3]))
    assert max(y.ranks()) <= 3


# ---- deterministic TT-SVD rounding -------------------------------------------------------------

def test_det_fixed_ranks_parity(P, O):
    x = O.synthetic_perturbed_tt(5, 20, 10, 1e-5, 1234)
    y_ref = O.round_deterministic(x, ranks=[10] * 4)
    y_gpu = P.round_deterministic(to_device(x), target_ranks=[10] * 4)
    assert y_gpu.ranks() == y_ref.ranks
    assert rel_err_vs_ref(y_ref, y_gpu) <= 1e-10


def test_det_tolerance_parity(P, O):
    x = O.random_gaussian_tt([6, 5, 6, 5], [1, 5, 6, 4, 1], 41)
    y_ref = O.round_deterministic(x, eps=1e-3)
    y_gpu = P.round_deterministic(to_device(x), eps=1e-3)
    assert y_gpu.ranks() == y_ref.ranks
    assert rel_err_vs_ref(y_ref, y_gpu) <= 1e-10


def test_estimate_norm_matches_oracle(P, O):
    x = O.synthetic_perturbed_tt(4, 10, 5, 1e-5, 99)
    for rng_mode in (0, 1):
        ref = O.estimate_norm_krp(x, 64, 7000, rng=rng_mode)
        got = P.estimate_norm_krp(to_device(x), 64, 7000, rng=rng_mode)
        assert abs(got - ref) <= 1e-12 * ref


# ---- batched rounding (config 5a) ------------------------------------------------------------

def test_batched_fixed_krp_config5a_parity(P, O):
    """Config 5a shapes (d=8, n=16, rank 16 + 1e-6 rank 48, l=20): tensor b of the batch equals
    round_fixed_krp(Y_b, {20}x7, derive_seed(7, b)) of the oracle."""
    B = 24
    xs = [O.two_part_tt(8, 16, 16, 48, 1e-6, O.derive_seed(1005, b)) for b in range(B)]
    n, r, _ = xs[0].shape()
    batch = P.TTBatch.from_flats(n, r, [x.flat() for x in xs])
    out = P.round_fixed_krp_batched(batch, [20] * 7, 7)
    _, on, orr, _ = out.shape()
    assert orr == [1, 16, 20, 20, 20, 20, 20, 20, 1]
    flats = out.flats()
    for b in (0, 5, B - 1):
        y_ref = O.round_fixed_krp(xs[b], [20] * 7, O.derive_seed(7, b), rng=O.PHILOX)
        assert y_ref.ranks == orr
        y_gpu = O.TT.from_flat(len(on), on, orr, flats[b])
        assert O.relative_error(y_ref, y_gpu) <= 1e-10


@pytest.mark.parametrize("d,n,r1,r2,l", [(4, 8, 3, 5, 6), (4, 16, 8, 16, 12), (5, 12, 10, 20, 28),
                                          (4, 40, 4, 8, 30), (5, 16, 10, 20, 18), (4, 16, 12, 36, 17)])
def test_batched_shapes_parity(P, O, d, n, r1, r2, l):
    """Batched QR dispatch (register column owners: 1..4 columns per warp, 1..12 row
    chunks; > 512 rows: the shared-memory kernel) against the oracle, rank-deficient
    last bond included."""
    B = 6
    xs = [O.two_part_tt(d, n, r1, r2, 1e-6, O.derive_seed(77, b)) for b in range(B)]
    nn, r, _ = xs[0].shape()
    out = P.round_fixed_krp_batched(P.TTBatch.from_flats(nn, r, [x.flat() for x in xs]), [l] * (d - 1), 5)
    _, on, orr, _ = out.shape()
    flats = out.flats()
    for b in (0, B - 1):
        y_ref = O.round_fixed_krp(xs[b], [l] * (d - 1), O.derive_seed(5, b), rng=O.PHILOX)
        assert y_ref.ranks == orr
        assert O.relative_error(y_ref, O.TT.from_flat(len(on), on, orr, flats[b])) <= 1e-10


def test_batched_equals_single(P, O):
    xs = [O.two_part_tt(5, 20, 6, 10, 1e-4, 40 + b) for b in range(3)]
    n, r, _ = xs[0].shape()
    outb = P.round_fixed_krp_batched(P.TTBatch.from_flats(n, r, [x.flat() for x in xs]), [8] * 4, 11)
    for b, x in enumerate(xs):
        single = P.round_fixed_krp(to_device(x), [8] * 4, O.derive_seed(11, b))
        _, on, orr, _ = outb.shape()
        yb = O.TT.from_flat(len(on), on, orr, outb.flats(b, 1)[0])
        assert O.relative_error(to_oracle(single), yb) <= 1e-12


def test_device_kernel_sum_input_matches_oracle(P, O):
    """The device generator of the config-4 input equals the oracle's (exp differs by <= ulps)."""
    dev = P.TTTensor.kernel_sum(3, 16, 4, 3, 0.3, 1004)
    ref = O.kernel_sum_tt(3, 16, 4, 3, 0.3, 1004)
    assert dev.ranks() == ref.ranks
    a, b = dev.flat(), ref.flat()
    assert np.max(np.abs(a - b)) <= 1e-15 * np.max(np.abs(b))


def test_adaptive_config4_small_parity(P, O):
    """Config 4 structure at reduced size (d=5, n=32, 6 terms of rank 5): identical ranks."""
    x = O.kernel_sum_tt(5, 32, 5, 6, 0.3, 1004)
    y_ref = O.round_adaptive_krp(x, tolerance=1e-6, f_init=0.1, f_inc=0.04, seed=7, rng=O.PHILOX)
    y_gpu = P.round_adaptive_krp(to_device(x), P.AdaptiveConfig(tolerance=1e-6, f_init=0.1, f_inc=0.04, seed=7))
    assert y_gpu.ranks() == y_ref.ranks
    assert rel_err_vs_ref(y_ref, y_gpu) <= 1e-10


# ---- edge cases across the entry points ----------------------------------------------------------

def _zero_tt(O, n, r):
    return O.TT.from_cores([np.zeros((r[k], n[k], r[k + 1])) for k in range(len(n))])


@pytest.mark.parametrize("shape", [
    ([7], [1, 1]),                       # d = 1
    ([6, 5], [1, 3, 1]),                 # d = 2
    ([1, 4, 1, 3], [1, 1, 2, 2, 1]),     # unit mode sizes
    ([3, 2, 3], [1, 3, 3, 1]),           # ranks at their caps (r_k = prod of modes)
])
def test_edge_shapes_all_paths(P, O, shape):
    """Ragged / degenerate shapes through fixed, adaptive, deterministic and
    Rand-Orth-TT rounding: the device matches the oracle (ranks and values)."""
    n, r = shape
    x = O.random_gaussian_tt(n, r, 1234)
    d = len(n)
    tx = to_device(x)
    targets = [5] * (d - 1)  # larger than several caps: l_eff = min(l, rows, cols)
    ref = O.round_fixed_krp(x, targets, 3, rng=O.PHILOX)
    y = P.round_fixed_krp(tx, targets, 3)
    assert y.ranks() == ref.ranks
    assert rel_err_vs_ref(ref, y) <= 1e-10
    ref = O.round_adaptive_krp(x, tolerance=1e-8, f_init=0.5, f_inc=0.5, seed=4, rng=O.PHILOX)
    y = P.round_adaptive_krp(tx, P.AdaptiveConfig(tolerance=1e-8, f_init=0.5, f_inc=0.5, seed=4))
    assert y.ranks() == ref.ranks
    assert rel_err_vs_ref(ref, y) <= 1e-10
    ref = O.round_deterministic(x, eps=1e-12)
    y = P.round_deterministic(tx, eps=1e-12)
    assert y.ranks() == ref.ranks
    assert rel_err_vs_ref(ref, y) <= 1e-10
    if d > 1:
        ref = O.round_rand_orth_tt(x, targets, 6, rng=O.PHILOX)
        y = P.round_rand_orth_tt(tx, targets, 6)
        assert y.ranks() == ref.ranks
        assert rel_err_vs_ref(ref, y) <= 1e-10


def test_zero_tensor_inputs(P, O):
    """An all-zero tensor: every sketch is zero, Householder takes tau = 0, the
    result is the zero tensor with the capped ranks (no NaN anywhere)."""
    n, r = [4, 5, 4], [1, 3, 3, 1]
    z = _zero_tt(O, n, r)
    y = P.round_fixed_krp(to_device(z), [2, 2], 1)
    ref = O.round_fixed_krp(z, [2, 2], 1, rng=O.PHILOX)
    assert y.ranks() == ref.ranks
    f = y.flat()
    assert np.all(np.isfinite(f))
    assert P.norm_exact(y) == 0.0
    yd = P.round_deterministic(to_device(z), target_ranks=[2, 2])
    assert np.all(np.isfinite(yd.flat())) and P.norm_exact(yd) == 0.0


def test_nan_free_rank_deficient_sketch(P, O):
    """Exactly rank-deficient padded input (true ranks 2 stored as 6): fixed
    rounding to 6 keeps an orthonormal basis (QR of a rank-2 sketch) and
    reproduces the tensor (the last bond of configs 3/5 behaves like this)."""
    x = O.random_gaussian_tt([6, 6, 6, 6], [1, 2, 2, 2, 1], 99)
    cores = x.cores()
    pad = [1, 6, 6, 6, 1]
    padded = []
    for k, c in enumerate(cores):
        zc = np.zeros((pad[k], c.shape[1], pad[k + 1]))
        zc[:c.shape[0], :, :c.shape[2]] = c
        padded.append(zc)
    xp = O.TT.from_cores(padded)
    y = P.round_fixed_krp(to_device(xp), [6, 6, 6], 2)
    assert np.all(np.isfinite(y.flat()))
    assert rel_err_vs_ref(xp, y) <= 1e-10
    assert left_orth_defect(y.cores()) <= 1e-12


# ---- TTF1 files (io.cpp, test_io.cpp) ----------------------------------------------------------------

def _ttf1_bytes(n, r, flat, magic=b"TTF1"):
    import struct
    return magic + struct.pack("<I", len(n)) + struct.pack(f"<{len(n)}I", *n) + \
        struct.pack(f"<{len(r)}I", *r) + np.asarray(flat, dtype="<f8").tobytes()


def test_ttf1_round_trip_and_format(P, O, tmp_path):
    """test_io.cpp:34-46: round trip bit identical, and the bytes are exactly the
    reference layout (magic, u32 d, n, r, fp64 cores)."""
    x = O.random_gaussian_tt([4, 5, 3], [1, 2, 3, 1], 11)
    n, r, _ = x.shape()
    t = to_device(x)
    p1 = tmp_path / "a.ttf1"
    t.write_ttf1(str(p1))
    assert p1.read_bytes() == _ttf1_bytes(n, r, x.flat())
    back = P.TTTensor.read_ttf1(str(p1))
    assert back.ranks() == r and np.array_equal(back.flat(), x.flat())
    p2 = tmp_path / "b.ttf1"
    back.write_ttf1(str(p2))
    assert p2.read_bytes() == p1.read_bytes()


def test_ttf1_rejects_malformed(P, O, tmp_path):
    """test_io.cpp:48-90: bad magic, rank-chain violation, truncated payload."""
    x = O.random_gaussian_tt([3, 3], [1, 2, 1], 5)
    n, r, _ = x.shape()
    good = _ttf1_bytes(n, r, x.flat())
    cases = {"magic.ttf1": (_ttf1_bytes(n, r, x.flat(), magic=b"TTF2"), "IoError"),
             "chain.ttf1": (_ttf1_bytes(n, [2, 2, 1], x.flat()), "BoundaryRankNotOne"),
             "short.ttf1": (good[:-9], "IoError")}
    for name, (data, code) in cases.items():
        p = tmp_path / name
        p.write_bytes(data)
        with pytest.raises(P.TTRoundError) as e:
            P.TTTensor.read_ttf1(str(p))
        assert e.value.code == code
    with pytest.raises(P.TTRoundError) as e:
        P.TTTensor.read_ttf1(str(tmp_path / "missing.ttf1"))
    assert e.value.code == "IoError"


def test_cli_round_matches_api(P, O, tmp_path):
    """The `round` command (tools/ttround_main.cpp:142-184 mirror): TTF1 in, TTF1
    out, the reference's JSON record; krp-fix with the reference stream equals the
    oracle's xoshiro rounding; krp-adapt-r runs the compression pass."""
    import json
    import subprocess
    import sys
    x = O.two_part_tt(5, 12, 6, 18, 1e-6, 321)
    inp, out = tmp_path / "x.ttf1", tmp_path / "y.ttf1"
    to_device(x).write_ttf1(str(inp))
    cmd = [sys.executable, "-m", "paper_2511_03598_b200.cli", "round", str(inp), str(out), "--algo", "krp-fix",
           "--ranks", "8", "8", "8", "8", "--seed", "7"]
    res = subprocess.run(cmd, capture_output=True, text=True, cwd=__import__("os").path.dirname(__import__("os").path.dirname(__file__)))
    assert res.returncode == 0, res.stderr
    rec = json.loads(res.stdout.strip().splitlines()[-1])
    assert set(rec) >= {"algorithm", "mode", "target", "rel_error", "ranks", "wall_seconds", "flops_total", "seed"}
    y = P.TTTensor.read_ttf1(str(out))
    ref = O.round_fixed_krp(x, [8] * 4, 7, rng=O.XOSHIRO)
    assert y.ranks() == ref.ranks == rec["ranks"]
    assert rel_err_vs_ref(ref, y) <= 1e-10
    cmd[cmd.index("krp-fix")] = "krp-adapt-r"
    i = cmd.index("--ranks")
    del cmd[i:i + 5]
    cmd += ["--tol", "1e-4"]
    res = subprocess.run(cmd, capture_output=True, text=True, cwd=__import__("os").path.dirname(__import__("os").path.dirname(__file__)))
    assert res.returncode == 0, res.stderr
    assert json.loads(res.stdout.strip().splitlines()[-1])["mode"] == "tolerance"
    bad = subprocess.run(cmd[:4] + [str(tmp_path / "nope.ttf1"), str(out)], capture_output=True, text=True,
                         cwd=__import__("os").path.dirname(__import__("os").path.dirname(__file__)))
    assert bad.returncode == 2 and "IoError" in bad.stderr


def test_cli_bench_synthetic(P, O, tmp_path):
    """`bench-synthetic` (ttround_main.cpp:178-210 mirror): the synthetic instance is
    the oracle's synthetic_perturbed_tt bit for bit (reference stream), the CSV has the
    reference header and one row per (target|tol, seed, algorithm) — Orth-Rand rows
    omitted (out of scope) — and the krp-fix rows equal the oracle's round_fixed_krp
    of that instance with the same seed."""
    import csv
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = tmp_path / "b.csv"
    cmd = [sys.executable, "-m", "paper_2511_03598_b200.cli", "bench-synthetic", "--d", "4", "--n", "10", "--rank",
           "5", "--eps-pert", "1e-5", "--targets", "5,6", "--tols", "1e-3", "--seeds", "2", "--csv", str(out)]
    res = subprocess.run(cmd, capture_output=True, text=True, cwd=root)
    assert res.returncode == 0, res.stderr
    summ = json.loads(res.stdout.strip().splitlines()[-1])
    assert summ["x_ranks"] == [1, 10, 10, 10, 1] and summ["omitted_algorithms"] == ["orth-rand"]
    rows = list(csv.reader(open(out)))
    assert ",".join(rows[0]) == ("algorithm,mode,target,rel_error,ranks,wall_seconds,flops_total,flops_gemm,"
                                 "flops_qr,flops_svd,flops_sketch,rng_draws,seed")
    body = rows[1:]
    assert len(body) == 2 * 2 * 3 + 1 * 2 * 3
    syn = O.synthetic_perturbed_tt(4, 10, 5, 1e-5, 20250807)
    for r in body:
        if r[0] == "krp-fix":
            ref = O.round_fixed_krp(syn, [int(float(r[2]))] * 3, int(r[12]), rng=O.XOSHIRO)
            assert r[4] == "x".join(str(v) for v in ref.ranks)
            assert abs(float(r[3]) - O.relative_error(syn, ref)) <= 1e-8 * max(1e-12, float(r[3])) + 1e-15
    bad = subprocess.run(cmd[:4] + ["--d", "1"], capture_output=True, text=True, cwd=root)
    assert bad.returncode == 2 and "InvalidArgument" in bad.stderr


# ---- BASELINE full sizes: size-independent properties ------------------------------------------

@pytest.mark.parametrize("cfg", ["3", "5b"])
def test_full_size_fixed_rank_properties(P, cfg):
    """Configs 3 and 5b at their full BASELINE sizes (2.3 GB / 18.4 GB of cores):
    the expected rank vector, left-orthogonal cores, error at the
    noise level of the input (X + eps Z rounded to a rank >= rank(X)), bitwise
    determinism, and the CUDA-graph plan == the eager call."""
    from paper_2511_03598_b200.seeds import derive_seed
    if cfg == "3":
        d, n, rx, rz, eps, ell, seed = 30, 64, 100, 300, 1e-8, 110, 1003
    else:
        d, n, rx, rz, eps, ell, seed = 20, 128, 300, 700, 1e-8, 320, 1005
    ctx = P.Context(0)
    modes = [n] * d
    x = P.TTTensor.random_philox(modes, [1] + [rx] * (d - 1) + [1], derive_seed(seed, 1), ctx)
    z = P.TTTensor.random_philox(modes, [1] + [rz] * (d - 1) + [1], derive_seed(seed, 2), ctx)
    x = P.scaled(x, 1.0 / P.norm_exact(x))
    z = P.scaled(z, eps / P.norm_exact(z))
    y = P.formal_sum([x, z])
    del z
    out = P.round_fixed_krp(y, [ell] * (d - 1), 7)
    expect = [1, n] + [ell] * (d - 2) + [1]
    assert out.ranks() == expect
    # left-orthogonality of cores 0..d-2 (on the device: ||V^T V - I|| via GEMM)
    for k in (0, 1, d // 2, d - 2):
        v = out.cores()[k]
        rl, nn, rr = v.shape
        m = v.reshape(rl * nn, rr, order="F")
        assert np.linalg.norm(m.T @ m - np.eye(rr)) <= 1e-11
    # randomized rounding error at the noise level: rounding to >= rank(X) keeps X;
    # the per-bond noise residuals add up over the d-1 bonds (~ eps sqrt(d-1))
    bound = 3 * eps * np.sqrt(d - 1)
    err = P.relative_error(y, out)
    assert err <= bound, err
    assert P.relative_error(x, out) <= bound
    again = P.round_fixed_krp(y, [ell] * (d - 1), 7)
    assert np.array_equal(again.flat(), out.flat())
    plan = P.FixedKrpPlan(y, [ell] * (d - 1), 7)
    plan.execute()
    assert np.array_equal(plan.output.flat(), out.flat())
    plan.close()


# ---- BASELINE full sizes: oracle parity ----------------------------------------------------------

def _dev_to_oracle(O, y):
    n, r, _ = y.shape()
    return O.TT.from_flat(len(n), n, r, y.flat())


@pytest.mark.parametrize("cfg", ["2", "3", "4", "5b-d4"])
def test_full_size_config_oracle_parity(P, O, cfg):
    """North-star gate at the FULL BASELINE sizes of configs 2 (adaptive, 143 MB),
    3 (fixed, 2.3 GB) and 4 (adaptive, 1.6 GB), and config 5b at full mode size and
    ranks (n=128, rank 300 + 1e-8 rank 700, l=320) on a d=4 slice (two full
    1000 x 128 x 1000 middle cores; the full d=20 oracle run is ~4 TF on the host,
    the full 5b size is covered by test_full_size_fixed_rank_properties): the device input is downloaded into
    the oracle, both sides draw the same Philox factors, adaptive runs must select
    identical rank vectors and ||Y_gpu - Y_ref|| / ||Y_ref|| <= 1e-10 (TT arithmetic)."""
    ctx = P.Context(0)
    if cfg == "2":
        y = P.TTTensor.two_part_philox(16, 32, 30, 170, 1e-6, 1002, ctx)
        kw = dict(tolerance=1e-4, f_init=0.1, f_inc=0.05, seed=7)
    elif cfg == "3":
        y = P.TTTensor.two_part_philox(30, 64, 100, 300, 1e-8, 1003, ctx)
    elif cfg == "5b-d4":
        y = P.TTTensor.two_part_philox(4, 128, 300, 700, 1e-8, 1005, ctx)
    else:
        y = P.TTTensor.kernel_sum(12, 128, 20, 20, 0.3, 1004, ctx)
        kw = dict(tolerance=1e-6, f_init=0.1, f_inc=0.04, seed=7)
    x = _dev_to_oracle(O, y)
    if cfg in ("3", "5b-d4"):
        tr = [110] * 29 if cfg == "3" else [320] * 3
        y_gpu = P.round_fixed_krp(y, tr, 7)
        y_ref = O.round_fixed_krp(x, tr, 7, rng=O.PHILOX)
    else:
        y_gpu = P.round_adaptive_krp(y, P.AdaptiveConfig(**kw))
        y_ref = O.round_adaptive_krp(x, rng=O.PHILOX, **kw)
    del y, x
    assert y_gpu.ranks() == y_ref.ranks
    assert O.relative_error(y_ref, _dev_to_oracle(O, y_gpu)) <= 1e-10


@pytest.mark.parametrize("cfg", ["5b", "3-det"])
def test_full_size_headline_oracle_parity(P, O, cfg):
    """The north-star gate on the two largest calls at their FULL BASELINE sizes:
    config 5b round_fixed_krp(Y, {320}x19, 7) at d = 20 (18.4 GB of cores,
    round_rand.cpp:52-64) and config 3's comparison call
    round_deterministic(Y, {100}x29) (2.3 GB, orthogonalize.cpp:129-140). The
    device input is downloaded into the oracle, which runs on its OpenBLAS/LAPACK
    backend (the same algorithms on all host cores; the plain-loop port would take
    minutes here). Both sides draw the same Philox factors; the rank vectors must be
    the expected ones and ||Y_gpu - Y_ref|| / ||Y_ref|| <= 1e-10 in TT
    arithmetic (the oracle's stable formal-difference relative_error)."""
    import os
    ctx = P.Context(0)
    if cfg == "5b":
        y = P.TTTensor.two_part_philox(20, 128, 300, 700, 1e-8, 1005, ctx)
        y_gpu = P.round_fixed_krp(y, [320] * 19, 7)
        expect = [1, 128] + [320] * 18 + [1]
    else:
        y = P.TTTensor.two_part_philox(30, 64, 100, 300, 1e-8, 1003, ctx)
        y_gpu = P.round_deterministic(y, target_ranks=[100] * 29)
        expect = [1, 64] + [100] * 27 + [64, 1]
    assert y_gpu.ranks() == expect
    with O.backend_scope("blas", os.cpu_count() or 1):
        x = _dev_to_oracle(O, y)
        del y
        if cfg == "5b":
            y_ref = O.round_fixed_krp(x, [320] * 19, 7, rng=O.PHILOX)
        else:
            y_ref = O.round_deterministic(x, ranks=[100] * 29)
        del x
        assert y_ref.ranks == expect
        err = O.relative_error(y_ref, _dev_to_oracle(O, y_gpu))
    assert err <= 1e-10, err


def test_full_batch_config5a_all_tensors_oracle_parity(P, O):
    """Config 5a at its full size: every one of the 4096 tensors of the batched
    round (12.9 GB generated on the device) equals the oracle's round_fixed_krp of
    the same downloaded input with the per-tensor seed derive_seed(7, b): identical
    ranks and ||Y_gpu - Y_ref|| / ||Y_ref|| <= 1e-10 for each b."""
    from paper_2511_03598_b200.seeds import derive_seed
    ctx = P.Context(0)
    batch = P.TTBatch.two_part_philox(4096, 8, 16, 16, 48, 1e-6, derive_seed(1005, 1000), ctx)
    out = P.round_fixed_krp_batched(batch, [20] * 7, 7)
    _, n, r, _ = batch.shape()
    _, on, orr, _ = out.shape()
    assert orr == [1, 16, 20, 20, 20, 20, 20, 20, 1]
    worst = 0.0
    chunk = 512
    for b0 in range(0, 4096, chunk):
        xs = batch.flats(b0, chunk)
        ys = out.flats(b0, chunk)
        for i in range(chunk):
            x = O.TT.from_flat(len(n), n, r, xs[i])
            y_ref = O.round_fixed_krp(x, [20] * 7, O.derive_seed(7, b0 + i), rng=O.PHILOX)
            assert y_ref.ranks == orr
            worst = max(worst, O.relative_error(y_ref, O.TT.from_flat(len(on), on, orr, ys[i])))
    assert worst <= 1e-10, worst


def test_full_batch_config5a_sampled_oracle_parity(P, O):
    """Config 5a at its full size (4096 tensors, 12.9 GB, generated on the device):
    sampled tensors of the batched result equal the oracle's round_fixed_krp of the
    same (downloaded) input with the per-tensor seed derive_seed(7, b)."""
    from paper_2511_03598_b200.seeds import derive_seed
    ctx = P.Context(0)
    batch = P.TTBatch.two_part_philox(4096, 8, 16, 16, 48, 1e-6, derive_seed(1005, 1000), ctx)
    out = P.round_fixed_krp_batched(batch, [20] * 7, 7)
    _, n, r, _ = batch.shape()
    _, on, orr, _ = out.shape()
    assert orr == [1, 16, 20, 20, 20, 20, 20, 20, 1]
    for b in (0, 1, 2047, 4095):
        x = O.TT.from_flat(len(n), n, r, batch.flats(b, 1)[0])
        y_ref = O.round_fixed_krp(x, [20] * 7, O.derive_seed(7, b), rng=O.PHILOX)
        assert y_ref.ranks == orr
        assert O.relative_error(y_ref, O.TT.from_flat(len(on), on, orr, out.flats(b, 1)[0])) <= 1e-10


# ---- flop accounting (flops.hpp:12-37): the device counters charge the reference's formulas ----

@pytest.mark.parametrize("case", ["fixed", "adaptive2", "adaptive4"])
def test_counters_match_oracle(P, O, case):
    """The device charges exactly the reference's flop counts — in particular the
    adaptive sketch, which the device appends in larger chunks (Sketch::ensure)
    but charges as the reference's column-exact appends when the columns are used."""
    if case == "fixed":
        x = O.two_part_tt(6, 16, 8, 20, 1e-4, 1001)
    elif case == "adaptive2":
        x = O.two_part_tt(6, 32, 30, 170, 1e-6, 1002)
    else:
        x = O.kernel_sum_tt(5, 32, 5, 6, 0.3, 1004)
    y = to_device(x)
    ctx = y.ctx
    ctx.reset_counters()
    O.flops_reset()
    if case == "fixed":
        P.round_fixed_krp(y, [12] * 5, 7)
        O.round_fixed_krp(x, [12] * 5, 7, rng=O.PHILOX)
    else:
        f_inc = 0.05 if case == "adaptive2" else 0.04
        tol = 1e-4 if case == "adaptive2" else 1e-6
        P.round_adaptive_krp(y, P.AdaptiveConfig(tolerance=tol, f_init=0.1, f_inc=f_inc, seed=7))
        O.round_adaptive_krp(x, tolerance=tol, f_init=0.1, f_inc=f_inc, seed=7, rng=O.PHILOX)
    dev, ref = ctx.counters(), O.flops_get()
    assert (dev.gemm, dev.qr, dev.svd, dev.sketch) == (ref["gemm"], ref["qr"], ref["svd"], ref["sketch"])


# ---- the reference's sketch-level API at the boundary (sketch.hpp:13-67, round_rand.hpp:37-39) ----

@pytest.mark.parametrize("rng", [0, 1])
def test_sketch_objects_match_oracle(P, O, rng):
    """GaussianStream -> draw_gaussian_factors -> append_gaussian_columns (bitwise, both
    generators: the reference stream continues across the calls, sketch.cpp:44-65; Philox
    takes the set's next global columns), krp_partial_contractions_rl and
    append_krp_contractions (1e-12, tests/test_sketch.cpp:54-77; the lower modes keep
    their width, sketch.hpp:33-34; the kept columns are untouched by the append)."""
    x = O.two_part_tt(6, 10, 4, 9, 1e-3, 3101)
    xd = to_device(x)
    st = P.GaussianStream(17, rng)
    f = P.draw_gaussian_factors(xd, 2, 6, st)
    P.append_gaussian_columns(f, 3, st)
    if rng == 1:
        first = O.draw_factors(x, 2, 6, 17, rng=rng)
        extra = O.draw_factors(x, 2, 3, 17, rng=rng, col0=6)
    else:  # one sequential stream: 5 factors of 10 x 6, then 5 blocks of 10 x 3, column-major
        seq = O.gaussian_matrix(5 * 10 * 9, 1, 17).ravel()
        first = [seq[q * 60:(q + 1) * 60].reshape(6, 10).T for q in range(5)]
        extra = [seq[300 + q * 30:300 + (q + 1) * 30].reshape(3, 10).T for q in range(5)]
    for k in range(2, 7):
        assert np.array_equal(f.at_mode(k), np.hstack([first[k - 2], extra[k - 2]]))
    w = P.krp_partial_contractions_rl(xd, f)
    wref = O.krp_contractions(x, [f.at_mode(k) for k in range(2, 7)])
    for k in range(2, 7):
        assert np.abs(w.at_mode(k) - wref[k - 2]).max() <= 1e-12 * (1 + np.abs(wref[k - 2]).max())
    before = {k: w.at_mode(k) for k in range(2, 7)}
    fresh = P.draw_gaussian_factors(xd, 4, 4, st)
    P.append_krp_contractions(w, xd, fresh)
    wf = O.krp_contractions(x, [fresh.at_mode(k) for k in range(4, 7)], start_mode=4)
    for k in range(2, 7):
        got = w.at_mode(k)
        assert np.array_equal(got[:, :9], before[k])
        if k < 4:
            assert got.shape[1] == 9
        else:
            assert got.shape[1] == 13
            assert np.abs(got[:, 9:] - wf[k - 4]).max() <= 1e-12 * (1 + np.abs(wf[k - 4]).max())
    with pytest.raises(P.TTRoundError) as e:
        P.draw_gaussian_factors(xd, 1, 3, st)
    assert e.value.code == "InvalidArgument"


@pytest.mark.parametrize("rng", [0, 1])
def test_generate_residual_sketch_matches_oracle(P, O, rng):
    """generate_residual_sketch (round_rand.cpp:80-94): the fresh factors for modes
    k+1..d come from the same stream position / global columns on both sides; S and the
    grown widths match, and residual_norm_estimate equals ||S||/sqrt(b)."""
    x = O.two_part_tt(6, 10, 4, 9, 1e-3, 3102)
    xd = to_device(x)
    st = P.GaussianStream(23, rng)
    w = P.krp_partial_contractions_rl(xd, P.draw_gaussian_factors(xd, 2, 5, st))
    c1 = x.cores()[1]
    z = c1.reshape(c1.shape[0] * c1.shape[1], -1, order="F")  # V(X_2): (r_1 n) x r_2
    w3 = w.at_mode(3)
    q, _ = np.linalg.qr(z @ w3[:, :2])
    s = P.generate_residual_sketch(xd, z, q, w, 2, 4, st)
    s_ref, widths = O.residual_sketch(x, 5, 23, rng, z, q, 2, 4)
    assert np.abs(s - s_ref).max() <= 1e-12 * (1 + np.abs(s_ref).max())
    assert [w.at_mode(k).shape[1] for k in range(2, 7)] == widths
    assert abs(P.residual_norm_estimate(s, 4) - O.residual_norm_estimate(s_ref, 4)) <= 1e-12 * (1 + np.linalg.norm(s))
    with pytest.raises(P.TTRoundError) as e:
        P.residual_norm_estimate(s, 0)
    assert e.value.code == "InvalidArgument"


def test_dot_random_gaussian_and_constructor_checks(P, O):
    """dot (tensor.cpp:244-256) <= 1e-12; random_gaussian_tt from the reference stream is
    bitwise the oracle's; TTTensor(vector<Core>) checks in the reference's order, including
    the finiteness scan (tensor.cpp:66-79), also on the flat upload."""
    modes, ranks = [6, 5, 7, 4], [1, 3, 5, 2, 1]
    g = P.TTTensor.random_gaussian(modes, ranks, 99)
    go = O.random_gaussian_tt(modes, ranks, 99)
    assert np.array_equal(g.flat(), go.flat())
    h = O.random_gaussian_tt(modes, [1, 2, 4, 3, 1], 5)
    ref = O.dot(go, h)
    assert abs(P.dot(g, to_device(h)) - ref) <= 1e-12 * O.norm_exact(go) * O.norm_exact(h)
    with pytest.raises(P.TTRoundError) as e:
        P.dot(g, to_device(O.random_gaussian_tt([6, 5, 7, 5], ranks, 1)))
    assert e.value.code == "ModeSizeMismatch"
    cases = [([], "EmptyCoreList"), ([np.ones((2, 3, 1))], "BoundaryRankNotOne"),
             ([np.ones((1, 3, 2)), np.ones((3, 3, 1))], "RankChainMismatch"),
             ([np.full((1, 3, 1), np.nan)], "InvalidArgument"), ([np.full((1, 3, 1), np.inf)], "InvalidArgument")]
    for cores, code in cases:
        with pytest.raises(P.TTRoundError) as e:
            P.TTTensor.from_cores(cores)
        assert e.value.code == code
    flat = go.flat().copy()
    flat[7] = np.inf
    with pytest.raises(P.TTRoundError) as e:
        P.TTTensor.from_flat(modes, ranks, flat)
    assert e.value.code == "InvalidArgument"
    ok = P.TTTensor.from_cores([np.ones((1, 2, 2)), np.ones((2, 2, 1))])
    assert ok.ranks() == [1, 2, 1]


# ---- TT-GMRES cookie harness (solver.cpp; csrc/tt_gmres.cu) ----------------------------------

def _dense_kron_apply(terms, ot):
    n, _, _ = ot.shape()
    x = ot.dense().reshape(tuple(n), order="F")
    out = np.zeros_like(x)
    for term in terms:
        y = x
        for k, a in enumerate(term):
            y = np.moveaxis(np.tensordot(a, y, axes=([1], [k])), 0, k)
        out += y
    return out


def test_cookie_problem_and_apply_match_oracle(P, O):
    """build_cookie_problem + apply_operator on the device against the oracle's
    (solver.cpp:81-151): same right-hand side, same operator terms applied to a
    random TT (strided-batch DMMA GEMMs vs the loop), identities copied."""
    op, rhs = P.cookie_problem(2, 8, 3, 1.0, 5.0)
    terms, orhs = O.cookie_problem(2, 8, 3, 1.0, 5.0)
    assert np.array_equal(rhs.flat(), orhs.flat())
    x = O.random_gaussian_tt([64, 3, 3], [1, 4, 2, 1], 8)
    dev = P.apply_operator(op, to_device(x))
    ref = O.apply_operator(terms, x)
    assert len(dev) == len(ref) == 3
    for d, r in zip(dev, ref):
        assert d.ranks() == r.ranks
        assert np.linalg.norm(d.flat() - r.flat()) <= 1e-13 * np.linalg.norm(r.flat())
    # an explicit operator (KronOp.of) and the identity-only case (test_solver.cpp:62-69)
    eye = P.KronOp.of([[np.eye(4), np.eye(5)]])
    y = O.random_gaussian_tt([4, 5], [1, 3, 1], 5)
    assert np.array_equal(P.apply_operator(eye, to_device(y))[0].flat(), y.flat())


@pytest.mark.parametrize("strategy", [0, 1, 2])
def test_gmres_device_matches_oracle(P, O, strategy):
    """tt_gmres on the device vs the oracle (solver.cpp:241-363), the small cookie
    problem of test_solver.cpp:109-125 with the reference's xoshiro sketches:
    same iteration count and rank history, Arnoldi estimates and the solution
    equal to rounding, dense residual <= 1e-4."""
    op, rhs = P.cookie_problem(2, 8, 4, 1.0, 10.0)
    dev = P.tt_gmres(op, rhs, rel_tolerance=1e-5, max_iterations=120, strategy=strategy, seed=4, rng=P.RNG_XOSHIRO)
    ref = O.tt_gmres_cookie(2, 8, 4, 1.0, 10.0, rel_tolerance=1e-5, max_iterations=120, strategy=strategy, seed=4)
    assert dev["converged"] and ref["converged"]
    assert dev["iterations"] == ref["iterations"]
    assert dev["max_rank_history"] == ref["max_rank_history"]
    np.testing.assert_allclose(dev["residual_history"], ref["residual_history"], rtol=1e-6)
    np.testing.assert_allclose(dev["true_residual_history"], ref["true_residual_history"], rtol=1e-5)
    assert rel_err_vs_ref(ref["solution"], dev["solution"]) <= 1e-8
    terms, orhs = O.cookie_problem(2, 8, 4, 1.0, 10.0)
    n, _, _ = orhs.shape()
    b = orhs.dense().reshape(tuple(n), order="F")
    x = to_oracle(dev["solution"])
    assert np.linalg.norm(b - _dense_kron_apply(terms, x)) / np.linalg.norm(b) <= 1e-4


def test_gmres_identity_operator_one_iteration(P, O):
    """test_solver.cpp:96-107."""
    op = P.KronOp.of([[np.eye(6), np.eye(4)]])
    b = O.random_gaussian_tt([6, 4], [1, 2, 1], 12)
    r = P.tt_gmres(op, to_device(b), rel_tolerance=1e-10)
    assert r["converged"] and r["iterations"] == 1
    assert rel_err_vs_ref(b, r["solution"]) <= 1e-9


def test_gmres_criterion8_on_device(P, O):
    """The reference's acceptance criterion 8 (acceptance.cpp:335-383, printed in
    test_output.txt:34) run through the device harness: the deterministic and the
    three seeded AdaptiveKRPSum runs converge in 17 iterations to the dense
    residual 4.42e-07; rank histories stay inside the 2x band."""
    op, rhs = P.cookie_problem(3, 16, 8, 1.0, 10.0)
    terms, orhs = O.cookie_problem(3, 16, 8, 1.0, 10.0)
    n, _, _ = orhs.shape()
    bd = orhs.dense().reshape(tuple(n), order="F")
    det = P.tt_gmres(op, rhs, rel_tolerance=1e-6, max_iterations=250, strategy=P.GMRES_DETERMINISTIC,
                     track_true_residual=False)
    assert det["converged"] and det["iterations"] == 17
    for seed in (1, 2, 3):
        r = P.tt_gmres(op, rhs, rel_tolerance=1e-6, max_iterations=250, strategy=P.GMRES_ADAPTIVE_KRP_SUM, seed=seed,
                       track_true_residual=False, rng=P.RNG_XOSHIRO)
        assert r["converged"] and r["iterations"] == 17
        resid = np.linalg.norm(bd - _dense_kron_apply(terms, to_oracle(r["solution"]))) / np.linalg.norm(bd)
        assert f"{resid:.2g}" == "4.4e-07"
        c = min(len(r["max_rank_history"]), len(det["max_rank_history"]))
        ratio = max([1.0] + [max(x / y, y / x) for x, y in zip(r["max_rank_history"][:c], det["max_rank_history"][:c])])
        assert ratio <= 2.0


def test_cli_cookie(P, O, tmp_path):
    """`cookie` (ttround_main.cpp:246-296 mirror): JSON summary with the reference's
    keys and the iteration CSV with its header; the run equals the API call; an
    unknown strategy is rejected."""
    import csv
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = tmp_path / "c.csv"
    cmd = [sys.executable, "-m", "paper_2511_03598_b200.cli", "cookie", "--params", "2", "--grid", "8", "--nsamples",
           "4", "--tol", "1e-5", "--strategy", "det", "--max-iters", "120", "--csv", str(out)]
    res = subprocess.run(cmd, capture_output=True, text=True, cwd=root)
    assert res.returncode == 0, res.stderr
    summ = json.loads(res.stdout.strip().splitlines()[-1])
    assert set(summ) >= {"converged", "iterations", "strategy", "arnoldi_residual", "solution_ranks",
                         "rounding_seconds", "seed", "true_residual", "csv"}
    assert summ["converged"] and summ["strategy"] == "det"
    ref = O.tt_gmres_cookie(2, 8, 4, 1.0, 10.0, rel_tolerance=1e-5, max_iterations=120, strategy=O.DETERMINISTIC)
    assert summ["iterations"] == ref["iterations"] and summ["solution_ranks"] == ref["solution"].ranks
    rows = list(csv.reader(open(out)))
    assert ",".join(rows[0]) == "iteration,rel_residual,max_tt_rank,cum_rounding_seconds"
    assert len(rows) - 1 == summ["iterations"]
    assert [int(r[2]) for r in rows[1:]] == ref["max_rank_history"]
    bad = subprocess.run(cmd[:4] + ["--strategy", "nope"], capture_output=True, text=True, cwd=root)
    assert bad.returncode != 0


_LR_QR_SCRIPT = r"""
import sys, numpy as np
sys.path[:0] = [sys.argv[1], sys.argv[2], sys.argv[3]]
import paper_2511_03598_b200 as P, py_oracle as O
from helpers import rel_err_vs_ref, to_oracle
# config-5a shapes, 64 tensors: the fused sweep + QR + M kernel (TTR_LR_QR=1)
b = P.TTBatch.two_part_philox(64, 8, 16, 16, 48, 1e-6, 1005)
o = P.round_fixed_krp_batched(b, [20] * 7, 7)
for i in (0, 31, 63):
    n, r = b.shape()[1], b.shape()[2]
    xo = O.TT.from_flat(len(n), n, r, b.flats(i, 1)[0])
    ref = O.round_fixed_krp(xo, [20] * 7, O.derive_seed(7, i), rng=O.PHILOX)
    no, ro = o.shape()[1], o.shape()[2]
    got = O.TT.from_flat(len(no), no, ro, o.flats(i, 1)[0])
    assert ro == ref.ranks, (ro, ref.ranks)
    assert O.relative_error(ref, got) <= 1e-10
print("ok")
"""


def test_batched_fused_qr_epilogue_opt_in(P, O):
    """The opt-in fused sweep + per-tensor QR + M = Q^T V kernel (TTR_LR_QR=1, read
    once per process, so in a subprocess) against the oracle on config-5a shapes."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    root = os.path.dirname(here)
    env = dict(os.environ, TTR_LR_QR="1")
    r = subprocess.run([sys.executable, "-c", _LR_QR_SCRIPT, root, os.path.join(root, "oracle"), here],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr



_BATCH_CQR_SCRIPT = r"""
import sys, numpy as np
sys.path[:0] = [sys.argv[1], sys.argv[2], sys.argv[3]]
import paper_2511_03598_b200 as P, py_oracle as O
from test_gpu_parity import _padded_low_rank
# config-5a shapes, 64 tensors (TTR_BATCH_CQR=1: the per-tensor QRs of modes 2..6 by K4e)
b = P.TTBatch.two_part_philox(64, 8, 16, 16, 48, 1e-6, 1005)
o = P.round_fixed_krp_batched(b, [20] * 7, 7)
n, r = b.shape()[1], b.shape()[2]
no, ro = o.shape()[1], o.shape()[2]
for i in (0, 31, 63):
    xo = O.TT.from_flat(len(n), n, r, b.flats(i, 1)[0])
    ref = O.round_fixed_krp(xo, [20] * 7, O.derive_seed(7, i), rng=O.PHILOX)
    assert ro == ref.ranks, (ro, ref.ranks)
    assert O.relative_error(ref, O.TT.from_flat(len(no), no, ro, o.flats(i, 1)[0])) <= 1e-10
# exactly rank-deficient members (true rank 8 stored as 64): their sketches are
# singular, the Cholesky QR breaks down and those tensors are redone on the
# Householder path; the full-rank members keep the batched result
xs = [O.two_part_tt(8, 16, 16, 48, 1e-6, O.derive_seed(1005, i)) for i in range(6)]
for i in (1, 4):
    xs[i] = _padded_low_rank(O, [16] * 8, [1] + [8] * 7 + [1], [1] + [64] * 7 + [1], 50 + i)
bb = P.TTBatch.from_flats(n, r, [x.flat() for x in xs])
ob = P.round_fixed_krp_batched(bb, [20] * 7, 9)
for i in range(6):
    ref = O.round_fixed_krp(xs[i], [20] * 7, O.derive_seed(9, i), rng=O.PHILOX)
    got = O.TT.from_flat(len(no), no, ro, ob.flats(i, 1)[0])
    assert np.all(np.isfinite(got.flat()))
    assert O.relative_error(ref, got) <= 1e-10, i
print("ok")
"""


@pytest.mark.parametrize("mode", ["1", "0"])
def test_batched_cholesky_qr_modes(P, O, mode):
    """The batched sweep with its per-tensor QRs by batched CholeskyQR2/sCQR3
    (TTR_BATCH_CQR=1, the default) and by the batched Householder QR only
    (TTR_BATCH_CQR=0; read once per process, so in a subprocess): oracle parity on
    config-5a shapes, and rank-deficient members (Cholesky breakdown) redone on
    the Householder path."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    root = os.path.dirname(here)
    env = dict(os.environ, TTR_BATCH_CQR=mode)
    r = subprocess.run([sys.executable, "-c", _BATCH_CQR_SCRIPT, root, os.path.join(root, "oracle"), here],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr


def test_adaptive_plan_qr_breakdown_in_replay(P, O):
    """Sketch blocks tall enough for the fused Cholesky-QR kernel (K4f as the thin QR
    of the initial and growth blocks, rows > 512): the plan replays bitwise the
    eager call; refilled with an all-zero tensor every captured Cholesky-QR kernel
    breaks down (zero Gram matrix), the replay raises the plan's flag, the call is
    redone eagerly — checked QRs falling back to the Householder panels — and
    re-recorded with those QRs on the Householder path; the result is the zero
    tensor with the oracle's ranks, and the next replay needs no further redo."""
    x1 = O.two_part_tt(5, 48, 8, 28, 1e-6, 3401)
    cfg = P.AdaptiveConfig(tolerance=1e-4, f_init=0.1, f_inc=0.05, seed=7)
    t = to_device(x1)
    plan = P.AdaptiveKrpPlan(t, cfg)
    eager = P.round_adaptive_krp(to_device(x1), cfg)
    ref = O.round_adaptive_krp(x1, tolerance=1e-4, f_init=0.1, f_inc=0.05, seed=7, rng=O.PHILOX)
    plan.execute()
    assert np.array_equal(plan.output.flat(), eager.flat())
    assert eager.ranks() == ref.ranks and rel_err_vs_ref(ref, eager) <= 1e-10
    assert plan.rerecords() == 0
    zero = np.zeros_like(x1.flat())
    P.copy_from_host(t, zero)
    plan.execute()
    assert plan.rerecords() == 1
    out = plan.output
    assert np.all(np.isfinite(out.flat()))
    n, r, _ = x1.shape()
    xz = O.TT.from_flat(len(n), n, r, zero)
    refz = O.round_adaptive_krp(xz, tolerance=1e-4, f_init=0.1, f_inc=0.05, seed=7, rng=O.PHILOX)
    assert out.ranks() == refz.ranks
    assert P.norm_exact(out) == 0.0
    plan.execute()
    assert plan.rerecords() == 1
    plan.close()


def test_adaptive_plan_replays_and_rerecords(P, O):
    """ttr_plan_adaptive_krp: the graph replay of the recorded growth decisions is
    bitwise the eager call; refilled with data that decides differently, the plan
    notices on the device, redoes the call and re-records (output = eager on the
    new data, identical ranks to the oracle)."""
    x1 = O.two_part_tt(6, 16, 6, 30, 1e-6, 3301)
    x2 = O.two_part_tt(6, 16, 10, 26, 1e-3, 3302)  # same formal ranks, other decisions
    cfg = P.AdaptiveConfig(tolerance=1e-4, f_init=0.1, f_inc=0.05, seed=7)
    t = to_device(x1)
    plan = P.AdaptiveKrpPlan(t, cfg)
    eager = P.round_adaptive_krp(to_device(x1), cfg)
    for _ in range(2):
        plan.execute()
        assert np.array_equal(plan.output.flat(), eager.flat())
    assert plan.rerecords() == 0
    P.copy_from_host(t, x2.flat())
    plan.execute()
    assert plan.rerecords() == 1
    e2 = P.round_adaptive_krp(to_device(x2), cfg)
    assert plan.output.ranks() == e2.ranks()
    assert np.array_equal(plan.output.flat(), e2.flat())
    ref = O.round_adaptive_krp(x2, tolerance=1e-4, f_init=0.1, f_inc=0.05, seed=7, rng=O.PHILOX)
    assert e2.ranks() == ref.ranks
    plan.execute()  # replays the re-recorded graph
    assert plan.rerecords() == 1 and np.array_equal(plan.output.flat(), e2.flat())
    plan.close()
