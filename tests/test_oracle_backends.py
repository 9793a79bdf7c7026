"""The oracle's OpenBLAS/LAPACK backend (used for the full-size parity checks
and the CPU baseline) restates the same algorithms as its plain-loop backend
(which tests/test_oracle_golden.py pins to the reference's own printed run):
identical rank vectors and agreement to rounding on every rounding path, plus
the pinned seeded-run numbers under the BLAS backend too."""
import pytest

import py_oracle as O

pytestmark = pytest.mark.skipif(not O.blas_available(), reason="oracle built without OpenBLAS")


@pytest.fixture
def blas():
    prev = O.backend()
    yield lambda: O.set_backend("blas", 4)
    O.set_backend(prev, 0)


def _both(fn, blas):
    O.set_backend("port", 4)
    a = fn()
    blas()
    b = fn()
    return a, b


@pytest.mark.parametrize("rng", [O.XOSHIRO, O.PHILOX])
def test_fixed_rank_agrees(blas, rng):
    x = O.two_part_tt(8, 20, 10, 40, 1e-4, 1001)
    a, b = _both(lambda: O.round_fixed_krp(x, [15] * 7, 7, rng=rng), blas)
    assert a.ranks == b.ranks
    assert O.relative_error(a, b) <= 1e-12


def test_deterministic_agrees(blas):
    x = O.two_part_tt(6, 16, 12, 30, 1e-6, 1003)
    for kw in (dict(ranks=[10] * 5), dict(eps=1e-5)):
        a, b = _both(lambda: O.round_deterministic(x, **kw), blas)
        assert a.ranks == b.ranks
        assert O.relative_error(a, b) <= 1e-12


def test_adaptive_agrees(blas):
    x = O.two_part_tt(8, 32, 30, 170, 1e-6, 1002)
    a, b = _both(lambda: O.round_adaptive_krp(x, tolerance=1e-4, f_init=0.1, f_inc=0.05, seed=7, rng=O.PHILOX), blas)
    assert a.ranks == b.ranks
    assert O.relative_error(a, b) <= 1e-10


def test_krp_contractions_agree(blas):
    x = O.two_part_tt(5, 12, 9, 21, 1e-3, 1005)
    f = O.draw_factors(x, 2, 17, 3, rng=O.PHILOX)
    a, b = _both(lambda: O.krp_contractions(x, f), blas)
    import numpy as np
    for wa, wb in zip(a, b):
        assert np.linalg.norm(wa - wb) <= 1e-12 * (1 + np.linalg.norm(wa))


def test_norm_and_error_agree(blas):
    x = O.two_part_tt(7, 10, 6, 14, 1e-2, 1006)
    y = O.two_part_tt(7, 10, 5, 9, 1e-2, 1007)
    (na, ea), (nb, eb) = _both(lambda: (O.norm_exact(x), O.relative_error(x, y)), blas)
    assert abs(na - nb) <= 1e-13 * na
    assert abs(ea - eb) <= 1e-12 * ea


def test_flop_charges_identical(blas):
    """The backend changes the arithmetic, never the charged flops (linalg.cpp:25-61)."""
    x = O.two_part_tt(6, 16, 8, 20, 1e-4, 1001)

    def run():
        O.flops_reset()
        O.round_fixed_krp(x, [12] * 5, 7, rng=O.PHILOX)
        O.round_deterministic(x, ranks=[6] * 5)
        return O.flops_get()
    a, b = _both(run, blas)
    assert a == b


def test_golden_numbers_under_blas(blas):
    """The reference's printed seeded-run numbers (proj/test_output.txt:29-31:
    criterion 3 det err 9.99e-06, criterion 5 norm-estimator bands 0.468 / 0.65 /
    0.878) also come out of the BLAS backend."""
    import numpy as np
    blas()
    syn = O.synthetic_perturbed_tt(5, 20, 10, 1e-5, 20250807)
    dense = syn.dense()
    det10 = O.round_deterministic(syn, ranks=[10] * 4)
    assert f"{np.linalg.norm(dense - det10.dense()) / np.linalg.norm(dense):.3g}" == "9.99e-06"
    for d, want in ((3, "0.468"), (4, "0.65"), (5, "0.878")):
        syn = O.synthetic_perturbed_tt(d, 15, 6, 1e-5, 5000 + d)
        truth = O.norm_exact(syn)
        es = np.array([O.estimate_norm_krp(syn, 64, O.derive_seed(31415, d * 10000 + t)) for t in range(1000)])
        assert f"{(es.max() - es.min()) / truth:.3g}" == want
