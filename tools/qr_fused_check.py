"""K4f check: thin_qr with the speculation tag (Cholesky-QR panels) on a few shapes,
against numpy: A = QR, Q^T Q = I, R upper; timing vs the Householder panels.
Run with TTR_QR_CQR=1 (the panels are read once per process)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_03598_b200 as P

rng = np.random.default_rng(5)

def check(name, a, expect_break=None):
    q, r, bd = P.thin_qr_speculative(a)
    if bd:
        print(f"{name}: breakdown flagged")
        assert expect_break is not False, name
        return
    assert expect_break is not True, name
    n = a.shape[1]
    orth = np.linalg.norm(q.T @ q - np.eye(n))
    res = np.linalg.norm(a - q @ r) / np.linalg.norm(a)
    low = np.linalg.norm(np.tril(r, -1))
    # column-wise residual (graded matrices)
    cres = np.max(np.linalg.norm(a - q @ r, axis=0) / np.maximum(np.linalg.norm(a, axis=0), 1e-300))
    print(f"{name}: orth {orth:.2e} res {res:.2e} colres {cres:.2e} tril {low:.1e}")
    assert orth <= 1e-12 * n and res <= 1e-13 and low == 0.0, name

for (m, n) in [(8192, 96), (20000, 110), (40960, 64), (3000, 40), (40960, 320)]:
    check(f"gauss {m}x{n}", rng.standard_normal((m, n)))
# graded columns + near dependence: cond ~ 1e9
m, n = 12000, 96
a = rng.standard_normal((m, n))
a[:, 40:] = a[:, :56] @ rng.standard_normal((56, 56)) * 1.0 + 1e-9 * rng.standard_normal((m, 56))
check("near-dependent 1e-9", a)
a = rng.standard_normal((m, n)) * np.logspace(0, -10, n)
check("graded 1e-10", a)
# the 5b sketch structure: rank 300 + 1e-8 x tail, 320 columns
m = 40960
u = rng.standard_normal((m, 300)) @ rng.standard_normal((300, 320)) + 1e-8 * rng.standard_normal((m, 320))
check("5b-like 40960x320", u)
# single-panel QRs (the adaptive growth blocks): the fused kernel as a plain thin QR
for (m, n) in [(25600, 16), (960, 10), (12800, 32), (3000, 5), (47000, 20)]:
    check(f"single-panel gauss {m}x{n}", rng.standard_normal((m, n)))
a = rng.standard_normal((25600, 16)) * np.logspace(0, -12, 16)
check("single-panel graded 1e-12", a)
# the checked (non-speculating) call: breakdown -> Householder rerun inside thin_qr
a = rng.standard_normal((9000, 30)) @ rng.standard_normal((30, 64))
q, r = P.thin_qr(a)
print("checked rank-deficient: orth", np.linalg.norm(q.T @ q - np.eye(64)), "res", np.linalg.norm(a - q @ r) / np.linalg.norm(a))
assert np.linalg.norm(q.T @ q - np.eye(64)) <= 1e-12 and np.linalg.norm(a - q @ r) <= 1e-13 * np.linalg.norm(a)
a = np.zeros((4000, 12)); a[:, :5] = rng.standard_normal((4000, 5))
q, r = P.thin_qr(a)
assert np.linalg.norm(a - q @ r) <= 1e-13 * np.linalg.norm(a), "zero columns"
# exactly rank deficient
a = rng.standard_normal((9000, 30)) @ rng.standard_normal((30, 64))
check("rank-deficient", a, expect_break=None)
print("ok")
