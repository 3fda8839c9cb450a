"""K6 recompression kernel vs numpy's QR/SVD truncation (hmatrix.py:412-426)."""

import numpy as np
import pytest

from gold import golden

pytestmark = pytest.mark.gpu


def _lr(rng, m, n, r, decay=0.5):
    U = rng.standard_normal((m, r)) + 1j * rng.standard_normal((m, r))
    V = rng.standard_normal((r, n)) + 1j * rng.standard_normal((r, n))
    return U * (decay ** np.arange(r)), V


@pytest.mark.parametrize("m,n,k", [(30, 40, 5), (192, 192, 40), (384, 384, 90), (192, 384, 150), (108, 108, 40), (108, 108, 80), (108, 108, 120), (108, 54, 70),
                                   (60, 50, 80)])
def test_truncate_matches_numpy(m, n, k):
    from oracle.hcompress import truncate
    from paper_2408_17116_b200.lowrank import truncate_lowrank
    rng = np.random.default_rng(m + n + k)
    U, V = _lr(rng, m, n, k, 0.7)
    for tol in (1e-4, 1e-8):
        Ug, Vg = truncate_lowrank(U, V, tol)
        Uo, Vo = truncate(U, V, tol)
        assert abs(Ug.shape[1] - Uo.shape[1]) <= 1
        A = U @ V
        assert np.linalg.norm(Ug @ Vg - A) <= 2 * tol * np.linalg.norm(A, 2) * np.sqrt(min(m, n))
        assert np.linalg.norm(Ug @ Vg - Uo @ Vo) <= 2 * tol * np.linalg.norm(A, 2) * np.sqrt(min(m, n))


@pytest.mark.parametrize("m,n,k,case", [(384, 192, 60, "plain"), (1536, 768, 64, "plain"),
                                        (192, 384, 48, "unbalanced"), (384, 384, 64, "dependent"),
                                        (768, 96, 33, "zero_cols"), (50, 40, 64, "wide")])
def test_gram_path_truncation(m, n, k, case):
    """Gram-path recompression (k <= 64, tol >= 1e-5): balanced Grams + pivoted Cholesky.
    Cases: scaled factors (U tiny / V huge), linearly dependent concatenations, zero
    columns, k > min(m, n)."""
    from oracle.hcompress import truncate
    from paper_2408_17116_b200.lowrank import truncate_lowrank
    rng = np.random.default_rng(m * 7 + n + k)
    U, V = _lr(rng, m, n, k, 0.8)
    if case == "unbalanced":
        U[:, ::2] *= 1e-9
        V[::2] *= 1e9
    elif case == "dependent":
        U[:, k // 2:] = U[:, :k - k // 2] * (1 + 1e-3j)
    elif case == "zero_cols":
        U[:, 3] = 0
        V[7] = 0
    A = U @ V
    for tol in (1e-4, 1e-5):
        Ug, Vg = truncate_lowrank(U, V, tol)
        Uo, Vo = truncate(U, V, tol)
        assert abs(Ug.shape[1] - Uo.shape[1]) <= 1
        s0 = np.linalg.norm(A, 2)
        assert np.linalg.norm(Ug @ Vg - A, 2) <= 2 * tol * s0
        assert np.linalg.norm(Ug @ Vg - Uo @ Vo, 2) <= 3 * tol * s0


@pytest.mark.parametrize("m,n", [(108, 108), (192, 192), (150, 120)])
def test_dense_svd_truncation(m, n):
    from oracle.hcompress import svd_lowrank
    from paper_2408_17116_b200.lowrank import svd_truncate
    rng = np.random.default_rng(m * n)
    U, V = _lr(rng, m, n, min(m, n), 0.85)
    P = U @ V
    for tol in (1e-4, 1e-6):
        Wg, Zg = svd_truncate(P, tol)
        Wo, Zo = svd_lowrank(P, tol)
        assert abs(Wg.shape[1] - Wo.shape[1]) <= 1
        assert np.linalg.norm(Wg @ Zg - P, 2) <= 2 * tol * np.linalg.norm(P, 2)


def test_truncate_golden_kat():
    from paper_2408_17116_b200.lowrank import truncate_lowrank
    g = golden("aca.npz")
    UV = g["UV"]
    W, s, Zh = np.linalg.svd(UV)
    r = int(g["rank"])
    U = W[:, :r] * s[:r]
    Ut, Vt = truncate_lowrank(np.concatenate([U, 0.3 * U[:, :2]], 1),
                              np.concatenate([Zh[:r], Zh[:2] * 1j], 0), 1e-6)
    assert Ut.shape[1] == int(g["trunc_rank"])
    assert np.abs(Ut @ Vt - g["trunc_UV"]).max() <= 1e-12 * np.abs(g["trunc_UV"]).max()
