"""T0: the seeded input generators (synth/) against the paper's printed sizes and
closed forms.  CPU only."""
import json
import os

import numpy as np
import pytest

import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _dense(ptr, col, val, n):
    D = np.zeros((n, n))
    for i in range(n):
        D[i, col[ptr[i]:ptr[i + 1]]] = val[ptr[i]:ptr[i + 1]]
    return D


def _check_csr(ptr, col, n):
    assert ptr[0] == 0 and np.all(np.diff(ptr) >= 0)
    assert col.min() >= 0 and col.max() < n
    rows = np.repeat(np.arange(n), np.diff(ptr))
    # strictly increasing columns inside each row
    same = rows[1:] == rows[:-1]
    assert np.all(col[1:][same] > col[:-1][same])


def test_paper_problem_sizes():
    """the 150^3 Poisson system has 3,375,000 unknowns and
    23,490,000 nonzeros; SPEC.md:542-544 small cases."""
    g = json.load(open(os.path.join(GOLD, "paper_problem_sizes.json")))
    for case in g["cases"]:
        ptr, col, val, f = synth.poisson3d(case["n"])
        assert len(ptr) - 1 == case["rows"]
        assert ptr[-1] == case["nnz"]
        if "value" in case:
            assert val.tolist() == [case["value"]]
        if case["n"] <= 2:
            _check_csr(ptr, col, case["rows"])


@pytest.mark.parametrize("dims", [(3, 4, 5), (7, 1, 2), (1, 1, 9), (5, 5, 5)])
def test_poisson_nnz_closed_form(dims):
    nx, ny, nz = dims
    ptr, col, val, f = synth.poisson3d(nx, ny, nz)
    N = nx * ny * nz
    assert ptr[-1] == 7 * N - 2 * (nx * ny + ny * nz + nx * nz)
    _check_csr(ptr, col, N)
    D = _dense(ptr, col, val, N)
    assert np.array_equal(D, D.T)
    # exact integer values 6(n+1)^2 and -(n+1)^2
    s = float((nx + 1) ** 2)
    assert set(np.unique(val).tolist()) <= {6 * s, -s}


def test_poisson_256_scaling_is_exact():
    """h = 1/257: 1/h^2 = 66049 and 6/h^2 = 396294 exactly (§8c)."""
    ptr, col, val, f = synth.poisson3d(2, h=1.0 / 257)
    assert 396294.0 in val and -66049.0 in val


def test_var_coef_symmetric_and_diag():
    ptr, col, val, f = synth.var_coef_poisson3d(6)
    N = 216
    _check_csr(ptr, col, N)
    D = _dense(ptr, col, val, N)
    assert np.array_equal(D, D.T)  # bitwise symmetric by construction
    off = D - np.diag(np.diag(D))
    assert np.all(off <= 0)
    # interior rows: diagonal = sum of |off-diagonals| (zero row sum up to rounding)
    idx = np.arange(N)
    x, y, z = idx % 6, (idx // 6) % 6, idx // 36
    interior = (x > 0) & (x < 5) & (y > 0) & (y < 5) & (z > 0) & (z < 5)
    rs = np.abs(off).sum(1)
    assert np.allclose(np.diag(D)[interior], rs[interior], rtol=1e-14, atol=0)
    assert np.all(np.diag(D)[~interior] > rs[~interior])
    assert np.all(np.linalg.eigvalsh(D) > 0)


def test_convdiff_stencil():
    ptr, col, val, f = synth.convdiff3d(4)
    N = 64
    D = _dense(ptr, col, val, N) / 25.0
    i = 1 + 4 * (1 + 4 * 1)  # interior node (1,1,1)
    assert D[i, i] == 9
    assert D[i, i - 1] == -2 and D[i, i - 4] == -2 and D[i, i - 16] == -2
    assert D[i, i + 1] == -1 and D[i, i + 4] == -1 and D[i, i + 16] == -1
    assert not np.array_equal(D, D.T)


def test_permutation_roundtrip():
    ptr, col, val, f = synth.poisson3d(4)
    f = np.arange(64, dtype=float)
    p2, c2, v2, f2 = synth.permute_symmetric(ptr, col, val, f)
    _check_csr(p2, c2, 64)
    perm = np.random.default_rng(synth.SEED_PERM).permutation(64)
    A = _dense(ptr, col, val, 64)
    B = _dense(p2, c2, v2, 64)
    assert np.array_equal(B, A[np.ix_(perm, perm)])
    assert np.array_equal(f2, f[perm])


def test_weak_poisson_shape():
    """configs[4] generator (§8c): n x n x (n P) box, h = 1/(n+1) in every
    direction, nnz = 7N - 2(nx ny + ny nz + nx nz); P = 1 is the cube problem."""
    n, P = 6, 3
    p, c, v, f = synth.weak_poisson(P, n)
    N = n * n * n * P
    assert len(f) == N and p[-1] == 7 * N - 2 * (n * n + n * n * P + n * n * P)
    d = np.repeat(np.arange(N), np.diff(p)) == c
    assert np.all(v[d] == 6.0 * (n + 1) ** 2) and np.all(v[~d] == -float((n + 1) ** 2))
    p1, c1, v1, f1 = synth.weak_poisson(1, n)
    q, e, w, g = synth.poisson3d(n)
    assert np.array_equal(p1, q) and np.array_equal(c1, e) and np.array_equal(v1, w)
    assert synth.problem_rows("poisson", n) == n ** 3 and np.array_equal(synth.rhs_slice("poisson", n, 2, 5), np.ones(3))
