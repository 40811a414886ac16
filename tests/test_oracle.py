"""T1: the oracle (oracle/) pinned against what the paper and mathematics fix --
worked examples (tests/golden/, each with its citation), closed forms,
invariants, special cases that reduce to a library routine, and brute force on
tiny inputs.  CPU only.  See DESIGN.md §4 for the pin table."""
import json
import math
import os

import numpy as np
import pytest

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    return json.load(open(os.path.join(GOLD, name)))


def csr_from_dense(D):
    D = np.asarray(D, float)
    ptr, col, val = [0], [], []
    for i in range(D.shape[0]):
        for j in range(D.shape[1]):
            if D[i, j] != 0:
                col.append(j)
                val.append(D[i, j])
        ptr.append(len(col))
    return oracle.Csr(np.array(ptr), np.array(col, np.int32), np.array(val), D.shape[1])


def problem(case):
    kind = case["problem"]
    if kind == "dense":
        return csr_from_dense(case["dense"])
    if kind == "poisson1d":
        p, c, v, _ = synth.poisson1d(case["n"])
    elif kind == "poisson2d":
        p, c, v, _ = synth.poisson2d(case["n"])
    elif kind == "poisson3d_unit":
        p, c, v, _ = synth.poisson3d(case["n"], scaled=False)
    else:
        raise ValueError(kind)
    return oracle.Csr(p, c, v)


def poisson(n, **kw):
    p, c, v, f = synth.poisson3d(n, **kw)
    return oracle.Csr(p, c, v), f


# ---------------------------------------------------------------- strength

def test_strength_examples():
    for case in gold("strength_examples.json")["cases"]:
        A = csr_from_dense(case["dense"])
        S = oracle.strength(A, case["eps"])
        rows = np.repeat(np.arange(A.nrows), np.diff(A.ptr))
        got = sorted([int(rows[k]), int(A.col[k])] for k in range(A.nnz) if S[k])
        assert got == sorted(case["strong_offdiag"])


def test_strength_rejects_nonpositive_diagonal():
    with pytest.raises(oracle.OracleError):
        oracle.strength(csr_from_dense([[1, -1], [-1, 0.0]]))
    with pytest.raises(oracle.OracleError):
        oracle.strength(csr_from_dense([[-1, 0.5], [0.5, 2]]))


def test_strength_poisson_all_strong_and_symmetric():
    A, _ = poisson(5)
    S = oracle.strength(A)
    rows = np.repeat(np.arange(A.nrows), np.diff(A.ptr))
    off = rows != A.col
    assert np.all(S[off] == 1) and np.all(S[~off] == 0)


# ------------------------------------------------------------- aggregation

def test_aggregation_examples():
    for case in gold("aggregation_examples.json")["cases"]:
        A = problem(case)
        idv, cnt = oracle.aggregate(A, oracle.strength(A))
        assert idv.tolist() == case["id"], case["name"]
        assert cnt == case["count"], case["name"]


def _aggregation_invariants(A, S, idv, cnt):
    n = A.nrows
    assert idv.min() == 0 and idv.max() == cnt - 1
    assert len(np.unique(idv)) == cnt  # every aggregate non-empty
    # aggregates are connected in the strength graph
    rows = np.repeat(np.arange(n), np.diff(A.ptr))
    import scipy.sparse as sp
    import scipy.sparse.csgraph as cg
    m = S.astype(bool) & (idv[rows] == idv[A.col])
    G = sp.csr_matrix((np.ones(m.sum()), (rows[m], A.col[m])), shape=(n, n))
    ncomp, lab = cg.connected_components(G, directed=False)
    # each aggregate is exactly one connected component
    pairs = set(zip(idv.tolist(), lab.tolist()))
    assert len(pairs) == cnt


@pytest.mark.parametrize("gen", ["poisson", "varcoef", "convdiff", "poisson_perm"])
def test_aggregation_invariants(gen):
    p, c, v, _ = synth.problem(gen, 9)
    A = oracle.Csr(p, c, v)
    S = oracle.strength(A)
    idv, cnt = oracle.aggregate(A, S)
    assert b"phase 3" not in oracle.lib().or_last_error()  # Phase 3 never fires (§8c L2 v)
    _aggregation_invariants(A, S, idv, cnt)
    assert cnt < A.nrows


def test_aggregation_deterministic():
    A, _ = poisson(8)
    S = oracle.strength(A)
    a1 = oracle.aggregate(A, S)[0]
    a2 = oracle.aggregate(A, S)[0]
    assert np.array_equal(a1, a2)


# ------------------------------------------------------------ prolongation

def test_tentative_p():
    """indicator matrix, row sums 1, Pt^T Pt = diag(sizes)."""
    idv = np.array([0, 0, 1, 1, 1, 1], np.int32)
    Pt = oracle.tentative_p(idv, 2)
    D = Pt.to_dense()
    assert np.array_equal(D.sum(1), np.ones(6))
    assert np.array_equal(D.T @ D, np.diag([2.0, 4.0]))
    A, _ = poisson(6)
    idv, cnt = oracle.aggregate(A, oracle.strength(A))
    D = oracle.tentative_p(idv, cnt).to_dense()
    assert np.array_equal(D.sum(1), np.ones(A.nrows))
    assert np.array_equal(D.T @ D, np.diag(np.bincount(idv).astype(float)))


def test_smoothed_p_examples():
    for case in gold("smoothed_p_examples.json")["cases"]:
        A = problem(case)
        S = oracle.strength(A)
        idv, cnt = oracle.aggregate(A, S)
        P = oracle.smooth_p(A, S, idv, cnt).to_dense()
        if "P" in case:
            np.testing.assert_allclose(P, case["P"], rtol=1e-15, atol=0)
        else:
            np.testing.assert_allclose(P * 9, case["P_times_9"], rtol=1e-14, atol=1e-14)


def test_smoothed_p_diagonal_matrix_is_scaled_tentative():
    """SPEC.md:221 (garbled; §8c): A diagonal -> P = (1 - omega) Pt."""
    A = csr_from_dense(np.diag([2.0, 3.0, 5.0]))
    S = oracle.strength(A)
    idv, cnt = oracle.aggregate(A, S)
    P = oracle.smooth_p(A, S, idv, cnt, omega=2.0 / 3.0).to_dense()
    assert np.array_equal(P, (1.0 - 2.0 / 3.0) * np.eye(3))


def test_smoothed_p_omega_zero_is_tentative():
    A, _ = poisson(5)
    S = oracle.strength(A)
    idv, cnt = oracle.aggregate(A, S)
    P0 = oracle.smooth_p(A, S, idv, cnt, omega=0.0).to_dense()
    assert np.array_equal(P0, oracle.tentative_p(idv, cnt).to_dense())


def test_smoothed_p_row_sums():
    """Row sum of P = 1 - omega * (sum_j A_F(i,j)) / D_F(i): exactly 1 where the
    filtered row sums to zero (interior Poisson rows), < 1 at Dirichlet rows."""
    A, _ = poisson(7, scaled=False)
    S = oracle.strength(A)
    idv, cnt = oracle.aggregate(A, S)
    P = oracle.smooth_p(A, S, idv, cnt)
    rs = P.to_dense().sum(1)
    deg = np.diff(A.ptr) - 1
    interior = deg == 6
    np.testing.assert_allclose(rs[interior], 1.0, rtol=0, atol=1e-15)
    # boundary: row sum of A is 6 - deg, D_F = 6 -> 1 - (2/3)(6-deg)/6
    np.testing.assert_allclose(rs[~interior], 1 - (2 / 3) * (6 - deg[~interior]) / 6, atol=1e-15)


# --------------------------------------------------------- transpose, SpGEMM

def _random_sparse(rng, m, n, density):
    D = rng.standard_normal((m, n)) * (rng.random((m, n)) < density)
    return D


def test_transpose_and_spgemm_vs_dense():
    """spgemm equals the dense product to 1e-12 max|entry| for n <= 50."""
    rng = np.random.default_rng(0)
    for trial in range(20):
        m, k, n = rng.integers(1, 50, 3)
        A = _random_sparse(rng, m, k, 0.2)
        B = _random_sparse(rng, k, n, 0.2)
        cA, cB = csr_from_dense(A), csr_from_dense(B)
        assert np.array_equal(oracle.transpose(cA).to_dense(), A.T)
        C = oracle.spgemm(cA, cB)
        ref = A @ B
        assert np.max(np.abs(C.to_dense() - ref)) <= 1e-12 * max(1.0, np.abs(ref).max())
        # structural pattern: (i,J) present iff some k has A(i,k) != 0 and B(k,J) != 0
        pat = (np.abs(A) > 0).astype(int) @ (np.abs(B) > 0).astype(int) > 0
        got = np.zeros_like(pat)
        rows = np.repeat(np.arange(C.nrows), np.diff(C.ptr))
        got[rows, C.col] = True
        assert np.array_equal(got, pat)


def test_spgemm_keeps_cancellation_zeros():
    """structural zeros from cancellation are kept."""
    A = csr_from_dense([[1.0, 1.0]])
    B = csr_from_dense([[1.0], [-1.0]])
    C = oracle.spgemm(A, B)
    assert C.nnz == 1 and C.val[0] == 0.0


# ------------------------------------------------------------------- RAP

def _two_level(A, smoothed):
    S = oracle.strength(A)
    idv, cnt = oracle.aggregate(A, S)
    P = oracle.smooth_p(A, S, idv, cnt) if smoothed else oracle.tentative_p(idv, cnt)
    R = oracle.transpose(P)
    return P, R, oracle.spgemm(R, oracle.spgemm(A, P))


def test_rap_examples():
    for case in gold("rap_examples.json")["cases"]:
        A = problem(case)
        P, R, Ac = _two_level(A, case["smoothed"])
        D = Ac.to_dense()
        if "Ac" in case:
            assert np.array_equal(D, np.array(case["Ac"], float)), case["name"]
        else:
            key = [k for k in case if k.startswith("Ac_times_")][0]
            s = float(key.split("_")[-1])
            np.testing.assert_allclose(D * s, case[key], rtol=1e-14, atol=1e-13)


def test_rap_1d_plain_gives_1d_stencil():
    """Plain aggregation of the 1D Laplacian with contiguous aggregates gives
    exactly the 1D stencil [-1, 2, -1] (first/last row 1 plus Dirichlet 1)."""
    p, c, v, _ = synth.poisson1d(30)
    A = oracle.Csr(p, c, v)
    P, R, Ac = _two_level(A, smoothed=False)
    D = Ac.to_dense()
    m = D.shape[0]
    ref = 2 * np.eye(m) - np.eye(m, k=1) - np.eye(m, k=-1)
    assert np.array_equal(D, ref)


def test_rap_2d_box_aggregates():
    """2D unit 5-point with a x b box aggregates (plain): diagonal 2(a+b),
    x-neighbour -b, y-neighbour -a, in the interior of the coarse grid."""
    nx = ny = 12
    a, b = 3, 2
    p, c, v, _ = synth.poisson2d(nx, ny)
    A = oracle.Csr(p, c, v)
    idx = np.arange(nx * ny)
    X, Y = idx % nx, idx // nx
    cx = nx // a
    idv = ((X // a) + cx * (Y // b)).astype(np.int32)
    Pt = oracle.tentative_p(idv, cx * (ny // b))
    Ac = oracle.spgemm(oracle.transpose(Pt), oracle.spgemm(A, Pt)).to_dense()
    I = 1 + cx * 1  # an interior coarse node (1,1)
    # block sum: 4ab (diagonals) - 2 (internal edges)
    internal_edges = (a - 1) * b + (b - 1) * a
    assert Ac[I, I] == 4 * a * b - 2 * internal_edges
    assert 4 * a * b - 2 * internal_edges == 2 * (a + b)
    assert Ac[I, I + 1] == -b and Ac[I, I - 1] == -b
    assert Ac[I, I + cx] == -a and Ac[I, I - cx] == -a


def test_rap_plain_preserves_total_sum():
    A, _ = poisson(6, scaled=False)
    P, R, Ac = _two_level(A, smoothed=False)
    assert Ac.val.sum() == A.val.sum()


@pytest.mark.parametrize("gen", ["poisson", "varcoef", "poisson_perm"])
def test_rap_galerkin_symmetric(gen):
    p, c, v, _ = synth.problem(gen, 8)
    A = oracle.Csr(p, c, v)
    P, R, Ac = _two_level(A, smoothed=True)
    D = Ac.to_dense()
    assert np.max(np.abs(D - D.T)) <= 1e-12 * np.abs(D).max()
    # R is exactly P^T
    assert np.array_equal(R.to_dense(), P.to_dense().T)
    # brute force: dense R A P
    ref = P.to_dense().T @ A.to_dense() @ P.to_dense()
    assert np.max(np.abs(D - ref)) <= 1e-12 * np.abs(ref).max()


# -------------------------------------------------------------- smoothers

def test_spai0_examples():
    """[[2,-1],[-1,2]] -> 0.4; unit 3D Poisson interior 6/42,
    face 6/41, edge 6/40, corner 6/39 (closed form a_ii / sum_j a_ij^2)."""
    A = csr_from_dense([[2, -1], [-1, 2]])
    h = oracle.Hierarchy(A, coarse_enough=1, max_levels=2)
    # 2x2 aggregates into one -> two levels
    assert h.nlevels == 2
    np.testing.assert_allclose(h.smoother(0), [0.4, 0.4], rtol=1e-15)
    A, _ = poisson(4, scaled=False)
    h = oracle.Hierarchy(A, coarse_enough=10)
    m = h.smoother(0)
    deg = np.diff(A.ptr) - 1
    for d, ref in ((6, 6 / 42), (5, 6 / 41), (4, 6 / 40), (3, 6 / 39)):
        np.testing.assert_allclose(m[deg == d], ref, rtol=1e-15)


def test_spai0_is_frobenius_optimal():
    """SPAI-0 minimises |I - M A|_F over diagonal M."""
    p, c, v, _ = synth.var_coef_poisson3d(3)
    A = oracle.Csr(p, c, v)
    h = oracle.Hierarchy(A, coarse_enough=5)
    m = h.smoother(0)
    D = A.to_dense()
    base = np.linalg.norm(np.eye(27) - np.diag(m) @ D)
    for i in range(27):
        for s in (1e-3, -1e-3):
            mm = m.copy()
            mm[i] *= 1 + s
            assert np.linalg.norm(np.eye(27) - np.diag(mm) @ D) > base


def test_jacobi_setup_and_exact_diagonal_sweep():
    """Jacobi m = omega/a_ii; omega = 1 on a diagonal system is
    exact in one sweep."""
    A = csr_from_dense(np.diag([2.0, 4.0, 8.0, 16.0]))
    h = oracle.Hierarchy(A, coarse_enough=1, relax="damped_jacobi", jacobi_omega=1.0,
                         max_levels=3)
    # diagonal matrix: every row is its own aggregate -> stagnation -> 1 level
    assert h.nlevels == 1
    A, _ = poisson(4)
    h = oracle.Hierarchy(A, coarse_enough=10, relax="damped_jacobi")
    np.testing.assert_allclose(h.smoother(0), 0.72 / A.to_dense().diagonal(), rtol=1e-15)
    hb = oracle.Hierarchy(csr_from_dense([[2.0, -1], [-1, 2]]), coarse_enough=1,
                          relax="damped_jacobi", jacobi_omega=1.0)
    x = hb.relax(0, np.array([2.0, 4.0]), np.zeros(2))
    np.testing.assert_allclose(x, [1.0, 2.0], rtol=1e-15)  # omega/a_ii * f from zero


def _cheb_T(K, t):
    t = np.asarray(t, float)
    out = np.where(np.abs(t) <= 1, np.cos(K * np.arccos(np.clip(t, -1, 1))),
                   np.cosh(K * np.arccosh(np.maximum(np.abs(t), 1))) * np.sign(t) ** K)
    return out


def test_chebyshev_bounds():
    """§8c: Gershgorin bound of D^-1 A is exactly 2 on the fine
    constant-coefficient Poisson matrix; A = I -> lmax = 1, lmin = 1/30."""
    A, _ = poisson(6)
    h = oracle.Hierarchy(A, coarse_enough=20, relax="chebyshev")
    lmax, lmin, d, c = h.smoother(0)
    assert lmax == 2.0 and lmin == 2.0 / 30
    assert d == (lmax + lmin) / 2 and c == (lmax - lmin) / 2
    h = oracle.Hierarchy(csr_from_dense([[1.0, 0.0], [0.0, 1.0]]), coarse_enough=1,
                         relax="chebyshev")
    assert h.nlevels == 1  # identity: stagnation


@pytest.mark.parametrize("scaled", [0, 1])
def test_chebyshev_relax_closed_form(scaled):
    """K steps of the Chebyshev recurrence from x = 0 equal the closed-form
    Chebyshev polynomial: x = (I - T_K((dI - M)/c) / T_K(d/c)) M^-1 g, with
    M = D^-1 A, g = D^-1 f (scaled) or M = A, g = f (unscaled); T_K evaluated
    with cos/cosh (textbook Chebyshev iteration, Saad 2003 §12.3)."""
    p, c, v, _ = synth.poisson1d(40)
    A = oracle.Csr(p, c, v)
    h = oracle.Hierarchy(A, coarse_enough=5, relax="chebyshev", cheb_scaled=scaled)
    lmax, lmin, d, cc = h.smoother(0)
    Ad = A.to_dense()
    M = np.diag(1 / np.diag(Ad)) @ Ad if scaled else Ad
    f = synth.random_vector(40)
    x = h.relax(0, f, np.zeros(40))
    # error polynomial: x = (I - T_K((dI - M)/c)/T_K(d/c)) M^-1 (D^-1 f or f)
    w, V = np.linalg.eig(M)
    K = 5
    pw = 1 - _cheb_T(K, (d - w.real) / cc) / _cheb_T(K, d / cc)
    rhs = (f / np.diag(Ad)) if scaled else f
    ref = (V @ np.diag(pw / w.real) @ np.linalg.inv(V) @ rhs).real
    np.testing.assert_allclose(x, ref, rtol=1e-9, atol=1e-12 * np.abs(ref).max())


def test_smoother_shift_invariance_and_fixed_point():
    """relax(x + delta, f + A delta) = relax(x, f) + delta; f = A u
    leaves u unchanged."""
    for relax in ("spai0", "damped_jacobi", "chebyshev"):
        A, _ = poisson(5)
        h = oracle.Hierarchy(A, coarse_enough=10, relax=relax)
        n = A.nrows
        rng = np.random.default_rng(1)
        x, f, dl = rng.standard_normal((3, n))
        Ad = A.to_dense()
        lhs = h.relax(0, f + Ad @ dl, x + dl)
        rhs = h.relax(0, f, x) + dl
        np.testing.assert_allclose(lhs, rhs, rtol=0, atol=1e-12 * np.abs(rhs).max())
        u = rng.standard_normal(n)
        np.testing.assert_allclose(h.relax(0, Ad @ u, u), u, rtol=1e-12)


def test_smoothers_contract_1d():
    """10 sweeps with f = 0 reduce |u| on 1D Poisson n = 32."""
    p, c, v, _ = synth.poisson1d(32)
    A = oracle.Csr(p, c, v)
    for relax in ("spai0", "damped_jacobi", "chebyshev"):
        h = oracle.Hierarchy(A, coarse_enough=4, relax=relax)
        u = synth.random_vector(32)
        n0 = np.linalg.norm(u)
        for _ in range(10):
            u = h.relax(0, np.zeros(32), u)
        assert np.linalg.norm(u) < n0


# -------------------------------------------------------- coarse LU solve

def test_lu_matches_library_solve():
    rng = np.random.default_rng(3)
    for n in (1, 2, 5, 40, 120):
        A = rng.standard_normal((n, n)) + n * np.eye(n) * (rng.random() < 0.5)
        b = rng.standard_normal(n)
        lu, piv = oracle.lu_factor(A)
        x = oracle.lu_solve(lu, piv, b)
        ref = np.linalg.solve(A, b)
        assert np.linalg.norm(A @ x - b) <= 1e-10 * np.linalg.norm(b) * np.linalg.cond(A) / 1e2 + 1e-12
        np.testing.assert_allclose(x, ref, rtol=1e-8, atol=1e-10)
        # PA = LU to 1e-10
        L = np.tril(lu, -1) + np.eye(n)
        U = np.triu(lu)
        PA = A.copy()
        for k in range(n):
            PA[[k, piv[k]]] = PA[[piv[k], k]]
        assert np.max(np.abs(PA - L @ U)) <= 1e-10 * np.abs(A).max()


def test_lu_singular_is_error():
    with pytest.raises(oracle.OracleError):
        oracle.lu_factor(np.array([[1.0, 2.0], [2.0, 4.0]]))


# ----------------------------------------------------------------- setup

def test_hierarchy_single_level_and_stagnation():
    """size <= coarse_enough -> one level; identity ->
    stagnation -> dense solve."""
    A, _ = poisson(4)
    h = oracle.Hierarchy(A, coarse_enough=64)
    assert h.nlevels == 1
    I = csr_from_dense(np.eye(10))
    h = oracle.Hierarchy(I, coarse_enough=1)
    assert h.nlevels == 1
    with pytest.raises(oracle.OracleError):
        oracle.Hierarchy(A, coarse_enough=1, dense_max=10, max_levels=1)


def test_hierarchy_sizes_decrease_and_complexity():
    """sizes strictly decrease; operator complexity < 2 and
    grid complexity < 1.5 at 32^3."""
    A, _ = poisson(16)
    h = oracle.Hierarchy(A, coarse_enough=100)
    rows = [h.info(l)["rows"] for l in range(h.nlevels)]
    assert all(a > b for a, b in zip(rows, rows[1:])) and len(rows) >= 2
    A, _ = poisson(32)
    h = oracle.Hierarchy(A)
    op, grid = h.complexities()
    assert op < 2.0 and grid < 1.5
    for l in range(h.nlevels - 1):
        P = h.matrix(l, "P")
        assert np.all(np.diff(P.ptr) >= 1)  # no empty rows of P
        assert np.array_equal(h.matrix(l, "R").to_dense() if P.nrows < 5000 else 0,
                              P.to_dense().T if P.nrows < 5000 else 0)


def test_hierarchy_levels_match_components():
    """Level l+1 of or_setup equals R (A P) built from the single operations,
    with the per-level strength threshold eps_l = 0.08 * 0.5^l (R1)."""
    A, _ = poisson(10)
    h = oracle.Hierarchy(A, coarse_enough=50)
    Al = A
    for l in range(h.nlevels - 1):
        S = oracle.strength(Al, 0.08 * 0.5 ** l)
        idv, cnt = oracle.aggregate(Al, S)
        assert np.array_equal(idv, h.aggregates(l))
        P = oracle.smooth_p(Al, S, idv, cnt)
        Pl = h.matrix(l, "P")
        assert np.array_equal(P.ptr, Pl.ptr) and np.array_equal(P.col, Pl.col)
        assert np.array_equal(P.val, Pl.val)
        Ac = oracle.spgemm(oracle.transpose(P), oracle.spgemm(Al, P))
        An = h.matrix(l + 1, "A")
        assert np.array_equal(Ac.ptr, An.ptr) and np.array_equal(Ac.col, An.col)
        assert np.array_equal(Ac.val, An.val)
        Al = An


# ---------------------------------------------------------------- V-cycle

def test_vcycle_single_level_is_direct_solve():
    A, f = poisson(5)
    h = oracle.Hierarchy(A, coarse_enough=1000)
    assert h.nlevels == 1
    z = h.precond(f)
    assert np.linalg.norm(A.to_dense() @ z - f) <= 1e-10 * np.linalg.norm(f)


def test_vcycle_zero_rhs_and_linearity_and_symmetry():
    """SPEC.md:359, 366-368, 378-379."""
    for relax in ("spai0", "damped_jacobi", "chebyshev"):
        A, _ = poisson(10)
        h = oracle.Hierarchy(A, coarse_enough=50, relax=relax)
        n = A.nrows
        assert np.all(h.precond(np.zeros(n)) == 0)
        rng = np.random.default_rng(7)
        r1, r2 = rng.standard_normal((2, n))
        a, b = 0.7, -1.3
        z = h.precond(a * r1 + b * r2)
        ref = a * h.precond(r1) + b * h.precond(r2)
        assert np.linalg.norm(z - ref) <= 1e-11 * np.linalg.norm(ref)
        lhs = h.precond(r1) @ r2
        rhs = r1 @ h.precond(r2)
        assert abs(lhs - rhs) <= 1e-10 * abs(lhs)


def _dense_vcycle_operator(h, l):
    """Brute-force error-propagation operator E_l of Algorithm 2 from dense
    factors: E_L = 0 (exact solve);
    E_l = S_l (I - P_l (I - E_{l+1}) A_{l+1}^-1 R_l A_l) S_l for npre = npost = 1."""
    A = h.matrix(l, "A").to_dense()
    n = A.shape[0]
    if l == h.nlevels - 1:
        return np.zeros((n, n))
    P = h.matrix(l, "P").to_dense()
    R = h.matrix(l, "R").to_dense()
    Ac = h.matrix(l + 1, "A").to_dense()
    Ec = _dense_vcycle_operator(h, l + 1)
    if h.prm.relax == 2:
        lmax, lmin, d, c = h.smoother(l)
        M = np.diag(1 / np.diag(A)) @ A
        w, V = np.linalg.eig(M)
        pw = _cheb_T(h.prm.cheb_degree, (d - w.real) / c) / _cheb_T(h.prm.cheb_degree, d / c)
        S = (V @ np.diag(pw) @ np.linalg.inv(V)).real
    else:
        S = np.eye(n) - np.diag(h.smoother(l)) @ A
    C = np.eye(n) - P @ (np.eye(Ac.shape[0]) - Ec) @ np.linalg.solve(Ac, R @ A)
    return S @ C @ S


@pytest.mark.parametrize("relax", ["spai0", "damped_jacobi", "chebyshev"])
def test_vcycle_brute_force(relax):
    """M = (I - E) A^-1 with E the dense V-cycle error operator (2-3 levels)."""
    A, _ = poisson(7)
    h = oracle.Hierarchy(A, coarse_enough=20, relax=relax)
    assert h.nlevels >= 3
    E = _dense_vcycle_operator(h, 0)
    Ad = A.to_dense()
    Mref = (np.eye(A.nrows) - E) @ np.linalg.inv(Ad)
    r = synth.random_vector(A.nrows)
    z = h.precond(r)
    ref = Mref @ r
    assert np.linalg.norm(z - ref) <= 1e-10 * np.linalg.norm(ref)


def test_stationary_vcycle_contracts():
    """SPEC.md:380 / §8c: u <- u + M (f - A u) on 16^3 Poisson decreases the
    residual strictly monotonically, by a factor < 0.5 per cycle after the first
    cycle (checked over 8 cycles; the asymptotic factor approaches ~0.55)."""
    A, f = poisson(16)
    h = oracle.Hierarchy(A, coarse_enough=100)
    Ad_mv = lambda x: oracle.spmv(A, x)
    u = np.zeros(A.nrows)
    res = [np.linalg.norm(f)]
    for _ in range(8):
        u = h.vcycle(0, f, u)
        res.append(np.linalg.norm(f - Ad_mv(u)))
    ratios = np.array(res[1:]) / np.array(res[:-1])
    assert np.all(ratios < 1.0) and np.all(ratios[1:] < 0.5), ratios
    # same through or_vcycle starting from u vs u + precond(f - Au)
    u2 = u + h.precond(f - Ad_mv(u))
    u3 = h.vcycle(0, f, u)
    np.testing.assert_allclose(u3, u2, rtol=1e-10, atol=1e-14 * np.abs(u2).max())


# --------------------------------------------------------------------- CG

def test_cg_identity_and_diag():
    """SPEC.md:420-421."""
    I = csr_from_dense(np.eye(5))
    f = np.arange(1.0, 6.0)
    r = oracle.cg(I, f)
    assert r["iters"] == 1 and np.allclose(r["x"], f, rtol=1e-15)
    D = csr_from_dense(np.diag([1.0, 2.0, 3.0]))
    r = oracle.cg(D, np.ones(3), tol=1e-12)
    assert r["iters"] <= 3
    np.testing.assert_allclose(r["x"], [1, 0.5, 1 / 3], rtol=1e-12)


def test_cg_finite_termination_distinct_eigenvalues():
    """CG terminates in k iterations for k distinct eigenvalues (exact arithmetic
    bound; here k = 4 with repeated eigenvalues on a 40x40 diagonal)."""
    d = np.repeat([1.0, 2.0, 5.0, 11.0], 10)
    r = oracle.cg(csr_from_dense(np.diag(d)), np.ones(40), tol=1e-12)
    assert r["iters"] == 4


def test_cg_unpreconditioned_poisson_and_scaling_invariance():
    """iteration count invariant under (alpha A, alpha f);
    solution equals the dense direct solve."""
    p, c, v, f = synth.poisson2d(8)
    A = oracle.Csr(p, c, v)
    base = oracle.cg(A, f, tol=1e-8)
    np.testing.assert_allclose(base["x"], np.linalg.solve(A.to_dense(), f), rtol=1e-7)
    assert base["iters"] <= 65  # n + 1
    for a in (1e-3, 1e3, 2.0 ** -10, 2.0 ** 10):
        r = oracle.cg(oracle.Csr(p, c, v * a), f * a, tol=1e-8)
        assert r["iters"] == base["iters"]


def test_cg_a_norm_error_monotone():
    """§8c: CG's A-norm error decreases monotonically (tiny grid, AMG-preconditioned)."""
    A, f = poisson(6)
    h = oracle.Hierarchy(A, coarse_enough=20)
    Ad = A.to_dense()
    xs = np.linalg.solve(Ad, f)
    errs = []
    for k in range(1, 8):
        r = oracle.cg(A, f, tol=0.0, maxiter=k, hier=h)
        e = r["x"] - xs
        errs.append(e @ Ad @ e)
    assert all(b < a for a, b in zip(errs, errs[1:]) if a > 1e-28)


def test_cg_amg_small_grids_and_true_residual():
    """true residual reported; <= 30 its at 32^3 and
    growth <= 1.5x per refinement; tiny grids match the dense solve."""
    A, f = poisson(6)
    h = oracle.Hierarchy(A, coarse_enough=20)
    r = oracle.cg(A, f, hier=h, tol=1e-10)
    np.testing.assert_allclose(r["x"], np.linalg.solve(A.to_dense(), f), rtol=1e-8)
    its = []
    for n in (16, 32):
        A, f = poisson(n)
        h = oracle.Hierarchy(A)
        r = oracle.cg(A, f, hier=h)
        assert r["status"] == oracle.OK
        true = np.linalg.norm(f - oracle.spmv(A, r["x"])) / np.linalg.norm(f)
        assert abs(true - r["rel_resid"]) <= 1e-12
        assert r["rel_resid"] <= 1.01e-8
        its.append(r["iters"])
    assert its[1] <= 30 and its[1] <= 1.5 * its[0]


def test_cg_zero_rhs_and_breakdown():
    A, f = poisson(4)
    r = oracle.cg(A, np.zeros(A.nrows), x0=np.ones(A.nrows))
    assert r["iters"] == 0 and np.all(r["x"] == 0) and r["rel_resid"] == 0
    N = csr_from_dense(-np.eye(3))
    r = oracle.cg(N, np.ones(3))
    assert r["status"] == oracle.BREAKDOWN


# --------------------------------------------------------------- BiCGStab

def test_bicgstab_examples():
    """SPEC.md:429-431."""
    r = oracle.bicgstab(csr_from_dense(np.eye(4)), np.arange(1.0, 5.0))
    assert r["iters"] == 1
    A = csr_from_dense([[2.0, 1.0], [0.0, 2.0]])
    r = oracle.bicgstab(A, np.array([3.0, 2.0]))
    assert r["rel_resid"] <= 1e-8
    np.testing.assert_allclose(r["x"], [1.0, 1.0], rtol=1e-8)
    r = oracle.bicgstab(A, np.zeros(2))
    assert r["iters"] == 0 and r["status"] == oracle.OK


def test_bicgstab_amg_convdiff():
    p, c, v, f = synth.convdiff3d(10)
    A = oracle.Csr(p, c, v)
    h = oracle.Hierarchy(A, coarse_enough=50, relax="damped_jacobi")
    r = oracle.bicgstab(A, f, hier=h, tol=1e-10)
    assert r["status"] == oracle.OK
    np.testing.assert_allclose(r["x"], np.linalg.solve(A.to_dense(), f), rtol=1e-8)
    assert r["vcycles"] in (2 * r["iters"], 2 * r["iters"] - 1)


# --------------------------------------------------------------------- GMRES

def test_gmres_examples():
    """A = I: one step; the SPEC's non-symmetric 2x2 example is
    solved in <= 2 steps; f = 0 -> 0 steps."""
    r = oracle.gmres(csr_from_dense(np.eye(4)), np.arange(1.0, 5.0))
    assert r["iters"] == 1 and np.allclose(r["x"], np.arange(1.0, 5.0), rtol=1e-15)
    A = csr_from_dense([[2.0, 1.0], [0.0, 2.0]])
    r = oracle.gmres(A, np.array([3.0, 2.0]), tol=1e-12)
    assert r["iters"] <= 2
    np.testing.assert_allclose(r["x"], [1.0, 1.0], rtol=1e-12)
    r = oracle.gmres(A, np.zeros(2))
    assert r["iters"] == 0 and r["status"] == oracle.OK


def test_gmres_minimises_residual_over_krylov_space():
    """Brute force: after k steps (no restart, M = I, x0 = 0) GMRES returns
    argmin_{x in K_k(A, f)} |f - A x|, computed here from an explicit Krylov
    basis with numpy least squares; the residual estimate is non-increasing."""
    rng = np.random.default_rng(11)
    n = 24
    D = np.eye(n) * 4 + rng.standard_normal((n, n)) * 0.4
    A = csr_from_dense(D)
    f = rng.standard_normal(n)
    for k in range(1, 9):
        r = oracle.gmres(A, f, tol=0.0, maxiter=k, m=50, history=True)
        K = np.empty((n, k))
        v = f / np.linalg.norm(f)
        for j in range(k):  # orthonormal Krylov basis (numpy QR for stability)
            K[:, j] = v
            Q, _ = np.linalg.qr(K[:, :j + 1])
            v = D @ Q[:, j]
        Q, _ = np.linalg.qr(K)
        c, *_ = np.linalg.lstsq(D @ Q, f, rcond=None)
        np.testing.assert_allclose(r["x"], Q @ c, rtol=1e-9, atol=1e-12)
        h = r["history"]
        assert np.all(np.diff(h) <= 1e-12 * h[0])


def test_gmres_full_terminates_and_restart():
    """Without restart GMRES terminates in <= n steps (exact arithmetic bound);
    with restarts it still converges on a diagonally dominant system; the
    AMG-preconditioned solve of a small conv-diff system matches the dense solve."""
    rng = np.random.default_rng(5)
    n = 12
    D = np.eye(n) * 3 + rng.standard_normal((n, n)) * 0.3
    A = csr_from_dense(D)
    f = rng.standard_normal(n)
    r = oracle.gmres(A, f, tol=1e-12, maxiter=100, m=100)
    assert r["iters"] <= n and r["status"] == oracle.OK
    np.testing.assert_allclose(r["x"], np.linalg.solve(D, f), rtol=1e-10)
    r = oracle.gmres(A, f, tol=1e-10, maxiter=200, m=3)
    assert r["status"] == oracle.OK and r["iters"] > 3
    np.testing.assert_allclose(r["x"], np.linalg.solve(D, f), rtol=1e-8)
    p, c, v, f = synth.convdiff3d(10)
    A = oracle.Csr(p, c, v)
    h = oracle.Hierarchy(A, coarse_enough=50, relax="damped_jacobi")
    r = oracle.gmres(A, f, hier=h, tol=1e-10, m=30)
    assert r["status"] == oracle.OK and r["rel_resid"] <= 1e-10
    np.testing.assert_allclose(r["x"], np.linalg.solve(A.to_dense(), f), rtol=1e-8)
    assert r["vcycles"] >= r["iters"] + 1


def test_cheb_step_composes_to_relax():
    """or_cheb_step (one step of the Chebyshev recurrence, the loop body of
    or_relax) chained K times equals one or_relax call bitwise, from a non-zero
    x, scaled and unscaled; step 0 on a diagonal A from x = 0 is alpha_0 f / a_ii
    (scaled: alpha_0 = 1/d with d = (1 + 1/30)/2 for D^-1 A = I)."""
    for scaled in (1, 0):
        p, c, v, f = synth.problem("varcoef", 12)
        h = oracle.Hierarchy(oracle.Csr(p, c, v), relax="chebyshev", cheb_scaled=scaled, coarse_enough=100)
        rng = np.random.default_rng(3)
        for l in range(h.nlevels - 1):
            n = h.info(l)["rows"]
            fl, x = rng.standard_normal(n), rng.standard_normal(n)
            xs, ps, a = x.copy(), np.zeros(n), 0.0
            for k in range(h.prm.cheb_degree):
                xs, ps, a = h.cheb_step(l, k, fl, xs, ps, a)
            assert np.array_equal(xs, h.relax(l, fl, x)), (scaled, l)
    # step 0 from x = 0: r = f exactly (A 0 = 0), so x_1 = p_1 = (1/d) (f / a_ii)
    # (scaled) with d = (lmax + lmin) / 2 of the level's Gershgorin bounds
    p, c, v, f = synth.problem("varcoef", 12)
    h = oracle.Hierarchy(oracle.Csr(p, c, v), relax="chebyshev", coarse_enough=100)
    A = h.matrix(0, "A")
    diag = np.array([A.val[A.ptr[i]:A.ptr[i + 1]][A.col[A.ptr[i]:A.ptr[i + 1]] == i][0] for i in range(A.nrows)])
    lmax, lmin, d, cc = h.smoother(0)
    assert d == (lmax + lmin) / 2 and lmin == lmax * (1.0 / 30.0)
    fl = np.random.default_rng(4).standard_normal(A.nrows)
    x1, p1, a0 = h.cheb_step(0, 0, fl, np.zeros(A.nrows), np.zeros(A.nrows), 0.0)
    assert a0 == 1.0 / d and np.array_equal(x1, p1)
    assert np.array_equal(x1, a0 * (fl / diag))
