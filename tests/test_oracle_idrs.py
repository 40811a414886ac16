"""Pins of the oracle's IDR(s) (or_idrs; PAPER.md:212 lists IDR(s), the
bi-orthogonal variant of van Gijzen & Sonneveld 2011) against facts that do not
come from its own code:
* IDR(1) with the minimal-residual omega (kappa = 0) and shadow vector
  r0/|r0| is mathematically BiCGStab (Sonneveld & van Gijzen 2008, §5): after k
  full cycles (2k preconditioned products) x equals BiCGStab's x after k
  iterations, with and without the AMG preconditioner;
* small non-symmetric systems converge to numpy's dense solve within the
  finite-termination bound n + n/s of exact arithmetic (plus slack);
* the shadow space is orthonormal and reproduces an independent Python
  implementation of the stated counter-based generator + MGS.
CPU only."""
import numpy as np
import pytest

import oracle
import synth


def splitmix64(z):
    m = (1 << 64) - 1
    z = (z + 0x9E3779B97F4A7C15) & m
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    return z ^ (z >> 31)


def test_shadow_space_generator_and_orthonormality():
    n, s = 37, 4
    P = oracle.idrs_shadow(n, s)
    raw = np.array([[2.0 * ((splitmix64(0x181105704 + j * n + i) >> 11) * 2.0 ** -53) - 1.0 for i in range(n)]
                    for j in range(s)])
    Q = raw.copy()
    for j in range(s):  # modified Gram-Schmidt, in order
        for q in range(j):
            Q[j] = Q[j] - np.dot(Q[q], Q[j]) * Q[q]
        Q[j] = Q[j] / np.linalg.norm(Q[j])
    assert np.max(np.abs(P - Q)) <= 1e-14
    assert np.max(np.abs(P @ P.T - np.eye(s))) <= 1e-14
    assert np.array_equal(P, oracle.idrs_shadow(n, s))


@pytest.mark.parametrize("precond", [False, True])
def test_idr1_is_bicgstab(precond):
    p, c, v, f = synth.problem("convdiff", 10)
    A = oracle.Csr(p, c, v)
    H = oracle.Hierarchy(A, coarse_enough=100) if precond else None
    P = (f / np.linalg.norm(f)).reshape(1, -1)  # x0 = 0: r0 = f
    for k in (1, 2, 3, 5):
        b = oracle.bicgstab(A, f, tol=0.0, maxiter=k, hier=H)
        i = oracle.idrs(A, f, tol=0.0, maxiter=2 * k, s=1, kappa=0.0, P=P, hier=H)
        assert b["iters"] == k and i["iters"] == 2 * k
        assert np.linalg.norm(b["x"] - i["x"]) <= 1e-10 * np.linalg.norm(b["x"]), k


@pytest.mark.parametrize("s", [1, 2, 4, 8])
def test_idrs_small_nonsymmetric_exact(s):
    rng = np.random.default_rng(5704 + s)
    n = 40
    D = rng.standard_normal((n, n)) * (rng.random((n, n)) < 0.15)
    D += np.diag(np.abs(D).sum(1) + 1.0)  # non-symmetric, diagonally dominant
    ptr = np.zeros(n + 1, np.int64)
    cols, vals = [], []
    for i in range(n):
        nz = np.nonzero(D[i])[0]
        cols += list(nz)
        vals += list(D[i, nz])
        ptr[i + 1] = len(cols)
    A = oracle.Csr(ptr, np.array(cols, np.int32), np.array(vals))
    f = rng.standard_normal(n)
    o = oracle.idrs(A, f, tol=1e-12, maxiter=500, s=s)
    assert o["status"] == 0
    assert o["iters"] <= n + n / s + 10, o["iters"]
    xs = np.linalg.solve(D, f)
    assert np.linalg.norm(o["x"] - xs) <= 1e-9 * np.linalg.norm(xs)


def test_idrs_preconditioned_convergence_and_history():
    p, c, v, f = synth.problem("convdiff", 12)
    A = oracle.Csr(p, c, v)
    H = oracle.Hierarchy(A, coarse_enough=100)
    o = oracle.idrs(A, f, tol=1e-8, maxiter=200, s=4, hier=H, history=True)
    assert o["status"] == 0 and o["rel_resid"] <= 1.01e-8
    assert o["vcycles"] == o["iters"]
    h = o["history"]
    assert h[0] == pytest.approx(np.linalg.norm(f)) and h[-1] <= 1e-8 * h[0]
    # the same problem unpreconditioned needs many more products
    u = oracle.idrs(A, f, tol=1e-8, maxiter=2000, s=4)
    assert u["status"] == 0 and u["iters"] > 2 * o["iters"]
    # zero right-hand side
    z = oracle.idrs(A, np.zeros_like(f), s=4, hier=H)
    assert z["iters"] == 0 and np.all(z["x"] == 0)
