"""SELL-C-sigma store: inside aligned 256-row windows the rows
of a SELL / TMA matrix are stored sorted by length, so slices pad less; the
kernels map a stored slot back to its row for the row-local operands.  It is a
storage choice only: every row sum is formed from the same entries in the same
order, so every result must be BITWISE equal to the unsorted store (the
default; AMGB_SIGMA=1 turns sorting on), and within the usual tolerance of the
oracle.  GPU only."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import paper_1811_05704_b200 as amgb  # noqa: E402
import synth  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float64)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def setup_pair(p, c, v, fmt=None, **kw):
    old = os.environ.get("AMGB_FORMAT")
    if fmt:
        os.environ["AMGB_FORMAT"] = fmt
    try:
        h_plain = amgb.setup(p, c, v, **kw)
        os.environ["AMGB_SIGMA"] = "1"
        try:
            h_sig = amgb.setup(p, c, v, **kw)
        finally:
            del os.environ["AMGB_SIGMA"]
    finally:
        if fmt:
            if old is None:
                del os.environ["AMGB_FORMAT"]
            else:
                os.environ["AMGB_FORMAT"] = old
    return h_sig, h_plain


def level_ops_equal(ha, hb):
    for l in range(ha.nlevels - 1):
        n = ha.level_info(l)["rows"]
        nc = ha.level_info(l + 1)["rows"]
        x, fl, xc = synth.random_vector(n), synth.random_vector(n)[::-1].copy(), synth.random_vector(nc)
        for op, xin, fin, ny in ((amgb.OP_SPMV_A, x, None, n), (amgb.OP_RESIDUAL, x, fl, n),
                                 (amgb.OP_RELAX, x, fl, n), (amgb.OP_SPMV_P, xc, None, n),
                                 (amgb.OP_SPMV_R, x, None, nc)):
            ya = host(ha.level_op(l, op, x=dev(xin), f=dev(fin) if fin is not None else None, ny=ny))
            yb = host(hb.level_op(l, op, x=dev(xin), f=dev(fin) if fin is not None else None, ny=ny))
            assert np.array_equal(ya, yb), (l, op)


# 48^3: P0 has rows of 1..6 entries -> sorted; 41^3: the last 256-row window
# is ragged (68921 rows).  fmt forces SELL-32 / TMA on every level, so the
# sorted layout runs in both kernels on A, P and R (a forced TMA format falls
# back to SELL-32 for rows too wide for its shared-memory stages; the default
# policy stores P0 padding-free in the TMA-CSR format, which needs no sorting).
@pytest.mark.parametrize("n,fmt", [(48, "tma"), (41, "tma"), (41, "sell"), (30, "sell"), (30, "tma")])
def test_sigma_bitwise_equal(n, fmt):
    p, c, v, f = synth.problem("poisson", n)
    hs, hp = setup_pair(p, c, v, fmt=fmt, coarse_enough=200)
    masks = [hs.level_info(l)["sigma_mask"] for l in range(hs.nlevels - 1)]
    assert masks[0] & 2, masks  # P0 sorted
    assert all(hp.level_info(l)["sigma_mask"] == 0 for l in range(hp.nlevels))
    i0s, i0p = hs.level_info(0), hp.level_info(0)
    assert i0s["padded_nnz_P"] < i0p["padded_nnz_P"]
    assert i0s["padded_nnz_P"] >= i0s["nnz_P"]
    level_ops_equal(hs, hp)
    r = synth.random_vector(len(f))
    assert np.array_equal(host(hs.precond(dev(r))), host(hp.precond(dev(r))))
    xs, its, rels, sts = hs.solve(dev(f), tol=1e-8)
    xp, itp, relp, stp = hp.solve(dev(f), tol=1e-8)
    assert sts == stp == amgb.OK and its == itp and rels == relp
    assert np.array_equal(host(xs), host(xp))
    A = oracle.Csr(p, c, v)
    o = oracle.cg(A, f, tol=1e-8, maxiter=100, hier=oracle.Hierarchy(A, coarse_enough=200))
    assert abs(its - o["iters"]) <= 1
    if its == o["iters"]:
        assert np.linalg.norm(host(xs) - o["x"]) <= 1e-8 * np.linalg.norm(o["x"])


@pytest.mark.parametrize("kw", [{"relax": "chebyshev", "gen": "varcoef"},
                                {"relax": "damped_jacobi", "solver": "bicgstab", "gen": "convdiff"},
                                {"gen": "poisson_perm", "reorder": 1},
                                {"gen": "poisson", "precision": "mixed"}])
def test_sigma_bitwise_equal_variants(kw):
    kw = dict(kw)
    gen = kw.pop("gen")
    p, c, v, f = synth.problem(gen, 42)
    hs, hp = setup_pair(p, c, v, fmt="sell", coarse_enough=200, **kw)
    assert any(hs.level_info(l)["sigma_mask"] for l in range(hs.nlevels - 1))
    xs, its, _, sts = hs.solve(dev(f), tol=1e-8, maxiter=200)
    xp, itp, _, stp = hp.solve(dev(f), tol=1e-8, maxiter=200)
    assert sts == stp == amgb.OK and its == itp
    assert np.array_equal(host(xs), host(xp))


@pytest.mark.parametrize("k", [2, 4, 8])
def test_sigma_batched(k):
    p, c, v, f = synth.problem("poisson", 44)
    hs, hp = setup_pair(p, c, v, fmt="tma", coarse_enough=200)  # P0 sorted in the TMA format
    assert hs.level_info(0)["sigma_mask"] & 2
    F = torch.stack([dev(f * (1.0 + 0.25 * j)) if j % 2 == 0 else dev(synth.random_vector(len(f)))
                     for j in range(k)])
    Xs, its, _, sts = hs.solve_batched(F, tol=1e-8)
    Xp, itp, _, stp = hp.solve_batched(F, tol=1e-8)
    assert sts == stp == amgb.OK and list(its) == list(itp)
    assert np.array_equal(host(Xs), host(Xp))
