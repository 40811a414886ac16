"""GPU setup phase (params setup_device = "gpu", the default on a device;
SURVEY §8f rank 3; gsetup.cu):
strength, aggregation (Phase 1 reproduced exactly by dependency-propagation
rounds), smoothed P, R = P^T, A P, R (A P) and the smoother data on the device,
the coarse inverse on the host.  The device steps perform the
host's operations in the host's order without FMA contraction, so the whole
hierarchy must be BITWISE equal to the host setup's (which tests/
test_setup_parity.py pins bitwise to the oracle), and so must the solve.
GPU only."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import paper_1811_05704_b200 as amgb  # noqa: E402
import synth  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float64)).cuda()


def problem(gen, n):
    return synth.poisson2d(n) if gen == "poisson2d" else synth.problem(gen, n)


def assert_same_hierarchy(hg, hh):
    assert hg.nlevels == hh.nlevels
    for l in range(hh.nlevels):
        ig, ih = hg.level_info(l), hh.level_info(l)
        for k in ("rows", "nnz_A", "nnz_P", "cols_P", "aggregates", "is_coarsest"):
            assert ig[k] == ih[k], (l, k, ig[k], ih[k])
        eg, eh = hg.export_level(l), hh.export_level(l)
        assert eg.keys() == eh.keys()
        for k in eh:
            a, b = eg[k], eh[k]
            for x, y in zip(a, b) if isinstance(a, tuple) else [(a, b)]:
                assert np.array_equal(x, y), (l, k)
                if x.dtype == np.float64:  # bitwise, incl. signed zeros
                    assert np.array_equal(x.view(np.int64), y.view(np.int64)), (l, k)


CASES = [
    ("poisson", 32, {}),
    ("poisson", 41, {}),
    ("poisson_perm", 24, {}),
    ("varcoef", 24, {"relax": "chebyshev"}),
    ("convdiff", 20, {"relax": "damped_jacobi", "solver": "bicgstab"}),
    ("poisson", 30, {"coarsening": "aggregation"}),
    ("poisson2d", 120, {}),
]


@pytest.mark.parametrize("gen,n,kw", CASES)
def test_gpu_setup_bitwise_equal_to_host(gen, n, kw):
    p, c, v, f = problem(gen, n)
    kw = dict(kw, coarse_enough=200)
    hh = amgb.setup(p, c, v, setup_device="host", **kw)
    hg = amgb.setup(p, c, v, **kw)
    assert_same_hierarchy(hg, hh)
    xh, ith, relh, _ = hh.solve(dev(f), tol=1e-8, maxiter=200)
    xg, itg, relg, _ = hg.solve(dev(f), tol=1e-8, maxiter=200)
    torch.cuda.synchronize()
    assert ith == itg and relh == relg
    assert np.array_equal(xh.cpu().numpy(), xg.cpu().numpy())


def test_gpu_setup_matches_oracle_hierarchy():
    p, c, v, f = synth.problem("poisson", 28)
    hg = amgb.setup(p, c, v, setup_device="gpu", coarse_enough=100)
    ho = oracle.Hierarchy(oracle.Csr(p, c, v), coarse_enough=100)
    assert hg.nlevels == ho.nlevels
    for l in range(ho.nlevels - 1):
        eg = hg.export_level(l)
        for which in "APR":
            M = ho.matrix(l, which)
            gp, gc, gv = eg[which]
            assert np.array_equal(gp, M.ptr) and np.array_equal(gc, M.col)
            assert np.array_equal(gv, M.val), (l, which)


def test_gpu_setup_long_rows_fall_back_to_host_routines():
    """A row longer than the device kernels' per-thread lists (256 entries in
    P's pass, 512 columns in a product row) is computed by the host routine:
    still bitwise the host hierarchy."""
    n2 = 80
    p, c, v, f = synth.poisson2d(n2)
    n = len(p) - 1
    rows = [list(zip(c[p[i]:p[i + 1]], v[p[i]:p[i + 1]])) for i in range(n)]
    hub = 0
    far = list(range(n // 2 - 1500, n // 2 + 1500))  # 3000 weak couplings of row 0
    for j in far:
        rows[hub].append((j, -1e-3))
        rows[j].append((hub, -1e-3))
    for j in far:  # keep diagonal dominance
        rows[j] = [(cc, vv + 1e-3 if cc == j else vv) for cc, vv in rows[j]]
    rows[hub] = [(cc, vv + 3.5 if cc == hub else vv) for cc, vv in rows[hub]]
    ptr = np.zeros(n + 1, np.int64)
    cols, vals = [], []
    for i, r in enumerate(rows):
        r.sort()
        cols += [cc for cc, _ in r]
        vals += [vv for _, vv in r]
        ptr[i + 1] = len(cols)
    col, val = np.array(cols, np.int32), np.array(vals)
    hh = amgb.setup(ptr, col, val, coarse_enough=50, eps_strong=0.001, setup_device="host")
    hg = amgb.setup(ptr, col, val, coarse_enough=50, eps_strong=0.001, setup_device="gpu")
    assert_same_hierarchy(hg, hh)


def test_gpu_setup_errors():
    p, c, v, f = synth.problem("poisson", 12)
    v = v.copy()
    bad_row = 17
    for k in range(p[bad_row], p[bad_row + 1]):
        if c[k] == bad_row:
            v[k] = -1.0
    with pytest.raises(amgb.AmgError) as e:
        amgb.setup(p, c, v, setup_device="gpu", coarse_enough=50)
    assert e.value.code == amgb.E_ZERO_DIAG and "row 17" in str(e.value)
    # a host-only handle builds on the host whatever setup_device says
    hh = amgb.setup(p, c, synth.problem("poisson", 12)[2], setup_device="gpu", device=-1, coarse_enough=50)
    assert hh.nlevels >= 2


@pytest.mark.parametrize("gen,n,kw", [("poisson", 48, {}), ("poisson", 41, {"precision": "mixed"}),
                                      ("poisson_perm", 40, {}), ("varcoef", 42, {"relax": "chebyshev"})])
def test_device_format_conversion_matches_host(gen, n, kw):
    """The SELL-32 / TMA (+ offset dictionary) arrays built on the device
    (convert.cuh, the default) equal the host converters' (AMGB_HOST_CONVERT=1):
    same stored sizes, dictionary slices and bitwise the same solve."""
    import os
    p, c, v, f = problem(gen, n)
    hd = amgb.setup(p, c, v, **kw)
    os.environ["AMGB_HOST_CONVERT"] = "1"
    try:
        hh = amgb.setup(p, c, v, **kw)
    finally:
        del os.environ["AMGB_HOST_CONVERT"]
    for l in range(hh.nlevels):
        a, b = hd.level_info(l), hh.level_info(l)
        assert (a["padded_nnz_A"], a["dict_slices_A"], a["dev_bytes"]) == \
            (b["padded_nnz_A"], b["dict_slices_A"], b["dev_bytes"]), l
    r = synth.random_vector(len(f))
    assert np.array_equal(hd.precond(dev(r)).cpu().numpy(), hh.precond(dev(r)).cpu().numpy())
    xd, itd, reld, _ = hd.solve(dev(f), tol=1e-8)
    xh, ith, relh, _ = hh.solve(dev(f), tol=1e-8)
    torch.cuda.synchronize()
    assert itd == ith and reld == relh
    assert np.array_equal(xd.cpu().numpy(), xh.cpu().numpy())


def random_mmatrix(n, deg, seed):
    """Unstructured non-symmetric M-matrix: deg random off-diagonal entries per
    row with independent magnitudes, so the strength pattern is NOT symmetric
    (exercises S versus S^T in the device aggregation)."""
    rng = np.random.default_rng(seed)
    rows = np.repeat(np.arange(n), deg)
    cols = (rows + rng.integers(1, n, size=n * deg)) % n
    vals = -rng.uniform(0.01, 1.0, size=n * deg) ** 3
    import scipy.sparse as sp
    M = sp.coo_matrix((vals, (rows, cols)), shape=(n, n)).tocsr()
    M.sum_duplicates()
    d = np.asarray(abs(M).sum(axis=1)).ravel() + 0.5
    M = (M + sp.diags(d)).tocsr()
    M.sort_indices()
    return M.indptr.astype(np.int64), M.indices.astype(np.int32), M.data.astype(np.float64), np.ones(n)


@pytest.mark.parametrize("case", ["poisson256", "varcoef96", "random"])
def test_gpu_aggregation_bitwise(case):
    """Aggregates, roots (via the hierarchy) and every level of the GPU setup --
    aggregation included -- bitwise equal to the host builder's, at the
    headline size 256^3, on log-random coefficients, and on an unstructured
    matrix with a non-symmetric strength pattern; the finest level's aggregates
    also equal the oracle's or_aggregate."""
    if case == "poisson256":
        p, c, v, f = synth.problem("poisson", 256)
    elif case == "varcoef96":
        p, c, v, f = synth.problem("varcoef", 96)
    else:
        p, c, v, f = random_mmatrix(60000, 6, 11)
    hg = amgb.setup(p, c, v)                        # device (default)
    hh = amgb.setup(p, c, v, device=-1)             # host builder, host-only handle
    assert hg.nlevels == hh.nlevels >= 2
    for l in range(hh.nlevels - 1):
        ag, ah = hg.export_level(l)["aggregates"], hh.export_level(l)["aggregates"]
        assert np.array_equal(ag, ah), (case, l, int(np.sum(ag != ah)))
    if case != "poisson256":
        assert_same_hierarchy(hg, hh)
    A = oracle.Csr(p, c, v)
    ido, cnt = oracle.aggregate(A, oracle.strength(A, 0.08))
    assert np.array_equal(hg.export_level(0)["aggregates"], ido)
