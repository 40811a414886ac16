"""T3-T5: the CUDA path (libamgb.so through the C ABI) against the oracle on
the same seeded inputs.  GPU only (-m gpu).

Tolerances:
* kernel level: |y - y_oracle|_i <= 8 (len_i + 2) u (|A||x| + |f|)_i, the
  standard a-priori bound for a row sum evaluated in a different order / with
  FMA (u = 2^-53);
* V-cycle: |z - z_oracle| <= 1e-12 |z_oracle|;
* solve: iterations within +-1 of the oracle; at equal iteration count
  |x - x_oracle| / |x_oracle| <= 1e-8 (BASELINE.json north_star; §8c).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import paper_1811_05704_b200 as amgb  # noqa: E402
import synth  # noqa: E402

U = 2.0 ** -53


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float64)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def abs_csr(M):
    return oracle.Csr(M.ptr, M.col, np.abs(M.val), M.ncols)


def row_bound(M, x, f=None):
    lens = np.diff(M.ptr).astype(float)
    b = oracle.spmv(abs_csr(M), np.abs(x))
    if f is not None:
        b = b + np.abs(f)
    return 8 * (lens + 2) * U * b + 1e-300


def okw(kw):
    o = dict(kw)
    if "coarsening" in o:
        o["smoothed"] = 1 - o.pop("coarsening")
    return o


LEVEL_CASES = [
    ("poisson", 33, {"coarse_enough": 200}),           # ragged: 35937 rows, not a multiple of 32
    ("poisson_perm", 20, {"coarse_enough": 100}),
    ("varcoef", 22, {"relax": "chebyshev", "coarse_enough": 100}),
    ("convdiff", 18, {"relax": "damped_jacobi", "coarse_enough": 100}),
    ("poisson", 17, {"coarsening": 1, "coarse_enough": 30}),
]


@pytest.mark.parametrize("gen,n,kw", LEVEL_CASES)
def test_level_kernels_match_oracle(gen, n, kw):
    p, c, v, f = synth.problem(gen, n)
    h = amgb.setup(p, c, v, **kw)
    o = oracle.Hierarchy(oracle.Csr(p, c, v), **okw(kw))
    assert h.nlevels == o.nlevels >= 2
    rng = np.random.default_rng(synth.SEED_VEC)
    for l in range(h.nlevels - 1):
        A, P, R = o.matrix(l, "A"), o.matrix(l, "P"), o.matrix(l, "R")
        x = rng.standard_normal(A.nrows)
        fl = rng.standard_normal(A.nrows)
        xc = rng.standard_normal(P.ncols)
        for op, M, xin, fin in ((amgb.OP_SPMV_A, A, x, None), (amgb.OP_SPMV_P, P, xc, None),
                                (amgb.OP_SPMV_R, R, x, None), (amgb.OP_RESIDUAL, A, x, fl)):
            y = host(h.level_op(l, op, x=dev(xin), f=dev(fin) if fin is not None else None,
                                ny=M.nrows))
            ref = oracle.spmv(M, xin)
            if fin is not None:
                ref = fin - ref
            err = np.abs(y - ref)
            assert np.all(err <= row_bound(M, xin, fin)), (l, op, err.max())
        # one smoother call from a non-zero x
        y = host(h.level_op(l, amgb.OP_RELAX, x=dev(x), f=dev(fl), ny=A.nrows))
        ref = o.relax(l, fl, x)
        assert np.linalg.norm(y - ref) <= 1e-12 * np.linalg.norm(ref), l
    # coarsest solve
    L = h.nlevels - 1
    fl = rng.standard_normal(o.info(L)["rows"])
    y = host(h.level_op(L, amgb.OP_COARSE, f=dev(fl), ny=len(fl)))
    ref = o.vcycle(L, fl, np.zeros_like(fl))
    assert np.linalg.norm(y - ref) <= 1e-10 * np.linalg.norm(ref)


@pytest.mark.parametrize("gen,n,kw", LEVEL_CASES)
def test_vcycle_matches_oracle(gen, n, kw):
    p, c, v, f = synth.problem(gen, n)
    h = amgb.setup(p, c, v, **kw)
    o = oracle.Hierarchy(oracle.Csr(p, c, v), **okw(kw))
    r = synth.random_vector(len(f))
    z = host(h.precond(dev(r)))
    ref = o.precond(r)
    assert np.linalg.norm(z - ref) <= 1e-12 * np.linalg.norm(ref)
    # linearity and zero input
    z2 = host(h.precond(dev(2.5 * r)))
    assert np.linalg.norm(z2 - 2.5 * z) <= 1e-12 * np.linalg.norm(z2)
    assert np.all(host(h.precond(dev(np.zeros_like(r)))) == 0)


SOLVE_CASES = [
    # configs[0]: 32^3 Poisson, SA + SPAI-0, CG
    ("poisson", 32, {}, 100),
    ("poisson_perm", 30, {}, 100),
    ("varcoef", 32, {"relax": "chebyshev"}, 200),
    ("convdiff", 24, {"relax": "damped_jacobi", "solver": "bicgstab"}, 200),
    ("poisson", 25, {"npre": 2, "npost": 2, "coarse_enough": 500}, 100),
    ("poisson", 20, {"coarsening": 1, "coarse_enough": 300}, 100),
]


def oracle_solve(p, c, v, f, kw, tol, maxiter, x0=None):
    A = oracle.Csr(p, c, v)
    k = okw(kw)
    solver = k.pop("solver", "cg")
    k.pop("use_graph", None)
    hier = oracle.Hierarchy(A, **k)
    fn = oracle.bicgstab if solver == "bicgstab" else oracle.cg
    return fn(A, f, x0=x0, tol=tol, maxiter=maxiter, hier=hier)


@pytest.mark.parametrize("graph", [1, 0])
@pytest.mark.parametrize("gen,n,kw,maxiter", SOLVE_CASES)
def test_solve_matches_oracle(gen, n, kw, maxiter, graph):
    p, c, v, f = synth.problem(gen, n)
    h = amgb.setup(p, c, v, use_graph=graph, **kw)
    o = oracle_solve(p, c, v, f, kw, 1e-8, maxiter)
    x, iters, rel, st = h.solve(dev(f), tol=1e-8, maxiter=maxiter)
    assert st == amgb.OK and o["status"] == oracle.OK
    assert abs(iters - o["iters"]) <= 1, (iters, o["iters"])
    assert rel <= 1.01e-8
    true = np.linalg.norm(f - oracle.spmv(oracle.Csr(p, c, v), host(x))) / np.linalg.norm(f)
    assert abs(true - rel) <= 1e-12
    if iters != o["iters"]:
        x, iters, rel, st = h.solve(dev(f), tol=0.0, maxiter=o["iters"])
    xh = host(x)
    assert np.linalg.norm(xh - o["x"]) <= 1e-8 * np.linalg.norm(o["x"])
    s = h.stats()
    assert s["iters"] == iters and s["kernel_launches"] > 0


def test_solve_initial_guess_and_maxiter():
    p, c, v, f = synth.poisson3d(20)
    h = amgb.setup(p, c, v, coarse_enough=200)
    x0 = synth.random_vector(len(f))
    o = oracle_solve(p, c, v, f, {"coarse_enough": 200}, 1e-9, 3, x0=x0)
    x, iters, rel, st = h.solve(dev(f), x=dev(x0), tol=1e-9, maxiter=3)
    assert st == amgb.NOT_CONVERGED and o["status"] == oracle.NOT_CONVERGED and iters == 3
    assert np.linalg.norm(host(x) - o["x"]) <= 1e-10 * np.linalg.norm(o["x"])
    x, iters, rel, st = h.solve(dev(f), tol=1e-8, maxiter=0)
    assert iters == 0 and st == amgb.NOT_CONVERGED


def test_zero_rhs_and_single_level():
    p, c, v, f = synth.poisson3d(10)
    h = amgb.setup(p, c, v)  # 1000 rows <= coarse_enough: one level, direct solve
    assert h.nlevels == 1
    x, iters, rel, st = h.solve(dev(np.zeros_like(f)), x=dev(np.ones_like(f)))
    assert iters == 0 and rel == 0.0 and st == amgb.OK and np.all(host(x) == 0)
    x, iters, rel, st = h.solve(dev(f), tol=1e-10)
    assert iters == 1 and rel <= 1e-10
    ref = np.linalg.solve(oracle.Csr(p, c, v).to_dense(), f)
    assert np.linalg.norm(host(x) - ref) <= 1e-10 * np.linalg.norm(ref)


def test_cg_breakdown_is_flagged():
    p, c, v, f = synth.poisson3d(6)
    h = amgb.setup(p, c, -v, coarse_enough=10000)  # negative definite, 1 level
    x, iters, rel, st = h.solve(dev(f))
    o = oracle.cg(oracle.Csr(p, c, -v), f, hier=oracle.Hierarchy(oracle.Csr(p, c, -v),
                                                                  coarse_enough=10000))
    assert st == amgb.BREAKDOWN and o["status"] == oracle.BREAKDOWN


def test_solve_host_end_to_end():
    p, c, v, f = synth.poisson3d(30)
    h = amgb.setup(p, c, v)
    o = oracle_solve(p, c, v, f, {}, 1e-8, 100)
    x, iters, rel, st = h.solve_host(f, tol=1e-8)
    assert st == amgb.OK and abs(iters - o["iters"]) <= 1
    if iters == o["iters"]:
        assert np.linalg.norm(x - o["x"]) <= 1e-8 * np.linalg.norm(o["x"])
    # explicit initial guess: restarting from the solution needs 0 iterations
    x2, iters2, rel2, st2 = h.solve_host(f, x0=x, tol=1e-8)
    assert iters2 == 0 and np.array_equal(x2, x)


def test_configs1_150_permuted_full_size():
    """BASELINE.json configs[1]: 150^3 randomly permuted Poisson, CG + SA-AMG,
    at full size against the oracle (iterations +-1, x within 1e-8)."""
    p, c, v, f = synth.problem("poisson_perm", 150)
    h = amgb.setup(p, c, v)
    x, iters, rel, st = h.solve(dev(f), tol=1e-8, maxiter=100)
    o = oracle_solve(p, c, v, f, {}, 1e-8, 100)
    assert st == amgb.OK and abs(iters - o["iters"]) <= 1, (iters, o["iters"])
    if iters != o["iters"]:
        x, iters, rel, st = h.solve(dev(f), tol=0.0, maxiter=o["iters"])
    assert np.linalg.norm(host(x) - o["x"]) <= 1e-8 * np.linalg.norm(o["x"])


@pytest.mark.parametrize("n", [1, 2, 5, 31, 33])
def test_tiny_systems(n):
    """Degenerate sizes: 1x1 .. a few rows (single level: the dense coarse solve
    is the whole preconditioner, so CG converges in one iteration)."""
    p, c, v, f = synth.poisson3d(n, 1, 1)
    h = amgb.setup(p, c, v)
    x, iters, rel, st = h.solve(dev(f), tol=1e-12)
    ref = np.linalg.solve(oracle.Csr(p, c, v).to_dense(), f)
    assert st == amgb.OK and iters == 1
    assert np.linalg.norm(host(x) - ref) <= 1e-12 * np.linalg.norm(ref)


def test_maxiter_one_and_two_levels_ragged():
    """maxiter = 1 and 2 (odd/even iterations of the two-iteration graph body),
    on a ragged two-level hierarchy, against the oracle."""
    p, c, v, f = synth.problem("poisson_perm", 13)  # 2197 rows
    for maxiter in (1, 2, 3):
        h = amgb.setup(p, c, v, coarse_enough=200)
        o = oracle_solve(p, c, v, f, {"coarse_enough": 200}, 0.0, maxiter)
        x, iters, rel, st = h.solve(dev(f), tol=0.0, maxiter=maxiter)
        assert iters == maxiter == o["iters"] and st == amgb.NOT_CONVERGED
        assert np.linalg.norm(host(x) - o["x"]) <= 1e-12 * np.linalg.norm(o["x"])
        s = h.stats()
        assert s["iters"] == maxiter and s["vcycles"] == maxiter and s["alg_bytes"] > 0


def test_device_loop_and_host_loop_agree():
    """The conditional-WHILE device loop and the host loop give identical results."""
    import os
    p, c, v, f = synth.problem("varcoef", 20)
    h = amgb.setup(p, c, v, relax="chebyshev", coarse_enough=100)
    x1, it1, rel1, _ = h.solve(dev(f), tol=1e-9)
    h.set_profile(1)  # profile mode uses the host loop
    x2, it2, rel2, _ = h.solve(dev(f), tol=1e-9)
    h.set_profile(0)
    assert it1 == it2 and np.array_equal(host(x1), host(x2))


def test_misaligned_vector_views():
    """f and x as 8-B-offset views (buf[1:n+1]): the paired 16-B vector kernels
    take their scalar loop (stats flag bit 2), and the solve still matches the
    oracle (iterations +-1, x within 1e-8 at equal count) and the host rejects
    wrong lengths instead of reading past a buffer."""
    p, c, v, f = synth.problem("poisson", 41)  # TMA store, odd n (68,921)
    n = len(f)
    h = amgb.setup(p, c, v)
    fb = torch.zeros(n + 2, dtype=torch.float64, device="cuda")
    xb = torch.zeros(n + 2, dtype=torch.float64, device="cuda")
    fb[1:n + 1] = dev(f)
    fv, xv = fb[1:n + 1], xb[1:n + 1]
    assert fv.data_ptr() % 16 == 8 and xv.data_ptr() % 16 == 8
    x, iters, rel, st = h.solve(fv, xv, tol=1e-8, maxiter=100)
    assert h.stats()["flags"] & 4, "scalar vector-kernel loop expected"
    o = oracle_solve(p, c, v, f, {}, 1e-8, 100)
    assert st == amgb.OK and abs(iters - o["iters"]) <= 1 and rel <= 1.01e-8
    if iters != o["iters"]:
        xv.zero_()
        x, iters, rel, st = h.solve(fv, xv, tol=0.0, maxiter=o["iters"])
    assert np.linalg.norm(host(xv) - o["x"]) <= 1e-8 * np.linalg.norm(o["x"])
    assert host(xb)[0] == 0.0 and host(xb)[n + 1] == 0.0  # nothing written outside the view
    # aligned run: bit 2 clear; the same iteration count
    x2, it2, _, _ = h.solve(dev(f), tol=1e-8, maxiter=100)
    assert not (h.stats()["flags"] & 4) and abs(it2 - iters) <= 1
    # wrong lengths are rejected on the host
    with pytest.raises(ValueError):
        h.solve(dev(f[:-1]))
    with pytest.raises(ValueError):
        h.solve_host(f[:-1])
    with pytest.raises(ValueError):
        h.solve_host_stream([f], xs=[np.empty(n - 1)])
