"""amg_solve_host_stream: a sequence of independent solves with host buffers,
transfers overlapped with the solves through double-buffered staging vectors.
Every system's result must be BITWISE that of amg_solve_host on the same
system (same kernels, same device vectors' arithmetic), for pinned and pageable
buffers, repeated and distinct right-hand sides.  GPU only."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import paper_1811_05704_b200 as amgb  # noqa: E402
import synth  # noqa: E402


def pinned(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float64)).pin_memory().numpy()


@pytest.mark.parametrize("gen,n,kw,pin", [("poisson", 34, {}, True), ("poisson", 34, {}, False),
                                          ("poisson_perm", 28, {}, True),
                                          ("convdiff", 22, {"relax": "damped_jacobi", "solver": "bicgstab"}, True)])
def test_host_stream_matches_host_solves(gen, n, kw, pin):
    p, c, v, f = synth.problem(gen, n)
    h = amgb.setup(p, c, v, coarse_enough=200, **kw)
    fs = [f, synth.random_vector(len(f)), f * 0.5, np.zeros_like(f), synth.random_vector(len(f), seed=7)]
    if pin:
        fs = [pinned(a) for a in fs]
    xs_out = [pinned(np.zeros_like(f)) if pin else np.zeros_like(f) for _ in fs]
    xs, its, rels, vcs, st = h.solve_host_stream(fs, xs_out, tol=1e-8, maxiter=200)
    assert st == amgb.OK
    A = oracle.Csr(p, c, v)
    for j, fj in enumerate(fs):
        xr, itr, relr, str_ = h.solve_host(fj, None, tol=1e-8, maxiter=200)
        assert str_ == amgb.OK and its[j] == itr and rels[j] == relr, j
        assert np.array_equal(xs[j], xr), j
        if np.any(fj):
            assert vcs[j] >= its[j] > 0
            res = fj - oracle.spmv(A, xs[j])
            assert np.linalg.norm(res) <= 1.01e-8 * np.linalg.norm(fj)
        else:
            assert its[j] == 0 and not np.any(xs[j])


def test_host_stream_repeated_buffers_and_edge_cases():
    p, c, v, f = synth.problem("poisson", 30)
    h = amgb.setup(p, c, v, coarse_enough=200)
    fp = pinned(f)
    xp = pinned(np.zeros_like(f))
    xs, its, rels, vcs, st = h.solve_host_stream([fp] * 4, [xp] * 4, tol=1e-8)  # one buffer each way
    xr, itr, relr, _ = h.solve_host(f, None, tol=1e-8)
    assert st == amgb.OK and its == [itr] * 4 and np.array_equal(xp, xr)
    assert h.solve_host_stream([], [], tol=1e-8)[4] == amgb.OK  # k = 0: nothing to do
    xs, its, rels, vcs, st = h.solve_host_stream([f], tol=1e-12, maxiter=2)
    assert st == amgb.NOT_CONVERGED and its == [2]
